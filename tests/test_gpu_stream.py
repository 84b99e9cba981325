"""GPU parity of the read-stationary streaming kernels (k_stream FP32 + FP64 retry units)
on inputs built to hit their edge cases: haplotypes of length 1..2 (event windows that
overlap), one-haplotype batches (an empty lane), batches with more haplotypes than one
unit holds (unit splitting), lanes of very different total length, every tiling width,
degenerate reads inside streams, and units where only some lanes underflow (partial FP64
retry units).  Checked against the C oracle (pinned bit-exactly to the reference by
tests/test_oracle_golden.py) with the north_star bars of test_gpu_parity.py."""
import numpy as np
import pytest

from oracle import oracle
from paper_2411_11547_b200 import _native, datagen, default_configs
from paper_2411_11547_b200.errors import DataError
from paper_2411_11547_b200.model import FlatBatches
from paper_2411_11547_b200.pipeline import config_tuples

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
RETRY_REL_TOL = 1e-9
F32 = config_tuples(default_configs("f32"))
KIND = _native.ST_KIND_MASK
SEED_CHUNK = 20240811 + 17


def _flat(rng, batches):
    """batches: list of (read_lengths, hap_lengths, mode); mode 'derived' makes reads
    substrings of the first haplotype (high likelihood), 'random' independent bases
    (FP32 underflow for long pairs), 'degenerate' ins+del qualities that sum past 1."""
    rb, bq, iq, dq, gq, hb = [], [], [], [], [], []
    rlen, hlen, bro, bho = [], [], [0], [0]
    for reads, haps, mode in batches:
        base = rng.integers(0, 4, size=max(haps) + max(reads), dtype=np.int8)
        for n in haps:
            h = base[:n].copy()
            hits = rng.random(n) < 0.01
            h[hits] = (h[hits] + 1) % 4
            hb.append(h)
            hlen.append(n)
        for m in reads:
            if mode == "random":
                r = rng.integers(0, 4, size=m, dtype=np.int8)
            else:
                start = int(rng.integers(0, max(1, min(haps) - m + 1))) if m <= min(haps) else 0
                r = base[start:start + m].copy()
            rb.append(r)
            bq.append(rng.integers(10, 41, size=m).astype(np.uint8))
            if mode == "degenerate":
                iq.append(np.full(m, 2, np.uint8)); dq.append(np.full(m, 2, np.uint8))
            else:
                iq.append(rng.integers(30, 46, size=m).astype(np.uint8))
                dq.append(rng.integers(30, 46, size=m).astype(np.uint8))
            gq.append(np.full(m, 10, np.uint8))
            rlen.append(m)
        bro.append(bro[-1] + len(reads))
        bho.append(bho[-1] + len(haps))
    cat = np.concatenate
    return FlatBatches(read_bases=cat(rb), bq=cat(bq), iq=cat(iq), dq=cat(dq), gq=cat(gq),
                       read_off=np.concatenate([[0], np.cumsum(rlen)]).astype(np.int64),
                       hap_bases=cat(hb), hap_off=np.concatenate([[0], np.cumsum(hlen)]).astype(np.int64),
                       batch_read_off=np.asarray(bro, np.int64), batch_hap_off=np.asarray(bho, np.int64))


def _check(engine, flat):
    ofl = oracle.Flat(**flat.as_dict())
    ref32, k32 = oracle.score(ofl, "f32")
    # plain FP32 semantics: identical flag set, values within 1e-4
    s, st, _ = engine.score(flat, F32, 0)
    assert np.array_equal(st & KIND, k32)
    ok = k32 == 0
    assert np.all(np.isfinite(s[ok])) and np.all(np.isnan(s[~ok]))
    if ok.any():
        assert (np.abs(s[ok] - ref32[ok]) / np.abs(ref32[ok])).max() <= REL_TOL
    # FP64 retry: exactly the reference's FP32 flag set retried, values within 1e-9
    s, st, _ = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    flagged = k32 == 1
    assert np.array_equal((st & _native.ST_RETRIED_F64) != 0, flagged)
    rest = ~flagged
    assert np.array_equal(st[rest] & KIND, k32[rest])
    okr = rest & (k32 == 0)
    if okr.any():
        assert (np.abs(s[okr] - ref32[okr]) / np.abs(ref32[okr])).max() <= REL_TOL
    if flagged.any():
        pr, ph = flat.pair_index()
        idx = np.flatnonzero(flagged)
        acc64, st64 = oracle.score_raw(ofl, "f64", 0, pairs=(pr[idx], ph[idx]))
        ref64 = oracle.finish(acc64, st64, 0)
        assert np.array_equal(st[idx] & KIND, st64)
        fin = st64 == 0
        if fin.any():
            assert (np.abs(s[idx][fin] - ref64[fin]) / np.abs(ref64[fin])).max() <= RETRY_REL_TOL
    return k32


def test_tiny_haplotypes_overlapping_windows(engine, rng):
    # haplotypes of 1..3 rows: FIRST/LAST events of consecutive pairs inside one window
    flat = _flat(rng, [([30, 31, 7], [1, 2, 3, 1, 2, 40, 1], "derived"),
                       ([100, 1, 2], [2, 1, 1, 1, 5], "derived"),
                       ([63, 64], [1] * 20, "random")])
    _check(engine, flat)


def test_single_haplotype_batches_empty_lane(engine, rng):
    flat = _flat(rng, [([m], [n], "derived") for m, n in [(5, 9), (50, 300), (127, 128), (250, 600),
                                                         (255, 40), (400, 450), (511, 700)]])
    _check(engine, flat)


def test_many_haplotypes_split_units_and_unbalanced_lanes(engine, rng):
    # 40 haplotypes per read (> 2 x 15 per unit), lengths spread 1..600
    haps = [int(x) for x in rng.integers(1, 601, size=40)]
    haps[3] = 600
    haps[7] = 1
    flat = _flat(rng, [([60, 180, 250], haps, "derived"), ([120], [600, 5, 5, 5, 5], "derived")])
    _check(engine, flat)


def test_every_tiling_width(engine, rng):
    # read lengths across all single-stripe widths W = 16 .. 512 and their edges (143, 175,
    # 207, 239: the odd-K tilings (16, 9 / 11 / 13 / 15) with a padded emission chunk)
    ms = [1, 14, 15, 16, 31, 32, 47, 48, 63, 64, 95, 96, 127, 128, 143, 159, 175, 191, 192, 207, 223, 239,
          255, 256, 383, 384, 511]
    flat = _flat(rng, [([m, max(1, m // 2)], [int(x) for x in rng.integers(50, 400, size=5)], "derived")
                       for m in ms])
    _check(engine, flat)


def test_long_reads_striped_team_and_sequential_modes(engine, rng):
    # reads past every single-stripe width (FP32 511, FP64 255, exact 511): a few units run
    # in team mode (a CTA's warps on one unit's stripes, column progress flags), many in
    # sequential mode; 'random' long pairs underflow (striped FP64 retries), 'derived'
    # ones land in the guard band (striped exact reruns, second-stage FP64)
    few = _flat(rng, [([1023, 700, 513], [1024, 1500, 37, 2000], "random"),
                      ([600, 900], [800, 1200, 5], "derived"),
                      ([1000], [2047, 1], "degenerate")])
    k32 = _check(engine, few)
    assert (k32 == 1).any() and (k32 == 0).any()
    many = _flat(rng, [([int(m) for m in rng.integers(512, 1024, size=6)],
                        [int(n) for n in rng.integers(100, 1600, size=5)], mode)
                       for mode in ["random", "derived"] * 24])
    _check(engine, many)


def test_partial_underflow_units_and_degenerate_reads(engine, rng):
    # 'random' reads underflow against long haplotypes but not short ones: FP64 retry
    # units hold a subset of each lane; degenerate reads share batches with normal ones
    flat = _flat(rng, [([200, 220, 90], [20, 30, 400, 500, 600, 10, 550], "random"),
                       ([150, 150], [300, 310, 320, 330], "degenerate"),
                       ([240, 16, 250], [250, 260, 270, 280, 290, 300], "derived"),
                       ([180], [40, 60, 80, 590, 595, 600, 50, 70, 90, 100], "random")])
    k32 = _check(engine, flat)
    assert (k32 == 1).any() and (k32 == 0).any() and (k32 == 3).any()


def test_chunked_score_matches_resident_path(engine):
    """phmm_score pipelines calls over chunk contexts (automatic for >= 2^20 pairs,
    phmm_set_pipeline forces it); results must equal the one-pass prepare/execute/fetch
    path bit for bit (FP32 + guard band + FP64 retry)."""
    from paper_2411_11547_b200 import datagen
    piped = _native.Context(0)
    piped.set_pipeline(4)
    derived = datagen.workload("c2", num_batches=520)          # 33,280 pairs -> 4 chunks
    indep = datagen.generate_synthetic_flat(num_batches=520, reads_per_batch=16, haps_per_batch=4,
                                            read_len_spec=120, hap_len_spec=200, seed=SEED_CHUNK,
                                            mode="independent")     # every pair underflows FP32
    for flat, flags in ((derived, 0), (derived, _native.FLAG_EXACT), (indep, 0),
                        (indep, _native.FLAG_RETRY_F64)):
        a, sa, st = piped.score(flat, F32, flags)
        engine.prepare(flat, F32, flags)
        engine.execute()
        b, sb, _ = engine.fetch()
        assert np.array_equal(a, b, equal_nan=True) and np.array_equal(sa, sb)
        assert st.num_pairs == flat.num_pairs
    # ramped automatic pipelining is exercised by the 1M-pair test (test_gpu_parity.py)
    piped.close()
    with pytest.raises(Exception):
        engine.set_pipeline(9)


def test_chunked_score_rejects_invalid_chunk_and_recovers(engine):
    from paper_2411_11547_b200 import datagen
    from paper_2411_11547_b200.errors import DataError
    piped = _native.Context(0)
    piped.set_pipeline(4)
    flat = datagen.workload("c2", num_batches=520)
    bad = FlatBatches(**{f: np.array(getattr(flat, f), copy=True) for f in FlatBatches.FIELDS})
    bad.hap_bases[-3] = 9                                     # last chunk: invalid base code
    with pytest.raises(DataError):
        piped.score(bad, F32, 0)
    bad = FlatBatches(**{f: np.array(getattr(flat, f), copy=True) for f in FlatBatches.FIELDS})
    bad.bq[5] = 200                                           # first chunk: invalid quality
    with pytest.raises(DataError):
        piped.score(bad, F32, 0)
    a, sa, _ = piped.score(flat, F32, 0)                     # the context is still healthy
    engine.prepare(flat, F32, 0)
    engine.execute()
    b, sb, _ = engine.fetch()
    assert np.array_equal(a, b, equal_nan=True) and np.array_equal(sa, sb)
    piped.close()


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_random_batches_all_modes_against_oracle(engine, seed):
    """Random batch shapes: 1-12 reads x 1-24 haplotypes, read lengths 1-520 (every
    tiling and the striped legacy path), haplotype lengths 1-700, qualities over the full
    0..93 range (incl. gcp 0 and degenerate indels), N bases.  Fast FP32 / retry /
    exact / f64-config results against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    rb, bq, iq, dq, gq, hb, rlen, hlen, bro, bho = [], [], [], [], [], [], [], [], [0], [0]
    for _ in range(int(rng.integers(4, 9))):
        nr, nh = int(rng.integers(1, 13)), int(rng.integers(1, 25))
        hl = [int(x) for x in rng.integers(1, 701, size=nh)]
        base = rng.integers(0, 5, size=max(hl) + 600, dtype=np.int8)
        for n in hl:
            h = base[:n].copy()
            hit = rng.random(n) < 0.02
            h[hit] = rng.integers(0, 5, size=int(hit.sum()))
            hb.append(h); hlen.append(n)
        for _ in range(nr):
            m = int(rng.integers(1, 521)) if rng.random() < 0.8 else int(rng.integers(1, 40))
            st = int(rng.integers(0, 300))
            r = base[st:st + m].copy() if rng.random() < 0.7 else rng.integers(0, 5, size=m, dtype=np.int8)
            if r.shape[0] < m:
                r = np.concatenate([r, rng.integers(0, 5, size=m - r.shape[0], dtype=np.int8)])
            rb.append(r); rlen.append(m)
            bq.append(rng.integers(0, 94, size=m).astype(np.uint8))
            low = rng.random() < 0.1
            iq.append(rng.integers(1 if low else 20, 94, size=m).astype(np.uint8))
            dq.append(rng.integers(1 if low else 20, 94, size=m).astype(np.uint8))
            g = np.full(m, int(rng.choice([10, 10, 10, 3, 0, 40])), np.uint8)
            gq.append(g)
        bro.append(bro[-1] + nr); bho.append(bho[-1] + nh)
    cat = np.concatenate
    flat = FlatBatches(read_bases=cat(rb), bq=cat(bq), iq=cat(iq), dq=cat(dq), gq=cat(gq),
                       read_off=np.concatenate([[0], np.cumsum(rlen)]).astype(np.int64),
                       hap_bases=cat(hb), hap_off=np.concatenate([[0], np.cumsum(hlen)]).astype(np.int64),
                       batch_read_off=np.asarray(bro, np.int64), batch_hap_off=np.asarray(bho, np.int64))
    _check(engine, flat)
    ofl = oracle.Flat(**flat.as_dict())
    ref32, k32 = oracle.score(ofl, "f32")
    s, st, _ = engine.score(flat, F32, _native.FLAG_EXACT)         # exact mode: bit-identical
    assert np.array_equal(st & KIND, k32) and np.array_equal(s, ref32, equal_nan=True)
    ref64, k64 = oracle.score(ofl, "f64")
    s, st, _ = engine.score(flat, config_tuples(default_configs("f64")), 0)
    assert np.array_equal(st & KIND, k64) and np.array_equal(s, ref64, equal_nan=True)


def test_long_haplotypes_ring_mode_all_modes(engine, rng):
    """Haplotypes longer than a sub-warp slot's row-code capacity (P=4: 510, P=16: 2046,
    P=32: 4094 rows) stream in ring mode (row codes restaged every half ring): short
    reads x haplotypes of 511-8000 bases, and long (striped) reads x 4095-6000-base
    haplotypes; fast FP32, FP64 retry, exact mode and f64 configurations."""
    flat = _flat(rng, [([60, 14, 250], [511, 512, 1100, 2047, 2048, 2049], "derived"),
                       ([120, 255], [4095, 4096, 4097, 8000], "derived"),
                       ([90, 200], [5000, 3, 600], "random"),
                       ([700, 1023], [4095, 6000], "derived"),
                       ([600], [4500, 10], "random")])
    k32 = _check(engine, flat)
    assert (k32 == 0).any()
    ofl = oracle.Flat(**flat.as_dict())
    ref32, _ = oracle.score(ofl, "f32")
    s, st, _ = engine.score(flat, F32, _native.FLAG_EXACT)
    assert np.array_equal(st & KIND, k32) and np.array_equal(s, ref32, equal_nan=True)
    ref64, k64 = oracle.score(ofl, "f64")
    s, st, _ = engine.score(flat, config_tuples(default_configs("f64")), 0)
    assert np.array_equal(st & KIND, k64) and np.array_equal(s, ref64, equal_nan=True)


@pytest.mark.parametrize("scale", [0, 24, 120])
def test_guard_band_adversarial_qualities(engine, scale):
    """Adversarial transition qualities for the guard band: low gap-
    continuation (eps near 1: g_i up to n) and low deletion / insertion qualities make
    n*Gsum huge, and small boundary scales put short, high-likelihood pairs (|score| of a
    few units) near the band.  Flag sets must equal the reference's and values stay
    within 1e-4 relative."""
    from paper_2411_11547_b200 import EngineConfig
    rng = np.random.default_rng(4242 + scale)
    rb, bq, iq, dq, gq, hb, rlen, hlen, bro, bho = [], [], [], [], [], [], [], [], [0], [0]
    for _ in range(40):
        nr, nh = int(rng.integers(1, 6)), int(rng.integers(1, 8))
        hl = [int(x) for x in rng.integers(1, 400, size=nh)]
        base = rng.integers(0, 4, size=max(hl) + 300, dtype=np.int8)
        for n in hl:
            hb.append(base[:n].copy()); hlen.append(n)
        for _ in range(nr):
            m = int(rng.integers(1, 120))
            st0 = int(rng.integers(0, 200))
            rb.append(base[st0:st0 + m].copy()); rlen.append(m)
            bq.append(rng.integers(20, 94, size=m).astype(np.uint8))
            iq.append(rng.integers(4, 12, size=m).astype(np.uint8))    # delta + zeta < 1
            dq.append(rng.integers(4, 12, size=m).astype(np.uint8))
            gq.append(rng.integers(1, 4, size=m).astype(np.uint8))
        bro.append(bro[-1] + nr); bho.append(bho[-1] + nh)
    cat = np.concatenate
    flat = FlatBatches(read_bases=cat(rb), bq=cat(bq), iq=cat(iq), dq=cat(dq), gq=cat(gq),
                       read_off=np.concatenate([[0], np.cumsum(rlen)]).astype(np.int64),
                       hap_bases=cat(hb), hap_off=np.concatenate([[0], np.cumsum(hlen)]).astype(np.int64),
                       batch_read_off=np.asarray(bro, np.int64), batch_hap_off=np.asarray(bho, np.int64))
    cfg = config_tuples([EngineConfig(32, 32, "f32", scale_log2=scale)])
    ofl = oracle.Flat(**flat.as_dict())
    pr, ph = flat.pair_index()
    acc, kind = oracle.score_raw(ofl, "f32", scale)
    ref = oracle.finish(acc, kind, scale)
    # the (one) config binds reads <= 1024: every pair is scored
    s, st, _ = engine.score(flat, cfg, 0)
    assert np.array_equal(st & KIND, kind)
    ok = kind == 0
    assert ok.sum() > 100
    rel = np.abs(s[ok] - ref[ok]) / np.maximum(np.abs(ref[ok]), 1e-300)
    assert rel.max() <= REL_TOL, rel.max()


def test_device_budget_streams_in_bounded_chunks(engine):
    """phmm_set_device_budget: a call ~4x over the bound streams through three chunk
    contexts reused round-robin (many chunks); results equal the resident path bitwise and
    the device working set stays within the bound (+ fixed per-context scratch)."""
    flat = datagen.workload("c3", num_batches=48)
    want, wst, _ = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    ctx = _native.Context(0)
    budget = 6 << 20
    ctx.set_device_budget(budget)
    got, gst, stats = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(got, want, equal_nan=True) and np.array_equal(gst, wst)
    assert stats.num_pairs == flat.num_pairs and stats.device_ms > 0
    assert ctx.device_bytes() <= budget * 1.25 + (8 << 20), ctx.device_bytes()
    # an invalid chunk in the middle is reported and the context recovers
    bad = datagen.workload("c3", num_batches=48)
    bad.bq = bad.bq.copy()
    bad.bq[bad.read_off[bad.batch_read_off[30]]] = 200
    with pytest.raises(DataError):
        ctx.score(bad, F32, _native.FLAG_RETRY_F64)
    again, _, _ = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(again, want, equal_nan=True)
    ctx.close()


def test_run_device_budget_matches_unbounded():
    from paper_2411_11547_b200 import default_configs, run
    flat = datagen.workload("c3", num_batches=24)
    a, ra = run(flat, default_configs("f32"), retry_f64=True)
    b, rb = run(flat, default_configs("f32"), retry_f64=True, device_budget_bytes=2 << 20)
    assert np.array_equal(a, b, equal_nan=True) and ra.total_cells == rb.total_cells
    assert ra.errors == rb.errors and ra.retried == rb.retried


def test_100k_base_haplotype_linear_device_memory(engine, rng):
    """A 100,000-base haplotype (and a long striped read against it) scores in every mode
    without a per-haplotype-length scratch blow-up: the ring-mode row codes and the
    grid-capped boundary columns keep the device working set bounded (reference.py:77-123
    handles any n in linear space)."""
    flat = _flat(rng, [([80, 250], [100000, 300], "derived"),
                       ([700], [100000], "derived"),
                       ([150], [100000], "random")])
    ctx = _native.Context(0)
    k32 = _check(ctx, flat)
    assert (k32 == 0).any() and (k32 == 1).any()
    ofl = oracle.Flat(**flat.as_dict())
    ref64, k64 = oracle.score(ofl, "f64")
    s, st, _ = ctx.score(flat, config_tuples(default_configs("f64")), 0)
    assert np.array_equal(st & KIND, k64) and np.array_equal(s, ref64, equal_nan=True)
    assert ctx.device_bytes() < (1536 << 20), ctx.device_bytes()
    ctx.close()


def test_c3_device_scratch_is_small(engine):
    """Boundary-column scratch only where a read needs stripes: c3 (reads <= 250) keeps the
    whole context's device working set near its inputs + per-pair lists."""
    flat = datagen.workload("c3")
    ctx = _native.Context(0)
    ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    # inputs ~6.5 MB + per-pair buffers (acc, status, unit/entry lists sized for every pair)
    per_pair = 200 * flat.num_pairs
    assert ctx.device_bytes() < flat.nbytes() + per_pair + (64 << 20), ctx.device_bytes()
    ctx.close()


def test_automatic_ramp_of_a_large_call_bit_identical():
    """The automatic chunk ramp of the largest calls ((1,5,10,10,5,1) from 8M pairs: six
    chunk contexts, device-built second-stage FP64 units on a side stream) against the one
    pass of the same context, bit for bit, with the FP64 retry."""
    flat = datagen.workload("c5", num_batches=16384)                    # 8.4M pairs
    assert flat.num_pairs >= 8_000_000
    ctx = _native.Context(0)
    got, gst, st = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    ctx.set_pipeline(1)
    want, wst, _ = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(got, want, equal_nan=True) and np.array_equal(gst, wst)
    assert st.num_pairs == flat.num_pairs and st.device_ms > 0
    assert ((gst & _native.ST_RETRIED_F64) != 0).mean() > 0.2            # the retry path ran
    ctx.close()


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_pipeline_depths_bit_identical(engine, n):
    """phmm_set_pipeline(n): n equal chunk contexts give bit-identical results to the one
    pass (pairs are independent), with the FP64 retry and the guard band in play."""
    flat = datagen.workload("c3", num_batches=40)
    want, wst, _ = engine.score(flat, F32, _native.FLAG_RETRY_F64)   # < 2^20 pairs: one pass
    ctx = _native.Context(0)
    ctx.set_pipeline(n)
    got, gst, st = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(got, want, equal_nan=True) and np.array_equal(gst, wst)
    assert st.num_pairs == flat.num_pairs and st.device_ms > 0
    ctx.set_pipeline(1)                                            # never pipeline
    got1, gst1, _ = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(got1, want, equal_nan=True) and np.array_equal(gst1, wst)
    ctx.close()

"""GPU parity: the CUDA engine (through the C-ABI) against the reference's outputs.

Bars (BASELINE.json north_star):
  * exact mode and f64 configs: bit-identical to the reference (same kernel arithmetic);
  * fast FP32 mode: identical numeric-overflow (retry) set, per-pair log10 within
    1e-4 relative (REL_TOL below);
  * FP64 retry: retried pairs within 1e-9 relative of the reference's f64 scores (the
    fast FP64 kernel, FMA + folded recurrence); f64 CONFIGS use the bit-exact FP64 kernel.
Golden fixtures come from the reference itself (tests/golden/make_golden.py); the
full-size configs are checked against the C oracle, which tests/test_oracle_golden.py
pins bit-exactly to the reference.
"""
import numpy as np
import pytest

from conftest import GOLDEN, golden_flat, load_golden
from oracle import oracle
from paper_2411_11547_b200 import _native, datagen, default_configs
from paper_2411_11547_b200.pipeline import config_tuples

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4          # fast FP32 path vs reference FP32 (north_star)
RETRY_REL_TOL = 1e-9    # FP64 retry vs reference FP64 (north_star)
F32 = config_tuples(default_configs("f32"))
F64 = config_tuples(default_configs("f64"))
KIND = _native.ST_KIND_MASK


def _rel(a, b):
    return np.abs(a - b) / np.abs(b)


def _check_fast(scores, status, ref, ref_kind, label):
    kinds = status & KIND
    assert np.array_equal(kinds, ref_kind), label + ": flag sets differ"
    ok = ref_kind == 0
    assert np.all(np.isfinite(scores[ok])) and np.all(np.isnan(scores[~ok]))
    if ok.any():
        worst = _rel(scores[ok], ref[ok]).max()
        assert worst <= REL_TOL, "%s: max rel err %.3e" % (label, worst)


@pytest.mark.parametrize("name", GOLDEN)
def test_exact_mode_bit_identical_to_reference_f32(engine, name):
    z = load_golden(name)
    scores, status, _ = engine.score(golden_flat(z), F32, _native.FLAG_EXACT)
    assert np.array_equal(status & KIND, z["ref_f32_kind"])
    assert np.array_equal(scores, z["ref_f32"], equal_nan=True)


@pytest.mark.parametrize("name", GOLDEN)
def test_f64_configs_bit_identical_to_reference_f64(engine, name):
    z = load_golden(name)
    scores, status, _ = engine.score(golden_flat(z), F64, 0)
    assert np.array_equal(status & KIND, z["ref_f64_kind"])
    assert np.array_equal(scores, z["ref_f64"], equal_nan=True)


@pytest.mark.parametrize("name", GOLDEN)
def test_fast_mode_matches_reference_f32(engine, name):
    z = load_golden(name)
    scores, status, stats = engine.score(golden_flat(z), F32, 0)
    _check_fast(scores, status, z["ref_f32"], z["ref_f32_kind"], name)


@pytest.mark.parametrize("name", GOLDEN)
def test_retry_f64_rescues_exactly_the_reference_flag_set(engine, name):
    z = load_golden(name)
    scores, status, _ = engine.score(golden_flat(z), F32, _native.FLAG_RETRY_F64)
    flagged32 = z["ref_f32_kind"] == 1
    retried = (status & _native.ST_RETRIED_F64) != 0
    assert np.array_equal(retried, flagged32)
    # retried pairs carry the reference's f64 result (or its f64 flag)
    assert np.array_equal(status[retried] & KIND, z["ref_f64_kind"][retried])
    got, want = scores[retried], z["ref_f64"][retried]
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin)
    if fin.any():
        assert _rel(got[fin], want[fin]).max() <= RETRY_REL_TOL
    rest = ~retried
    _check_fast(scores[rest], status[rest], z["ref_f32"][rest], z["ref_f32_kind"][rest], name)


@pytest.mark.parametrize("wl,batches", [("c1", None), ("c1_independent", None), ("c2", None),
                                        ("c3", None), ("c4", 16), ("c4_underflow", 8)])
def test_full_size_configs_against_oracle(engine, wl, batches):
    """BASELINE configs at full size (c4 prefixes) vs the C oracle (reference-pinned)."""
    flat = datagen.workload(wl, num_batches=batches)
    ofl = oracle.Flat(**flat.as_dict())
    ref32, k32 = oracle.score(ofl, "f32")
    scores, status, stats = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    flagged = k32 == 1
    assert np.array_equal((status & _native.ST_RETRIED_F64) != 0, flagged)
    rest = ~flagged
    _check_fast(scores[rest], status[rest], ref32[rest], k32[rest], wl)
    if flagged.any():
        pr, ph = flat.pair_index()
        idx = np.flatnonzero(flagged)
        acc64, st64 = oracle.score_raw(ofl, "f64", 0, pairs=(pr[idx], ph[idx]))
        ref64 = oracle.finish(acc64, st64, 0)
        assert np.array_equal(status[idx] & KIND, st64)
        fin = st64 == 0
        assert _rel(scores[idx][fin], ref64[fin]).max() <= RETRY_REL_TOL
    assert stats.total_cells == int((flat.read_len[flat.pair_index()[0]]
                                     * flat.hap_len[flat.pair_index()[1]]).sum())


def test_fast_path_carries_the_bulk(engine):
    """On the GATK-shaped config most pairs are accepted from the fast kernel."""
    flat = datagen.workload("c3", num_batches=16)
    _, status, stats = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    assert stats.fast_pairs >= 0.7 * stats.num_pairs
    assert stats.fast_pairs + stats.exact_pairs + stats.f64_pairs <= stats.num_pairs


def test_results_are_deterministic_and_order_independent(engine):
    flat = datagen.workload("c3", num_batches=6)
    a, sa, _ = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    b, sb, _ = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    assert np.array_equal(a, b, equal_nan=True) and np.array_equal(sa, sb)
    # reverse the batch order: every pair keeps its bits
    from paper_2411_11547_b200.model import FlatBatches
    B = flat.num_batches
    parts = []
    for bidx in reversed(range(B)):
        r0, r1 = flat.batch_read_off[bidx], flat.batch_read_off[bidx + 1]
        h0, h1 = flat.batch_hap_off[bidx], flat.batch_hap_off[bidx + 1]
        parts.append((r0, r1, h0, h1))
    ro, ho = flat.read_off, flat.hap_off
    sel_r = np.concatenate([np.arange(ro[r0], ro[r1]) for r0, r1, _, _ in parts])
    sel_h = np.concatenate([np.arange(ho[h0], ho[h1]) for _, _, h0, h1 in parts])
    rl = np.concatenate([np.diff(ro[r0:r1 + 1]) for r0, r1, _, _ in parts])
    hl = np.concatenate([np.diff(ho[h0:h1 + 1]) for _, _, h0, h1 in parts])
    rev = FlatBatches(read_bases=flat.read_bases[sel_r], bq=flat.bq[sel_r], iq=flat.iq[sel_r],
                      dq=flat.dq[sel_r], gq=flat.gq[sel_r],
                      read_off=np.concatenate([[0], np.cumsum(rl)]),
                      hap_bases=flat.hap_bases[sel_h], hap_off=np.concatenate([[0], np.cumsum(hl)]),
                      batch_read_off=np.concatenate([[0], np.cumsum([r1 - r0 for r0, r1, _, _ in parts])]),
                      batch_hap_off=np.concatenate([[0], np.cumsum([h1 - h0 for _, _, h0, h1 in parts])]))
    c, sc, _ = engine.score(rev, F32, _native.FLAG_RETRY_F64)
    N = [int((flat.batch_read_off[i + 1] - flat.batch_read_off[i])
             * (flat.batch_hap_off[i + 1] - flat.batch_hap_off[i])) for i in range(B)]
    starts = np.concatenate([[0], np.cumsum(N)])
    expect = np.concatenate([a[starts[i]:starts[i + 1]] for i in reversed(range(B))])
    assert np.array_equal(c, expect, equal_nan=True)


def test_prepare_execute_fetch_is_rerunnable(engine):
    flat = datagen.workload("c2", num_batches=32)
    engine.prepare(flat, F32, 0)
    engine.execute()
    a, sa, st1 = engine.fetch()
    engine.execute()
    b, sb, st2 = engine.fetch()
    assert np.array_equal(a, b) and np.array_equal(sa, sb)
    c, sc, _ = engine.score(flat, F32, 0)
    assert np.array_equal(a, c)
    assert st2.device_ms > 0 and st2.fast_ms > 0 and st2.kernel_launches >= 2


def test_million_pair_gatk_call_against_oracle(engine):
    """A >= 1M-pair GATK-shaped call (the c5 prefix of 2,048 batches = 1,048,576 pairs)
    with the FP64 retry: the big-call branches (3 ramped pipelined chunk contexts, longer
    device-built retry units) against the oracle -- f32 for every pair, f64 on the
    flagged subset; chunked-call stats are filled (device time span, FP32 phases)."""
    flat = datagen.workload("c5", num_batches=2048)
    assert flat.num_pairs >= 1 << 20
    ofl = oracle.Flat(**flat.as_dict())
    ref32, k32 = oracle.score(ofl, "f32")
    scores, status, stats = engine.score(flat, F32, _native.FLAG_RETRY_F64)
    flagged = k32 == 1
    assert flagged.mean() > 0.1
    assert np.array_equal((status & _native.ST_RETRIED_F64) != 0, flagged)
    rest = ~flagged
    _check_fast(scores[rest], status[rest], ref32[rest], k32[rest], "c5[:2048]")
    pr, ph = flat.pair_index()
    idx = np.flatnonzero(flagged)
    acc64, st64 = oracle.score_raw(ofl, "f64", 0, pairs=(pr[idx], ph[idx]))
    ref64 = oracle.finish(acc64, st64, 0)
    assert np.array_equal(status[idx] & KIND, st64)
    fin = st64 == 0
    assert _rel(scores[idx][fin], ref64[fin]).max() <= RETRY_REL_TOL
    assert stats.num_pairs == flat.num_pairs
    assert stats.device_ms > 0 and stats.fast_ms > 0 and stats.h2d_ms > 0

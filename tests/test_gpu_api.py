"""The drop-in API on the GPU engine — the reference's own black-box tests
(pkg/tests/test_reference.py, test_wavefront.py, test_pipeline.py, test_acceptance.py)
re-pointed at paper_2411_11547_b200."""
import math

import numpy as np
import pytest

from conftest import make_hap, make_read, random_pair
from paper_2411_11547_b200 import (Batch, EngineConfig, Haplotype, ReadRecord, default_configs,
                                   enumerate_work_items, forward_reference,
                                   forward_reference_linear_space, forward_wavefront,
                                   forward_wavefront_batch, forward_wavefront_counted, run,
                                   select_config, throughput)
from paper_2411_11547_b200.datagen import generate_synthetic, generate_verification_pairs
from paper_2411_11547_b200.errors import (BudgetError, ConfigTooSmallError,
                                          DegenerateTransitionError, NumericOverflowError)

pytestmark = pytest.mark.gpu

LOG10_MATCH_081 = -0.0915149811213503       # test_reference.py:14-30
LOG10_MISMATCH_003 = -1.5228787452803376
SEED = 20240811


def _hand_read():
    return make_read("A", base_q=10, ins_q=40, del_q=40, gcp_q=10)


def test_hand_cases():
    assert forward_reference(_hand_read(), make_hap("A")).log10_likelihood == pytest.approx(LOG10_MATCH_081, abs=1e-9)
    assert forward_reference(_hand_read(), make_hap("C")).log10_likelihood == pytest.approx(LOG10_MISMATCH_003, abs=1e-9)
    for prec in ("f32", "f64"):
        wf = forward_wavefront(_hand_read(), make_hap("A"), EngineConfig(2, 4, prec))
        assert wf.log10_likelihood == pytest.approx(LOG10_MATCH_081, abs=1e-6 if prec == "f32" else 1e-9)


def test_path_enumeration_small_instances(rng):
    from itertools import product  # noqa: F401

    def path_sum(read, hap):
        # independent exponential oracle (reference tests/oracles.py:18-57)
        q = 10.0 ** (-read.base_qual.astype(float) / 10)
        d = 10.0 ** (-read.ins_qual.astype(float) / 10)
        z = 10.0 ** (-read.del_qual.astype(float) / 10)
        e = 10.0 ** (-read.gcp_qual.astype(float) / 10)
        a, b = 1.0 - d - z, 1.0 - e
        m, n = read.length, hap.length

        def lam(i, j):
            r, h = read.bases[i - 1], hap.bases[j - 1]
            return 1.0 - q[i - 1] if (r == h or r == 4 or h == 4) else q[i - 1] / 3.0

        def v(i, j, s):
            if i == 0:
                return 1.0 / n if s == "D" else 0.0
            if j == 0:
                return 0.0
            if s == "M":
                return lam(i, j) * (a[i - 1] * v(i - 1, j - 1, "M") + b[i - 1] * v(i - 1, j - 1, "I")
                                    + b[i - 1] * v(i - 1, j - 1, "D"))
            if s == "I":
                return d[i - 1] * v(i - 1, j, "M") + e[i - 1] * v(i - 1, j, "I")
            return z[i - 1] * v(i, j - 1, "M") + e[i - 1] * v(i, j - 1, "D")
        return sum(v(m, j, "M") + v(m, j, "I") for j in range(1, n + 1))

    for _ in range(40):
        m, n = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        read = ReadRecord(rng.integers(0, 5, size=m, dtype=np.int8), rng.integers(0, 41, m),
                          rng.integers(10, 94, m), rng.integers(10, 94, m), rng.integers(0, 94, m))
        hap = Haplotype(rng.integers(0, 5, size=n, dtype=np.int8))
        expected = path_sum(read, hap)
        if expected > 0:
            assert forward_reference(read, hap).log10_likelihood == pytest.approx(math.log10(expected), abs=1e-12)


def test_degenerate_and_underflow_errors(rng):
    with pytest.raises(DegenerateTransitionError):
        forward_reference(make_read("ACG", ins_q=2, del_q=2), make_hap("ACG"))
    with pytest.raises(ConfigTooSmallError):
        forward_wavefront(make_read("ACGTACGTACGT"), make_hap("ACGT"), EngineConfig(2, 4))
    read, hap = random_pair(rng, 700, 700, mutation_rate=0.10, base_q=(10, 11))
    assert forward_reference(read, hap).log10_likelihood < -70
    with pytest.raises(NumericOverflowError, match="double precision"):
        forward_wavefront(read, hap, EngineConfig(32, 32, "f32"))


def test_double_precision_matches_reference_bitwise(rng):
    for _ in range(40):
        n = int(rng.integers(1, 160))
        m = int(rng.integers(1, n + 1))
        read, hap = random_pair(rng, m, n)
        expected = forward_reference(read, hap).log10_likelihood
        for p, k in [(2, 4), (4, 8), (16, 16), (32, 8)]:
            if p * k >= m:
                assert forward_wavefront(read, hap, EngineConfig(p, k, "f64")).log10_likelihood == expected


def test_single_precision_close_to_double(rng):
    worst = 0.0
    for _ in range(30):
        n = int(rng.integers(1, 700))
        m = int(rng.integers(1, n + 1))
        read, hap = random_pair(rng, m, n, base_q=(15, 41))
        expected = forward_reference(read, hap).log10_likelihood
        got = forward_wavefront(read, hap, EngineConfig(32, 32, "f32"))
        worst = max(worst, abs(got.log10_likelihood - expected))
    assert worst <= 1e-3


def test_step_count_is_rows_plus_lanes(rng):
    # test_wavefront.py:50-55: the reference's step count n + p, for any config
    for m, n, p, k in [(1, 1, 2, 4), (5, 200, 4, 8), (60, 3, 32, 8), (256, 64, 32, 8), (17, 17, 4, 8)]:
        read, hap = random_pair(rng, m, n)
        _, steps = forward_wavefront_counted(read, hap, EngineConfig(p, k, "f64"))
        assert steps == n + p


def test_engine_wavefront_steps():
    from paper_2411_11547_b200 import _native
    from paper_2411_11547_b200.wavefront import engine_wavefront_steps
    P, K, Q = _native.fast_geometry(100, 150)
    assert engine_wavefront_steps(100, 150) == Q * (150 + P - 1)


def test_padding_and_tiling_invariance(rng):
    for precision in ("f32", "f64"):
        for _ in range(10):
            n = int(rng.integers(1, 100))
            m = int(rng.integers(1, min(n, 64) + 1))
            read, hap = random_pair(rng, m, n)
            values = {forward_wavefront(read, hap, EngineConfig(p, k, precision)).log10_likelihood
                      for p, k in [(2, 4), (4, 8), (8, 8), (16, 16), (32, 32)] if p * k >= m}
            assert len(values) == 1


def test_batch_matches_per_item_and_isolates_failures(rng):
    good, hap = random_pair(rng, 20, 40)
    too_long, _ = random_pair(rng, 60, 70)
    batches = [Batch((good, too_long), (hap,))]
    items = enumerate_work_items(batches)
    out = np.full(len(items), np.nan)
    errors = forward_wavefront_batch(batches, items, EngineConfig(4, 8, "f64"), out)
    assert errors == [(1, "config-too-small")]
    assert math.isfinite(out[0]) and math.isnan(out[1])
    assert out[0] == forward_wavefront(good, hap, EngineConfig(4, 8, "f64")).log10_likelihood


def test_run_report_and_errors(rng):
    shapes = [(3, 2), (1, 3), (2, 2)]
    batches = []
    for r, h in shapes:
        reads = tuple(random_pair(rng, int(rng.integers(5, 60)), 64)[0] for _ in range(r))
        haps = tuple(random_pair(rng, 5, int(rng.integers(10, 80)))[1] for _ in range(h))
        batches.append(Batch(reads, haps))
    scores, report = run(batches, workers=2)
    assert scores.shape[0] == 13 and np.all(np.isfinite(scores))
    expected = sum(b.reads[i].length * b.haps[j].length for b in batches
                   for i in range(len(b.reads)) for j in range(len(b.haps)))
    assert report.total_cells == expected
    assert report.gcups == report.total_cells / (report.wall_seconds * 1e9)
    assert sum(s.cells for s in report.per_config.values()) == expected


def test_run_oversized_reads_and_budget(rng):
    fine, hap = random_pair(rng, 20, 50)
    oversized, _ = random_pair(rng, 200, 220)
    batches = [Batch((fine, oversized), (hap,))]
    scores, report = run(batches, configs=[EngineConfig(4, 8, "f64")])
    assert math.isfinite(scores[0]) and math.isnan(scores[1])
    assert report.errors == [(1, "config-too-small")]
    assert report.total_cells == fine.length * hap.length
    with pytest.raises(BudgetError):
        run(batches, budget_bytes=64)


def test_run_empty_and_workers():
    scores, report = run([])
    assert scores.shape == (0,) and report.total_cells == 0 and report.gcups == 0.0
    assert report.errors == []
    with pytest.raises(ValueError):
        run([], workers=0)
    assert throughput(2_500_000_000, 2.0) == 1.25


def test_run_worker_and_budget_independent():
    batches = generate_synthetic(6, 5, 4, (10, 40), (20, 60), 7, mode="derived")
    base, rep = run(batches, workers=1)
    for w in (2, 8):
        assert np.array_equal(run(batches, workers=w)[0], base)
    assert np.array_equal(run(batches, workers=2, budget_bytes=1 << 14)[0], base)
    assert rep.errors == []


def test_run_matches_direct_engine_calls():
    batches = generate_synthetic(2, 5, 4, (10, 40), (20, 60), 7, mode="derived")
    configs = default_configs("f64")
    scores, _ = run(batches, configs=configs)
    for item in enumerate_work_items(batches)[::5]:
        b = batches[item.batch_index]
        read = b.reads[item.read_index]
        want = forward_wavefront(read, b.haps[item.hap_index], select_config(read.length, configs))
        assert scores[item.global_id] == want.log10_likelihood


def test_retry_f64_gives_finite_scores_for_underflowing_pairs():
    batches = generate_synthetic(10, 25, 4, 100, 150, SEED, mode="independent", base_qual=30,
                                 indel_qual=45, gcp_qual=10)
    s32, r32 = run(batches)
    assert len(r32.errors) == 1000 and np.all(np.isnan(s32))
    s, r = run(batches, retry_f64=True)
    assert r.errors == [] and len(r.retried) == 1000 and np.all(np.isfinite(s))
    s64, _ = run(batches, configs=default_configs("f64"))
    assert np.max(np.abs(s - s64) / np.abs(s64)) <= 1e-9
    assert r.total_cells == r32.total_cells == 1000 * 100 * 150


def test_acceptance_oracle_equivalence_sample():
    pairs = generate_verification_pairs(400, SEED)
    f32, f64 = default_configs("f32"), default_configs("f64")
    worst = 0.0
    for batch in pairs:
        read, hap = batch.reads[0], batch.haps[0]
        oracle = forward_reference_linear_space(read, hap).log10_likelihood
        assert forward_wavefront(read, hap, select_config(read.length, f64)).log10_likelihood == oracle
        got = forward_wavefront(read, hap, select_config(read.length, f32)).log10_likelihood
        worst = max(worst, abs(got - oracle))
    assert worst <= 1e-3


def test_scale_invariance():
    for batch in generate_verification_pairs(100, SEED + 4, max_read_len=256, max_hap_len=256):
        read, hap = batch.reads[0], batch.haps[0]
        a = forward_reference_linear_space(read, hap, scale_log2=0).log10_likelihood
        b = forward_reference_linear_space(read, hap, scale_log2=120).log10_likelihood
        assert abs(a - b) < 1e-12


def test_forward_matrices_bit_identical_to_reference():
    """forward_matrices (GPU k_matrices) against the reference's own forward_matrices on the
    fixtures tests/golden/make_matrices_golden.py produced: every M, I, D entry bitwise."""
    import os
    from conftest import ROOT
    from paper_2411_11547_b200 import DpMatrices, forward_matrices
    z = np.load(os.path.join(ROOT, "tests", "golden", "matrices.npz"))
    for i in range(int(z["count"])):
        read = ReadRecord(z["%d_bases" % i], z["%d_bq" % i], z["%d_iq" % i], z["%d_dq" % i], z["%d_gq" % i])
        hap = Haplotype(z["%d_hap" % i])
        mats = forward_matrices(read, hap, int(z["%d_scale" % i]))
        assert isinstance(mats, DpMatrices)
        for k in ("M", "I", "D"):
            want = z["%d_%s" % (i, k)]
            got = getattr(mats, k)
            assert got.shape == want.shape and np.array_equal(got.view(np.uint64), want.view(np.uint64)), (i, k)


def test_forward_matrices_score_matches_forward_reference(rng):
    from paper_2411_11547_b200 import forward_matrices
    read, hap = random_pair(rng, 40, 55)
    mats = forward_matrices(read, hap)
    acc = 0.0
    for j in range(1, hap.length + 1):
        acc = acc + (mats.M[read.length, j] + mats.I[read.length, j])
    assert math.log10(acc) == forward_reference(read, hap).log10_likelihood
    with pytest.raises(DegenerateTransitionError):
        forward_matrices(make_read("A", base_q=10, ins_q=0, del_q=0, gcp_q=10), make_hap("A"))

"""The CPU oracle (oracle/phmm_oracle.c) against the reference's own outputs.

tests/golden/*.npz were produced by tests/golden/make_golden.py, which imports
and runs the reference package (pairhmm.run with default f32 and f64 configs).
Bit-identical agreement here is what pins the oracle used by the GPU parity tests.
"""
import numpy as np
import pytest

from conftest import GOLDEN, GOLDEN_DIR, load_golden
from oracle import oracle


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


def test_phred_table_matches_reference():
    z = np.load(GOLDEN_DIR + "/prob_tables.npz")
    assert np.array_equal(z["phred_to_prob"], oracle.PHRED_TO_PROB)
    assert float(z["log10_2"]) == float(oracle.LOG10_2) == 0.30102999566398120


@pytest.mark.parametrize("name", GOLDEN)
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_oracle_bit_identical_to_reference(name, precision):
    z = load_golden(name)
    flat = oracle.Flat.from_npz(z)
    scores, status = oracle.score(flat, precision)
    ref = z["ref_" + precision]
    kind = z["ref_" + precision + "_kind"]
    assert np.array_equal(status, kind)
    assert np.array_equal(scores, ref, equal_nan=True)


def test_golden_fixtures_cover_the_edge_cases():
    kinds = set()
    for name in GOLDEN:
        z = load_golden(name)
        kinds |= set(np.unique(z["ref_f32_kind"]).tolist())
    assert kinds == {0, 1, 2, 3}     # ok, numeric-overflow, config-too-small, degenerate

"""The restated generator reproduces the reference generator's stream exactly.

The golden fixtures hold inputs made by the reference's own
pairhmm.datagen (tests/golden/make_golden.py); regenerating them here with
paper_2411_11547_b200.datagen must give identical arrays.
"""
import json

import numpy as np
import pytest

from conftest import golden_flat, load_golden
from paper_2411_11547_b200 import datagen
from paper_2411_11547_b200.model import FlatBatches

SYNTH = ["c1_derived", "c1_independent", "c2_prefix", "c3_prefix", "c4_prefix", "c4_underflow",
         "short_mixed"]


def _same(a: FlatBatches, b: FlatBatches):
    for f in FlatBatches.FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype and np.array_equal(x, y), f


@pytest.mark.parametrize("name", SYNTH)
def test_generate_synthetic_matches_reference_fixture(name):
    z = load_golden(name)
    params = json.loads(str(z["params"]))
    flat = datagen.generate_synthetic_flat(*params["args"], **params["kw"])
    _same(flat, golden_flat(z))
    objs = FlatBatches.from_batches(datagen.generate_synthetic(*params["args"], **params["kw"]))
    _same(objs, flat)


def test_verification_pairs_match_reference_fixture():
    z = load_golden("verify_pairs")
    n, seed = json.loads(str(z["params"]))["generate_verification_pairs"]
    _same(FlatBatches.from_batches(datagen.generate_verification_pairs(n, seed)), golden_flat(z))


def test_workload_prefix_property():
    # generation is sequential per batch: a shorter run is a prefix of a longer one
    a = datagen.workload("c3", num_batches=2)
    b = datagen.workload("c3", num_batches=3)
    ra = a.read_off[-1]
    assert np.array_equal(a.read_bases, b.read_bases[:ra])
    assert np.array_equal(a.hap_bases, b.hap_bases[:a.hap_off[-1]])


def test_workload_shapes():
    c2 = datagen.workload("c2", num_batches=4)
    assert c2.num_pairs == 4 * 16 * 4
    assert set(np.unique(c2.read_len)) == {250} and set(np.unique(c2.hap_len)) == {250}

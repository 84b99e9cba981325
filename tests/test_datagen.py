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


@pytest.fixture(scope="module")
def native_gen():
    from paper_2411_11547_b200.build import build_host
    build_host()


@pytest.mark.parametrize("name", SYNTH)
def test_native_generator_matches_reference_fixture(native_gen, name):
    """csrc/datagen.cpp (PCG64 + numpy's bounded-integer algorithms) draws the reference
    generator's stream element for element."""
    z = load_golden(name)
    params = json.loads(str(z["params"]))
    flat = datagen._native_flat(*(params["args"] + [params["kw"].get(k, d) for k, d in (
        ("mode", "independent"), ("mutation_rate", datagen.DEFAULT_MUTATION_RATE),
        ("base_qual", datagen.DEFAULT_BASE_QUAL), ("indel_qual", datagen.DEFAULT_INDEL_QUAL),
        ("gcp_qual", datagen.DEFAULT_GCP_QUAL))]))
    assert flat is not None
    _same(flat, golden_flat(z))


@pytest.mark.parametrize("kw", [
    dict(num_batches=40, reads_per_batch=7, haps_per_batch=3, read_len_spec=(1, 300),
         hap_len_spec=(1, 200), seed=5, mode="derived", mutation_rate=0.2),
    dict(num_batches=30, reads_per_batch=3, haps_per_batch=5, read_len_spec=(1, 40),
         hap_len_spec=(1, 40), seed=6, mode="independent", base_qual=(0, 93), indel_qual=(0, 93),
         gcp_qual=(0, 5)),
    dict(num_batches=25, reads_per_batch=4, haps_per_batch=2, read_len_spec=60, hap_len_spec=60,
         seed=7, mode="derived", base_qual=17, indel_qual=(44, 45), gcp_qual=(9, 11)),
    dict(num_batches=300, reads_per_batch=64, haps_per_batch=8, read_len_spec=(50, 250),
         hap_len_spec=(100, 600), seed=datagen.SEED + 4, mode="derived")])
def test_native_generator_matches_numpy_stream(native_gen, kw):
    """Edge shapes (reads longer than the shortest haplotype, equal lengths -> empty start
    range, full quality range, fixed specs, c5's first 300 batches) against the numpy
    restatement."""
    _same(datagen.generate_synthetic_flat(**kw, native=True), datagen.generate_synthetic_flat(**kw, native=False))

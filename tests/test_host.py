"""Host-side logic of the drop-in run() (no GPU): the native flattening of Batch objects at a
size that spreads the copy over several threads, and the error list built from the engine's
per-pair status bytes."""
import numpy as np

from paper_2411_11547_b200 import _native, datagen
from paper_2411_11547_b200.model import FlatBatches, _flatten_ext
from paper_2411_11547_b200.pipeline import errors_from_status


def test_native_flatten_multithreaded_copy_matches_source():
    flat = datagen.workload("c2", num_batches=256)        # 4,096 reads x 250: 5 MB, 3 copy threads
    batches = flat.to_batches()
    assert _flatten_ext() is not None
    a = FlatBatches.from_batches(batches)
    for k in FlatBatches.FIELDS:
        assert np.array_equal(getattr(a, k), getattr(flat, k)), k


def test_errors_from_status_pairs_in_order():
    st = np.zeros(10, np.uint8)
    st[[2, 5, 7]] = [_native.ST_OVERFLOW, _native.ST_TOO_SMALL, _native.ST_DEGENERATE | _native.ST_RETRIED_F64]
    st[8] = _native.ST_RETRIED_F64                       # retried and scored: not an error
    assert errors_from_status(st) == [(2, "numeric-overflow"), (5, "config-too-small"),
                                      (7, "degenerate-transition")]
    assert errors_from_status(np.zeros(0, np.uint8)) == []


def test_native_flatten_falls_back_to_the_serial_walk():
    # one record whose track is a bytes object (buffer protocol, not an ndarray): the
    # threaded view pass bails out and the serial walk produces the same arrays
    flat = datagen.workload("c2", num_batches=256)
    batches = flat.to_batches()
    rec = batches[200].reads[3]
    object.__setattr__(rec, "ins_qual", bytes(np.asarray(rec.ins_qual)))
    a = FlatBatches.from_batches(batches)
    for k in FlatBatches.FIELDS:
        assert np.array_equal(getattr(a, k), getattr(flat, k)), k

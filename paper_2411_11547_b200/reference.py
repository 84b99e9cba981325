"""Double-precision scoring entry points (mirror of reference reference.py:161-175).

forward_matrices returns the complete FP64 DP matrices of one pair (GPU k_matrices).
forward_reference / forward_reference_linear_space score one pair in float64
with boundary scale 2^scale_log2 and the f64 flush policy (prob.py:39), like the
reference's oracle.  Here they run on the GPU's bit-exact FP64 kernel
(k_exact<double>), whose arithmetic order equals reference.py:106-122, so the
result is bit-identical to the reference's oracle for any read length (no
p*k limit: the engine stripes long reads).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import NumericOverflowError
from .model import Batch, FlatBatches, Score
from .prob import build_transitions


def _f64(read, hap, scale_log2: int) -> Score:
    build_transitions(read)                     # degenerate-transition raises here
    flat = FlatBatches.from_batches([Batch((read,), (hap,))])
    cfg = [(1, read.length, 1, int(scale_log2))]
    scores, status, _ = _native.context(0).score(flat, cfg, 0)
    if (status[0] & _native.ST_KIND_MASK) != _native.ST_OK:
        raise NumericOverflowError("accumulator out of range; retry in double precision or with "
                                   "a different scale")
    return Score(float(scores[0]))


def forward_reference(read, hap, scale_log2: int = 0) -> Score:
    return _f64(read, hap, scale_log2)


def forward_reference_linear_space(read, hap, scale_log2: int = 0) -> Score:
    return _f64(read, hap, scale_log2)


@dataclass(frozen=True)
class DpMatrices:
    """The filled (m+1) x (n+1) float64 tables, boundaries included (reference.py:126-132)."""

    M: np.ndarray
    I: np.ndarray
    D: np.ndarray


def forward_matrices(read, hap, scale_log2: int = 0) -> DpMatrices:
    """Fill and return the complete dynamic-programming matrices of one pair on the GPU
    (k_matrices: bit-identical to the reference's _full_kernel, reference.py:150-156)."""
    build_transitions(read)                     # degenerate-transition raises here
    M, I, D = _native.context(0).forward_matrices(read, hap, scale_log2)
    return DpMatrices(M, I, D)

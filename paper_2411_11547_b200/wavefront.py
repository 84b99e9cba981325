"""Single-pair and item-list entry points of the GPU wavefront engine.

Mirror of the reference's wavefront.py public API (wavefront.py:441-505):

  forward_wavefront(read, hap, cfg) -> Score
  forward_wavefront_counted(read, hap, cfg) -> (Score, steps)
  forward_wavefront_batch(batches, items, cfg, out, errors=None) -> errors

Errors behave like the reference: a read longer than cfg.m_max raises
ConfigTooSmallError, a degenerate transition raises DegenerateTransitionError and
an out-of-range accumulator raises NumericOverflowError (single pair) or is
recorded as (global_id, kind) with NaN in ``out`` (batch).  All scoring runs in
libphmm.so on the GPU.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .errors import ConfigTooSmallError, NumericOverflowError
from .model import Batch, FlatBatches, Score
from .pipeline import config_tuples, engine_flags
from .prob import build_transitions


def _score_pairs(reads, haps, cfg, device=0):
    """Score pairs (reads[i], haps[i]) as single-pair batches with one config."""
    flat = FlatBatches.from_batches([Batch((r,), (h,)) for r, h in zip(reads, haps)])
    ctx = _native.context(device)
    return ctx.score(flat, config_tuples([cfg]), engine_flags())


def _single(read, hap, cfg):
    if read.length > cfg.m_max:
        raise ConfigTooSmallError("read length %d exceeds %d (p=%d, k=%d)"
                                  % (read.length, cfg.m_max, cfg.p, cfg.k))
    build_transitions(read)            # raises DegenerateTransitionError like stage_read
    scores, status, _ = _score_pairs([read], [hap], cfg)
    if (status[0] & _native.ST_KIND_MASK) == _native.ST_OVERFLOW:
        raise NumericOverflowError("accumulator out of range; retry in double precision or with "
                                   "a different scale")
    return Score(float(scores[0]))


def forward_wavefront(read, hap, cfg) -> Score:
    """Score one read/haplotype pair on the GPU engine."""
    return _single(read, hap, cfg)


def forward_wavefront_counted(read, hap, cfg):
    """As forward_wavefront, also returning the step count of the reference's lane-tiled
    schedule, n + p (wavefront.py:314-315, pinned by test_wavefront.py:54-55).  The
    engine's own schedule is reported by engine_wavefront_steps()."""
    score = _single(read, hap, cfg)
    return score, hap.length + cfg.p


def engine_wavefront_steps(m: int, n: int) -> int:
    """Wavefront steps the B200 engine's per-pair tiling executes for an m x n pair:
    (n + P - 1) per stripe for its sub-warp size P."""
    P, _, Q = _native.fast_geometry(int(m), int(n))
    return Q * (n + P - 1)


def forward_wavefront_batch(batches, items, cfg, out, errors=None) -> list:
    """Score ``items`` (WorkItem list) with one config into out[global_id]; failures
    are appended to ``errors`` as (global_id, kind) in item order and leave NaN."""
    if errors is None:
        errors = []
    items = list(items)
    if not items:
        return errors
    reads = [batches[w.batch_index].reads[w.read_index] for w in items]
    haps = [batches[w.batch_index].haps[w.hap_index] for w in items]
    scores, status, _ = _score_pairs(reads, haps, cfg)
    kinds = status & _native.ST_KIND_MASK
    for w, s, k in zip(items, scores.tolist(), kinds.tolist()):
        if k == _native.ST_OK:
            out[w.global_id] = s
        else:
            out[w.global_id] = np.nan
            errors.append((w.global_id, _native.KIND_NAMES[k]))
    return errors

"""Worst relative deviation of the engine from the C oracle (reference-pinned) per workload:
fast FP32 pairs (bar 1e-4) and FP64-retried pairs (bar 1e-9).  GPU required.

usage: python tools/accuracy.py [workload[:batches] ...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_2411_11547_b200 import _native, datagen, default_configs  # noqa: E402
from paper_2411_11547_b200.pipeline import config_tuples  # noqa: E402

F32 = config_tuples(default_configs("f32"))
ctx = _native.Context(0)
for spec in (sys.argv[1:] or ["c1", "c2", "c3", "c4:16", "c4_underflow:8"]):
    name, _, nb = spec.partition(":")
    flat = datagen.workload(name, num_batches=int(nb) if nb else None)
    ofl = oracle.Flat(**flat.as_dict())
    ref32, k32 = oracle.score(ofl, "f32")
    scores, status, stats = ctx.score(flat, F32, _native.FLAG_RETRY_F64)
    kind = status & _native.ST_KIND_MASK
    fast = (k32 == 0) & ((status & (_native.ST_RETRIED_F64 | _native.ST_EXACT_F32)) == 0)
    exact = (k32 == 0) & ((status & _native.ST_EXACT_F32) != 0)
    rel = lambda a, b: np.abs(a - b) / np.abs(b)  # noqa: E731
    line = "%-14s pairs %7d  fast %7d max rel %.2e" % (name, len(scores), fast.sum(),
                                                       rel(scores[fast], ref32[fast]).max() if fast.any() else 0)
    line += "  exact %5d max rel %.1e" % (exact.sum(), rel(scores[exact], ref32[exact]).max() if exact.any() else 0)
    flagged = k32 == 1
    line += "  flag sets equal %s" % np.array_equal((status & _native.ST_RETRIED_F64) != 0, flagged)
    if flagged.any():
        pr, ph = flat.pair_index()
        idx = np.flatnonzero(flagged)
        acc64, st64 = oracle.score_raw(ofl, "f64", 0, pairs=(pr[idx], ph[idx]))
        ref64 = oracle.finish(acc64, st64, 0)
        fin = st64 == 0
        line += "  f64 %6d max rel %.2e" % (idx.size, rel(scores[idx][fin], ref64[fin]).max())
    print(line, flush=True)

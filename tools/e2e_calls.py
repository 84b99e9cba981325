"""Wall time of repeated phmm_score calls (pinned inputs, caller-owned result buffers, like
bench.py's e2e loop); PHMM_TRACE=1 adds the per-chunk host timeline on stderr.

usage: python tools/e2e_calls.py [workload[:num_batches]] [calls] [--retry] [--pipeline=n]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_11547_b200 import _native, datagen, default_configs  # noqa: E402
from paper_2411_11547_b200.pipeline import config_tuples  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "c5"
name, _, nb = spec.partition(":")
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 10
flags = _native.FLAG_RETRY_F64 if "--retry" in sys.argv else 0
flat = bench.pinned_copy(datagen.workload(name, num_batches=int(nb) if nb else None))
cfg = config_tuples(default_configs("f32"))
ctx = _native.Context(0)
for a in sys.argv:
    if a.startswith("--pipeline="):
        ctx.set_pipeline(int(a.split("=", 1)[1]))
res = np.empty(flat.num_pairs, np.float64)
st = np.empty(flat.num_pairs, np.uint8)
for i in range(calls):
    t0 = time.perf_counter()
    _, _, stats = ctx.score(flat, cfg, flags, out=res, status=st)
    dt = time.perf_counter() - t0
    print("%s call %d: %.1f ms  e2e %.0f GCUPS  device span %.1f ms  plan %.1f ms" % (
        name, i, dt * 1e3, stats.total_cells / dt / 1e9, stats.device_ms, stats.plan_ms), file=sys.stderr, flush=True)

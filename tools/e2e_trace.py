"""e2e breakdown: phmm_score from pinned host buffers, PHMM_TRACE phases on stderr.

usage: PHMM_TRACE=1 python tools/e2e_trace.py [workload] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2411_11547_b200 import _native, datagen, default_configs  # noqa: E402
from paper_2411_11547_b200.pipeline import config_tuples  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
flat = bench.pinned_copy(datagen.workload(name))
cfg = config_tuples(default_configs("f32"))
ctx = _native.Context(0)
for i in range(reps):
    t0 = time.perf_counter()
    out, st, stats = ctx.score(flat, cfg, _native.FLAG_RETRY_F64 if "--retry" in sys.argv else 0)
    dt = time.perf_counter() - t0
    print("%s call %d: %.3f ms  e2e %.0f GCUPS  plan %.3f h2d %.3f dev %.3f d2h %.3f" % (
        name, i, dt * 1e3, stats.total_cells / dt / 1e9, stats.plan_ms, stats.h2d_ms, stats.device_ms, stats.d2h_ms),
        file=sys.stderr, flush=True)

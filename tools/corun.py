"""Co-scheduling experiment: an FP32-stream workload and an FP64 workload on two contexts
(two streams), alone and concurrently; PHMM_OCC_CAP caps CTAs per SM for both.

usage: PHMM_OCC_CAP=1 python tools/corun.py [reps]
"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_11547_b200 import _native, datagen, default_configs  # noqa: E402
from paper_2411_11547_b200.pipeline import config_tuples  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
a = _native.Context(0)
b = _native.Context(0)
f32 = datagen.workload("c2")                                     # k_stream<kFast32,16,16>
f64 = datagen.generate_synthetic_flat(512, 16, 4, 250, 250, 7, mode="derived")   # exact FP64 (32,8)
a.prepare(f32, config_tuples(default_configs("f32")), 0)
b.prepare(f64, config_tuples(default_configs("f64")), 0)
import torch  # noqa: E402


def loop(ctx, n, out):
    t0 = time.perf_counter()
    for _ in range(n):
        ctx.execute()
    out.append(time.perf_counter() - t0)


for c in (a, b):
    c.execute()
res = {}
for name, ctxs in (("fp32 alone", [a]), ("fp64 alone", [b]), ("both", [a, b])):
    outs = [[] for _ in ctxs]
    th = [threading.Thread(target=loop, args=(c, reps, o)) for c, o in zip(ctxs, outs)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    wall = time.perf_counter() - t0
    res[name] = wall
    print("%-11s wall %.2f ms per rep  (threads %s)" % (name, wall / reps * 1e3,
          ", ".join("%.2f" % (o[0] / reps * 1e3) for o in outs)))
print("overlap efficiency: serial %.2f ms vs concurrent %.2f ms" % (
    (res["fp32 alone"] + res["fp64 alone"]) / reps * 1e3, res["both"] / reps * 1e3))

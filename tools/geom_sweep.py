"""Tiling sweep: device time of the fast kernel on one workload per forced geometry.

usage: python tools/geom_sweep.py c2 16x16 32x8 8x16 ...
Each geometry runs in a fresh process (PHMM_FAST_GEOM is read once per process); scores
are compared with the default tiling's (must agree to 1e-5 relative).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
from paper_2411_11547_b200 import _native, datagen, default_configs
from paper_2411_11547_b200.pipeline import config_tuples
flat = datagen.workload(%r)
ctx = _native.Context(0)
cells = None
ctx.prepare(flat, config_tuples(default_configs("f32")), 0)
ts = []
for i in range(6):
    ctx.execute()
    d, f, n = ctx.last_timing()
    if i >= 1: ts.append((d, f))
s, st, stats = ctx.fetch()
np.save("/tmp/geom_scores.npy", s)
print(json.dumps({"device_ms": float(np.median([t[0] for t in ts])), "fast_ms": float(np.median([t[1] for t in ts])),
                  "cells": int(stats.total_cells), "computed": int(stats.computed_cells)}))
'''


def run(wl, geom):
    env = dict(os.environ)
    if geom != "auto":
        env["PHMM_FAST_GEOM"] = geom
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, wl)], env=env, capture_output=True, text=True)
    if out.returncode != 0:
        return {"error": out.stderr[-400:]}
    import numpy as np
    res = json.loads(out.stdout.strip().splitlines()[-1])
    res["scores"] = np.load("/tmp/geom_scores.npy")
    return res


if __name__ == "__main__":
    import numpy as np
    wl = sys.argv[1]
    base = run(wl, "auto")
    print("auto: fast %.3f ms  device %.3f ms  GCUPS(fast) %.0f" % (base["fast_ms"], base["device_ms"], base["cells"] / base["fast_ms"] / 1e6))
    for g in sys.argv[2:]:
        r = run(wl, g)
        if "error" in r:
            print(g, "ERROR", r["error"])
            continue
        ok = np.isfinite(base["scores"])
        rel = np.max(np.abs(r["scores"][ok] - base["scores"][ok]) / np.abs(base["scores"][ok])) if ok.any() else 0
        print("%-6s fast %.3f ms  device %.3f ms  GCUPS(fast) %.0f  computed/true %.3f  max rel vs auto %.1e"
              % (g, r["fast_ms"], r["device_ms"], r["cells"] / r["fast_ms"] / 1e6, r["computed"] / r["cells"], rel))

import sys, os, subprocess, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2411_11547_b200 import _native, default_configs
from paper_2411_11547_b200.pipeline import config_tuples
import test_gpu_stream as T
F32 = config_tuples(default_configs("f32"))
rng = np.random.default_rng(5)
cases = {
  "1x1": [([100], [150], "derived")],
  "1x2": [([100], [150, 150], "derived")],
  "1x3": [([100], [150, 140, 130], "derived")],
  "m20": [([20], [50], "derived")],
  "m250": [([250], [300], "derived")],
}
mode = sys.argv[1] if len(sys.argv) > 1 else "run"
eng = _native.context(0)
out = {}
for name, spec in cases.items():
    flat = T._flat(np.random.default_rng(7), spec)
    s, st, stats = eng.score(flat, F32, _native.FLAG_EXACT)
    out[name] = s
np.savez("/tmp/dbg_%s.npz" % os.environ.get("PHMM_NO_STREAM", "0"), **out)

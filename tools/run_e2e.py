import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2411_11547_b200 import datagen, default_configs, run
cfg = default_configs("f32")
for name in ("c3", "c2", "c3"):
    kw = dict(datagen.WORKLOADS[name]); batches = datagen.generate_synthetic(**kw)
    run(batches, cfg)
    ts = []
    for _ in range(8):
        t0 = time.perf_counter(); _, rep = run(batches, cfg); ts.append(time.perf_counter() - t0)
    print(name, "run() ms: %s  gcups(median) %.0f" % (" ".join("%.1f" % (t * 1e3) for t in ts), rep.total_cells / np.median(ts) / 1e9))

"""Wall time of the stages of the drop-in pipeline.run(list[Batch]) on c2 / c3: native
flattening into the page-locked arena, budget check, engine call, per-config accounting.

usage: python tools/run_stages.py [workload] [reps]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_11547_b200 import datagen, default_configs, pipeline  # noqa: E402
from paper_2411_11547_b200.model import FlatBatches  # noqa: E402
from paper_2411_11547_b200.partition import check_budget  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
batches = datagen.generate_synthetic(**dict(datagen.WORKLOADS[name]))
cfg = default_configs("f32")
pipeline.run(batches, cfg)
rows = []
for _ in range(reps):
    t = [time.perf_counter()]
    flat = FlatBatches.from_batches(batches, pipeline._arena())
    t.append(time.perf_counter())
    check_budget(flat, cfg, pipeline.DEFAULT_BUDGET_BYTES)
    t.append(time.perf_counter())
    scores, status, stats = pipeline.score_flat(flat, cfg, False, False, 0, None)
    t.append(time.perf_counter())
    pipeline._config_cells(flat, cfg, status, 1e-3)
    pipeline.errors_from_status(status)
    t.append(time.perf_counter())
    _, rep = pipeline.run(batches, cfg)
    t.append(time.perf_counter())
    rows.append(np.diff(t) * 1e3)
med = np.median(np.array(rows), axis=0)
print("%s: flatten %.2f  budget %.2f  score %.2f  accounting %.2f  | run() %.2f ms" % ((name,) + tuple(med)))

# c5 (10M pairs) end to end through phmm_score (pinned inputs), pipelined vs one pass
python - <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import bench
from paper_2411_11547_b200 import _native, datagen, default_configs
from paper_2411_11547_b200.pipeline import config_tuples
flat = bench.pinned_copy(datagen.workload("c5"))
cfg = config_tuples(default_configs("f32"))
ctx = _native.Context(0)
for flags, name in ((_native.FLAG_RETRY_F64, "retry"),):
    for i in range(3):
        t0 = time.perf_counter()
        out, st, stats = ctx.score(flat, cfg, flags)
        dt = time.perf_counter() - t0
        print("c5 %s call %d: %.1f ms  e2e %.0f GCUPS  plan %.1f ms" % (name, i, dt * 1e3, stats.total_cells / dt / 1e9, stats.plan_ms), flush=True)
PY

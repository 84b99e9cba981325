"""Run the engine on one workload for profiling: prepare, warm execute, then N executes.

usage: python tools/profile_run.py [workload[:num_batches]] [num_executes] [--retry] [--exact]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_11547_b200 import _native, datagen, default_configs  # noqa: E402
from paper_2411_11547_b200.pipeline import config_tuples  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "c2"
name, _, nb = spec.partition(":")          # "c5:2442" = the first 2442 batches of c5
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
flags = (_native.FLAG_RETRY_F64 if "--retry" in sys.argv else 0) | (_native.FLAG_EXACT if "--exact" in sys.argv else 0)
flat = datagen.workload(name, num_batches=int(nb) if nb else None)
ctx = _native.Context(0)
ctx.prepare(flat, config_tuples(default_configs("f32")), flags)
for _ in range(reps):
    ctx.execute()
    print("%s device %.3f ms fast %.3f ms launches %d" % ((name,) + ctx.last_timing()))
_, _, st = ctx.fetch()
print({k: v for k, v in st.as_dict().items()})

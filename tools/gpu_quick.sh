# GPU check of a kernel change: the -m gpu suite, then a short bench (c5 headline + c2/c3/c4)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_quick.json"))
print(round(d["value"], 1), round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 1),
      {k: round(v, 2) for k, v in d["roofline"]["phases_ms"].items()}, round(d["roofline"]["frac"], 4))
for s in d["secondary"]:
    print(s["workload"][:3], round(s["gcups"]), round(s["device_ms"], 3), s.get("flags"), round(s["fp32_phase_gcups"]))
PY

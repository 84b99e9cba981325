timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value',d['value'],'fast',d['roofline']['achieved'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'], 'c3', d['secondary'][0]['gcups'], d['secondary'][0]['fast_ms'])"

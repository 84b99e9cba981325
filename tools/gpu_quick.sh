timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value',round(d['value']),'fast',round(d['roofline']['achieved']),'frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value']), 'c3', round(d['secondary'][0]['gcups']), d['secondary'][0]['fast_ms'], d['secondary'][0]['device_ms'], 'engine', d['engine'])"
for W in ${PROFILE_WORKLOADS:-}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_${W}.csv python tools/profile_run.py $W 2 --retry > gpurun_out/launches_${W}.log 2>&1
  python tools/launches.py gpurun_out/launches_${W}.csv
done

# scratch GPU session used during development: parity tests, c2/c3 timings, c3 launch list
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
for i in 1 2; do python tools/profile_run.py c2 4 | tail -2 | head -1; python tools/profile_run.py c3 4 --retry | tail -2 | head -1; done
python tools/profile_run.py c3 1 --retry | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py c3 2 --retry > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c3.csv

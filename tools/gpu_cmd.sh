# scratch GPU session used during development: A/B timings, parity tests, c3 launch list
AB_VARIANTS="PHMM_NO_STREAM=0" AB_NOTEST=1 bash tools/ab.sh
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py c3 2 --retry > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c3.csv

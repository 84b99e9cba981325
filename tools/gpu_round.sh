# one GPU session: smoke, GPU tests, bench, launch list (+ optional ncu capture)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
for W in ${PROFILE_WORKLOADS:-c2}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_${W}.csv python tools/profile_run.py $W 2 --retry > gpurun_out/launches_${W}.log 2>&1
done
if [ -n "$NCU_FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_stream<.int.0," -s 1 -c 1 \
     -o gpurun_out/prof_kstream_c2 python tools/profile_run.py c2 2 > gpurun_out/prof_c2.log 2>&1
fi
ls gpurun_out

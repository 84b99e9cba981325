# one GPU iteration: parity suite, c5 e2e timeline, device timings (c5/c3/c2/c4)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
PHMM_TRACE=1 timeout 300 python tools/e2e_trace.py c5 3 --retry 2>&1 | grep -E "chunk|call|prepare\]" | tail -14
for W in "c5 3 --retry" "c3 6 --retry" "c2 6" "c4 4 --retry"; do
  timeout 600 python tools/profile_run.py $W 2>&1 | grep -v "^{" | tail -2
done
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi

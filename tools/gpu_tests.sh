# GPU session: smoke + the -m gpu suite (+ optional extra command in $EXTRA)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu.log
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi

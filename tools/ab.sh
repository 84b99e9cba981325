# A/B timing of the engine on c2/c3 (device/fast ms per execute) + GPU parity tests
for W in ${AB_WORKLOADS:-c2 c3}; do
  for V in ${AB_VARIANTS:?set AB_VARIANTS to the env settings to compare}; do
    echo "== $W $V"; env $V timeout 300 python tools/profile_run.py $W 4 --retry 2>&1 | tail -3
  done
done
if [ -z "$AB_NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
  tail -15 gpurun_out/pytest_gpu.log
fi

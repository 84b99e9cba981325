# quick A/B timing on the GPU: engine device/FP32-phase time for c5 (retry), c2, c3, c4
for W in ${PERF_WORKLOADS:-"c5 3 --retry" "c2 6" "c3 6 --retry" "c4 4 --retry"}; do
  timeout 600 python tools/profile_run.py $W 2>&1 | grep -v "^{" | tail -2
done

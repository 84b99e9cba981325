# ncu --set full captures (source-level) of the c5 top FP32 bin and the FP64 retry kernel
for K in ${KERNELS:-"0, 16, 14, 0" "1, 32, 8, 0"}; do
  tag=$(echo "$K" | tr -d ' ' | tr ',' '_')
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_stream<$K>" -s ${SKIP:-0} -c 1 \
     -o gpurun_out/prof_c5_$tag python tools/profile_run.py ${WL:-c5} 1 --retry > gpurun_out/prof_c5_$tag.log 2>&1
  echo "ncu $tag rc=$?"; tail -2 gpurun_out/prof_c5_$tag.log
done

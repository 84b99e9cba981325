# ncu --set full captures (source-level) of the c5 top FP32 bin and the FP64 retry kernel
# KERNELS: "MODE,P,K" triples (demangled k_stream<(int)MODE, (int)P, (int)K, (bool)0>)
for K in ${KERNELS:-"0,16,14" "1,32,8"}; do
  IFS=, read MODE P KK <<< "$K"
  tag="${MODE}_${P}_${KK}"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k "regex:k_stream<.int.$MODE, .int.$P, .int.$KK, .bool.0>" -s ${SKIP:-0} -c 1 \
     -o gpurun_out/prof_${WL:-c5}_$tag python tools/profile_run.py ${WL:-c5} 1 --retry > gpurun_out/prof_${WL:-c5}_$tag.log 2>&1
  echo "ncu $tag rc=$?"; tail -2 gpurun_out/prof_${WL:-c5}_$tag.log
done

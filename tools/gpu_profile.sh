# ncu launch list + full capture of the top kernel (one GPU, one process)
set -x
W=${1:-c2}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_${W}.csv python tools/profile_run.py $W 2 ${2:-} > gpurun_out/launches_${W}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_stream<.int.0," -s 1 -c 1 \
   -o gpurun_out/prof_kstream_${W} python tools/profile_run.py $W 2 ${2:-} > gpurun_out/prof_${W}.log 2>&1
ls -la gpurun_out

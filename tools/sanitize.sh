# compute-sanitizer memcheck / racecheck / synccheck on a reduced GPU test subset that
# covers every k_stream mode: single-stripe units (event windows, empty lanes, split
# units), striped team + sequential modes with the cp.async column ring and the
# shared-memory progress flags, ring-buffered row codes, device-built retry units,
# the per-pair post-pass kernels and k_matrices.  Logs under gpurun_out/.
SUB="tests/test_gpu_stream.py::test_tiny_haplotypes_overlapping_windows tests/test_gpu_stream.py::test_single_haplotype_batches_empty_lane tests/test_gpu_stream.py::test_many_haplotypes_split_units_and_unbalanced_lanes tests/test_gpu_stream.py::test_long_reads_striped_team_and_sequential_modes tests/test_gpu_stream.py::test_partial_underflow_units_and_degenerate_reads tests/test_gpu_stream.py::test_long_haplotypes_ring_mode_all_modes tests/test_gpu_api.py::test_forward_matrices_bit_identical_to_reference"
for TOOL in ${TOOLS:-memcheck racecheck synccheck}; do
  EXTRA_OPTS=""
  [ "$TOOL" = "memcheck" ] && EXTRA_OPTS="--leak-check no"
  [ "$TOOL" = "racecheck" ] && EXTRA_OPTS="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $TOOL $EXTRA_OPTS --print-limit 100000 --show-backtrace no \
     --log-file gpurun_out/sanitize_${TOOL}.log \
     python -m pytest $SUB -x -q -p no:cacheprovider > gpurun_out/sanitize_${TOOL}_pytest.log 2>&1
  echo "$TOOL rc=$?"
  tail -3 gpurun_out/sanitize_${TOOL}_pytest.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_${TOOL}.log | tail -3
  # distinct hazard / error sites (kernel, source line) with counts
  grep -E "(Write|Read) Thread|Invalid|at .* in .*:[0-9]+" gpurun_out/sanitize_${TOOL}.log \
    | sed -E 's/Thread \([0-9,]+\)//; s/\+0x[0-9a-f]+//; s/block \([0-9,]+\)//' | sort | uniq -c | sort -rn \
    > gpurun_out/sanitize_${TOOL}_sites.txt
  head -20 gpurun_out/sanitize_${TOOL}_sites.txt
  if [ $(stat -c %s gpurun_out/sanitize_${TOOL}.log) -gt 4000000 ]; then
    head -c 2000000 gpurun_out/sanitize_${TOOL}.log > gpurun_out/sanitize_${TOOL}.head.log
    tail -c 200000 gpurun_out/sanitize_${TOOL}.log > gpurun_out/sanitize_${TOOL}.tail.log
    rm gpurun_out/sanitize_${TOOL}.log
  fi
done

for mode in 0 1; do
  echo "PHMM_BAND_SERIAL=$mode"
  PHMM_BAND_SERIAL=$mode python tools/profile_run.py c2 6 | head -6
  PHMM_BAND_SERIAL=$mode python tools/profile_run.py c3 4 --retry | head -4
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_run.py c2 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c2.csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_run.py c3 2 --retry > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c3.csv

for U in 2 3 4 6 8; do
  echo "== PHMM_LANE_UNITS=$U"
  for W in "c3 6 --retry" "c3 6" "c2 6" "c4 4 --retry"; do
    PHMM_LANE_UNITS=$U timeout 300 python tools/profile_run.py $W 2>&1 | grep -v "^{" | tail -1
  done
done

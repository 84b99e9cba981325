# e2e of c5 through phmm_score for several chunk weightings (PHMM_CHUNK_WEIGHTS)
for W in ${WEIGHTS:-"1,2,2,2,1" "1,3,4,4,3,1" "1,2,4,4,4,1" "1,4,6,4,1" "1,3,4,4,4" "1,2,3,3,3,2,1"}; do
  echo "== $W"
  PHMM_CHUNK_WEIGHTS=$W timeout 300 python tools/e2e_calls.py c5 8 --retry 2>&1 | tail -6 | awk '{print $4}' | tr '\n' ' '; echo
done

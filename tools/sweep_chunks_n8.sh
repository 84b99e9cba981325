# e2e of the per-GPU share of c5 at N = 8 (1.25M pairs) and N = 4 (2.5M) through phmm_score
# for several ramped chunk weightings
for NB in ${NBS:-2442 4883}; do
 for W in ${WEIGHTS:-"1,3,5,5,3,1" "1,2,2,1" "1,3,3,1" "1,4,4,1" "1,2,4,2,1" "1,4,1" "1,2,1" "1,3,5,3,1"}; do
  echo "== c5:$NB $W $(PHMM_CHUNK_WEIGHTS=$W timeout 300 python tools/e2e_calls.py c5:$NB 8 --retry 2>&1 | tail -5 | awk '{printf "%s/%s ", $4, $10}')"
 done
done

# e2e of the small calls (c2, c3) through phmm_score, one pass vs ramped chunk weightings
# (--pipeline=n enables chunking for calls below 2^20 pairs; PHMM_CHUNK_WEIGHTS sets the ramp)
for WL in ${WLS:-c2 c3}; do
 for W in ${WEIGHTS:-"NOCHUNK" "1,1" "1,2" "1,3" "1,2,2" "1,2,3" "1,3,3" "1,2,2,1" "1,3,5" "1,4,4,2"}; do
  if [ "$W" = "NOCHUNK" ]; then V="NOCHUNK=1"; P=1; else V="PHMM_CHUNK_WEIGHTS=$W"; P=$(echo $W | tr ',' '\n' | wc -l); fi
  echo "== $WL $V $(env $V timeout 300 python tools/e2e_calls.py $WL 12 --pipeline=$P $( [ "$WL" = c3 ] && echo --retry) 2>&1 | tail -8 | awk '{printf "%s ", $4}')"
 done
done

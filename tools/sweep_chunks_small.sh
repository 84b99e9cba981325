# e2e of the small calls (c2, c3) through phmm_score for several chunk weightings
for WL in "c2" "c3"; do
 for W in "1,1,1" "1,2" "1,3" "1,2,2" "1,2,3" "NOCHUNK"; do
  if [ "$W" = "NOCHUNK" ]; then V="NOCHUNK=1"; else V="PHMM_CHUNK_WEIGHTS=$W"; fi
  echo "== $WL $V $(env $V timeout 300 python tools/e2e_calls.py $WL 10 $([ "$V" = NOCHUNK=1 ] && echo --pipeline=1) $( [ "$WL" = c3 ] && echo --retry) 2>&1 | tail -6 | awk '{printf "%s ", $4}')"
 done
done

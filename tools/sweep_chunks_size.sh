for NB in 2442 4883 9766; do
 for W in "1,1,1" "1,2,2,2,1" "1,3,4,4,3,1" "NOCHUNK"; do
  if [ "$W" = "NOCHUNK" ]; then V="NOCHUNK=1"; else V="PHMM_CHUNK_WEIGHTS=$W"; fi
  echo "== c5:$NB $V $(env $V timeout 300 python tools/e2e_calls.py c5:$NB 6 --retry $([ "$V" = NOCHUNK=1 ] && echo --pipeline=1) 2>&1 | tail -4 | awk '{printf "%s/%s ", $4, $10}')"
 done
 echo "   device one-pass: $(timeout 300 python tools/profile_run.py c5 2 --retry 2>&1 | head -0)"
done

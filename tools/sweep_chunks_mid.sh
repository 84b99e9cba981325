for NB in 256 512 1024; do
 for V in "PHMM_CHUNK_WEIGHTS=1,3,4,4,3,1" "PHMM_CHUNK_WEIGHTS=1,2,2,1" "NOCHUNK=1"; do
  echo "== c5:$NB $V $(env $V timeout 300 python tools/e2e_calls.py c5:$NB 8 --retry $([ "$V" = NOCHUNK=1 ] && echo --pipeline=1) 2>&1 | tail -5 | awk '{printf "%s ", $4}')"
 done
done

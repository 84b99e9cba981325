# e2e A/B of c5 through phmm_score: default vs an env setting ($AB)
for V in "X=1" "${AB:?set AB}" "X=1" "$AB"; do
  echo "== $V"; env $V timeout 300 python tools/e2e_calls.py c5 8 --retry 2>&1 | tail -7 | awk '{print $4, $10}' | tr '\n' ' '; echo
done

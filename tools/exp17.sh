for rep in 1 2; do for cps in 2 4 8; do for c in c2 c5; do
  echo "cps=$cps $c $(PG_COMMIT_PER_SM=$cps timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -1)"
done; done; done

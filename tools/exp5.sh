for rep in 1 2; do
for mb in 1 4 16 1000000; do
for c in c2 c5; do
  echo "mark_batch=$mb $c $(PG_MARK_BATCH=$mb timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -1)"
done; done; done

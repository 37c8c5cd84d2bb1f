for rep in 1 2 3; do for mb in 0 34 40; do
  echo "persist=$mb c2 $(PG_L2_PERSIST_MB=$mb timeout 300 python tools/prof_round.py --config c2 --reps 5 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
done; done

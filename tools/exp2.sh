for g in 16 32; do
  for c in c5 c2; do
    echo "gather=$g $c $(PG_SELL_GATHER=$g timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
  done
done

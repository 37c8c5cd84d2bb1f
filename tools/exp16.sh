for rep in 1 2; do for g in 16 32 8; do
  echo "gather=$g c3 $(PG_SELL_GATHER=$g timeout 300 python tools/prof_round.py --config c3 --reps 3 --debug-flags 0x1000 --solve 2>&1 | tail -2 | tr '\n' ' ')"
done; done

for rep in 1 2; do for l in build/var/*.so; do for c in c5 c2; do
  echo "$(basename $l) $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -1)"
done; done; done

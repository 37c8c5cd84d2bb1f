for rep in 1 2 3; do for l in build/var/*.so; do for c in c2 c5 c3; do
  wl=--worklist; [ $c = c3 ] && wl=
  echo "$(basename $l) $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags 0x1000 --solve $wl 2>&1 | tail -2 | tr '\n' ' ')"
done; done; done

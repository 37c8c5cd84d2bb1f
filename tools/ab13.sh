#!/usr/bin/env bash
# A/B of library variants under build/var: first-round kernel time and best
# full solve (C2/C5 with the worklist as in the bench, C3 dense), two passes
for rep in 1 2; do
for l in build/var/*.so; do
  for c in ${CONFIGS:-c2 c5 c3}; do
    wl=--worklist; [ $c = c3 ] && wl=
    echo "$(basename $l) $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --debug-flags 0x1000 --reps 10 --solve $wl 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
done

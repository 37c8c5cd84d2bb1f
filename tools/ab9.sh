#!/usr/bin/env bash
# A/B of library variants (build/var/*.so) on full solves: worklist C2/C5, C3, C1
for rep in 1 2; do
for v in build/var/*.so; do
  for c in c2 c5 c3 c1; do
    echo "$(basename $v) $c $(PG_LIB=$v timeout 300 python tools/prof_round.py --config $c --reps 3 --solve $( [ $c != c3 ] && [ $c != c1 ] && echo --worklist ) 2>&1 | tail -1)"
  done
done
done

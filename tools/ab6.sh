#!/usr/bin/env bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -1
for rep in 1 2; do
for l in build/var/*.so; do
  for c in ${CONFIGS:-c2 c5 c3}; do
    echo "$l $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --reps 10 --solve $( [ $c != c3 ] && echo --worklist ) 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
done

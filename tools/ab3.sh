#!/usr/bin/env bash
# A/B on one box: per variant, C2 first-round kernels and best-of-3 solves (+ C5, C3)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -k "not c3 and not c4 and not c5" 2>&1 | tail -1
for rep in 1 2; do
for l in build/var/*.so; do
  for c in ${CONFIGS:-c2 c5}; do
    echo "$l $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --reps 10 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
done

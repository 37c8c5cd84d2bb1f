#!/usr/bin/env bash
# A/B timing of library variants under build/var (GPU box): parity tests with
# the in-tree library, then per variant the first-round kernels and the best
# of 3 full solves for C2/C3/C1, and the C2 first round without phase 2
# (variants built with -DPG_SELL_DEBUG=1).
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for l in build/var/*.so; do
  for c in ${CONFIGS:-c2 c3 c1}; do
    echo "$l $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --debug-flags 0x1000 --reps 5 --solve 2>&1 | tail -2 | tr '\n' ' ')"
  done
  echo "$l c2 nophase2 $(PG_LIB=$l timeout 300 python tools/prof_round.py --config c2 --debug-flags 0x10000 --reps 5 2>&1 | tail -1)"
done

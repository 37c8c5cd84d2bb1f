#!/usr/bin/env bash
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "FAILED|Error|passed|failed" | tail -8
for rep in 1 2; do
for k in 0 1; do
  for c in c2 c5 c3 c1; do
    echo "kind_if=$k $c $(PG_KIND_IF=$k timeout 300 python tools/prof_round.py --config $c --reps 3 --solve $( [ $c != c3 ] && [ $c != c1 ] && echo --worklist ) 2>&1 | tail -1)"
  done
done
done

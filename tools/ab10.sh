#!/usr/bin/env bash
# A/B of the round-kind heuristics: PG_DENSE_DIV x PG_DENSE_DEG x PG_LIST_GATE x PG_WL_WEIGHTS
for rep in 1 2; do
for spec in "4 1e30 1 2,4,2,1" "1 1 1 8,32,2,1" "1 0.7 1 8,32,2,1" "1 1.5 1 8,32,2,1" "2 1 1 8,32,2,1" "0.5 1 1 8,32,2,1"; do
  set -- $spec
  for c in c2 c5; do
    echo "div=$1 deg=$2 gate=$3 w=$4 $c $(PG_DENSE_DIV=$1 PG_DENSE_DEG=$2 PG_LIST_GATE=$3 PG_WL_WEIGHTS=$4 timeout 300 python tools/prof_round.py --config $c --reps 3 --solve --worklist 2>&1 | tail -1)"
  done
done
done

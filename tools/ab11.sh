#!/usr/bin/env bash
# variants x round-kind heuristics (PG_DENSE_DIV PG_DENSE_DEG PG_LIST_GATE PG_WL_WEIGHTS)
for rep in 1 2; do
for v in build/var/*.so; do
for spec in "4 1e30 1 2,4,2,1" "1 0.5 1 8,32,2,1" "1 0.15 1 8,32,2,1"; do
  set -- $spec
  for c in c2 c5; do
    echo "$(basename $v) div=$1 deg=$2 gate=$3 w=$4 $c $(PG_LIB=$v PG_DENSE_DIV=$1 PG_DENSE_DEG=$2 PG_LIST_GATE=$3 PG_WL_WEIGHTS=$4 timeout 300 python tools/prof_round.py --config $c --reps 3 --solve --worklist 2>&1 | tail -1)"
  done
done
done
done

#!/usr/bin/env bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -1
for rep in 1 2; do
for hy in 0 1; do
  for c in c2 c5; do
    echo "hybrid=$hy $c $(PG_HYBRID=$hy timeout 300 python tools/prof_round.py --config $c --reps 3 --solve --worklist 2>&1 | tail -1)"
  done
done
done

#!/usr/bin/env bash
# A/B: parity subset with the in-tree library, then per variant the first-round kernel time and best-of-3 solves
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -k "not c3 and not c4 and not c5" 2>&1 | tail -2
for l in build/var/*.so; do
  for c in ${CONFIGS:-c2}; do
    echo "$l $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --debug-flags 0x1000 --reps 10 --solve 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
if [ -f build/var/dbg.so ]; then
  for f in 0x10000 0x40000; do echo "dbg c2 flags $f $(PG_LIB=build/var/dbg.so timeout 300 python tools/prof_round.py --config c2 --debug-flags $f --reps 10 2>&1 | tail -1)"; done
fi

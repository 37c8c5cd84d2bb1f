for mb in 0 64 96; do
  for c in c5 c2; do
    echo "persist=$mb $c $(PG_L2_PERSIST_MB=$mb timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
for f in 0x1000 0x10000 0x40000; do
  for c in c5 c2; do
    echo "dbg $f $c $(PG_LIB=build/var/dbg.so timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags $f 2>&1 | tail -1)"
  done
done

timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do
for c in c5 c2 c3; do
  wl=--worklist; [ $c = c3 ] && wl=
  echo "default $c $(timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve $wl 2>&1 | tail -2 | tr '\n' ' ')"
done
for mb in 16 32; do
  echo "persist=$mb c2 $(PG_L2_PERSIST_MB=$mb timeout 300 python tools/prof_round.py --config c2 --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
done
echo "persist=0 c5 $(PG_L2_PERSIST_MB=0 timeout 300 python tools/prof_round.py --config c5 --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
done

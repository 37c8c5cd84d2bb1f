timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do
for p in 1 0; do
for c in c2 c5 c3 c1; do
  wl=--worklist; [ $c = c3 ] && wl=; [ $c = c1 ] && wl=
  echo "pdl=$p $c $(PG_PDL=$p timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve $wl 2>&1 | tail -1)"
done; done; done

for rep in 1 2; do
for l in build/var/*.so; do for c in c5 c2; do
  echo "$(basename $l) $c $(PG_LIB=$l timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
done; done
for mb in 40 64; do
  echo "persist=$mb c5 $(PG_L2_PERSIST_MB=$mb PG_LIB=build/var/a_base.so timeout 300 python tools/prof_round.py --config c5 --reps 3 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
done
done

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do
for f in 1 0; do
for c in c2 c3 c1; do
  wl=--worklist; [ $c = c3 ] && wl=; [ $c = c1 ] && wl=
  echo "fuse=$f $c $(PG_FUSE_SPLIT=$f timeout 300 python tools/prof_round.py --config $c --reps 3 --debug-flags 0x1000 --solve $wl 2>&1 | tail -2 | tr '\n' ' ')"
done; done; done

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do
for c in c2 c5 c3; do
  wl=--worklist; [ $c = c3 ] && wl=
  echo "$c $(timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags 0x1000 --solve $wl 2>&1 | tail -2 | tr '\n' ' ')"
done
done

#!/usr/bin/env bash
# persisting-L2 window over the gathered bounds (PG_L2_PERSIST_MB) on C5 / C2 / C3
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p.name, 'L2', p.L2_cache_size>>20, 'MB')"
for rep in 1 2; do
for mb in 0 40 64 80 96; do
  for c in c5 c2 c3; do
    echo "persist=$mb $c $(PG_L2_PERSIST_MB=$mb timeout 300 python tools/prof_round.py --config $c --reps 3 --solve $( [ $c != c3 ] && echo --worklist ) 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
done

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -3
for rep in 1 2; do
for g in 16 def; do
  for c in c5; do
    if [ $g = def ]; then unset PG_SELL_GATHER; else export PG_SELL_GATHER=$g; fi
    echo "gather=$g $c $(timeout 300 python tools/prof_round.py --config $c --reps 5 --debug-flags 0x1000 --solve --worklist 2>&1 | tail -2 | tr '\n' ' ')"
  done
done
done
unset PG_SELL_GATHER
python -c "
import sys; sys.path.insert(0,'.')
from instances import generators as G
from paper_2009_07785_b200.engine import Session
with Session(G.config_instance('c5')) as s: print(s.info())"

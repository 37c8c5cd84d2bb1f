#!/usr/bin/env bash
# quick GPU iteration: parity subset, kernel timing, bench C2, optional ncu of k_sell
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -k "${PYTEST_K:-not c3 and not c4 and not c5}" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_${TAG}.log
for c in ${CONFIGS:-c2}; do timeout 300 python tools/prof_round.py --config $c --reps 20 2>&1 | tail -1; done
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_${TAG}.json').read().strip().splitlines()[-1]); print('value',d['value'],'parity',d['parity'],'roofline',d['roofline']['achieved'],d['roofline']['frac'],d['roofline']['launch_us'],'e2e',d['e2e']['value'])"
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu=$?"
fi

#!/usr/bin/env bash
# round-2 GPU pass: tests (incl. full-size parity), bench, optional ncu
TAG=${1:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_${TAG}.log
[ "$2" = "tests" ] && exit 0
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench=$?"; tail -1 gpurun_out/bench_${TAG}.json | cut -c1-300
if [ "$2" = "ncu" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_sell=$?"
fi

#!/usr/bin/env bash
# One GPU-box pass: parity tests, a short bench, optional ncu of k_tiles.
# usage: tools/gpu_check.sh [tag] [ncu]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.log 2>&1; echo "bench=$?"; tail -2 gpurun_out/bench_${TAG}.log | cut -c1-1500
if [ "$2" = "ncu" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 1 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu=$?"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python tools/prof_round.py --reps 2 --solve --host-loop > /dev/null 2>&1; echo "launches=$?"
fi

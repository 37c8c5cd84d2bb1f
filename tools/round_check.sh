#!/usr/bin/env bash
# One GPU-box pass: build check, parity tests, bench C2, ncu launch list of the
# bench command, one `ncu --set full` capture of the dominant kernel (k_tiles).
# usage: tools/round_check.sh TAG [noprof]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench=$?"; tail -1 gpurun_out/bench_${TAG}.json | cut -c1-600
[ "$2" = "noprof" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/launches_${TAG}.log 2>&1; echo "launches=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 2 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_tiles=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_round -s 2 -c 1 -o gpurun_out/profr_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncur_${TAG}.log 2>&1; echo "ncu_round=$?"

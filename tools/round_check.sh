#!/usr/bin/env bash
# One GPU-box pass: parity tests, smoke, bench C2, ncu launch list of the
# bench command (host loop: ncu cannot see kernel nodes of conditional graphs),
# one `ncu --set full` capture of the dominant kernel (k_sell), all configs.
# usage: tools/round_check.sh TAG [noprof|all]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench=$?"; tail -1 gpurun_out/bench_${TAG}.json | cut -c1-400
[ "$2" = "noprof" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --loop host > gpurun_out/launches_${TAG}.log 2>&1; echo "launches=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_sell=$?"
if [ "$2" = "all" ]; then
  for c in c1 c3 c4 c5; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "$c rc=$?"; tail -1 gpurun_out/bench_${TAG}_$c.json | cut -c1-300
  done
  timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_${TAG}_ref.json | cut -c1-300
fi

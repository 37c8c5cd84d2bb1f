#!/usr/bin/env bash
# Final evidence pass (one B200): GPU tests, smoke, parity report, bench C2,
# the reference arm, every config with the geomean, Narrow32 lines, launch
# lists (C2, C5; host loop) and ncu --set full captures of k_sell (C2, C5).
TAG=${1:-r2g}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/pytest_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke=$?"
timeout 900 python tools/parity_report.py gpurun_out/parity_${TAG}.json > gpurun_out/parity_${TAG}.log 2>&1; echo "parity=$?"
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo "bench c2=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err; echo "bench ref=$?"
timeout 1800 python bench.py --config all --steps 5 > gpurun_out/bench_${TAG}_all.json 2> gpurun_out/bench_${TAG}_all.err; echo "bench all=$?"
for c in c2 c3; do timeout 600 python bench.py --config $c --scalar f32 --steps 3 > gpurun_out/bench_${TAG}_f32_$c.json 2> gpurun_out/bench_${TAG}_f32_$c.err; echo "f32 $c=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --loop host > gpurun_out/launches_${TAG}.log 2>&1; echo "launches=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_${TAG}_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --loop host > gpurun_out/launches_${TAG}_c5.log 2>&1; echo "launches_c5=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_${TAG} python tools/prof_round.py --reps 3 > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu_sell=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sell -s 2 -c 1 -o gpurun_out/prof_${TAG}_c5 python tools/prof_round.py --config c5 --reps 3 > gpurun_out/ncu_${TAG}_c5.log 2>&1; echo "ncu_sell_c5=$?"

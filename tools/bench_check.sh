#!/usr/bin/env bash
# bench.py in its driver forms on a 1-GPU box
TAG=${1:-bc}
mkdir -p gpurun_out
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err; echo "c2 rc=$? $(( $(date +%s)-t0 ))s"; tail -1 gpurun_out/bench_${TAG}_c2.json | cut -c1-200
for c in ${CONFIGS:-c5 c4}; do
t0=$(date +%s); timeout 900 python bench.py --config $c --steps 5 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "$c rc=$? $(( $(date +%s)-t0 ))s"; tail -1 gpurun_out/bench_${TAG}_$c.json | cut -c1-200
done
timeout 300 python bench.py --gpus 2 > gpurun_out/bench_${TAG}_g2.out 2>&1; echo "gpus2 rc=$?"; tail -2 gpurun_out/bench_${TAG}_g2.out
if [ -n "$REF" ]; then t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_${TAG}_ref.json 2>&1; echo "ref rc=$? $(( $(date +%s)-t0 ))s"; tail -1 gpurun_out/bench_${TAG}_ref.json | cut -c1-200; fi

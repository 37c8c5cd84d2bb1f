#!/usr/bin/env bash
# All benchmark configurations on one GPU (gpurun), JSON lines into gpurun_out/.
TAG=${1:-all}
mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --worklist 1 > gpurun_out/bench_${TAG}_c2wl.json 2>&1; echo "c2wl rc=$?"
timeout 900 python bench.py --config c4 --steps 3 --warmup 3 --nodes ${C4_NODES:-8192} > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err; echo "c4 rc=$?"
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "c5 rc=$?"
timeout 900 python bench.py --impl reference --config c2 --steps 2 --warmup 1 > gpurun_out/bench_${TAG}_ref_c2.json 2>&1; echo "ref rc=$?"

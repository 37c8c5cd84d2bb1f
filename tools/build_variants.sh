#!/usr/bin/env bash
# build library variants into build/var/NAME.so: tools/build_variants.sh "NAME:-DFLAG=1 -DX=2" ...
set -e
mkdir -p build/var
rm -f build/var/*.so
pids=()
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -Xcompiler -fPIC -shared $flags \
    -o build/var/$name.so paper_2009_07785_b200/csrc/engine.cu -ldl &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
ls build/var

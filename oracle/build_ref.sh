#!/usr/bin/env bash
# ORACLE build recipe (test infrastructure only).
# Compiles the UNMODIFIED reference sources where they lie under
# /root/reference/proj (never copied into this repo) plus oracle/ref_shim.cpp
# into oracle/_ref/ (git-ignored; travels to the GPU box with gpurun).
# Outputs:
#   oracle/_ref/libpropgate_ref.so   reference engines + generators + MPS + shim
#   oracle/_ref/acceptance           the reference's own acceptance suite
# The reference CMake is not used (GTest / CLI11 / google-benchmark absent).
# No -march flags: the binaries must run on the GPU box's host CPU too.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${PROPGATE_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
JSON_INC="${PROPGATE_JSON_INC:-$(python3 -c 'import site,os;print(next((os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann") for p in site.getsitepackages() if os.path.isdir(os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann"))),""))')}"
if [ ! -d "$REF/core/src" ]; then
  echo "build_ref: reference not found at $REF (expected on the CPU container only)" >&2
  exit 3
fi
mkdir -p "$OUT"
SRCS="$REF/core/src/model.cpp $REF/core/src/generators.cpp $REF/core/src/seq_engine.cpp $REF/core/src/par_engine.cpp $REF/core/src/mps.cpp $REF/core/src/harness.cpp"
CXX="${CXX:-g++}"
FLAGS="-O2 -std=c++20 -pthread -I$REF/core/include -I$REF/core/src -I$JSON_INC"
# build objects once (PIC), then link the shared library and the acceptance binary
OBJ="$OUT/obj"; mkdir -p "$OBJ"
pids=()
for s in $SRCS; do
  o="$OBJ/$(basename "${s%.cpp}").o"
  if [ ! -f "$o" ] || [ "$s" -nt "$o" ]; then $CXX $FLAGS -fPIC -c "$s" -o "$o" & pids+=($!); fi
done
$CXX $FLAGS -fPIC -c "$HERE/ref_shim.cpp" -o "$OBJ/ref_shim.o" & pids+=($!)
if [ ! -f "$OBJ/acceptance.o" ]; then
  $CXX $FLAGS -I"$REF/tests" -DPROPGATE_FIXTURE_DIR="\"$REF/tests/fixtures\"" -fPIC -c "$REF/tests/acceptance.cpp" -o "$OBJ/acceptance.o" & pids+=($!)
fi
for p in "${pids[@]}"; do wait "$p"; done
LIBOBJS="$OBJ/model.o $OBJ/generators.o $OBJ/seq_engine.o $OBJ/par_engine.o $OBJ/mps.o $OBJ/harness.o"
$CXX -shared -pthread -o "$OUT/libpropgate_ref.so" $LIBOBJS "$OBJ/ref_shim.o"
$CXX -pthread -o "$OUT/acceptance" $LIBOBJS "$OBJ/acceptance.o"
# drop-in check: reference types/engines + the GPU engine via include/propgate_b200.hpp
REPO="$(cd "$HERE/.." && pwd)"
if [ -f "$REPO/paper_2009_07785_b200/libpropgate_b200.so" ]; then
  $CXX $FLAGS -I"$REPO/include" -c "$REPO/tests/cpp/gpu_dropin.cpp" -o "$OBJ/gpu_dropin.o"
  $CXX -pthread -o "$OUT/gpu_dropin" $LIBOBJS "$OBJ/gpu_dropin.o" \
      -L"$REPO/paper_2009_07785_b200" -lpropgate_b200 -Wl,-rpath,'$ORIGIN/../../paper_2009_07785_b200'
fi
# the reference's bench harness with EngineId::Gpu:
# patched COPIES of harness.hpp / harness.cpp (oracle/patch_harness.py) +
# tests/cpp/harness_gpu.cpp, linked with the GPU engine
if [ -f "$REPO/paper_2009_07785_b200/libpropgate_b200.so" ]; then
  PATCHED="$OUT/patched"
  python3 "$HERE/patch_harness.py" "$REF" "$PATCHED"
  PFLAGS="-O2 -std=c++20 -pthread -I$PATCHED -I$REF/core/include -I$REF/core/src -I$JSON_INC -I$REPO/include"
  $CXX $PFLAGS -c "$PATCHED/harness.cpp" -o "$OBJ/harness_gpu_patched.o"
  $CXX $PFLAGS -c "$REPO/tests/cpp/harness_gpu.cpp" -o "$OBJ/harness_gpu_main.o"
  $CXX -pthread -o "$OUT/harness_gpu" "$OBJ/model.o" "$OBJ/generators.o" "$OBJ/seq_engine.o" \
      "$OBJ/par_engine.o" "$OBJ/mps.o" "$OBJ/harness_gpu_patched.o" "$OBJ/harness_gpu_main.o" \
      -L"$REPO/paper_2009_07785_b200" -lpropgate_b200 -Wl,-rpath,'$ORIGIN/../../paper_2009_07785_b200'
fi
echo "build_ref: ok -> $OUT"

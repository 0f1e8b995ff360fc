#!/usr/bin/env bash
# Builds oracle/_ref/: the REFERENCE's own unmodified sources (/root/reference/proj/src) with
# the test-infrastructure stand-ins (oracle/ref_shim: Eigen/Core, doctest.h; nlohmann json from
# the image's cudnn_frontend) into libglmref.so + oracle/ref_harness.cpp, and the reference's
# own unit tests (test_tensor, test_quant, test_model, test_corruption, test_tensor_io).
# TEST INFRASTRUCTURE ONLY. Outputs go to oracle/_ref/ (git-ignored, shipped
# to the GPU box by gpurun). Without /root/reference (the GPU box) it keeps a prebuilt _ref.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${GLM_REFERENCE:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; keeping prebuilt $OUT" >&2
  exit 0
fi
JSON="$(python3 -c 'import site,os;print(next(os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann") for p in site.getsitepackages() if os.path.isdir(os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann"))))')"
mkdir -p "$OUT/obj"
CXX="/usr/bin/g++ -std=c++20 -O2 -fPIC -I$HERE/ref_shim -I$JSON -I$REF/include"
objs=()
for f in tensor quant model corruption tensor_io; do
  o="$OUT/obj/$f.o"
  if [ ! -f "$o" ] || [ "$REF/src/$f.cpp" -nt "$o" ] || [ "$HERE/ref_shim/Eigen/Core" -nt "$o" ]; then
    $CXX -c "$REF/src/$f.cpp" -o "$o"
  fi
  objs+=("$o")
done
stale=0
[ -f "$OUT/libglmref.so" ] || stale=1
for dep in "$HERE/ref_harness.cpp" "$HERE/liboracle.so" "${objs[@]}"; do
  [ "$dep" -nt "$OUT/libglmref.so" ] && stale=1
done
if [ "$stale" = 1 ]; then
  $CXX -shared "$HERE/ref_harness.cpp" "${objs[@]}" -L"$HERE" -loracle -Wl,-rpath,'$ORIGIN/..' -ldl -lpthread -o "$OUT/libglmref.so"
fi
for t in test_tensor test_quant test_model test_corruption test_tensor_io; do
  if [ ! -x "$OUT/$t" ] || [ "$REF/tests/$t.cpp" -nt "$OUT/$t" ] || [ "$OUT/obj/tensor.o" -nt "$OUT/$t" ]; then
    $CXX -I"$REF/tests" "$REF/tests/$t.cpp" "${objs[@]}" -o "$OUT/$t"
  fi
done
echo "build_ref: $OUT/libglmref.so + reference unit tests"

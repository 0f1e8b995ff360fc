for L in a b; do GLM130B_LIB=build/ab/$L/libglm130b.so timeout 300 python -m pytest tests/test_gpu_qlinear.py -m gpu -q -x -k "tcgen05_integer or glm130b_k" 2>&1 | tail -1; done
for L in a b; do GLM130B_LIB=build/ab/$L/libglm130b.so GLM_GEMV_TC=2 python tools/tc_trace.py 12288 36864 16 2>&1 | grep -v "^[0-9] {" | sed "s/^/$L /"; done
for L in a b; do echo "== $L"; GLM130B_LIB=build/ab/$L/libglm130b.so GLM_GEMV_TC=2 timeout 300 python tools/r2_mk_probe.py 8 12 16; done
echo "== imma"; timeout 300 python tools/r2_mk_probe.py 8 12 16

GLM130B_LIB=build/ab/c/libglm130b.so timeout 300 python -m pytest tests/test_gpu_qlinear.py -m gpu -q -x 2>&1 | tail -1
for L in a b c; do for D in 0 15; do echo "$L DBG $D"; GLM130B_LIB=build/ab/$L/libglm130b.so GLM_TC_DBG=$D python tools/tc_trace.py 12288 36864 16 2>&1 | grep -E "bench|digits|transcode end"; done; done

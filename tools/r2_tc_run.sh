set -x
timeout 600 python -m pytest tests/test_gpu_qlinear.py -m gpu -q -x 2>&1 | tail -5
for T in 0 2; do GLM_GEMV_TC=$T timeout 300 python tools/r2_mk_probe.py 2 4 8 12 16; done

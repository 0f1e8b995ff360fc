# parity of the multi-token GEMV, then RT=1 vs RT=2 per M on the GLM-130B shapes
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q > gpurun_out/check.log 2>&1; tail -3 gpurun_out/check.log
for rt in 1 2; do
  for M in 4 8 12 16; do
    GLM_MK_RT=$rt python - <<PY
import sys; sys.path.insert(0, '.')
from paper_2210_02414_b200 import glm
out = []
for K, N in [(12288, 36864), (12288, 12288), (12288, 65536), (32768, 12288)]:
    for bits in (4, 8):
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        us = q.bench($M, iters=20, flush=False)
        out.append(f"{bits}b {K}x{N} {us:6.1f}us {K*N*bits/8/us/1e3:5.0f}GB/s")
        del q
print("RT=$rt M=$M", " | ".join(out))
PY
  done
done

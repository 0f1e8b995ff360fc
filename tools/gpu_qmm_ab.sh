# qmm parity + prefill/qlinear A/B against a previous library: tools/gpu_qmm_ab.sh OLD_LIB
OLD=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q > gpurun_out/check.log 2>&1; tail -3 gpurun_out/check.log
for L in "$OLD" paper_2210_02414_b200/libglm130b.so "$OLD" paper_2210_02414_b200/libglm130b.so; do
  echo "== $L"
  GLM130B_LIB=$L timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c1-300
  GLM130B_LIB=$L python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2210_02414_b200 import glm
out = []
for K, N in [(12288, 36864), (32768, 12288)]:
    for bits in (4, 8):
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        for M in (256, 2048):
            us = q.bench(M, iters=10, flush=False)
            out.append(f"{bits}b {K}x{N} M{M} {us:7.1f}us {2*M*K*N/us/1e6:5.0f}TF")
        del q
print(" | ".join(out))
PY
done

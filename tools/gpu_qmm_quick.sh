# qlinear + prefill parity, GEMM timing, config-3 launch list (tools/gpu_qmm_quick.sh)
timeout 1500 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_model.py -x -q 2>&1 | tail -2
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2210_02414_b200 import glm
out = []
for K, N in [(12288, 36864), (32768, 12288)]:
    for bits in (4, 8):
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        for M in (256, 2048, 8192):
            us = q.bench(M, iters=10, flush=False)
            out.append(f"{bits}b {K}x{N} M{M} {us:7.1f}us {2*M*K*N/us/1e6:5.0f}TF")
        del q
print("\n".join(out))
PY
for i in 1 2; do timeout 600 python tools/bench_prefill.py 2>&1 | tail -2 | cut -c60-110; done
bash tools/ncu_prefill_list.sh | head -4

"""Multi-token INT4 GEMV probe: QLinear.bench at the four GLM-130B shapes for M tokens (weights
streamed from HBM every launch); env switches select the kernel variant (GLM_GEMV_IMMA, GLM_MK_RT)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02414_b200 import glm

Ms = [int(v) for v in sys.argv[1:]] or [3, 4, 8, 12, 16]
for K, N in [(12288, 36864), (12288, 12288), (12288, 32768), (32768, 12288)]:
    q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, 4, "column")
    for M in Ms:
        us = q.bench(M, iters=30, flush=False)
        b = K * N // 2 + 4 * N + 2 * M * (K + N)
        print(json.dumps({"K": K, "N": N, "M": M, "us": round(us, 2), "TB/s": round(b / us / 1e6, 3),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("GLM_")}}), flush=True)
    del q

import os, sys
sys.path.insert(0, '.')
from paper_2210_02414_b200 import glm
for bits in (4, 8):
    for K, N in [(12288, 36864), (12288, 12288), (12288, 65536), (32768, 12288)]:
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        for M in (8, 16):
            us = q.bench(M, iters=20, flush=False)
            print(os.environ.get("GLM_QMM_MIN_M", "17"), bits, K, N, M, round(us, 1), round(K * N * bits / 8 / us / 1e3), "GB/s", flush=True)
        del q

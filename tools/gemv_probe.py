import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2210_02414_b200 import glm
shapes = [(12288, 36864), (12288, 12288), (12288, 65536), (32768, 12288)]
for bits in (4, 8):
    for K, N in shapes:
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        for M in (1, 16):
            us = q.bench(M, iters=20, flush=False)
            gb = K * N * bits / 8 / 1e9
            print(f"int{bits} K={K} N={N} M={M}: {us:.1f} us  {gb / (us * 1e-6):.0f} GB/s", flush=True)
        del q

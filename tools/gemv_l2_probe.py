"""INT4 M=1 GEMV on L2-resident weights vs HBM-streamed ones: separates the kernel's
consumption rate from HBM latency/bandwidth."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02414_b200 import glm
for K, N in [(12288, 2048), (12288, 4096), (12288, 8192), (12288, 16384), (12288, 36864)]:
    q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, 4, "column")
    us = q.bench(1, iters=50, flush=False)
    print(f"K={K} N={N} ({K * N / 2 / 2**20:.0f} MiB): {us:.2f} us {K * N / 2 / us / 1e3:.0f} GB/s", flush=True)
    del q

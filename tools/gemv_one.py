"""One GEMV shape for ncu: python tools/gemv_one.py K N bits M"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2210_02414_b200 import glm
K, N, bits, M = (int(v) for v in sys.argv[1:5])
q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
us = q.bench(M, iters=5, flush=False)
print(f"K={K} N={N} bits={bits} M={M}: {us:.1f} us {K * N * bits / 8 / us / 1e3:.0f} GB/s")

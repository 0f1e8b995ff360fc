"""INT4 M=1 GEMV bandwidth at the four GLM-130B shapes (used with GLM_M1_WARPS / GLM_M1_STAGES)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02414_b200 import glm
tot_b = tot_us = 0.0
for K, N in [(12288, 36864), (12288, 12288), (12288, 65536), (32768, 12288)]:
    q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, 4, "column")
    us = q.bench(1, iters=20, flush=False)
    b = K * N / 2
    tot_b += b
    tot_us += us
    print(f"  K={K} N={N}: {us:.1f} us {b / us / 1e3:.0f} GB/s")
    del q
print(f"warps={os.environ.get('GLM_M1_WARPS', '16')} stages={os.environ.get('GLM_M1_STAGES', '3')}: layer {tot_us:.1f} us, {tot_b / tot_us / 1e3:.0f} GB/s")

"""One INT4 multi-token GEMV shape for ncu (tools/mk_probe.py M K N [bits])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02414_b200 import glm

M, K, N = (int(v) for v in sys.argv[1:4])
bits = int(sys.argv[4]) if len(sys.argv) > 4 else 4
q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
print(M, K, N, bits, "us", q.bench(M, iters=10, flush=False))

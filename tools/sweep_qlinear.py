"""BASELINE config 5: quantized-linear sweep. W4A16 and W8A16, per-output-channel scales,
M in {1, 16, 256, 2048} at the four GLM-130B (K, N) shapes, against the HBM and tensor
rooflines of MEASURED_PEAKS.json. M <= 16 runs the decode GEMV, larger M the tcgen05 GEMM.
Weights larger than L2 (>= 75 MB) are streamed from HBM every launch; one JSON line each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02414_b200 import glm

here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    pk = json.load(open(os.path.join(here, "MEASURED_PEAKS.json")))
    hbm, tc = pk["hbm_gbs"], pk["bf16_tflops"]  # burst figures: each point is one kernel timed alone
except (OSError, KeyError, ValueError):
    hbm, tc = 6650.0, 1400.0
for bits in (4, 8):
    for K, N in [(12288, 36864), (12288, 12288), (12288, 32768), (32768, 12288)]:
        q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
        for M in (1, 16, 256, 2048):
            us = q.bench(M, iters=20 if M <= 256 else 5, flush=False)
            wbytes = K * N * bits // 8
            nbytes = wbytes + 4 * N + 2 * M * (K + N)
            flop = 2.0 * M * K * N
            t_roof = max(nbytes / (hbm * 1e9), flop / (tc * 1e12)) * 1e6
            print(json.dumps({"bits": bits, "K": K, "N": N, "M": M, "us": round(us, 2),
                              "GB/s": round(nbytes / us / 1e3, 1), "TFLOP/s": round(flop / us / 1e6, 1),
                              "bound": "hbm" if nbytes / (hbm * 1e9) > flop / (tc * 1e12) else "tensor",
                              "roofline_us": round(t_roof, 2), "frac": round(t_roof / us, 3)}), flush=True)
        del q

"""BASELINE config 3: one GLM-130B-shaped block (hidden 12288, 96 heads, FFN 32768) INT4 / INT8
prefill of 4 [gMASK] samples of 2048 tokens (P = 2046, C = 2047, one [sop]) through the
tcgen05 GEMM + tensor-core flash attention. Synthetic counter-based weights; small vocab
(the head is not part of the block). Prints one JSON line per precision."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2210_02414_b200 import glm

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--bits", type=int, nargs="+", default=[4, 8])
ap.add_argument("--separate", action="store_true", help="one prefill call per sample instead of one packed call")
a = ap.parse_args()
torch.cuda.set_device(0)
d, H, f = 12288, 96, 32768
for bits in a.bits:
    cfg = glm.GLMConfig(num_layers=1, hidden=d, num_heads=H, ffn_hidden=f, vocab=1024)
    m = glm.Model(cfg, bits=bits, axis="column", max_batch=a.batch, max_ctx=a.seq + 8, head_bf16=True)
    m.init_synthetic(2210)
    rng = np.random.default_rng(0)
    P = a.seq - 2
    samples = []
    for b in range(a.batch):
        toks = [int(v) for v in rng.integers(6, 1000, size=P)] + [2, 3]
        pos, C = glm.gmask_layout(P, 1)
        samples.append((toks, pos[:a.seq], C))

    def run():
        if a.separate:
            for b, (toks, pos, C) in enumerate(samples):
                m.prefill(toks, pos, C, seq=b, logits=False)
        else:  # packed: one call, M = batch * seq rows through every linear
            m.prefill_batch([(b, toks, pos, C) for b, (toks, pos, C) in enumerate(samples)], logits=False)

    run()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(a.iters):
        run()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) * 1e3 / a.iters
    n = a.seq * a.batch
    lin_flop = 2.0 * n * (d * 3 * d + d * d + 2 * d * f + f * d)
    # attention (dense upper bound, QK^T and PV): the gMASK prefix is bidirectional
    att_flop = 4.0 * a.batch * a.seq * a.seq * d
    print(json.dumps({"config": "BASELINE configs[2]: one GLM-130B block prefill", "bits": bits,
                      "seq": a.seq, "batch": a.batch, "ms": ms, "tokens_per_s": n / ms * 1e3,
                      "linear_tflop": lin_flop / 1e12, "attention_tflop": att_flop / 1e12,
                      "tflops": (lin_flop + att_flop) / (ms * 1e-3) / 1e12,
                      "mode": "separate calls" if a.separate else "packed (one call)",
                      "timing": "host wall clock around synchronised prefill calls (includes host copies)"}),
          flush=True)
    del m

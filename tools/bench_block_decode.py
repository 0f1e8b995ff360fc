"""BASELINE config 2: one GLM-130B-shaped block (hidden 12288, 96 heads, FFN 32768) W4A16
decode at batch 1 with a 2048-token KV cache, on one GPU. Synthetic counter-based weights,
small vocab (the 150528-row head is not part of the block). Device-timed CUDA-graph steps.
Bytes per token: INT4 codes + scales of the block and the K/V cache read."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2210_02414_b200 import glm

torch.cuda.set_device(0)
ap = argparse.ArgumentParser()
ap.add_argument("--kv", type=int, default=2048, help="cached tokens at the first timed step")
ap.add_argument("--max-ctx", type=int, default=0, help="model max_ctx (default kv + 64)")
args = ap.parse_args()
d, H, f, KV = 12288, 96, 32768, args.kv
cfg = glm.GLMConfig(num_layers=1, hidden=d, num_heads=H, ffn_hidden=f, vocab=1024)
m = glm.Model(cfg, bits=4, axis="column", max_batch=1, max_ctx=args.max_ctx or KV + 64, head_bf16=True)
m.init_synthetic(2210)
P = KV - 2
rng = np.random.default_rng(0)
pos, C = glm.gmask_layout(P, 0)
m.prefill([int(v) for v in rng.integers(6, 1000, size=P)] + [2], pos[:C], C, logits=False)
m.decode_step([3], [P], logits=False)
steps = 50
ms, gemv_ms, launches = m.bench_decode(1, steps, warmup=5)
w_bytes = (d * 3 * d + d * d + 2 * d * f + f * d) // 2 + 4 * (3 * d + d + 2 * f + d)
kv_bytes = 2 * (KV + steps // 2) * d * 2
print(json.dumps({"config": f"BASELINE configs[1]: one GLM-130B block W4A16 decode, batch 1, KV {KV} (max_ctx {args.max_ctx or KV + 64})",
                  "ms_per_token": ms, "gemv_ms": gemv_ms, "launches_per_step": launches,
                  "block_bytes_per_token": w_bytes + kv_bytes,
                  "achieved_GB/s": (w_bytes + kv_bytes) / (ms * 1e-3) / 1e9,
                  "note": "step includes embed + 1024-row head + argmax (small)"}), flush=True)

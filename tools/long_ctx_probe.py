"""Decode many steps of one GLM-130B-width block at a ~2048-token cache (debug probe)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2210_02414_b200 import glm

KV = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
d = int(sys.argv[2]) if len(sys.argv) > 2 else 12288
H = d // 128
cfg = glm.GLMConfig(num_layers=1, hidden=d, num_heads=H, vocab=1024)
m = glm.Model(cfg, bits=4, axis="column", max_batch=1, max_ctx=KV + 64, head_bf16=True)
m.init_synthetic(2210)
P = KV - 2
rng = np.random.default_rng(0)
pos, C = glm.gmask_layout(P, 0)
m.prefill([int(v) for v in rng.integers(6, 1000, size=P)] + [2], pos[:C], C, logits=False)
tok, p = 3, P
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 60):
    nxt, _ = m.decode_step([tok], [p], logits=False)
    tok, p = int(nxt[0]), p + 1
    if i % 10 == 0:
        print("step", i, "len", P + 1 + i + 1, flush=True)
print("ok")

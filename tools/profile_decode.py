"""Profiling window for ncu: builds the GLM-130B INT4 model, prefills, warms up, then runs
`--steps` decode steps between cudaProfilerStart/Stop (use ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2210_02414_b200 import glm
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--layers", type=int, default=70)
ap.add_argument("--bits", type=int, default=4)
ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
torch.cuda.set_device(0)
cfg = dict(bench.G)
cfg["num_layers"] = a.layers
m = glm.Model(glm.GLMConfig(**cfg), bits=a.bits, axis="column", max_ctx=256, head_bf16=True, max_batch=a.batch)
m.init_synthetic(2210)
pos, C = glm.gmask_layout(127, 0)
for b in range(a.batch):
    m.prefill([7] * 127 + [2], pos[:C], C, seq=b, logits=False)
tok, p = [3] * a.batch, [127] * a.batch
for _ in range(3):
    nxt, _ = m.decode_step(tok, p, logits=False)
    tok, p = [int(v) for v in nxt], [q + 1 for q in p]
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    nxt, _ = m.decode_step(tok, p, logits=False)
    tok, p = [int(v) for v in nxt], [q + 1 for q in p]
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled", a.steps, "decode steps")

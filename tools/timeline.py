"""Device timeline of one GLM-130B decode step (diagnostics). Uses glm_debug_trace_start/
stop: thread 0 of every CTA of the decode kernels stamps %globaltimer at kernel entry, after
the programmatic-dependency wait, (GEMV) when its activations are ready, and at exit.
Prints, per kernel instance of layers 10..11, first entry / first post-wait / last exit
relative to the previous kernel's last exit."""
import argparse
import collections
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2210_02414_b200 import glm
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=70)
ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--prompt", type=int, default=127, help="prompt tokens before [gMASK] (cache length)")
ap.add_argument("--first", type=int, default=40, help="first kernel instance printed")
a = ap.parse_args()
torch.cuda.set_device(0)
cfg = dict(bench.G)
cfg["num_layers"] = a.layers
m = glm.Model(glm.GLMConfig(**cfg), bits=4, axis="column", max_ctx=max(256, a.prompt + 64), head_bf16=True,
              max_batch=a.batch)
m.init_synthetic(2210)
pos, Cl = glm.gmask_layout(a.prompt, 0)
for b in range(a.batch):
    m.prefill([7] * a.prompt + [2], pos[:Cl], Cl, seq=b, logits=False)
tok, p = [3] * a.batch, [a.prompt] * a.batch
for _ in range(3):
    nxt, _ = m.decode_step(tok, p, logits=False)
    tok, p = [int(v) for v in nxt], [q + 1 for q in p]
cap = 1 << 22
glm._check(glm.lib().glm_debug_trace_start(cap))
nxt, _ = m.decode_step(tok, p, logits=False)
buf = np.zeros(2 * cap, np.uint64)
n = C.c_int64()
glm._check(glm.lib().glm_debug_trace_stop(glm._p(buf), cap, C.byref(n)))
rec = buf[:2 * n.value].reshape(-1, 2)
t = rec[:, 0].astype(np.int64)
tag = (rec[:, 1] >> 32).astype(np.int64)
t0 = t.min()
t = t - t0
fam = (tag // 10) * 10
kind = tag % 10
names = {10: "gemv", 20: "ln", 30: "attn", 40: "act", 50: "head"}
endkind = {10: 3, 20: 2, 30: 2, 40: 2, 50: 2}
# post-wait stamps of one kernel instance are released together: cluster them in time
w = np.where(kind == 1)[0]
w = w[np.argsort(t[w])]
inst = []
blk = ((rec[:, 1] >> 8) & 0xFFFFFF).astype(np.int64)
for i in w:
    # a GEMV CTA id seen twice starts the next launch (grids of other kernels are 3-D: no dedupe)
    if (inst and inst[-1]["fam"] == fam[i] and t[i] - inst[-1]["wait_last"] < 20000
            and (fam[i] != 10 or blk[i] not in inst[-1]["blocks"])):
        inst[-1]["wait_last"] = t[i]
        inst[-1]["n"] += 1
        inst[-1]["blocks"].add(blk[i])
    else:
        inst.append({"fam": int(fam[i]), "wait": int(t[i]), "wait_last": int(t[i]), "n": 1, "blocks": {blk[i]}})
for k, c in enumerate(inst):
    nxt = inst[k + 1]["wait"] if k + 1 < len(inst) else t.max() + 1
    sel = (fam == c["fam"]) & (t >= c["wait"]) & (t <= nxt)
    ends = t[sel & (kind == endkind[c["fam"]])]
    c["end"] = int(ends.max()) if ends.size else c["wait"]
    c["end_min"] = int(ends.min()) if ends.size else c["wait"]
    rdy = t[sel & (kind == 2)] if c["fam"] == 10 else np.array([])
    c["ready"] = int(rdy.max()) if rdy.size else None
    xa = t[sel & (kind == 4)] if c["fam"] == 10 else np.array([])
    c["xarr"] = int(xa.max()) if xa.size else None
    mxd = t[sel & (kind == 5)] if c["fam"] == 10 else np.array([])
    c["maxd"] = int(mxd.max()) if mxd.size else None
    st7 = t[sel & (kind == 7)] if c["fam"] == 10 else np.array([])
    c["lnstat"] = int(st7.max()) if st7.size else None
    # entry (kind 0) of this instance: the earliest entry stamp after the previous instance's release
    ent = t[(fam == c["fam"]) & (kind == 0) & (t <= c["wait"]) & (t >= (inst[k - 1]["wait"] if k > 0 else 0))]
    c["entry"] = int(ent.min()) if ent.size else None
print(f"{len(rec)} records, {len(inst)} kernel instances, step span {t.max() / 1e3:.1f} us")
total = collections.Counter()
gaps = collections.Counter()
prev_end = None
for i, c in enumerate(inst):
    gap = (c["wait"] - prev_end) / 1e3 if prev_end is not None else 0.0
    dur = (c["end"] - c["wait"]) / 1e3
    total[names[c["fam"]]] += dur
    gaps[names[c["fam"]]] += gap
    if a.first <= i < a.first + 16:
        rdy = (c["ready"] - c["wait"]) / 1e3 if c["ready"] else float("nan")
        tail = (c["end"] - c["end_min"]) / 1e3
        xa = (c["xarr"] - c["wait"]) / 1e3 if c.get("xarr") else float("nan")
        md = (c["maxd"] - c["wait"]) / 1e3 if c.get("maxd") else float("nan")
        lst = (c["lnstat"] - c["wait"]) / 1e3 if c.get("lnstat") else float("nan")
        ent = (c["wait"] - c["entry"]) / 1e3 if c.get("entry") else float("nan")
        print(f"{i:4d} {names[c['fam']]:5s} CTAs {c['n']:4d} released {c['wait'] / 1e3:9.1f} us (+{gap:5.2f} after prev end,"
              f" first entry {ent:5.2f} before)  x-arrived +{xa:5.2f} ln-stats +{lst:5.2f} max +{md:5.2f} x-ready +{rdy:5.2f}"
              f"  work {dur:6.2f}  end spread {tail:5.2f}")
    prev_end = c["end"]
print("post-wait -> last end, summed per family (us):", {k: round(v, 1) for k, v in total.items()})
# LayerNorm phases: post-wait -> loads done (23) -> cluster reduction done (24) -> end
for c in inst[a.first:a.first + 16]:
    if c["fam"] != 20:
        continue
    nxt = [d["wait"] for d in inst if d["wait"] > c["wait"]]
    hi = nxt[0] if nxt else t.max() + 1
    sel = (fam == 20) & (t >= c["wait"]) & (t <= hi)
    l3, l4 = t[sel & (kind == 3)], t[sel & (kind == 4)]
    if l3.size and l4.size:
        print(f"ln: loads done +{(l3.max() - c['wait']) / 1e3:.2f}  reduced +{(l4.max() - c['wait']) / 1e3:.2f}  end +{(c['end'] - c['wait']) / 1e3:.2f} us")
print("previous end -> release gaps, summed per family (us):", {k: round(v, 1) for k, v in gaps.items()})

for c in inst[a.first:a.first + 16]:
    if c["fam"] != 30:
        continue
    nxt = [d["wait"] for d in inst if d["wait"] > c["wait"]]
    hi = nxt[0] if nxt else t.max() + 1
    sel = (fam == 30) & (t >= c["wait"]) & (t <= hi)
    ph = [t[sel & (kind == k)] for k in (3, 4, 5)]
    if all(x.size for x in ph):
        print("attn: q ready +%.2f  scores +%.2f  P.V +%.2f  end +%.2f us" % tuple(
            [(x.max() - c["wait"]) / 1e3 for x in ph] + [(c["end"] - c["wait"]) / 1e3]))

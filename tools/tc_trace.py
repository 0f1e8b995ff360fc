"""Per-CTA timeline of one k_gemv_tc_i4 launch (diagnostics): entry (10), after the dependency
wait (11), each k-slice's digits ready (12), transcode done (13), ns from the first entry.
python tools/tc_trace.py K N M"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2210_02414_b200 import glm

K, N, M = (int(v) for v in sys.argv[1:4])
q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, 4, "column")
x = np.random.default_rng(0).normal(size=(M, K))
print(q.plan(M), "bench us", q.bench(M, iters=20, flush=False))
q(x)
cap = 1 << 20
glm._check(glm.lib().glm_debug_trace_start(cap))
q(x)
buf = np.zeros(2 * cap, np.uint64)
n = C.c_int64()
glm._check(glm.lib().glm_debug_trace_stop(glm._p(buf), cap, C.byref(n)))
rec = buf[:2 * n.value].reshape(-1, 2)
t = rec[:, 0].astype(np.int64)
tag = (rec[:, 1] >> 32).astype(np.int64)
blk = ((rec[:, 1] >> 8) & 0xFFFFFF).astype(np.int64)
t = t - t[tag == 10].min()
print("records", len(t), "span us", t.max() / 1e3)
for name, k in (("entry", 10), ("post-wait", 11), ("x landed", 14), ("max done", 15), ("digits", 12), ("transcode end", 13)):
    v = t[tag == k] / 1e3
    if len(v):
        print(f"{name:14s} n={len(v):4d} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
d = {}
for ti, tg, b in zip(t, tag, blk):
    d.setdefault(b, {}).setdefault(tg, []).append(ti / 1e3)
for b in sorted(d)[:2]:
    print(b, {k: [round(x, 2) for x in v] for k, v in sorted(d[b].items())})

"""Per-stage pipeline timeline of CTA 0 of one quantized-matmul launch (GLM_QMM_TRACE=1).
Stamps: 0 producer passed slot-free wait, 5 producer issued copies, 1 transcode group 0
saw the weights, 2 group 0 finished (A in TMEM), 3 issuer saw A ready, 4 issuer committed."""
import os, sys
os.environ["GLM_QMM_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2210_02414_b200 import glm
K, N, bits, M = (int(v) for v in sys.argv[1:5])
q = glm.QLinear.synthetic(1, 3, K, N, 5.6e-4, bits, "column")
q.bench(M, iters=2, flush=False)
t = np.zeros((256, 8), np.int64)
glm._check(glm.lib().glm_debug_qmm_trace(glm._p(t)))
t0 = t[0, 0]
ev = [0, 5, 1, 2, 3, 4]
names = ["slot_free", "copies_out", "deq_seen", "deq_done", "mma_start", "mma_commit"]
print("stage " + " ".join(f"{n:>11s}" for n in names))
for i in list(range(0, 40)) + list(range(200, 216)):
    print(f"{i:5d} " + " ".join(f"{(t[i, e] - t0) if t[i, e] else -1:11d}" for e in ev))
n = 250
for e, nm in zip(ev, names):
    v = t[:n, e]
    v = v[v > 0]
    if len(v) > 10:
        d = np.diff(np.sort(v))
        print(f"{nm:12s} median spacing {np.median(d):8.1f} cycles over {len(v)} stamps")
g0 = np.arange(0, n, 4)
print("group0 latency seen->done median", np.median(t[g0, 2] - t[g0, 1]), " done->mma_start", np.median(t[g0, 3] - t[g0, 2]),
      " mma_start->commit", np.median(t[g0, 4] - t[g0, 3]), " copies_out->seen", np.median(t[g0, 1] - t[g0, 5]))

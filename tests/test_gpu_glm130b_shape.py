"""Parity at the GLM-130B shape (d 12288, 96 heads x 128, ffn 32768, vocab 150528) — the shapes
the headline numbers are quoted on (BASELINE configs 2-5), against the CPU oracle:

  (a) codes + FP64 scales of every linear of the GPU's synthetic init (glm_model_init_synthetic,
      the weights bench.py runs) == the oracle's quantize_absmax (quant.cpp:113-143) of the same
      counter-based values (or_gen_quantize), byte for byte, kRow and kColumn, 70-layer model;
  (b) one G-shaped block (glm_block_forward) in prefill over > 4 token tiles (the tcgen05 GEMM's
      token-group walk, qmm_tc.cu, and the paired W1|V GeGLU GEMM at M > 1024) plus
      teacher-forced decode rows against the oracle block (model.cpp:198-224): sublayer taps
      and block output <= 1e-2 of their max;
  (c) the quantized linear at the four G (K, N) shapes for M in {1, 16, 256, 2048, 8192} against
      x . dequantize(q) on 256 sampled output columns (quant.cpp:188-221 + tensor.cpp:135-155);
  (d) the bf16 tied head over the full 150528-token vocabulary (model.cpp:225) against the
      oracle's h . E^T, batch 1 (fp32 h) and batch 2 (bf16 h on the tensor cores), argmax included;
  (e) batched decode of 8 sequences through one G block (multi-token integer-MMA GEMV, streaming
      attention of 3+ sequences) against the oracle block of each sequence;
  (f) one G block under Megatron tensor parallelism at t = 4 and 8 (emulated group on one GPU).
"""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

pytestmark = pytest.mark.gpu
D, H, F, V = 12288, 96, 32768, 150528
EMBED_ID = 0xFFFF0000  # gen.cuh kEmbedTensorId


def stds(L):
    """init_parameters stds (model.cpp:69-104) for an L-layer GLM-130B-shaped model."""
    fac = (2.0 * L) ** -0.5
    xav = lambda a, b: (2.0 / (a + b)) ** 0.5  # noqa: E731
    return {"init": 0.0052, "v": xav(D, D) * fac, "out": xav(D, D) * fac, "ffn": xav(D, F) * fac, "w2": xav(F, D) * fac}


def oracle_linear(seed, L, layer, which, bits, axis):
    s = stds(L)
    tid = layer * 8 + which
    if which == O.QKV:
        return O.gen_quantize(seed, tid, D, 3 * D, bits, axis, s["init"], s["v"], 2 * D)
    if which == O.OUT:
        return O.gen_quantize(seed, tid, D, D, bits, axis, s["out"])
    if which in (O.W1, O.V):
        return O.gen_quantize(seed, tid, D, F, bits, axis, s["ffn"])
    return O.gen_quantize(seed, tid, F, D, bits, axis, s["w2"])


SHAPE = {O.QKV: (D, 3 * D), O.OUT: (D, D), O.W1: (D, F), O.V: (D, F), O.W2: (F, D)}


@pytest.mark.parametrize("axis", ["column", "row"])
def test_synthetic_init_codes_bit_exact_70_layers(axis):
    L, seed = 70, 2210
    m = glm.Model(glm.GLMConfig(num_layers=L, hidden=D, num_heads=H, ffn_hidden=F, vocab=V), bits=4, axis=axis,
                  max_ctx=8, head_bf16=True)
    m.init_synthetic(seed)
    for layer in (0, 37, 69):
        for which in range(5):
            payload, scales = m.export_linear(layer, which, *SHAPE[which])
            ref = oracle_linear(seed, L, layer, which, 4, axis)
            assert np.array_equal(scales, ref["scales"]), (layer, which)
            assert np.array_equal(payload, ref["payload"]), (layer, which)
    del m


def g_block(bits, axis, seed, max_ctx, head_bf16=False, max_batch=2):
    m = glm.Model(glm.GLMConfig(num_layers=1, hidden=D, num_heads=H, ffn_hidden=F, vocab=V), bits=bits, axis=axis,
                  max_ctx=max_ctx, max_batch=max_batch, head_bf16=head_bf16)
    m.init_synthetic(seed)
    return m


@pytest.mark.parametrize("bits,axis,n", [(4, "column", 1100), (8, "row", 300)])
def test_g_block_prefill_and_decode_match_oracle(bits, axis, n):
    seed, G = 77, 3
    m = g_block(bits, axis, seed, max_ctx=n + G + 1)
    W = {}
    for which in range(5):
        payload, scales = m.export_linear(0, which, *SHAPE[which])
        ref = oracle_linear(seed, 1, 0, which, bits, axis)
        assert np.array_equal(payload, ref["payload"]) and np.array_equal(scales, ref["scales"]), which
        W[which] = O.dequantize(ref)
        del ref
    ones, zeros = np.ones(D), np.zeros(D)
    N = n + G
    P = n - 1                                  # prefix, [gMASK] at P: context length C = n
    pos = list(range(P)) + [P] + [P + j for j in range(G)]
    C = n
    rng = np.random.default_rng(bits)
    x = rng.normal(0.0, 1.0, size=(N, D))
    mask = np.arange(N)[None, :] < np.maximum(C, np.arange(N)[:, None] + 1)  # corruption.cpp:338-367
    out, attn, ff = O.block_forward(x, W, (ones, zeros, ones, zeros), pos, mask, H, alpha=np.sqrt(2.0))
    del W
    m.enable_taps(True)
    y = m.block_forward(0, x[:n].astype(np.float32), pos[:n], "prefill", seq=0, context_length=C)
    ta, tf = m.taps(n)
    rows = [(y, ta[0], tf[0], slice(0, n))]
    for r in range(n, N):
        yr = m.block_forward(0, x[r:r + 1].astype(np.float32), pos[r:r + 1], "decode")
        ta, tf = m.taps(1)
        rows.append((yr, ta[0], tf[0], slice(r, r + 1)))
    for (yg, tag, tfg, sl) in rows:
        for got, ref, name in ((tag, attn[sl], "attention"), (tfg, ff[sl], "geglu"), (yg, out[sl], "block output")):
            err = np.abs(got.astype(np.float64) - ref).max()
            assert err <= 1e-2 * np.abs(ref).max(), (name, sl, err, np.abs(ref).max())


def test_g_block_batched_decode_8_sequences_match_oracle():
    """Batched decode at the G shape (the rows behind the batch sweep): one G block, 8 sequences
    with their own prefixes (21..84 tokens) prefilled into their caches, then two decode steps of
    8 rows each — the multi-token integer-MMA GEMV (k_gemv_mk_i4, M = 8) and the streaming
    attention of 3+ sequences (k_attn_decode_ring) — against the oracle block per sequence."""
    seed, bits, axis, B = 91, 4, "column", 8
    m = g_block(bits, axis, seed, max_ctx=96, max_batch=B)
    W = {w: O.dequantize(oracle_linear(seed, 1, 0, w, bits, axis)) for w in range(5)}
    ones, zeros = np.ones(D), np.zeros(D)
    rng = np.random.default_rng(B)
    lens = [21 + 9 * b for b in range(B)]
    xs, ref_out, ref_attn = [], [], []
    for b, n in enumerate(lens):
        N = n + 2
        x = rng.normal(0.0, 1.0, size=(N, D))
        pos = list(range(n - 1)) + [n - 1, n - 1, n]  # prefix, [gMASK] at n-1, two generated rows
        mask = np.arange(N)[None, :] < np.maximum(n, np.arange(N)[:, None] + 1)
        out, attn, _ff = O.block_forward(x, W, (ones, zeros, ones, zeros), pos, mask, H, alpha=np.sqrt(2.0))
        xs.append((x, pos))
        ref_out.append(out[n:])
        ref_attn.append(attn[n:])
        m.block_forward(0, x[:n].astype(np.float32), pos[:n], "prefill", seq=b, context_length=n)
    del W
    m.enable_taps(True)
    for j in range(2):
        rows = np.stack([xs[b][0][lens[b] + j] for b in range(B)]).astype(np.float32)
        pos = [xs[b][1][lens[b] + j] for b in range(B)]
        y = m.block_forward(0, rows, pos, "decode")
        ta, _tf = m.taps(B)
        for b in range(B):
            for got, ref, name in ((ta[0][b], ref_attn[b][j], "attention"), (y[b], ref_out[b][j], "block output")):
                err = np.abs(got.astype(np.float64) - ref).max()
                assert err <= 1e-2 * np.abs(ref).max(), (name, b, j, err, np.abs(ref).max())


@pytest.mark.parametrize("t", [4, 8])
def test_g_block_tensor_parallel_matches_oracle(t):
    """Megatron tensor parallelism at the G shape: t rank-models of one GLM-130B block (heads
    96 / t, ffn 32768 / t per rank, INT4 kColumn synthetic weights quantized on the full
    matrices) on one GPU through the emulated group, prefill (allreduce after out_proj / ffn_w2)
    and decode (the fused push / sum inside the LayerNorm) via glm_block_forward, against the
    oracle block; every rank holds the same output."""
    seed, bits, axis, n = 92, 4, "column", 64
    group = glm.EmulatedGroup(t)
    ms = [glm.Model(glm.GLMConfig(num_layers=1, hidden=D, num_heads=H, ffn_hidden=F, vocab=1024), bits=bits,
                    axis=axis, max_ctx=n + 4, tp_rank=r, tp_size=t) for r in range(t)]
    glm.run_ranks([lambda m=m: m.init_comm_emulated(group) for m in ms])
    for m in ms:
        m.init_synthetic(seed)
    W = {w: O.dequantize(oracle_linear(seed, 1, 0, w, bits, axis)) for w in range(5)}
    ones, zeros = np.ones(D), np.zeros(D)
    N = n + 2
    rng = np.random.default_rng(t)
    x = rng.normal(0.0, 1.0, size=(N, D))
    pos = list(range(n - 1)) + [n - 1, n - 1, n]
    mask = np.arange(N)[None, :] < np.maximum(n, np.arange(N)[:, None] + 1)
    out, attn, ff = O.block_forward(x, W, (ones, zeros, ones, zeros), pos, mask, H, alpha=np.sqrt(2.0))
    del W
    for m in ms:
        m.enable_taps(True)
    res = glm.run_ranks([lambda m=m: (m.block_forward(0, x[:n].astype(np.float32), pos[:n], "prefill", seq=0,
                                                      context_length=n), m.taps(n)) for m in ms])
    rows = [(res[0][0], res[0][1][0][0], res[0][1][1][0], slice(0, n))]
    for r in range(1, t):
        assert np.array_equal(res[r][0], res[0][0])
    for j in range(2):
        rr = glm.run_ranks([lambda m=m: (m.block_forward(0, x[n + j:n + j + 1].astype(np.float32), pos[n + j:n + j + 1],
                                                         "decode"), m.taps(1)) for m in ms])
        for r in range(1, t):
            assert np.array_equal(rr[r][0], rr[0][0])
        rows.append((rr[0][0], rr[0][1][0][0], rr[0][1][1][0], slice(n + j, n + j + 1)))
    for yg, tag, tfg, sl in rows:
        for got, ref, name in ((tag, attn[sl], "attention"), (tfg, ff[sl], "geglu"), (yg, out[sl], "block output")):
            err = np.abs(got.astype(np.float64) - ref).max()
            assert err <= 1e-2 * np.abs(ref).max(), (t, name, sl, err, np.abs(ref).max())
    del ms, group


G_SHAPES = [(D, 3 * D), (D, D), (D, F), (F, D)]


@pytest.mark.parametrize("K,N", G_SHAPES)
def test_qlinear_g_shapes_up_to_8192_rows(K, N):
    seed, tid, sigma = 5, 900 + K // 1024 + N // 1024, 5.6e-4
    rng = np.random.default_rng(K + N)
    cols = np.sort(rng.choice(N, size=256, replace=False))
    for bits, axis, Ms in ((4, "column", (1, 16, 256, 2048, 8192)), (8, "row", (1, 2048))):
        lin = glm.QLinear.synthetic(seed, tid, K, N, sigma, bits, axis)
        q = O.gen_quantize(seed, tid, K, N, bits, axis, sigma)
        exp = lin.export()
        assert np.array_equal(exp["payload"], q["payload"]) and np.array_equal(exp["scales"], q["scales"])
        Wc = O.dequantize_cols(q, cols)
        del q, exp
        for M in Ms:
            x = rng.normal(0.0, 1.0, size=(M, K)).astype(np.float32)
            y = lin(x)[:, cols].astype(np.float64)
            ref = x.astype(np.float64) @ Wc
            err = np.abs(y - ref).max()
            assert err <= 5e-3 * np.abs(ref).max(), (bits, M, err, np.abs(ref).max())
        del lin


def oracle_head(h, seed, chunk=16384):
    """logits = h . E^T over the full vocabulary (model.cpp:225), E generated in row chunks."""
    out = np.empty((h.shape[0], V))
    for r0 in range(0, V, chunk):
        nr = min(chunk, V - r0)
        E = O.gen_rows(seed, EMBED_ID, r0, nr, D, 0.0052)
        out[:, r0:r0 + nr] = h @ E.T
    return out


def test_bf16_head_full_vocabulary():
    """Zero sublayers (the echo chain): h = LN(alpha LN(alpha e)) with e the embedding row of the
    input token, so the head's input is known exactly on the CPU and the whole 150528 x 12288
    head (3.7 GB bf16) is checked against h . E^T."""
    seed = 31
    m = g_block(4, "column", seed, max_ctx=32, head_bf16=True)
    m.zero_sublayers(True)
    alpha = np.sqrt(2.0)
    toks = [17, 150000]
    for b, t in enumerate(toks):
        m.prefill([5, 6, 7, 2], [0, 1, 2, 3], 4, seq=b, logits=False)
    e = np.stack([O.gen_rows(seed, EMBED_ID, t, 1, D, 0.0052)[0] for t in toks])
    ones, zeros = np.ones(D), np.zeros(D)
    h = O.layer_norm(alpha * O.layer_norm(alpha * e, ones, zeros), ones, zeros)
    ref = oracle_head(h, seed)
    nxt1, l1 = m.decode_step([toks[0]], [4])                  # batch 1: fp32 h x bf16 E
    err1 = np.abs(l1[0] - ref[0]).max()
    assert err1 <= 1e-4 * np.abs(ref[0]).max(), err1
    assert int(nxt1[0]) == int(np.argmax(ref[0]))
    m.reset()
    for b in range(2):
        m.prefill([5, 6, 7, 2], [0, 1, 2, 3], 4, seq=b, logits=False)
    nxt2, l2 = m.decode_step(toks, [4, 4])                    # batch 2: bf16 h on the tensor cores
    for b in range(2):
        err = np.abs(l2[b] - ref[b]).max()
        assert err <= 1e-2 * np.abs(ref[b]).max(), (b, err)
        top = np.sort(ref[b])[-2:]
        if top[1] - top[0] > 2 * err:
            assert int(nxt2[b]) == int(np.argmax(ref[b]))

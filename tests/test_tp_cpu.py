"""Megatron tensor parallelism, host side, on CPU with torch.distributed (gloo, world size 2).

The B200 path shards every quantized linear exactly as `glm_model_create(..., tp_rank,
tp_size)` does (paper_2210_02414_b200/csrc/model.cu, `mk(...)` / ShardSpec):

  qkv    [d, 3d]  column-parallel: local column j -> (j // dl) * d + r*dl + j % dl
  out    [d, d]   row-parallel:    local row i    -> r*dl + i
  w1, v  [d, f]   column-parallel: local column j -> r*fl + j
  w2     [f, d]   row-parallel:    local row i    -> r*fl + i
  head   tied embedding, vocab-sharded; logits all-gathered, argmax via max-allreduce

with one fp32 allreduce (here: float64 sum) of the row-parallel partial outputs after
out_proj and after w2. Quantization runs on the FULL matrix before sharding, so each shard
is a slice of the reference QuantizedMatrix.

These tests run that decomposition with the oracle's float64 ops on two gloo ranks and
require the gathered result to equal the single-process oracle forward
(oracle/oracle.cpp or_forward = model.cpp:166-226 on dequantize(quantize_model(p))) to
1e-10, for every layer's sublayer taps, the logits and the greedy token.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as O

CFG = dict(num_layers=2, hidden=64, num_heads=4, vocab=96, seed=77)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard_cols(which, d, f, r, t):
    """Full column indices of rank r's local columns (model.cpp ShardSpec)."""
    dl, fl = d // t, f // t
    if which == O.QKV:
        j = np.arange(3 * dl)
        return (j // dl) * d + r * dl + j % dl
    if which in (O.W1, O.V):
        return r * fl + np.arange(fl)
    return np.arange(d)  # out, w2: all columns


def shard_rows(which, d, f, r, t):
    dl, fl = d // t, f // t
    if which == O.OUT:
        return r * dl + np.arange(dl)
    if which == O.W2:
        return r * fl + np.arange(fl)
    return np.arange(d)  # qkv, w1, v: all rows


def dequantized(p, layer, which, bits, axis):
    rows, cols = p.shape(which)
    payload, scales = p.qpayload(layer, which)
    return O.dequantize(dict(payload=payload, scales=scales, rows=rows, cols=cols, bits=bits, axis=axis,
                             scheme="absmax"))


def allreduce(x):
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def tp_forward(p, sample, r, t, bits, axis):
    """Rank r's share of forward (model.cpp:166-226) with Megatron shards + gloo collectives."""
    d, H, f, V, L = p.hidden, p.num_heads, p.ffn, p.vocab, p.num_layers
    dh, Hl = d // H, H // t
    alpha = (2.0 * L) ** 0.5
    E = p.tensor(0, O.EMBED)
    x = E[np.asarray(sample["tokens"])]
    mask = O.build_mask(sample)
    attn_taps, ffn_taps = [], []
    for layer in range(L):
        W = {w: dequantized(p, layer, w, bits, axis) for w in (O.QKV, O.OUT, O.W1, O.V, O.W2)}
        sh = {w: W[w][np.ix_(shard_rows(w, d, f, r, t), shard_cols(w, d, f, r, t))] for w in W}
        qkv = x @ sh[O.QKV]  # [n, 3 dl] = [q_r | k_r | v_r]
        heads = []
        for h in range(Hl):
            q = qkv[:, h * dh:(h + 1) * dh]
            k = qkv[:, Hl * dh + h * dh:Hl * dh + (h + 1) * dh]
            v = qkv[:, 2 * Hl * dh + h * dh:2 * Hl * dh + (h + 1) * dh]
            heads.append(O.attention(q, k, v, sample["positions"], mask))
        a = allreduce(np.concatenate(heads, axis=1) @ sh[O.OUT])  # row-parallel out_proj
        attn_taps.append(a)
        x = O.layer_norm(alpha * x + a, p.tensor(layer, 5), np.zeros(d))
        g = O.gelu(x @ sh[O.W1]) * (x @ sh[O.V])
        y = allreduce(g @ sh[O.W2])  # row-parallel w2
        ffn_taps.append(y)
        x = O.layer_norm(alpha * x + y, p.tensor(layer, 6), np.zeros(d))
    Vl = V // t
    logits_local = x @ E[r * Vl:(r + 1) * Vl].T  # vocab-sharded tied head
    gathered = [torch.zeros(logits_local.shape, dtype=torch.float64) for _ in range(t)]
    dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(logits_local)))
    logits = np.concatenate([g.numpy() for g in gathered], axis=1)
    # greedy token: (value, -index) max-allreduce, smallest id on ties
    j = int(np.argmax(logits_local[-1]))
    key = torch.tensor([logits_local[-1, j], -(r * Vl + j)], dtype=torch.float64)
    keys = [torch.zeros(2, dtype=torch.float64) for _ in range(t)]
    dist.all_gather(keys, key)
    best = max(keys, key=lambda k: (float(k[0]), float(k[1])))
    return logits, int(-best[1]), np.stack(attn_taps), np.stack(ffn_taps)


def _worker(rank, world, port, bits, axis, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = O.Params(**CFG)
        p.quantize(bits, axis)
        prefix = [6 + (37 * i + 11) % 80 for i in range(9)]
        sample = O.gmask_sample(prefix, [17, 29])
        logits, tok, at, ft = tp_forward(p, sample, rank, world, bits, axis)
        if rank == 0:
            np.savez(out, logits=logits, tok=tok, at=at, ft=ft)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bits,axis", [(8, "row"), (4, "column")])
def test_tensor_parallel_decomposition_matches_single_device(tmp_path, bits, axis):
    world = 2
    out = str(tmp_path / "tp.npz")
    mp.spawn(_worker, args=(world, free_port(), bits, axis, out), nprocs=world, join=True)
    got = np.load(out)
    p = O.Params(**CFG)
    p.quantize(bits, axis)
    prefix = [6 + (37 * i + 11) % 80 for i in range(9)]
    sample = O.gmask_sample(prefix, [17, 29])
    ref, at, ft = p.forward(sample, taps=True)
    assert np.abs(got["logits"] - ref).max() <= 1e-10 * np.abs(ref).max()
    assert np.abs(got["at"] - at).max() <= 1e-10 * np.abs(at).max()
    assert np.abs(got["ft"] - ft).max() <= 1e-10 * np.abs(ft).max()
    assert int(got["tok"]) == int(np.argmax(ref[-1]))


def test_shard_maps_partition_every_linear():
    d, f = 64, 176
    for t in (1, 2, 4, 8):
        if d % t or f % t:
            continue
        for w, (K, N) in {O.QKV: (d, 3 * d), O.OUT: (d, d), O.W1: (d, f), O.V: (d, f), O.W2: (f, d)}.items():
            cells = set()
            for r in range(t):
                rows, cols = shard_rows(w, d, f, r, t), shard_cols(w, d, f, r, t)
                block = {(int(i), int(j)) for i in rows for j in cols}
                assert not (cells & block), (w, t, r)
                cells |= block
            assert len(cells) == K * N, (w, t)


# ---- the device side of the same maps (one B200: every rank's model built in one process) ----
@pytest.mark.gpu
@pytest.mark.parametrize("t", [2, 4, 8])
@pytest.mark.parametrize("bits,axis", [(4, "column"), (4, "row"), (8, "row")])
def test_device_shards_are_slices_of_the_full_quantized_matrices(t, bits, axis):
    from paper_2210_02414_b200 import glm
    cfg = glm.GLMConfig(num_layers=1, hidden=512, num_heads=8, vocab=264)
    full = glm.Model(cfg, bits=bits, axis=axis, max_ctx=16)
    full.init_synthetic(5)
    d = cfg.hidden
    f = full.cfg.ffn_hidden or O.default_ffn_hidden(d, cfg.num_heads)
    shapes = {O.QKV: (d, 3 * d), O.OUT: (d, d), O.W1: (d, f), O.V: (d, f), O.W2: (f, d)}

    def codes(payload, rows, cols):
        return (O.unpack_int4(payload, rows * cols) if bits == 4 else payload).reshape(rows, cols)

    ref = {}
    for w, (K, N) in shapes.items():
        pl, sc = full.export_linear(0, w, K, N)
        ref[w] = (codes(pl, K, N), sc)
    for r in range(t):
        m = glm.Model(cfg, bits=bits, axis=axis, max_ctx=16, tp_rank=r, tp_size=t)
        m.init_synthetic(5)
        for w, (K, N) in shapes.items():
            rows, cols = shard_rows(w, d, f, r, t), shard_cols(w, d, f, r, t)
            pl, sc = m.export_linear(0, w, len(rows), len(cols))
            assert np.array_equal(codes(pl, len(rows), len(cols)), ref[w][0][np.ix_(rows, cols)]), (w, r)
            want = ref[w][1][rows] if axis == "row" else ref[w][1][cols]
            assert np.array_equal(sc, want), (w, r)
        del m

"""Zeropoint models on the B200: QuantPolicy{scheme = kZeropoint} (quant.hpp:53-58) applied by
quantize_model to the five linears of every layer (quant.cpp:284-311, quantize_zeropoint
:145-186, dequantization s * (code + z) :188-221). The GEMVs / GEMMs accumulate x . code; the
zero points enter every consumer as the rank-1 term zt[m] * zvec[n] (zt = sums of the fp16
activations the MMA reads times zeta). Same gates as test_gpu_model: codes / scales / zero points
bit-exact against the oracle's quantize_zeropoint, per-layer sublayer taps and logits against the
oracle forward of the dequantized zeropoint model, prefill and decode."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm
from test_gpu_model import PREFIX, check_logits, check_taps, oracle_rows

pytestmark = pytest.mark.gpu


def build_zp(bits, axis, layers=3, hidden=512, heads=8, vocab=262, seed=77, max_batch=1, tp=None):
    p = O.Params(layers, hidden, heads, vocab=vocab, seed=seed)
    m = glm.Model(glm.GLMConfig(num_layers=layers, hidden=hidden, num_heads=heads, vocab=vocab), bits=bits, axis=axis,
                  max_batch=max_batch, max_ctx=256, scheme="zeropoint")
    m.load_reference_params(lambda layer, slot: p.tensor(0, O.EMBED) if slot == "embed" else p.tensor(layer, slot))
    ref = {(layer, w): O.quantize(p.tensor(layer, w), bits, axis, scheme="zeropoint")
           for layer in range(layers) for w in range(5)}
    p.quantize(bits, axis, scheme="zeropoint")
    return p, m, ref


@pytest.mark.parametrize("bits,axis", [(4, "column"), (8, "row"), (4, "row"), (8, "whole")])
def test_zeropoint_model_matches_oracle(bits, axis):
    p, m, ref = build_zp(bits, axis)
    shapes = {0: (512, 1536), 1: (512, 512), 2: (512, 1368), 3: (512, 1368), 4: (1368, 512)}
    for (layer, w), q in ref.items():
        payload, scales = m.export_linear(layer, w, *shapes[w])
        zps = m.export_zero_points(layer, w, *shapes[w])
        assert np.array_equal(payload, q["payload"]), (layer, w)
        assert np.array_equal(scales, q["scales"]) and np.array_equal(zps, q["zero_points"]), (layer, w)
    acc = m.memory()
    groups = sum(len(q["scales"]) for q in ref.values())
    assert acc["scale_bytes"] == 2 * groups * 8  # scales + zero points (quant.cpp:352-353)
    gen = [40, 100, 200, 57, 9]
    sample = O.gmask_sample(PREFIX, gen)
    refl, at, ft, zero = oracle_rows(p, sample)
    C = sample["context_length"]
    m.enable_taps(True)
    lp = m.prefill(sample["tokens"][:C], sample["positions"][:C], C)
    pa, pf = m.taps(C)
    check_taps(pa, at, slice(0, C))
    check_taps(pf, ft, slice(0, C))
    rows = [lp]
    for j in range(len(gen) + 1):
        _, lg = m.decode_step([sample["tokens"][C + j]], [sample["positions"][C + j]])
        a, f = m.taps(1)
        check_taps(a, at[:, C + j:C + j + 1])
        check_taps(f, ft[:, C + j:C + j + 1])
        rows.append(lg)
    m.enable_taps(False)
    check_logits(np.concatenate(rows, 0).astype(np.float64), refl, zero)


def test_zeropoint_canonical_payload_equals_gpu_quantization():
    """glm_model_set_quantized_zp with the oracle's canonical matrices (incl. a constant column
    whose scale is 0 and whose value is the zero point, quant.cpp:166-171 / :209-216) gives the
    same logits as quantizing on the GPU; an absmax payload is rejected by a zeropoint model."""
    p, m, ref = build_zp(4, "column", layers=2)
    m2 = glm.Model(m.cfg, bits=4, axis="column", max_ctx=256, scheme="zeropoint")
    m2.set_embedding(p.tensor(0, O.EMBED))
    for (layer, w), q in ref.items():
        m2.set_quantized(layer, w, q["payload"], q["scales"], q["zero_points"])
    for layer in range(2):
        for which, v in ((m.LN1G, 1.0), (m.LN2G, 1.0), (m.LN1B, 0.0), (m.LN2B, 0.0)):
            m2.set_tensor(layer, which, np.full(512, v))
    sample = O.gmask_sample(PREFIX[:40])
    C = sample["context_length"]
    a = m.prefill(sample["tokens"][:C], sample["positions"][:C], C)
    b = m2.prefill(sample["tokens"][:C], sample["positions"][:C], C)
    assert np.array_equal(a, b)
    _, da = m.decode_step([3], [sample["positions"][C - 1]])
    _, db = m2.decode_step([3], [sample["positions"][C - 1]])
    assert np.array_equal(da, db)
    # constant column: scale 0, codes 0, the column's value is its zero point
    w = p.tensor(0, 1).copy()
    w[:, 7] = 0.0123
    qc = O.quantize(w, 4, "column", scheme="zeropoint")
    assert qc["scales"][7] == 0.0 and qc["zero_points"][7] == 0.0123
    m2.set_quantized(0, 1, qc["payload"], qc["scales"], qc["zero_points"])
    _, zps = m2.export_linear(0, 1, 512, 512), m2.export_zero_points(0, 1, 512, 512)
    assert zps[7] == 0.0123
    with pytest.raises(glm.ContractError):
        m2.set_quantized(0, 1, qc["payload"], qc["scales"])
    with pytest.raises(glm.ContractError):
        m2.init_synthetic(1)


def test_zeropoint_batched_decode_equals_single_sequences():
    p, m, _ = build_zp(4, "column", layers=2, max_batch=3)
    seqs = [PREFIX[:30], PREFIX[5:50], PREFIX[10:21]]
    samples = [O.gmask_sample(s) for s in seqs]
    singles = []
    for b, smp in enumerate(samples):
        C = smp["context_length"]
        m.prefill(smp["tokens"][:C], smp["positions"][:C], C, seq=b, logits=False)
    toks = [3, 3, 3]
    pos = [smp["positions"][smp["context_length"] - 1] for smp in samples]
    _, batched = m.decode_step(toks, pos)
    for b, smp in enumerate(samples):
        m1 = build_zp(4, "column", layers=2)[1]
        C = smp["context_length"]
        m1.prefill(smp["tokens"][:C], smp["positions"][:C], C, logits=False)
        _, lg = m1.decode_step([3], [pos[b]])
        singles.append(lg[0])
    np.testing.assert_allclose(batched, np.array(singles), rtol=0, atol=2e-3 * np.abs(np.array(singles)).max())

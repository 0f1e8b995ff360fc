"""PrecisionPolicy kHalfEmulated on the B200 (tensor.hpp:18-29; storage_round at model.cpp:148,
197, 213-223): the embedding rows, the attention / GeGLU sublayer outputs, every DeepNorm output
and the attention scores divided by softmax_prescale are held as binary16. Gated like
test_gpu_model.py against the oracle's forward under the same policy, which tests/
test_ref_pinned.py pins to the reference's own forward with that policy."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

pytestmark = pytest.mark.gpu
PREFIX = [6 + (37 * i + 11) % 256 for i in range(126)]


@pytest.mark.parametrize("bits,axis,prescale,hidden,heads", [(8, "row", 1.0, 512, 8), (4, "column", 8.0, 512, 8),
                                                             (4, "column", 4.0, 256, 2)])
def test_half_storage_prefill_and_decode_match_oracle(bits, axis, prescale, hidden, heads):
    p = O.Params(4, hidden, heads, vocab=262, seed=1234)
    m = glm.Model(glm.GLMConfig(num_layers=4, hidden=hidden, num_heads=heads, vocab=262), bits=bits, axis=axis,
                  max_ctx=256)
    m.load_reference_params(lambda layer, slot: p.tensor(0, O.EMBED) if slot == "embed" else p.tensor(layer, slot))
    p.quantize(bits, axis)
    m.set_precision(True, prescale)
    gen = [40, 100, 200, 57]
    sample = O.gmask_sample(PREFIX[:90], gen)  # 90-row prefix: the tcgen05 / mma.sync prefill paths
    ref, at, ft = p.forward(sample, taps=True, half=True, prescale=prescale)
    zero = p.forward(sample, zero_sublayers=True, half=True, prescale=prescale)
    wide = p.forward(sample)
    C = sample["context_length"]
    m.enable_taps(True)
    lp = m.prefill(sample["tokens"][:C], sample["positions"][:C], C)
    pa, pf = m.taps(C)
    rows = [lp]
    for layer in range(4):
        for g, r in ((pa[layer], at[layer, :C]), (pf[layer], ft[layer, :C])):
            assert np.abs(g - r).max() <= 1e-2 * np.abs(r).max(), layer
    for j in range(len(gen) + 1):
        _, lg = m.decode_step([sample["tokens"][C + j]], [sample["positions"][C + j]])
        a, f = m.taps(1)
        for layer in range(4):
            for g, r in ((a[layer, 0], at[layer, C + j]), (f[layer, 0], ft[layer, C + j])):
                assert np.abs(g - r).max() <= 1e-2 * np.abs(r).max(), (j, layer)
        rows.append(lg)
    gpu = np.concatenate(rows).astype(np.float64)
    # The sublayer taps above are the discriminating gate. The logits sit on a residual that is
    # rounded to binary16 after every DeepNorm: the GPU rounds fp32 values, the oracle f64 ones,
    # so an element within fp32 error of a rounding boundary may land one fp16 ulp (2^-11
    # relative) apart; those flips put a ~1e-4 floor under the logit difference, ~1% of
    # Delta_ref. Gate: 1e-3 of max|logit| (north_star: 1e-2), 3% of Delta_ref.
    err, delta = np.abs(gpu - ref).max(), np.abs(ref - zero).max()
    assert err <= 1e-3 * np.abs(ref).max() and err <= 3e-2 * delta, (err, delta)
    # the policy is visible: the half-storage result is closer to its own oracle than to the wide one
    assert err < np.abs(gpu - wide).max()
    m.set_precision(False)
    m.reset()
    lw = m.prefill(sample["tokens"][:C], sample["positions"][:C], C).astype(np.float64)
    assert np.abs(lw - wide[:C]).max() <= 1e-2 * np.abs(wide[:C] - p.forward(sample, zero_sublayers=True)[:C]).max()


def test_precision_contract():
    m = glm.Model(glm.GLMConfig(num_layers=1, hidden=256, num_heads=4, vocab=262), bits=8)
    with pytest.raises(glm.ContractError):
        m.set_precision(True, 0.0)

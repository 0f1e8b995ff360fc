"""Op-level block functions on the B200 (glm_deepnorm_residual / glm_geglu / glm_attention,
model.hpp:70-80) against the oracle's float64 ops, including the LayerNorm statistics on rows
whose mean is large against their spread (loaded checkpoints with big LN biases): the kernels
merge (count, mean, M2) partials instead of forming E[z^2] - mean^2, so they keep fp32
precision where the one-pass formula cancels (tensor.cpp:256-274 computes two passes)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows", [1, 3, 16, 40, 300])
@pytest.mark.parametrize("d,offset", [(512, 0.0), (512, 300.0), (12288, 0.0), (12288, 1000.0)])
def test_deepnorm_residual_matches_oracle(rows, d, offset):
    rng = np.random.default_rng(rows + d)
    alpha = 11.832159566199232
    x = (offset + rng.normal(0, 1, size=(rows, d))).astype(np.float32)
    y = rng.normal(0, 0.05, size=(rows, d)).astype(np.float32)
    g = (1 + 0.1 * rng.normal(size=d)).astype(np.float32)
    b = (0.1 * rng.normal(size=d)).astype(np.float32)
    out = glm.deepnorm_residual(x, y, alpha, g, b)
    ref = O.layer_norm(alpha * x.astype(np.float64) + y, g, b)
    # fp32 inputs of magnitude |alpha x| carry ~6e-8 * alpha * offset of rounding in z itself
    tol = 2e-5 + 4e-7 * alpha * offset
    assert np.abs(out - ref).max() <= tol * np.abs(ref).max(), np.abs(out - ref).max()


def test_geglu_op_matches_oracle():
    rng = np.random.default_rng(3)
    d, f, n = 512, 1368, 512
    qs = [glm.quantize_absmax(rng.normal(0, 0.02, size=s), 4, "column") for s in ((d, f), (d, f), (f, n))]
    lins = [glm.QLinear.from_payload(q) for q in qs]
    for M in (1, 7, 40):
        x = rng.normal(size=(M, d))
        y = glm.geglu(x, *lins)
        w1, v, w2 = (O.dequantize(q) for q in qs)
        ref = (O.gelu(x @ w1) * (x @ v)) @ w2
        assert np.abs(y - ref).max() <= 1e-2 * np.abs(ref).max()


def test_attention_op_matches_oracle_and_raises_policy_error():
    rng = np.random.default_rng(4)
    sample = O.gmask_sample([6 + i for i in range(50)], [7, 8, 9])
    mask = O.build_mask(sample)
    n = sample["n"]
    for dh in (64, 128):
        q, k, v = (rng.normal(size=(n, dh)) for _ in range(3))
        out = glm.attention(q, k, v, sample["positions"], mask)
        ref = O.attention(q, k, v, sample["positions"], mask)
        assert np.abs(out - ref).max() <= 1e-4 * np.abs(ref).max()
    dead = mask.copy()
    dead[3, :] = False
    with pytest.raises(glm.PolicyError):
        glm.attention(q, k, v, sample["positions"], dead)

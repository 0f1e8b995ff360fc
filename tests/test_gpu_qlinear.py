"""Quantized-linear parity: the W4A16/W8A16 GEMV (M <= 16) and its 16-row slabs against
y = x . dequantize(q) (quant.cpp:188-221 + tensor.cpp:135-155).

Two bars: (1) exact-arithmetic check against a float64 evaluation of the kernel's own
contract (activations rounded to fp16 after the kRow fold, fp32 scale) -> only fp32
accumulation error remains: <= 2e-6 of max|y|. The INT4 decode GEMVs run on the integer MMA
(gemv.cu k_gemv_i4 at one token, k_gemv_mk_i4 at 2..16): their contract re-quantizes each fp16
activation vector to 16-bit fixed point, x_int = rint(x * (32512 / max|x|)), per token
(k_gemv_i4) or per (token, k-split) on the plan's 64-element chunk boundaries (k_gemv_mk_i4 and
its tcgen05 twin k_gemv_tc_i4, QLinear.plan), and the products and sums are exact integers, so only the fp32 scaling and the
k-split reduction round: <= 2e-6 (one split) / 4e-6 (several) of max|y|;
(2) the reference check against the oracle's float64 x . dequantize(q),
max|dy| <= 5e-3 max|y| (fp16 activation rounding)."""
import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

pytestmark = pytest.mark.gpu


def contract_tol(ksplit):
    return 2e-6 if ksplit == 1 else 4e-6


DIGIT_Q = np.float32(32512.0)  # gemv.cu kDigitQ


def imma_activations(xh):
    """The integer-MMA GEMV's view of fp16 activations (gemv.cu digits_group): per row,
    x_int = rint(x * fp32(32512 / max|x|)) of the exact product and s_x = max|x| / 32512."""
    xh32 = xh.astype(np.float32)
    out = np.zeros(xh.shape, np.float64)
    for m in range(xh.shape[0]):
        mx = np.float32(np.abs(xh32[m]).max()) if xh.shape[1] else np.float32(0)
        if mx == 0:
            continue
        inv = np.float32(DIGIT_Q / mx)
        xi = np.rint(xh32[m].astype(np.float64) * np.float64(inv)).astype(np.int64)  # FFMA: one rounding
        assert np.abs(xi).max() <= 32512
        out[m] = xi.astype(np.float64) * np.float64(np.float32(mx / DIGIT_Q))
    return out


def kernel_view(xh, kind, ksplit, nch):
    """The activations the MMA multiplies: fp16 values (HMMA kernels), fixed point per token
    (k_gemv_i4) or fixed point per (token, k-split) with splits at chunks nch * s / ksplit."""
    if kind == "i4_single":
        return imma_activations(xh)
    if kind in ("i4_multi", "i4_tc"):
        out = np.zeros(xh.shape, np.float64)
        for s in range(ksplit):
            k0, k1 = 64 * (nch * s // ksplit), min(xh.shape[1], 64 * (nch * (s + 1) // ksplit))
            if k1 > k0:
                out[:, k0:k1] = imma_activations(xh[:, k0:k1])
        return out
    return xh.astype(np.float64)


def kernel_contract(x, q, lin):
    """float64 evaluation of what the kernel glm_qlinear picks for these M rows computes
    (DESIGN.md "Quantized linear"); returns (contract, ksplit)."""
    K, N = q["rows"], q["cols"]
    kind, ksplit, nch = lin.plan(x.shape[0])
    codes = O.codes_of(q).reshape(K, N).astype(np.float64)
    s = q["scales"]
    x32 = x.astype(np.float32)
    if q["axis"] == "row":
        S = s.max()
        fold = (s / S).astype(np.float32) if S > 0 else np.zeros(K, np.float32)
        xv = kernel_view((x32 * fold[None, :]).astype(np.float16), kind, ksplit, nch)
        return (xv @ codes) * np.float64(np.float32(S)), ksplit
    xv = kernel_view(x32.astype(np.float16), kind, ksplit, nch)
    cs = (s if q["axis"] == "column" else np.full(N, s[0])).astype(np.float32).astype(np.float64)
    return (xv @ codes) * cs[None, :], ksplit


SHAPES = [(64, 16), (512, 1536), (1368, 512), (512, 1368), (200, 90), (4096, 1024)]


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("axis", ["row", "column", "whole"])
@pytest.mark.parametrize("K,N", SHAPES)
def test_qlinear_matches_contract_and_oracle(bits, axis, K, N):
    rng = np.random.default_rng(K * 7 + N + bits)
    w = rng.normal(0, 0.02, size=(K, N))
    q = glm.quantize_absmax(w, bits, axis)
    lin = glm.QLinear.from_payload(q)
    for M in (1, 2, 3, 8, 9, 16, 37):
        x = rng.normal(0, 1, size=(M, K))
        y = lin(x).astype(np.float64)
        c, ks = kernel_contract(x, q, lin)
        assert np.abs(y - c).max() <= contract_tol(ks) * np.abs(c).max() + 1e-30, (M, np.abs(y - c).max())
        ref = x @ O.dequantize(q)
        assert np.abs(y - ref).max() <= 5e-3 * np.abs(ref).max(), (M, np.abs(y - ref).max())


def test_qlinear_glm130b_k_dimension_with_split_k():
    # K = 12288 (GLM-130B hidden) exercises ksplit > 1 and long per-warp chunk streams
    rng = np.random.default_rng(1)
    K, N = 12288, 512
    w = rng.normal(0, 5.6e-4, size=(K, N))
    for bits, axis in ((4, "column"), (8, "row")):
        q = glm.quantize_absmax(w, bits, axis)
        lin = glm.QLinear.from_payload(q)
        for M in (1, 2, 5, 16):
            x = rng.normal(0, 1, size=(M, K))
            y = lin(x).astype(np.float64)
            c, ks = kernel_contract(x, q, lin)
            if bits == 4 and M > 1:
                assert ks > 1, "the per-split activation contract is not exercised"
            assert np.abs(y - c).max() <= contract_tol(ks) * np.abs(c).max()


def test_qlinear_kernel_selection():
    """Decode GEMV dispatch (gemv.cu gemv_launch): INT4 one token on the integer-MMA
    single-token kernel, 2..16 on the integer-MMA multi-token kernel; INT8 on the fp16 kernels;
    more than 16 rows on the tcgen05 GEMM."""
    lin4 = glm.QLinear.synthetic(1, 0, 12288, 4096, 0.02, 4, "column")
    lin8 = glm.QLinear.synthetic(1, 1, 12288, 4096, 0.02, 8, "row")
    assert lin4.plan(1)[0] == "i4_single"
    for M in (2, 3, 8, 16):
        assert lin4.plan(M)[0] == "i4_multi"
        assert lin8.plan(M)[0] in ("f16_multi", "f16_tma")
    assert lin8.plan(1)[0] in ("f16_tma", "f16_multi")
    assert lin4.plan(17)[0] == lin8.plan(300)[0] == "tcgen05"
    assert lin4.plan(1)[2] == 12288 // 64


def test_qlinear_quantize_handle_equals_payload_handle():
    rng = np.random.default_rng(2)
    w = rng.normal(0, 0.01, size=(256, 128))
    a = glm.QLinear.quantize(w, 4, "row")
    b = glm.QLinear.from_payload(glm.quantize_absmax(w, 4, "row"))
    x = rng.normal(size=(4, 256))
    assert np.array_equal(a(x), b(x))
    assert np.array_equal(a.device_bytes(), b.device_bytes())


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("axis", ["row", "column", "whole"])
def test_zeropoint_qlinear_matches_oracle(bits, axis):
    """quantize_zeropoint payloads (quant.cpp:145-186) on the GPU: the MMA accumulates x.code
    and the zero points enter as a rank-1 epilogue term; constant groups (quant.cpp:209-216)
    included. Reference: the oracle's x . dequantize(q)."""
    rng = np.random.default_rng(bits * 10 + len(axis))
    K, N = 640, 384
    w = rng.normal(0.01, 0.02, size=(K, N))
    w[:, 5] = 0.037        # constant column
    w[7, :] = -0.011       # constant row
    q = O.quantize(w, bits, axis, scheme="zeropoint")
    lin = glm.QLinear.from_payload(q)
    deq = O.dequantize(q)
    for M in (1, 5, 16, 37, 300):
        x = rng.normal(0, 1, size=(M, K))
        y = lin(x).astype(np.float64)
        ref = x @ deq
        assert np.abs(y - ref).max() <= 5e-3 * np.abs(ref).max(), (M, np.abs(y - ref).max())


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("K,N", [(4096, 1024), (1024, 4096)])
def test_tcgen05_gemm_token_tile_boundaries(bits, K, N):
    """M > 16 runs the tcgen05 GEMM (qmm_tc.cu) on 256-token tiles: partial tiles (17, 255),
    an exact tile (256), a tile plus one row (257) and several tiles (600), with the planner's
    split-K (partials + reduce) and unsplit (direct scaled output) variants across the shapes."""
    rng = np.random.default_rng(bits + K)
    w = rng.normal(0, 0.02, size=(K, N))
    q = glm.quantize_absmax(w, bits, "column")
    lin = glm.QLinear.from_payload(q)
    deq = O.dequantize(q)
    for M in (17, 255, 256, 257, 600):
        x = rng.normal(0, 1, size=(M, K))
        y = lin(x).astype(np.float64)
        ref = x @ deq
        assert np.abs(y - ref).max() <= 5e-3 * np.abs(ref).max(), (M, np.abs(y - ref).max())


TC_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tests")
from paper_2210_02414_b200 import glm
from oracle import pyoracle as O
from test_gpu_qlinear import kernel_contract, contract_tol
rng = np.random.default_rng(5)
for K, N, axis in ((12288, 1024, "column"), (4096, 1536, "row"), (1368, 512, "whole")):
    w = rng.normal(0, 0.02, size=(K, N))
    q = glm.quantize_absmax(w, 4, axis)
    lin = glm.QLinear.from_payload(q)
    for M in (2, 5, 16):
        assert lin.plan(M)[0] == "i4_tc", lin.plan(M)
        x = rng.normal(0, 1, size=(M, K))
        x[0, 7] = 40.0  # one large activation: per-slice scales differ
        y = lin(x).astype(np.float64)
        c, ks = kernel_contract(x, q, lin)
        assert np.abs(y - c).max() <= contract_tol(ks) * np.abs(c).max(), (K, N, M)
        ref = x @ O.dequantize(q)
        assert np.abs(y - ref).max() <= 5e-3 * np.abs(ref).max()
print("ok")
"""


def test_qlinear_tcgen05_integer_kernel_contract():
    """The opt-in tcgen05 kind::i8 decode GEMV (gemv_tc.cu, GLM_GEMV_TC=2) computes exactly the
    integer-MMA multi-token contract (per (token, k-split) fixed point) at 2..16 tokens."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GLM_GEMV_TC="2")
    r = subprocess.run([sys.executable, "-c", TC_SCRIPT, root], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]

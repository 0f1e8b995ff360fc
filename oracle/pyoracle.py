"""ctypes binding of the CPU oracle (oracle/liboracle.so). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

AXIS = {"row": 0, "column": 1, "whole": 2}
SCHEME = {"absmax": 0, "zeropoint": 1}
QKV, OUT, W1, V, W2, EMBED = 0, 1, 2, 3, 4, 7


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Config(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("hidden", C.c_int), ("num_heads", C.c_int),
                ("ffn_hidden", C.c_int), ("vocab", C.c_int), ("init_method_std", C.c_double),
                ("layernorm_eps", C.c_double), ("deepnorm_alpha", C.c_double)]


class Sample(C.Structure):
    _fields_ = [("n", C.c_int), ("tokens", C.POINTER(C.c_int)), ("positions", C.POINTER(C.c_int)),
                ("span_id", C.POINTER(C.c_int)), ("span_offset", C.POINTER(C.c_int)),
                ("segment", C.POINTER(C.c_int)), ("span_rank", C.POINTER(C.c_int)),
                ("num_spans", C.c_int), ("unidirectional", C.c_int)]


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            subprocess.check_call(["make", "-s", "-C", _HERE])
        L = C.CDLL(path)
        d, i64, i32, p = C.c_double, C.c_int64, C.c_int, C.c_void_p
        L.or_last_error.restype = C.c_char_p
        L.or_rng_normal.argtypes = [C.c_uint64, i64, d, d, p]
        L.or_default_ffn_hidden.argtypes = [i32, i32]
        L.or_deepnorm_alpha.argtypes = [i32]
        L.or_deepnorm_alpha.restype = d
        L.or_quantize.argtypes = [p, i64, i64, i32, i32, i32, p, p, p, p]
        L.or_dequantize.argtypes = [p, i64, p, p, i64, i64, i32, i32, i32, p]
        L.or_pack_int4.argtypes = [p, i64, p]
        L.or_unpack_int4.argtypes = [p, i64, i64, p]
        L.or_group_count.argtypes = [i64, i64, i32]
        L.or_group_count.restype = i64
        L.or_params_init_reference.argtypes = [C.POINTER(Config), C.c_uint64]
        L.or_params_init_reference.restype = p
        L.or_params_init_philox.argtypes = [C.POINTER(Config), C.c_uint64]
        L.or_params_init_philox.restype = p
        L.or_params_free.argtypes = [p]
        L.or_params_shape.argtypes = [p, i32, C.POINTER(i64), C.POINTER(i64)]
        L.or_params_tensor.argtypes = [p, i32, i32]
        L.or_params_tensor.restype = C.POINTER(d)
        L.or_params_quantize.argtypes = [p, i32, i32, i32]
        L.or_params_qpayload.argtypes = [p, i32, i32, C.POINTER(C.POINTER(C.c_int8)), C.POINTER(i64),
                                         C.POINTER(C.POINTER(d)), C.POINTER(i64)]
        L.or_forward.argtypes = [p, C.POINTER(Sample), p, p, p, i32]
        L.or_rope_rotate.argtypes = [p, i64, i64, p, p]
        L.or_softmax_rows.argtypes = [p, i64, i64, p]
        L.or_layer_norm.argtypes = [p, i64, i64, p, p, d, p]
        L.or_gelu.argtypes = [p, i64, p]
        L.or_attention.argtypes = [p, p, p, i64, i64, p, p, p]
        L.or_build_mask.argtypes = [C.POINTER(Sample), p]
        L.or_half_round.argtypes = [d]
        L.or_half_round.restype = d
        L.or_philox_bf16.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_float]
        L.or_philox_bf16.restype = C.c_uint16
        L.or_gen_matrix.argtypes = [C.c_uint64, C.c_uint32, i64, i64, C.c_float, C.c_float, i64, p]
        L.or_gen_quantize.argtypes = [C.c_uint64, C.c_uint32, i64, i64, C.c_float, C.c_float, i64, i32, i32, p, p]
        L.or_qlinear_full.argtypes = [p, i64, i64, i64, p, p, i32, i32, p]
        L.or_fnv1a64.argtypes = [p, i64, C.c_uint64]
        L.or_fnv1a64.restype = C.c_uint64
        L.or_qlinear_cols.argtypes = [p, i64, i64, i64, p, p, i32, i32, p, i64, p]
        L.or_forward_policy.argtypes = [p, C.POINTER(Sample), i32, d, p, p, p, i32]
        L.or_gen_rows.argtypes = [C.c_uint64, C.c_uint32, i64, i64, i64, C.c_float, C.c_float, i64, p]
        L.or_dequantize_cols.argtypes = [p, p, i64, i64, i32, i32, p, i64, p]
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().or_last_error().decode())


def rng_normal(seed, n, mean=0.0, std=1.0):
    out = np.empty(n, np.float64)
    lib().or_rng_normal(seed, n, mean, std, _ptr(out))
    return out


def default_ffn_hidden(hidden, heads):
    return lib().or_default_ffn_hidden(hidden, heads)


def group_count(rows, cols, axis):
    return lib().or_group_count(rows, cols, AXIS[axis])


def quantize(w, bits, axis="row", scheme="absmax"):
    """quantize_absmax / quantize_zeropoint (quant.cpp:113-186). Returns dict."""
    w = np.ascontiguousarray(w, np.float64)
    rows, cols = w.shape
    nbytes = (rows * cols + 1) // 2 if bits == 4 else rows * cols
    payload = np.zeros(max(nbytes, 1), np.int8)
    g = lib().or_group_count(rows, cols, AXIS[axis])
    scales = np.zeros(max(g, 1), np.float64)
    zp = np.zeros(max(g, 1), np.float64)
    cg = np.zeros(max(g, 1), np.uint8)
    _check(lib().or_quantize(_ptr(w), rows, cols, bits, SCHEME[scheme], AXIS[axis], _ptr(payload),
                             _ptr(scales), _ptr(zp), _ptr(cg)))
    out = dict(bits=bits, axis=axis, scheme=scheme, rows=rows, cols=cols,
               payload=payload[:nbytes], scales=scales[:g])
    if scheme == "zeropoint":
        out.update(zero_points=zp[:g], constant_group=cg[:g])
    return out


def dequantize(q):
    out = np.empty((q["rows"], q["cols"]), np.float64)
    zp = q.get("zero_points")
    _check(lib().or_dequantize(_ptr(np.ascontiguousarray(q["payload"])), len(q["payload"]),
                               _ptr(np.ascontiguousarray(q["scales"])),
                               _ptr(zp) if zp is not None else None, q["rows"], q["cols"], q["bits"],
                               SCHEME[q["scheme"]], AXIS[q["axis"]], _ptr(out)))
    return out


def pack_int4(codes):
    codes = np.ascontiguousarray(codes, np.int8)
    out = np.zeros((len(codes) + 1) // 2, np.int8)
    _check(lib().or_pack_int4(_ptr(codes), len(codes), _ptr(out)))
    return out


def unpack_int4(packed, count):
    packed = np.ascontiguousarray(packed, np.int8)
    out = np.zeros(max(count, 0), np.int8)
    _check(lib().or_unpack_int4(_ptr(packed), len(packed), count, _ptr(out)))
    return out


def codes_of(q):
    if q["bits"] == 4:
        return unpack_int4(q["payload"], q["rows"] * q["cols"])
    return np.asarray(q["payload"], np.int8)


class Params:
    """init_parameters (model.cpp:69-104) or the counter-based generator."""

    def __init__(self, num_layers, hidden, num_heads, vocab=262, seed=1234, ffn_hidden=0,
                 init="reference"):
        self.cfg = Config(num_layers, hidden, num_heads, ffn_hidden, vocab, 0.0052, 1e-5, 0.0)
        fn = lib().or_params_init_reference if init == "reference" else lib().or_params_init_philox
        self.h = fn(C.byref(self.cfg), seed)
        if not self.h:
            raise OracleError(1, lib().or_last_error().decode())
        self.num_layers, self.hidden, self.num_heads, self.vocab = num_layers, hidden, num_heads, vocab
        r, c = C.c_int64(), C.c_int64()
        lib().or_params_shape(self.h, W1, C.byref(r), C.byref(c))
        self.ffn = c.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_params_free(self.h)
            self.h = None

    def shape(self, which):
        r, c = C.c_int64(), C.c_int64()
        _check(lib().or_params_shape(self.h, which, C.byref(r), C.byref(c)))
        return r.value, c.value

    def tensor(self, layer, which):
        r, c = self.shape(which)
        p = lib().or_params_tensor(self.h, layer, which)
        return np.ctypeslib.as_array(p, shape=(r, c)).copy()

    def quantize(self, bits, axis="row", scheme="absmax"):
        _check(lib().or_params_quantize(self.h, bits, SCHEME[scheme], AXIS[axis]))

    def qpayload(self, layer, which):
        pl, nb = C.POINTER(C.c_int8)(), C.c_int64()
        sc, ns = C.POINTER(C.c_double)(), C.c_int64()
        _check(lib().or_params_qpayload(self.h, layer, which, C.byref(pl), C.byref(nb), C.byref(sc),
                                        C.byref(ns)))
        return (np.ctypeslib.as_array(pl, shape=(nb.value,)).copy(),
                np.ctypeslib.as_array(sc, shape=(ns.value,)).copy())

    def forward(self, sample, taps=False, zero_sublayers=False, half=False, prescale=1.0):
        """forward (model.cpp:166-226); half / prescale: PrecisionPolicy kHalfEmulated."""
        n = sample["n"]
        logits = np.empty((n, self.vocab), np.float64)
        at = np.empty((self.num_layers, n, self.hidden)) if taps else None
        ft = np.empty((self.num_layers, n, self.hidden)) if taps else None
        s, keep = make_sample(sample)
        _check(lib().or_forward_policy(self.h, C.byref(s), int(half), float(prescale), _ptr(logits), _ptr(at),
                                       _ptr(ft), int(zero_sublayers)))
        del keep
        return (logits, at, ft) if taps else logits


def _iarr(x):
    a = np.ascontiguousarray(np.asarray(x, np.int32))
    return a, a.ctypes.data_as(C.POINTER(C.c_int))


def make_sample(sample):
    keep = []
    fields = {}
    for k in ("tokens", "positions", "span_id", "span_offset", "segment", "span_rank"):
        a, p = _iarr(sample[k])
        keep.append(a)
        fields[k] = p
    s = Sample(sample["n"], fields["tokens"], fields["positions"], fields["span_id"],
               fields["span_offset"], fields["segment"], fields["span_rank"],
               len(sample["span_rank"]), int(sample.get("unidirectional", 0)))
    return s, keep


def gmask_sample(prefix_tokens, gen_tokens=()):
    """A [gMASK] sample as corrupt_gmask lays it out (corruption.cpp:249-293):
    prefix at positions 0..P-1, [gMASK] (id 2) at P (context length C = P+1), then
    [sop] (id 3) and the generated tokens at positions P + max(0, j-1)."""
    P = len(prefix_tokens)
    toks = list(prefix_tokens) + [2] + [3] + list(gen_tokens)
    pos = list(range(P)) + [P] + [P + max(0, j - 1) for j in range(len(gen_tokens) + 1)]
    span_id = [-1] * (P + 1) + [0] * (len(gen_tokens) + 1)
    span_off = [-1] * (P + 1) + list(range(len(gen_tokens) + 1))
    n = len(toks)
    return dict(n=n, tokens=toks, positions=pos, span_id=span_id, span_offset=span_off,
                segment=[0] * n, span_rank=[0], context_length=P + 1)


def build_mask(sample):
    n = sample["n"]
    m = np.zeros((n, n), np.uint8)
    s, keep = make_sample(sample)
    _check(lib().or_build_mask(C.byref(s), _ptr(m)))
    return m.astype(bool)


def rope_rotate(x, positions):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    pa, _ = _iarr(positions)
    lib().or_rope_rotate(_ptr(x), x.shape[0], x.shape[1], _ptr(pa), _ptr(out))
    return out


def softmax_rows(x):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    _check(lib().or_softmax_rows(_ptr(x), x.shape[0], x.shape[1], _ptr(out)))
    return out


def layer_norm(x, gain, bias, eps=1e-5):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    lib().or_layer_norm(_ptr(x), x.shape[0], x.shape[1], _ptr(np.ascontiguousarray(gain, np.float64)),
                        _ptr(np.ascontiguousarray(bias, np.float64)), eps, _ptr(out))
    return out


def gelu(x):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    lib().or_gelu(_ptr(x), x.size, _ptr(out))
    return out


def attention(q, k, v, positions, mask):
    q, k, v = (np.ascontiguousarray(a, np.float64) for a in (q, k, v))
    out = np.empty_like(v)
    pa, _ = _iarr(positions)
    m = np.ascontiguousarray(mask, np.uint8)
    _check(lib().or_attention(_ptr(q), _ptr(k), _ptr(v), q.shape[0], q.shape[1], _ptr(pa), _ptr(m),
                              _ptr(out)))
    return out


def half_round(x):
    return lib().or_half_round(float(x))


def philox_bf16(seed, tensor_id, flat, sigma):
    return lib().or_philox_bf16(seed, tensor_id, flat, sigma)


def gen_matrix(seed, tensor_id, rows, cols, sigma_lo, sigma_hi=None, split_col=None):
    out = np.empty((rows, cols), np.float64)
    sigma_hi = sigma_lo if sigma_hi is None else sigma_hi
    split_col = cols if split_col is None else split_col
    lib().or_gen_matrix(seed, tensor_id, rows, cols, sigma_lo, sigma_hi, split_col, _ptr(out))
    return out


def gen_rows(seed, tensor_id, row0, nrows, cols, sigma_lo, sigma_hi=None, split_col=None):
    """Rows [row0, row0 + nrows) of gen_matrix(seed, tensor_id, ., cols, ...)."""
    out = np.empty((nrows, cols), np.float64)
    sigma_hi = sigma_lo if sigma_hi is None else sigma_hi
    split_col = cols if split_col is None else split_col
    lib().or_gen_rows(seed, tensor_id, row0, nrows, cols, sigma_lo, sigma_hi, split_col, _ptr(out))
    return out


def dequantize_cols(q, cols):
    """dequantize(q) (quant.cpp:188-221, absmax) restricted to output columns `cols`: [rows, len(cols)]."""
    cols = np.ascontiguousarray(cols, np.int64)
    out = np.empty((q["rows"], len(cols)), np.float64)
    _check(lib().or_dequantize_cols(_ptr(np.ascontiguousarray(q["payload"])), _ptr(np.ascontiguousarray(q["scales"])),
                                    q["rows"], q["cols"], q["bits"], AXIS[q["axis"]], _ptr(cols), len(cols), _ptr(out)))
    return out


def block_forward(x, W, ln, positions, mask, num_heads, alpha, eps=1e-5):
    """One GLM block (model.cpp:198-224) in float64 on hidden states x [n, d]: W = dense
    (dequantized) [in, out] matrices indexed QKV / OUT / W1 / V / W2; ln = (g1, b1, g2, b2);
    mask [n, n] bool. Per head (model.cpp:141-152): RoPE(q), RoPE(k) (tensor.cpp:335-394,
    or_rope_rotate), scores / sqrt(dh), invisible -> -inf, wide softmax (tensor.cpp:221-254),
    P . v; then out_proj, deepnorm_residual (model.cpp:125-131), geglu (model.cpp:133-135),
    deepnorm_residual. Returns (out, attention sublayer output, GeGLU sublayer output)."""
    x = np.ascontiguousarray(x, np.float64)
    n, d = x.shape
    dh = d // num_heads
    qkv = x @ W[QKV]
    pos_all = np.tile(np.asarray(positions, np.int32), num_heads)

    def heads(a):  # [n, d] -> [H * n, dh] (head-major rows)
        return np.ascontiguousarray(a.reshape(n, num_heads, dh).transpose(1, 0, 2).reshape(num_heads * n, dh))

    rq = rope_rotate(heads(qkv[:, :d]), pos_all).reshape(num_heads, n, dh)
    rk = rope_rotate(heads(qkv[:, d:2 * d]), pos_all).reshape(num_heads, n, dh)
    vh = heads(qkv[:, 2 * d:]).reshape(num_heads, n, dh)
    sc = np.einsum("hid,hjd->hij", rq, rk) / np.sqrt(dh)
    sc[:, ~np.asarray(mask, bool)] = -np.inf
    if np.isneginf(sc.max(axis=2)).any():
        raise OracleError(4, "[tensorcore] softmax row is entirely -inf; no distribution is defined")
    sc = np.exp(sc - sc.max(axis=2, keepdims=True))
    sc /= sc.sum(axis=2, keepdims=True)
    att = np.einsum("hij,hjd->hid", sc, vh).transpose(1, 0, 2).reshape(n, d)
    attn = att @ W[OUT]
    g1, b1, g2, b2 = ln
    h = layer_norm(alpha * x + attn, g1, b1, eps)
    ff = (gelu(h @ W[W1]) * (h @ W[V])) @ W[W2]
    out = layer_norm(alpha * h + ff, g2, b2, eps)
    return out, attn, ff


def qlinear_cols(x, q, cols):
    x = np.ascontiguousarray(x, np.float64)
    M, K = x.shape
    cols = np.ascontiguousarray(cols, np.int64)
    y = np.empty((M, len(cols)), np.float64)
    _check(lib().or_qlinear_cols(_ptr(x), M, K, q["cols"], _ptr(np.ascontiguousarray(q["payload"])),
                                 _ptr(np.ascontiguousarray(q["scales"])), q["bits"], AXIS[q["axis"]],
                                 _ptr(cols), len(cols), _ptr(y)))
    return y


def fnv1a64(data, h=1469598103934665603):
    """FNV-1a-64 (offset 1469598103934665603, prime 1099511628211), SURVEY §8c hashes."""
    a = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if isinstance(data, (bytes, bytearray))
                             else np.asarray(data).view(np.uint8).ravel())
    return lib().or_fnv1a64(_ptr(a), a.size, h)


def gen_quantize(seed, tensor_id, K, N, bits, axis, sigma_lo, sigma_hi=None, split_col=None):
    """Counter-based weights quantized with quantize_absmax, streamed (no double matrix)."""
    sigma_hi = sigma_lo if sigma_hi is None else sigma_hi
    split_col = N if split_col is None else split_col
    nb = (K * N + 1) // 2 if bits == 4 else K * N
    payload = np.empty(nb, np.int8)
    scales = np.empty(K if axis == "row" else N, np.float64)
    _check(lib().or_gen_quantize(seed, tensor_id, K, N, sigma_lo, sigma_hi, split_col, bits, AXIS[axis],
                                 _ptr(payload), _ptr(scales)))
    return dict(bits=bits, scheme="absmax", axis=axis, rows=K, cols=N, payload=payload, scales=scales)


def qlinear_full(x, q):
    x = np.ascontiguousarray(np.atleast_2d(x), np.float64)
    y = np.empty((x.shape[0], q["cols"]), np.float64)
    _check(lib().or_qlinear_full(_ptr(x), x.shape[0], q["rows"], q["cols"], _ptr(np.ascontiguousarray(q["payload"])),
                                 _ptr(np.ascontiguousarray(q["scales"])), q["bits"], AXIS[q["axis"]], _ptr(y)))
    return y


def mask_sample(tokens, spans, permutation, mask_id=1, sop_id=3):
    """A [MASK] blank-infilling sample laid out as corrupt_mask does (corruption.cpp:190-247):
    Part A = the text with each span replaced by one [MASK] placeholder (sequential positions),
    Part B = the spans in `permutation` order, each [sop] + its tokens, every Part-B input
    carrying its span's placeholder position. spans = [(start, length), ...] sorted by start.
    Token ids: [MASK] = 1, [sop] = 3 (corruption.hpp:17-19)."""
    toks, pos, span_id, span_off = [], [], [], []
    placeholder = []
    cursor = 0
    for (start, length) in spans:
        while cursor < start:
            toks.append(tokens[cursor]); pos.append(len(toks) - 1); span_id.append(-1); span_off.append(-1)
            cursor += 1
        placeholder.append(len(toks))
        toks.append(mask_id); pos.append(len(toks) - 1); span_id.append(-1); span_off.append(-1)
        cursor = start + length
    while cursor < len(tokens):
        toks.append(tokens[cursor]); pos.append(len(toks) - 1); span_id.append(-1); span_off.append(-1)
        cursor += 1
    C = len(toks)
    rank = [0] * len(spans)
    for r, s in enumerate(permutation):
        rank[s] = r
    for s in permutation:
        start, length = spans[s]
        for j in range(length + 1):
            toks.append(sop_id if j == 0 else tokens[start + j - 1])
            pos.append(placeholder[s]); span_id.append(s); span_off.append(j)
    n = len(toks)
    return dict(n=n, tokens=toks, positions=pos, span_id=span_id, span_offset=span_off, segment=[0] * n,
                span_rank=rank, context_length=C)

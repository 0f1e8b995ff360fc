"""ctypes binding of include/glm130b.h with the reference's names and error classes.

Mirrors the glmlab operator API (quantize_absmax / quantize_zeropoint / dequantize /
pack_int4 / unpack_int4, quant.hpp:44-51; GLMConfig + forward, model.hpp:15-91) so the
parity tests read like the reference's own tests. All compute happens in
libglm130b.so on the GPU; there is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

LIB_PATH = os.environ.get("GLM130B_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libglm130b.so")
_LIB = None

AXIS = {"row": 0, "column": 1, "whole": 2}
SCHEME = {"absmax": 0, "zeropoint": 1}
DTYPE = {np.dtype(np.float64): 0, np.dtype(np.float32): 1}
GLM_BF16 = 2


class GLMError(RuntimeError):
    """glmlab::Error (common.hpp:28-36): message carries the "[module] ..." tag."""
    code = -1


class ContractError(GLMError):
    code = 1


class DimensionError(GLMError):
    code = 2


class FormatError(GLMError):
    code = 3


class PolicyError(GLMError):
    code = 4


class CudaError(GLMError):
    code = 5


class NcclError(GLMError):
    code = 6


_ERRORS = {c.code: c for c in (ContractError, DimensionError, FormatError, PolicyError, CudaError, NcclError)}


class _Config(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("hidden", C.c_int), ("num_heads", C.c_int),
                ("ffn_hidden", C.c_int), ("vocab", C.c_int), ("init_method_std", C.c_double),
                ("layernorm_eps", C.c_double), ("deepnorm_alpha", C.c_double)]


class _Memory(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("element_count", "quant_payload_bytes", "scale_bytes",
                                         "half_baseline_bytes", "wide_baseline_bytes",
                                         "device_weight_bytes", "device_head_bytes", "device_kv_bytes")]


# name -> (restype, argtypes); every symbol declared in include/glm130b.h
P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
SIGNATURES = {
    "glm_last_error": (C.c_char_p, []),
    "glm_version": (C.c_char_p, []),
    "glm_group_count": (I64, [I64, I64, I32]),
    "glm_payload_bytes": (I64, [I64, I64, I32]),
    "glm_quantize_weight": (I32, [P, I32, I64, I64, I32, I32, I32, P, P, P, P]),
    "glm_quantize_weight_device": (I32, [P, I32, I64, I64, I32, I32, I32, P, P, P, P, P]),
    "glm_dequantize": (I32, [P, I64, P, P, I64, I64, I32, I32, I32, P]),
    "glm_pack_int4": (I32, [P, I64, P]),
    "glm_unpack_int4": (I32, [P, I64, I64, P]),
    "glm_qweight_create": (I32, [P, P, I64, I64, I32, I32, C.POINTER(P)]),
    "glm_qweight_quantize": (I32, [P, I32, I64, I64, I32, I32, C.POINTER(P)]),
    "glm_qweight_synthetic": (I32, [C.c_uint64, C.c_uint32, I64, I64, C.c_float, I32, I32, C.POINTER(P)]),
    "glm_qweight_destroy": (I32, [P]),
    "glm_qweight_export": (I32, [P, P, P]),
    "glm_qweight_device_bytes": (I64, [P]),
    "glm_qweight_device_copy": (I32, [P, P]),
    "glm_debug_qmm_trace": (I32, [P]),
    "glm_debug_gemv_plan": (I32, [P, I64, P]),
    "glm_debug_plan_shape": (I32, [I64, I64, I32, I64, P]),
    "glm_qlinear": (I32, [P, P, I64, P, P]),
    "glm_qlinear_host": (I32, [P, P, I64, P]),
    "glm_qlinear_bench": (I32, [P, I64, I32, I32, C.POINTER(D)]),
    "glm_model_create": (I32, [C.POINTER(_Config), I32, I32, I32, I32, I32, I32, I32, C.POINTER(P)]),
    "glm_model_destroy": (I32, [P]),
    "glm_debug_trace_start": (I32, [I64]),
    "glm_debug_trace_stop": (I32, [P, I64, P]),
    "glm_model_set_quantized": (I32, [P, I32, I32, P, I64, P, I64]),
    "glm_model_set_scheme": (I32, [P, I32]),
    "glm_model_set_quantized_zp": (I32, [P, I32, I32, P, I64, P, P, I64]),
    "glm_model_export_zero_points": (I32, [P, I32, I32, P]),
    "glm_model_get_config": (I32, [P, P]),
    "glm_model_load_quantized": (I32, [C.c_char_p, I32, I32, I32, I32, I32, P]),
    "glm_qweight_create_ex": (I32, [P, P, P, I64, I64, I32, I32, I32, P]),
    "glm_model_prefill_batch": (I32, [P, I32, P, P, P, P, P, P]),
    "glm_tp_unique_id": (I32, [P]),
    "glm_tp_emulated_group_create": (I32, [I32, C.POINTER(P)]),
    "glm_tp_emulated_group_destroy": (I32, [P]),
    "glm_model_init_comm_emulated": (I32, [P, P]),
    "glm_model_init_comm": (I32, [P, P]),
    "glm_model_set_embedding": (I32, [P, P]),
    "glm_model_set_embedding_rows": (I32, [P, I64, I64, P]),
    "glm_model_set_tensor": (I32, [P, I32, I32, P]),
    "glm_model_init_synthetic": (I32, [P, C.c_uint64]),
    "glm_model_export_linear": (I32, [P, I32, I32, P, P]),
    "glm_model_memory": (I32, [P, C.POINTER(_Memory)]),
    "glm_model_prefill": (I32, [P, I32, P, P, I32, I32, P]),
    "glm_model_decode_step": (I32, [P, I32, P, P, P, P]),
    "glm_model_cached_length": (I32, [P, I32]),
    "glm_model_reset": (I32, [P]),
    "glm_model_enable_taps": (I32, [P, I32]),
    "glm_model_get_taps": (I32, [P, P, P]),
    "glm_model_zero_sublayers": (I32, [P, I32]),
    "glm_model_set_precision": (I32, [P, I32, D]),
    "glm_block_forward": (I32, [P, I32, I32, I32, P, P, I32, I32, P]),
    "glm_block_forward_host": (I32, [P, I32, I32, I32, P, P, I32, I32]),
    "glm_deepnorm_residual": (I32, [P, P, I64, I64, D, P, P, D, P, P]),
    "glm_deepnorm_residual_host": (I32, [P, P, I64, I64, D, P, P, D, P]),
    "glm_geglu": (I32, [P, P, P, P, I64, P, P]),
    "glm_geglu_host": (I32, [P, P, P, P, I64, P]),
    "glm_attention": (I32, [P, P, P, I64, I64, P, P, P, P]),
    "glm_attention_host": (I32, [P, P, P, I64, I64, P, P, P]),
    "glm_model_bench_decode": (I32, [P, I32, I32, I32, C.POINTER(D), C.POINTER(D), C.POINTER(I32)]),
}


def lib():
    """Loads libglm130b.so (raises if it was not built: there is no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()) first; "
                              "this package has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def _check(rc):
    if rc != 0:
        msg = lib().glm_last_error().decode()
        raise _ERRORS.get(rc, GLMError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def group_count(rows, cols, axis="row"):
    return lib().glm_group_count(rows, cols, AXIS[axis])


def payload_bytes(rows, cols, bits):
    return lib().glm_payload_bytes(rows, cols, bits)


def _weights(w):
    w = np.asarray(w)
    if w.dtype == np.uint16:  # raw bf16 bits
        return np.ascontiguousarray(w), GLM_BF16
    if w.dtype not in (np.float64, np.float32):
        w = w.astype(np.float64)
    return np.ascontiguousarray(w), DTYPE[w.dtype]


def quantize_weight(w, bits, axis="row", scheme="absmax"):
    """QuantizedMatrix as a dict (quant.hpp:26-42), computed on the GPU."""
    w, dt = _weights(w)
    if w.ndim != 2:
        raise DimensionError("[quantlab] expected a matrix")
    rows, cols = w.shape
    g = group_count(rows, cols, axis)
    pb = payload_bytes(rows, cols, bits) if bits in (4, 8) else 0
    payload = np.zeros(max(pb, 1), np.int8)
    scales = np.zeros(max(g, 1), np.float64)
    zp = np.zeros(max(g, 1), np.float64)
    cg = np.zeros(max(g, 1), np.uint8)
    _check(lib().glm_quantize_weight(_p(w), dt, rows, cols, bits, SCHEME[scheme], AXIS[axis], _p(payload),
                                     _p(scales), _p(zp), _p(cg)))
    q = dict(bits=bits, scheme=scheme, axis=axis, rows=rows, cols=cols, payload=payload[:pb], scales=scales[:g])
    if scheme == "zeropoint":
        q.update(zero_points=zp[:g], constant_group=cg[:g])
    return q


def quantize_absmax(w, bits, axis="row"):
    return quantize_weight(w, bits, axis, "absmax")


def quantize_zeropoint(w, bits, axis="row"):
    return quantize_weight(w, bits, axis, "zeropoint")


def dequantize(q):
    out = np.empty((q["rows"], q["cols"]), np.float64)
    payload = np.ascontiguousarray(q["payload"], np.int8)
    scales = np.ascontiguousarray(q["scales"], np.float64)
    zp = q.get("zero_points")
    zp = None if zp is None else np.ascontiguousarray(zp, np.float64)
    _check(lib().glm_dequantize(_p(payload), len(payload), _p(scales), _p(zp), q["rows"], q["cols"], q["bits"],
                                SCHEME[q["scheme"]], AXIS[q["axis"]], _p(out)))
    return out


def pack_int4(codes):
    codes = np.ascontiguousarray(codes, np.int8)
    out = np.zeros((len(codes) + 1) // 2, np.int8)
    _check(lib().glm_pack_int4(_p(codes), len(codes), _p(out)))
    return out


def unpack_int4(packed, count):
    packed = np.ascontiguousarray(packed, np.int8)
    out = np.zeros(max(count, 0), np.int8)
    _check(lib().glm_unpack_int4(_p(packed), len(packed), count, _p(out)))
    return out


def deepnorm_residual(x, y, alpha, gain, bias, eps=1e-5):
    """deepnorm_residual (model.hpp:70-71, model.cpp:125-131) on the GPU: LN(alpha x + y)."""
    x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
    y = np.ascontiguousarray(np.atleast_2d(y), np.float32)
    if x.shape != y.shape:
        raise DimensionError("[glmmodel] deepnorm_residual operands must share a shape")
    g = np.ascontiguousarray(gain, np.float32)
    b = np.ascontiguousarray(bias, np.float32)
    out = np.empty_like(x)
    _check(lib().glm_deepnorm_residual_host(_p(x), _p(y), x.shape[0], x.shape[1], alpha, _p(g), _p(b), eps, _p(out)))
    return out


def geglu(x, w1, v, w2):
    """geglu (model.hpp:74, model.cpp:133-135) with quantized W1, V, W2 (QLinear handles)."""
    x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
    y = np.empty((x.shape[0], w2.cols), np.float32)
    _check(lib().glm_geglu_host(w1.h, v.h, w2.h, _p(x), x.shape[0], _p(y)))
    return y


def attention(q, k, v, positions, mask):
    """Single-head attention (model.hpp:78-80, model.cpp:137-152) with a boolean mask."""
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    pos = np.ascontiguousarray(positions, np.int32)
    mk = np.ascontiguousarray(mask, np.uint8)
    n, dh = q.shape
    out = np.empty((n, dh), np.float32)
    _check(lib().glm_attention_host(_p(q), _p(k), _p(v), n, dh, _p(pos), _p(mk), _p(out)))
    return out


class QLinear:
    """Quantized linear y = x . dequantize(q) on the B200 (device layout handle)."""

    def __init__(self, handle, rows, cols, bits, axis):
        self.h, self.rows, self.cols, self.bits, self.axis = handle, rows, cols, bits, axis

    @classmethod
    def from_payload(cls, q):
        h = C.c_void_p()
        payload = np.ascontiguousarray(q["payload"], np.int8)
        scales = np.ascontiguousarray(q["scales"], np.float64)
        if q.get("scheme", "absmax") == "zeropoint":
            zp = np.ascontiguousarray(q["zero_points"], np.float64)
            _check(lib().glm_qweight_create_ex(_p(payload), _p(scales), _p(zp), q["rows"], q["cols"], q["bits"],
                                               SCHEME["zeropoint"], AXIS[q["axis"]], C.byref(h)))
        else:
            _check(lib().glm_qweight_create(_p(payload), _p(scales), q["rows"], q["cols"], q["bits"],
                                            AXIS[q["axis"]], C.byref(h)))
        return cls(h, q["rows"], q["cols"], q["bits"], q["axis"])

    @classmethod
    def quantize(cls, w, bits, axis="row"):
        w, dt = _weights(w)
        h = C.c_void_p()
        _check(lib().glm_qweight_quantize(_p(w), dt, w.shape[0], w.shape[1], bits, AXIS[axis], C.byref(h)))
        return cls(h, w.shape[0], w.shape[1], bits, axis)

    @classmethod
    def synthetic(cls, seed, tensor_id, rows, cols, sigma, bits, axis="column"):
        h = C.c_void_p()
        _check(lib().glm_qweight_synthetic(seed, tensor_id, rows, cols, sigma, bits, AXIS[axis], C.byref(h)))
        return cls(h, rows, cols, bits, axis)

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.glm_qweight_destroy(self.h)
            self.h = None

    def export(self):
        pb = payload_bytes(self.rows, self.cols, self.bits)
        payload = np.zeros(pb, np.int8)
        scales = np.zeros(group_count(self.rows, self.cols, self.axis), np.float64)
        _check(lib().glm_qweight_export(self.h, _p(payload), _p(scales)))
        return dict(bits=self.bits, scheme="absmax", axis=self.axis, rows=self.rows, cols=self.cols,
                    payload=payload, scales=scales)

    def device_bytes(self):
        n = lib().glm_qweight_device_bytes(self.h)
        out = np.zeros(n, np.uint8)
        _check(lib().glm_qweight_device_copy(self.h, _p(out)))
        return out

    def __call__(self, x):
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        y = np.empty((x.shape[0], self.cols), np.float32)
        _check(lib().glm_qlinear_host(self.h, _p(x), x.shape[0], _p(y)))
        return y

    GEMV_KINDS = ("f16_single", "i4_single", "i4_multi", "f16_multi", "f16_tma", "tcgen05", "i4_tc")

    def plan(self, M):
        """(kernel, ksplit, nch) glm_qlinear uses for M rows (glm_debug_gemv_plan)."""
        out = np.zeros(3, np.int32)
        _check(lib().glm_debug_gemv_plan(self.h, M, _p(out)))
        return self.GEMV_KINDS[out[0]], int(out[1]), int(out[2])

    @classmethod
    def plan_for(cls, rows, cols, bits, M):
        """(kernel, ksplit, nch, grid) of a [rows, cols] weight for M rows (host only)."""
        out = np.zeros(4, np.int32)
        _check(lib().glm_debug_plan_shape(rows, cols, bits, M, _p(out)))
        return cls.GEMV_KINDS[out[0]], int(out[1]), int(out[2]), int(out[3])

    def bench(self, M, iters=20, flush=True):
        us = C.c_double()
        _check(lib().glm_qlinear_bench(self.h, M, iters, int(flush), C.byref(us)))
        return us.value


@dataclass
class GLMConfig:
    """GLMConfig (model.hpp:15-31)."""
    num_layers: int = 2
    hidden: int = 64
    num_heads: int = 4
    ffn_hidden: int = 0
    vocab: int = 262
    init_method_std: float = 0.0052
    layernorm_eps: float = 1e-5
    deepnorm_alpha: float = 0.0

    def c(self):
        return _Config(self.num_layers, self.hidden, self.num_heads, self.ffn_hidden, self.vocab,
                       self.init_method_std, self.layernorm_eps, self.deepnorm_alpha)


def gmask_layout(prefix_len, n_gen):
    """Positions of a [gMASK] sample (corruption.cpp:266-290): prefix 0..P-1, [gMASK] at P,
    generation input j at P + max(0, j-1). Returns (positions, context_length)."""
    P = prefix_len
    pos = list(range(P)) + [P] + [P + max(0, j - 1) for j in range(n_gen)]
    return pos, P + 1


def tp_unique_id() -> bytes:
    """128-byte NCCL unique id (glm_tp_unique_id); rank 0 creates it, every rank passes it
    to Model.init_comm."""
    uid = np.zeros(128, np.uint8)
    _check(lib().glm_tp_unique_id(_p(uid)))
    return uid.tobytes()


class EmulatedGroup:
    """Single-GPU test group of tensor-parallel rank-models (glm_tp_emulated_group_create):
    the same sharded model code, with collectives emulated by stream-ordered sums behind a
    host barrier. Each rank must be driven from its own thread (see run_ranks)."""

    def __init__(self, size):
        h = C.c_void_p()
        _check(lib().glm_tp_emulated_group_create(size, C.byref(h)))
        self.h, self.size = h, size

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.glm_tp_emulated_group_destroy(self.h)
            self.h = None


def run_ranks(fns):
    """Run fns[r]() on one thread per rank (ctypes releases the GIL inside the library);
    returns the results in rank order and re-raises the first failure."""
    import threading
    out, err = [None] * len(fns), [None] * len(fns)

    def body(r):
        try:
            out[r] = fns[r]()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    ts = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out


class Model:
    """GLM model on the B200: quantized linears, fp32 residual stream, KV cache."""

    QKV, OUT, W1, V, W2, LN1G, LN1B, LN2G, LN2B = range(9)

    def __init__(self, cfg: GLMConfig, bits=8, axis="row", max_batch=1, max_ctx=256, head_bf16=False,
                 tp_rank=0, tp_size=1, scheme="absmax"):
        self.cfg = cfg
        self.bits, self.axis, self.scheme = bits, axis, scheme
        self._c = cfg.c()
        h = C.c_void_p()
        _check(lib().glm_model_create(C.byref(self._c), bits, AXIS[axis], max_batch, max_ctx, int(head_bf16),
                                      tp_rank, tp_size, C.byref(h)))
        self.h = h
        if scheme != "absmax":  # QuantPolicy::scheme (quant.hpp:53-58)
            _check(lib().glm_model_set_scheme(self.h, SCHEME[scheme]))

    def __del__(self):
        if getattr(self, "h", None) and _LIB is not None:
            _LIB.glm_model_destroy(self.h)
            self.h = None

    @classmethod
    def load_quantized(cls, directory, max_batch=1, max_ctx=256, head_bf16=False, tp_rank=0, tp_size=1):
        """load_quantized_model (quant.cpp:450-491) of a reference checkpoint directory."""
        h = C.c_void_p()
        _check(lib().glm_model_load_quantized(os.fsencode(directory), max_batch, max_ctx, int(head_bf16), tp_rank,
                                              tp_size, C.byref(h)))
        self = cls.__new__(cls)
        self.h = h
        cfg = _Config()
        import json
        with open(os.path.join(directory, "manifest.json")) as fh:
            man = json.load(fh)
        jc, jp = man["config"], man["policy"]
        self.cfg = GLMConfig(num_layers=jc["num_layers"], hidden=jc["hidden"], num_heads=jc["num_heads"],
                             ffn_hidden=jc["ffn_hidden"], vocab=jc["vocab"])
        self.bits, self.axis, self.scheme = jp["bits"], jp["axis"], jp.get("scheme", "absmax")
        self._c = self.cfg.c()
        del cfg
        return self

    def set_quantized(self, layer, which, payload, scales, zero_points=None):
        """A canonical QuantizedMatrix (payload int8 bytes, FP64 scales [, FP64 zero points of a
        zeropoint model]) of linear `which`."""
        payload = np.ascontiguousarray(payload, np.int8)
        scales = np.ascontiguousarray(scales, np.float64)
        if zero_points is not None:
            zps = np.ascontiguousarray(zero_points, np.float64)
            if zps.size != scales.size:
                raise FormatError("[quantlab] zero point count differs from the scale count")
            _check(lib().glm_model_set_quantized_zp(self.h, layer, which, _p(payload), payload.size, _p(scales), _p(zps),
                                                    scales.size))
            return
        _check(lib().glm_model_set_quantized(self.h, layer, which, _p(payload), payload.size, _p(scales), scales.size))

    def init_comm_emulated(self, group: "EmulatedGroup"):
        """Join a single-GPU emulated rank group (test hook; call from this rank's thread)."""
        _check(lib().glm_model_init_comm_emulated(self.h, group.h))

    def init_comm(self, unique_id: bytes):
        """Join the tensor-parallel group (NCCL over NVLink); no-op at tp_size == 1."""
        uid = np.frombuffer(bytes(unique_id), np.uint8).copy()
        if uid.size != 128:
            raise ContractError("[glmmodel] NCCL unique id must be 128 bytes")
        _check(lib().glm_model_init_comm(self.h, _p(uid)))

    # -- weights --
    def set_embedding(self, e):
        e = np.ascontiguousarray(e, np.float64)
        _check(lib().glm_model_set_embedding(self.h, _p(e)))

    def set_tensor(self, layer, which, values):
        v = np.ascontiguousarray(values, np.float64)
        _check(lib().glm_model_set_tensor(self.h, layer, which, _p(v)))

    def load_reference_params(self, tensor_fn):
        """tensor_fn(layer, slot) -> float64 array; slot in QKV..W2 and 'embed'."""
        self.set_embedding(tensor_fn(0, "embed"))
        d = self.cfg.hidden
        for layer in range(self.cfg.num_layers):
            for which in (self.QKV, self.OUT, self.W1, self.V, self.W2):
                self.set_tensor(layer, which, tensor_fn(layer, which))
            for which in (self.LN1G, self.LN2G):
                self.set_tensor(layer, which, np.ones(d))
            for which in (self.LN1B, self.LN2B):
                self.set_tensor(layer, which, np.zeros(d))

    def init_synthetic(self, seed):
        _check(lib().glm_model_init_synthetic(self.h, seed))

    def export_linear(self, layer, which, rows, cols):
        payload = np.zeros(payload_bytes(rows, cols, self.bits), np.int8)
        scales = np.zeros(group_count(rows, cols, self.axis), np.float64)
        _check(lib().glm_model_export_linear(self.h, layer, which, _p(payload), _p(scales)))
        return payload, scales

    def export_zero_points(self, layer, which, rows, cols):
        zps = np.zeros(group_count(rows, cols, self.axis), np.float64)
        _check(lib().glm_model_export_zero_points(self.h, layer, which, _p(zps)))
        return zps

    def memory(self):
        m = _Memory()
        _check(lib().glm_model_memory(self.h, C.byref(m)))
        return {n: getattr(m, n) for n, _ in _Memory._fields_}

    # -- inference --
    def prefill(self, tokens, positions, context_length=None, seq=0, logits=True):
        tokens = np.ascontiguousarray(tokens, np.int32)
        positions = np.ascontiguousarray(positions, np.int32)
        n = len(tokens)
        out = np.empty((n, self.cfg.vocab), np.float32) if logits else None
        _check(lib().glm_model_prefill(self.h, seq, _p(tokens), _p(positions), n,
                                       n if context_length is None else context_length, _p(out)))
        return out

    def prefill_batch(self, samples, logits=True):
        """Packed prefill (pack_samples, corruption.cpp:295-334): samples = [(seq, tokens,
        positions, context_length), ...]; one batch through the linears, per-sample attention."""
        seqs = np.array([s[0] for s in samples], np.int32)
        lens = np.array([len(s[1]) for s in samples], np.int32)
        ctx = np.array([s[3] for s in samples], np.int32)
        toks = np.ascontiguousarray(np.concatenate([np.asarray(s[1], np.int32) for s in samples]))
        poss = np.ascontiguousarray(np.concatenate([np.asarray(s[2], np.int32) for s in samples]))
        out = np.zeros((int(lens.sum()), self.cfg.vocab), np.float32) if logits else None
        _check(lib().glm_model_prefill_batch(self.h, len(samples), _p(seqs), _p(lens), _p(ctx), _p(toks), _p(poss),
                                             _p(out)))
        return out

    def decode_step(self, tokens, positions, logits=True):
        tokens = np.ascontiguousarray(np.atleast_1d(tokens), np.int32)
        positions = np.ascontiguousarray(np.atleast_1d(positions), np.int32)
        b = len(tokens)
        nxt = np.empty(b, np.int32)
        out = np.empty((b, self.cfg.vocab), np.float32) if logits else None
        _check(lib().glm_model_decode_step(self.h, b, _p(tokens), _p(positions), _p(nxt), _p(out)))
        return nxt, out

    def block_forward(self, layer, x, positions, mode="prefill", seq=0, context_length=None):
        """glm_block_forward_host: one GLM block (model.cpp:198-224) of `layer` on hidden
        states x [n, hidden]; prefill fills the layer's KV cache of `seq`, decode appends row b
        to sequence b. Returns the block output."""
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32).copy()
        pos = np.ascontiguousarray(np.atleast_1d(positions), np.int32)
        n = x.shape[0]
        ctx = n if context_length is None else context_length
        _check(lib().glm_block_forward_host(self.h, layer, {"prefill": 0, "decode": 1}[mode], seq, _p(x), _p(pos), n,
                                            ctx))
        return x

    def cached_length(self, seq=0):
        return lib().glm_model_cached_length(self.h, seq)

    def reset(self):
        _check(lib().glm_model_reset(self.h))

    def enable_taps(self, on=True):
        _check(lib().glm_model_enable_taps(self.h, int(on)))

    def taps(self, rows):
        a = np.empty((self.cfg.num_layers, rows, self.cfg.hidden), np.float32)
        f = np.empty_like(a)
        _check(lib().glm_model_get_taps(self.h, _p(a), _p(f)))
        return a, f

    def set_precision(self, half_storage=False, softmax_prescale=1.0):
        """PrecisionPolicy (tensor.hpp:18-29): binary16 storage emulation at the reference's
        storage_round points, attention scores stored / softmax_prescale."""
        _check(lib().glm_model_set_precision(self.h, int(half_storage), float(softmax_prescale)))

    def zero_sublayers(self, on=True):
        _check(lib().glm_model_zero_sublayers(self.h, int(on)))

    def bench_decode(self, batch, steps, warmup=3):
        ms, gemv, launches = C.c_double(), C.c_double(), C.c_int()
        _check(lib().glm_model_bench_decode(self.h, batch, steps, warmup, C.byref(ms), C.byref(gemv),
                                            C.byref(launches)))
        return ms.value, gemv.value, launches.value

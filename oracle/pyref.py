"""ctypes binding of oracle/_ref/libglmref.so: the REFERENCE's own sources (glmlab,
/root/reference/proj/src) built with the test-infrastructure stand-ins (oracle/build_ref.sh).
TEST INFRASTRUCTURE ONLY: tests/ use it to pin the oracle against the reference itself, and
bench.py's CPU baseline / reference arm time the reference's path with it."""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(_HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "libglmref.so")
_LIB = None
AXIS = {"row": 0, "column": 1, "whole": 2}


def available():
    return os.path.exists(LIB_PATH)


def build():
    """oracle/build_ref.sh (needs /root/reference; keeps a prebuilt _ref otherwise)."""
    subprocess.check_call(["make", "-s", "-C", _HERE])
    subprocess.check_call([os.path.join(_HERE, "build_ref.sh")])


def blas_path():
    """numpy's bundled ILP64 OpenBLAS (scipy_openblas64_), the dgemm behind the stand-in's product."""
    import numpy
    libs = glob.glob(os.path.join(os.path.dirname(os.path.dirname(numpy.__file__)), "numpy.libs", "libscipy_openblas64_*.so"))
    return libs[0] if libs else None


def lib(blas_threads=None):
    global _LIB
    if _LIB is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (oracle/build_ref.sh)")
        L = C.CDLL(LIB_PATH)
        p, i32, i64, u64 = C.c_void_p, C.c_int, C.c_int64, C.c_uint64
        L.ref_last_error.restype = C.c_char_p
        L.ref_use_blas.argtypes = [C.c_char_p, i32]
        L.ref_forward.argtypes = [i32, i32, i32, i32, u64, i32, i32, p, p, i32, i32, i32, i32, C.c_double, p]
        L.ref_quantize_hashes.argtypes = [i32, i32, i32, i32, u64, i32, i32, p, p, p, p]
        L.ref_bench_layer_decode.argtypes = [u64, i32, i32, i32, i32, i32, i32, i64, p, p, p]
        bp = blas_path()
        if bp:
            _check(L, L.ref_use_blas(bp.encode(), int(blas_threads or os.cpu_count() or 1)))
        _LIB = L
    return _LIB


def _check(L, rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {L.ref_last_error().decode()}")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def forward(layers, hidden, heads, vocab, seed, bits, axis, tokens, positions, context_length, unidirectional=False,
            half=False, prescale=1.0):
    """forward(dequantize_model(quantize_model(init_parameters(cfg, Rng(seed)), policy)), gMASK sample)
    (model.cpp:166-226 on quant.cpp:284-342); bits 0 = unquantized; half: PrecisionPolicy
    kHalfEmulated with softmax_prescale. Logits [n, vocab]."""
    L = lib()
    t = np.ascontiguousarray(tokens, np.int32)
    pos = np.ascontiguousarray(positions, np.int32)
    out = np.empty((len(t), vocab), np.float64)
    _check(L, L.ref_forward(layers, hidden, heads, vocab, seed, bits, AXIS[axis], _ptr(t), _ptr(pos), len(t),
                            context_length, int(unidirectional), int(half), float(prescale), _ptr(out)))
    return out


def quantize_hashes(layers, hidden, heads, vocab, seed, bits, axis):
    L = lib()
    hp, hs, pb, ns = C.c_uint64(), C.c_uint64(), C.c_int64(), C.c_int64()
    _check(L, L.ref_quantize_hashes(layers, hidden, heads, vocab, seed, bits, AXIS[axis], C.byref(hp), C.byref(hs),
                                    C.byref(pb), C.byref(ns)))
    return f"{hp.value:016x}", f"{hs.value:016x}", pb.value, ns.value


def bench_layer_decode(seed=2210, bits=4, axis="column", ctx=130, warmup=1, steps=3, threads=None, head_vocab=16384):
    """Seconds per decode token through one GLM-130B-shaped layer on the reference's own ops
    (oracle/ref_harness.cpp ref_bench_layer_decode), setup seconds, and head seconds for a
    `head_vocab`-row slice of the tied table."""
    L = lib(threads)
    sps, setup, head = C.c_double(), C.c_double(), C.c_double()
    _check(L, L.ref_bench_layer_decode(seed, bits, AXIS[axis], ctx, warmup, steps, int(threads or os.cpu_count() or 1),
                                       head_vocab, C.byref(sps), C.byref(setup), C.byref(head)))
    return sps.value, setup.value, head.value

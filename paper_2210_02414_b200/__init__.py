"""B200-native GLM-130B quantized inference hot path (arXiv 2210.02414).

The product is the C ABI shared library `libglm130b.so` built from `csrc/` for sm_100a
(declared in include/glm130b.h). This package is a thin ctypes binding over that ABI —
the same binding a maintainer of the reference would add — used by
bench.py and the tests. It never falls back to CPU code: if the library is missing,
importing `lib()` raises.
"""
from .glm import (  # noqa: F401
    GLMError, ContractError, DimensionError, FormatError, PolicyError, CudaError,
    lib, LIB_PATH, group_count, payload_bytes, quantize_absmax, quantize_zeropoint, quantize_weight,
    dequantize, pack_int4, unpack_int4, QLinear, Model, GLMConfig, gmask_layout,
    deepnorm_residual, geglu, attention, EmulatedGroup, run_ranks,
)

"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol
include/glm130b.h declares, the ctypes binding covers them, and the header is valid C.
No compute call runs here (there is no GPU in the build container)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2210_02414_b200 import glm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "glm130b.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:glm_status|int64_t|int|const char\s*\*)\s+(glm_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = declared_functions()
    assert len(names) >= 30
    for must in ("glm_quantize_weight", "glm_dequantize", "glm_pack_int4", "glm_unpack_int4", "glm_qlinear",
                 "glm_model_prefill", "glm_model_decode_step", "glm_model_memory"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(glm.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    assert sorted(glm.SIGNATURES) == declared_functions()


def test_header_is_valid_c_and_cpp():
    for lang, std in (("c", "-std=c99"), ("c++", "-std=c++17")):
        subprocess.run(["/usr/bin/gcc", "-x", lang, std, "-fsyntax-only", "-Wall", "-Werror", HEADER], check=True)


def test_pure_host_entry_points_work_without_gpu():
    lib = glm.lib()
    assert lib.glm_group_count(3, 5, 0) == 3 and lib.glm_group_count(3, 5, 1) == 5 and lib.glm_group_count(3, 5, 2) == 1
    assert lib.glm_payload_bytes(3, 5, 4) == 8 and lib.glm_payload_bytes(3, 5, 8) == 15
    assert b"sm_100a" in lib.glm_version()


def _has_gpu():
    try:
        return subprocess.run(["nvidia-smi"], capture_output=True).returncode == 0
    except FileNotFoundError:
        return False


@pytest.mark.skipif(_has_gpu(), reason="a GPU is present; the no-GPU failure mode is not observable")
def test_compute_fails_loudly_without_gpu():
    with pytest.raises(glm.CudaError):
        glm.quantize_absmax([[1.0, -2.0, 0.5]], 8)
    with pytest.raises(glm.CudaError):
        glm.Model(glm.GLMConfig(num_layers=1, hidden=256, num_heads=4), bits=8)


def test_policy_errors_are_raised_before_device_work():
    with pytest.raises(glm.ContractError):
        glm.quantize_absmax([[1.0, 2.0]], 5)
    with pytest.raises(glm.ContractError):
        glm.Model(glm.GLMConfig(num_layers=0, hidden=256, num_heads=4))
    with pytest.raises(glm.ContractError):
        glm.Model(glm.GLMConfig(num_layers=1, hidden=256, num_heads=3))


def build_cpp_test():
    """Compile tests/cpp/test_quant_capi.cpp against include/glm130b.hpp + libglm130b.so."""
    out = os.path.join(ROOT, "build", "test_quant_capi")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(glm.LIB_PATH)
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_quant_capi.cpp"), "-L" + libdir, "-lglm130b",
                    "-Wl,-rpath," + libdir, "-o", out], check=True)
    return out


def build_cpp_block_test():
    """Compile tests/cpp/test_block_capi.cpp: the product through glm130b.hpp, checked against
    the CPU oracle (oracle/liboracle.so, test infrastructure) linked into the test binary."""
    out = os.path.join(ROOT, "build", "test_block_capi")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libdir = os.path.dirname(glm.LIB_PATH)
    odir = os.path.join(ROOT, "oracle")
    if not os.path.exists(os.path.join(odir, "liboracle.so")):
        subprocess.run(["make", "-s", "-C", odir], check=True)
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_block_capi.cpp"), "-L" + libdir, "-lglm130b",
                    "-L" + odir, "-loracle", "-Wl,-rpath," + libdir + ":" + odir, "-o", out], check=True)
    return out


def test_cpp_wrapper_compiles_and_links():
    assert os.path.exists(build_cpp_test())
    assert os.path.exists(build_cpp_block_test())


@pytest.mark.skipif(_has_gpu(), reason="a GPU is present; the no-GPU failure mode is not observable")
def test_cpp_wrapper_raises_cuda_error_without_gpu():
    r = subprocess.run([build_cpp_test(), "--no-gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr

"""The C++ caller's view of the boundary on a B200: tests/cpp/test_quant_capi.cpp runs the
reference's quantization KATs (test_quant.cpp:40-75, :188-215), the quantized linear against
x . dequantize(q), and a C++ host decode loop through include/glm130b.hpp."""
import subprocess

import pytest

from test_capi import build_cpp_block_test, build_cpp_test


@pytest.mark.gpu
def test_cpp_host_path_on_gpu():
    r = subprocess.run([build_cpp_test()], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_block_api_matches_oracle():
    """tests/cpp/test_block_capi.cpp: deepnorm_residual / attention / geglu op by op and the
    glm_block_forward layer chain (prefill + teacher-forced decode) against the oracle's taps."""
    r = subprocess.run([build_cpp_block_test()], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout

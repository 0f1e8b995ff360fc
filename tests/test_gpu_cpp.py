"""The C++ caller's view of the boundary on a B200: tests/cpp/test_quant_capi.cpp runs the
reference's quantization KATs (test_quant.cpp:40-75, :188-215), the quantized linear against
x . dequantize(q), and a C++ host decode loop through include/glm130b.hpp."""
import subprocess

import pytest

from test_capi import build_cpp_test


@pytest.mark.gpu
def test_cpp_host_path_on_gpu():
    r = subprocess.run([build_cpp_test()], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout

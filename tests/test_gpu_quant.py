"""GPU quantization parity: codes, packed payloads and FP64 scales from the B200 kernels
must equal the reference bit for bit (quant.cpp:19-255), checked against the pinned CPU
oracle and the reference's golden FNV hashes. Mirrors test_quant.cpp."""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

pytestmark = pytest.mark.gpu
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


@pytest.fixture(scope="module")
def tiny():
    return O.Params(4, 512, 8, vocab=262, seed=1234)


@pytest.mark.parametrize("case", GOLD["tiny_quantize_model"], ids=lambda c: f"int{c['bits']}-{c['axis']}")
def test_gpu_quantize_model_matches_reference_hashes(tiny, case):
    hp = hs = 1469598103934665603
    for layer in range(4):
        for w in (O.QKV, O.OUT, O.W1, O.V, O.W2):
            q = glm.quantize_absmax(tiny.tensor(layer, w), case["bits"], case["axis"])
            hp = O.fnv1a64(q["payload"], hp)
            hs = O.fnv1a64(q["scales"], hs)
    assert "%016x" % hp == case["payload_fnv"]
    assert "%016x" % hs == case["scales_fnv"]


def test_absmax_worked_row():  # test_quant.cpp:40-53
    q = glm.quantize_absmax(np.array([[1.0, -2.0, 0.5]]), 8, "row")
    assert q["scales"][0] == 2.0 / 127.0
    assert O.codes_of(q).tolist() == [64, -127, 32]
    back = glm.dequantize(q)[0]
    np.testing.assert_allclose(back, [1.007874, -2.0, 0.503937], rtol=1e-6)


def test_zeropoint_worked_row_and_constant_group():  # test_quant.cpp:77-114
    q = glm.quantize_zeropoint(np.array([[0.0, 0.5, 1.0]]), 8, "row")
    assert q["zero_points"][0] == 127.0 and O.codes_of(q).tolist() == [-127, 0, 127]
    np.testing.assert_allclose(glm.dequantize(q)[0], [0.0, 0.5, 1.0], atol=1e-12)
    qc = glm.quantize_zeropoint(np.full((2, 5), -3.75), 4, "row")
    assert qc["constant_group"][0] == 1
    assert (glm.dequantize(qc) == -3.75).all()


def test_degenerate_and_error_cases():  # test_quant.cpp:55-75
    z = np.zeros((3, 4))
    qz = glm.quantize_absmax(z, 8, "row")
    assert (glm.dequantize(qz) == z).all() and (qz["scales"] == 0).all()
    s = 0.03125
    grid = np.array([[4 * s, -127 * s, 10 * s], [127 * s, 0.0, -77 * s]])
    np.testing.assert_array_equal(glm.dequantize(glm.quantize_absmax(grid, 8, "whole")), grid)
    with pytest.raises(glm.ContractError):
        glm.quantize_absmax(np.array([[1.0, np.inf]]), 8, "row")
    with pytest.raises(glm.ContractError):
        glm.quantize_absmax(np.array([[np.nan, 1.0]]), 4, "column")
    with pytest.raises(glm.ContractError):
        glm.quantize_absmax(grid, 5, "row")
    with pytest.raises(glm.FormatError):
        q = glm.quantize_absmax(grid, 8, "row")
        q["payload"] = q["payload"][:-1]
        glm.dequantize(q)


@pytest.mark.parametrize("scheme", ["absmax", "zeropoint"])
def test_random_shapes_bit_exact(scheme):  # test_quant.cpp:116-139, acceptance.cpp:524-554
    rng = np.random.default_rng(31)
    for trial in range(60):
        r, c = (int(v) for v in rng.integers(1, 70, size=2))
        w = rng.normal(0, 10.0 ** rng.integers(-3, 3), size=(r, c))
        if trial % 7 == 0:
            w[rng.integers(0, r)] = 0.0  # all-zero group
        for bits in (4, 8):
            for axis in ("row", "column", "whole"):
                g = glm.quantize_weight(w, bits, axis, scheme)
                o = O.quantize(w, bits, axis, scheme)
                assert np.array_equal(g["payload"], o["payload"]), (r, c, bits, axis)
                assert np.array_equal(g["scales"].view(np.uint64), o["scales"].view(np.uint64))
                if scheme == "zeropoint":
                    assert np.array_equal(g["zero_points"], o["zero_points"])
                    assert np.array_equal(g["constant_group"], o["constant_group"])
                back = glm.dequantize(g)
                assert np.array_equal(back, O.dequantize(o))


def test_float32_and_bf16_inputs_are_widened_exactly():
    rng = np.random.default_rng(5)
    w32 = rng.normal(0, 0.02, size=(33, 47)).astype(np.float32)
    g = glm.quantize_absmax(w32, 4, "column")
    o = O.quantize(w32.astype(np.float64), 4, "column")
    assert np.array_equal(g["payload"], o["payload"]) and np.array_equal(g["scales"], o["scales"])
    bf = (w32.view(np.uint32) >> 16).astype(np.uint16)
    wide = (bf.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    g = glm.quantize_absmax(bf, 8, "row")
    o = O.quantize(wide, 8, "row")
    assert np.array_equal(g["payload"], o["payload"]) and np.array_equal(g["scales"], o["scales"])


def test_pack_unpack():  # test_quant.cpp:188-215
    vals = np.array([a for a in range(-7, 8) for _ in range(2)], np.int8)
    for n in (1, 2, 7, 16, len(vals)):
        packed = glm.pack_int4(vals[:n])
        assert np.array_equal(packed, O.pack_int4(vals[:n]))
        assert np.array_equal(glm.unpack_int4(packed, n), vals[:n])
    for bad in (8, -8):
        with pytest.raises(glm.ContractError):
            glm.pack_int4(np.array([0, bad], np.int8))
    with pytest.raises(glm.FormatError):
        glm.unpack_int4(np.zeros(3, np.int8), 7)


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("axis", ["row", "column", "whole"])
def test_qweight_export_round_trip_and_layout(bits, axis):
    rng = np.random.default_rng(bits * 10 + len(axis))
    K, N = 200, 90  # ragged: K % 64 != 0, N % 16 != 0
    w = rng.normal(0, 0.01, size=(K, N))
    q = glm.quantize_absmax(w, bits, axis)
    ql = glm.QLinear.from_payload(q)
    e = ql.export()
    assert np.array_equal(e["payload"], q["payload"]) and np.array_equal(e["scales"], q["scales"])
    # the device layout places code(k, n) where layout.cuh says: 16-feature row tiles x
    # 64-k chunks in mma.sync fragment order (Np/Kp padded to 128)
    dev = ql.device_bytes()
    codes = O.codes_of(q).reshape(K, N)
    nch, chunk = ((K + 127) // 128 * 128) // 64, (512 if bits == 4 else 1024)
    for k, n in [(0, 0), (1, 0), (0, 1), (9, 8), (63, 15), (64, 16), (K - 1, N - 1), (130, 77), (31, 89), (199, 64)]:
        rt, c, row, kk = n // 16, k // 64, n % 16, k % 64
        g, rsel, j, kc = row & 7, row >> 3, kk >> 4, kk & 15
        hi, t, r = kc & 1, (kc & 7) >> 1, rsel | ((kc >> 3) << 1)
        lane = g * 4 + t
        base = (rt * nch + c) * chunk
        if bits == 4:
            p = r + 4 * hi
            byte = dev[base + lane * 16 + j * 4 + p // 2]
            got = ((int(byte) >> (4 * (p & 1))) & 0xF) - 8
        else:
            half, jj, wd, b = j >> 1, j & 1, r >> 1, (r & 1) * 2 + hi
            got = int(dev[base + half * 512 + lane * 16 + jj * 8 + wd * 4 + b]) - 128
        assert got == codes[k, n], (k, n)


def test_qweight_rejects_minus_eight():
    bad = {"payload": O.pack_int4(np.array([0, 1], np.int8)), "scales": np.ones(1), "rows": 1, "cols": 2,
           "bits": 4, "axis": "row"}
    bad["payload"] = np.array([8], np.int8)  # low nibble 8 == code -8, never produced by quant.cpp:223-240
    with pytest.raises(glm.ContractError):
        glm.QLinear.from_payload(bad)

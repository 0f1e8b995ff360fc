"""Pins the CPU oracle (oracle/liboracle.so) against the reference's own golden values
(tests/golden/reference_golden.json) and known-answer tests from the reference test
suite. CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def test_rng_stream_matches_reference():
    # rng.hpp:30-32: a fresh normal_distribution per draw
    got = O.rng_normal(1234, 4)
    assert got.tolist() == GOLD["rng_1234_normal_0_1"]
    assert got[1] != GOLD["rng_1234_reused_distribution_second"]


@pytest.fixture(scope="module")
def tiny():
    return O.Params(4, 512, 8, vocab=262, seed=1234)


def test_tiny_init_bit_exact(tiny):
    g = GOLD["tiny_init"]
    E = tiny.tensor(0, O.EMBED)
    assert E[0, :3].tolist() == [g["E00"], g["E01"], g["E02"]]
    assert tiny.tensor(0, O.QKV)[0, 0] == g["L0_qkv_00"]
    assert tiny.tensor(3, O.W2).ravel()[-1] == g["L3_ffn_w2_last"]
    assert tiny.ffn == 1368


@pytest.mark.parametrize("case", GOLD["tiny_quantize_model"], ids=lambda c: f"int{c['bits']}-{c['axis']}")
def test_quantize_model_hashes(tiny, case):
    hp = hs = 1469598103934665603
    nb = ns = 0
    for layer in range(4):
        for w in (O.QKV, O.OUT, O.W1, O.V, O.W2):
            q = O.quantize(tiny.tensor(layer, w), case["bits"], case["axis"])
            hp = O.fnv1a64(q["payload"], hp)
            hs = O.fnv1a64(q["scales"], hs)
            nb += len(q["payload"])
            ns += len(q["scales"])
            if layer == 0 and w == O.QKV:
                assert q["scales"][0] == case["L0_qkv_s0"]
                assert O.codes_of(q)[:4].tolist() == case["L0_qkv_codes"]
    assert nb == case["payload_bytes"] and ns == case["nscales"]
    assert "%016x" % hp == case["payload_fnv"]
    assert "%016x" % hs == case["scales_fnv"]


def tiny_sample():
    return O.gmask_sample([6 + (37 * i + 11) % 256 for i in range(126)])


def test_tiny_forward_matches_reference_logits():
    p = O.Params(4, 512, 8, vocab=262, seed=1234)
    s = tiny_sample()
    fp64 = p.forward(s)
    p.quantize(8, "row")
    lq = p.forward(s)
    g = GOLD["tiny_forward_int8_row"]
    np.testing.assert_allclose(lq[-1, :4], g["last_row_logits_0_3"], rtol=0, atol=1e-12)
    assert abs(np.abs(lq - fp64).max() - g["max_abs_int8_minus_fp64"]) < 1e-6
    lz = p.forward(s, zero_sublayers=True)
    assert abs(np.abs(lq - lz).max() - g["max_abs_delta_ref_sublayers_zeroed"]) < 1e-4


def test_absmax_worked_row():  # test_quant.cpp:40-53
    k = GOLD["kats"]["absmax_row"]
    q = O.quantize(np.array([k["w"]]), 8, "row")
    assert abs(q["scales"][0] - 2.0 / 127.0) <= 1e-15 * (2.0 / 127.0)
    assert O.codes_of(q).tolist() == k["codes"]
    back = O.dequantize(q)[0]
    np.testing.assert_allclose(back, k["deq"], rtol=1e-6)


def test_zeropoint_worked_row():  # test_quant.cpp:77-91
    k = GOLD["kats"]["zeropoint_row"]
    q = O.quantize(np.array([k["w"]]), 8, "row", "zeropoint")
    assert abs(q["scales"][0] - 1 / 254) < 1e-17
    assert q["zero_points"][0] == 127.0
    assert O.codes_of(q).tolist() == k["codes"]
    np.testing.assert_allclose(O.dequantize(q)[0], k["w"], atol=1e-12)


def test_degenerate_and_errors():  # test_quant.cpp:55-75
    z = np.zeros((3, 4))
    q = O.quantize(z, 8, "row")
    assert (O.dequantize(q) == 0).all() and (q["scales"] == 0).all()
    s = 0.03125
    grid = np.array([[4 * s, -127 * s, 10 * s], [127 * s, 0.0, -77 * s]])
    q = O.quantize(grid, 8, "whole")
    np.testing.assert_allclose(O.dequantize(q), grid, rtol=1e-15)
    with pytest.raises(O.OracleError) as e:
        O.quantize(np.array([[1.0, np.inf]]), 8, "row")
    assert e.value.code == 1
    with pytest.raises(O.OracleError) as e:
        O.quantize(grid, 5, "row")
    assert e.value.code == 1


def test_roundtrip_bound_and_fixed_point():  # test_quant.cpp:116-139
    rng = np.random.default_rng(31)
    for _ in range(100):
        r, c = rng.integers(1, 9, size=2)
        w = rng.normal(0, 10.0 ** rng.integers(-3, 3), size=(r, c))
        for bits in (4, 8):
            for axis in ("row", "column", "whole"):
                q = O.quantize(w, bits, axis)
                back = O.dequantize(q)
                g = {"row": np.arange(r)[:, None].repeat(c, 1), "column": np.arange(c)[None, :].repeat(r, 0),
                     "whole": np.zeros((r, c), int)}[axis]
                assert (np.abs(back - w) <= q["scales"][g] / 2 + 1e-12).all()
                q2 = O.quantize(back, bits, axis)
                assert (O.codes_of(q2) == O.codes_of(q)).all()


def test_pack_unpack_bijection():  # test_quant.cpp:188-215
    for a in range(-7, 8):
        assert O.unpack_int4(O.pack_int4([a]), 1).tolist() == [a]
        for b in range(-7, 8):
            assert O.unpack_int4(O.pack_int4([a, b]), 2).tolist() == [a, b]
    for bad in (8, -8):
        with pytest.raises(O.OracleError):
            O.pack_int4([bad])
    with pytest.raises(O.OracleError) as e:
        O.unpack_int4(np.zeros(3, np.int8), 7)
    assert e.value.code == 3


def test_model_constants():  # test_model.cpp:32-35, :478; test_model.cpp:188
    k = GOLD["kats"]
    assert abs(O.lib().or_deepnorm_alpha(70) - k["deepnorm_alpha_70"]) < 1e-6
    assert abs(1 / O.lib().or_deepnorm_alpha(70) - k["deepnorm_factor_70"]) < 1e-6
    for h, n, f in k["default_ffn_hidden"]:
        assert O.default_ffn_hidden(h, n) == f


def test_half_round_kats():  # test_tensor.cpp:186-207
    for x, y in GOLD["kats"]["half_round"]:
        assert O.half_round(x) == y
    assert math.isinf(O.half_round(65520.0))


def test_rope_properties():  # test_model.cpp:118-166
    q = np.array([[1.0, 0.0]])
    assert O.rope_rotate(q, [0]).tolist() == [[1.0, 0.0]]
    k1 = O.rope_rotate(q, [1])
    assert abs((q * k1).sum() - math.cos(1.0)) < 1e-12
    rng = np.random.default_rng(9)
    for _ in range(20):
        d = 2 * rng.integers(1, 16)
        a, b = rng.normal(size=(1, d)), rng.normal(size=(1, d))
        delta = int(rng.integers(-8, 9))
        ref = None
        for _ in range(4):
            m = int(rng.integers(max(0, -delta), 300))
            dot = (O.rope_rotate(a, [m]) * O.rope_rotate(b, [m + delta])).sum()
            ref = dot if ref is None else ref
            assert abs(dot - ref) < 1e-10


def test_softmax_layernorm_closed_forms():  # test_tensor.cpp:45-127
    np.testing.assert_allclose(O.softmax_rows(np.zeros((1, 3))), [[1 / 3] * 3])
    np.testing.assert_allclose(O.softmax_rows(np.array([[1000.0, 0.0]])), [[1.0, 0.0]], atol=1e-300)
    np.testing.assert_allclose(O.softmax_rows(np.array([[0.0, math.log(3)]])), [[0.25, 0.75]])
    with pytest.raises(O.OracleError) as e:
        O.softmax_rows(np.array([[-np.inf, -np.inf]]))
    assert e.value.code == 4
    x = np.random.default_rng(0).normal(size=(4, 32))
    y = O.layer_norm(x, np.ones(32), np.zeros(32))
    assert np.abs(y.mean(1)).max() < 1e-10 and np.abs(y.var(1) - 1).max() < 1e-3


def test_gmask_mask_closed_form():  # corruption.cpp:338-367 == j < max(C, i+1)
    s = O.gmask_sample(list(range(6, 30)), list(range(40, 52)))
    m = O.build_mask(s)
    C = s["context_length"]
    i = np.arange(s["n"])[:, None]
    j = np.arange(s["n"])[None, :]
    assert (m == (j < np.maximum(C, i + 1))).all()
    assert s["positions"][C:C + 3] == [C - 1, C - 1, C]


def test_attention_kats():  # test_model.cpp:204-241
    out = O.attention(np.array([[1.0, 2, 3, 4]]), np.full((1, 4), 0.5), np.array([[9.0, -1, 2.5, 0]]), [0],
                      np.ones((1, 1)))
    np.testing.assert_allclose(out, [[9.0, -1, 2.5, 0]], rtol=1e-12)
    with pytest.raises(O.OracleError) as e:
        O.attention(np.ones((1, 4)), np.ones((1, 4)), np.ones((1, 4)), [0], np.zeros((1, 1)))
    assert e.value.code == 4


def test_philox_generator_is_deterministic_and_normal():
    w = O.gen_matrix(7, 3, 256, 512, 1.0)
    assert np.array_equal(w, O.gen_matrix(7, 3, 256, 512, 1.0))
    assert abs(w.mean()) < 0.01 and abs(w.std() - 1) < 0.01
    # values are bf16-representable
    f = w.astype(np.float32).view(np.uint32)
    assert (f & 0xFFFF == 0).all()


def test_numpy_block_oracle_equals_or_forward_taps():
    """pyoracle.block_forward (the G-shape block oracle, model.cpp:198-224 restated over the
    oracle's ops + numpy GEMMs) chained from the embedding rows reproduces or_forward's
    per-layer sublayer taps and final logits (tiny config, INT4 kColumn weights)."""
    import numpy as np
    from oracle import pyoracle as O

    p = O.Params(2, 256, 4, vocab=262, seed=5)
    p.quantize(4, "column")
    sample = O.gmask_sample([6 + (37 * i + 11) % 256 for i in range(30)], [40, 41])
    ref, at, ft = p.forward(sample, taps=True)
    n = sample["n"]
    mask = O.build_mask(sample)
    x = p.tensor(0, O.EMBED)[sample["tokens"]]
    ones, zeros = np.ones(256), np.zeros(256)
    alpha = np.sqrt(4.0)
    for layer in range(2):
        W = {w: p.tensor(layer, w) for w in range(5)}
        x, attn, ff = O.block_forward(x, W, (ones, zeros, ones, zeros), sample["positions"], mask, 4, alpha)
        assert np.abs(attn - at[layer]).max() <= 1e-12 * np.abs(at[layer]).max()
        assert np.abs(ff - ft[layer]).max() <= 1e-12 * np.abs(ft[layer]).max()
    logits = x @ p.tensor(0, O.EMBED).T
    assert np.abs(logits - ref).max() <= 1e-12 * np.abs(ref).max()
    assert n == ref.shape[0]


def test_oracle_chunked_generation_and_column_dequantize():
    import numpy as np
    from oracle import pyoracle as O

    a = O.gen_matrix(3, 5, 10, 7, 0.1)
    assert np.array_equal(a[4:7], O.gen_rows(3, 5, 4, 3, 7, 0.1))
    for bits, axis in ((4, "column"), (8, "row"), (4, "whole")):
        q = O.quantize(np.random.default_rng(bits).normal(size=(33, 21)), bits, axis)
        assert np.array_equal(O.dequantize_cols(q, [0, 5, 20]), O.dequantize(q)[:, [0, 5, 20]])

"""Quantized-checkpoint loader: glm_model_load_quantized reads the
directory the reference's save_quantized_model writes (quant.cpp:409-448: manifest.json +
GLMT tensors, tensor_io.cpp:68-97) and puts the canonical payloads/scales on the GPU without
re-quantizing. The fixture directory is written here byte-for-byte in the reference format
from the oracle's quantize_model output (pinned to the reference hashes in
test_oracle_golden.py)."""
import json
import os
import struct

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2210_02414_b200 import glm

NAMES = ["qkv", "out_proj", "ffn_w1", "ffn_v", "ffn_w2"]


def write_glmt(path, array, dtype):
    """tensor_io.cpp:68-97: "GLMT", u8 version 1, u8 dtype (0 f64, 1 f32, 2 i8), u32 rank,
    u64 dims, raw little-endian payload."""
    a = np.ascontiguousarray(array)
    code = {"f64": 0, "f32": 1, "i8": 2}[dtype]
    with open(path, "wb") as f:
        f.write(b"GLMT" + bytes([1, code]) + struct.pack("<I", a.ndim))
        for d in a.shape:
            f.write(struct.pack("<Q", d))
        f.write(a.astype({"f64": "<f8", "f32": "<f4", "i8": "i1"}[dtype]).tobytes())


def write_checkpoint(dirpath, p, bits, axis, scheme="absmax"):
    """save_quantized_model (quant.cpp:409-448) of the oracle's params under (bits, scheme, axis);
    zeropoint matrices add .zeros.glmt and "constant_groups" (write_quantized_matrix, :367-387)."""
    os.makedirs(dirpath, exist_ok=True)
    d, f = p.hidden, p.ffn
    man = {"config": {"num_layers": p.num_layers, "hidden": d, "num_heads": p.num_heads, "ffn_hidden": f,
                      "vocab": p.vocab, "dropout": 0.0, "init_method_std": 0.0052, "layernorm_eps": 1e-5,
                      "deepnorm_alpha": (2.0 * p.num_layers) ** 0.5},
           "policy": {"bits": bits, "scheme": scheme, "axis": axis}, "matrices": []}
    write_glmt(os.path.join(dirpath, "embedding.glmt"), p.tensor(0, O.EMBED), "f64")
    payloads = {}
    for layer in range(p.num_layers):
        for w, nm in enumerate(NAMES):
            q = O.quantize(p.tensor(layer, w), bits, axis, scheme=scheme)
            payloads[(layer, w)] = q
            name = f"layer{layer}.{nm}"
            entry = {"name": name, "bits": bits, "scheme": scheme, "axis": axis, "rows": q["rows"], "cols": q["cols"]}
            write_glmt(os.path.join(dirpath, name + ".codes.glmt"), np.asarray(q["payload"], np.int8), "i8")
            write_glmt(os.path.join(dirpath, name + ".scales.glmt"), q["scales"], "f64")
            if scheme == "zeropoint":
                write_glmt(os.path.join(dirpath, name + ".zeros.glmt"), q["zero_points"], "f64")
                entry["constant_groups"] = [int(c) for c in q["constant_group"]]
            man["matrices"].append(entry)
        for v, slot in (("ln1_gain", 5), ("ln2_gain", 6)):
            write_glmt(os.path.join(dirpath, f"layer{layer}.{v}.glmt"), p.tensor(layer, slot).reshape(-1), "f64")
        for v in ("ln1_bias", "ln2_bias"):
            write_glmt(os.path.join(dirpath, f"layer{layer}.{v}.glmt"), np.zeros(d), "f64")
    with open(os.path.join(dirpath, "manifest.json"), "w") as fh:
        json.dump(man, fh, indent=2)
    return payloads


@pytest.fixture(scope="module")
def ckpt(tmp_path_factory):
    p = O.Params(2, 256, 4, vocab=300, seed=21)
    path = str(tmp_path_factory.mktemp("ckpt"))
    payloads = write_checkpoint(path, p, 4, "column")
    return p, path, payloads


def corrupt(path, name, offset, data):
    with open(os.path.join(path, name), "r+b") as fh:
        fh.seek(offset)
        fh.write(data)


@pytest.mark.parametrize("mutation,err", [
    (lambda d: corrupt(d, "layer0.ffn_v.codes.glmt", 0, b"XLMT"), glm.FormatError),       # magic
    (lambda d: corrupt(d, "layer0.qkv.scales.glmt", 4, bytes([2])), glm.FormatError),     # version
    (lambda d: corrupt(d, "embedding.glmt", 5, bytes([7])), glm.FormatError),            # dtype
    (lambda d: os.truncate(os.path.join(d, "layer0.ffn_w2.codes.glmt"), 40), glm.FormatError),
    (lambda d: os.remove(os.path.join(d, "layer0.ln2_bias.glmt")), glm.FormatError),
    (lambda d: open(os.path.join(d, "manifest.json"), "w").write("{\"config\": [1, 2"), glm.FormatError),
])
def test_malformed_checkpoints_fail_before_device_work(tmp_path, mutation, err):
    p = O.Params(1, 128, 2, vocab=64, seed=3)
    write_checkpoint(str(tmp_path), p, 8, "row")
    mutation(str(tmp_path))
    with pytest.raises(err):
        glm.Model.load_quantized(str(tmp_path))


def test_policy_and_shape_mismatches_are_format_errors(tmp_path):
    p = O.Params(1, 128, 2, vocab=64, seed=3)
    write_checkpoint(str(tmp_path), p, 8, "row")
    man_path = os.path.join(str(tmp_path), "manifest.json")
    man = json.load(open(man_path))
    man["matrices"][1]["cols"] = 129
    json.dump(man, open(man_path, "w"))
    with pytest.raises(glm.FormatError):
        glm.Model.load_quantized(str(tmp_path))
    man["matrices"][1]["cols"] = 128
    man["policy"]["scheme"] = "zeropoint"  # the matrices are absmax: not the manifest policy
    json.dump(man, open(man_path, "w"))
    with pytest.raises(glm.FormatError):
        glm.Model.load_quantized(str(tmp_path))
    man["policy"]["scheme"] = "nf4"
    json.dump(man, open(man_path, "w"))
    with pytest.raises(glm.FormatError):
        glm.Model.load_quantized(str(tmp_path))


def test_zeropoint_checkpoint_without_zero_points_fails_before_device_work(tmp_path):
    p = O.Params(1, 128, 2, vocab=64, seed=3)
    write_checkpoint(str(tmp_path), p, 4, "column", scheme="zeropoint")
    os.remove(os.path.join(str(tmp_path), "layer0.ffn_v.zeros.glmt"))
    with pytest.raises(glm.FormatError):
        glm.Model.load_quantized(str(tmp_path))


@pytest.mark.gpu
@pytest.mark.parametrize("bits,axis", [(4, "row"), (8, "column")])
def test_zeropoint_checkpoint_matches_the_reference_quantized_model(tmp_path, bits, axis):
    """load_quantized_model of a zeropoint checkpoint (quant.cpp:450-491 reads .zeros.glmt):
    codes, scales and zero points byte-exact on the device, taps and logits vs the oracle's
    forward of the same quantized model."""
    p = O.Params(2, 256, 4, vocab=300, seed=23)
    payloads = write_checkpoint(str(tmp_path), p, bits, axis, scheme="zeropoint")
    m = glm.Model.load_quantized(str(tmp_path), max_ctx=64)
    assert m.scheme == "zeropoint"
    for (layer, w), q in payloads.items():
        pl, sc = m.export_linear(layer, w, q["rows"], q["cols"])
        zp = m.export_zero_points(layer, w, q["rows"], q["cols"])
        assert np.array_equal(pl, np.asarray(q["payload"], np.int8)) and np.array_equal(sc, q["scales"]), (layer, w)
        assert np.array_equal(zp, q["zero_points"]), (layer, w)
    p.quantize(bits, axis, scheme="zeropoint")
    sample = O.gmask_sample([6 + (7 * i) % 250 for i in range(20)], [40, 41])
    ref, at, ft = p.forward(sample, taps=True)
    zero = p.forward(sample, zero_sublayers=True)
    m.enable_taps(True)
    lg = m.prefill(sample["tokens"], sample["positions"], sample["context_length"]).astype(np.float64)
    ga, gf = m.taps(sample["n"])
    for layer in range(2):
        assert np.abs(ga[layer] - at[layer]).max() <= 1e-2 * np.abs(at[layer]).max()
        assert np.abs(gf[layer] - ft[layer]).max() <= 1e-2 * np.abs(ft[layer]).max()
    assert np.abs(lg - ref).max() <= 1e-2 * np.abs(ref - zero).max()


@pytest.mark.gpu
def test_loaded_checkpoint_matches_the_reference_quantized_model(ckpt):
    p, path, payloads = ckpt
    m = glm.Model.load_quantized(path, max_ctx=64)
    for (layer, w), q in payloads.items():
        pl, sc = m.export_linear(layer, w, q["rows"], q["cols"])
        assert np.array_equal(pl, np.asarray(q["payload"], np.int8)) and np.array_equal(sc, q["scales"]), (layer, w)
    p.quantize(4, "column")
    sample = O.gmask_sample([6 + (7 * i) % 250 for i in range(20)], [40, 41])
    ref, at, ft = p.forward(sample, taps=True)
    zero = p.forward(sample, zero_sublayers=True)
    m.enable_taps(True)
    lg = m.prefill(sample["tokens"], sample["positions"], sample["context_length"]).astype(np.float64)
    ga, gf = m.taps(sample["n"])
    for layer in range(2):
        assert np.abs(ga[layer] - at[layer]).max() <= 1e-2 * np.abs(at[layer]).max()
        assert np.abs(gf[layer] - ft[layer]).max() <= 1e-2 * np.abs(ft[layer]).max()
    assert np.abs(lg - ref).max() <= 1e-2 * np.abs(ref - zero).max()


@pytest.mark.gpu
def test_cpp_wrapper_loads_the_checkpoint(ckpt):
    import subprocess
    from test_capi import build_cpp_test
    _, path, _ = ckpt
    r = subprocess.run([build_cpp_test(), "--checkpoint", path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "0 failed" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("bits,byte", [(4, 0x08), (4, 0x80), (8, 0x80)])
def test_codes_outside_the_absmax_range_are_rejected(tmp_path, bits, byte):
    """The streaming loader validates every payload like glm_qweight_create: an INT4 nibble of
    -8 or an INT8 code of -128 cannot come out of quantize_absmax (quant.cpp:19-31)."""
    p = O.Params(1, 128, 2, vocab=64, seed=3)
    write_checkpoint(str(tmp_path), p, bits, "column")
    header = 4 + 2 + 4 + 8  # rank-1 GLMT header
    corrupt(str(tmp_path), "layer0.ffn_w1.codes.glmt", header + 5, bytes([byte]))
    with pytest.raises(glm.ContractError):
        glm.Model.load_quantized(str(tmp_path))

"""The reference itself as the oracle's anchor: the reference's own unmodified
sources (glmlab, /root/reference/proj/src) built with the test-infrastructure stand-ins
(oracle/build_ref.sh -> oracle/_ref). Checked here on the CPU:
  * the reference's own unit tests pass under the stand-ins (test_tensor, test_quant,
    test_model, test_corruption, test_tensor_io) — the stand-ins do not change its behaviour;
  * quantize_model's payload / scale hashes from the reference == the committed goldens == the
    oracle restatement (all four policies);
  * forward(dequantize_model(quantize_model(init_parameters(Rng 1234)))) of the config-1 sample
    from the reference == the oracle restatement's forward to 1e-10, INT8 kRow and INT4 kColumn,
    gMASK and unidirectional."""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as O
from oracle import pyref as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_golden.json")))
PREFIX = [6 + (37 * i + 11) % 256 for i in range(126)]


@pytest.fixture(scope="module", autouse=True)
def ref_built():
    if not R.available():
        if not os.path.isdir("/root/reference/proj/src"):
            pytest.skip("oracle/_ref not built and the reference sources are absent")
        R.build()


@pytest.mark.parametrize("name", ["test_tensor", "test_quant", "test_model", "test_corruption", "test_tensor_io"])
def test_reference_unit_tests_pass_under_the_stand_ins(name):
    exe = os.path.join(R.REF_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=R.REF_DIR)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed |" in r.stdout


@pytest.mark.parametrize("policy", GOLD["tiny_quantize_model"], ids=lambda p: f"int{p['bits']}-{p['axis']}")
def test_reference_quantize_hashes_equal_goldens_and_oracle(policy):
    hp, hs, pb, ns = R.quantize_hashes(4, 512, 8, 262, 1234, policy["bits"], policy["axis"])
    assert (hp, hs, pb, ns) == (policy["payload_fnv"], policy["scales_fnv"], policy["payload_bytes"], policy["nscales"])
    p = O.Params(4, 512, 8, vocab=262, seed=1234)
    h1 = h2 = 1469598103934665603
    for layer in range(4):
        for w in range(5):
            q = O.quantize(p.tensor(layer, w), policy["bits"], policy["axis"])
            h1 = O.fnv1a64(q["payload"], h1)
            h2 = O.fnv1a64(q["scales"], h2)
    assert (f"{h1:016x}", f"{h2:016x}") == (hp, hs)


@pytest.mark.parametrize("bits,axis,uni", [(8, "row", False), (4, "column", False), (8, "row", True), (0, "row", False)])
def test_reference_forward_equals_oracle(bits, axis, uni):
    sample = O.gmask_sample(PREFIX)
    ref = R.forward(4, 512, 8, 262, 1234, bits, axis, sample["tokens"], sample["positions"], sample["context_length"],
                    unidirectional=uni)
    p = O.Params(4, 512, 8, vocab=262, seed=1234)
    if bits:
        p.quantize(bits, axis)
    if uni:
        sample["unidirectional"] = 1
    ora = p.forward(sample)
    assert np.abs(ref - ora).max() <= 1e-10 * np.abs(ref).max()
    if bits == 8 and not uni:
        np.testing.assert_allclose(ref[-1, :4], GOLD["tiny_forward_int8_row"]["last_row_logits_0_3"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("prescale", [1.0, 8.0])
def test_reference_half_storage_forward_equals_oracle(prescale):
    """PrecisionPolicy kHalfEmulated (tensor.hpp:18-29; storage_round at model.cpp:148, 197,
    213-223): the reference's forward with binary16 storage == the oracle's restatement."""
    sample = O.gmask_sample(PREFIX[:60], [40, 41])
    ref = R.forward(4, 512, 8, 262, 1234, 8, "row", sample["tokens"], sample["positions"], sample["context_length"],
                    half=True, prescale=prescale)
    p = O.Params(4, 512, 8, vocab=262, seed=1234)
    p.quantize(8, "row")
    ora = p.forward(sample, half=True, prescale=prescale)
    assert np.abs(ref - ora).max() <= 1e-10 * np.abs(ref).max()
    wide = p.forward(sample)
    assert np.abs(ora - wide).max() > 1e-6  # the policy changes the result

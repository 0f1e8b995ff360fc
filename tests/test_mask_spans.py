"""[MASK] multi-span blank infilling (corruption.cpp:190-247, mask rules
:338-367). corrupt_mask lays the spans out in permutation order after the context, so the
general visibility rule (context bidirectional and blind to spans; spans see the context,
permutation-earlier spans fully and their own span causally) reduces to the closed form
j < max(C, i + 1) the B200 kernels apply. The CPU test proves that reduction on random
samples with the oracle's general mask builder; the GPU test runs prefill of Part A plus
teacher-forced decode of every span in permutation order against the oracle forward."""
import numpy as np
import pytest

from oracle import pyoracle as O


def random_mask_sample(rng, n_text=40, n_spans=3):
    tokens = [int(v) for v in rng.integers(6, 250, size=n_text)]
    starts = sorted(rng.choice(np.arange(0, n_text - 4, 5), size=n_spans, replace=False))
    spans = [(int(s), int(rng.integers(1, 4))) for s in starts]
    perm = [int(v) for v in rng.permutation(n_spans)]
    return O.mask_sample(tokens, spans, perm)


@pytest.mark.parametrize("seed", range(8))
def test_general_mask_reduces_to_the_closed_form(seed):
    s = random_mask_sample(np.random.default_rng(seed), n_spans=1 + seed % 4)
    m = O.build_mask(s)
    n, C = s["n"], s["context_length"]
    closed = np.array([[j < max(C, i + 1) for j in range(n)] for i in range(n)])
    assert np.array_equal(m, closed)


@pytest.mark.gpu
def test_mask_sample_prefill_then_span_decode_matches_oracle():
    from paper_2210_02414_b200 import glm
    from test_gpu_model import build, check_logits, check_taps, oracle_rows
    p, m, _ = build(8, "row")
    s = random_mask_sample(np.random.default_rng(11), n_text=60, n_spans=3)
    ref, at, ft, zero = oracle_rows(p, s)
    C = s["context_length"]
    m.reset()
    m.enable_taps(True)
    lp = m.prefill(s["tokens"][:C], s["positions"][:C], C)
    rows = [lp]
    dtaps_a, dtaps_f = [], []
    for i in range(C, s["n"]):
        _, ld = m.decode_step([s["tokens"][i]], [s["positions"][i]])
        rows.append(ld)
        a, f = m.taps(1)
        dtaps_a.append(a)
        dtaps_f.append(f)
    m.enable_taps(False)
    gpu = np.concatenate(rows, 0).astype(np.float64)
    check_logits(gpu, ref, zero)
    check_taps(np.concatenate(dtaps_a, axis=1), at[:, C:], slice(None))
    check_taps(np.concatenate(dtaps_f, axis=1), ft[:, C:], slice(None))

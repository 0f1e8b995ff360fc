"""Decode / prefill plan selection (host logic, no GPU): which kernel glm_qlinear runs and how
it splits K, for the GLM-130B shapes (glm_debug_plan_shape). The parity tests read the same
plan (QLinear.plan) to model each kernel's exact activation contract."""
import pytest

from paper_2210_02414_b200 import glm

G = [(12288, 36864), (12288, 12288), (12288, 65536), (32768, 12288)]  # qkv, out, W1|V, W2


@pytest.mark.parametrize("K,N", G)
def test_int4_kernel_selection_and_split(K, N):
    nch = K // 64
    kind, ks, nch_, grid = glm.QLinear.plan_for(K, N, 4, 1)
    assert (kind, nch_) == ("i4_single", nch)
    assert 1 <= ks <= 32 and nch // ks >= 4 and 1 <= grid <= 148
    for M in (2, 3, 8, 16):
        kind, ks, _, grid = glm.QLinear.plan_for(K, N, 4, M)
        assert kind == "i4_multi"
        # one resident activation slice of every token per CTA (96 KB, gemv.cu kMkXBytes)
        slice_chunks = -(-nch // ks)
        assert slice_chunks * 128 * M <= 96 * 1024
        assert 1 <= grid <= 148
    for M in (17, 256, 8192):
        kind, ks, _, grid = glm.QLinear.plan_for(K, N, 4, M)
        assert kind == "tcgen05" and ks >= 1 and grid >= 1


@pytest.mark.parametrize("K,N", G)
def test_int8_kernel_selection(K, N):
    assert glm.QLinear.plan_for(K, N, 8, 1)[0] == "f16_tma"
    for M in (2, 16):
        assert glm.QLinear.plan_for(K, N, 8, M)[0] in ("f16_multi", "f16_tma")
    assert glm.QLinear.plan_for(K, N, 8, 300)[0] == "tcgen05"


def test_plan_rejects_bad_arguments():
    with pytest.raises(glm.DimensionError):
        glm.QLinear.plan_for(12288, 12288, 4, 0)
    with pytest.raises(glm.ContractError):
        glm.QLinear.plan_for(12288, 12288, 3, 1)


def test_opt_in_tcgen05_decode_plan():
    """GLM_GEMV_TC=2 moves INT4 2..16-token GEMVs to the tcgen05 kernel: 128-feature items,
    k-slices of <= 64 chunks, one CTA per SM."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, sys.argv[1]); from paper_2210_02414_b200 import glm\n"
        "for K, N in %r:\n"
        "    nch = K // 64\n"
        "    assert glm.QLinear.plan_for(K, N, 4, 1)[0] == 'i4_single'\n"
        "    for M in (2, 8, 16):\n"
        "        kind, ks, _, grid = glm.QLinear.plan_for(K, N, 4, M)\n"
        "        assert kind == 'i4_tc' and -(-nch // ks) <= 64 and 1 <= grid <= 148, (K, N, M, kind, ks, grid)\n"
        "print('ok')\n" % (G,))
    r = subprocess.run([sys.executable, "-c", code, root], env=dict(os.environ, GLM_GEMV_TC="2"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr

"""Pin the CPU oracle against the reference's own goldens and known-answer tests.

CPU-only.  If these pass, every GPU parity test that compares against the oracle is
transitively a comparison against the reference implementation.
"""

import numpy as np
import pytest
from conftest import unpack_keep
from gen import digest, wan_like

import oracle


def test_masker_goldens_bit_exact(manifest, golden_masks):
    for case in manifest["masks"]:
        i, k, p = case["idx"], case["k_frac"], case["p_frac"]
        probs = golden_masks[f"c{i}_probs"]
        t_n = probs.shape[1]
        assert np.array_equal(oracle.top_k_keep(probs, k), unpack_keep(golden_masks[f"c{i}_topk"], t_n)), case
        assert np.array_equal(oracle.top_p_keep(probs, p), unpack_keep(golden_masks[f"c{i}_topp"], t_n)), case
        assert np.array_equal(oracle.hybrid_keep(probs, k, p), unpack_keep(golden_masks[f"c{i}_hybrid"], t_n)), case


def test_pooled_goldens(manifest, golden_pooled):
    for case in manifest["pooled"]:
        i = case["idx"]
        got = oracle.pooled_probs(golden_pooled[f"p{i}_q"], golden_pooled[f"p{i}_k"], case["b_q"], case["b_kv"])
        assert np.array_equal(got, golden_pooled[f"p{i}_probs"]), case


@pytest.mark.parametrize("idx", range(5))
def test_attention_goldens(manifest, golden_attention, idx):
    case = manifest["attention"][idx]
    tag, n, d, t_n = case["tag"], case["n"], case["d"], case["t_n"]
    q, k, v, do = wan_like(case["seed"], n, d, case["b_q"], case["b_kv"], case["s"], heads=case["heads"])
    assert digest(q, k, v, do) == case["digest"], "input regeneration drifted"
    keep = unpack_keep(golden_attention[f"{tag}_keep"], t_n)
    exact = golden_attention[f"{tag}_out"].dtype == np.float64
    tol = 1e-10 if exact else 2e-6
    for h in range(case["heads"]):
        if case["mask"][0] == "hybrid":
            probs = oracle.pooled_probs(q[h], k[h], case["b_q"], case["b_kv"])
            assert np.array_equal(oracle.hybrid_keep(probs, case["mask"][1], case["mask"][2]), keep[h])
        dq, dk, dv, out, lse = oracle.attention_backward(q[h], k[h], v[h], keep[h], case["b_q"], case["b_kv"], do[h])
        for name, got in (("out", out), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
            want = golden_attention[f"{tag}_{name}"][h].astype(np.float64)
            err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-12)
            assert err <= tol, (tag, h, name, err)


# --- the reference test suite's hand-written known answers (test_masker.py) ---------

def _keep_cols(keep):
    return set(np.flatnonzero(keep[0]))


def test_kat_top_k_rows():
    assert _keep_cols(oracle.top_k_keep(np.array([[0.1] * 10]), 0.2)) == {0, 1}  # test_masker.py:67-70
    assert _keep_cols(oracle.top_k_keep(np.array([[0.6, 0.2, 0.1, 0.1]]), 0.5)) == {0, 1}  # :78-80
    assert oracle.top_k_keep(np.array([[0.1] * 10]), 1.0).all()  # :73-75


def test_kat_top_p_rows():
    assert _keep_cols(oracle.top_p_keep(np.array([[0.6, 0.2, 0.1, 0.1]]), 0.6)) == {0}  # :83-85
    assert _keep_cols(oracle.top_p_keep(np.array([[0.4, 0.3, 0.2, 0.1]]), 1.0)) == {0, 1, 2, 3}  # :88-90
    assert _keep_cols(oracle.top_p_keep(np.array([[0.4, 0.3, 0.2, 0.1]]), 0.65)) == {0, 1}  # :93-95
    assert _keep_cols(oracle.top_p_keep(np.array([[0.2, 0.5, 0.3]]), 0.0)) == {1}  # :98-100


def test_kat_hybrid_rows():
    assert _keep_cols(oracle.hybrid_keep(np.array([[0.1] * 10]), 0.2, 0.6)) == {0, 1, 2, 3, 4, 5}  # :103-107
    assert _keep_cols(oracle.hybrid_keep(np.array([[0.6, 0.2, 0.1, 0.1]]), 0.5, 0.6)) == {0, 1}  # :110-113


def test_kat_top_k_count_ieee_trap():
    # 0.07 * 100 == 7.000000000000001 in IEEE double, so K = 8 (SURVEY.md §7 "Hard parts")
    assert oracle.top_k_count(0.07, 100) == 8
    assert oracle.top_k_count(0.0, 50) == 1


def test_kat_pool_ragged():
    x = np.arange(10, dtype=np.float64).reshape(5, 2)  # test_numerics.py:77-82
    assert np.array_equal(oracle.block_mean_pool(x, 2), np.array([[1.0, 2.0], [5.0, 6.0], [8.0, 9.0]]))


def test_oracle_tiled_vs_token_level():
    rng = np.random.Generator(np.random.PCG64(9))
    n, d = 40, 6
    q, k, v = (rng.normal(size=(n, d)) for _ in range(3))
    keep = rng.random((oracle.attention.np.ceil(n / 8).astype(int), 14)) < 0.5
    keep[~keep.any(axis=1), 0] = True
    out, _, visited = oracle.sparse_forward(q, k, v, keep, 8, 3)
    want = oracle.masked_attention_tokens(q, k, v, oracle.expand_keep(keep, 8, 3, n))
    assert np.abs(out - want).max() <= 1e-10
    assert visited == keep.sum()


def test_oracle_wan_like_sparsity_calibration():
    # the structured generator must actually produce a sparse hybrid mask
    q, k, _, _ = wan_like(11, 8192, 64, 128, 64, 0.9)
    probs = oracle.pooled_probs(q[0], k[0], 128, 64)
    keep = oracle.hybrid_keep(probs, 0.03, 0.2)
    assert 0.85 < 1 - keep.mean() < 0.99

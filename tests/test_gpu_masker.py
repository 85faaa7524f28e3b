"""GPU masker parity: K1 pooled map, K2 select (bit-exact vs the reference's goldens),
K3 block lists, and the reference's masker known-answer tests run through the GPU."""

import numpy as np
import pytest
import torch
from conftest import unpack_keep
from gen import wan_like

import oracle
import paper_2602_13515_b200 as spa
from paper_2602_13515_b200 import _lib
from paper_2602_13515_b200 import masker as mk

pytestmark = pytest.mark.gpu


def pm_from_rows(rows):
    probs = np.atleast_2d(np.asarray(rows, dtype=np.float64))
    t_m, t_n = probs.shape
    return mk.PooledMap(probs, b_q=t_n, b_kv=t_m, n_tokens=t_m * t_n)


def kept_cols(bm, row=0):
    return set(np.flatnonzero(bm.keep_numpy()[row]))


def test_select_bit_exact_on_reference_goldens(manifest, golden_masks):
    """Every golden pooled map (hand rows, ties, zeros, c06/c07 random rows, Wan-size
    maps) → identical keep matrices for top-k, top-p and hybrid."""
    for case in manifest["masks"]:
        i, k, p = case["idx"], case["k_frac"], case["p_frac"]
        pm = pm_from_rows(golden_masks[f"c{i}_probs"])
        t_n = pm.probs.shape[1]
        cfg = mk.SparsityConfig(k, p, pm.b_q, pm.b_kv)
        for name, bm in (("topk", mk.top_k_mask(pm, k)), ("topp", mk.top_p_mask(pm, p)),
                         ("hybrid", mk.hybrid_mask(pm, cfg))):
            want = unpack_keep(golden_masks[f"c{i}_{name}"], t_n)
            assert np.array_equal(bm.keep_numpy(), want), (case, name)


# --- the reference masker KATs (test_masker.py:67-119), through the GPU ---------------

def test_kat_rows():
    assert kept_cols(mk.top_k_mask(pm_from_rows([[0.1] * 10]), 0.2)) == {0, 1}
    assert mk.top_k_mask(pm_from_rows([[0.1] * 10]), 1.0).keep.all()
    assert kept_cols(mk.top_k_mask(pm_from_rows([[0.6, 0.2, 0.1, 0.1]]), 0.5)) == {0, 1}
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.6, 0.2, 0.1, 0.1]]), 0.6)) == {0}
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.4, 0.3, 0.2, 0.1]]), 1.0)) == {0, 1, 2, 3}
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.4, 0.3, 0.2, 0.1]]), 0.65)) == {0, 1}
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.2, 0.5, 0.3]]), 0.0)) == {1}
    pm = pm_from_rows([[0.1] * 10])
    assert kept_cols(mk.hybrid_mask(pm, mk.SparsityConfig(0.2, 0.6, pm.b_q, pm.b_kv))) == {0, 1, 2, 3, 4, 5}
    pm = pm_from_rows([[0.6, 0.2, 0.1, 0.1]])
    assert kept_cols(mk.hybrid_mask(pm, mk.SparsityConfig(0.5, 0.6, pm.b_q, pm.b_kv))) == {0, 1}


def test_c06_top_p_minimality_vs_exhaustive_prefix():
    """test_acceptance.py:151-162 — GPU prefix count == exhaustive oracle on 500 rows."""
    rng = np.random.Generator(np.random.PCG64(31))
    edges = (1.0, 0.5, 1e-9)
    for trial in range(500):
        t_n = int(rng.integers(1, 13))
        row = rng.dirichlet(np.ones(t_n) * float(rng.uniform(0.2, 4.0)))
        p = edges[trial % 3] if trial % 7 == 0 else float(rng.uniform(0.01, 1.0))
        bm = mk.top_p_mask(pm_from_rows([row]), p)
        order = np.argsort(-row, kind="stable")
        want = next((L for L in range(1, t_n + 1) if float(row[order[:L]].sum()) >= p - 1e-12), t_n)
        assert int(bm.keep.sum()) == want


def test_c07_hybrid_is_union():
    rng = np.random.Generator(np.random.PCG64(47))
    for _ in range(60):
        t_m, t_n = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        pm = pm_from_rows(rng.dirichlet(np.ones(t_n), size=t_m))
        cfg = mk.SparsityConfig(float(rng.uniform(0.01, 1.0)), float(rng.uniform(0.01, 1.0)), pm.b_q, pm.b_kv)
        union = mk.top_k_mask(pm, cfg.k_frac) | mk.top_p_mask(pm, cfg.p_frac)
        assert np.array_equal(mk.hybrid_mask(pm, cfg).keep, union.keep)


def test_select_negative_entries_replay_numpy_binary_search():
    # rows sum to 1 but hold negative entries: the cumsum is not monotone, so the
    # count must follow numpy's binary search exactly (masker.py:133-134)
    rows = np.array([[0.9, -0.4, 0.3, 0.2], [0.7, 0.6, -0.5, 0.2], [1.5, -0.25, -0.25, 0.0]])
    pm = pm_from_rows(rows)
    for p in (0.1, 0.5, 0.85, 1.0):
        assert np.array_equal(mk.top_p_mask(pm, p).keep_numpy(), oracle.top_p_keep(rows, p)), p


def test_select_large_rows_ties():
    # T_n = 1500 with many exact ties (quantised values): order must be stable by column
    rng = np.random.Generator(np.random.PCG64(77))
    raw = rng.integers(1, 6, size=(33, 1500)).astype(np.float64)
    probs = raw / raw.sum(axis=1, keepdims=True)
    pm = pm_from_rows(probs)
    for k, p in ((0.03, 0.2), (0.0, 0.5), (0.5, 0.0), (0.01, 1.0)):
        bm = mk.hybrid_mask(pm, mk.SparsityConfig(k, p, pm.b_q, pm.b_kv))
        assert np.array_equal(bm.keep_numpy(), oracle.hybrid_keep(probs, k, p)), (k, p)


def test_pooled_map_goldens_float64(manifest, golden_pooled):
    for case in manifest["pooled"]:
        i = case["idx"]
        cfg = mk.SparsityConfig(0.5, 0.5, case["b_q"], case["b_kv"])
        pm = mk.pooled_map(golden_pooled[f"p{i}_q"], golden_pooled[f"p{i}_k"], cfg)
        want = golden_pooled[f"p{i}_probs"]
        got = np.asarray(pm.probs)
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-12, case


def test_pooled_map_reference_kats():
    cfg = mk.SparsityConfig(0.5, 0.5, 2, 2)
    pm = mk.pooled_map(np.zeros((4, 3)), np.zeros((4, 3)), cfg)  # test_masker.py:32-35
    assert np.array_equal(np.asarray(pm.probs), np.full((2, 2), 0.5))
    cfg = mk.SparsityConfig(0.5, 0.5, 4, 4)  # :38-41
    rng = np.random.Generator(np.random.PCG64(0))
    pm = mk.pooled_map(rng.normal(size=(4, 2)), rng.normal(size=(4, 2)), cfg)
    assert np.array_equal(np.asarray(pm.probs), np.array([[1.0]]))
    with pytest.raises(ValueError):  # :59-64
        mk.pooled_map(np.zeros((4, 3)), np.zeros((4, 2)), cfg)
    with pytest.raises(ValueError):
        mk.pooled_map(np.zeros((4, 3)), np.zeros((6, 3)), cfg)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32])
def test_pooled_map_bf16_inputs_match_oracle(dtype):
    q, k, _, _ = wan_like(11, 8192, 64, 128, 64, 0.9)
    cfg = mk.SparsityConfig(0.03, 0.2, 128, 64)
    qt = torch.tensor(q[0], device="cuda").to(dtype)
    kt = torch.tensor(k[0], device="cuda").to(dtype)
    pm = mk.pooled_map(qt, kt, cfg)
    want = oracle.pooled_probs(qt.double().cpu().numpy(), kt.double().cpu().numpy(), 128, 64)
    assert np.abs(pm.probs.cpu().numpy() - want).max() <= 1e-13
    keep = mk.hybrid_mask(pm, cfg).keep_numpy()
    assert (keep == oracle.hybrid_keep(want, 0.03, 0.2)).mean() >= 0.999


def test_pooled_map_batched_matches_per_head():
    q, k, _, _ = wan_like(5, 1000, 128, 128, 64, 0.8, heads=3)
    qt = torch.tensor(q, device="cuda").to(torch.bfloat16).view(1, 3, 1000, 128)
    kt = torch.tensor(k, device="cuda").to(torch.bfloat16).view(1, 3, 1000, 128)
    cfg = mk.SparsityConfig(0.1, 0.5, 128, 64)
    pm = mk.pooled_map(qt, kt, cfg)
    assert tuple(pm.probs.shape) == (1, 3, 8, 16)
    for h in range(3):
        want = oracle.pooled_probs(qt[0, h].double().cpu().numpy(), kt[0, h].double().cpu().numpy(), 128, 64)
        assert np.abs(pm.probs[0, h].cpu().numpy() - want).max() <= 1e-13


def test_pooled_map_rejects_nonfinite():
    q = np.zeros((8, 4))
    q[3, 1] = np.nan
    with pytest.raises(FloatingPointError):
        mk.pooled_map(q, np.zeros((8, 4)), mk.SparsityConfig(0.5, 0.5, 2, 2))


def test_block_mask_validation():
    with pytest.raises(ValueError, match="at least one"):
        mk.BlockMask(np.array([[True, False], [False, False]]), 2, 2, 4)
    with pytest.raises(ValueError, match="grid"):
        mk.BlockMask(np.ones((2, 3), dtype=bool), b_q=2, b_kv=2, n_tokens=4)
    bm = mk.BlockMask(np.array([[True, False, False, False]]), b_q=4, b_kv=1, n_tokens=4)
    assert bm.sparsity() == 0.75 and bm.kept_blocks() == 1


def _lists(keep_u8, bh, t_m, t_n):
    dev = keep_u8.device
    nnz_cap = bh * t_m * t_n
    row_ptr = torch.empty(bh * t_m + 1, device=dev, dtype=torch.int32)
    col_ptr = torch.empty(bh * t_n + 1, device=dev, dtype=torch.int32)
    row_idx = torch.full((nnz_cap,), -1, device=dev, dtype=torch.int32)
    col_idx = torch.full((nnz_cap,), -1, device=dev, dtype=torch.int32)
    row_order = torch.empty(bh * t_m, device=dev, dtype=torch.int32)
    col_order = torch.empty(bh * t_n, device=dev, dtype=torch.int32)
    scratch = torch.empty(bh * (t_m + t_n), device=dev, dtype=torch.int32)
    rc = _lib.load().spa2_build_lists(_lib.ptr(keep_u8), bh, t_m, t_n, _lib.ptr(row_ptr), _lib.ptr(row_idx),
                                      _lib.ptr(col_ptr), _lib.ptr(col_idx), _lib.ptr(row_order),
                                      _lib.ptr(col_order), _lib.ptr(scratch), torch.cuda.current_stream().cuda_stream)
    _lib.check(rc, "build_lists")
    return [t.cpu().numpy() for t in (row_ptr, row_idx, col_ptr, col_idx, row_order, col_order)]


@pytest.mark.parametrize("bh,t_m,t_n,density", [(1, 8, 16, 0.5), (3, 37, 71, 0.1), (2, 256, 512, 0.05),
                                                 (1, 591, 1182, 0.03)])
def test_build_lists(bh, t_m, t_n, density):
    rng = np.random.Generator(np.random.PCG64(bh * 1000 + t_m))
    keep = rng.random((bh, t_m, t_n)) < density
    keep[..., 0] |= ~keep.any(axis=-1)
    row_ptr, row_idx, col_ptr, col_idx, row_order, col_order = _lists(
        torch.tensor(keep.astype(np.uint8), device="cuda"), bh, t_m, t_n)
    flat = keep.reshape(bh * t_m, t_n)
    assert row_ptr[0] == 0 and row_ptr[-1] == keep.sum()
    for r in range(bh * t_m):
        assert np.array_equal(row_idx[row_ptr[r]:row_ptr[r + 1]], np.flatnonzero(flat[r]))
    cols = keep.transpose(0, 2, 1).reshape(bh * t_n, t_m)
    for c in range(bh * t_n):
        assert np.array_equal(col_idx[col_ptr[c]:col_ptr[c + 1]], np.flatnonzero(cols[c]))
    rc, cc = np.diff(row_ptr), np.diff(col_ptr)
    # launch orders: head-major (L2 residency), longest-first inside each head
    for order, cnt, per in ((row_order, rc, t_m), (col_order, cc, t_n)):
        assert sorted(order.tolist()) == list(range(bh * per))
        for h in range(bh):
            seg = order[h * per:(h + 1) * per]
            assert np.all(seg // per == h) and np.all(np.diff(cnt[seg]) <= 0)


def test_public_names():
    for name in ("SparsityConfig", "PooledMap", "BlockMask", "pooled_map", "top_k_mask", "top_p_mask",
                 "hybrid_mask", "expand_mask"):
        assert hasattr(spa, name)


@pytest.mark.parametrize("n,heads,s,k,p", [(32760, 12, 0.9, 0.03, 0.2), (4096, 2, 0.0, 0.1, 0.9), (777, 3, 0.5, 0.2, 0.5),
                                           (75600 // 8, 1, 0.8, 0.03, 0.16), (1000, 1, 0.7, 0.0, 0.3)])
def test_fused_softmax_select_is_bit_identical(n, heads, s, k, p):
    """sparse_attention's mask path (pooled scores + softmax inside the select kernel) gives
    exactly hybrid_mask(pooled_map(q, k)) — the map never leaves shared memory."""
    from paper_2602_13515_b200 import attention as at
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    q, kk, _ = wan_like_qkv(1, heads, n, 128, s, seed=n + heads)
    cfg = spa.SparsityConfig(k, p, 128, 64)
    fused = at._hybrid_mask_device(q, kk, cfg, None, fused=True)
    twostep = at._hybrid_mask_device(q, kk, cfg, None, fused=False)
    assert torch.equal(fused, twostep)


def test_cfg2_end_to_end_mask_disagreement():
    """configs[1] (12 heads, N = 32760): the operator's masks (GPU pooled map, fp64 from bf16
    inputs) against the float64 oracle's pooled map + hybrid rule on the same bf16 inputs.
    The select is bit-exact given a map; only pooled-score rounding (<= 1e-13) can flip a
    near-tie at the selection boundary.  The disagreement is recorded (parity_measured.json)."""
    import parity
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
    res = spa.sparse_attention(q, k, v, spa.SparsityConfig(0.03, 0.2, 128, 64))
    got = res.mask_used.keep_numpy()[0]
    diff_blocks = diff_rows = 0
    for h in range(12):
        probs = oracle.pooled_probs(q[0, h].double().cpu().numpy(), k[0, h].double().cpu().numpy(), 128, 64)
        want = oracle.hybrid_keep(probs, 0.03, 0.2)
        diff_blocks += int((got[h] != want).sum())
        diff_rows += int((got[h] != want).any(axis=1).sum())
    parity.RECORD.append({"test": parity.CURRENT_TEST["id"], "name": "cfg2_mask", "key": "mask",
                          "disagree_blocks": diff_blocks, "disagree_rows": diff_rows, "total_blocks": int(got.size),
                          "total_rows": int(got.shape[0] * got.shape[1])})
    assert diff_blocks <= 1e-4 * got.size, (diff_blocks, diff_rows)


@pytest.mark.parametrize("n,d,b_q,b_kv", [(1000, 128, 128, 64), (777, 64, 128, 64), (300, 128, 64, 64), (4100, 128, 256, 128)])
def test_block_mean_pool_entry_point(n, d, b_q, b_kv):
    """spa2_block_mean_pool (K1a alone, the reference's numerics.block_mean_pool) equals the
    oracle's float64 pooling bit for bit on bf16 inputs, ragged tails included."""
    g = torch.Generator(device="cuda").manual_seed(n + d + b_q)
    q = torch.randn(1, 2, n, d, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(1, 2, n, d, device="cuda", generator=g).to(torch.bfloat16)
    t_m, t_n = -(-n // b_q), -(-n // b_kv)
    ws = torch.full((2 * (t_m + t_n) * d,), float("nan"), device="cuda", dtype=torch.float64)
    st = torch.cuda.current_stream()
    _lib.call("spa2_block_mean_pool", _lib.view4(q), _lib.view4(k), _lib.DTYPE_CODES[q.dtype], 1, 2, n, d, b_q, b_kv,
              _lib.ptr(ws), _lib.ptr(ws[2 * t_m * d:]), None, st.cuda_stream, stream_obj=st)
    torch.cuda.synchronize()
    qbar = ws[:2 * t_m * d].view(2, t_m, d).cpu().numpy()
    kbar = ws[2 * t_m * d:].view(2, t_n, d).cpu().numpy()
    for h in range(2):
        np.testing.assert_array_equal(qbar[h], oracle.masker.block_mean_pool(q[0, h].double().cpu().numpy(), b_q))
        np.testing.assert_array_equal(kbar[h], oracle.masker.block_mean_pool(k[0, h].double().cpu().numpy(), b_kv))

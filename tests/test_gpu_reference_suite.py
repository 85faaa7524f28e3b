"""The reference's own test suite, run through the ``sparseattn_lab`` shim on the GPU.

* test_masker.py (/root/reference/pkg/tests/test_masker.py) ported unchanged: the select
  kernel takes the pooled map directly, so masks must be bit-identical to the reference's
  rules for any map and geometry (SURVEY.md §8c "port rules").
* test_attention.py ported at the kernels' shapes: d in {64, 128} and (b_q, b_kv) =
  (128, 64) (or coarser multiples / all-ones masks, which are refined exactly), with the
  reference's float64 tolerances replaced by the stated bf16 tolerance (tests/parity.py)
  against the float64 oracle run on the same bf16-rounded inputs — or exact equality
  where the bf16 arithmetic is exact (N = 1, zero gradients, identical kernels).

Inputs are numpy, as in the reference; results come back as numpy float64.
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle
from gen import to_bf16
from parity import assert_close
from sparseattn_lab import attention as at
from sparseattn_lab import masker as mk
from sparseattn_lab import numerics as nm

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- masker (test_masker.py)

def pm_from_rows(rows):  # test_masker.py:11-15
    probs = np.atleast_2d(np.asarray(rows, dtype=np.float64))
    t_m, t_n = probs.shape
    return mk.PooledMap(probs, b_q=t_n, b_kv=t_m, n_tokens=t_m * t_n)


def kept_cols(bm, row=0):
    assert isinstance(bm.keep, np.ndarray) and not bm.keep.flags.writeable  # reference types
    return set(np.flatnonzero(bm.keep[row]))


def test_pooled_map_zeros_is_uniform():  # test_masker.py:32-35
    cfg = mk.SparsityConfig(0.5, 0.5, 2, 2)
    pm = mk.pooled_map(np.zeros((4, 3)), np.zeros((4, 3)), cfg)
    assert isinstance(pm.probs, np.ndarray) and not pm.probs.flags.writeable
    np.testing.assert_array_equal(pm.probs, np.full((2, 2), 0.5))


def test_pooled_map_single_block():  # test_masker.py:38-41
    cfg = mk.SparsityConfig(0.5, 0.5, 4, 4)
    pm = mk.pooled_map(nm.make_rng(0).normal(size=(4, 2)), nm.make_rng(1).normal(size=(4, 2)), cfg)
    np.testing.assert_array_equal(pm.probs, np.array([[1.0]]))


def test_pooled_map_matches_by_hand_oracle():  # test_masker.py:44-56
    rng = nm.make_rng(5)
    q = rng.normal(size=(8, 4))
    k = rng.normal(size=(8, 4))
    cfg = mk.SparsityConfig(0.5, 0.5, 3, 2)
    pm = mk.pooled_map(q, k, cfg)
    qb = np.array([q[0:3].mean(axis=0), q[3:6].mean(axis=0), q[6:8].mean(axis=0)])
    kb = np.array([k[0:2].mean(axis=0), k[2:4].mean(axis=0), k[4:6].mean(axis=0), k[6:8].mean(axis=0)])
    s = qb @ kb.T / np.sqrt(4)
    want = np.array([np.exp(r - r.max()) / np.exp(r - r.max()).sum() for r in s])
    np.testing.assert_allclose(pm.probs, want, atol=1e-12)


def test_pooled_map_rejects_mismatched_shapes():  # test_masker.py:59-64
    cfg = mk.SparsityConfig(0.5, 0.5, 2, 2)
    with pytest.raises(ValueError):
        mk.pooled_map(np.zeros((4, 3)), np.zeros((4, 2)), cfg)
    with pytest.raises(ValueError):
        mk.pooled_map(np.zeros((4, 3)), np.zeros((6, 3)), cfg)


def test_pooled_map_rejects_non_finite():  # numerics.py:29-32
    cfg = mk.SparsityConfig(0.5, 0.5, 2, 2)
    q = np.zeros((4, 3))
    q[1, 2] = np.inf
    with pytest.raises(FloatingPointError):
        mk.pooled_map(q, np.zeros((4, 3)), cfg)


def test_top_k_uniform_row_tie_rule():  # test_masker.py:67-70
    assert kept_cols(mk.top_k_mask(pm_from_rows([[0.1] * 10]), 0.2)) == {0, 1}


def test_top_k_full_fraction_keeps_all():  # test_masker.py:73-75
    assert mk.top_k_mask(pm_from_rows([[0.1] * 10]), 1.0).keep.all()


def test_top_k_sink_row():  # test_masker.py:78-80
    assert kept_cols(mk.top_k_mask(pm_from_rows([[0.6, 0.2, 0.1, 0.1]]), 0.5)) == {0, 1}


def test_top_p_sink_row_keeps_only_sink():  # test_masker.py:83-85
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.6, 0.2, 0.1, 0.1]]), 0.6)) == {0}


def test_top_p_full_mass_keeps_all_nonzero():  # test_masker.py:88-90
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.4, 0.3, 0.2, 0.1]]), 1.0)) == {0, 1, 2, 3}


def test_top_p_two_needed():  # test_masker.py:93-95
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.4, 0.3, 0.2, 0.1]]), 0.65)) == {0, 1}


def test_top_p_zero_keeps_single_largest():  # test_masker.py:98-100
    assert kept_cols(mk.top_p_mask(pm_from_rows([[0.2, 0.5, 0.3]]), 0.0)) == {1}


def test_hybrid_uniform_row_top_p_dominates():  # test_masker.py:103-107
    pm = pm_from_rows([[0.1] * 10])
    assert kept_cols(mk.hybrid_mask(pm, mk.SparsityConfig(0.2, 0.6, pm.b_q, pm.b_kv))) == {0, 1, 2, 3, 4, 5}


def test_hybrid_sink_row_top_k_dominates():  # test_masker.py:110-113
    pm = pm_from_rows([[0.6, 0.2, 0.1, 0.1]])
    assert kept_cols(mk.hybrid_mask(pm, mk.SparsityConfig(0.5, 0.6, pm.b_q, pm.b_kv))) == {0, 1}


def test_hybrid_k_one_keeps_everything():  # test_masker.py:116-119
    pm = pm_from_rows(nm.make_rng(3).dirichlet(np.ones(7), size=4))
    assert mk.hybrid_mask(pm, mk.SparsityConfig(1.0, 0.1, pm.b_q, pm.b_kv)).keep.all()


def random_pm(seed, t_m=6, t_n=9, alpha=1.0):  # test_masker.py:150-152
    return pm_from_rows(nm.make_rng(seed).dirichlet(np.full(t_n, alpha), size=t_m))


@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 10**6), k_frac=st.floats(0.0, 1.0), p_frac=st.floats(0.0, 1.0))
def test_hybrid_is_elementwise_or(seed, k_frac, p_frac):  # test_masker.py:155-161
    pm = random_pm(seed)
    cfg = mk.SparsityConfig(k_frac, p_frac, pm.b_q, pm.b_kv)
    want = mk.top_k_mask(pm, k_frac).keep | mk.top_p_mask(pm, p_frac).keep
    np.testing.assert_array_equal(mk.hybrid_mask(pm, cfg).keep, want)


@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 10**6), k_frac=st.floats(0.0, 1.0))
def test_top_k_cardinality(seed, k_frac):  # test_masker.py:164-170
    pm = random_pm(seed)
    t_n = pm.probs.shape[1]
    counts = mk.top_k_mask(pm, k_frac).keep.sum(axis=1)
    assert np.all(counts == max(1, int(np.ceil(k_frac * t_n))))


@settings(max_examples=200, deadline=None)
@given(seed=st.integers(0, 10**6), t_n=st.integers(1, 12), p_frac=st.floats(0.0, 1.0),
       alpha=st.sampled_from([0.3, 1.0, 5.0]))
def test_top_p_minimality_vs_prefix_oracle(seed, t_n, p_frac, alpha):  # test_masker.py:173-186
    probs = nm.make_rng(seed).dirichlet(np.full(t_n, alpha), size=3)
    bm = mk.top_p_mask(pm_from_rows(probs), p_frac)
    for i, row in enumerate(probs):
        assert bm.keep[i].sum() == min(oracle.top_p_count(row, p_frac), t_n)


@settings(max_examples=100, deadline=None)
@given(seed=st.integers(0, 10**6), lo=st.floats(0.0, 1.0), hi=st.floats(0.0, 1.0))
def test_masks_monotone_in_fraction(seed, lo, hi):  # test_masker.py:189-196
    lo, hi = min(lo, hi), max(lo, hi)
    pm = random_pm(seed)
    assert not (mk.top_k_mask(pm, lo).keep & ~mk.top_k_mask(pm, hi).keep).any()
    assert not (mk.top_p_mask(pm, lo).keep & ~mk.top_p_mask(pm, hi).keep).any()


def test_masks_deterministic():  # test_masker.py:199-204
    pm = random_pm(77)
    cfg = mk.SparsityConfig(0.3, 0.7, pm.b_q, pm.b_kv)
    np.testing.assert_array_equal(mk.hybrid_mask(pm, cfg).keep, mk.hybrid_mask(pm, cfg).keep)


def test_hybrid_supersets_both_rules():  # test_masker.py:207-215
    pm = random_pm(41, alpha=0.4)
    cfg = mk.SparsityConfig(0.25, 0.5, pm.b_q, pm.b_kv)
    hy, tk, tp = mk.hybrid_mask(pm, cfg), mk.top_k_mask(pm, cfg.k_frac), mk.top_p_mask(pm, cfg.p_frac)
    assert np.all(hy.keep.sum(axis=1) >= np.maximum(tk.keep.sum(axis=1), tp.keep.sum(axis=1)))
    assert hy.sparsity() <= min(tk.sparsity(), tp.sparsity())


def test_mask_csv_round_trip_of_gpu_mask(tmp_path):  # test_masker.py:243-253
    pm = random_pm(13)
    bm = mk.hybrid_mask(pm, mk.SparsityConfig(0.2, 0.5, pm.b_q, pm.b_kv))
    p = tmp_path / "mask.csv"
    mk.write_mask_csv(p, bm)
    back = mk.read_mask_csv(p)
    np.testing.assert_array_equal(back.keep, bm.keep)
    assert (back.b_q, back.b_kv, back.n_tokens) == (bm.b_q, bm.b_kv, bm.n_tokens)


# ----------------------------------------------------------- attention (test_attention.py)

D_VALUES = (64, 128)


def rand_qkv(seed, n, d):  # test_attention.py:12-14, rounded to the bf16 values the GPU computes on
    rng = nm.make_rng(seed)
    return tuple(to_bf16(rng.normal(size=(n, d))) for _ in range(3))


def random_mask(seed, n, b_q=128, b_kv=64, density=0.5):  # test_attention.py:17-22
    rng = nm.make_rng(seed)
    t_m, t_n = nm.num_blocks(n, b_q), nm.num_blocks(n, b_kv)
    keep = rng.random((t_m, t_n)) < density
    keep[~keep.any(axis=1), 0] = True
    return mk.BlockMask(keep, b_q, b_kv, n)


@pytest.mark.parametrize("d", D_VALUES)
def test_dense_single_token_returns_v(d):  # test_attention.py:29-31 — exact in bf16 (one key, P = 1)
    q, k, v = rand_qkv(0, 1, d)
    res = at.dense_attention(q, k, v)
    assert isinstance(res.out, np.ndarray) and res.out.shape == (1, d)
    np.testing.assert_array_equal(res.out, v)
    np.testing.assert_allclose(res.lse, (q @ k.T / np.sqrt(d))[:, 0], atol=2e-3)


@pytest.mark.parametrize("d", D_VALUES)
def test_dense_zero_queries_average_v(d):  # test_attention.py:34-37
    _, k, v = rand_qkv(1, 7, d)
    res = at.dense_attention(np.zeros((7, d)), k, v)
    assert_close(f"zero_q.d{d}", res.out, np.tile(v.mean(axis=0), (7, 1)), "out")
    np.testing.assert_allclose(res.lse, np.log(7.0), atol=1e-6)


@pytest.mark.parametrize("d", D_VALUES)
def test_dense_matches_naive_oracle(d):  # test_attention.py:40-42
    q, k, v = rand_qkv(2, 16, d)
    out, lse = oracle.dense_attention(q, k, v)
    res = at.dense_attention(q, k, v)
    assert_close(f"dense16.d{d}.out", res.out, out, "out")
    assert_close(f"dense16.d{d}.lse", res.lse, lse, "lse")


@pytest.mark.parametrize("d", D_VALUES)
def test_dense_lse_consistent(d):  # test_attention.py:45-49
    q, k, v = rand_qkv(3, 12, d)
    s = q @ k.T / np.sqrt(d)
    want = np.log(np.exp(s - s.max(1, keepdims=True)).sum(1)) + s.max(1)
    assert_close(f"lse12.d{d}", at.dense_attention(q, k, v).lse, want, "lse")


def test_dense_shape_mismatch():  # test_attention.py:52-54
    with pytest.raises(ValueError):
        at.dense_attention(np.zeros((4, 64)), np.zeros((4, 128)), np.zeros((4, 64)))


def test_unsupported_head_dim_raises():  # d outside {64, 128} is a ValueError, no fallback
    with pytest.raises(ValueError, match="head dim"):
        at.dense_attention(np.zeros((4, 5)), np.zeros((4, 5)), np.zeros((4, 5)))


def test_unsupported_block_geometry_raises():  # b_q not a multiple of 64
    q, k, v = rand_qkv(4, 256, 64)
    bm = random_mask(4, 256, b_q=32, b_kv=64)
    with pytest.raises(ValueError, match="b_q=128"):
        at.sparse_attention_with_mask(q, k, v, bm)


@pytest.mark.parametrize("d", D_VALUES)
def test_sparse_full_k_frac_equals_dense(d):  # test_attention.py:57-62 — same kernels, same tiles: bit-equal
    q, k, v = rand_qkv(4, 300, d)
    res = at.sparse_attention(q, k, v, mk.SparsityConfig(1.0, 0.5, 128, 64))
    assert res.mask_used.keep.all()
    np.testing.assert_array_equal(res.out, at.dense_attention(q, k, v).out)


@pytest.mark.parametrize("d", D_VALUES)
def test_sparse_diagonal_mask_per_block_oracle(d):  # test_attention.py:65-71
    q, k, v = rand_qkv(5, 256, d)
    bm = mk.BlockMask(np.eye(2, dtype=bool), b_q=128, b_kv=128, n_tokens=256)
    res = at.sparse_attention_with_mask(q, k, v, bm)
    for blk in range(2):
        sl = slice(128 * blk, 128 * blk + 128)
        assert_close(f"diag.d{d}.{blk}", res.out[sl], oracle.dense_attention(q[sl], k[sl], v[sl])[0], "out")


def test_sparse_default_config_smoke():  # test_attention.py:74-78 (paper defaults at the kernel grid)
    rng = nm.make_rng(6)
    n, d = 4096, 64
    off = lambda b: np.repeat(rng.normal(size=(-(-n // b), d)), b, axis=0)[:n]
    q, k, v = to_bf16(rng.normal(size=(n, d)) + off(128)), to_bf16(rng.normal(size=(n, d)) + off(64)), \
        to_bf16(rng.normal(size=(n, d)))
    res = at.sparse_attention(q, k, v, mk.SparsityConfig(0.03, 0.2, 128, 64))
    assert np.all(np.isfinite(res.out))
    assert 0.5 <= res.mask_used.sparsity() < 1.0
    assert isinstance(res.mask_used.keep, np.ndarray)


@pytest.mark.parametrize("d", D_VALUES)
def test_with_mask_all_ones_equals_dense(d):  # test_attention.py:80-83
    q, k, v = rand_qkv(7, 320, d)
    res = at.sparse_attention_with_mask(q, k, v, at.full_mask(320))
    np.testing.assert_array_equal(res.out, at.dense_attention(q, k, v).out)


@pytest.mark.parametrize("d", D_VALUES)
def test_with_mask_single_block_rows(d):  # test_attention.py:86-97
    q, k, v = rand_qkv(8, 384, d)
    keep = np.array([[True, False, False], [False, False, True], [False, True, False]])
    bm = mk.BlockMask(keep, b_q=128, b_kv=128, n_tokens=384)
    res = at.sparse_attention_with_mask(q, k, v, bm)
    for i in range(3):
        j = int(np.flatnonzero(keep[i])[0])
        sl_q, sl_k = slice(128 * i, 128 * i + 128), slice(128 * j, 128 * j + 128)
        s = q[sl_q] @ k[sl_k].T / np.sqrt(d)
        p = np.exp(s - s.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        assert_close(f"single_rows.d{d}.{i}", res.out[sl_q], p @ v[sl_k], "out")


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
@pytest.mark.parametrize("d", D_VALUES)
def test_with_mask_matches_token_level_oracle(seed, d):  # test_attention.py:100-107
    n = 300 + 97 * seed  # ragged tails
    q, k, v = rand_qkv(100 + seed, n, d)
    bm = random_mask(seed, n)
    res = at.sparse_attention_with_mask(q, k, v, bm)
    want = oracle.masked_attention_tokens(q, k, v, mk.expand_mask(bm))
    assert_close(f"token_oracle.s{seed}.d{d}", res.out, want, "out")


@pytest.mark.parametrize("d", D_VALUES)
def test_block_visit_order_invariance(d):  # test_attention.py:110-121
    n = 700
    q, k, v = rand_qkv(9, n, d)
    bm = random_mask(9, n, density=0.7)
    base = at.sparse_attention_with_mask(q, k, v, bm)
    shuffler = nm.make_rng(1234)
    for _ in range(5):
        permuted = at.sparse_attention_with_mask(q, k, v, bm, _block_order=lambda i, kept: shuffler.permutation(kept))
        assert_close(f"visit.d{d}.out", permuted.out, base.out, "out")
        assert_close(f"visit.d{d}.lse", permuted.lse, base.lse, "lse")


def test_block_visit_order_hook_sees_the_mask_grid():  # attention.py:97-99 on a coarse (256, 128) mask
    n, d = 600, 64
    q, k, v = rand_qkv(19, n, d)
    bm = random_mask(19, n, b_q=256, b_kv=128, density=0.6)
    seen = []
    res = at.sparse_attention_with_mask(q, k, v, bm, _block_order=lambda i, kept: seen.append((i, list(kept))) or
                                        kept[::-1])
    assert sorted(seen) == [(i, list(np.flatnonzero(bm.keep[i]))) for i in range(bm.keep.shape[0])]
    want = oracle.masked_attention_tokens(q, k, v, mk.expand_mask(bm))
    assert_close("visit_coarse.out", res.out, want, "out")


@pytest.mark.parametrize("d", D_VALUES)
def test_renormalization_weights_sum_to_one(d):  # test_attention.py:124-132
    n = 500
    q, k, v = rand_qkv(10, n, d)
    bm = random_mask(10, n)
    res = at.sparse_attention_with_mask(q, k, v, bm)
    em = mk.expand_mask(bm)
    s = q @ k.T / np.sqrt(d)
    weights = np.exp(s - res.lse[:, None]) * em
    np.testing.assert_allclose(weights.sum(axis=1), 1.0, atol=2e-3)  # fp32 LSE


@settings(max_examples=10, deadline=None)
@given(seed=st.integers(0, 10**6))
def test_output_rows_convex_in_selected_v(seed):  # test_attention.py:135-146 (+ bf16 output rounding)
    n, d = 256, 64
    q, k, v = rand_qkv(seed, n, d)
    bm = random_mask(seed, n)
    res = at.sparse_attention_with_mask(q, k, v, bm)
    em = mk.expand_mask(bm).astype(bool)
    for a in range(n):
        sel = v[em[a]]
        lo, hi = sel.min(axis=0), sel.max(axis=0)
        slack = 2 ** -8 * np.maximum(np.abs(lo), np.abs(hi))
        assert np.all(res.out[a] >= lo - slack) and np.all(res.out[a] <= hi + slack)


@pytest.mark.parametrize("geometry", [(128, 64), (256, 128), (128, 192)])
def test_counter_counts_exactly_kept_blocks(geometry):  # test_attention.py:149-155
    n = 900
    q, k, v = rand_qkv(11, n, 64)
    bm = random_mask(11, n, *geometry, density=0.4)
    ctr = at.BlockCounter()
    at.sparse_attention_with_mask(q, k, v, bm, counter=ctr)
    assert ctr.count == bm.kept_blocks()


def test_counter_full_mask_counts_one_block():  # the reference visits full_mask(N)'s single block once
    q, k, v = rand_qkv(11, 300, 64)
    ctr = at.BlockCounter()
    at.sparse_attention_with_mask(q, k, v, at.full_mask(300), counter=ctr)
    assert ctr.count == 1


def test_counter_with_derived_mask():  # test_attention.py:158-163
    q, k, v = rand_qkv(12, 1024, 64)
    ctr = at.BlockCounter()
    res = at.sparse_attention(q, k, v, mk.SparsityConfig(0.1, 0.3, 128, 64), counter=ctr)
    assert ctr.count == res.mask_used.kept_blocks()


def test_mask_token_count_mismatch():  # test_attention.py:166-169
    q, k, v = rand_qkv(13, 128, 64)
    with pytest.raises(ValueError, match="tokens"):
        at.sparse_attention_with_mask(q, k, v, at.full_mask(256))


def test_non_finite_inputs_raise():  # numerics.py:29-32 via attention._check_qkv (attention.py:50-59)
    q, k, v = rand_qkv(13, 128, 64)
    for bad in ("q", "k", "v"):
        args = {"q": q.copy(), "k": k.copy(), "v": v.copy()}
        args[bad][3, 5] = np.nan
        with pytest.raises(FloatingPointError):
            at.sparse_attention(args["q"], args["k"], args["v"], mk.SparsityConfig(0.5, 0.5, 128, 64))


@pytest.mark.parametrize("d", D_VALUES)
def test_backward_zero_dout(d):  # test_attention.py:175-178 — exact zeros
    q, k, v = rand_qkv(14, 200, d)
    g = at.attention_backward(q, k, v, at.full_mask(200), np.zeros((200, d)))
    assert not g.dq.any() and not g.dk.any() and not g.dv.any()


@pytest.mark.parametrize("d", D_VALUES)
def test_backward_dense_mask_vs_oracle(d):  # test_attention.py:194-195 (FD-pinned oracle: test_oracle.py)
    n = 260
    q, k, v = rand_qkv(15, n, d)
    w = to_bf16(nm.make_rng(15 + 991).normal(size=(n, d)))
    g = at.attention_backward(q, k, v, at.full_mask(n), w)
    dq, dk, dv, _, _ = oracle.attention_backward(q, k, v, np.ones((1, 1), bool), n, n, w)
    for name, got, want in (("dq", g.dq, dq), ("dk", g.dk, dk), ("dv", g.dv, dv)):
        assert_close(f"bwd_dense.d{d}.{name}", got, want, name)


@pytest.mark.parametrize("d", D_VALUES)
def test_backward_dropped_column_gets_zero_grad(d):  # test_attention.py:198-204
    n = 256
    keep = np.array([[True, False], [True, False]])
    bm = mk.BlockMask(keep, b_q=128, b_kv=128, n_tokens=n)
    q, k, v = rand_qkv(16, n, d)
    w = to_bf16(nm.make_rng(16 + 991).normal(size=(n, d)))
    g = at.attention_backward(q, k, v, bm, w)
    assert not g.dk[128:].any()
    assert not g.dv[128:].any()
    dq, dk, dv, _, _ = oracle.attention_backward(q, k, v, keep, 128, 128, w)
    for name, got, want in (("dq", g.dq, dq), ("dk", g.dk, dk), ("dv", g.dv, dv)):
        assert_close(f"bwd_dropped.d{d}.{name}", got, want, name)


@pytest.mark.parametrize("seed", [21, 22, 23])
@pytest.mark.parametrize("d", D_VALUES)
def test_backward_random_masks_vs_oracle(seed, d):  # test_attention.py:207-211
    n = 333 + seed
    bm = random_mask(seed, n, density=0.5)
    q, k, v = rand_qkv(seed, n, d)
    w = to_bf16(nm.make_rng(seed + 991).normal(size=(n, d)))
    g = at.attention_backward(q, k, v, bm, w)
    dq, dk, dv, _, _ = oracle.attention_backward(q, k, v, bm.keep, 128, 64, w)
    for name, got, want in (("dq", g.dq, dq), ("dk", g.dk, dk), ("dv", g.dv, dv)):
        assert_close(f"bwd_random.s{seed}.d{d}.{name}", got, want, name)

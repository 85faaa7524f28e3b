"""The reference's own masker tests that need no GPU, run through the ``sparseattn_lab`` shim.

Ported from /root/reference/pkg/tests/test_masker.py (line numbers cited per test).  The
shim resolves ``sparseattn_lab.masker`` to this package's module; numpy callers get the
reference's types (read-only numpy arrays) and the reference's exceptions.  Everything here
runs on the host — BlockMask / PooledMap validation, expand_mask, sparsity, mask CSV —
so these checks also run in the CPU-only CI.
"""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2602_13515_b200 as spa
from sparseattn_lab import attention as at
from sparseattn_lab import masker as mk
from sparseattn_lab import numerics as nm


def test_shim_resolves_to_the_gpu_modules():
    import sparseattn_lab.attention
    import sparseattn_lab.masker

    assert sparseattn_lab.masker is spa.masker and sparseattn_lab.attention is spa.attention
    assert mk.hybrid_mask is spa.hybrid_mask and at.sparse_attention is spa.sparse_attention


def test_config_validation():  # test_masker.py:22-29
    mk.SparsityConfig(0.0, 1.0, 1, 1)
    with pytest.raises(ValueError):
        mk.SparsityConfig(-0.1, 0.5, 4, 4)
    with pytest.raises(ValueError):
        mk.SparsityConfig(0.5, 1.5, 4, 4)
    with pytest.raises(ValueError):
        mk.SparsityConfig(0.5, 0.5, 0, 4)


def test_expand_single_block():  # test_masker.py:122-124
    bm = mk.BlockMask(np.ones((1, 1), dtype=bool), b_q=3, b_kv=3, n_tokens=3)
    got = mk.expand_mask(bm)
    assert isinstance(got, np.ndarray) and got.dtype == np.float64
    np.testing.assert_array_equal(got, np.ones((3, 3)))


def test_expand_block_diagonal():  # test_masker.py:127-132
    bm = mk.BlockMask(np.eye(2, dtype=bool), b_q=2, b_kv=2, n_tokens=4)
    want = np.zeros((4, 4))
    want[:2, :2] = 1.0
    want[2:, 2:] = 1.0
    np.testing.assert_array_equal(mk.expand_mask(bm), want)


@settings(max_examples=50, deadline=None)
@given(seed=st.integers(0, 10**6), n=st.integers(2, 30), b_q=st.integers(1, 7), b_kv=st.integers(1, 7))
def test_expand_every_token_matches_its_block(seed, n, b_q, b_kv):  # test_masker.py:135-147
    rng = nm.make_rng(seed)
    t_m, t_n = nm.num_blocks(n, b_q), nm.num_blocks(n, b_kv)
    keep = rng.random((t_m, t_n)) < 0.5
    keep[~keep.any(axis=1), 0] = True
    bm = mk.BlockMask(keep, b_q, b_kv, n)
    em = mk.expand_mask(bm)
    assert em.shape == (n, n)
    for a in range(n):
        for b in range(n):
            assert em[a, b] == float(keep[a // b_q, b // b_kv])


def test_block_mask_rejects_empty_row():  # test_masker.py:225-228
    keep = np.array([[True, False], [False, False]])
    with pytest.raises(ValueError, match="at least one"):
        mk.BlockMask(keep, 2, 2, 4)


def test_block_mask_rejects_wrong_grid():  # test_masker.py:231-233
    with pytest.raises(ValueError, match="grid"):
        mk.BlockMask(np.ones((2, 3), dtype=bool), b_q=2, b_kv=2, n_tokens=4)


def test_block_mask_rejects_wrong_rank():  # masker.py:75-76
    with pytest.raises(ValueError, match="rank 2"):
        mk.BlockMask(np.ones((2,), dtype=bool), b_q=2, b_kv=2, n_tokens=4)


def test_sparsity_value():  # test_masker.py:236-240
    keep = np.array([[True, False, False, False]])
    bm = mk.BlockMask(keep, b_q=4, b_kv=1, n_tokens=4)
    assert bm.sparsity() == 0.75
    assert bm.kept_blocks() == 1


def test_host_containers_are_readonly_reference_types():  # masker.py:56-58, 73-75
    bm = mk.BlockMask(np.array([[1, 0], [1, 1]]), b_q=2, b_kv=2, n_tokens=4)
    assert isinstance(bm.keep, np.ndarray) and bm.keep.dtype == bool and not bm.keep.flags.writeable
    with pytest.raises(ValueError):
        bm.keep[0, 0] = False
    pm = mk.PooledMap(np.array([[0.25, 0.75], [0.5, 0.5]]), b_q=2, b_kv=2, n_tokens=4)
    assert isinstance(pm.probs, np.ndarray) and not pm.probs.flags.writeable
    # the reference-style caller expression (cli.py:149-150) works on host objects
    assert float((pm.probs * bm.keep).sum(axis=1)[0]) == 0.25


def test_pooled_map_validation_on_host():  # masker.py:54-62
    with pytest.raises(ValueError, match="sum to 1"):
        mk.PooledMap(np.array([[0.5, 0.6]]), 1, 1, 2)
    with pytest.raises(FloatingPointError):
        mk.PooledMap(np.array([[np.nan, 1.0]]), 1, 1, 2)
    with pytest.raises(ValueError):  # ShapeError is a ValueError
        mk.PooledMap(np.ones((1, 1, 1)), 1, 1, 1)
    batched = mk.BlockMask(np.ones((1, 2, 2, 2), dtype=bool), 2, 2, 4)  # [B, H, T_m, T_n] extension
    assert batched.kept_blocks() == 8


def test_union_of_host_masks_stays_on_host():  # masker.py:94-97
    a = mk.BlockMask(np.array([[1, 0], [0, 1]]), 2, 2, 4)
    b = mk.BlockMask(np.array([[0, 1], [0, 1]]), 2, 2, 4)
    u = a | b
    assert isinstance(u.keep, np.ndarray)
    np.testing.assert_array_equal(u.keep, [[True, True], [False, True]])
    with pytest.raises(ValueError, match="geometry"):
        a | mk.BlockMask(np.array([[1, 1]]), 2, 1, 2)


def test_mask_csv_round_trip(tmp_path):  # test_masker.py:243-253 (host mask; GPU-derived masks in test_formats)
    rng = nm.make_rng(13)
    keep = rng.random((6, 9)) < 0.4
    keep[~keep.any(axis=1), 0] = True
    bm = mk.BlockMask(keep, b_q=9, b_kv=6, n_tokens=54)
    p = tmp_path / "mask.csv"
    mk.write_mask_csv(p, bm)
    back = mk.read_mask_csv(p)
    np.testing.assert_array_equal(back.keep, bm.keep)
    assert (back.b_q, back.b_kv, back.n_tokens) == (bm.b_q, bm.b_kv, bm.n_tokens)
    lines = p.read_text().splitlines()
    assert lines[0] == f"b_q={bm.b_q},b_kv={bm.b_kv},n_tokens={bm.n_tokens}"
    assert lines[1].startswith("c0,")


def test_full_mask_is_the_reference_host_mask():  # attention.py:46-47
    fm = at.full_mask(16)
    assert isinstance(fm.keep, np.ndarray) and fm.keep.shape == (1, 1) and fm.keep.all()
    assert (fm.b_q, fm.b_kv, fm.n_tokens) == (16, 16, 16)


def test_block_counter_interface():  # attention.py:36-43
    c = at.BlockCounter()
    c.hit(0, 1)
    c.hit(2, 3)
    assert c.count == 2

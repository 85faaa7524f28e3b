"""Masks with b_q = 64 (SURVEY.md §7 scopes b ∈ {64, 128}) and other 64-row multiples.

The kernels tile 128 query rows; a b_q = 64 mask pairs two mask rows per query block, the
block lists carry which half keeps each tile (csrc/common.cuh list entries), and the
forward / dQ / dK/dV kernels give the other half's rows P = 0 for that tile.  Checked against
the float64 oracle at the mask's own geometry (fwd, LSE, dq, dk, dv), ragged N (incl. a last
query block without a bottom half), the masker → operator path with b_q = 64, the counter and
the visit-order hook on the mask's grid."""

import numpy as np
import pytest
import torch

import oracle
import paper_2602_13515_b200 as spa
from gen import random_keep, wan_like
from parity import assert_close

pytestmark = pytest.mark.gpu


def _check(n, d, b_q, b_kv, density, seed, heads=1):
    q, k, v, do = wan_like(seed, n, d, b_q, b_kv, 0.6, heads=heads)
    t_m, t_n = -(-n // b_q), -(-n // b_kv)
    keep = np.stack([random_keep(seed + h, t_m, t_n, density) for h in range(heads)])
    t = lambda x: torch.tensor(x, device="cuda").to(torch.bfloat16).view(1, heads, n, d)  # noqa: E731
    qd, kd, vd = (t(x).requires_grad_(True) for x in (q, k, v))
    bm = spa.BlockMask(torch.tensor(keep.reshape(1, heads, t_m, t_n), device="cuda"), b_q, b_kv, n)
    res = spa.sparse_attention_with_mask(qd, kd, vd, bm)
    res.out.backward(t(do))
    for h in range(heads):
        dq, dk, dv, out, lse = oracle.attention_backward(q[h], k[h], v[h], keep[h], b_q, b_kv, do[h])
        tag = f"bq{b_q}.bkv{b_kv}.n{n}.d{d}.h{h}"
        assert_close(f"{tag}.out", res.out[0, h], out, "out")
        assert_close(f"{tag}.lse", res.lse[0, h], lse, "lse")
        assert_close(f"{tag}.dq", qd.grad[0, h], dq, "dq")
        assert_close(f"{tag}.dk", kd.grad[0, h], dk, "dk")
        assert_close(f"{tag}.dv", vd.grad[0, h], dv, "dv")
        # key blocks no query row keeps get exact zeros (attention.py:152-157)
        tok_keep = oracle.expand_keep(keep[h], b_q, b_kv, n).any(axis=0)
        assert not kd.grad[0, h][torch.tensor(~tok_keep, device="cuda")].any()


@pytest.mark.parametrize("n,d,b_q,b_kv,density", [
    (1000, 128, 64, 64, 0.3), (777, 64, 64, 64, 0.5), (1100, 128, 64, 128, 0.4), (600, 128, 192, 64, 0.4),
    (129, 64, 64, 64, 0.6), (64, 128, 64, 64, 1.0), (4100, 128, 64, 64, 0.05)])
def test_bq64_fwd_bwd_vs_oracle(n, d, b_q, b_kv, density):
    _check(n, d, b_q, b_kv, density, seed=n + b_q)


def test_bq64_batched_heads():
    _check(900, 128, 64, 64, 0.25, seed=7, heads=3)


def test_bq64_masker_to_operator():
    """hybrid mask at b_q = 64 from the masker, then the operator (the reference's
    sparse_attention with SparsityConfig(k, p, 64, 64))."""
    n, d = 2048, 128
    q, k, v, _ = wan_like(11, n, d, 64, 64, 0.8)
    cfg = spa.SparsityConfig(0.1, 0.3, 64, 64)
    qt, kt, vt = (torch.tensor(x[0], device="cuda").to(torch.bfloat16) for x in (q, k, v))
    res = spa.sparse_attention(qt, kt, vt, cfg)
    keep = res.mask_used.keep_numpy()
    assert keep.shape == (32, 32)
    probs = spa.pooled_map(qt, kt, cfg).probs.cpu().numpy()
    assert np.array_equal(keep, oracle.hybrid_keep(probs, 0.1, 0.3))
    out, lse, _ = oracle.sparse_forward(*(x.double().cpu().numpy() for x in (qt, kt, vt)), keep, 64, 64)
    assert_close("bq64.masker.out", res.out, out, "out")
    ctr = spa.BlockCounter()
    spa.sparse_attention_with_mask(qt, kt, vt, res.mask_used, counter=ctr)
    assert ctr.count == res.mask_used.kept_blocks()


def test_bq64_visit_order_hook_on_mask_grid():
    n, d = 640, 64
    q, k, v, _ = wan_like(13, n, d, 64, 64, 0.5)
    keep = random_keep(13, 10, 10, 0.5)
    bm = spa.BlockMask(keep, 64, 64, n)
    seen = []

    def visit(i, kept):
        seen.append((i, list(kept)))
        return kept[::-1]

    res = spa.sparse_attention_with_mask(q[0], k[0], v[0], bm, _block_order=visit)
    assert sorted(seen) == [(i, list(np.flatnonzero(keep[i]))) for i in range(10)]
    out, _, _ = oracle.sparse_forward(q[0], k[0], v[0], keep, 64, 64)
    assert_close("bq64.visit.out", res.out, out, "out")

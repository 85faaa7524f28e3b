"""Wan2.1-14B 720p attention shape (configs[3]: N=75600, d=128, k=0.03, p=0.16), two heads:
T_n = 1182 key blocks (2048-wide selection path), ragged tails (80-row query / 16-row key
block).  Masks bit-exact vs the oracle on the GPU's own pooled map, forward + dQ checked on a
slice of query blocks, dK/dV checked exactly for chosen key blocks (their full column lists, with the oracle's own
forward statistics)."""

import math

import numpy as np
import pytest
import torch
from parity import assert_close

import oracle
import paper_2602_13515_b200 as spa
from paper_2602_13515_b200.synthetic import wan_like_qkv

pytestmark = pytest.mark.gpu
N, D, H = 75600, 128, 2


@pytest.fixture(scope="module")
def run():
    q, k, v = wan_like_qkv(1, H, N, D, 0.8, seed=14)
    do = torch.randn(q.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(15)).to(q.dtype)
    qs, ks, vs = (t.clone().requires_grad_(True) for t in (q, k, v))
    cfg = spa.SparsityConfig(0.03, 0.16, 128, 64)
    res = spa.sparse_attention(qs, ks, vs, cfg)
    res.out.backward(do)
    torch.cuda.synchronize()
    host = [t[0].double().cpu().numpy() for t in (q, k, v, do)]
    return res, (qs.grad[0], ks.grad[0], vs.grad[0]), host, cfg


def test_mask_bit_exact_and_sparse(run):
    res, _, host, cfg = run
    q, k = host[0], host[1]
    pm = spa.pooled_map(torch.tensor(q[0], device="cuda").to(torch.bfloat16),
                        torch.tensor(k[0], device="cuda").to(torch.bfloat16), cfg)
    probs = pm.probs.cpu().numpy()
    keep = res.mask_used.keep_numpy()[0, 0]
    assert keep.shape == (591, 1182)
    assert np.array_equal(keep, oracle.hybrid_keep(probs, 0.03, 0.16))
    assert 0.9 < res.mask_used.sparsity() < 0.99


@pytest.mark.parametrize("h", [0, 1])
def test_forward_and_dq_on_row_slices(run, h):
    res, (dq, _, _), host, _ = run
    q, k, v, do = (x[h] for x in host)
    keep = res.mask_used.keep_numpy()[0, h]
    for blocks in (slice(0, 6), slice(586, 591)):  # includes the 80-row tail block
        rows = slice(blocks.start * 128, min(blocks.stop * 128, N))
        out, lse, _ = oracle.sparse_forward(q[rows], k, v, keep[blocks], 128, 64)
        assert_close(f"h{h} out{blocks}", res.out[0, h, rows], out, "out")
        assert_close(f"h{h} lse{blocks}", res.lse[0, h, rows], lse, "lse")
        dq_ref, _, _, _, _ = oracle.attention_backward(q[rows], k, v, keep[blocks], 128, 64, do[rows])
        assert_close(f"h{h} dq{blocks}", dq[h, rows], dq_ref, "dq")


def test_dkdv_for_key_blocks(run):
    res, (_, dk, dv), host, _ = run
    h = 0
    q, k, v, do = (x[h] for x in host)
    keep = res.mask_used.keep_numpy()[0, h]
    scale = 1.0 / math.sqrt(D)
    for j in (int(np.argmax(keep.sum(axis=0))), 1181):  # the most-kept key block and the 16-row tail
        kv = slice(j * 64, min((j + 1) * 64, N))
        dk_ref = np.zeros((kv.stop - kv.start, D))
        dv_ref = np.zeros_like(dk_ref)
        for i in np.flatnonzero(keep[:, j]):
            rows = slice(i * 128, min((i + 1) * 128, N))
            # row statistics (O, LSE) from the float64 oracle forward of query block i, so the
            # check is independent of the GPU forward
            out_i, lse_i, _ = oracle.sparse_forward(q[rows], k, v, keep[i:i + 1], 128, 64)
            p = np.exp((q[rows] @ k[kv].T) * scale - lse_i[:, None])
            delta = (do[rows] * out_i).sum(axis=1)
            dv_ref += p.T @ do[rows]
            ds = p * (do[rows] @ v[kv].T - delta[:, None])
            dk_ref += (ds.T @ q[rows]) * scale
        if keep[:, j].any():
            assert_close(f"dk{j}", dk[h, kv], dk_ref, "dk")
            assert_close(f"dv{j}", dv[h, kv], dv_ref, "dv")
        else:
            assert not dk[h, kv].any() and not dv[h, kv].any()

"""Tiny and ragged sequence lengths: the TMA out-of-bounds / ragged-tail path when a whole
problem is smaller than one key block (64) or one query block (128), forward and backward.

The reference has no block-size floor (attention.py:87-102); the kernels tile N into 128-row
query blocks and 64-row key blocks, so N < 64 means a single partial key block whose rows past
N are zero-filled by TMA on load and clipped on store, and masked to -inf in the softmax.
Checked against the float64 oracle on the same bf16 inputs, through autograd (torch in)."""

import numpy as np
import pytest
import torch

import oracle
import paper_2602_13515_b200 as spa
from gen import random_keep, wan_like
from parity import assert_close

pytestmark = pytest.mark.gpu

SIZES = (1, 2, 17, 63, 64, 65, 127, 128, 129, 191)


def _run(n, d, keep, seed):
    q, k, v, do = wan_like(seed, n, d, 128, 64, 0.0, heads=1)
    t = lambda x: torch.tensor(x[0], device="cuda").to(torch.bfloat16)
    qd, kd, vd = (t(x).requires_grad_(True) for x in (q, k, v))
    bm = spa.BlockMask(torch.tensor(keep, device="cuda"), 128, 64, n)
    res = spa.sparse_attention_with_mask(qd, kd, vd, bm)
    res.out.backward(t(do))
    dq, dk, dv, out, lse = oracle.attention_backward(q[0], k[0], v[0], keep, 128, 64, do[0])
    tag = f"n{n}.d{d}"
    assert_close(f"{tag}.out", res.out, out, "out")
    assert_close(f"{tag}.lse", res.lse, lse, "lse")
    if n == 1:
        # one key: P = 1 and dS = dP - δ = 0 exactly; the GPU's dP (tensor core) and δ (fp32 dot
        # product) round differently, so dq/dk are zero up to fp32 rounding of |dO|·|v|
        scale = float(np.abs(do).max() * np.abs(v).max() * d)
        assert float(qd.grad.abs().max()) <= 1e-5 * scale and float(kd.grad.abs().max()) <= 1e-5 * scale
    else:
        assert_close(f"{tag}.dq", qd.grad, dq, "dq")
        assert_close(f"{tag}.dk", kd.grad, dk, "dk")
    assert_close(f"{tag}.dv", vd.grad, dv, "dv")
    return res, (qd.grad, kd.grad, vd.grad)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("d", (64, 128))
def test_tiny_full_mask(n, d):
    t_m, t_n = -(-n // 128), -(-n // 64)
    _run(n, d, np.ones((t_m, t_n), bool), seed=n * 3 + d)


@pytest.mark.parametrize("n", (129, 191, 300))
@pytest.mark.parametrize("d", (64, 128))
def test_tiny_random_mask(n, d):
    t_m, t_n = -(-n // 128), -(-n // 64)
    keep = random_keep(n + d, t_m, t_n, 0.5)
    _, (dq, dk, dv) = _run(n, d, keep, seed=n * 5 + d)
    # key blocks no query block keeps get exact zeros (attention.py:152-157)
    for j in np.flatnonzero(~keep.any(axis=0)):
        assert not dk[64 * j:64 * (j + 1)].any() and not dv[64 * j:64 * (j + 1)].any()


def test_single_token_is_exact():  # test_attention.py:29-31 at the kernel's shapes, torch path
    for d in (64, 128):
        x = torch.randn(3, 1, d, device="cuda").to(torch.bfloat16)
        res = spa.dense_attention(x[0], x[1], x[2])
        assert torch.equal(res.out, x[2])

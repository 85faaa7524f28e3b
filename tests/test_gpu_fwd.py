"""GPU forward parity (K4) against the reference's goldens and the float64 oracle, plus the
reference's attention known-answer tests (test_attention.py) run through the GPU."""

import math

import numpy as np
import pytest
import torch
from conftest import unpack_keep
from gen import random_keep, wan_like
from parity import assert_close

import oracle
import paper_2602_13515_b200 as spa
from paper_2602_13515_b200 import _lib
from paper_2602_13515_b200 import masker as mk

pytestmark = pytest.mark.gpu
BQ, BKV = 128, 64


def bf(x):
    return torch.tensor(np.asarray(x), device="cuda").to(torch.bfloat16)


def case_inputs(case):
    return wan_like(case["seed"], case["n"], case["d"], case["b_q"], case["b_kv"], case["s"], heads=case["heads"])


@pytest.mark.parametrize("idx", range(5))
def test_forward_matches_reference_goldens(manifest, golden_attention, idx):
    case = manifest["attention"][idx]
    tag, n, t_n = case["tag"], case["n"], case["t_n"]
    q, k, v, _ = case_inputs(case)
    keep = unpack_keep(golden_attention[f"{tag}_keep"], t_n)
    for h in range(case["heads"]):
        bm = mk.BlockMask(keep[h], BQ, BKV, n)
        res = spa.sparse_attention_with_mask(bf(q[h]), bf(k[h]), bf(v[h]), bm)
        assert_close(f"{tag}[{h}].out", res.out, golden_attention[f"{tag}_out"][h], "out")
        assert_close(f"{tag}[{h}].lse", res.lse, golden_attention[f"{tag}_lse"][h], "lse")


def test_cfg1_end_to_end_masker_plus_forward(manifest, golden_attention):
    """configs[0]: B=1 H=2 N=1024 d=64, hybrid k=0.1/p=0.9, batched [B,H,N,d] call."""
    case = next(c for c in manifest["attention"] if c["tag"] == "cfg1")
    q, k, v, _ = case_inputs(case)
    q4, k4, v4 = (bf(x).view(1, 2, 1024, 64) for x in (q, k, v))
    res = spa.sparse_attention(q4, k4, v4, spa.SparsityConfig(0.1, 0.9, BQ, BKV))
    want_keep = unpack_keep(golden_attention["cfg1_keep"], case["t_n"])
    assert np.array_equal(res.mask_used.keep_numpy()[0], want_keep)
    assert_close("cfg1.out", res.out[0], golden_attention["cfg1_out"], "out")
    assert_close("cfg1.lse", res.lse[0], golden_attention["cfg1_lse"], "lse")


@pytest.mark.parametrize("n,d,density,heads", [(1000, 128, 0.3, 2), (4096, 128, 0.05, 1), (777, 64, 0.5, 3),
                                               (64, 64, 1.0, 1), (128, 128, 1.0, 1), (8192, 64, 0.08, 2)])
def test_forward_random_masks_vs_oracle(n, d, density, heads):
    q, k, v, _ = wan_like(n + d, n, d, BQ, BKV, 0.5, heads=heads)
    t_m, t_n = -(-n // BQ), -(-n // BKV)
    keep = np.stack([random_keep(n * 7 + h, t_m, t_n, density) for h in range(heads)])
    bm = mk.BlockMask(keep.reshape(1, heads, t_m, t_n), BQ, BKV, n)
    res = spa.sparse_attention_with_mask(bf(q).view(1, heads, n, d), bf(k).view(1, heads, n, d),
                                         bf(v).view(1, heads, n, d), bm)
    for h in range(heads):
        out, lse, _ = oracle.sparse_forward(q[h], k[h], v[h], keep[h], BQ, BKV)
        assert_close(f"h{h}.out", res.out[0, h], out, "out")
        assert_close(f"h{h}.lse", res.lse[0, h], lse, "lse")


def test_forward_strided_bnhd_layout():
    """Wan/flash layout [B, N, H, d] passed as a permuted view (strided TMA descriptors)."""
    B, N, H, d = 2, 640, 3, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    base = [torch.randn(B, N, H, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3)]
    q, k, v = (t.permute(0, 2, 1, 3) for t in base)  # [B,H,N,d] views, token stride H*d
    assert not q.is_contiguous()
    cfg = spa.SparsityConfig(0.2, 0.5, BQ, BKV)
    res = spa.sparse_attention(q, k, v, cfg)
    res_c = spa.sparse_attention(q.contiguous(), k.contiguous(), v.contiguous(), cfg)
    assert torch.equal(res.mask_used.keep, res_c.mask_used.keep)
    assert torch.equal(res.out, res_c.out)
    keep = res.mask_used.keep_numpy()
    for b in range(B):
        for h in range(H):
            out, _, _ = oracle.sparse_forward(q[b, h].double().cpu().numpy(), k[b, h].double().cpu().numpy(),
                                              v[b, h].double().cpu().numpy(), keep[b, h], BQ, BKV)
            assert_close(f"b{b}h{h}", res.out[b, h], out, "out")


def test_full_mask_equals_dense_and_sdpa():
    """test_attention.py:126-129 — all-ones mask == dense; cross-checked with torch SDPA."""
    n, d = 512, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    a = spa.sparse_attention_with_mask(q, k, v, spa.full_mask(n))
    b = spa.dense_attention(q, k, v)
    assert torch.equal(a.out, b.out)
    ref = torch.nn.functional.scaled_dot_product_attention(q.float()[None, None], k.float()[None, None],
                                                           v.float()[None, None])[0, 0]
    assert_close("full", a.out, ref, "out")
    s = (q.double() @ k.double().t()) / math.sqrt(d)
    assert_close("lse", a.lse, torch.logsumexp(s, dim=1), "lse")


def test_single_block_rows_and_diagonal():
    """test_attention.py:309-343 at the kernel grid: each query block keeps exactly one
    key block; its output is plain softmax attention over that block."""
    n, d = 512, 64
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
    keep = np.zeros((4, 8), dtype=bool)
    for i, j in enumerate((0, 7, 3, 4)):
        keep[i, j] = True
    res = spa.sparse_attention_with_mask(q, k, v, mk.BlockMask(keep, BQ, BKV, n))
    for i, j in enumerate((0, 7, 3, 4)):
        qi, kj, vj = q[i * 128:(i + 1) * 128].double(), k[j * 64:(j + 1) * 64].double(), v[j * 64:(j + 1) * 64].double()
        want = torch.softmax(qi @ kj.t() / math.sqrt(d), dim=1) @ vj
        assert_close(f"row{i}", res.out[i * 128:(i + 1) * 128], want, "out")


def test_visit_order_invariance():
    """test_attention.py:356-367 — a permuted per-row visit order changes nothing beyond
    float rounding (the kernel's online softmax is order-invariant)."""
    n, d = 1024, 128
    q, k, v, _ = wan_like(9, n, d, BQ, BKV, 0.5)
    keep = random_keep(9, 8, 16, 0.7)
    bm = mk.BlockMask(keep, BQ, BKV, n)
    base = spa.sparse_attention_with_mask(bf(q[0]), bf(k[0]), bf(v[0]), bm)
    rng = np.random.Generator(np.random.PCG64(1234))
    for _ in range(3):
        perm = spa.sparse_attention_with_mask(bf(q[0]), bf(k[0]), bf(v[0]), bm,
                                              _block_order=lambda i, kept: rng.permutation(kept))
        assert_close("perm", perm.out, base.out.float(), "out")
        assert_close("perm.lse", perm.lse, base.lse, "lse")


def test_renormalisation_and_convexity():
    """test_attention.py:370-392 — Σ_kept exp(s - lse) == 1 per row; outputs are convex
    combinations of the selected v rows."""
    n, d = 384, 64
    q, k, v, _ = wan_like(10, n, d, BQ, BKV, 0.3)
    keep = random_keep(10, 3, 6, 0.5)
    bm = mk.BlockMask(keep, BQ, BKV, n)
    res = spa.sparse_attention_with_mask(bf(q[0]), bf(k[0]), bf(v[0]), bm)
    em = oracle.expand_keep(keep, BQ, BKV, n).astype(bool)
    s = q[0] @ k[0].T / math.sqrt(d)
    lse = res.lse.double().cpu().numpy()
    w = np.exp(s - lse[:, None]) * em
    assert np.abs(w.sum(axis=1) - 1.0).max() <= 5e-3
    out = res.out.double().cpu().numpy()
    for a in range(n):
        sel = v[0][em[a]]
        assert np.all(out[a] >= sel.min(axis=0) - 1e-2) and np.all(out[a] <= sel.max(axis=0) + 1e-2)


def test_counter_counts_exactly_kept_blocks():
    """test_attention.py:395-409 — the device-side counter equals kept blocks."""
    n, d = 2000, 128
    q, k, v, _ = wan_like(11, n, d, BQ, BKV, 0.9)
    keep = random_keep(11, 16, 32, 0.4)
    bm = mk.BlockMask(keep, BQ, BKV, n)
    ctr = spa.BlockCounter()
    spa.sparse_attention_with_mask(bf(q[0]), bf(k[0]), bf(v[0]), bm, counter=ctr)
    assert ctr.count == bm.kept_blocks() == int(keep.sum())
    ctr2 = spa.BlockCounter()
    res = spa.sparse_attention(bf(q[0]), bf(k[0]), bf(v[0]), spa.SparsityConfig(0.1, 0.3, BQ, BKV), counter=ctr2)
    assert ctr2.count == res.mask_used.kept_blocks()


def test_errors():
    q = torch.zeros(8, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="tokens"):  # test_attention.py:412-415
        spa.sparse_attention_with_mask(q, q, q, spa.full_mask(16))
    with pytest.raises(ValueError):
        spa.sparse_attention_with_mask(q, q, torch.zeros(8, 32, device="cuda"), spa.full_mask(8))
    bad = q.clone()
    bad[3, 3] = float("inf")
    with pytest.raises(FloatingPointError):
        spa.sparse_attention_with_mask(bad, q, q, spa.full_mask(8), check_finite="sync")
    for args in ((q, bad, q), (q, q, bad), (bad, q, q)):
        with pytest.raises(FloatingPointError):
            spa.sparse_attention(*args, spa.SparsityConfig(0.5, 0.5, BQ, BKV), check_finite="sync")
    with pytest.raises(spa.ShapeError):
        spa.sparse_attention_with_mask(q[None], q[None], q[None], spa.full_mask(8))
    with pytest.raises(ValueError, match="head dim"):
        z = torch.zeros(8, 48, device="cuda", dtype=torch.bfloat16)
        spa.sparse_attention_with_mask(z, z, z, spa.full_mask(8))


def test_non_finite_verdict_is_deferred_for_torch_callers():
    """No host sync on the hot path: a torch caller's non-finite input raises at the latest at
    the next operator call, in its own backward once the scan has landed, or at
    check_pending() (numerics.FiniteGuard)."""
    q = torch.randn(300, 64, device="cuda").to(torch.bfloat16)
    bad = q.clone()
    bad[7, 1] = float("nan")
    cfg = spa.SparsityConfig(0.5, 0.5, BQ, BKV)
    spa.sparse_attention(q, q, bad, cfg)  # returns without a sync
    with pytest.raises(FloatingPointError):
        spa.check_pending()
    spa.check_pending()  # consumed
    spa.sparse_attention_with_mask(bad, q, q, spa.full_mask(300))
    torch.cuda.synchronize()
    with pytest.raises(FloatingPointError):  # the next call enforces the landed verdict
        spa.sparse_attention(q, q, q, cfg)
    qs = bad.clone().requires_grad_(True)
    res = spa.sparse_attention(qs, q, q, cfg)
    torch.cuda.synchronize()
    with pytest.raises(FloatingPointError):  # ... and so does the call's own backward
        res.out.sum().backward()
    spa.check_pending()
    g = spa.attention_backward(q, q, q, spa.full_mask(300), bad)  # d_out is scanned too
    with pytest.raises(FloatingPointError):
        spa.check_pending()
    assert g.dq.shape == q.shape
    res = spa.sparse_attention(q, q, bad, cfg, check_finite=False)  # opt-out: no verdict at all
    spa.check_pending()


def test_numpy_in_numpy_out():
    q, k, v, _ = wan_like(12, 300, 64, BQ, BKV, 0.0)
    res = spa.sparse_attention_with_mask(q[0], k[0], v[0], spa.full_mask(300))
    assert isinstance(res.out, np.ndarray) and res.out.dtype == np.float64 and res.out.shape == (300, 64)
    out, _ = oracle.dense_attention(q[0], k[0], v[0])
    assert_close("np", res.out, out, "out")


def test_probe_tmem_a_operand():
    """The TS form of tcgen05.mma (A = P packed in TMEM) used by the forward's PV step."""
    for n_, k_ in ((64, 64), (128, 64), (128, 128)):
        a = torch.randn(128, k_, device="cuda").to(torch.bfloat16)
        b = torch.randn(k_, n_, device="cuda").to(torch.bfloat16)  # stored [k, n] -> MN-major B
        d = torch.empty(128, n_, device="cuda")
        rc = _lib.load_diag().spa2_probe_gemm(_lib.ptr(a), _lib.ptr(b), _lib.ptr(d), 128, n_, k_, 0, 1, 2,
                                         torch.cuda.current_stream().cuda_stream)
        _lib.check_diag(rc, "probe")
        torch.cuda.synchronize()
        want = a.float() @ b.float()
        assert (d - want).abs().max().item() <= 1e-3 * want.abs().max().item()

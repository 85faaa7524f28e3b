"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic: head ranges,
head all-gather, and the Ulysses sequence<->head all-to-all (round trip, exact placement,
autograd through the exchange)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_13515_b200 import dist as pdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, fn):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
    finally:
        dist.destroy_process_group()


def _spawn(fn, world=2):
    mp.spawn(_run, args=(world, _free_port(), fn), nprocs=world, join=True)


def test_head_range_partitions():
    for H in (1, 5, 12, 40):
        for world in (1, 2, 3, 4, 8):
            ranges = [pdist.head_range(H, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [h1 - h0 for h0, h1 in ranges]
            assert max(sizes) - min(sizes) <= 1
    assert pdist.head_range(40, 3, 8) == (15, 20)


def _check_gather(rank, world):
    H = 5
    full = torch.arange(2 * H * 3 * 4, dtype=torch.float32).reshape(2, H, 3, 4)
    local = pdist.shard_heads(full)
    h0, h1 = pdist.head_range(H, rank, world)
    assert torch.equal(local, full[:, h0:h1])
    assert torch.equal(pdist.gather_heads(local * 2, H), full * 2)


def test_gather_heads_uneven():
    _spawn(_check_gather)


def _check_ulysses(rank, world):
    B, N, H, d = 2, 8, 4, 3
    g = torch.Generator().manual_seed(0)
    full = torch.randn(B, N, H, d, generator=g)  # the unsharded activations, same on every rank
    n_loc = N // world
    x_local = full[:, rank * n_loc:(rank + 1) * n_loc].clone()
    y = pdist.seq_to_head(x_local)
    hp = H // world
    assert torch.equal(y, full[:, :, rank * hp:(rank + 1) * hp])  # full sequence, my heads
    back = pdist.head_to_seq(y)
    assert torch.equal(back, x_local)
    # autograd through the exchange: d/dx sum(w * seq_to_head(x)) = head_to_seq(w) on my shard
    xr = x_local.clone().requires_grad_(True)
    w = torch.randn(B, N, hp, d, generator=torch.Generator().manual_seed(1 + rank))
    (pdist.seq_to_head(xr) * w).sum().backward()
    assert torch.allclose(xr.grad, pdist.head_to_seq(w))
    with pytest.raises(ValueError):  # heads must split evenly across ranks
        pdist.seq_to_head(torch.zeros(1, 2, 3, 4))


def test_ulysses_all_to_all_round_trip_and_grad():
    _spawn(_check_ulysses)




class RefKernels:
    """float64 dense-softmax restatement of the per-group compute (no masker): stands in for
    the B200 kernels so the overlapped Ulysses exchange logic runs on CPU with gloo."""

    def forward(self, q, k, v, o_out):
        s = (q.double() @ k.double().transpose(-1, -2)) / q.shape[-1] ** 0.5
        p = torch.softmax(s, dim=-1)
        o_out.copy_((p @ v.double()).to(o_out.dtype))
        return p

    def backward(self, p, q, k, v, o, do, dq_out, dk_out, dv_out):
        with torch.enable_grad():  # autograd backward runs with grad mode off
            qd, kd, vd = (t.double().detach().requires_grad_(True) for t in (q, k, v))
            s = (qd @ kd.transpose(-1, -2)) / q.shape[-1] ** 0.5
            out = torch.softmax(s, dim=-1) @ vd
            out.backward(do.double())
        for g, dst in ((qd.grad, dq_out), (kd.grad, dk_out), (vd.grad, dv_out)):
            dst.copy_(g.to(dst.dtype))


def _dense(q, k, v):  # [B, N, H, d] -> [B, N, H, d]
    qh, kh, vh = (t.permute(0, 2, 1, 3) for t in (q, k, v))
    p = torch.softmax((qh @ kh.transpose(-1, -2)) / q.shape[-1] ** 0.5, dim=-1)
    return (p @ vh).permute(0, 2, 1, 3)


def _check_ulysses_overlapped(rank, world):
    B, N, H, d = 2, 12, 6, 8  # 3 heads per rank in 2 groups (uneven group sizes)
    g = torch.Generator().manual_seed(3)
    full = [torch.randn(B, N, H, d, generator=g, dtype=torch.float64) for _ in range(4)]
    n_loc = N // world
    sl = slice(rank * n_loc, (rank + 1) * n_loc)
    q, k, v = (t[:, sl].clone().requires_grad_(True) for t in full[:3])
    uly = pdist.UlyssesAttention(cfg=None, groups=2, kernels=RefKernels())
    out = uly(q, k, v)
    ref = [t.clone().requires_grad_(True) for t in full[:3]]
    want = _dense(*ref)
    assert torch.allclose(out, want[:, sl], atol=1e-12)
    out.backward(full[3][:, sl])
    want.backward(full[3])
    for got, r in zip((q, k, v), ref):
        assert torch.allclose(got.grad, r.grad[:, sl], atol=1e-12)


def test_ulysses_overlapped_operator_matches_single_process():
    """UlyssesAttention: per-group exchange (send packing, strided head views of the receive
    buffers, outputs written into the return exchange's send buffers, unpacking) and its
    backward, against unsharded attention — exact up to float64 rounding."""
    _spawn(_check_ulysses_overlapped)

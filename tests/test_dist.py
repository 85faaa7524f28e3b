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



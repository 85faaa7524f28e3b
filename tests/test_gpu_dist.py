"""The multi-GPU operator paths executed end to end: two processes (ranks) share the one lease
GPU and talk over gloo (CUDA tensors staged through host memory — NCCL needs one GPU per
rank).  A configs[3]-like slice (N = 4096, H = 8, d = 128, k = 0.03, p = 0.16):

* head sharding (dist.sparse_attention_head_sharded + gather_heads) and
* the overlapped Ulysses operator (dist.UlyssesAttention: per-head-group all-to-all, strided
  head views of the receive buffers, kernels writing into the return exchange's buffers),

forward AND backward, must be BIT-EQUAL to the single-process operator on the same inputs:
every output tile is computed by one CTA with a fixed accumulation order, whichever rank,
head group or memory layout it comes from."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N, H, D = 4096, 8, 128


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    q, k, v = wan_like_qkv(1, H, N, D, 0.8, seed=31)
    do = torch.randn(q.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(32)).to(q.dtype)
    return q, k, v, do


def _worker(rank, world, port, groups):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_13515_b200 as spa
        from paper_2602_13515_b200 import dist as sdist

        cfg = spa.SparsityConfig(0.03, 0.16, 128, 64)
        q, k, v, do = _inputs()
        # single-process operator on the whole problem
        qs, ks, vs = (t.clone().requires_grad_(True) for t in (q, k, v))
        ref = spa.sparse_attention(qs, ks, vs, cfg)
        ref.out.backward(do)
        assert 0.85 < ref.mask_used.sparsity() < 0.99

        # (a) head sharding + all-gather
        h0, h1 = sdist.head_range(H, rank, world)
        qr, kr, vr = (t.clone().requires_grad_(True) for t in (q, k, v))  # replicated inputs
        o_gathered, res = sdist.sparse_attention_head_sharded(qr, kr, vr, cfg, gather=True)
        assert torch.equal(o_gathered, ref.out.detach()), "head-sharded O"
        res.out.backward(do[:, h0:h1])
        ql, kl, vl = (t.grad[:, h0:h1] for t in (qr, kr, vr))
        assert not qr.grad[:, :h0].any() and not qr.grad[:, h1:].any()  # other ranks' heads
        for name, g, r in (("dq", ql, qs.grad), ("dk", kl, ks.grad), ("dv", vl, vs.grad)):
            assert torch.equal(sdist.gather_heads(g.contiguous(), H), r), f"head-sharded {name}"

        # (b) Ulysses: sequence-sharded [B, N/P, H, d] activations
        n_loc = N // world
        sl = slice(rank * n_loc, (rank + 1) * n_loc)
        seq = lambda t: t.permute(0, 2, 1, 3)[:, sl].contiguous()  # noqa: E731
        qu, ku, vu = (seq(t).requires_grad_(True) for t in (q, k, v))
        uly = sdist.UlyssesAttention(cfg, groups=groups)
        out = uly(qu, ku, vu)
        assert torch.equal(out, seq(ref.out.detach())), "Ulysses O"
        out.backward(seq(do))
        for name, g, r in (("dq", qu.grad, qs.grad), ("dk", ku.grad, ks.grad), ("dv", vu.grad, vs.grad)):
            assert torch.equal(g, seq(r)), f"Ulysses {name}"
        spa.check_pending()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("groups", [1, 3])
def test_head_sharded_and_ulysses_bit_equal_to_single_process(groups):
    mp.spawn(_worker, args=(2, _free_port(), groups), nprocs=2, join=True)

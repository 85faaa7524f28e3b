"""Multi-GPU plumbing for the sparse-attention operator.

Every kernel's work item lives inside one (batch, head), so the operator shards by head
with no data-path collective:

* ``head_range`` / ``shard_heads`` / ``gather_heads`` — contiguous head ranges per rank
  (balanced when H % world != 0), optional all-gather of outputs.
* ``seq_to_head`` / ``head_to_seq`` — the Ulysses all-to-all for sequence-parallel callers
  (a DiT whose activations are sharded along the sequence): ``[B, N/P, H, d]`` ↔
  ``[B, N, H/P, d]``, differentiable (``torch.distributed.nn.functional.all_to_all_single``).
* ``ulysses_sparse_attention`` — seq-sharded q/k/v in, seq-sharded output out, with the
  local heads' sparse attention (masker + forward + autograd backward) in between.

One process per GPU; ``torch.distributed`` with NCCL on the box (gloo works for the host
logic and is what the CPU tests use).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _world(group) -> tuple[int, int]:
    return dist.get_rank(group), dist.get_world_size(group)


def head_range(H: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [h0, h1) of rank `rank`; the first H % world ranks get one extra head."""
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def shard_heads(x: torch.Tensor, group=None) -> torch.Tensor:
    """This rank's head slice of a replicated [B, H, N, d] tensor (a view, no copy)."""
    rank, world = _world(group)
    h0, h1 = head_range(x.shape[1], rank, world)
    return x[:, h0:h1]


def gather_heads(x_local: torch.Tensor, H: int, group=None) -> torch.Tensor:
    """All-gather head slices [B, h_r, ...] from every rank into [B, H, ...] (uneven OK)."""
    rank, world = _world(group)
    sizes = [head_range(H, r, world) for r in range(world)]
    hmax = max(h1 - h0 for h0, h1 in sizes)
    pad = torch.zeros((x_local.shape[0], hmax) + tuple(x_local.shape[2:]), dtype=x_local.dtype,
                      device=x_local.device)
    pad[:, : x_local.shape[1]] = x_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    return torch.cat([b[:, : h1 - h0] for b, (h0, h1) in zip(bufs, sizes)], dim=1)


def _a2a(x: torch.Tensor, group) -> torch.Tensor:
    if x.requires_grad:
        from torch.distributed.nn.functional import all_to_all_single

        out = torch.empty_like(x)
        return all_to_all_single(out, x, group=group)
    out = torch.empty_like(x)
    dist.all_to_all_single(out, x, group=group)
    return out


def seq_to_head(x: torch.Tensor, group=None) -> torch.Tensor:
    """Ulysses forward exchange: sequence-sharded [B, N/P, H, d] -> head-sharded
    [B, N, H/P, d] (rank r receives heads [r·H/P, (r+1)·H/P) of every sequence chunk)."""
    _, world = _world(group)
    B, n_loc, H, d = x.shape
    if H % world:
        raise ValueError(f"Ulysses needs H % world == 0 (H={H}, world={world})")
    hp = H // world
    send = x.reshape(B, n_loc, world, hp, d).permute(2, 0, 1, 3, 4).contiguous()  # [P, B, N/P, H/P, d]
    recv = _a2a(send, group)  # [P (source = sequence chunk), B, N/P, H/P, d]
    return recv.permute(1, 0, 2, 3, 4).reshape(B, world * n_loc, hp, d)


def head_to_seq(y: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse exchange: head-sharded [B, N, H/P, d] -> sequence-sharded [B, N/P, H, d]."""
    _, world = _world(group)
    B, N, hp, d = y.shape
    if N % world:
        raise ValueError(f"Ulysses needs N % world == 0 (N={N}, world={world})")
    n_loc = N // world
    send = y.reshape(B, world, n_loc, hp, d).permute(1, 0, 2, 3, 4).contiguous()  # [P (dest chunk), B, N/P, H/P, d]
    recv = _a2a(send, group)  # [P (source = head group), B, N/P, H/P, d]
    return recv.permute(1, 2, 0, 3, 4).reshape(B, n_loc, world * hp, d)


def sparse_attention_head_sharded(q, k, v, cfg, group=None, gather: bool = False, **kw):
    """Run this rank's heads of replicated [B, H, N, d] inputs; optionally all-gather O."""
    from .attention import sparse_attention

    res = sparse_attention(shard_heads(q, group), shard_heads(k, group), shard_heads(v, group), cfg, **kw)
    if gather:
        return gather_heads(res.out, q.shape[1], group), res
    return res.out, res


def ulysses_sparse_attention(q_l, k_l, v_l, cfg, group=None, **kw):
    """Sequence-sharded [B, N/P, H, d] q/k/v -> sequence-sharded output, differentiable.
    The block mask is built per local head over the full sequence, exactly as one GPU
    would (the masker needs the whole sequence of a head)."""
    from .attention import sparse_attention

    q, k, v = (seq_to_head(t, group).permute(0, 2, 1, 3) for t in (q_l, k_l, v_l))  # [B, H/P, N, d] views
    res = sparse_attention(q, k, v, cfg, **kw)
    out = head_to_seq(res.out.permute(0, 2, 1, 3), group)
    return out, res

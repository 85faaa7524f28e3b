"""Multi-GPU plumbing for the sparse-attention operator.

Every kernel's work item lives inside one (batch, head), so the operator shards by head
with no data-path collective:

* ``head_range`` / ``shard_heads`` / ``gather_heads`` — contiguous head ranges per rank
  (balanced when H % world != 0), all-gather of outputs / gradients.
* ``seq_to_head`` / ``head_to_seq`` — the plain Ulysses all-to-all for sequence-parallel
  callers: ``[B, N/P, H, d]`` ↔ ``[B, N, H/P, d]``.
* ``UlyssesAttention`` — the fused, overlapped sequence-parallel operator: sequence-sharded
  q/k/v in, sequence-sharded output out, differentiable.  The local heads are processed
  in head groups; the all-to-all of group g+1 runs on a communication stream while the
  masker + forward (or the backward kernels) of group g run on the compute stream, and
  the received buffers are handed to the TMA-fed kernels AS STRIDED VIEWS (no unpacking
  copy): the receive layout [P (source chunk)][n_loc][h_g][d] of one batch row is exactly a
  [h_g, N, d] tensor with strides (d, h_g·d).  Likewise the kernels write O (forward) and
  dQ/dK/dV (backward) straight into the return exchange's send buffers.  Only the pack of
  the caller's [B, N/P, H, d] activations into per-destination chunks (and the matching
  unpack of the returned chunks) remain as copies, because a collective needs contiguous
  per-peer buffers.

One process per GPU; NCCL on the box.  With the gloo backend (CPU tests, or several
processes sharing one GPU in the GPU tests) CUDA tensors are staged through host memory.
"""

from __future__ import annotations

import math

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


def _staged(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _all_gather(bufs: list[torch.Tensor], x: torch.Tensor, group) -> None:
    if _staged(group) and x.is_cuda:
        host = [torch.empty(b.shape, dtype=b.dtype) for b in bufs]
        dist.all_gather(host, x.cpu(), group=group)
        for b, h in zip(bufs, host):
            b.copy_(h)
        return
    dist.all_gather(bufs, x, group=group)


def _all_to_all(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """all_to_all_single over contiguous buffers split along dim 0 (staged for gloo + CUDA)."""
    if _staged(group) and inp.is_cuda:
        h_out = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(h_out, inp.cpu(), group=group)
        out.copy_(h_out)
        return
    dist.all_to_all_single(out, inp, group=group)


def gather_heads(x_local: torch.Tensor, H: int, group=None) -> torch.Tensor:
    """All-gather head slices [B, h_r, ...] from every rank into [B, H, ...] (uneven OK)."""
    rank, world = _world(group)
    sizes = [head_range(H, r, world) for r in range(world)]
    hmax = max(h1 - h0 for h0, h1 in sizes)
    if all(h1 - h0 == hmax for h0, h1 in sizes) and x_local.is_contiguous():
        pad = x_local
    else:
        pad = torch.zeros((x_local.shape[0], hmax) + tuple(x_local.shape[2:]), dtype=x_local.dtype,
                          device=x_local.device)
        pad[:, : x_local.shape[1]] = x_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    _all_gather(bufs, pad.contiguous(), group)
    return torch.cat([b[:, : h1 - h0] for b, (h0, h1) in zip(bufs, sizes)], dim=1)


def _seq_to_head(x: torch.Tensor, group) -> torch.Tensor:
    _, world = _world(group)
    B, n_loc, H, d = x.shape
    if H % world:
        raise ValueError(f"Ulysses needs H % world == 0 (H={H}, world={world})")
    hp = H // world
    send = x.reshape(B, n_loc, world, hp, d).permute(2, 0, 1, 3, 4).contiguous()  # [P, B, N/P, H/P, d]
    recv = torch.empty_like(send)  # [P (source = sequence chunk), B, N/P, H/P, d]
    _all_to_all(recv, send, group)
    return recv.permute(1, 0, 2, 3, 4).reshape(B, world * n_loc, hp, d)


def _head_to_seq(y: torch.Tensor, group) -> torch.Tensor:
    _, world = _world(group)
    B, N, hp, d = y.shape
    if N % world:
        raise ValueError(f"Ulysses needs N % world == 0 (N={N}, world={world})")
    n_loc = N // world
    send = y.reshape(B, world, n_loc, hp, d).permute(1, 0, 2, 3, 4).contiguous()  # [P (dest chunk), B, N/P, H/P, d]
    recv = torch.empty_like(send)  # [P (source = head group), B, N/P, H/P, d]
    _all_to_all(recv, send, group)
    return recv.permute(1, 2, 0, 3, 4).reshape(B, n_loc, world * hp, d)


class _Exchange(torch.autograd.Function):
    """The two exchanges are inverse permutations, so each one's adjoint is the other."""

    @staticmethod
    def forward(ctx, x, to_heads, group):
        ctx.to_heads, ctx.group = to_heads, group
        return _seq_to_head(x, group) if to_heads else _head_to_seq(x, group)

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        return (_head_to_seq(g, ctx.group) if ctx.to_heads else _seq_to_head(g, ctx.group)), None, None


def seq_to_head(x: torch.Tensor, group=None) -> torch.Tensor:
    """Ulysses forward exchange: sequence-sharded [B, N/P, H, d] -> head-sharded
    [B, N, H/P, d] (rank r receives heads [r·H/P, (r+1)·H/P) of every sequence chunk).
    Differentiable (the adjoint is ``head_to_seq``)."""
    return _Exchange.apply(x, True, group)


def head_to_seq(y: torch.Tensor, group=None) -> torch.Tensor:
    """Inverse exchange: head-sharded [B, N, H/P, d] -> sequence-sharded [B, N/P, H, d]."""
    return _Exchange.apply(y, False, group)


def sparse_attention_head_sharded(q, k, v, cfg, group=None, gather: bool = False, **kw):
    """Run this rank's heads of replicated [B, H, N, d] inputs; optionally all-gather O."""
    from .attention import sparse_attention

    res = sparse_attention(shard_heads(q, group), shard_heads(k, group), shard_heads(v, group), cfg, **kw)
    if gather:
        return gather_heads(res.out, q.shape[1], group), res
    return res.out, res


# ---------------------------------------------------------------------------------------
# Fused, overlapped Ulysses (§8f row 1)
# ---------------------------------------------------------------------------------------

class GroupKernels:
    """The per-head-group compute of ``UlyssesAttention`` on [1, h, N, d] strided views:
    the B200 kernels (finiteness scan + masker + forward; δ/dQ/dK/dV), writing their outputs
    into caller-provided views.  Tests substitute a float64 torch restatement to check the
    exchange logic on CPU."""

    def __init__(self, cfg):
        self.cfg = cfg

    def forward(self, q, k, v, o_out):
        from . import attention as at
        from .masker import BlockMask
        from .numerics import finite_guard

        flag = finite_guard.new_flag(q.device)
        at._scan_finite(flag, v)
        keep = at._hybrid_mask_device(q, k, self.cfg, flag)
        finite_guard.submit(flag, "q, k or v (Ulysses group)", block=False, device=q.device)
        B, H, N, d = q.shape
        bm = BlockMask._trusted(keep, self.cfg.b_q, self.cfg.b_kv, N)
        lists = at.mask_lists(bm, B, H, N)
        _, lse = at.fwd(q, k, v, lists, 1.0 / math.sqrt(d), o=o_out)
        return (lists, lse, bm)

    def backward(self, saved, q, k, v, o, do, dq_out, dk_out, dv_out):
        from . import attention as at

        lists, lse, _ = saved
        at.bwd(q, k, v, o, do, lse, lists, 1.0 / math.sqrt(q.shape[-1]), dq=dq_out, dk=dk_out, dv=dv_out)


def _head_view(buf: torch.Tensor) -> torch.Tensor:
    """[P, n_loc, h, d] receive / send buffer of one batch row as a [1, h, N, d] strided view."""
    P, n_loc, h, d = buf.shape
    return buf.view(P * n_loc, h, d).permute(1, 0, 2).unsqueeze(0)


class _UlyssesFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q_l, k_l, v_l, mod):
        out_l, saved = mod._forward(q_l, k_l, v_l)
        ctx.mod = mod
        ctx.saved = saved
        return out_l

    @staticmethod
    def backward(ctx, do_l):
        dq, dk, dv = ctx.mod._backward(ctx.saved, do_l.contiguous())
        ctx.saved = None
        return dq, dk, dv, None


class UlyssesAttention:
    """Sequence-parallel sparse attention: ``self(q_l, k_l, v_l)`` with sequence-sharded
    [B, N/P, H, d] inputs returns the sequence-sharded [B, N/P, H, d] output, differentiable.
    Rank r computes heads {p·H/P + h : h in its local range} for the FULL sequence — the
    masker needs a head's whole sequence, exactly as on one GPU — so results equal the
    single-GPU operator's.  ``groups`` head groups per rank pipeline the exchange against
    the compute (see the module docstring)."""

    def __init__(self, cfg, group=None, groups: int = 4, kernels=None):
        self.cfg = cfg
        self.group = group
        self.groups = groups
        self.kernels = kernels if kernels is not None else GroupKernels(cfg)
        self._comm = None
        self._events: list[tuple] = []

    def __call__(self, q_l, k_l, v_l):
        return _UlyssesFn.apply(q_l, k_l, v_l, self)

    # ---- helpers ----
    def _streams(self, dev):
        if dev.type != "cuda":
            return None
        if self._comm is None:
            self._comm = torch.cuda.Stream(dev)
        return self._comm

    def _bounds(self, hp):
        G = max(1, min(self.groups, hp))
        return [(g * hp // G, (g + 1) * hp // G) for g in range(G)]

    def comm_ms(self, reps: int) -> float:
        """Mean all-to-all device time per call over the last `reps` fwd+bwd calls (events on
        the communication stream; the transfers overlap the compute)."""
        ev = self._events[-reps:]
        if not ev:
            return 0.0
        torch.cuda.synchronize()
        return sum(sum(a.elapsed_time(b) for a, b in call) for call in ev) / len(ev)

    def _exchange(self, chunks_in, dev, comm, record):
        """all-to-all of each (send, recv) pair on the communication stream."""
        for send, recv in chunks_in:
            if comm is not None and record is not None:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(comm)
                _all_to_all(recv, send, self.group)
                b.record(comm)
                record.append((a, b))
            else:
                _all_to_all(recv, send, self.group)

    def _forward(self, q_l, k_l, v_l):
        rank, P = _world(self.group)
        B, n_loc, H, d = q_l.shape
        if H % P:
            raise ValueError(f"Ulysses needs H % world == 0 (H={H}, world={P})")
        hp = H // P
        dev = q_l.device
        comm = self._streams(dev)
        main = torch.cuda.current_stream(dev) if comm is not None else None
        record = [] if comm is not None else None
        out_l = torch.empty_like(q_l)
        xs = [t.reshape(B, n_loc, P, hp, d) for t in (q_l, k_l, v_l)]
        saved = {"groups": [], "shape": (B, n_loc, H, d)}
        bounds = self._bounds(hp)
        # 1. every group's input exchange, issued up front on the comm stream
        recvs, ev_in = [], []
        if comm is not None:
            comm.wait_stream(main)
        for g0, g1 in bounds:
            hg = g1 - g0
            per_b = []
            with torch.cuda.stream(comm) if comm is not None else _null():
                for b in range(B):
                    pairs = []
                    for x in xs:
                        send = x[b, :, :, g0:g1].permute(1, 0, 2, 3).contiguous()  # [P (dest), n_loc, hg, d]
                        pairs.append((send, torch.empty_like(send)))
                    self._exchange(pairs, dev, comm, record)
                    per_b.append([r for _, r in pairs])
                e = torch.cuda.Event() if comm is not None else None
                if e is not None:
                    e.record(comm)
            recvs.append(per_b)
            ev_in.append(e)
        # 2. per group: compute on the main stream as soon as its inputs land; the output
        #    exchange of group g overlaps the compute of group g+1
        for gi, (g0, g1) in enumerate(bounds):
            if comm is not None:
                main.wait_event(ev_in[gi])
            grp = []
            for b in range(B):
                rq, rk, rv = recvs[gi][b]
                if comm is not None:
                    for t in (rq, rk, rv):
                        t.record_stream(main)
                o_send = torch.empty_like(rq)  # written by the kernel in the return exchange's layout
                qv, kv, vv, ov = (_head_view(t) for t in (rq, rk, rv, o_send))
                st = self.kernels.forward(qv, kv, vv, ov)
                grp.append((rq, rk, rv, o_send, st))
            saved["groups"].append(grp)
            e = torch.cuda.Event() if comm is not None else None
            if e is not None:
                e.record(main)
            with torch.cuda.stream(comm) if comm is not None else _null():
                if comm is not None:
                    comm.wait_event(e)
                for b in range(B):
                    o_send = grp[b][3]
                    o_recv = torch.empty_like(o_send)  # [P (source = head owner), n_loc, hg, d]
                    self._exchange([(o_send, o_recv)], dev, comm, record)
                    out_l.view(B, n_loc, P, hp, d)[b, :, :, g0:g1].copy_(o_recv.permute(1, 0, 2, 3))
        if comm is not None:
            main.wait_stream(comm)
            out_l.record_stream(comm)
        saved["record"] = record
        return out_l, saved

    def _backward(self, saved, do_l):
        rank, P = _world(self.group)
        B, n_loc, H, d = saved["shape"]
        hp = H // P
        dev = do_l.device
        comm = self._streams(dev)
        main = torch.cuda.current_stream(dev) if comm is not None else None
        record = saved["record"]
        grads = [torch.empty((B, n_loc, H, d), device=dev, dtype=do_l.dtype) for _ in range(3)]
        dox = do_l.reshape(B, n_loc, P, hp, d)
        bounds = self._bounds(hp)
        if comm is not None:
            comm.wait_stream(main)
        recvs, ev_in = [], []
        for g0, g1 in bounds:
            per_b = []
            with torch.cuda.stream(comm) if comm is not None else _null():
                for b in range(B):
                    send = dox[b, :, :, g0:g1].permute(1, 0, 2, 3).contiguous()
                    recv = torch.empty_like(send)
                    self._exchange([(send, recv)], dev, comm, record)
                    per_b.append(recv)
                e = torch.cuda.Event() if comm is not None else None
                if e is not None:
                    e.record(comm)
            recvs.append(per_b)
            ev_in.append(e)
        for gi, (g0, g1) in enumerate(bounds):
            if comm is not None:
                main.wait_event(ev_in[gi])
            sends = []
            for b in range(B):
                rq, rk, rv, o_send, st = saved["groups"][gi][b]
                rdo = recvs[gi][b]
                if comm is not None:
                    rdo.record_stream(main)
                dq_s, dk_s, dv_s = (torch.empty_like(rq) for _ in range(3))
                self.kernels.backward(st, *(_head_view(t) for t in (rq, rk, rv, o_send, rdo, dq_s, dk_s, dv_s)))
                sends.append((dq_s, dk_s, dv_s))
            e = torch.cuda.Event() if comm is not None else None
            if e is not None:
                e.record(main)
            with torch.cuda.stream(comm) if comm is not None else _null():
                if comm is not None:
                    comm.wait_event(e)
                for b in range(B):
                    for gsend, gout in zip(sends[b], grads):
                        grecv = torch.empty_like(gsend)
                        self._exchange([(gsend, grecv)], dev, comm, record)
                        gout.view(B, n_loc, P, hp, d)[b, :, :, g0:g1].copy_(grecv.permute(1, 0, 2, 3))
        if comm is not None:
            main.wait_stream(comm)
            for g in grads:
                g.record_stream(comm)
            self._events.append(record)
            self._events = self._events[-64:]
        return tuple(grads)


class _null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def ulysses_sparse_attention(q_l, k_l, v_l, cfg, group=None, groups: int = 4):
    """Sequence-sharded [B, N/P, H, d] q/k/v -> sequence-sharded output (differentiable),
    through the overlapped ``UlyssesAttention``."""
    return UlyssesAttention(cfg, group=group, groups=groups)(q_l, k_l, v_l)

"""Block-sparse attention forward / backward on the GPU, with autograd.

Drop-in for ``sparseattn_lab.attention`` (attention.py:22-166): same names, arguments,
result types and errors.  Compute runs in ``libspa2.so``:

* ``sparse_attention_with_mask`` -> K4 tcgen05 forward (O bf16, LSE fp32 natural log);
* ``attention_backward`` / autograd -> K5 δ, K6 dK/dV (KV-major lists), K7 dQ (row lists);
* ``sparse_attention`` = K1 pooled map -> K2 hybrid select -> K3 lists -> K4.

Inputs are [N, d] (the reference contract) or [B, H, N, d]; they are computed in bf16
(the reference's float64 is out of reach of tensor cores); results come back in the
caller's container (numpy in -> numpy float64 out).  The kernels use b_q = 128 and
b_kv = 64 (the paper's setting); masks at coarser multiples of that grid
(or all-ones masks such as ``full_mask``) are refined exactly, other geometries raise.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .masker import BlockMask, SparsityConfig, _pooled_probs, _select, top_k_count
from .numerics import finite_guard, from_device, num_blocks, to_device4

BQ, BKV = 128, 64
SUPPORTED_HEAD_DIMS = (64, 128)


@dataclass(frozen=True)
class AttentionOutput:
    """attention.py:22-26."""

    out: object
    lse: object
    mask_used: BlockMask


@dataclass(frozen=True)
class AttentionGrads:
    """attention.py:29-33."""

    dq: object
    dk: object
    dv: object


class BlockCounter:
    """Counts computed (query block, key block) pairs of the mask's grid (attention.py:36-43).
    On the kernels' native grid (b_q, b_kv) = (128, 64) the forward counts the tiles it
    computed on the device; a coarser mask is refined into several kernel tiles per mask
    block, so the count is then the mask's kept blocks (what the reference's loop visits)."""

    def __init__(self):
        self.count = 0

    def hit(self, i: int, j: int) -> None:
        self.count += 1


def full_mask(n: int) -> BlockMask:
    """One all-kept block covering everything (attention.py:46-47); a host mask, as in the
    reference."""
    return BlockMask(np.ones((1, 1), dtype=bool), b_q=n, b_kv=n, n_tokens=n)


# --------------------------------------------------------------------------------------
# block lists
# --------------------------------------------------------------------------------------

@dataclass(frozen=True)
class BlockLists:
    """CSR block lists over flattened (b, h, block) rows / columns, on the device."""

    row_ptr: torch.Tensor
    row_idx: torch.Tensor
    row_order: torch.Tensor
    col_ptr: torch.Tensor
    col_idx: torch.Tensor
    col_order: torch.Tensor
    shape: tuple  # (B, H, T_m, T_n)
    half: bool = False  # entries carry half-block codes (a b_q = 64·odd mask): kernels take b_q = 64


def _mask_on(bm: BlockMask, device: torch.device | None) -> torch.Tensor:
    """The mask's device keep tensor on ``device``: a host (numpy) mask is uploaded there (cached
    per device); a CUDA mask must already live there (the kernels take raw device pointers)."""
    keep = bm.dev
    if device is None or keep.device == device:
        return keep
    if not bm.on_host:
        raise ValueError(f"BlockMask is on {keep.device}, the inputs are on {device}")
    key = ("dev", str(device))
    hit = bm._cache.get(key)
    if hit is None:
        hit = bm._cache[key] = keep.to(device)
    return hit


def _native_keep(bm: BlockMask, B: int, H: int, N: int, device: torch.device | None = None) -> torch.Tensor:
    """keep at the kernel grid (128, 64) as uint8 codes [B, H, T_m, T_n]: 0 dropped, 1 kept.

    Masks on coarser grids (b_q ∈ 128ℕ, b_kv ∈ 64ℕ) are refined exactly.  Masks with
    b_q = 64·odd (e.g. the b_q = 64 of SURVEY §7) pair two 64-row mask rows per 128-row kernel
    query block: code 1 = both halves keep the tile, 2 = only the top half (rows 0-63),
    3 = only the bottom half — the kernels give the other half's rows P = 0 for that tile
    (list entries carry the code in bits 30-31, see csrc/common.cuh)."""
    t_m, t_n = num_blocks(N, BQ), num_blocks(N, BKV)
    keep = _mask_on(bm, device)
    if keep.dim() == 2:
        keep = keep.view(1, 1, *keep.shape)
    codes = None
    if (bm.b_q, bm.b_kv) != (BQ, BKV):
        if bm.b_q % BQ == 0 and bm.b_kv % BKV == 0:
            keep = keep.repeat_interleave(bm.b_q // BQ, dim=-2).repeat_interleave(bm.b_kv // BKV, dim=-1)
            keep = keep[..., :t_m, :t_n]
        elif bm.b_q % (BQ // 2) == 0 and bm.b_kv % BKV == 0:
            t_h = num_blocks(N, BQ // 2)  # 64-row halves
            k64 = keep.repeat_interleave(bm.b_q // (BQ // 2), dim=-2).repeat_interleave(bm.b_kv // BKV, dim=-1)
            k64 = k64[..., :t_h, :t_n]
            if t_h % 2:  # the last query block has no bottom half inside N
                k64 = torch.cat([k64, torch.zeros_like(k64[..., :1, :])], dim=-2)
            top, bot = k64[..., 0::2, :], k64[..., 1::2, :]
            codes = torch.where(top & bot, 1, torch.where(top, 2, torch.where(bot, 3, 0))).to(torch.uint8)
        elif bool(keep.all()):
            keep = torch.ones((*keep.shape[:2], t_m, t_n), device=keep.device, dtype=torch.bool)
        else:
            raise ValueError(f"GPU kernels use b_q={BQ} (or 64), b_kv={BKV}; mask geometry (b_q={bm.b_q}, "
                             f"b_kv={bm.b_kv}) is not a multiple of it")
    if codes is None:
        codes = keep.view(torch.uint8) if keep.dtype == torch.bool else keep.to(torch.uint8)
    if codes.shape[0] != B or codes.shape[1] != H:
        if codes.shape[0] == 1 and codes.shape[1] == 1:
            codes = codes.expand(B, H, t_m, t_n)
        else:
            raise ValueError(f"mask batch/head dims {tuple(codes.shape[:2])} do not match inputs ({B}, {H})")
    return codes.contiguous()


def _half_codes(bm: BlockMask) -> bool:
    """True if the mask's query geometry is a 64-row multiple that is not a 128-row one."""
    return (bm.b_q, bm.b_kv) != (BQ, BKV) and bm.b_q % BQ != 0 and bm.b_q % (BQ // 2) == 0 and bm.b_kv % BKV == 0


def build_lists(keep_u8: torch.Tensor, half: bool = False) -> BlockLists:
    """K3 on a uint8 [B, H, T_m, T_n] keep-code tensor (see ``_native_keep``)."""
    B, H, t_m, t_n = keep_u8.shape
    bh, dev = B * H, keep_u8.device
    cap = max(1, bh * t_m * t_n)
    i32 = dict(device=dev, dtype=torch.int32)
    lists = BlockLists(
        row_ptr=torch.empty(bh * t_m + 1, **i32), row_idx=torch.empty(cap, **i32), row_order=torch.empty(bh * t_m, **i32),
        col_ptr=torch.empty(bh * t_n + 1, **i32), col_idx=torch.empty(cap, **i32), col_order=torch.empty(bh * t_n, **i32),
        shape=(B, H, t_m, t_n), half=half)
    scratch = torch.empty(bh * (t_m + t_n), **i32)
    st = torch.cuda.current_stream(dev)
    _lib.call("spa2_build_lists", _lib.ptr(keep_u8), bh, t_m, t_n, _lib.ptr(lists.row_ptr), _lib.ptr(lists.row_idx),
              _lib.ptr(lists.col_ptr), _lib.ptr(lists.col_idx), _lib.ptr(lists.row_order), _lib.ptr(lists.col_order),
              _lib.ptr(scratch), st.cuda_stream, stream_obj=st)
    return lists


def _lists_with_order(bm: BlockMask, B: int, H: int, N: int, visit, device=None) -> BlockLists:
    """Row lists honouring the reference's ``_block_order`` test hook (attention.py:74-81,
    97-99), which is called with the MASK grid's row index and kept columns, as in the
    reference; its order is then refined to the kernel grid (mask column j covers kernel
    columns j·(b_kv/64) ...).  Test-only: copies the mask to the host."""
    keep_u8 = _native_keep(bm, B, H, N, device)
    base = build_lists(keep_u8, half=_half_codes(bm))
    t_m, t_n = keep_u8.shape[-2:]
    mk = bm.keep_numpy().astype(bool)
    mk = np.broadcast_to(mk.reshape((1, 1) + mk.shape[-2:]) if mk.ndim == 2 else mk, (B, H) + mk.shape[-2:])
    rq = bm.b_q // BQ if bm.b_q % BQ == 0 else None
    rk = bm.b_kv // BKV if bm.b_kv % BKV == 0 else None
    half = rq is None and bm.b_q % (BQ // 2) == 0 and rk is not None  # b_q = 64·odd: two mask rows per block
    codes = keep_u8.cpu().numpy()
    idx = []
    for b in range(B):
        for h in range(H):
            orders = {}  # the hook runs once per MASK row, as in the reference

            def order_of(i_m):
                if i_m not in orders:
                    orders[i_m] = [int(j) for j in visit(i_m, np.flatnonzero(mk[b, h, i_m]))]
                return orders[i_m]

            for r in range(t_m):
                if half:  # the union of the two halves' orders; entries carry the half code
                    out, seen = [], set()
                    for hrow in (2 * r, 2 * r + 1):
                        i_m = hrow * (BQ // 2) // bm.b_q
                        if hrow * (BQ // 2) >= N or i_m >= mk.shape[-2]:
                            continue
                        for j in order_of(i_m):
                            for c in range(j * rk, min((j + 1) * rk, t_n)):
                                if c not in seen:
                                    seen.add(c)
                                    out.append(c | ((int(codes[b, h, r, c]) - 1) << 30))
                    idx.append(np.asarray(out, dtype=np.int64).astype(np.int32))
                    continue
                if rq is None or rk is None:  # all-ones mask of an arbitrary geometry
                    i_m = min(r * BQ // bm.b_q, mk.shape[-2] - 1)
                    order = order_of(i_m)
                    seen, out = set(), []
                    for j in order:
                        for c in range(t_n):
                            if c * BKV < (j + 1) * bm.b_kv and (c + 1) * BKV > j * bm.b_kv and c not in seen:
                                seen.add(c)
                                out.append(c)
                else:
                    order = order_of(r // rq)
                    out = [c for j in order for c in range(j * rk, min((j + 1) * rk, t_n))]
                idx.append(np.asarray(out, dtype=np.int32))
    flat = torch.tensor(np.concatenate(idx) if idx else np.zeros(0, np.int32), device=keep_u8.device)
    return BlockLists(base.row_ptr, flat, base.row_order, base.col_ptr, base.col_idx, base.col_order, base.shape,
                      base.half)


def mask_lists(bm: BlockMask, B: int, H: int, N: int, device: torch.device | None = None) -> BlockLists:
    """Block lists of ``bm`` for a [B, H, N, d] problem on ``device`` (default: the mask's own),
    cached on the (immutable) mask."""
    key = ("lists", B, H, N, None if device is None else str(device))
    hit = bm._cache.get(key)
    if hit is None:
        hit = build_lists(_native_keep(bm, B, H, N, device), half=_half_codes(bm))
        bm._cache[key] = hit
    return hit


# --------------------------------------------------------------------------------------
# kernel launchers
# --------------------------------------------------------------------------------------

def _check_kernel_shape(q4: torch.Tensor) -> None:
    d = q4.shape[-1]
    if d not in SUPPORTED_HEAD_DIMS:
        raise ValueError(f"GPU kernels support head dim d in {SUPPORTED_HEAD_DIMS}, got d={d}")


def fwd(q4, k4, v4, lists: BlockLists, scale: float, counter: torch.Tensor | None = None,
        o: torch.Tensor | None = None):
    """K4: returns (O [B,H,N,d] bf16, LSE [B,H,N] fp32).  ``o`` may be a preallocated strided
    [B,H,N,d] view to write O into (e.g. a collective's send buffer)."""
    B, H, N, d = q4.shape
    if o is None:
        o = torch.empty((B, H, N, d), device=q4.device, dtype=q4.dtype)
    lse = torch.empty((B, H, N), device=q4.device, dtype=torch.float32)
    st = torch.cuda.current_stream(q4.device)
    _lib.call("spa2_fwd", _lib.view4(q4), _lib.view4(k4), _lib.view4(v4), _lib.view4(o), _lib.ptr(lse),
              _lib.DTYPE_CODES[q4.dtype], B, H, N, d, BQ // 2 if lists.half else BQ, BKV, _lib.ptr(lists.row_ptr),
              _lib.ptr(lists.row_idx), _lib.ptr(lists.row_order), scale, _lib.ptr(counter), st.cuda_stream, stream_obj=st)
    return o, lse


def bwd(q4, k4, v4, o4, do4, lse, lists: BlockLists, scale: float, dq=None, dk=None, dv=None):
    """K5-K7: returns (dQ, dK, dV) bf16 [B,H,N,d] (optionally written into given strided views)."""
    B, H, N, d = q4.shape
    if dq is None:
        dq = torch.empty((B, H, N, d), device=q4.device, dtype=q4.dtype)
    if dk is None:
        dk = torch.empty((B, H, N, d), device=q4.device, dtype=q4.dtype)
    if dv is None:
        dv = torch.empty((B, H, N, d), device=q4.device, dtype=q4.dtype)
    delta = torch.empty((B, H, N), device=q4.device, dtype=torch.float32)
    st = torch.cuda.current_stream(q4.device)
    dt = _lib.DTYPE_CODES[q4.dtype]
    bq = BQ // 2 if lists.half else BQ  # b_q = 64 tells the kernels the lists carry half-block codes
    # δ = rowsum(dO ∘ O) is computed inside the dQ kernel (spa2_bwd_dq_delta)
    _lib.call("spa2_bwd_dq_delta", _lib.view4(q4), _lib.view4(k4), _lib.view4(v4), _lib.view4(o4), _lib.view4(do4),
              _lib.ptr(lse), _lib.ptr(delta), _lib.view4(dq), dt, B, H, N, d, bq, BKV, _lib.ptr(lists.row_ptr),
              _lib.ptr(lists.row_idx), _lib.ptr(lists.row_order), scale, st.cuda_stream, stream_obj=st)
    _lib.call("spa2_bwd_dkdv", _lib.view4(q4), _lib.view4(k4), _lib.view4(v4), _lib.view4(do4), _lib.ptr(lse),
              _lib.ptr(delta), _lib.view4(dk), _lib.view4(dv), dt, B, H, N, d, bq, BKV, _lib.ptr(lists.col_ptr),
              _lib.ptr(lists.col_idx), _lib.ptr(lists.col_order), scale, st.cuda_stream, stream_obj=st)
    return dq, dk, dv


class SparseAttentionFunction(torch.autograd.Function):
    """O, LSE = sparse_attention(q, k, v | block lists); the mask is a constant
    (SPEC.md:260), so only q, k, v receive gradients."""

    @staticmethod
    def forward(ctx, q4, k4, v4, lists, scale, counter, finite=None):
        o, lse = fwd(q4, k4, v4, lists, scale, counter)
        ctx.save_for_backward(q4, k4, v4, o, lse)
        ctx.lists = lists
        ctx.scale = scale
        ctx.finite = finite
        ctx.mark_non_differentiable(lse)
        return o, lse

    @staticmethod
    def backward(ctx, do, _dlse):
        if ctx.finite is not None:  # no gradients from non-finite inputs (numerics.py:29-32)
            finite_guard.resolve(ctx.finite)
        q4, k4, v4, o, lse = ctx.saved_tensors
        do = do.to(q4.dtype)
        if do.stride(-1) != 1 or any(s % 8 for s in do.stride()[:3]):
            do = do.contiguous()
        dq, dk, dv = bwd(q4, k4, v4, o, do, lse, ctx.lists, ctx.scale)
        return dq, dk, dv, None, None, None, None


# --------------------------------------------------------------------------------------
# reference-facing API
# --------------------------------------------------------------------------------------

def _host_finite(named) -> None:
    """numerics.ensure_finite (numerics.py:29-32) on the caller's own float64 arrays."""
    for name, x in named:
        if not isinstance(x, torch.Tensor) and not np.all(np.isfinite(np.asarray(x, dtype=np.float64))):
            raise FloatingPointError(f"non-finite values in {name}")


def _scan_finite(flag: torch.Tensor, *tensors: torch.Tensor) -> None:
    """K0: OR "has a NaN/Inf" of each bf16 [B,H,N,d] tensor into ``flag`` (no host sync)."""
    st = torch.cuda.current_stream(tensors[0].device)
    for t in tensors:
        B, H, N, d = t.shape
        _lib.call("spa2_check_finite", _lib.view4(t), _lib.DTYPE_CODES[t.dtype], B, H, N, d, _lib.ptr(flag),
                  st.cuda_stream, stream_obj=st)


_SIDE_STREAMS: dict = {}


def _scan_finite_side(flag: torch.Tensor, *tensors: torch.Tensor) -> torch.cuda.Event:
    """K0 on a per-device side stream, concurrent with the masker on the current stream (the
    scan only feeds the host-side verdict, nothing on the GPU waits for it).  Returns the event
    that marks its completion."""
    dev = tensors[0].device
    main = torch.cuda.current_stream(dev)
    side = _SIDE_STREAMS.get(dev)
    if side is None:
        side = _SIDE_STREAMS[dev] = torch.cuda.Stream(dev)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        _scan_finite(flag, *tensors)
        ev = torch.cuda.Event()
        ev.record(side)
    for t in tensors:
        t.record_stream(side)
    return ev


def _prepare(q, k, v, check_finite):
    """attention.py:50-59: same shapes (ValueError), rank (ShapeError), finite
    (FloatingPointError; numpy inputs are checked on the host exactly as the reference does,
    torch inputs by the K0 scan with a deferred verdict, see ``numerics.FiniteGuard``).
    Returns (q4, k4, v4, boundary, finite-flag or None)."""
    if check_finite:
        finite_guard.check_pending(block=False)  # verdicts of earlier calls that have landed
        _host_finite((("q", q), ("k", k), ("v", v)))
    q4, qb = to_device4(q, torch.bfloat16, "q")
    k4, _ = to_device4(k, torch.bfloat16, "k", device=qb.device)
    v4, _ = to_device4(v, torch.bfloat16, "v", device=qb.device)
    if not (q4.shape == k4.shape == v4.shape):
        raise ValueError(f"q/k/v shapes differ: {tuple(q4.shape)}, {tuple(k4.shape)}, {tuple(v4.shape)}")
    _check_kernel_shape(q4)
    q4, k4, v4 = (_tma_ready(t) for t in (q4, k4, v4))
    flag = finite_guard.new_flag(q4.device) if check_finite and not qb.numpy else None
    return q4, k4, v4, qb, flag


def _tma_ready(t: torch.Tensor) -> torch.Tensor:
    """TMA needs 16-byte aligned base and strides that are multiples of 8 elements."""
    if t.data_ptr() % 16 or any(s % 8 for s in t.stride()[:3]):
        return t.contiguous()
    return t


def _run(q4, k4, v4, bm: BlockMask, qb, counter, flag, check_finite, visit=None, side_event=None) -> AttentionOutput:
    B, H, N, d = q4.shape
    if bm.n_tokens != N:
        raise ValueError(f"mask built for {bm.n_tokens} tokens, inputs have {N}")
    lists = (mask_lists(bm, B, H, N, q4.device) if visit is None
             else _lists_with_order(bm, B, H, N, visit, q4.device))
    native = (bm.b_q, bm.b_kv) == (BQ, BKV)
    ctr = torch.zeros((1,), device=q4.device, dtype=torch.int64) if counter is not None and native else None
    verdict = None
    if flag is not None:
        verdict = finite_guard.submit(flag, "q, k or v", block=check_finite == "sync", device=q4.device,
                                      extra_event=side_event)
    o, lse = SparseAttentionFunction.apply(q4, k4, v4, lists, 1.0 / math.sqrt(d), ctr, verdict)
    if counter is not None:
        counter.count += int(ctr.item()) if native else bm.kept_blocks()
    return AttentionOutput(out=from_device(o, qb), lse=from_device(lse, qb, 1), mask_used=bm)


def sparse_attention_with_mask(q, k, v, bm: BlockMask, counter: BlockCounter | None = None, _block_order=None,
                               *, check_finite: bool | str = True) -> AttentionOutput:
    """Tiled attention restricted to ``bm``'s kept blocks (attention.py:73-114).

    ``out`` is differentiable w.r.t. torch inputs.  ``_block_order(i, kept)`` may permute
    the visit order of each row (the reference's test hook, called on the mask's own grid);
    the result does not depend on it beyond float rounding.  ``check_finite``: True (the
    reference's ``ensure_finite``; deferred for torch inputs, see ``numerics.FiniteGuard``),
    ``"sync"`` (raise before returning) or False.
    """
    q4, k4, v4, qb, flag = _prepare(q, k, v, check_finite)
    if flag is not None:
        _scan_finite(flag, q4, k4, v4)
    return _run(q4, k4, v4, bm, qb, counter, flag, check_finite, _block_order)


_FUSED_SELECT = os.environ.get("SPA2_FUSED_SELECT", "1") != "0"


def _hybrid_mask_device(q4, k4, cfg: SparsityConfig, flag: torch.Tensor | None, fused: bool | None = None):
    """hybrid_mask(pooled_map(q, k, cfg), cfg) as a device keep tensor, without materialising
    the map: the row softmax runs inside the select kernel (bit-identical masks;
    ``fused=False`` takes the two-step pooled_map + select path).  K1 ORs "q or k has a
    NaN/Inf" into ``flag``."""
    t_n = num_blocks(q4.shape[2], cfg.b_kv)
    if fused is None:
        fused = _FUSED_SELECT
    if fused and t_n <= 4096:
        scores = _pooled_probs(q4, k4, cfg.b_q, cfg.b_kv, flag, softmax=False)
        keep, _ = _select(scores, top_k_count(cfg.k_frac, t_n), cfg.p_frac, from_scores=True)
    else:
        probs = _pooled_probs(q4, k4, cfg.b_q, cfg.b_kv, flag)
        keep, _ = _select(probs, top_k_count(cfg.k_frac, probs.shape[-1]), cfg.p_frac)
    if q4.shape[0] == 1 and q4.shape[1] == 1:
        keep = keep[0, 0]
    return keep


def sparse_attention(q, k, v, cfg: SparsityConfig, counter: BlockCounter | None = None, *,
                     check_finite: bool | str = True) -> AttentionOutput:
    """Derive the hybrid mask from the current q/k, then run the kernel (attention.py:117-125).
    The mask is rebuilt on every call; nothing is cached across steps.
    Finiteness: K1 checks q and k while pooling them, K0 scans v; no host sync for torch
    callers (``check_finite`` as in ``sparse_attention_with_mask``)."""
    q4, k4, v4, qb, flag = _prepare(q, k, v, check_finite)
    side = _scan_finite_side(flag, v4) if flag is not None else None
    keep = _hybrid_mask_device(q4, k4, cfg, flag)
    bm = BlockMask._from_device(keep, cfg.b_q, cfg.b_kv, q4.shape[2], host=qb.numpy)
    return _run(q4, k4, v4, bm, qb, counter, flag, check_finite, side_event=side)


def dense_attention(q, k, v, *, check_finite: bool | str = True) -> AttentionOutput:
    """Full softmax attention (attention.py:62-70), computed by the same kernels with every
    block kept; ``mask_used`` is ``full_mask(N)`` as in the reference."""
    q4, k4, v4, qb, flag = _prepare(q, k, v, check_finite)
    if flag is not None:
        _scan_finite(flag, q4, k4, v4)
    return _run(q4, k4, v4, full_mask(q4.shape[2]), qb, None, flag, check_finite)


def attention_backward(q, k, v, bm: BlockMask, d_out, *, check_finite: bool | str = True) -> AttentionGrads:
    """Gradients of the masked attention output with the mask held constant
    (attention.py:128-166).  Like the reference it recomputes the forward for O and LSE."""
    if check_finite:
        _host_finite((("d_out", d_out),))
    q4, k4, v4, qb, flag = _prepare(q, k, v, check_finite)
    do4, _ = to_device4(d_out, torch.bfloat16, "d_out", device=qb.device)
    if do4.shape != q4.shape:
        raise ValueError(f"d_out shape {tuple(do4.shape)} != q shape {tuple(q4.shape)}")
    do4 = _tma_ready(do4)
    B, H, N, d = q4.shape
    if bm.n_tokens != N:
        raise ValueError(f"mask built for {bm.n_tokens} tokens, inputs have {N}")
    if flag is not None:
        _scan_finite(flag, q4, k4, v4, do4)
        finite_guard.submit(flag, "q, k, v or d_out", block=check_finite == "sync", device=q4.device)
    lists = mask_lists(bm, B, H, N, q4.device)
    scale = 1.0 / math.sqrt(d)
    with torch.no_grad():
        o, lse = fwd(q4, k4, v4, lists, scale)
        dq, dk, dv = bwd(q4, k4, v4, o, do4, lse, lists, scale)
    return AttentionGrads(dq=from_device(dq, qb), dk=from_device(dk, qb), dv=from_device(dv, qb))


__all__ = [
    "AttentionOutput", "AttentionGrads", "BlockCounter", "BlockLists", "full_mask", "dense_attention",
    "sparse_attention", "sparse_attention_with_mask", "attention_backward", "SparseAttentionFunction",
    "build_lists", "mask_lists",
]

"""Block-pooled maps and Top-k / Top-p / hybrid block masks on the GPU.

Drop-in for ``sparseattn_lab.masker`` (masker.py:30-153): same names, arguments and
errors.  ``pooled_map`` runs the K1 kernels (float64 pooling + pooled scores + softmax),
``top_k_mask`` / ``top_p_mask`` / ``hybrid_mask`` run the K2 select kernel, which is
bit-exact with the reference for any float64 pooled map (stable descending order, ties
to the lower column, strictly sequential float64 prefix sums).

Tensors live on the CUDA device.  ``PooledMap.probs`` is float64 [T_m, T_n] (or
[B, H, T_m, T_n] for batched inputs); ``BlockMask.keep`` is bool of the same rank.  As in
the reference both objects are frozen and must be treated as immutable: the block lists
a mask derives for the attention kernels are cached on it.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .numerics import ShapeError, from_device, num_blocks, to_device4

# masker.py:27 — absorbs cumulative-sum rounding when a prefix lands exactly on p_frac
P_SLACK = 1e-12


@dataclass(frozen=True)
class SparsityConfig:
    """Masking policy (masker.py:30-43)."""

    k_frac: float
    p_frac: float
    b_q: int
    b_kv: int

    def __post_init__(self):
        if not (0.0 <= self.k_frac <= 1.0):
            raise ValueError(f"k_frac out of [0,1]: {self.k_frac}")
        if not (0.0 <= self.p_frac <= 1.0):
            raise ValueError(f"p_frac out of [0,1]: {self.p_frac}")
        if self.b_q < 1 or self.b_kv < 1:
            raise ValueError(f"block sizes must be >= 1: b_q={self.b_q}, b_kv={self.b_kv}")


def _as_probs(probs) -> torch.Tensor:
    t = probs if isinstance(probs, torch.Tensor) else torch.as_tensor(np.asarray(probs, dtype=np.float64))
    if t.dim() not in (2, 4):
        raise ShapeError(f"expected rank 2 (or 4 for batched maps), got rank {t.dim()} with shape {tuple(t.shape)}")
    dev = t.device if t.is_cuda else torch.device("cuda", torch.cuda.current_device())
    _lib.require_device(dev)
    return t.to(device=dev, dtype=torch.float64).contiguous()


@dataclass(frozen=True)
class PooledMap:
    """Row-stochastic block-level attention map plus grid geometry (masker.py:46-62)."""

    probs: torch.Tensor
    b_q: int
    b_kv: int
    n_tokens: int

    def __post_init__(self):
        probs = _as_probs(self.probs)
        object.__setattr__(self, "probs", probs)
        if not bool(torch.isfinite(probs).all()):
            raise FloatingPointError("non-finite values in pooled map")
        if bool(((probs.sum(dim=-1) - 1.0).abs() > 1e-12).any()):
            raise ValueError("pooled map rows must sum to 1 within 1e-12")

    @classmethod
    def _trusted(cls, probs: torch.Tensor, b_q: int, b_kv: int, n_tokens: int) -> "PooledMap":
        """Built by the K1 kernels: already validated by construction (no device sync)."""
        obj = object.__new__(cls)
        for k, v in (("probs", probs), ("b_q", b_q), ("b_kv", b_kv), ("n_tokens", n_tokens)):
            object.__setattr__(obj, k, v)
        return obj


@dataclass(frozen=True)
class BlockMask:
    """Per-(query block, key block) keep matrix plus block geometry (masker.py:65-97)."""

    keep: torch.Tensor
    b_q: int
    b_kv: int
    n_tokens: int
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        k = self.keep if isinstance(self.keep, torch.Tensor) else torch.as_tensor(np.asarray(self.keep))
        if k.dim() not in (2, 4):
            raise ValueError(f"keep must be rank 2, got shape {tuple(k.shape)}")
        dev = k.device if k.is_cuda else torch.device("cuda", torch.cuda.current_device())
        _lib.require_device(dev)
        k = (k.to(device=dev) != 0).contiguous()
        object.__setattr__(self, "keep", k)
        t_m, t_n = num_blocks(self.n_tokens, self.b_q), num_blocks(self.n_tokens, self.b_kv)
        if tuple(k.shape[-2:]) != (t_m, t_n):
            raise ValueError(f"keep shape {tuple(k.shape)} does not match grid ({t_m}, {t_n}) "
                             f"for n_tokens={self.n_tokens}")
        if not bool(k.any(dim=-1).all()):
            raise ValueError("every query block must keep at least one key block")

    @classmethod
    def _trusted(cls, keep: torch.Tensor, b_q: int, b_kv: int, n_tokens: int) -> "BlockMask":
        """Built by the select kernel, which keeps >= 1 block per row by construction."""
        obj = object.__new__(cls)
        for k, v in (("keep", keep), ("b_q", b_q), ("b_kv", b_kv), ("n_tokens", n_tokens), ("_cache", {})):
            object.__setattr__(obj, k, v)
        return obj

    @property
    def grid(self) -> tuple[int, int]:
        return tuple(self.keep.shape[-2:])

    def sparsity(self) -> float:
        """1 - kept/total, counted in blocks (masker.py:88-89)."""
        return 1.0 - float(self.keep.sum()) / self.keep.numel()

    def kept_blocks(self) -> int:
        return int(self.keep.sum())

    def __or__(self, other: "BlockMask") -> "BlockMask":
        if (self.b_q, self.b_kv, self.n_tokens) != (other.b_q, other.b_kv, other.n_tokens):
            raise ValueError("mask geometry mismatch")
        return BlockMask._trusted(self.keep | other.keep, self.b_q, self.b_kv, self.n_tokens)

    def keep_numpy(self) -> np.ndarray:
        return self.keep.cpu().numpy()


# --------------------------------------------------------------------------------------
# K1: pooled map
# --------------------------------------------------------------------------------------

def pooled_map(q, k, cfg: SparsityConfig) -> PooledMap:
    """P̄ = softmax(mean-pool(Q, b_q) · mean-pool(K, b_kv)ᵀ / √d) (masker.py:100-110).

    Any float dtype is accepted; q/k are read in their own dtype and everything after the
    load is float64.  Raises ``FloatingPointError`` on non-finite q/k (numerics.py:29-32).
    """
    qt, qb = to_device4(q, None, "q")
    kt, _ = to_device4(k, None, "k", device=qb.device)
    if qt.shape[-1] != kt.shape[-1]:
        raise ValueError(f"q/k feature dims differ: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    if qt.shape[:-1] != kt.shape[:-1]:
        raise ValueError(f"q/k token counts differ: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    if kt.dtype != qt.dtype:
        kt = kt.to(qt.dtype)
    probs, flag = _pooled_probs(qt, kt, cfg.b_q, cfg.b_kv, check_finite=True)
    if flag is not None and int(flag.item()) != 0:
        raise FloatingPointError("non-finite values in q or k")
    if qb.rank == 2:
        probs = probs[0, 0]
    return PooledMap._trusted(probs, cfg.b_q, cfg.b_kv, qt.shape[2])


def _pooled_probs(qt: torch.Tensor, kt: torch.Tensor, b_q: int, b_kv: int, check_finite: bool, softmax: bool = True):
    """Launch K1 on [B,H,N,d] tensors; returns (probs [B,H,T_m,T_n] float64, flag|None).
    ``softmax=False`` returns the pre-softmax scores Q̄K̄ᵀ/√d (for spa2_select_scores)."""
    B, H, N, d = qt.shape
    t_m, t_n = num_blocks(N, b_q), num_blocks(N, b_kv)
    probs = torch.empty((B, H, t_m, t_n), device=qt.device, dtype=torch.float64)
    work = torch.empty((B * H * (t_m + t_n) * d,), device=qt.device, dtype=torch.float64)
    flag = torch.zeros((1,), device=qt.device, dtype=torch.int32) if check_finite else None
    st = torch.cuda.current_stream(qt.device)
    _lib.call("spa2_pooled_map" if softmax else "spa2_pooled_scores", _lib.view4(qt), _lib.view4(kt),
              _lib.DTYPE_CODES[qt.dtype], B, H, N, d, b_q, b_kv, _lib.ptr(probs), _lib.ptr(work), _lib.ptr(flag),
              st.cuda_stream, stream_obj=st)
    return probs, flag


# --------------------------------------------------------------------------------------
# K2: selection
# --------------------------------------------------------------------------------------

def top_k_count(k_frac: float, t_n: int) -> int:
    """K = max(1, ceil(k_frac * T_n)), evaluated in IEEE double (masker.py:118-119)."""
    return max(1, math.ceil(k_frac * t_n))


def _select(probs: torch.Tensor, k_count: int, p_frac: float | None,
            from_scores: bool = False) -> tuple[torch.Tensor, torch.Tensor]:
    t_n = probs.shape[-1]
    rows = probs.numel() // t_n
    keep = torch.empty(probs.shape, device=probs.device, dtype=torch.bool)
    counts = torch.empty(probs.shape[:-1], device=probs.device, dtype=torch.int32)
    thr = (p_frac - P_SLACK) if p_frac is not None else -math.inf
    st = torch.cuda.current_stream(probs.device)
    _lib.call("spa2_select_scores" if from_scores else "spa2_select", _lib.ptr(probs), rows, t_n, k_count, thr,
              _lib.ptr(keep), _lib.ptr(counts), st.cuda_stream, stream_obj=st)
    return keep, counts


def top_k_mask(pm: PooledMap, k_frac: float) -> BlockMask:
    """Keep the K largest entries per row, ties to the lower column (masker.py:122-128)."""
    keep, _ = _select(pm.probs, top_k_count(k_frac, pm.probs.shape[-1]), None)
    return BlockMask._trusted(keep, pm.b_q, pm.b_kv, pm.n_tokens)


def top_p_mask(pm: PooledMap, p_frac: float) -> BlockMask:
    """Keep the shortest descending prefix reaching p_frac (masker.py:131-142)."""
    keep, _ = _select(pm.probs, 1, p_frac)
    return BlockMask._trusted(keep, pm.b_q, pm.b_kv, pm.n_tokens)


def hybrid_mask(pm: PooledMap, cfg: SparsityConfig) -> BlockMask:
    """Top-k ∪ Top-p (masker.py:145-146), computed in one pass: both rules keep a prefix
    of the same stable order, so the union is its first max(K, cnt_p) columns."""
    keep, _ = _select(pm.probs, top_k_count(cfg.k_frac, pm.probs.shape[-1]), cfg.p_frac)
    return BlockMask._trusted(keep, pm.b_q, pm.b_kv, pm.n_tokens)


def expand_mask(bm: BlockMask) -> torch.Tensor:
    """Token-level 0/1 float64 matrix, entry (a, b) = keep[a // b_q, b // b_kv]
    (masker.py:149-153).  Materialises N×N — tests and analysis only."""
    n = bm.n_tokens
    full = bm.keep.repeat_interleave(bm.b_q, dim=-2).repeat_interleave(bm.b_kv, dim=-1)
    return full[..., :n, :n].to(torch.float64)


__all__ = [
    "P_SLACK", "SparsityConfig", "PooledMap", "BlockMask", "pooled_map", "top_k_count", "top_k_mask",
    "top_p_mask", "hybrid_mask", "expand_mask", "from_device",
]

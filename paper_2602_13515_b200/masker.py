"""Block-pooled maps and Top-k / Top-p / hybrid block masks on the GPU.

Drop-in for ``sparseattn_lab.masker`` (masker.py:30-186): same names, arguments, result
types and errors.  ``pooled_map`` runs the K1 kernels (float64 pooling + pooled scores +
softmax), ``top_k_mask`` / ``top_p_mask`` / ``hybrid_mask`` run the K2 select kernel, which
is bit-exact with the reference for any float64 pooled map (stable descending order, ties
to the lower column, strictly sequential float64 prefix sums).

Containers follow the caller, as in the reference's frozen dataclasses (masker.py:46-97):

* numpy in -> numpy out: ``PooledMap.probs`` is a read-only float64 ndarray and
  ``BlockMask.keep`` a read-only bool ndarray, exactly the reference's types, so callers
  such as ``pm.probs * bm.keep`` (cli.py:149-150) work unchanged.  The device copy the
  kernels need is made once and cached on the (immutable) object.
* torch in -> torch out: ``probs`` / ``keep`` are CUDA tensors ([T_m, T_n], or
  [B, H, T_m, T_n] for batched inputs) and nothing leaves the device.

``obj.dev`` is the device tensor in both cases (what the kernels consume).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .numerics import ShapeError, finite_guard, num_blocks, to_device4

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


def _device_of(t: torch.Tensor | None) -> torch.device:
    if t is not None and t.is_cuda:
        return t.device
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_13515_b200 requires a CUDA device (B200, sm_100a); none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _readonly(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    a.flags.writeable = False
    return a


@dataclass(frozen=True)
class PooledMap:
    """Row-stochastic block-level attention map plus grid geometry (masker.py:46-62)."""

    probs: object
    b_q: int
    b_kv: int
    n_tokens: int
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        p = self.probs
        if isinstance(p, torch.Tensor):
            if p.dim() not in (2, 4):
                raise ShapeError(f"expected rank 2 (or 4 for batched maps), got rank {p.dim()} with shape "
                                 f"{tuple(p.shape)}")
            dev = _device_of(p)
            _lib.require_device(dev)
            p = p.to(device=dev, dtype=torch.float64).contiguous()
            if not bool(torch.isfinite(p).all()):
                raise FloatingPointError("non-finite values in pooled map")
            if bool(((p.sum(dim=-1) - 1.0).abs() > 1e-12).any()):
                raise ValueError("pooled map rows must sum to 1 within 1e-12")
        else:  # the reference path: validated on the host, no device needed (numerics.py:21-32)
            p = np.asarray(p, dtype=np.float64)
            if p.ndim not in (2, 4):
                raise ShapeError(f"expected rank 2, got rank {p.ndim} with shape {p.shape}")
            if not np.all(np.isfinite(p)):
                raise FloatingPointError("non-finite values in pooled map")
            if np.any(np.abs(p.sum(axis=-1) - 1.0) > 1e-12):
                raise ValueError("pooled map rows must sum to 1 within 1e-12")
            p = _readonly(p)
        object.__setattr__(self, "probs", p)

    @classmethod
    def _trusted(cls, probs, b_q: int, b_kv: int, n_tokens: int, dev: torch.Tensor | None = None) -> "PooledMap":
        """Built by the K1 kernels: already validated by construction (no device sync)."""
        obj = object.__new__(cls)
        for k, v in (("probs", probs), ("b_q", b_q), ("b_kv", b_kv), ("n_tokens", n_tokens), ("_cache", {})):
            object.__setattr__(obj, k, v)
        if dev is not None:
            obj._cache["dev"] = dev
        return obj

    @property
    def on_host(self) -> bool:
        return not isinstance(self.probs, torch.Tensor)

    @property
    def dev(self) -> torch.Tensor:
        """float64 CUDA tensor of the map (cached upload for host maps)."""
        if not self.on_host:
            return self.probs
        hit = self._cache.get("dev")
        if hit is None:
            dev = _device_of(None)
            _lib.require_device(dev)
            hit = torch.from_numpy(np.array(self.probs)).to(dev)
            self._cache["dev"] = hit
        return hit


@dataclass(frozen=True)
class BlockMask:
    """Per-(query block, key block) keep matrix plus block geometry (masker.py:65-97)."""

    keep: object
    b_q: int
    b_kv: int
    n_tokens: int
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        k = self.keep
        t_m, t_n = num_blocks(self.n_tokens, self.b_q), num_blocks(self.n_tokens, self.b_kv)
        if isinstance(k, torch.Tensor):
            if k.dim() not in (2, 4):
                raise ValueError(f"keep must be rank 2, got shape {tuple(k.shape)}")
            dev = _device_of(k)
            _lib.require_device(dev)
            k = (k.to(device=dev) != 0).contiguous()
            if not bool(k.any(dim=-1).all()):
                raise ValueError("every query block must keep at least one key block")
        else:  # masker.py:71-86, on the host (rank 4 = the batched [B, H, T_m, T_n] extension)
            k = np.asarray(k)
            if k.ndim not in (2, 4):
                raise ValueError(f"keep must be rank 2, got shape {k.shape}")
            k = _readonly(k.astype(bool))
            if not np.all(k.any(axis=-1)):
                raise ValueError("every query block must keep at least one key block")
        if tuple(k.shape[-2:]) != (t_m, t_n):
            raise ValueError(f"keep shape {tuple(k.shape)} does not match grid ({t_m}, {t_n}) "
                             f"for n_tokens={self.n_tokens}")
        object.__setattr__(self, "keep", k)

    @classmethod
    def _trusted(cls, keep, b_q: int, b_kv: int, n_tokens: int, dev: torch.Tensor | None = None) -> "BlockMask":
        """Built by the select kernel, which keeps >= 1 block per row by construction."""
        obj = object.__new__(cls)
        for k, v in (("keep", keep), ("b_q", b_q), ("b_kv", b_kv), ("n_tokens", n_tokens), ("_cache", {})):
            object.__setattr__(obj, k, v)
        if dev is not None:
            obj._cache["dev"] = dev
        return obj

    @classmethod
    def _from_device(cls, keep_dev: torch.Tensor, b_q: int, b_kv: int, n_tokens: int, host: bool) -> "BlockMask":
        """Wrap a kernel-made device keep tensor; ``host`` = the caller passed numpy."""
        if host:
            return cls._trusted(_readonly(keep_dev.cpu().numpy()), b_q, b_kv, n_tokens, dev=keep_dev)
        return cls._trusted(keep_dev, b_q, b_kv, n_tokens)

    @property
    def on_host(self) -> bool:
        return not isinstance(self.keep, torch.Tensor)

    @property
    def dev(self) -> torch.Tensor:
        """bool CUDA tensor of the keep matrix (cached upload for host masks)."""
        if not self.on_host:
            return self.keep
        hit = self._cache.get("dev")
        if hit is None:
            dev = _device_of(None)
            _lib.require_device(dev)
            hit = torch.from_numpy(np.array(self.keep)).to(dev)
            self._cache["dev"] = hit
        return hit

    @property
    def grid(self) -> tuple[int, int]:
        return tuple(self.keep.shape[-2:])

    def sparsity(self) -> float:
        """1 - kept/total, counted in blocks (masker.py:88-89)."""
        if self.on_host:
            return 1.0 - self.keep.sum() / self.keep.size
        return 1.0 - float(self.keep.sum()) / self.keep.numel()

    def kept_blocks(self) -> int:
        return int(self.keep.sum())

    def __or__(self, other: "BlockMask") -> "BlockMask":
        if (self.b_q, self.b_kv, self.n_tokens) != (other.b_q, other.b_kv, other.n_tokens):
            raise ValueError("mask geometry mismatch")
        if self.on_host and other.on_host:
            return BlockMask(self.keep | other.keep, self.b_q, self.b_kv, self.n_tokens)
        return BlockMask._trusted(self.dev | other.dev, self.b_q, self.b_kv, self.n_tokens)

    def keep_numpy(self) -> np.ndarray:
        return np.asarray(self.keep) if self.on_host else self.keep.cpu().numpy()


# --------------------------------------------------------------------------------------
# K1: pooled map
# --------------------------------------------------------------------------------------

def pooled_map(q, k, cfg: SparsityConfig, *, check_finite: bool | str = True) -> PooledMap:
    """P̄ = softmax(mean-pool(Q, b_q) · mean-pool(K, b_kv)ᵀ / √d) (masker.py:100-110).

    Any float dtype is accepted; q/k are read in their own dtype and everything after the
    load is float64.  Non-finite q/k raise ``FloatingPointError`` (numerics.py:29-32):
    immediately for numpy callers, deferred for torch callers (``numerics.finite_guard``).
    """
    qt, qb = to_device4(q, None, "q")
    kt, _ = to_device4(k, None, "k", device=qb.device)
    if qt.shape[-1] != kt.shape[-1]:
        raise ValueError(f"q/k feature dims differ: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    if qt.shape[:-1] != kt.shape[:-1]:
        raise ValueError(f"q/k token counts differ: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    if kt.dtype != qt.dtype:
        kt = kt.to(qt.dtype)
    flag = finite_guard.new_flag(qt.device) if check_finite else None
    probs = _pooled_probs(qt, kt, cfg.b_q, cfg.b_kv, flag)
    if flag is not None:
        finite_guard.submit(flag, "q or k", block=qb.numpy or check_finite == "sync", device=qt.device)
    if qb.rank == 2:
        probs = probs[0, 0]
    if qb.numpy:
        return PooledMap._trusted(_readonly(probs.cpu().numpy()), cfg.b_q, cfg.b_kv, qt.shape[2], dev=probs)
    return PooledMap._trusted(probs, cfg.b_q, cfg.b_kv, qt.shape[2])


def _pooled_probs(qt: torch.Tensor, kt: torch.Tensor, b_q: int, b_kv: int, flag: torch.Tensor | None,
                  softmax: bool = True) -> torch.Tensor:
    """Launch K1 on [B,H,N,d] tensors; returns probs [B,H,T_m,T_n] float64.  ``flag`` (int32[1]
    or None) is OR-ed with "q or k has a non-finite entry".  ``softmax=False`` returns the
    pre-softmax scores Q̄K̄ᵀ/√d (for spa2_select_scores)."""
    B, H, N, d = qt.shape
    t_m, t_n = num_blocks(N, b_q), num_blocks(N, b_kv)
    probs = torch.empty((B, H, t_m, t_n), device=qt.device, dtype=torch.float64)
    work = torch.empty((B * H * (t_m + t_n) * d,), device=qt.device, dtype=torch.float64)
    st = torch.cuda.current_stream(qt.device)
    _lib.call("spa2_pooled_map" if softmax else "spa2_pooled_scores", _lib.view4(qt), _lib.view4(kt),
              _lib.DTYPE_CODES[qt.dtype], B, H, N, d, b_q, b_kv, _lib.ptr(probs), _lib.ptr(work), _lib.ptr(flag),
              st.cuda_stream, stream_obj=st)
    return probs


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


def _mask_from(pm: PooledMap, k_count: int, p_frac: float | None) -> BlockMask:
    keep, _ = _select(pm.dev, k_count, p_frac)
    return BlockMask._from_device(keep, pm.b_q, pm.b_kv, pm.n_tokens, host=pm.on_host)


def top_k_mask(pm: PooledMap, k_frac: float) -> BlockMask:
    """Keep the K largest entries per row, ties to the lower column (masker.py:122-128)."""
    return _mask_from(pm, top_k_count(k_frac, pm.probs.shape[-1]), None)


def top_p_mask(pm: PooledMap, p_frac: float) -> BlockMask:
    """Keep the shortest descending prefix reaching p_frac (masker.py:137-142)."""
    return _mask_from(pm, 1, p_frac)


def hybrid_mask(pm: PooledMap, cfg: SparsityConfig) -> BlockMask:
    """Top-k ∪ Top-p (masker.py:145-146), computed in one pass: both rules keep a prefix
    of the same stable order, so the union is its first max(K, cnt_p) columns."""
    return _mask_from(pm, top_k_count(cfg.k_frac, pm.probs.shape[-1]), cfg.p_frac)


def expand_mask(bm: BlockMask):
    """Token-level 0/1 float64 matrix, entry (a, b) = keep[a // b_q, b // b_kv]
    (masker.py:149-153).  Materialises N×N — tests and analysis only.  numpy for host
    masks (the reference's type), a CUDA tensor for device masks."""
    n = bm.n_tokens
    if bm.on_host:
        full = np.repeat(np.repeat(bm.keep, bm.b_q, axis=0), bm.b_kv, axis=1)
        return full[:n, :n].astype(np.float64)
    full = bm.keep.repeat_interleave(bm.b_q, dim=-2).repeat_interleave(bm.b_kv, dim=-1)
    return full[..., :n, :n].to(torch.float64)


# --------------------------------------------------------------------------------------
# serialisation (masker.py:159-186; writers byte-identical, see formats.py)
# --------------------------------------------------------------------------------------

def write_mask_csv(path, bm: BlockMask) -> None:
    from . import formats

    formats.write_mask_csv(path, bm)


def read_mask_csv(path) -> BlockMask:
    from . import formats

    keep, b_q, b_kv, n_tokens = formats.read_mask_csv(path)
    return BlockMask(keep, b_q=b_q, b_kv=b_kv, n_tokens=n_tokens)


def write_pooled_map_csv(path, pm: PooledMap) -> None:
    from . import formats

    formats.write_pooled_map_csv(path, pm)


__all__ = [
    "P_SLACK", "SparsityConfig", "PooledMap", "BlockMask", "pooled_map", "top_k_count", "top_k_mask",
    "top_p_mask", "hybrid_mask", "expand_mask", "write_mask_csv", "read_mask_csv",
    "write_pooled_map_csv",
]

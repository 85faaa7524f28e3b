"""Mask-quality measurements on the GPU at Wan sizes, without N×N materialisation
(SURVEY.md §8f row 3).

The reference measures mask quality with dense token-level matrices:

* retained mass τ of a query row = Σ_kept p (flowmatch._attn_stats / measure_tau_bar,
  flowmatch.py:408-434: ``(softmax(q kᵀ/√d) * expand_mask(bm)).sum(axis=1)``), and its mean
  τ̄; the mask-analyze report's block-level τ̄ (cli.py:147-150: ``(pm.probs * bm.keep)``);
* the exact error decomposition of one row (analysis.error_decompose, analysis.py:37-65)
  o − o_s = dropped + renorm with dropped = (p ∘ (1−m)) V, renorm = (1 − 1/τ)(p ∘ m) V, and
  the relative L1 aggregate Σ|o − o_s| / Σ|o| (analysis.relative_l1, analysis.py:192-200).

Here every quantity comes from two passes of the attention kernels — the sparse forward
(mask bm) and the dense forward (all blocks) — using only row statistics:

    τ      = exp(LSE_sparse − LSE_dense)      (LSE = log Σ exp over the kept / all keys)
    o_s    = sparse output,  o = dense output,  (p ∘ m) V = τ · o_s
    dropped = o − τ · o_s,   renorm = (τ − 1) · o_s,   dropped + renorm = o − o_s

so the cost is one dense and one sparse forward (O(N² d) tensor work, O(N d) memory).
Inputs are computed in bf16 (as the operator is); the terms carry the outputs' bf16
rounding (~2⁻⁸ relative), far below typical 95 %-sparsity errors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import attention as at
from .masker import BlockMask, PooledMap
from .numerics import from_device, to_device4


@dataclass(frozen=True)
class QualityReport:
    """Row-wise decomposition for every query row (analysis.ErrorReport, for all rows at once)."""

    tau: object           # [.., N] retained mass per query row
    dropped_term: object  # [.., N, d]
    renorm_term: object   # [.., N, d]
    total_error: object   # [.., N, d] = o − o_s
    aggregate: float      # Σ|o − o_s| / Σ|o|  (relative L1, analysis.py:192-200)
    tau_bar: float        # mean τ over all rows (flowmatch.py:434)


def _forwards(q, k, v, bm: BlockMask):
    q4, qb = to_device4(q, torch.bfloat16, "q")
    k4, _ = to_device4(k, torch.bfloat16, "k", device=qb.device)
    v4, _ = to_device4(v, torch.bfloat16, "v", device=qb.device)
    if not (q4.shape == k4.shape == v4.shape):
        raise ValueError(f"q/k/v shapes differ: {tuple(q4.shape)}, {tuple(k4.shape)}, {tuple(v4.shape)}")
    at._check_kernel_shape(q4)
    q4, k4, v4 = (at._tma_ready(t) for t in (q4, k4, v4))
    B, H, N, d = q4.shape
    if bm.n_tokens != N:
        raise ValueError(f"mask built for {bm.n_tokens} tokens, inputs have {N}")
    scale = 1.0 / math.sqrt(d)
    with torch.no_grad():
        o_s, lse_s = at.fwd(q4, k4, v4, at.mask_lists(bm, B, H, N), scale)
        o, lse = at.fwd(q4, k4, v4, at.mask_lists(at.full_mask(N), B, H, N), scale)
    return o_s, lse_s, o, lse, qb


def retained_mass(q, k, v, bm: BlockMask):
    """τ per query row: the softmax mass the mask keeps (flowmatch.py:408-434), from the
    sparse and dense log-sum-exps.  Returns [N] (or [B, H, N]) like the inputs' container."""
    _, lse_s, _, lse, qb = _forwards(q, k, v, bm)
    return from_device(torch.exp(lse_s.double() - lse.double()), qb, 1)


def tau_bar(q, k, v, bm: BlockMask) -> float:
    """Mean retained mass over all query rows (flowmatch.measure_tau_bar's statistic)."""
    _, lse_s, _, lse, _ = _forwards(q, k, v, bm)
    return float(torch.exp(lse_s.double() - lse.double()).mean())


def pooled_tau_bar(pm: PooledMap, bm: BlockMask) -> float:
    """Block-level retained mass of the mask-analyze report: mean over block rows of
    Σ_j P̄_ij keep_ij (cli.py:147-150), on the device."""
    return float((pm.dev * bm.dev.to(torch.float64)).sum(dim=-1).mean())


def error_decomposition(q, k, v, bm: BlockMask) -> QualityReport:
    """analysis.error_decompose (analysis.py:37-65) for every query row at once, plus the
    relative-L1 aggregate; o and o_s from the dense and sparse forward kernels."""
    o_s, lse_s, o, lse, qb = _forwards(q, k, v, bm)
    tau = torch.exp(lse_s.double() - lse.double())  # [B, H, N]
    os_, od = o_s.double(), o.double()
    kept_v = tau[..., None] * os_          # (p ∘ m) V
    dropped = od - kept_v                  # (p ∘ (1 − m)) V
    renorm = kept_v - os_                  # (1 − 1/τ)(p ∘ m) V
    total = dropped + renorm               # = o − o_s
    aggregate = float((od - os_).abs().sum() / od.abs().sum())
    return QualityReport(tau=from_device(tau, qb, 1), dropped_term=from_device(dropped, qb),
                         renorm_term=from_device(renorm, qb), total_error=from_device(total, qb),
                         aggregate=aggregate, tau_bar=float(tau.mean()))


__all__ = ["QualityReport", "retained_mass", "tau_bar", "pooled_tau_bar", "error_decomposition"]

"""float64 restatement of the reference block masker — TEST INFRASTRUCTURE ONLY.

Reference: ``sparseattn_lab/masker.py`` and ``sparseattn_lab/numerics.py``
(``/root/reference/pkg/src``).  Only tests, ``smoke()`` and bench's CPU legs use it.

The reference builds Top-k and Top-p masks with separate per-row loops and ORs them
(masker.py:122-146).  Both rules keep a prefix of the *same* stable descending order
(masker.py:113-115), so the hybrid mask is the first ``max(K, cnt_p)`` columns of
that order.  This module exposes the counts explicitly (``select_counts``) because
that is exactly the quantity the GPU select kernel computes; the keep matrices are
then rebuilt from the shared order.  ``tests/test_oracle.py`` pins every function
here against goldens produced by the reference itself.
"""

from __future__ import annotations

import math

import numpy as np

# masker.py:27 — slack subtracted from p_frac before the prefix search
P_SLACK = 1e-12


def block_mean_pool(x: np.ndarray, block: int) -> np.ndarray:
    """Means of consecutive ``block``-row groups; the ragged tail group is divided
    by its true row count (numerics.py:55-65, ``np.add.reduceat`` + true counts)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if block < 1:
        raise ValueError(f"block must be >= 1, got {block}")
    n = x.shape[0]
    starts = np.arange(0, n, block)
    group_sums = np.add.reduceat(x, starts, axis=0)
    group_sizes = np.minimum(starts + block, n) - starts
    return group_sums / group_sizes[:, None]


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """Row softmax with max subtraction (numerics.py:46-52)."""
    shifted = x - x.max(axis=1, keepdims=True)
    e = np.exp(shifted)
    return e / e.sum(axis=1, keepdims=True)


def pooled_probs(q: np.ndarray, k: np.ndarray, b_q: int, b_kv: int) -> np.ndarray:
    """Row-stochastic pooled map P̄ = softmax(Q̄ K̄ᵀ / √d) (masker.py:100-110)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    if q.shape != k.shape:
        raise ValueError(f"q/k shapes differ: {q.shape} vs {k.shape}")
    q_bar = block_mean_pool(q, b_q)
    k_bar = block_mean_pool(k, b_kv)
    return softmax_rows((q_bar @ k_bar.T) / math.sqrt(q.shape[1]))


def descending_order(row: np.ndarray) -> np.ndarray:
    """Stable argsort of the negated row: larger first, ties to the lower column
    (masker.py:113-115)."""
    return np.argsort(-row, kind="stable")


def top_k_count(k_frac: float, t_n: int) -> int:
    """K = max(1, ceil(k_frac * T_n)) in IEEE double (masker.py:118-119)."""
    return max(1, math.ceil(k_frac * t_n))


def top_p_count(row: np.ndarray, p_frac: float) -> int:
    """Length of the shortest descending prefix whose sequential float64 running sum
    reaches ``p_frac - P_SLACK``: ``searchsorted(cumsum, thr, 'left') + 1``
    (masker.py:131-134).  Not capped here; callers cap at T_n (masker.py:141)."""
    running = np.cumsum(row[descending_order(row)])
    return int(np.searchsorted(running, p_frac - P_SLACK, side="left")) + 1


def select_counts(probs: np.ndarray, k_frac: float | None, p_frac: float | None) -> np.ndarray:
    """Per-row kept-block count of the hybrid rule; ``None`` disables a rule.

    top-k only  -> K;  top-p only -> min(cnt_p, T_n);  hybrid -> min(max(K, cnt_p), T_n).
    """
    probs = np.ascontiguousarray(probs, dtype=np.float64)
    t_n = probs.shape[1]
    kk = top_k_count(k_frac, t_n) if k_frac is not None else 1
    out = np.empty(probs.shape[0], dtype=np.int64)
    for r, row in enumerate(probs):
        cnt = top_p_count(row, p_frac) if p_frac is not None else 1
        out[r] = min(max(kk, cnt), t_n)
    return out


def _keep_from_counts(probs: np.ndarray, counts: np.ndarray) -> np.ndarray:
    keep = np.zeros(probs.shape, dtype=bool)
    for r, row in enumerate(probs):
        keep[r, descending_order(row)[: counts[r]]] = True
    return keep


def top_k_keep(probs: np.ndarray, k_frac: float) -> np.ndarray:
    """Top-k keep matrix (masker.py:122-128)."""
    return _keep_from_counts(probs, select_counts(probs, k_frac, None))


def top_p_keep(probs: np.ndarray, p_frac: float) -> np.ndarray:
    """Top-p keep matrix (masker.py:137-142)."""
    return _keep_from_counts(probs, select_counts(probs, None, p_frac))


def hybrid_keep(probs: np.ndarray, k_frac: float, p_frac: float) -> np.ndarray:
    """Hybrid keep matrix = Top-k OR Top-p (masker.py:145-146), built from the shared
    descending order."""
    return _keep_from_counts(probs, select_counts(probs, k_frac, p_frac))

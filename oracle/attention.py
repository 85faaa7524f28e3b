"""float64 restatement of the reference attention kernels — TEST INFRASTRUCTURE ONLY.

Reference: ``sparseattn_lab/attention.py`` (``/root/reference/pkg/src``).  Used by
tests as the checker and by ``bench.py`` as the timed CPU baseline (kind "port");
never by the product package.

All functions are single-head: q, k, v are [N, d]; ``keep`` is the [T_m, T_n] block
keep matrix for block sizes (b_q, b_kv).
"""

from __future__ import annotations

import math

import numpy as np

# oracles.py:17 stands in -1e30 for -inf in its token-level loop; we do the same.
_MASKED = -1e30


def _f64(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def dense_attention(q, k, v):
    """Materialised softmax attention with LSE (attention.py:62-70)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    s = (q @ k.T) / math.sqrt(q.shape[1])
    m = s.max(axis=1)
    e = np.exp(s - m[:, None])
    z = e.sum(axis=1)
    return (e / z[:, None]) @ v, m + np.log(z)


def sparse_forward(q, k, v, keep, b_q: int, b_kv: int, visit=None):
    """Tiled online-softmax forward over kept blocks (attention.py:73-114).

    For every query block i the kept key blocks are visited in ascending j (or in the
    order returned by ``visit(i, kept)``, the reference's ``_block_order`` hook,
    attention.py:97-99).  Running state per row: max ``m``, normaliser ``z`` and the
    unnormalised accumulator; ``lse = m + ln z`` (attention.py:112-113).
    Returns (out [N,d], lse [N], visited_blocks).
    """
    q, k, v = _f64(q), _f64(k), _f64(v)
    keep = np.asarray(keep, dtype=bool)
    n, d = q.shape
    n_kv = k.shape[0]  # == n for the reference contract; bench samples pass a q slice
    scale = 1.0 / math.sqrt(d)
    out = np.empty((n, v.shape[1]))
    lse = np.empty(n)
    visited = 0
    for i in range(keep.shape[0]):
        rows = slice(i * b_q, min((i + 1) * b_q, n))
        qi = q[rows]
        m = np.full(qi.shape[0], -np.inf)
        z = np.zeros(qi.shape[0])
        acc = np.zeros((qi.shape[0], v.shape[1]))
        cols = np.flatnonzero(keep[i])
        if visit is not None:
            cols = visit(i, cols)
        for j in cols:
            kv = slice(j * b_kv, min((j + 1) * b_kv, n_kv))
            visited += 1
            s = (qi @ k[kv].T) * scale
            m_next = np.maximum(m, s.max(axis=1))
            decay = np.exp(m - m_next)  # exp(-inf) == 0 on the first visited block
            p = np.exp(s - m_next[:, None])
            z = decay * z + p.sum(axis=1)
            acc = decay[:, None] * acc + p @ v[kv]
            m = m_next
        out[rows] = acc / z[:, None]
        lse[rows] = m + np.log(z)
    return out, lse, visited


def attention_backward(q, k, v, keep, b_q: int, b_kv: int, d_out):
    """Gradients with the mask held constant (attention.py:128-166).

    The forward is recomputed for ``out``/``lse`` (attention.py:140); then per kept
    (i, j): P = exp(S*scale - lse), dV += Pᵀ dO, dS = P ∘ (dO Vᵀ - δ),
    dQ += dS K * scale, dK += dSᵀ Q * scale, with δ = rowsum(dO ∘ O) (attention.py:149).
    Dropped blocks contribute exactly zero.
    Returns (dq, dk, dv, out, lse).
    """
    q, k, v, d_out = _f64(q), _f64(k), _f64(v), _f64(d_out)
    keep = np.asarray(keep, dtype=bool)
    out, lse, _ = sparse_forward(q, k, v, keep, b_q, b_kv)
    n, d = q.shape
    n_kv = k.shape[0]
    scale = 1.0 / math.sqrt(d)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    delta = (d_out * out).sum(axis=1)
    for i in range(keep.shape[0]):
        rows = slice(i * b_q, min((i + 1) * b_q, n))
        qi, doi = q[rows], d_out[rows]
        for j in np.flatnonzero(keep[i]):
            kv = slice(j * b_kv, min((j + 1) * b_kv, n_kv))
            p = np.exp((qi @ k[kv].T) * scale - lse[rows][:, None])
            dv[kv] += p.T @ doi
            ds = p * (doi @ v[kv].T - delta[rows][:, None])
            dq[rows] += (ds @ k[kv]) * scale
            dk[kv] += (ds.T @ qi) * scale
    return dq, dk, dv, out, lse


def masked_attention_tokens(q, k, v, token_keep):
    """Token-level masked softmax attention, an independent check of the tiled kernel
    (oracles.py:36-54, written as one vectorised pass instead of explicit loops)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    token_keep = np.asarray(token_keep) != 0
    if not token_keep.any(axis=1).all():
        raise ValueError("a query row keeps no key")
    s = np.where(token_keep, (q @ k.T) / math.sqrt(q.shape[1]), _MASKED)
    e = np.exp(s - s.max(axis=1, keepdims=True))
    return (e / e.sum(axis=1, keepdims=True)) @ v


def expand_keep(keep, b_q: int, b_kv: int, n: int) -> np.ndarray:
    """Token-level 0/1 matrix of a block mask (masker.py:149-153)."""
    keep = np.asarray(keep, dtype=bool)
    return np.repeat(np.repeat(keep, b_q, axis=0), b_kv, axis=1)[:n, :n].astype(np.float64)

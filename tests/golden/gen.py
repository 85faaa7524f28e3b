"""Seeded numpy input generators shared by ``make_golden.py`` and the tests.

Inputs are drawn with PCG64 (numpy guarantees a bit-identical stream per seed) and
rounded to bfloat16 (round-to-nearest-even), because the GPU path computes on bf16
operands.  The reference is then run on the *same* bf16 values up-cast to float64,
so any output difference is the GPU's arithmetic, not input rounding.

``wan_like`` adds a per-block shared offset of scale ``s`` to q and k, which makes
the pooled map peaked the way real video-DiT attention is: with
s = 0 the hybrid rule only reaches ~80 % sparsity, with s ≈ 0.9 it reaches ~95 %.
"""

from __future__ import annotations

import hashlib

import numpy as np


def to_bf16(x: np.ndarray) -> np.ndarray:
    """Round float64 → bfloat16 (RNE) and return the exact value as float64."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of values that are already bf16-representable."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def wan_like(seed: int, n: int, d: int, b_q: int, b_kv: int, s: float, heads: int = 1):
    """q, k, v, d_out of shape [heads, n, d] (bf16-representable float64)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    t_m, t_n = -(-n // b_q), -(-n // b_kv)
    out = []
    for _ in range(heads):
        q = rng.normal(size=(n, d))
        k = rng.normal(size=(n, d))
        v = rng.normal(size=(n, d))
        do = rng.normal(size=(n, d))
        if s > 0:
            q = q + np.repeat(rng.normal(size=(t_m, d)) * s, b_q, axis=0)[:n]
            k = k + np.repeat(rng.normal(size=(t_n, d)) * s, b_kv, axis=0)[:n]
        out.append([to_bf16(t) for t in (q, k, v, do)])
    return [np.stack([h[i] for h in out]) for i in range(4)]


def random_keep(seed: int, t_m: int, t_n: int, density: float) -> np.ndarray:
    """Random block mask with at least one kept block per row (test_attention.py:261-266)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    keep = rng.random((t_m, t_n)) < density
    keep[~keep.any(axis=1), 0] = True
    return keep

"""Synthetic Wan2.1-shaped q/k/v generated directly on the GPU (benchmarks and tests).

There is no network for real activations, so inputs are i.i.d. N(0, 1) plus a per-block
shared offset N(0, s²) added to every b_q-row block of q and every b_kv-row block of k.
The offset makes the pooled map peaked like real video-DiT attention: at the
Wan2.1-1.3B shape s ≈ 0.9 with k = 0.03, p = 0.2 lands at ≈ 95 % block sparsity
(pure i.i.d. inputs only reach ≈ 80 %).
"""

from __future__ import annotations

import torch


def wan_like_qkv(B: int, H: int, N: int, d: int, s: float, seed: int = 0, b_q: int = 128, b_kv: int = 64,
                 device="cuda", dtype=torch.bfloat16):
    g = torch.Generator(device=device).manual_seed(seed)
    t_m, t_n = -(-N // b_q), -(-N // b_kv)

    def one(blocks, bsize):
        x = torch.randn(B, H, N, d, device=device, generator=g, dtype=torch.float32)
        if s > 0:
            off = torch.randn(B, H, blocks, d, device=device, generator=g, dtype=torch.float32) * s
            x += off.repeat_interleave(bsize, dim=2)[:, :, :N]
        return x.to(dtype)

    q = one(t_m, b_q)
    k = one(t_n, b_kv)
    v = torch.randn(B, H, N, d, device=device, generator=g, dtype=torch.float32).to(dtype)
    return q, k, v

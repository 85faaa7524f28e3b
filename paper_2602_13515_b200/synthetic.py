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


def latent_grid(N: int) -> tuple[int, int, int]:
    """(frames, rows, cols) of a video latent with N tokens: Wan2.1 480p / 81 frames is
    21 x 30 x 52 = 32760 and 720p is 21 x 45 x 80 = 75600; other N use 21 frames of a
    near-16:9 grid (the last frame is truncated)."""
    for grid in ((21, 30, 52), (21, 45, 80)):
        if grid[0] * grid[1] * grid[2] == N:
            return grid
    per = -(-N // 21)
    rows = max(1, int(round((per * 9 / 16) ** 0.5)))
    return 21, rows, -(-per // rows)


def video_like_qkv(B: int, H: int, N: int, d: int, s: float = 2.5, seed: int = 0, modes: int = 24,
                   device="cuda", dtype=torch.bfloat16):
    """Spatio-temporally CORRELATED synthetic q/k/v: i.i.d. N(0, 1) plus s times a smooth
    random feature field over the latent (frame, row, col) grid (a sum of `modes` random
    low-frequency Fourier modes, wavelengths ~ 6-8 latent cells), shared by q and k of a
    head.  Tokens attend to spatially / temporally nearby tokens, as in real video-DiT
    attention, so neighbouring key blocks tend to be kept together — unlike `wan_like_qkv`,
    whose per-block offsets make every mask row independent.  s = 2.5 gives ~95 % block
    sparsity at the Wan2.1-1.3B shape with k = 0.03, p = 0.2 (calibrated with the oracle)."""
    g = torch.Generator(device=device).manual_seed(seed)
    F, R, C = latent_grid(N)
    n = torch.arange(N, device=device)
    pos = torch.stack([n // (R * C), (n // C) % R, n % C], dim=1).to(torch.float32)  # [N, 3]
    scale = torch.tensor([6.0, 8.0, 8.0], device=device)
    x = torch.empty(B, H, N, d, device=device, dtype=torch.float32)
    out = []
    for which in range(3):
        x.normal_(generator=g)
        out.append(x.clone())
    q, k, v = out
    for b in range(B):
        for h in range(H):
            kvec = torch.randn(modes, 3, device=device, generator=g) / scale  # cycles per cell
            phase = torch.rand(modes, device=device, generator=g) * (2 * torch.pi)
            amp = torch.randn(modes, d, device=device, generator=g)
            waves = torch.cos(2 * torch.pi * pos @ kvec.T + phase)  # [N, modes]
            field = (waves @ amp) * (s / modes ** 0.5)
            q[b, h] += field
            k[b, h] += field
    return q.to(dtype), k.to(dtype), v.to(dtype)

"""Config 5: one sparse-attention distillation step on a Wan2.1-style DiT.

The reference's Algorithm 2 (``flowmatch.train_vd``, flowmatch.py:506-519, with the loss
``vd_loss`` flowmatch.py:354-367 and the shared loop ``_run_training`` 454-497): clone the
dense teacher, swap the student's self-attention for sparse attention, and fit the
student's velocity prediction to the frozen teacher's on the same noisy input; the gradient
of the mean squared difference drives an Adam step.  Here the model is a Wan2.1-style video
DiT (the reference only ships a toy denoiser; ``SPEC.md:9`` excludes Wan2.1, so the
architecture constants below are the public Wan2.1-1.3B values, random-initialised) and the
student's self-attention is this package's ``sparse_attention`` (tcgen05 kernels, autograd);
the teacher runs dense attention (cuDNN SDPA).

This is a caller of the hot path, not part of it: plain PyTorch modules around the operator.
"""

from __future__ import annotations

import copy
import math
from dataclasses import dataclass

import torch
import torch.nn as nn
import torch.nn.functional as F

from .attention import sparse_attention
from .masker import SparsityConfig


@dataclass(frozen=True)
class WanConfig:
    """Wan2.1 text-to-video DiT sizes (1.3B: dim 1536, 30 layers, 12 heads of 128)."""

    dim: int = 1536
    ffn_dim: int = 8960
    heads: int = 12
    layers: int = 30
    in_channels: int = 16
    patch: tuple[int, int, int] = (1, 2, 2)
    text_len: int = 512
    text_dim: int = 4096
    freq_dim: int = 256
    eps: float = 1e-6

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


WAN_1_3B = WanConfig()
# 480p, 81 frames: latent 21 x 60 x 104 -> patch (1, 2, 2) -> 21 * 30 * 52 = 32760 tokens
WAN_480P_LATENT = (21, 60, 104)


class RMSNorm(nn.Module):
    def __init__(self, dim: int, eps: float):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(dim))

    def forward(self, x):
        return F.rms_norm(x, (x.shape[-1],), self.weight, self.eps)


def rope_freqs(head_dim: int, grid: tuple[int, int, int], device) -> torch.Tensor:
    """3-D rotary angles: the head dim is split between frame / height / width axes
    (Wan: d - 4(d//6), 2(d//6), 2(d//6) channels).  Returns complex [N, head_dim // 2]."""
    f, h, w = grid
    c = head_dim // 2
    parts = [c - 2 * (c // 3), c // 3, c // 3]
    axes = []
    for size, n in zip((f, h, w), parts):
        inv = 1.0 / (10000 ** (torch.arange(n, device=device, dtype=torch.float64) / n))
        axes.append(torch.outer(torch.arange(size, device=device, dtype=torch.float64), inv))
    ff = axes[0][:, None, None, :].expand(f, h, w, parts[0])
    hh = axes[1][None, :, None, :].expand(f, h, w, parts[1])
    ww = axes[2][None, None, :, :].expand(f, h, w, parts[2])
    ang = torch.cat([ff, hh, ww], dim=-1).reshape(f * h * w, c)
    return torch.polar(torch.ones_like(ang), ang).to(torch.complex64)


def apply_rope(x: torch.Tensor, freqs: torch.Tensor) -> torch.Tensor:
    """x [B, N, H, d] real -> rotated pairs (interleaved as Wan)."""
    xc = torch.view_as_complex(x.float().reshape(*x.shape[:-1], -1, 2))
    return torch.view_as_real(xc * freqs[None, :, None, :]).flatten(-2).to(x.dtype)


class SelfAttention(nn.Module):
    def __init__(self, cfg: WanConfig):
        super().__init__()
        self.cfg = cfg
        self.qkv = nn.Linear(cfg.dim, 3 * cfg.dim)
        self.o = nn.Linear(cfg.dim, cfg.dim)
        self.norm_q = RMSNorm(cfg.dim, cfg.eps)
        self.norm_k = RMSNorm(cfg.dim, cfg.eps)
        self.sparse: SparsityConfig | None = None  # None: dense (teacher)

    def forward(self, x, freqs):
        B, N, _ = x.shape
        H, d = self.cfg.heads, self.cfg.head_dim
        q, k, v = self.qkv(x).chunk(3, dim=-1)
        q = apply_rope(self.norm_q(q).view(B, N, H, d), freqs)
        k = apply_rope(self.norm_k(k).view(B, N, H, d), freqs)
        v = v.view(B, N, H, d)
        if self.sparse is None:
            out = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2))
        else:
            # [B, N, H, d] passed as a [B, H, N, d] view: no copy, the kernels take strides
            out = sparse_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2), self.sparse).out
        return self.o(out.transpose(1, 2).reshape(B, N, H * d))


class CrossAttention(nn.Module):
    def __init__(self, cfg: WanConfig):
        super().__init__()
        self.cfg = cfg
        self.q = nn.Linear(cfg.dim, cfg.dim)
        self.kv = nn.Linear(cfg.dim, 2 * cfg.dim)
        self.o = nn.Linear(cfg.dim, cfg.dim)
        self.norm_q = RMSNorm(cfg.dim, cfg.eps)
        self.norm_k = RMSNorm(cfg.dim, cfg.eps)

    def forward(self, x, ctx):
        B, N, _ = x.shape
        H, d = self.cfg.heads, self.cfg.head_dim
        q = self.norm_q(self.q(x)).view(B, N, H, d).transpose(1, 2)
        k, v = self.kv(ctx).chunk(2, dim=-1)
        k = self.norm_k(k).view(B, -1, H, d).transpose(1, 2)
        v = v.view(B, -1, H, d).transpose(1, 2)
        out = F.scaled_dot_product_attention(q, k, v)
        return self.o(out.transpose(1, 2).reshape(B, N, H * d))


class DiTBlock(nn.Module):
    def __init__(self, cfg: WanConfig):
        super().__init__()
        self.norm1 = nn.LayerNorm(cfg.dim, eps=cfg.eps, elementwise_affine=False)
        self.attn = SelfAttention(cfg)
        self.norm3 = nn.LayerNorm(cfg.dim, eps=cfg.eps)
        self.cross = CrossAttention(cfg)
        self.norm2 = nn.LayerNorm(cfg.dim, eps=cfg.eps, elementwise_affine=False)
        self.ffn = nn.Sequential(nn.Linear(cfg.dim, cfg.ffn_dim), nn.GELU(approximate="tanh"),
                                 nn.Linear(cfg.ffn_dim, cfg.dim))
        self.modulation = nn.Parameter(torch.randn(1, 6, cfg.dim) / cfg.dim**0.5)

    def forward(self, x, e, ctx, freqs):
        m = (self.modulation + e).chunk(6, dim=1)  # shift/scale/gate for attention and FFN
        x = x + m[2] * self.attn(self.norm1(x) * (1 + m[1]) + m[0], freqs)
        x = x + self.cross(self.norm3(x), ctx)
        x = x + m[5] * self.ffn(self.norm2(x) * (1 + m[4]) + m[3])
        return x


class WanDiT(nn.Module):
    """Velocity predictor u(x_t, t, text) of a Wan2.1-style DiT (flow matching)."""

    def __init__(self, cfg: WanConfig = WAN_1_3B):
        super().__init__()
        self.cfg = cfg
        pc = cfg.in_channels * math.prod(cfg.patch)
        self.patch_in = nn.Linear(pc, cfg.dim)
        self.text_in = nn.Sequential(nn.Linear(cfg.text_dim, cfg.dim), nn.GELU(approximate="tanh"),
                                     nn.Linear(cfg.dim, cfg.dim))
        self.time_in = nn.Sequential(nn.Linear(cfg.freq_dim, cfg.dim), nn.SiLU(), nn.Linear(cfg.dim, cfg.dim))
        self.time_proj = nn.Sequential(nn.SiLU(), nn.Linear(cfg.dim, 6 * cfg.dim))
        self.blocks = nn.ModuleList([DiTBlock(cfg) for _ in range(cfg.layers)])
        self.head_norm = nn.LayerNorm(cfg.dim, eps=cfg.eps, elementwise_affine=False)
        self.head_mod = nn.Parameter(torch.randn(1, 2, cfg.dim) / cfg.dim**0.5)
        self.head = nn.Linear(cfg.dim, pc)

    def set_attention(self, sparse: SparsityConfig | None) -> None:
        """None: dense self-attention (teacher); a SparsityConfig: the sparse operator."""
        for b in self.blocks:
            b.attn.sparse = sparse

    def forward(self, latent, t, text):
        """latent [B, C, F, H, W], t [B] in [0, 1], text [B, L, text_dim] -> velocity like latent."""
        cfg = self.cfg
        B, C, Fr, Hh, Ww = latent.shape
        pf, ph, pw = cfg.patch
        grid = (Fr // pf, Hh // ph, Ww // pw)
        x = latent.view(B, C, grid[0], pf, grid[1], ph, grid[2], pw).permute(0, 2, 4, 6, 1, 3, 5, 7)
        x = self.patch_in(x.reshape(B, -1, C * pf * ph * pw))
        half = cfg.freq_dim // 2
        fr = torch.exp(-math.log(10000) * torch.arange(half, device=t.device, dtype=torch.float32) / half)
        emb = torch.cat([torch.cos(t[:, None].float() * 1000 * fr), torch.sin(t[:, None].float() * 1000 * fr)], -1)
        temb = self.time_in(emb.to(x.dtype))
        e = self.time_proj(temb).view(B, 6, cfg.dim)
        ctx = self.text_in(text)
        freqs = rope_freqs(cfg.head_dim, grid, latent.device)
        for blk in self.blocks:
            x = blk(x, e, ctx, freqs)
        shift, scale = (self.head_mod + temb[:, None]).chunk(2, dim=1)
        x = self.head(self.head_norm(x) * (1 + scale) + shift)
        x = x.view(B, *grid, C, pf, ph, pw).permute(0, 4, 1, 5, 2, 6, 3, 7)
        return x.reshape(B, C, Fr, Hh, Ww)


def make_student(teacher: WanDiT, cfg: SparsityConfig) -> WanDiT:
    """train_vd's clone-and-swap (flowmatch.py:513-514): same weights, sparse self-attention."""
    student = copy.deepcopy(teacher)
    student.set_attention(cfg)
    for p in student.parameters():
        p.requires_grad_(True)
    return student


def distill_step(student: WanDiT, teacher: WanDiT, opt: torch.optim.Optimizer, latent, t, text) -> torch.Tensor:
    """One step of Algorithm 2: x_t is shared, the teacher is frozen and dense, the loss is
    the mean squared velocity difference (vd_loss, flowmatch.py:354-367)."""
    with torch.no_grad():
        u_t = teacher(latent, t, text)
    u_s = student(latent, t, text)
    loss = F.mse_loss(u_s.float(), u_t.float())
    opt.zero_grad(set_to_none=True)
    loss.backward()
    opt.step()
    return loss.detach()


def synthetic_batch(cfg: WanConfig, latent_shape=WAN_480P_LATENT, batch: int = 1, seed: int = 0,
                    device="cuda", dtype=torch.bfloat16):
    """Flow-matching draw x_t = (1 - t) x0 + t ε on random latents and random text features."""
    g = torch.Generator(device=device).manual_seed(seed)
    x0 = torch.randn((batch, cfg.in_channels, *latent_shape), generator=g, device=device)
    eps = torch.randn(x0.shape, generator=g, device=device)
    t = torch.rand((batch,), generator=g, device=device)
    x_t = ((1 - t.view(-1, 1, 1, 1, 1)) * x0 + t.view(-1, 1, 1, 1, 1) * eps).to(dtype)
    text = torch.randn((batch, cfg.text_len, cfg.text_dim), generator=g, device=device).to(dtype)
    return x_t, t, text

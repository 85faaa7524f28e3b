"""Config 5 building blocks on the GPU: the Wan-style DiT with the sparse operator as its
self-attention (distill.py) — keep-everything sparse student == dense teacher, and one
Algorithm-2 step (flowmatch.train_vd) runs with finite loss and gradients."""

import pytest
import torch

import paper_2602_13515_b200 as spa
from paper_2602_13515_b200 import distill as ds

pytestmark = pytest.mark.gpu
TINY = ds.WanConfig(dim=256, ffn_dim=512, heads=2, layers=2, text_len=16, text_dim=64, freq_dim=32)
LATENT = (4, 16, 32)  # -> 4 * 8 * 16 = 512 tokens, head dim 128


def _models():
    torch.manual_seed(0)
    teacher = ds.WanDiT(TINY).cuda().to(torch.bfloat16)
    teacher.set_attention(None)
    return teacher


def test_keep_all_student_matches_dense_teacher():
    teacher = _models()
    student = ds.make_student(teacher, spa.SparsityConfig(1.0, 1.0, 128, 64))
    x_t, t, text = ds.synthetic_batch(TINY, LATENT, seed=1)
    with torch.no_grad():
        u_t = teacher(x_t, t, text).float()
        u_s = student(x_t, t, text).float()
    cos = torch.nn.functional.cosine_similarity(u_s.flatten(), u_t.flatten(), dim=0).item()
    assert cos > 0.999, cos


def test_distill_step_runs_and_updates_student():
    teacher = _models()
    for p in teacher.parameters():
        p.requires_grad_(False)
    student = ds.make_student(teacher, spa.SparsityConfig(0.25, 0.3, 128, 64))
    opt = torch.optim.AdamW(student.parameters(), lr=1e-3)
    x_t, t, text = ds.synthetic_batch(TINY, LATENT, seed=2)
    w0 = student.blocks[0].attn.qkv.weight.detach().clone()
    loss = ds.distill_step(student, teacher, opt, x_t, t, text)
    assert torch.isfinite(loss)
    g = student.blocks[0].attn.qkv.weight
    assert not torch.equal(w0, g.detach())  # the sparse operator's gradients reached q/k/v

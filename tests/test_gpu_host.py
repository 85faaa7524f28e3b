"""HostPipeline (host-buffer entry point used by bench.py's e2e leg): results equal the
device path bit for bit, including back-to-back calls whose copy-in overlaps the previous
call's copy-out."""

import pytest
import torch

import paper_2602_13515_b200 as spa
from paper_2602_13515_b200.host import HostPipeline
from paper_2602_13515_b200.synthetic import wan_like_qkv

pytestmark = pytest.mark.gpu


def _device_ref(q, k, v, do, cfg):
    qs, ks, vs = (t.clone().requires_grad_(True) for t in (q, k, v))
    res = spa.sparse_attention(qs, ks, vs, cfg, check_finite=False)
    res.out.backward(do)
    return [t.detach().cpu() for t in (res.out, qs.grad, ks.grad, vs.grad)]


@pytest.mark.parametrize("groups", [1, 3])
def test_host_pipeline_matches_device(groups):
    cfg = spa.SparsityConfig(0.1, 0.3, 128, 64)
    B, H, N, d = 1, 6, 2000, 128
    inputs = []
    for seed in (1, 2):
        q, k, v = wan_like_qkv(B, H, N, d, 0.9, seed=seed)
        do = torch.randn(q.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(seed)).to(q.dtype)
        inputs.append((q, k, v, do))
    refs = [_device_ref(*x, cfg) for x in inputs]
    pipe = HostPipeline(groups=groups)
    host_in = [[t.cpu().pin_memory() for t in x] for x in inputs]
    outs = [[torch.empty(B, H, N, d, dtype=torch.bfloat16).pin_memory() for _ in range(4)] for _ in inputs]
    for x, o in zip(host_in, outs):  # back to back, no sync in between
        pipe.fwd_bwd(*x, cfg, *o)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        for name, got, want in zip(("out", "dq", "dk", "dv"), o, r):
            assert torch.equal(got, want), name

"""Host-buffer entry point: fwd + bwd of the sparse-attention operator on tensors that live
in (pinned) host memory, with the PCIe transfers overlapped with the GPU compute.

A reference user calls the operator on host arrays (the reference is numpy,
attention.py:117-166).  Doing that naively serialises H2D of q/k/v/dO, the kernels, and
D2H of out/dq/dk/dv.  Here the heads are split into groups (every kernel's work lives
inside one head, so groups are independent problems) and three CUDA streams run a
software pipeline:

    copy-in  : H2D(group g+1)            (stream `h2d`)
    compute  : masker+fwd+bwd(group g)   (stream `comp`)
    copy-out : D2H(group g-1)            (stream `d2h`)

so the step approaches max(H2D, D2H, compute) instead of their sum.  Consecutive calls
pipeline too: the copy-in of call s+1 does not wait for the copy-out of call s (the two
directions of the link run concurrently), so a stream of calls is bound by
max(H2D, D2H, compute) per call.  Host inputs must already hold their data when the call
is made (written by the CPU or by completed copies); host outputs are valid once the
current stream (which waits for the copy-out) has been synchronised.
"""

from __future__ import annotations

import torch

from .attention import sparse_attention
from .masker import SparsityConfig


class HostPipeline:
    """Reusable streams + device buffers for repeated host-buffer fwd+bwd calls."""

    def __init__(self, device=None, groups: int = 4):
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.groups = groups
        self.h2d = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)

    def fwd_bwd(self, q, k, v, d_out, cfg: SparsityConfig, out=None, dq=None, dk=None, dv=None,
                check_finite: bool | str = True):
        """q, k, v, d_out: host tensors [B, H, N, d] (pinned for overlap).  Returns host
        (out, dq, dk, dv); pass preallocated pinned outputs to avoid allocations."""
        B, H, N, d = q.shape
        out = torch.empty_like(q, pin_memory=q.is_pinned()) if out is None else out
        dq = torch.empty_like(q, pin_memory=q.is_pinned()) if dq is None else dq
        dk = torch.empty_like(q, pin_memory=q.is_pinned()) if dk is None else dk
        dv = torch.empty_like(q, pin_memory=q.is_pinned()) if dv is None else dv
        G = max(1, min(self.groups, H))
        bounds = [(g * H // G, (g + 1) * H // G) for g in range(G)]
        main = torch.cuda.current_stream(self.device)
        # compute and copy-out follow the caller's stream; copy-in reads host memory only,
        # so it may run ahead of (and overlap) the previous call's copy-out
        for s in (self.comp, self.d2h):
            s.wait_stream(main)
        ev_in, ev_done = [], []
        dev_in = []
        with torch.cuda.stream(self.h2d):
            for h0, h1 in bounds:
                t = [x[:, h0:h1].to(self.device, non_blocking=True) for x in (q, k, v, d_out)]
                e = torch.cuda.Event()
                e.record(self.h2d)
                ev_in.append(e)
                dev_in.append(t)
        results = []
        for g, (h0, h1) in enumerate(bounds):
            self.comp.wait_event(ev_in[g])
            with torch.cuda.stream(self.comp):
                qg, kg, vg, dog = dev_in[g]
                for t in (qg, kg, vg, dog):
                    t.record_stream(self.comp)
                qs, ks, vs = (t.requires_grad_(True) for t in (qg, kg, vg))
                res = sparse_attention(qs, ks, vs, cfg, check_finite=check_finite)
                res.out.backward(dog)
                e = torch.cuda.Event()
                e.record(self.comp)
                ev_done.append(e)
                results.append((res.out.detach(), qs.grad, ks.grad, vs.grad))
            self.d2h.wait_event(ev_done[g])
            with torch.cuda.stream(self.d2h):
                for dst, src in zip((out, dq, dk, dv), results[g]):
                    src.record_stream(self.d2h)
                    dst[:, h0:h1].copy_(src, non_blocking=True)
        main.wait_stream(self.d2h)
        return out, dq, dk, dv

"""End-to-end (host-buffer) step time of HostPipeline.fwd_bwd at the bench shape for several
head-group counts, repeated windows, next to the PCIe duplex copy floor measured in between.

    python tools/e2e_sweep.py [groups ...]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200.host import HostPipeline  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

groups = [int(g) for g in sys.argv[1:]] or [3, 4, 6, 12]
dev = torch.device("cuda", 0)
q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
do = torch.randn(q.shape, device=dev).to(q.dtype)
cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, do))
outs = [torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(4)]
dev_bufs = [torch.empty_like(q) for _ in range(4)]
s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def duplex():
    s_in.wait_stream(torch.cuda.current_stream())
    s_out.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_in):
        for dst, src in zip(dev_bufs, (hq, hk, hv, hdo)):
            dst.copy_(src, non_blocking=True)
    with torch.cuda.stream(s_out):
        for dst, src in zip(outs, (q, k, v, do)):
            dst.copy_(src, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s_in)
    torch.cuda.current_stream().wait_stream(s_out)


host_ms = []
check = os.environ.get("E2E_CHECK_FINITE", "1") != "0"
for g in groups:
    pipe = HostPipeline(dev, groups=g)

    def step():
        t0 = time.perf_counter()
        pipe.fwd_bwd(hq, hk, hv, hdo, cfg, *outs, check_finite=check)
        host_ms.append(1e3 * (time.perf_counter() - t0))

    timed(step, 2)
    res = []
    for _ in range(4):
        res.append((timed(step, 20), timed(duplex, 5)))
    spa.check_pending()
    print(f"groups {g:2d}: e2e ms " + " ".join(f"{e:6.2f}" for e, _ in res) + "   pcie floor " +
          " ".join(f"{p:6.2f}" for _, p in res), flush=True)
    hm = sorted(host_ms)
    print(f"   host enqueue ms per call: median {hm[len(hm) // 2]:.2f} p90 {hm[int(0.9 * len(hm))]:.2f} "
          f"max {hm[-1]:.2f} (n={len(hm)})", flush=True)
    host_ms.clear()

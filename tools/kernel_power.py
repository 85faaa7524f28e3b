"""Energy per launch of the attention kernels under the board's power cap.

    python tools/kernel_power.py [--seconds 1.5] [--lib alt/x/libspa2.so]

Each stage (masker, forward, dQ, dK/dV, and a cuBLAS bf16 GEMM for reference) is launched back
to back for a fixed wall time at the Wan2.1-1.3B bench shape; NVML's total-energy counter and
a 5 ms sampler (SM clock, power, throttle reasons) give joules per launch, the mean SM clock
and the mean power.  Under a power cap, time per launch ~ energy per launch / cap, so the
joules tell which kernel to make cheaper.
"""

import argparse
import math
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=1.5)
    ap.add_argument("--lib", default=None)
    a = ap.parse_args()
    if a.lib:
        _lib.use_library(a.lib)
    import pynvml as nv

    import paper_2602_13515_b200 as spa
    from paper_2602_13515_b200 import attention as at
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
    do = torch.randn_like(q)
    cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
    B, H, N, d = q.shape
    keep = at._hybrid_mask_device(q, k, cfg, None)
    bm = spa.BlockMask._trusted(keep, 128, 64, N)
    lists = at.mask_lists(bm, B, H, N)
    scale = 1 / math.sqrt(d)
    o, lse = at.fwd(q, k, v, lists, scale)
    dq, dk, dv = at.bwd(q, k, v, o, do, lse, lists, scale)
    delta = torch.empty((B, H, N), device=q.device, dtype=torch.float32)
    st = torch.cuda.current_stream()
    dt = _lib.DTYPE_CODES[q.dtype]

    def k_dq():
        _lib.call("spa2_bwd_dq_delta", _lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(o), _lib.view4(do),
                  _lib.ptr(lse), _lib.ptr(delta), _lib.view4(dq), dt, B, H, N, d, 128, 64, _lib.ptr(lists.row_ptr),
                  _lib.ptr(lists.row_idx), _lib.ptr(lists.row_order), scale, st.cuda_stream, stream_obj=st)

    def k_dkdv():
        _lib.call("spa2_bwd_dkdv", _lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(do), _lib.ptr(lse),
                  _lib.ptr(delta), _lib.view4(dk), _lib.view4(dv), dt, B, H, N, d, 128, 64, _lib.ptr(lists.col_ptr),
                  _lib.ptr(lists.col_idx), _lib.ptr(lists.col_order), scale, st.cuda_stream, stream_obj=st)

    ga = torch.randn(8192, 8192, device=q.device, dtype=torch.bfloat16)
    gb = torch.randn(8192, 8192, device=q.device, dtype=torch.bfloat16)
    stages = [
        ("masker (pool+scores+select+lists)", lambda: at.build_lists(at._native_keep(spa.BlockMask._trusted(at._hybrid_mask_device(q, k, cfg, None), 128, 64, N), B, H, N))),
        ("fwd k_fwd", lambda: at.fwd(q, k, v, lists, scale)),
        ("dQ k_dq3 (+delta)", k_dq),
        ("dK/dV k_dkdv5", k_dkdv),
        ("cuBLAS bf16 GEMM 8192^3", lambda: torch.matmul(ga, gb)),
    ]
    for name, fn in stages:
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        samples = []
        stop = threading.Event()

        def sampler():
            while not stop.is_set():
                samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1e3,
                                nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                time.sleep(0.005)

        # launches per batch sized from one timed launch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        one = max(e0.elapsed_time(e1), 1e-3)
        n = max(10, int(a.seconds * 1e3 / one))
        th = threading.Thread(target=sampler, daemon=True)
        th.start()
        time.sleep(0.05)
        j0 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        j1 = nv.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set()
        th.join()
        ms = e0.elapsed_time(e1) / n
        load = samples[len(samples) // 5:] or samples
        mhz = sorted(s[0] for s in load)[len(load) // 2]
        watts = sum(s[1] for s in load) / len(load)
        capped = sum(1 for s in load if s[2] & nv.nvmlClocksEventReasonSwPowerCap) / len(load)
        mj = (j1 - j0) / n  # NVML energy counter is in mJ
        print(f"{name:36s} {ms:8.4f} ms/launch  {mj:8.2f} mJ/launch  SM {mhz:5d} MHz  {watts:6.0f} W  "
              f"power-capped {capped * 100:4.0f}% of samples  ({n} launches)")


if __name__ == "__main__":
    main()

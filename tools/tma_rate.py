"""TMA streaming micro-benchmark: aggregate L2->SMEM (or HBM->SMEM) bandwidth, no compute.
    python tools/tma_rate.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402

lib = _lib.load()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(4 * sms, dtype=torch.int64, device="cuda")
clk = 1.0e9 * 0  # filled below
for label, mb in (("L2-resident 32 MB", 32), ("L2-resident 96 MB", 96), ("HBM 2 GB", 2048)):
    rows = mb * 1024 * 1024 // 128
    buf = torch.empty(rows * 64, dtype=torch.bfloat16, device="cuda").normal_()
    for box, stages, ctas_per_sm in ((128, 2, 1), (128, 4, 1), (64, 4, 1), (128, 4, 2)):
        ctas = sms * ctas_per_sm
        iters = 400
        st = torch.cuda.current_stream().cuda_stream
        lib.spa2_probe_tma_rate(_lib.ptr(buf), rows, box, stages, 20, ctas, _lib.ptr(out), st)  # warm
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(lib.spa2_probe_tma_rate(_lib.ptr(buf), rows, box, stages, iters, ctas, _lib.ptr(out), st), "tma")
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        tb = ctas * iters * box * 128 / (ms * 1e-3) / 1e12
        per_sm_cyc = out[:ctas].double().mean().item()
        print(f"{label:20s} box {box:3d} rows ({box*128//1024} KB) stages {stages} ctas/SM {ctas_per_sm}: "
              f"{tb:6.2f} TB/s aggregate; {ctas_per_sm * iters * box * 128 / per_sm_cyc:6.1f} B/clk/SM")
    del buf

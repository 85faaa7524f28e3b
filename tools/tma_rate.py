"""TMA streaming micro-benchmark: aggregate L2->SMEM bandwidth, no compute.

    python tools/tma_rate.py

Measures how the per-SM fill rate depends on request size, ring depth, the number of
issuing warps per CTA, CTAs per SM, and tensor-map boxes vs 1-D bulk copies."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402

lib = _lib.load_diag()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(4 * 2 * sms, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
mb = 48
rows = mb * 1024 * 1024 // 256
buf = torch.empty(rows * 128, dtype=torch.bfloat16, device="cuda").normal_()
# (box_rows, chunks, stages, issuers, mode, ctas_per_sm)
cases = [
    (128, 1, 4, 1, 0, 1), (128, 2, 4, 1, 0, 1), (64, 2, 4, 1, 0, 1), (256, 2, 2, 1, 0, 1),
    (128, 1, 4, 2, 0, 1), (128, 2, 2, 2, 0, 1), (64, 2, 4, 2, 0, 1), (128, 2, 2, 3, 0, 1),
    (128, 1, 3, 4, 0, 1), (64, 2, 2, 4, 0, 1), (128, 2, 1, 4, 0, 1),
    (128, 1, 4, 1, 1, 1), (128, 2, 4, 1, 1, 1), (128, 2, 2, 2, 1, 1), (64, 2, 2, 4, 1, 1),
    (128, 2, 2, 1, 0, 2), (64, 2, 2, 2, 0, 2),
    # issuers on the same SM sub-partition (warp stride 4) vs adjacent warps
    (128, 2, 2, 2, 4 << 8, 1), (128, 1, 4, 2, 4 << 8, 1), (128, 2, 2, 2, 2 << 8, 1),
]
print(f"buffer {mb} MB (L2-resident), {sms} SMs")
for box, chunks, stages, issuers, mode, cps in cases:
    ctas = sms * cps
    iters = 300
    args = (_lib.ptr(buf), rows, box, chunks, stages, issuers, mode)
    _lib.check_diag(lib.spa2_probe_tma_rate2(*args, 10, ctas, _lib.ptr(out), st), "tma2")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check_diag(lib.spa2_probe_tma_rate2(*args, iters, ctas, _lib.ptr(out), st), "tma2")
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    req = box * 128 * chunks
    total = ctas * issuers * iters * req
    cyc = out.view(-1, 4)[:ctas, :issuers].double().max(dim=1).values.mean().item()
    print(f"req {req // 1024:3d} KB ({'box' if mode % 256 == 0 else 'bulk'} wstride {max(1, mode >> 8)} {box}x{chunks}) stages {stages} issuers {issuers} "
          f"ctas/SM {cps}: {total / (ms * 1e-3) / 1e12:6.2f} TB/s; {cps * issuers * iters * req / cyc:6.1f} B/clk/SM")

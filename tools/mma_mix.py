"""The dQ kernel's per-tile MMA sequence in isolation (spa2_probe_mma_mix): cycles per tile."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402

lib = _lib.load_diag()
sms = torch.cuda.get_device_properties(0).multi_processor_count
out = torch.zeros(sms + 1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
src = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
reps = 2000
for flags, label in ((1, "TS random"), (256 | 1, "TS warp-issue"), (256 | 17, "TS warp-issue S only"), (256 | 3, "TS warp-issue + noise"),
                     (256 | 512 | 1, "TS warp-issue + commits"), (256 | 1024 | 1, "TS warp-issue, wait S"),
                     (256 | 1536 | 3, "TS warp-issue + commits + wait S + noise"),
                     (256 | 2048 | 1, "TS warp-issue + TMA noise"), (256 | 2048 | 3, "TS warp-issue + TMA + TMEM noise"),
                     (256 | 2048 | 16 | 1, "TS warp-issue S only + TMA noise"), (2048 | 5, "SS + TMA noise"),
                     (4096 | 1, "3 issuing warps (S / dP / dQ)"), (4096 | 512 | 1, "3 issuing warps + commits")):
    for ctas in (1, sms):
        _lib.check_diag(lib.spa2_probe_mma_mix(10, flags, ctas, _lib.ptr(src), _lib.ptr(out), st), "mix")
        out.zero_()
        _lib.check_diag(lib.spa2_probe_mma_mix(reps, flags, ctas, _lib.ptr(src), _lib.ptr(out), st), "mix")
        torch.cuda.synchronize()
        cyc = out[:ctas].double().mean().item() / reps
        print(f"{label:28s} ctas {ctas:3d}: {cyc:7.1f} cycles per tile")

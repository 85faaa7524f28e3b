"""tcgen05.ld / tcgen05.st throughput per SM (diagnostic; numbers quoted in DESIGN.md §5).
Every warp reads (or writes) its TMEM lane quarter, 32x32b shapes; one CTA per SM."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402

lib = _lib.load_diag()
st = torch.cuda.current_stream().cuda_stream
ctas, reps = 148, 2048
cyc = torch.zeros(ctas * 16, dtype=torch.int64, device="cuda")
names = {0: "ld 32 col", 1: "ld 2x32 col", 2: "ld 16 col", 3: "st 16 col"}
bytes_per = {0: 4096, 1: 4096, 2: 2048, 3: 2048}
for mode in (0, 1, 2, 3):
    for warps in (1, 4, 8, 16):
        cyc.zero_()
        _lib.check_diag(lib.spa2_probe_tmem_rate(reps, mode, warps, ctas, _lib.ptr(cyc), st), "tmem")
        torch.cuda.synchronize()
        c = cyc.view(ctas, 16)[:, :warps].float()
        tot = warps * reps * bytes_per[mode]
        print(f"{names[mode]:12s} warps {warps:2d}: {c.mean().item() / reps:7.1f} cyc/instr per warp, "
              f"{tot / c.max(dim=1).values.mean().item():6.1f} B/clk/SM")

# loads while the tensor core is busy (warp 0 streams MMAs into other columns)
for mode, label in ((4, "ld 32 col + N=128 MMAs"), (5, "ld 32 col + N=64 MMAs")):
    for warps in (2, 5, 9):
        cyc.zero_()
        _lib.check_diag(lib.spa2_probe_tmem_rate(reps, mode, warps, ctas, _lib.ptr(cyc), st), "tmem")
        torch.cuda.synchronize()
        c = cyc.view(ctas, 16)[:, 1:warps].float()
        print(f"{label:24s} ld warps {warps - 1}: {c.mean().item() / reps:7.1f} cyc/instr per warp")

# mbarrier polls on an already-completed phase
mb = torch.zeros(4, dtype=torch.int64, device="cuda")
for mode, label in ((0, "try_wait"), (1, "test_wait"), (2, "mbar_wait()")):
    for threads in (32, 512):
        mb.zero_()
        _lib.check_diag(lib.spa2_probe_mbar_latency(4096, mode, threads, _lib.ptr(mb), st), "mbar")
        torch.cuda.synchronize()
        print(f"mbarrier {label:12s} {threads:3d} threads: {mb[0].item() / 4096:6.1f} cycles per poll (completed phase)")

"""mbarrier try_wait polls by three warps at a chosen shared-memory offset while the dK/dV tile's
SS MMA sequence runs (does barrier polling contend with the tensor core's operand fetch?)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2602_13515_b200 import _lib
lib = _lib.load_diag()
ctas = torch.cuda.get_device_properties(0).multi_processor_count
reps = 1000
cyc = torch.zeros(2 * ctas, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for which, name in ((0, "alone"), (256 | 2048 | 32768 | (1 << 16), "polls at 16K (Q tile)"), (256 | 2048 | 32768 | (6 << 16), "polls at 96K (P tile)"),
                    (256 | 2048 | 32768 | (9 << 16), "polls at 144K (no operand, upper half)"), (256 | 2048 | 32768 | (11 << 16), "polls at 176K")):
    lib.spa2_probe_dkdv_mix(reps, which, ctas, _lib.ptr(cyc), st)
    torch.cuda.synchronize()
    c = cyc[:ctas].double().mean().item()
    polls = cyc[ctas:].double().mean().item()
    print(f"{name:40s} {c / reps:7.1f} cyc per tile   polls/clk {polls / c:6.3f}")

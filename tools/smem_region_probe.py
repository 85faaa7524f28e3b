"""Which shared-memory addresses can other warps read (LDS.128) without slowing the tensor
core's SS operand fetch?  The dK/dV tile's MMA sequence (operands in [0, 128 KB): Q, dO, K, V,
P, dS) runs back to back while three warps stream conflict-free LDS.128 of a 32 KB region at
offset r x 16 KB (r = 0..10).  One CTA per SM.

    python tools/smem_region_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load_diag()
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    reps = 1000
    cyc = torch.zeros(2 * ctas, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    _lib.check_diag(lib.spa2_probe_dkdv_mix(reps, 0, ctas, _lib.ptr(cyc), st), "dkdv_mix")
    torch.cuda.synchronize()
    print(f"alone: {cyc[:ctas].double().mean().item() / reps:7.1f} cyc per tile")
    for ops, name in ((0, "all four"), (1, "S+dP (Q 0-32K, dO 32-64K, K 64-80K, V 80-96K)"),
                      (2, "dV+dK (dO, Q, P 96-112K, dS 112-128K)")):
        for r in range(11):
            which = ops | 256 | 1024 | 32768 | (r << 16)
            _lib.check_diag(lib.spa2_probe_dkdv_mix(reps, which, ctas, _lib.ptr(cyc), st), "dkdv_mix")
            torch.cuda.synchronize()
            c = cyc[:ctas].double().mean().item()
            staged = cyc[ctas:].double().mean().item()
            print(f"{name:48s} LDS [{16 * r:3d}K, {16 * r + 32:3d}K): {c / reps:7.1f} cyc per tile, LDS {staged / c:5.1f} B/clk")


if __name__ == "__main__":
    main()

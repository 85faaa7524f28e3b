"""Shared-memory contention probe: SS MMA (M=128, N=64) rate alone and with concurrent bulk-copy
writes, STS.128 stores and LDS.128 loads in other warps of the same CTA (one CTA per SM).

    python tools/smem_contend.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load_diag()
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    src = torch.zeros(16 * 1024 * 1024 + 65536, dtype=torch.uint8, device="cuda")
    out = torch.zeros(ctas * 4, dtype=torch.int64, device="cuda")
    reps = 4000
    names = {0: "MMA alone", 16: "A rotating (3 tiles)", 1: "+ bulk copies", 2: "+ STS.128", 4: "+ LDS.128",
             8: "+ TMEM loads", 3: "+ bulk + STS", 7: "+ bulk + STS + LDS", 8 | 16: "rot + TMEM loads",
             1 | 2 | 16: "rot + bulk + STS", 1 | 8 | 16: "rot + bulk + TMEM",
             32: "TS MMA alone", 32 | 8: "TS + TMEM loads", 32 | 1 | 8: "TS + bulk + TMEM loads"}
    for mode, name in names.items():
        rc = lib.spa2_probe_smem_contend(reps, mode, ctas, _lib.ptr(src), _lib.ptr(out), torch.cuda.current_stream().cuda_stream)
        _lib.check_diag(rc, "smem_contend")
        torch.cuda.synchronize()
        o = out.view(ctas, 4).double().mean(0)
        cyc = o[0].item()
        per = cyc / (reps * 8)
        bpc = [o[i].item() / cyc for i in (1, 2, 3)]
        mma_bpc = (2048 if mode & 32 else 6144) / per
        print(f"{name:22s} {per:6.1f} cyc per K=16 SS MMA ({mma_bpc:5.1f} B/clk operand reads)  "
              f"bulk {bpc[0]:5.1f}  STS/TMEM {bpc[1]:5.1f}  LDS {bpc[2]:5.1f} B/clk  total {mma_bpc + sum(bpc):6.1f} B/clk")

    reps = 1000
    cyc = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    cases = ((0, "dK/dV tile: S, dP, dV^T, dK^T"), (1, "S + dP only (K-major)"), (2, "dV^T + dK^T only (MN-major)"),
             (32, "S only"))
    for which, name in cases + tuple((w | 64, name + " [1 thread]") for w, name in cases):
        _lib.check_diag(lib.spa2_probe_dkdv_mix(reps, which, ctas, _lib.ptr(cyc), torch.cuda.current_stream().cuda_stream),
                        "dkdv_mix")
        torch.cuda.synchronize()
        per = cyc.double().mean().item() / reps
        groups = 1 if which & 32 else (4 if (which & 3) == 0 else 2)
        print(f"{name:34s} {per:7.1f} cyc per tile ({per / groups:6.1f} per 8-step group, {per / groups / 8:5.1f} per K step)")

    for mode, name in ((1, "tcgen05.cp 32 KB tile"), (2, "SS MMA group (8 x N=64)"), (3, "both, interleaved")):
        _lib.check_diag(lib.spa2_probe_cp_rate(reps, mode, ctas, _lib.ptr(cyc), torch.cuda.current_stream().cuda_stream),
                        "cp_rate")
        torch.cuda.synchronize()
        per = cyc.double().mean().item() / reps
        print(f"{name:34s} {per:7.1f} cyc per rep" + (f" ({32768 / per:5.1f} B/clk)" if mode == 1 else ""))


if __name__ == "__main__":
    main()

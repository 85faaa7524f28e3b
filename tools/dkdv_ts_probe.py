"""dK/dV MMA sequence with S and dP as TS MMAs (Q / dO read from TMEM) vs the SS form of the
current kernel, alone and with concurrent LDS.128 + tcgen05.st staging traffic (what staging
Q / dO into TMEM from the shared-memory operand slots would add), one CTA per SM.

    python tools/dkdv_ts_probe.py
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
    cases = ((0, "SS S/dP + dV^T/dK^T (current)"), (1, "SS S + dP only"), (128 | 1, "TS S + dP only"),
             (128, "TS S/dP + SS dV^T/dK^T"), (256, "SS tile + staging traffic"),
             (128 | 256, "TS tile + staging traffic"), (128 | 1 | 256, "TS S + dP + staging traffic"),
             (256 | 512, "SS tile + TMEM stores only"), (256 | 1024, "SS tile + LDS only"),
             (128 | 256 | 512, "TS tile + TMEM stores only"), (128 | 256 | 1024, "TS tile + LDS only"),
             (32 | 256 | 512, "SS S only + TMEM stores only"),
             (256 | 1024 | 8192, "SS tile + LDS of the P tile"), (256 | 1024 | 16384, "SS tile + LDS elsewhere"),
             (256 | 4096, "SS tile + STS into the Q tile"), (256 | 4096 | 8192, "SS tile + STS into the P tile"),
             (256 | 4096 | 16384, "SS tile + STS elsewhere"), (1 | 256 | 1024 | 16384, "SS S+dP + LDS elsewhere"),
             (2 | 256 | 4096 | 8192, "SS dV+dK + STS into the P tile"))
    for which, name in cases:
        st = torch.cuda.current_stream().cuda_stream
        _lib.check_diag(lib.spa2_probe_dkdv_mix(reps, which, ctas, _lib.ptr(cyc), st), "dkdv_mix")
        torch.cuda.synchronize()
        c = cyc[:ctas].double().mean().item()
        per = c / reps
        line = f"{name:34s} {per:7.1f} cyc per tile"
        if which & 256:
            staged = cyc[ctas:].double().mean().item()
            line += f"   staging {staged / c:6.1f} B/clk ({staged / reps / 1024:5.1f} KB per tile)"
        print(line)


if __name__ == "__main__":
    main()

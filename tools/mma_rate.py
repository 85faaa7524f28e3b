"""tcgen05 issue-rate micro-benchmark: cycles per MMA (M x N x 16) per operand layout.

    python tools/mma_rate.py            (on the GPU box)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402

CASES = [  # (name, m, n, k, a_mn, b_mn, a_tmem)
    ("S=QK^T  SS K/K  128x64", 128, 64, 128, 0, 0, 0),
    ("S pair  SS K/K  128x128", 128, 128, 128, 0, 0, 0),
    ("SS K/K  128x256", 128, 256, 128, 0, 0, 0),
    ("dV^T    SS MN/MN 128x64", 128, 64, 128, 1, 1, 0),
    ("dV^T2   SS MN/MN 128x128", 128, 128, 128, 1, 1, 0),
    ("PV      TS K/MN 128x128", 128, 128, 64, 0, 1, 1),
    ("PV      TS K/MN 128x64", 128, 64, 64, 0, 1, 1),
    ("PV      SS K/MN 128x128", 128, 128, 64, 0, 1, 0),
    ("M64     SS K/K  64x64", 64, 64, 128, 0, 0, 0),
    ("M64     SS K/K  64x128", 64, 128, 128, 0, 0, 0),
    ("M64     TS K/K  64x128", 64, 128, 128, 0, 0, 1),
    ("M64     TS K/MN 64x128", 64, 128, 128, 0, 1, 1),
    ("M64     TS K/K  64x256", 64, 256, 128, 0, 0, 1),
    # weight-stationary form (tcgen05.mma.ws): a_tmem bit 1
    ("WS M64  SS K/K  64x128", 64, 128, 128, 0, 0, 2),
    ("WS M64  TS K/K  64x128", 64, 128, 128, 0, 0, 3),
    ("WS M64  TS K/MN 64x128", 64, 128, 128, 0, 1, 3),
    ("WS M64  TS K/K  64x64", 64, 64, 128, 0, 0, 3),
    ("WS M128 TS K/K  128x64", 128, 64, 128, 0, 0, 3),
    ("WS M128 SS K/K  128x64", 128, 64, 128, 0, 0, 2),
]

def main():
    lib = _lib.load_diag()
    ctas = torch.cuda.get_device_properties(0).multi_processor_count
    out = torch.zeros(ctas, dtype=torch.int64, device="cuda")
    reps = 2000
    only = sys.argv[1:]
    for name, m, n, k, amn, bmn, at in CASES:
        if only and not any(o in name for o in only):
            continue
        for c in (1, ctas):
            rc = lib.spa2_probe_mma_rate(m, n, k, amn, bmn, at, reps, c, _lib.ptr(out), torch.cuda.current_stream().cuda_stream)
            _lib.check_diag(rc, name)
            torch.cuda.synchronize()
            cyc = out[:c].double().mean().item()
            per = cyc / (reps * 8)
            ideal = max(m, 128) * n / 256
            print(f"{name:28s} ctas={c:3d}  {per:7.1f} cyc/MMA  (pacing-law floor {ideal:5.1f}; "
                  f"{100 * ideal / per:5.1f}% of floor)")

if __name__ == "__main__":
    main()

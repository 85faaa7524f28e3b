"""fp32 reduction-into-L2 throughput (the dQ-partial traffic of a fused dK/dV/dQ backward).

    python tools/red_rate.py
"""

import sys

import torch

sys.path.insert(0, ".")
from paper_2602_13515_b200 import _lib  # noqa: E402

lib = _lib.load_diag()
st = torch.cuda.current_stream().cuda_stream
for nslots in (256, 3072):  # 16 MB (L2-resident) and 201 MB (the configs[1] dQ in fp32)
    dst = torch.zeros(nslots * 128 * 128, device="cuda")
    for mode, name in ((0, "red.v4 row per thread"), (2, "red.v4 coalesced"), (1, "st.v4 row per thread"),
                       (3, "TMA bulk reduce .add.f32")):
        for ctas in ((148,) if mode == 3 else (148, 296, 592)):
            tiles = 64
            _lib.check_diag(lib.spa2_probe_red_rate(_lib.ptr(dst), tiles, nslots, ctas, mode, st), "red")
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                lib.spa2_probe_red_rate(_lib.ptr(dst), tiles, nslots, ctas, mode, st)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            nbytes = ctas * tiles * 128 * 128 * 4
            print(f"{name:24s} dst {nslots * 64 / 1024:6.1f} MB ctas {ctas:4d}: {nbytes / ms / 1e6:8.1f} GB/s")

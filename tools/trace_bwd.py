"""Pipeline trace of the dK/dV kernel (CTA 0) at the bench shape — diagnostic.

    python tools/trace_bwd.py

Roles/kinds recorded by the kernel (spa2_debug_trace):
  producer 0: 1 before waiting for a free Q/dO stage, 2 after (loads issued next)
  mma      1: 1 before waiting for Q/dO of tile g, 2 after (S/dP issued next),
              3 before waiting for P/dS of tile g, 4 after (dV/dK issued next)
  softmax  2: 1 before waiting for S/dP of tile g, 2 after, 3 P/dS buffer free, 4 P/dS written
  epilog   3: 1 before waiting for the accumulators of item it, 2 after, 3 stores done

Needs a trace build: `bash tools/build_alt.sh trace -DSPA2_TRACE`, then run with
SPA2_LIB_PATH=alt/trace/libspa2.so (production kernels carry no trace code)."""
import math
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import _lib  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402


def main():
    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=0)
    do = torch.randn_like(q)
    cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
    bm = at._hybrid_mask_device(q, k, cfg, False)
    lists = at.mask_lists(bm, 1, 12, 32760)
    scale = 1 / math.sqrt(128)
    o, lse = at.fwd(q, k, v, lists, scale)
    at.bwd(q, k, v, o, do, lse, lists, scale)
    cap = 1 << 16
    buf = torch.zeros(2 + cap, dtype=torch.int64, device="cuda")
    _lib.load().spa2_debug_trace(_lib.ptr(buf), cap)
    at.bwd(q, k, v, o, do, lse, lists, scale)
    torch.cuda.synchronize()
    _lib.load().spa2_debug_trace(None, 0)
    R = cap // 4
    raw = buf[2:].view(4, R).cpu()
if not raw.any():
    sys.exit("no events recorded: run with SPA2_LIB_PATH=alt/trace/libspa2.so (tools/build_alt.sh trace -DSPA2_TRACE)")
    rec = defaultdict(dict)
    t0 = None
    nz = raw.nonzero().tolist()
    for role, slot in nz:
        t = int(raw[role, slot])
        t0 = t if t0 is None else min(t0, t)
    for role, slot in nz:
        rec[(role, slot // 8)][slot % 8] = int(raw[role, slot]) - t0
    n = len(nz)
    ev = [(0, 0)]
    tiles = sorted(i for (r, i) in rec if r == 2)
    print(f"events {n}; tiles traced {len(tiles)}")
    print("stage lifetime of tile g (cycles): load issued -> S/dP issued -> softmax done -> dV/dK issued -> "
          "stage reloaded (tile g+2)")
    cols = ["load->SdP", "SdP->smx_done", "smx->dVdK", "dVdK->reload", "smx wait S/dP", "smx wait Pbuf", "smx compute"]
    agg, cnt = defaultdict(float), 0
    for g in tiles[5:-3]:
        ld, sdp = rec.get((0, g), {}).get(2), rec.get((1, g), {}).get(2)
        smx, dvdk = rec.get((2, g), {}), rec.get((1, g), {}).get(4)
        rel = rec.get((0, g + 2), {}).get(2)
        if None in (ld, sdp, dvdk, rel) or 4 not in smx:
            continue
        row = (sdp - ld, smx[4] - sdp, dvdk - smx[4], rel - dvdk, smx[2] - smx[1], smx[3] - smx[2], smx[4] - smx[3])
        for i, x in enumerate(row):
            agg[i] += x
        cnt += 1
        if cnt <= 12:
            print(f"{g:4d} " + " ".join(f"{x:>14d}" for x in row))
    print("mean " + " ".join(f"{agg[i] / max(cnt, 1):>14.0f}" for i in range(len(cols))))
    print("     " + " ".join(f"{c:>14s}" for c in cols))
    done = [rec[(2, g)].get(4, 0) for g in tiles]
    per = sorted(b - a for a, b in zip(done, done[1:]))
    print("tile period cycles: median", per[len(per) // 2], "p10", per[len(per) // 10], "p90", per[9 * len(per) // 10])


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def timeline():
    """Per-tile event timeline (cycles relative to the first shown event) for a steady-state
    window: producer P1/P2 (wait free stage / load issued), MMA M2 (S/dP issued), M4 (dV
    issued), M5 (dK issued), elementwise E1/E2 (wait S / S landed), E3 (P buffer free), E5 (P
    stored), E4 (dS stored)."""
    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=0)
    do = torch.randn_like(q)
    cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
    bm = at._hybrid_mask_device(q, k, cfg, False)
    lists = at.mask_lists(bm, 1, 12, 32760)
    scale = 1 / math.sqrt(128)
    o, lse = at.fwd(q, k, v, lists, scale)
    at.bwd(q, k, v, o, do, lse, lists, scale)
    cap = 1 << 16
    buf = torch.zeros(2 + cap, dtype=torch.int64, device="cuda")
    _lib.load().spa2_debug_trace(_lib.ptr(buf), cap)
    at.bwd(q, k, v, o, do, lse, lists, scale)
    torch.cuda.synchronize()
    _lib.load().spa2_debug_trace(None, 0)
    R = cap // 4
    raw = buf[2:].view(4, R).cpu()
if not raw.any():
    sys.exit("no events recorded: run with SPA2_LIB_PATH=alt/trace/libspa2.so (tools/build_alt.sh trace -DSPA2_TRACE)")
    names = {0: "P", 1: "M", 2: "E", 3: "X"}
    ev = []
    for role, slot in raw.nonzero().tolist():
        ev.append((int(raw[role, slot]), f"{names[role]}{slot % 8}", slot // 8))
    ev.sort()
    lo = [e for e in ev if e[1][0] in "PME" and 40 <= e[2] < 46]
    t0 = lo[0][0]
    for t, kind, g in lo:
        print(f"{t - t0:7d} {kind} g={g}")


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "timeline":
    timeline()

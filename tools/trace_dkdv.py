"""Pipeline trace of the dK/dV kernel (CTA 0) from a -DSPA2_TRACE build.

    bash tools/build_alt.sh trace -DSPA2_TRACE
    python tools/trace_dkdv.py alt/trace/libspa2.so

Events (clock64 of lane 0 of the recording warp, tile index g = the CTA's running tile counter):
  S/dP warp: 25 loop entry, 22 item start, 26 K/V landed, 29 S issue (buffer free + Q landed),
             16 dP committed
  dV/dK warp: 27 loop entry, 17 dV issue (P(g) stored + dO landed), 28 dK issue (dS(g) stored),
             18 dK committed
  EW warp 2: 19 S(g) landed, 23 past the P-buffer wait (dV(g-1) done), 20 dP(g) landed,
             24 past the dS-buffer wait (dK(g-1) done), 21 dS(g) stored
The tensor pipe executes the MMA groups in issue order; each SS group (8 K=16 steps at N=64)
takes ~384 cycles, so with issue times known the pipe's idle time can be reconstructed.
"""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_13515_b200 import _lib  # noqa: E402

_lib.use_library(sys.argv[1] if len(sys.argv) > 1 else "alt/trace/libspa2.so")
import ctypes  # noqa: E402

import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

SLOTS = 2048
GROUP = 384  # cycles per SS MMA group (8 x 48)
lib = _lib.load()
lib.spa2_trace_fetch.argtypes = [ctypes.c_void_p]
buf = np.zeros(32 * SLOTS, dtype=np.uint64)
q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
do = torch.randn_like(q)
cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
for it in range(3):
    qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
    res = spa.sparse_attention(qs, ks, vs, cfg)
    res.out.backward(do)
    torch.cuda.synchronize()
    lib.spa2_trace_fetch(buf.ctypes.data)
ev = buf.reshape(32, SLOTS).astype(np.int64)
n = int((ev[18] > 0).sum())
t0 = ev[16:30][ev[16:30] > 0].min()
e = {kk: np.where(ev[kk, :n] > 0, ev[kk, :n] - t0, -1) for kk in range(16, 32)}
print(f"tiles traced: {n}")
per = np.diff(e[18])
print(f"dK commit period: median {np.median(per):.0f}, mean {per.mean():.0f} cycles/tile "
      f"(floor {4 * GROUP} for four SS groups)")
items = np.flatnonzero(ev[22, :n] > 0)
print(f"items: {len(items)}, mean tiles/item {n / max(1, len(items)):.1f}")


def stat(name, x):
    x = x[np.isfinite(x)]
    if len(x) == 0:
        return
    print(f"  {name:46s} median {np.median(x):7.0f}  mean {x.mean():7.0f}  p90 {np.percentile(x, 90):7.0f}")


g = np.arange(n)
stat("S issue(g) -> S landed(g) [EW]", e[19] - e[29])
stat("S issue(g) -> dP committed(g)", e[16] - e[29])
stat("dP committed(g) -> dP landed(g) [EW]", e[20] - e[16])
stat("S landed(g) -> P-buffer free(g) [EW]", e[23] - e[19])
stat("S landed(g) -> P computed(g) [EW math]", e[31] - e[19])
stat("P computed(g) -> P-buffer free(g) [wait dV(g-1)]", e[23] - e[31])
stat("P-buffer free(g) -> dV issue(g)", e[17] - e[23])
stat("dP landed(g) -> dS-buffer free(g)", e[24] - e[20])
stat("dS-buffer free(g) -> dS stored(g)", e[21] - e[24])
stat("dS stored(g) -> dK issue(g)", e[28] - e[21])
stat("dV issue(g) -> P-buffer free(g+1) (dV done)", e[23][1:] - e[17][:-1])
stat("dK issue(g) -> dS-buffer free(g+1) (dK done)", e[24][1:] - e[28][:-1])
stat("S issue(g+2) - S landed(g) [TMEM ring]", e[29][2:] - e[19][:-2])
stat("dK issue(g-1) -> dV warp loop entry(g)", e[27][1:] - e[28][:-1])
stat("dV warp loop entry(g) -> P-buffer free(g) [EW]", e[23] - e[27])
stat("dV warp loop entry(g) -> dV issue(g)", e[17] - e[27])
stat("dS stored(g-1) -> dK issue(g-1)", e[28] - e[21])
stat("S issue(g) -> S issue(g+1)", e[29][1:] - e[29][:-1])
stat("dP committed(g) -> S issue(g+1)", e[29][1:] - e[16][:-1])

# pipe reconstruction: groups in issue order, each GROUP cycles, start = max(issue, prev end)
iss = []
for gi in range(n):
    if e[29][gi] >= 0:
        iss.append((e[29][gi], "S", gi))
    if e[16][gi] >= 0:
        iss.append((e[16][gi] - 1, "dP", gi))  # committed right after issue
    if e[17][gi] >= 0:
        iss.append((e[17][gi], "dV", gi))
    if e[28][gi] >= 0:
        iss.append((e[28][gi], "dK", gi))
iss.sort()
end = iss[0][0]
idle = 0
idle_after = {}
for t, kind, gi in iss:
    if t > end:
        idle += t - end
        idle_after[kind] = idle_after.get(kind, 0) + t - end
    end = max(end, t) + GROUP
span = end - iss[0][0]
print(f"pipe model: span {span} cycles, busy {len(iss) * GROUP} ({100 * len(iss) * GROUP / span:.1f} %), idle {idle}")
print("  idle cycles before the next group, by the group that was waited for:",
      {kk: f"{vv / max(1, n):.0f}/tile" for kk, vv in idle_after.items()})
order = "".join({"S": "s", "dP": "p", "dV": "v", "dK": "k"}[kind] for _, kind, _ in iss[:80])
print(f"  issue order of the first groups: {order}")

# completion estimates (observed by a waiter; exact when the waiter was already waiting)
comp = []
for gi in range(n - 1):
    for kind, t in (("S", e[19][gi]), ("dP", e[20][gi]), ("dV", e[23][gi + 1]), ("dK", e[24][gi + 1])):
        if t >= 0:
            comp.append((t, kind))
comp.sort()
ct = np.array([c[0] for c in comp])
d = np.diff(ct)
print(f"completion spacing (all groups, sorted): median {np.median(d):.0f}, mean {d.mean():.0f}, "
      f"p25 {np.percentile(d, 25):.0f}, p75 {np.percentile(d, 75):.0f} cycles")
seq = "".join({"S": "s", "dP": "p", "dV": "v", "dK": "k"}[c[1]] for c in comp[:60])
print(f"  completion order: {seq}")

# raw timeline of a few consecutive tiles in the middle of an item
names = {31: "EW P computed", 29: "S issue", 16: "dP commit", 17: "dV issue", 28: "dK issue", 18: "dK commit", 19: "EW S landed",
         23: "EW P-buf free", 20: "EW dP landed", 24: "EW dS-buf free", 21: "EW dS stored", 27: "dV warp entry"}
g0 = int(items[len(items) // 2]) + 3 if len(items) > 2 else 100
rows = []
for gi in range(g0, min(n, g0 + 5)):
    for kk, nm in names.items():
        if e[kk][gi] >= 0:
            rows.append((e[kk][gi], gi, nm))
rows.sort()
base_t = rows[0][0]
print(f"timeline of tiles {g0}..{g0 + 4} (cycles from the first event):")
for t, gi, nm in rows:
    print(f"  {t - base_t:7d}  tile {gi:4d}  {nm}")

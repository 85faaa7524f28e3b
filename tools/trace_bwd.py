"""Pipeline trace of the dQ kernel (CTA 0) from a -DSPA2_TRACE build: per-tile event times.

    bash tools/build_alt.sh trace -DSPA2_TRACE
    python tools/trace_bwd.py alt/trace/libspa2.so

Events (clock64 of lane 0, CTA 0; tile index g = the CTA's running tile counter):
  9 S warp entry, 0 S committed, 6 item start (before staging wait), 10 after Q/dO staging +
  TMEM free, 7 dP warp entry, 1 dP committed, 8 dQ warp entry, 2 dQ committed,
  3 EW (warp 2) S landed, 4 EW dP landed, 5 EW dS stored.
"""

import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_13515_b200 import _lib  # noqa: E402

_lib.use_library(sys.argv[1] if len(sys.argv) > 1 else "alt/trace/libspa2.so")
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

SLOTS = 2048
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
    lib.spa2_trace_fetch(buf.ctypes.data)  # keeps the last step's trace
ev = buf.reshape(32, SLOTS).astype(np.int64)
n = int((ev[0] > 0).sum())
t0 = ev[ev > 0].min()
e = {k_: ev[k_, :n] - t0 for k_ in range(11)}
print(f"tiles traced: {n}")
per = np.diff(e[0])
print(f"S commit period: median {np.median(per):.0f}, mean {per.mean():.0f} cycles/tile")
items = np.flatnonzero(ev[6, :n] > 0)
print(f"items: {len(items)}, mean tiles/item {n / max(1, len(items)):.1f}")
def stat(name, x):
    x = x[np.isfinite(x)]
    print(f"  {name:42s} median {np.median(x):7.0f}  mean {x.mean():7.0f}  p90 {np.percentile(x, 90):7.0f}")
stat("S: entry -> committed", e[0] - e[9])
stat("dP: entry -> committed", e[1] - e[7])
stat("dQ: entry -> committed", e[2] - e[8])
stat("EW: S committed -> S landed (EW wake)", e[3] - e[0])
stat("EW: dP committed -> dP landed", e[4] - e[1])
stat("EW: dP landed -> dS stored", e[5] - e[4])
stat("EW: S landed -> dP landed", e[4] - e[3])
stat("dQ: dS stored -> dQ committed", e[2] - e[5])
last = ev[11, :n] - t0
stat("EW: dS stored (warp 2) -> last warp's dS stored", last - e[5])
stat("dQ: last warp's dS stored -> dQ committed", e[2] - last)
e12, e13 = ev[12, :n] - t0, ev[13, :n] - t0
stat("hop: last warp's dS stored -> dQ warp past ds_full wait", e12 - last)
e14 = ev[14, :n] - t0
stat("  of which: last warp's arrive instruction (release)", e14 - last)
stat("  of which: arrive done -> dQ warp past wait", e12 - e14)
stat("dQ warp: past wait -> dQ committed (issue)", e[2] - e12)
stat("dP warp: past dq_done wait -> dP committed", e[1] - e13)
stat("hop: dQ(g-2) committed -> dP warp past dq_done wait", e13[2:] - e[2][:-2])
stat("dP(g) commit - dQ(g-2) commit", e[1][2:] - e[2][:-2])
stat("S(g) commit - EW S landed(g-2)", e[0][2:] - e[3][:-2])
stat("EW: dS stored(g) -> S landed(g+1)", e[3][1:] - e[5][:-1])
b = items[1:]
stat("item boundary: start -> Q/dO ready", (e[10] - e[6])[b])
stat("item boundary: S period at first tile", (e[0][b] - e[0][b - 1]).astype(float))
print("first 12 tiles (cycles from start): S, dP, EW-S, EW-dP, dS, dQ")
for g in range(12):
    print(g, e[0][g], e[1][g], e[3][g], e[4][g], e[5][g], e[2][g])

print()
print("==== dK/dV kernel (CTA 0) ====")
d = ev[16:]
n2 = int((d[0] > 0).sum())
t1 = d[d > 0].min()
f = {k_: d[k_, :n2] - t1 for k_ in range(11)}
per = np.diff(f[0])
print(f"tiles traced: {n2}; dP commit period median {np.median(per):.0f}, mean {per.mean():.0f} cycles/tile")
it2 = np.flatnonzero(d[6, :n2] > 0)
print(f"items: {len(it2)}, mean tiles/item {n2 / max(1, len(it2)):.1f}")
stat("S/dP issue: entry -> dP committed", f[0] - f[9])
stat("dK issue committed - dP committed", f[2] - f[0])
stat("EW: dP committed -> S landed", f[3] - f[0])
stat("EW: S landed -> dP landed", f[4] - f[3])
stat("EW: dP landed -> dS stored", f[5] - f[4])
bb = it2[1:]
stat("item boundary: start -> K/V landed", (f[10] - f[6])[bb])
stat("item boundary: period at first tile", (f[0][bb] - f[0][bb - 1]).astype(float))
nb = np.setdiff1d(np.arange(1, n2), bb)
stat("period at other tiles", (f[0][nb] - f[0][nb - 1]).astype(float))

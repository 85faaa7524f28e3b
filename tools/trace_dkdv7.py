"""Event timeline of the key-pair dK/dV kernel (k_dkdv7, CTA 0) at the bench shape.
Needs a trace build: `bash tools/build_alt.sh trace -DSPA2_TRACE`, then
SPA2_LIB_PATH=alt/trace/libspa2.so SPA2_DKDV_VARIANT=7 python tools/trace_dkdv7.py
P1/P2 producer before/after waiting the Q slot of tile g; M1 Sᵀ(g) issue, M2 dPᵀ(g) issued,
M3 dV(g) issue (P ready), M4 dK(g) issue (dS ready); E1/E2 elementwise before/after Sᵀ landed,
E3 Pᵀ written, E4 dPᵀ landed, E5 dSᵀ written."""
import collections, math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import _lib  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=0)
do = torch.randn_like(q)
bm = at._hybrid_mask_device(q, k, spa.SparsityConfig(0.03, 0.2, 128, 64), False)
lists = at.mask_lists(bm, 1, 12, 32760)
scale = 1 / math.sqrt(128)
o, lse = at.fwd(q, k, v, lists, scale)
at.bwd(q, k, v, o, do, lse, lists, scale)
cap = 1 << 16
buf = torch.zeros(2 + cap, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.spa2_debug_trace(_lib.ptr(buf), cap)
at.bwd(q, k, v, o, do, lse, lists, scale)
torch.cuda.synchronize()
lib.spa2_debug_trace(None, 0)
R = cap // 4
raw = buf[2:].view(4, R).cpu()
if not raw.any():
    sys.exit("no events recorded: run with SPA2_LIB_PATH=alt/trace/libspa2.so (tools/build_alt.sh trace -DSPA2_TRACE)")
names = {0: "P", 1: "M", 2: "E", 3: "X"}
ev = sorted((int(raw[r, s]), f"{names[r]}{s % 8}", s // 8) for r, s in raw.nonzero().tolist())
# the dQ kernel of the same bwd call also writes role 1/2 events: keep the last launch's (dK/dV)
by = collections.defaultdict(dict)
for t, kd, g in ev:
    by[g][kd] = t
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 40
win = sorted((t, kd, g) for g in range(lo, lo + 4) for kd, t in by.get(g, {}).items())
t0 = win[0][0] if win else 0
for t, kd, g in win:
    print(f"{t - t0:7d} {kd} g={g}")
def avg(a, b):
    vals = [x[b] - x[a] for x in by.values() if a in x and b in x]
    return sum(vals) / max(1, len(vals))
for a, b in (("E1", "E2"), ("E2", "E3"), ("E3", "E4"), ("E4", "E5"), ("M1", "M2"), ("M2", "M3"), ("M3", "M4"),
             ("E3", "M3"), ("E5", "M4"), ("M1", "E2")):
    print(f"{a}->{b}: {avg(a, b):.0f} cycles")
m1 = sorted(x["M1"] for x in by.values() if "M1" in x)
d = sorted(b - a for a, b in zip(m1, m1[1:]))
if d:
    print("Sᵀ issue period: median", d[len(d) // 2])

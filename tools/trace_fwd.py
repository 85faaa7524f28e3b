"""Event timeline of the forward kernel (CTA 0; k_fwd3 numbers tiles by a CTA-global counter).
P1/P2 producer before/after waiting a free K slot for tile t; M2 S issue begins, M3 S issued,
M4 PV issue; E1/E2 softmax before/after S landed, E5 row max done, E4 P written.
Needs a trace build: `bash tools/build_alt.sh trace -DSPA2_TRACE`, then run with
SPA2_LIB_PATH=alt/trace/libspa2.so (production kernels carry no trace code)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import _lib  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=0)
bm = at._hybrid_mask_device(q, k, spa.SparsityConfig(0.03, 0.2, 128, 64), False)
lists = at.mask_lists(bm, 1, 12, 32760)
scale = 1 / math.sqrt(128)
at.fwd(q, k, v, lists, scale)
cap = 1 << 16
buf = torch.zeros(2 + cap, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.spa2_debug_trace(_lib.ptr(buf), cap)
at.fwd(q, k, v, lists, scale)
torch.cuda.synchronize()
lib.spa2_debug_trace(None, 0)
R = cap // 4
raw = buf[2:].view(4, R).cpu()
if not raw.any():
    sys.exit("no events recorded: run with SPA2_LIB_PATH=alt/trace/libspa2.so (tools/build_alt.sh trace -DSPA2_TRACE)")
names = {0: "P", 1: "M", 2: "E", 3: "X"}
ev = sorted((int(raw[r, s]), f"{names[r]}{s % 8}", s // 8) for r, s in raw.nonzero().tolist())
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 10
win = [e for e in ev if lo <= e[2] < lo + 5]
t0 = win[0][0]
for t, kind, g in win:
    print(f"{t - t0:7d} {kind} t={g}")
m2 = {g: t for t, kd, g in ev if kd == "M2"}
gs = sorted(m2)
d = sorted(m2[b] - m2[a] for a, b in zip(gs, gs[1:]) if b == a + 1)
print("S issue period: median", d[len(d) // 2], "n", len(d), "tiles", len(gs))

# per-stage averages over all tiles of CTA 0
import collections
by = collections.defaultdict(dict)
for t, kd, g in ev:
    by[g][kd] = t
def avg(a, b):
    v = [x[b] - x[a] for x in by.values() if a in x and b in x]
    return sum(v) / max(1, len(v))
for a, b in (("E1", "E2"), ("E2", "E5"), ("E5", "E4"), ("M2", "M3"), ("M3", "E2"), ("E4", "M4")):
    print(f"{a}->{b}: {avg(a, b):.0f} cycles")

"""Event timeline of the dQ kernel (CTA 0) at the bench shape — diagnostic.
M2 S/dP issue begins, M6 S issued, M3 S/dP issued, M7 dQ wait begins, M4 dQ issue begins, M5 dQ issued;
P1/P2 producer before/after waiting a free K slot of tile g; M2 S/dP issued; M4 dQ issued;
E1/E2 elementwise before/after S landed, E3 dP landed, E4 dS written.
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
do = torch.randn_like(q)
bm = at._hybrid_mask_device(q, k, spa.SparsityConfig(0.03, 0.2, 128, 64), False)
lists = at.mask_lists(bm, 1, 12, 32760)
scale = 1 / math.sqrt(128)
o, lse = at.fwd(q, k, v, lists, scale)
delta = torch.empty(1, 12, 32760, device="cuda")
st = torch.cuda.current_stream().cuda_stream
lib = _lib.load()
_lib.check(lib.spa2_bwd_delta(_lib.view4(o), _lib.view4(do), _lib.ptr(delta), 0, 1, 12, 32760, 128, st), "d")
dq = torch.empty_like(q)
cap = 1 << 16
buf = torch.zeros(2 + cap, dtype=torch.int64, device="cuda")


def run():
    _lib.check(lib.spa2_bwd_dq_delta(_lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(o), _lib.view4(do),
                                     _lib.ptr(lse), _lib.ptr(delta), _lib.view4(dq), 0, 1, 12, 32760, 128, 128, 64,
                                     _lib.ptr(lists.row_ptr), _lib.ptr(lists.row_idx), _lib.ptr(lists.row_order),
                                     scale, st), "dq")


run()
lib.spa2_debug_trace(_lib.ptr(buf), cap)
run()
torch.cuda.synchronize()
lib.spa2_debug_trace(None, 0)
R = cap // 4
raw = buf[2:].view(4, R).cpu()
if not raw.any():
    sys.exit("no events recorded: run with SPA2_LIB_PATH=alt/trace/libspa2.so (tools/build_alt.sh trace -DSPA2_TRACE)")
names = {0: "P", 1: "M", 2: "E", 3: "X"}
ev = sorted((int(raw[r, s]), f"{names[r]}{s % 8}", s // 8) for r, s in raw.nonzero().tolist())
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 40
win = [e for e in ev if lo <= e[2] < lo + 6]
t0 = win[0][0]
for t, kind, g in win:
    print(f"{t - t0:7d} {kind} g={g}")
# periods
m2 = {g: t for t, kd, g in ev if kd == "M2"}
gs = sorted(m2)
d = sorted(m2[b] - m2[a] for a, b in zip(gs, gs[1:]) if b == a + 1)
print("S/dP issue period: median", d[len(d) // 2], "p10", d[len(d) // 10], "p90", d[9 * len(d) // 10], "n", len(d))

x = {}
for t, kd, g in ev:
    if kd[0] == "X":
        x.setdefault(g, {})[int(kd[1:])] = t
print("per-warp dS-written times relative to warp 2 (cycles), tiles", lo, "..", lo + 5)
for g in range(lo, lo + 6):
    if g in x and 0 in x[g]:
        print(g, [x[g].get(w, 0) - x[g][0] for w in range(8)])

# per-stage averages over all tiles of CTA 0
import collections
by = collections.defaultdict(dict)
for t, kd, g in ev:
    by[g][kd] = t
def avg(a, b):
    v = [x[b] - x[a] for x in by.values() if a in x and b in x]
    return sum(v) / max(1, len(v))
for a, b in (("E1", "E2"), ("E2", "E3"), ("E3", "E4"), ("M2", "M3"), ("M3", "E2"), ("E4", "M4"), ("M4", "M5"), ("P2", "M2")):
    print(f"{a}->{b}: {avg(a, b):.0f} cycles")


"""Pipeline trace of the dQ kernel (CTA 0) at the bench shape — diagnostic.
producer 0: 1/2 before/after waiting for a free K slot of tile g
mma 1: 1 before waiting dq_done(g-2), 5 after, 2 K landed (S/dP issued next), 3/4 before/after waiting dS(g)
softmax 2: 1/2 before/after waiting S/dP(g), 4 dS written

Needs a trace build: `bash tools/build_alt.sh trace -DSPA2_TRACE`, then run with
SPA2_LIB_PATH=alt/trace/libspa2.so (production kernels carry no trace code)."""
import math, os, sys
from collections import defaultdict
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
lib.spa2_debug_trace(_lib.ptr(buf), cap)
_lib.check(lib.spa2_bwd_dq(_lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(do), _lib.ptr(lse), _lib.ptr(delta),
                           _lib.view4(dq), 0, 1, 12, 32760, 128, 128, 64, _lib.ptr(lists.row_ptr), _lib.ptr(lists.row_idx),
                           _lib.ptr(lists.row_order), scale, st), "dq")
torch.cuda.synchronize()
lib.spa2_debug_trace(None, 0)
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
cols = ["mma wait dq_done", "mma wait K", "mma wait dS", "smx wait S", "smx compute", "prod wait Kslot"]
agg, cnt = defaultdict(float), 0
for g in tiles[5:-3]:
    m, s_, pr = rec.get((1, g), {}), rec.get((2, g), {}), rec.get((0, g), {})
    try:
        row = (m[5] - m[1], m[2] - m[5], m[4] - m[3], s_[2] - s_[1], s_[4] - s_[2], pr[2] - pr[1])
    except KeyError:
        continue
    for i, x in enumerate(row):
        agg[i] += x
    cnt += 1
print("mean " + " ".join(f"{agg[i] / max(cnt, 1):>16.0f}" for i in range(len(cols))))
print("     " + " ".join(f"{c:>16s}" for c in cols))
done = [rec[(2, g)].get(4, 0) for g in tiles]
per = sorted(b - a for a, b in zip(done, done[1:]))
print("tile period cycles: median", per[len(per) // 2], "p10", per[len(per) // 10], "p90", per[9 * len(per) // 10])

"""Per-CTA timing of the three attention kernels from a -DSPA2_CTA_TIMES build.

    bash tools/build_alt.sh ctat -DSPA2_CTA_TIMES
    python tools/cta_times.py alt/ctat/libspa2.so

Runs bench-shape steps (Wan2.1-1.3B, 95 % hybrid sparsity), keeps the last step's per-CTA
start/end globaltimer stamps and SM ids, and reports per kernel: the span (first start to last
end), the CTA durations, the busy fraction of the span, and the nanoseconds per kept tile of
each CTA (tiles per CTA from the block lists and the kernels' static item deal).
"""

import ctypes
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_13515_b200 import _lib  # noqa: E402

_lib.use_library(sys.argv[1] if len(sys.argv) > 1 else "alt/ctat/libspa2.so")
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

MAX = 4096
SL = 8
lib = _lib.load()
for f in (lib.spa2_cta_fetch_fwd, lib.spa2_cta_fetch_bwd):
    f.argtypes = [ctypes.c_void_p]
fb = np.zeros(3 * MAX * SL, dtype=np.uint64)
bb = np.zeros(3 * MAX * SL, dtype=np.uint64)
q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
do = torch.randn_like(q)
cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
for it in range(4):
    qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
    res = spa.sparse_attention(qs, ks, vs, cfg)
    res.out.backward(do)
    torch.cuda.synchronize()
    lib.spa2_cta_fetch_fwd(fb.ctypes.data)
    lib.spa2_cta_fetch_bwd(bb.ctypes.data)
bm = res.mask_used
B, H, N, d = q.shape
lists = at.mask_lists(bm, B, H, N)
row_ptr = lists.row_ptr.cpu().numpy()
col_ptr = lists.col_ptr.cpu().numpy()
row_order = lists.row_order.cpu().numpy()
col_order = lists.col_order.cpu().numpy()
n_sm = torch.cuda.get_device_properties(0).multi_processor_count
clk = torch.cuda.clock_rate(0) if hasattr(torch.cuda, "clock_rate") else None


def tiles_persistent(ptr, order, grid):
    lens = np.diff(ptr)[order]
    out = np.zeros(grid, dtype=np.int64)
    items = np.zeros(grid, dtype=np.int64)
    for c in range(grid):
        sel = lens[c::grid]
        out[c] = sel.sum()
        items[c] = (sel > 0).sum()
    return out, items


def report(name, arr, kind, tiles, items):
    a = arr.reshape(3, MAX, SL)[kind].astype(np.int64)
    used = a[:, 0] > 0
    n = int(used.sum())
    st, en, sm = a[:n, 0], a[:n, 1], a[:n, 2]
    t0 = st.min()
    span = (en.max() - t0) / 1e3
    dur = (en - st) / 1e3
    print(f"\n== {name}: {n} CTAs on {len(np.unique(sm))} SMs, span {span:.1f} us")
    print(f"   CTA duration us: min {dur.min():.1f} median {np.median(dur):.1f} max {dur.max():.1f}; "
          f"start spread {(st.max() - t0) / 1e3:.1f} us, end spread {(en.max() - en.min()) / 1e3:.1f} us")
    per_sm = np.zeros(n_sm)
    np.add.at(per_sm, sm, dur)
    print(f"   SM busy (sum of CTA durations / span): mean {per_sm.mean() / span:.3f} min {per_sm.min() / span:.3f}")
    if kind in (1, 2) and (a[:n, 4] > 0).all():
        mhz = (a[:n, 5] - a[:n, 4]) / np.maximum(en - st, 1) * 1e3
        print(f"   SM clock over the CTA lifetime (clock64 / globaltimer): median {np.median(mhz):.0f} MHz "
              f"(min {mhz.min():.0f}, max {mhz.max():.0f})")
    if tiles is not None:
        t = tiles[:n]
        ok = t > 0
        nspt = dur[ok] * 1e3 / t[ok]
        print(f"   tiles/CTA: min {t.min()} median {int(np.median(t))} max {t.max()} (items/CTA median {int(np.median(items[:n]))})")
        print(f"   ns per tile per CTA: median {np.median(nspt):.1f} p10 {np.percentile(nspt, 10):.1f} p90 {np.percentile(nspt, 90):.1f}")
        if kind in (1, 2) and (a[:n, 4] > 0).all():
            cpt = (a[:n, 5] - a[:n, 4])[ok] / t[ok]
            print(f"   cycles per tile per CTA: median {np.median(cpt):.0f} p10 {np.percentile(cpt, 10):.0f} p90 {np.percentile(cpt, 90):.0f}")
        print(f"   ideal span (total tiles x median ns/tile / {n_sm} SMs): {t.sum() * np.median(nspt) / n_sm / 1e3:.1f} us")
    if kind == 0 and (a[:n, 6] > 0).all():  # true lifetime: kernel entry -> TMEM dealloc done
        st, en = a[:n, 3], a[:n, 6]
        t0 = st.min()
        print(f"   true lifetimes (entry -> dealloc done): median {np.median(en - st) / 1e3:.1f} us; "
              f"main loop (start of work -> last PV issued) median {np.median(a[:n, 7] - a[:n, 0]) / 1e3:.1f} us")
    if kind == 0:  # non-persistent: how many CTAs run on each SM over the span
        ev = []
        for s_, e_, m_ in zip(st, en, sm):
            ev += [(s_, m_, 1), (e_, m_, -1)]
        ev.sort()
        occ = np.zeros((n_sm, 4))
        cur = np.zeros(n_sm, dtype=int)
        last = np.full(n_sm, t0)
        for t_, m_, dlt in ev:
            occ[m_, min(cur[m_], 3)] += t_ - last[m_]
            last[m_] = t_
            cur[m_] += dlt
        tot = occ.sum(1, keepdims=True)
        fr = (occ / tot).mean(0)
        print(f"   fraction of each SM's time (first start to its last end) with 0/1/2/3+ CTAs: "
              f"{fr[0]:.3f} {fr[1]:.3f} {fr[2]:.3f} {fr[3]:.3f}")
        gaps = []
        for m_ in range(n_sm):
            sel = np.flatnonzero(sm == m_)
            ss, ee = np.sort(st[sel]), np.sort(en[sel])
            # a new CTA starts after one retires: match the k-th start beyond the first two to the (k-2)-th end
            if len(ss) > 2:
                gaps += list(ss[2:] - ee[:len(ss) - 2])
        gaps = np.asarray(gaps) / 1e3
        print(f"   retire -> next start on the SM (us): median {np.median(gaps):.2f} p90 {np.percentile(gaps, 90):.2f}")
        ent = a[:n, 3]
        if (ent > 0).all():
            pro = (st - ent) / 1e3
            print(f"   kernel entry -> start of work (prologue, us): median {np.median(pro):.2f} p90 {np.percentile(pro, 90):.2f}")
        for nm, i0, i1 in (("last PV issued -> epilogue start", 7, 4), ("epilogue start -> TMA store done", 4, 5),
                           ("TMA store done -> end", 5, 1), ("end -> dealloc done", 1, 6)):
            x, y = a[:n, i0], a[:n, i1]
            if (x > 0).all() and (y > 0).all():
                dd = (y - x) / 1e3
                print(f"   {nm} (us): median {np.median(dd):.2f} p90 {np.percentile(dd, 90):.2f}")
    return st, en, sm


fwd_tiles = np.diff(row_ptr)[row_order]
report("k_fwd", fb, 0, fwd_tiles, np.ones_like(fwd_tiles))
grid_b = n_sm
tq, iq = tiles_persistent(row_ptr, row_order, grid_b)
report("k_dq3", bb, 1, tq, iq)
tk, ik = tiles_persistent(col_ptr, col_order, grid_b)
report("k_dkdv5", bb, 2, tk, ik)
print(f"\nkept tiles {int(np.diff(row_ptr).sum())}, clock {clk}")

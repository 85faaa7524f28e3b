"""Static vs dynamic work assignment of the persistent kernels at the bench workload's hybrid
mask: per-CTA load (max / mean) for the current launch order (head-major, longest-first
within a head) dealt round-robin (static, today) and for dynamic list scheduling of the same
order (each item to the first CTA that frees up).  Per-item cost = kept tiles + `ovh` tiles."""
import heapq, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
bm = at._hybrid_mask_device(q, k, spa.SparsityConfig(0.03, 0.2, 128, 64), False)
keep = bm.keep.view(12, 256, 512).cpu().numpy()
for name, lens2d, ctas in (("fwd rows", keep.sum(-1), 296), ("dq rows", keep.sum(-1), 148),
                           ("dkdv cols", keep.sum(-2), 148)):
    for ovh in (0.0, 2.0):
        cost = np.concatenate([np.sort(r)[::-1] for r in lens2d]).astype(float)
        cost = cost + ovh * (cost > 0)
        rr = np.zeros(ctas)
        for i, c in enumerate(cost):
            rr[i % ctas] += c
        h = [(0.0, b) for b in range(ctas)]
        dyn = np.zeros(ctas)
        for c in cost:
            t, b = heapq.heappop(h)
            dyn[b] = t + c
            heapq.heappush(h, (t + c, b))
        m = cost.sum() / ctas
        print(f"{name:10s} ctas {ctas} ovh {ovh}: mean {m:.1f}  static round-robin max/mean {rr.max() / m:.3f}  "
              f"dynamic {dyn.max() / m:.3f}")

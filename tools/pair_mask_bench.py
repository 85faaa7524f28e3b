"""dK/dV kernel time on a mask whose adjacent key blocks are correlated (kept in pairs, as in
real video attention) versus an uncorrelated mask of the same block sparsity.  Run once per
SPA2_DKDV_VARIANT (the variant is chosen per process)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import masker as mk  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

H, N, d = 12, 32760, 128
t_m, t_n = -(-N // 128), -(-N // 64)
q, k, v = wan_like_qkv(1, H, N, d, 0.9, seed=5)
do = torch.randn_like(q)
rng = np.random.default_rng(0)
dens = 0.05
uncorr = rng.random((1, H, t_m, t_n)) < dens
pairs = rng.random((1, H, t_m, (t_n + 1) // 2)) < dens
corr = np.repeat(pairs, 2, axis=3)[..., :t_n]
for name, keep in (("uncorrelated", uncorr), ("paired", corr)):
    keep[..., np.arange(t_m), np.arange(t_m) * 2 % t_n] = True  # >= 1 kept block per row
    bm = mk.BlockMask(torch.as_tensor(keep, device="cuda"), 128, 64, N)
    spa.attention_backward(q, k, v, bm, do)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        spa.attention_backward(q, k, v, bm, do)
    b.record()
    torch.cuda.synchronize()
    print(f"variant {os.environ.get('SPA2_DKDV_VARIANT', '5')} {name:13s} sparsity {1 - keep.mean():.4f}  "
          f"fwd-less bwd {a.elapsed_time(b) / 10:.3f} ms")

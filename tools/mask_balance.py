"""Why do equal-sparsity masks run at different speeds?  Per-kernel time and list-length
statistics for top-k / top-p / hybrid masks at ~95 % block sparsity (Wan2.1-1.3B shape)."""
import math, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402

q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=0)
do = torch.randn_like(q)
scale = 1 / math.sqrt(128)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for name, cfg in (("top-k 0.049", spa.SparsityConfig(0.049023, 0.0, 128, 64)),
                  ("top-p 0.1996", spa.SparsityConfig(0.0, 0.199567, 128, 64)),
                  ("hybrid k.03 p.2", spa.SparsityConfig(0.03, 0.2, 128, 64))):
    bm = at._hybrid_mask_device(q, k, cfg, False)
    lists = at.mask_lists(bm, 1, 12, 32760)
    keep = bm.keep.view(12, 256, 512)
    rc, cc = keep.sum(-1).float(), keep.sum(-2).float()
    o, lse = at.fwd(q, k, v, lists, scale)
    tf = t(lambda: at.fwd(q, k, v, lists, scale))
    tb = t(lambda: at.bwd(q, k, v, o, do, lse, lists, scale))
    print(f"{name:16s} sparsity {bm.sparsity():.4f}  rows: mean {rc.mean():.1f} max {rc.max():.0f}  "
          f"cols: mean {cc.mean():.1f} max {cc.max():.0f} std {cc.std():.1f}  fwd {tf:.3f} ms  bwd {tb:.3f} ms")

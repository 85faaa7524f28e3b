"""Developer timing of the individual hot-path stages at a Wan2.1 shape (CUDA events).

    python tools/time_kernels.py [--n 32760 --heads 12 --d 128 --s 0.9 --k 0.03 --p 0.2]

Prints per-stage milliseconds and achieved TFLOP/s (kept-block FLOPs) / GB/s.  Not the
benchmark of record (that is bench.py); used to iterate on kernels.
"""

import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import attention as at  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402


def timed(fn, reps=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32760)
    ap.add_argument("--heads", type=int, default=12)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--s", type=float, default=0.9)
    ap.add_argument("--k", type=float, default=0.03)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--bwd", action="store_true")
    a = ap.parse_args()
    q, k, v = wan_like_qkv(1, a.heads, a.n, a.d, a.s, seed=0)
    do = torch.randn_like(q)
    cfg = spa.SparsityConfig(a.k, a.p, 128, 64)
    t_mask = timed(lambda: at._hybrid_mask_device(q, k, cfg, False))
    bm = at._hybrid_mask_device(q, k, cfg, False)
    if a.dense:
        bm = spa.BlockMask._trusted(torch.ones_like(bm.keep), 128, 64, a.n)
    B, H, N, d = q.shape
    t_lists = timed(lambda: at.build_lists(at._native_keep(bm, B, H, N)))
    lists = at.mask_lists(bm, B, H, N)
    scale = 1 / math.sqrt(d)
    t_fwd = timed(lambda: at.fwd(q, k, v, lists, scale))
    kept = int(bm.keep.sum())
    tiles = kept  # ragged tails ignored in this dev estimate
    fl_fwd = 4.0 * 128 * 64 * d * tiles
    print(f"shape B{B} H{H} N{N} d{d} sparsity {bm.sparsity():.4f} kept {kept}")
    print(f"masker (pool+score+softmax+select) {t_mask:.3f} ms   lists {t_lists:.3f} ms")
    print(f"fwd {t_fwd:.3f} ms  {fl_fwd / t_fwd / 1e9:.1f} TFLOP/s (kept)  "
          f"dense-equiv {4.0 * B * H * N * N * d / t_fwd / 1e9:.1f} TFLOP/s")
    if a.bwd:
        o, lse = at.fwd(q, k, v, lists, scale)
        t_bwd = timed(lambda: at.bwd(q, k, v, o, do, lse, lists, scale))
        print(f"bwd {t_bwd:.3f} ms  {10.0 * 128 * 64 * d * tiles / t_bwd / 1e9:.1f} TFLOP/s (kept)")


if __name__ == "__main__":
    main()

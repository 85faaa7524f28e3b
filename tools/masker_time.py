"""Masker stage timings at the bench shape (back-to-back launches between two CUDA events),
plus a bit-level checksum of the pooled scores so A/B builds can be compared for equality.

    python tools/masker_time.py [--lib alt/x/libspa2.so]
"""

import argparse
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_13515_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=None)
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    if a.lib:
        _lib.use_library(a.lib)
    import paper_2602_13515_b200 as spa
    from paper_2602_13515_b200 import attention as at
    from paper_2602_13515_b200 import masker as mk
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=1000)
    cfg = spa.SparsityConfig(0.03, 0.2, 128, 64)
    flag = torch.zeros((1,), dtype=torch.int32, device="cuda")

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    nbytes = q.numel() * 2
    t_k1 = timed(lambda: mk._pooled_probs(q, k, 128, 64, flag, softmax=False))
    t_k0 = timed(lambda: at._scan_finite(flag, v))
    t_mask = timed(lambda: at._hybrid_mask_device(q, k, cfg, flag))
    scores = mk._pooled_probs(q, k, 128, 64, flag, softmax=False)
    keep = at._hybrid_mask_device(q, k, cfg, flag)
    torch.cuda.synchronize()
    h = hashlib.sha256(scores.cpu().numpy().tobytes()).hexdigest()[:16]
    hk = hashlib.sha256(keep.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"K1 pool+scores {t_k1 * 1e3:7.1f} us ({2 * nbytes / t_k1 / 1e6:6.0f} GB/s on Q+K)   "
          f"K0 scan(v) {t_k0 * 1e3:6.1f} us ({nbytes / t_k0 / 1e6:6.0f} GB/s)   masker {t_mask * 1e3:6.1f} us   "
          f"scores sha {h} keep sha {hk} flag {int(flag.item())}")


if __name__ == "__main__":
    main()

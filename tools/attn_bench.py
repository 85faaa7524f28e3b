"""The reference's ``attn-bench`` (cli.py:200-241) on the B200 kernels: dense vs masked
attention at several sequence lengths and target sparsities, written as ``bench.csv`` and
``timings.json`` in the reference's layout (formats.py) so its tooling reads GPU runs.

    python tools/attn_bench.py --out runs/attn_bench [--sizes 4096,32760 --d 128 --sparsities 0.9,0.95 --reps 5]

Inputs are bf16 N(0,1) q/k/v (the reference uses float64 numpy); masks keep a fixed count of
random key blocks per query block as the reference's _bench_mask (cli.py:176-185); times are
CUDA-event seconds of the forward (the reference times sparse_attention_with_mask)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import formats as fm  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--sizes", default="4096,32760")
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--sparsities", default="0.8,0.9,0.95")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--format", choices=("csv", "json"), default="csv")
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    rng = np.random.Generator(np.random.PCG64(args.seed))
    b_q, b_kv, d = 128, 64, args.d
    rows, timings = [], []
    for n in (int(x) for x in args.sizes.split(",")):
        g = torch.Generator(device="cuda").manual_seed(n)
        q, k, v = (torch.randn(n, d, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
        t_m, t_n = -(-n // b_q), -(-n // b_kv)
        dense_bm = spa.BlockMask(torch.ones(t_m, t_n, dtype=torch.bool), b_q, b_kv, n)
        dense_out = spa.sparse_attention_with_mask(q, k, v, dense_bm).out
        dense_s = timed(lambda: spa.sparse_attention_with_mask(q, k, v, dense_bm), args.reps)
        for target in (float(x) for x in args.sparsities.split(",")):
            per_row = max(1, round((1.0 - target) * t_n))
            keep = np.zeros((t_m, t_n), dtype=bool)
            for i in range(t_m):
                keep[i, rng.choice(t_n, size=per_row, replace=False)] = True
            bm = spa.BlockMask(torch.as_tensor(keep), b_q, b_kv, n)
            counter = spa.BlockCounter()
            out = spa.sparse_attention_with_mask(q, k, v, bm, counter=counter).out
            sparse_s = timed(lambda: spa.sparse_attention_with_mask(q, k, v, bm), args.reps)
            total = keep.size
            assert counter.count == int(keep.sum()), "computed blocks must equal kept blocks"
            ratio = counter.count / total
            max_dev = float((out.float() - dense_out.float()).abs().max())
            rows.append([n, d, b_q, b_kv, 1.0 - ratio, counter.count, total, ratio, max_dev])
            timings.append({"n": n, "sparsity": 1.0 - ratio, "dense_s": dense_s, "sparse_s": sparse_s,
                            "speedup": dense_s / sparse_s})
            print(f"n={n} sparsity={1.0 - ratio:.4f} blocks {counter.count}/{total} speedup {dense_s / sparse_s:.2f}x")
    fm.write_table(args.out, "bench", fm.BENCH_HEADER, rows, args.format)
    fm.write_json(args.out, "timings", {"reps": args.reps, "entries": timings})


if __name__ == "__main__":
    main()

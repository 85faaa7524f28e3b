"""Config 4 (Wan2.1-14B 720p attention: N=75600, H=40, d=128, k=0.03, p=0.16): head-sharded
work per GPU at 1/2/4/8 GPUs, measured on one B200.

Head sharding has no data-path collective (each rank owns H/P heads end to end), so the
per-GPU step time for H/P heads IS the P-GPU step time; this tool measures it for P = 1, 2,
4, 8 and prints the implied speedup T(P=1)/T(P).  (The driver's multi-GPU bench runs the
same per-rank work on real ranks.)

    python tools/cfg4_scaling.py [--steps 5]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200.synthetic import wan_like_qkv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--rounds", type=int, default=5)
    args = ap.parse_args()
    N, D, H = 75600, 128, 40
    cfg = spa.SparsityConfig(0.03, 0.16, 128, 64)
    q, k, v = wan_like_qkv(1, H, N, D, 0.8, seed=40)
    do = torch.randn(q.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(41)).to(q.dtype)
    steps = {}
    for P in (1, 2, 4, 8):
        h = H // P
        qs, ks, vs, dos = (t[:, :h].contiguous() for t in (q, k, v, do))

        def step(qs=qs, ks=ks, vs=vs, dos=dos):
            a, b, c = (t.detach().requires_grad_(True) for t in (qs, ks, vs))
            res = spa.sparse_attention(a, b, c, cfg)
            res.out.backward(dos)
            return res

        steps[P] = (h, step, step().mask_used.sparsity())
    # the four per-rank workloads are timed in interleaved rounds (median over rounds), so every
    # P sees the same clock / power state instead of one long run per P
    times = {P: [] for P in steps}
    for _ in range(args.rounds):
        for P, (h, step, _) in steps.items():
            for _ in range(args.warmup):
                step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                step()
            e1.record()
            torch.cuda.synchronize()
            times[P].append(e0.elapsed_time(e1) / args.steps)
    spa.check_pending()
    results = []
    for P, (h, _, sp) in steps.items():
        ms = sorted(times[P])[len(times[P]) // 2]
        dense = 14 * h * N * N * D
        results.append({"gpus": P, "heads_per_gpu": h, "ms_per_step": ms, "block_sparsity": sp,
                        "dense_equiv_tflops_per_gpu": dense / ms / 1e9, "rounds_ms": [round(t, 3) for t in times[P]]})
    base = results[0]["ms_per_step"]
    for r in results:
        r["speedup_vs_1gpu"] = base / r["ms_per_step"]
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

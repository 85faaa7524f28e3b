"""Config 5: time one sparse-attention distillation step (Algorithm 2) on a random-init
Wan2.1-1.3B DiT at the 480p latent (32760 tokens), against the same step with a dense
student.

    python tools/distill_step.py [--layers 30] [--steps 3] [--warmup 2] [--k 0.03 --p 0.2]

Prints one JSON line per student (sparse, dense): ms/step, the block sparsity the masker
chose in the first layer, and the loss."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_13515_b200 as spa  # noqa: E402
from paper_2602_13515_b200 import distill as ds  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=30)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--k", type=float, default=0.03)
    ap.add_argument("--p", type=float, default=0.2)
    ap.add_argument("--dense-student", action="store_true", help="also time a dense-attention student")
    args = ap.parse_args()
    torch.manual_seed(0)
    cfg = ds.WanConfig(layers=args.layers)
    teacher = ds.WanDiT(cfg).cuda().to(torch.bfloat16).eval()
    teacher.set_attention(None)
    for p in teacher.parameters():
        p.requires_grad_(False)
    x_t, t, text = ds.synthetic_batch(cfg)
    runs = [("sparse", spa.SparsityConfig(args.k, args.p, 128, 64))]
    if args.dense_student:
        runs.append(("dense", None))
    for name, scfg in runs:
        student = ds.make_student(teacher, scfg) if scfg is not None else ds.make_student(teacher, spa.SparsityConfig(1, 1, 128, 64))
        if scfg is None:
            student.set_attention(None)
        student.train()
        opt = torch.optim.AdamW(student.parameters(), lr=1e-5, fused=True)
        sparsity = None
        if scfg is not None:  # the mask the first layer's masker picks on this input
            blk = student.blocks[0].attn
            with torch.no_grad():
                seen = {}
                orig = spa.attention._run

                def spy(q4, k4, v4, bm, *args, **kw):
                    seen.setdefault("sp", bm.sparsity())
                    return orig(q4, k4, v4, bm, *args, **kw)
                spa.attention._run = spy
                try:
                    student(x_t, t, text)
                finally:
                    spa.attention._run = orig
                sparsity = seen.get("sp")
            del blk
        for _ in range(args.warmup):
            loss = ds.distill_step(student, teacher, opt, x_t, t, text)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            loss = ds.distill_step(student, teacher, opt, x_t, t, text)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        print(json.dumps({"workload": "config 5: Wan2.1-1.3B DiT distillation step (random init, 480p latent, "
                                      "32760 tokens, teacher dense)", "student": name, "layers": args.layers,
                          "ms_per_step": ms, "block_sparsity_layer0": sparsity, "loss": float(loss),
                          "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
        del student, opt
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of record: sparse-attention fwd+bwd at 95 % block sparsity, Wan2.1 shape.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

One step = the trainable operator of the reference's hot path on one batch:
``sparse_attention(q, k, v, SparsityConfig(0.03, 0.2, 128, 64))`` (pooled map -> hybrid
Top-k∪Top-p select -> block lists -> block-sparse forward) followed by its backward
(δ, dQ, dK/dV).  Workload = BASELINE.json configs[1]: Wan2.1-1.3B 480p attention,
B=1, H=12, N=32760, d=128, bf16, synthetic inputs calibrated to ≈95 % block sparsity.
Multi-GPU: every rank runs its own 12-head problem (head sharding, no data-path
collective) -> weak scaling; timing = max over ranks.

value = dense-equivalent TFLOP/s = 14·B·H·N²·d / step time, summed over ranks.
"""

from __future__ import annotations

import argparse
import datetime as _dt
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn fwd+bwd ms & effective TFLOPS @95% sparsity, Wan2.1 shape, 1-8 GPU"
UNIT = "TFLOP/s (dense-equivalent, 14*B*H*N^2*d per step)"
WORKLOAD = dict(B=1, H=12, N=32760, d=128, b_q=128, b_kv=64, k_frac=0.03, p_frac=0.2, offset_scale=0.9)
FLOP_MULT = 14  # fwd 4 + bwd 10, per (query, key, feature) triple


def dense_equiv_flops(w=WORKLOAD) -> float:
    return float(FLOP_MULT) * w["B"] * w["H"] * w["N"] ** 2 * w["d"]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return {"bf16_tflops": float(pk["bf16_tflops"]), "bf16_tflops_sustained": float(pk["bf16_tflops_sustained"]),
                "hbm_gbs": float(pk["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------------------
# CPU arm: the reference algorithm (oracle port, float64 numpy) on the host's cores
# ---------------------------------------------------------------------------------------
_CPU = {}


def _cpu_worker_init(seed: int, n: int, d: int, s: float):
    import numpy as np
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    rng = np.random.Generator(np.random.PCG64(seed))
    b_q, b_kv = 128, 64
    t_m, t_n = -(-n // b_q), -(-n // b_kv)
    q = rng.normal(size=(n, d)) + np.repeat(rng.normal(size=(t_m, d)) * s, b_q, axis=0)[:n]
    k = rng.normal(size=(n, d)) + np.repeat(rng.normal(size=(t_n, d)) * s, b_kv, axis=0)[:n]
    v = rng.normal(size=(n, d))
    do = rng.normal(size=(n, d))
    _CPU.update(q=q, k=k, v=v, do=do, t_m=t_m)


def _cpu_sample(args):
    """Masker (pooled map + hybrid select for the sampled query blocks) + tiled forward +
    LSE-recompute backward over `rows` query blocks of one head, as the reference runs them
    (masker.py:100-146, attention.py:73-166).  Returns (seconds, kept blocks)."""
    import numpy as np

    import oracle

    start_blk, rows, k_frac, p_frac = args
    q, k, v, do, t_m = _CPU["q"], _CPU["k"], _CPU["v"], _CPU["do"], _CPU["t_m"]
    start_blk = start_blk % max(1, t_m - rows)
    sl = slice(start_blk * 128, (start_blk + rows) * 128)
    t0 = time.perf_counter()
    q_bar = oracle.block_mean_pool(q[sl], 128)
    k_bar = oracle.block_mean_pool(k, 64)
    probs = oracle.softmax_rows((q_bar @ k_bar.T) / math.sqrt(q.shape[1]))
    keep = oracle.hybrid_keep(probs, k_frac, p_frac)
    oracle.attention_backward(q[sl], k, v, keep, 128, 64, do[sl])  # includes the forward recompute
    return time.perf_counter() - t0, int(keep.sum())


def cpu_reference(steps: int, warmup: int, w=WORKLOAD, target_step_s: float = 0.12):
    """Time the CPU reference path on a bounded sample; returns a dict with value (same
    metric/unit as the GPU arm) and the sample description."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    workers = max(1, min(cores, w["B"] * w["H"]))
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers, initializer=_cpu_worker_init, initargs=(7, w["N"], w["d"], w["offset_scale"])) as pool:
        t1, _ = pool.apply(_cpu_sample, ((0, 1, w["k_frac"], w["p_frac"]),))
        rows = max(1, min(16, int(round(target_step_s / max(t1, 1e-3)))))
        times, kept = [], []
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_sample, [((it * 7 + r * 37), rows, w["k_frac"], w["p_frac"]) for r in range(workers)])
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
                kept.append(sum(x[1] for x in res))
    t_step = statistics.median(times)
    t_m = -(-w["N"] // w["b_q"])
    frac_of_job = workers * rows / (w["B"] * w["H"] * t_m)  # share of the job's query blocks per step
    value = dense_equiv_flops(w) * frac_of_job / t_step / 1e12
    full_job_ms = t_step / frac_of_job * 1e3
    return {
        "value": value, "unit": UNIT, "cores": workers, "kind": "port",
        "sample": (f"oracle/ float64 numpy port of the reference (masker + tiled fwd + LSE-recompute bwd), "
                   f"{workers} process(es) x {rows} query-block row(s) of one Wan2.1-1.3B head each per step "
                   f"(1 BLAS thread per process), {steps} steps; {statistics.mean(kept) / workers / rows:.1f} kept "
                   f"blocks per row; full 12-head job extrapolated to {full_job_ms / 1e3:.1f} s"),
        "full_job_ms": full_job_ms,
        "host_cores": cores,
    }


# ---------------------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["timestamp", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_uuid: str | None):
        self.proc = None
        self.path = os.path.join("/tmp", f"spa2_clocks_{os.getpid()}.csv")
        cmd = ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "100"]
        if device_uuid:
            cmd[1:1] = ["-i", device_uuid]
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(cmd, stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, t_start: float, t_end: float):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons, n_all = [], [], set(), 0
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) != len(self.FIELDS):
                    continue
                n_all += 1
                try:
                    ts = _dt.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if not (t_start - 0.05 <= ts <= t_end + 0.05):
                    continue
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                for name, val in zip(self.NAMES, parts[3:]):
                    if val.lower() == "active":
                        reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "samples_total": n_all}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------
def tile_flops(keep, N: int, d: int, mult: int) -> float:
    """Σ over kept (i, j) of mult · r_i · c_j · d with ragged true row/col counts."""
    import torch

    t_m, t_n = keep.shape[-2:]
    r = torch.full((t_m,), 128.0, device=keep.device, dtype=torch.float64)
    r[-1] = N - 128 * (t_m - 1)
    c = torch.full((t_n,), 64.0, device=keep.device, dtype=torch.float64)
    c[-1] = N - 64 * (t_n - 1)
    return float(mult * d * (keep.double() * r[:, None] * c[None, :]).sum())


def gpu_arm(args, rank: int, world: int, dev):
    import torch
    import torch.distributed as dist

    import paper_2602_13515_b200 as spa
    from paper_2602_13515_b200 import _lib
    from paper_2602_13515_b200 import attention as at
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    w = WORKLOAD
    B, H, N, d = w["B"], w["H"], w["N"], w["d"]
    cfg = spa.SparsityConfig(w["k_frac"], w["p_frac"], w["b_q"], w["b_kv"])
    q, k, v = wan_like_qkv(B, H, N, d, w["offset_scale"], seed=1000 + rank)
    do = torch.randn(q.shape, device=dev, generator=torch.Generator(device=dev).manual_seed(77 + rank)).to(q.dtype)

    def step():
        qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
        res = spa.sparse_attention(qs, ks, vs, cfg)
        res.out.backward(do)
        return res

    def barrier():
        if world > 1:
            dist.barrier()

    res = step()
    keep = res.mask_used.keep
    sparsity = res.mask_used.sparsity()
    for _ in range(max(0, args.warmup - 1)):
        step()
    torch.cuda.synchronize()

    timed_names = ("spa2_fwd", "spa2_bwd_dq_delta", "spa2_bwd_dkdv", "spa2_pooled_scores", "spa2_select_scores",
                   "spa2_pooled_map", "spa2_select", "spa2_build_lists")
    _lib.STATS.timing = {n: [] for n in timed_names}
    launches0 = _lib.STATS.launches
    uuid = None
    try:
        uuid = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        pass
    sampler = ClockSampler(uuid)
    time.sleep(0.6)  # nvidia-smi start-up
    barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    t_wall1 = time.time()
    clocks = sampler.stop(t_wall0, t_wall1)
    launches = _lib.STATS.launches - launches0
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    per_kernel_ms = {n: (sum(a.elapsed_time(b) for a, b in lst) / len(lst) if lst else 0.0)
                     for n, lst in _lib.STATS.timing.items()}
    _lib.STATS.timing = None

    # ---- roofline of the dominant kernel (tensor-bound attention kernels) ----
    kflops = {"spa2_fwd": tile_flops(keep, N, d, 4), "spa2_bwd_dq_delta": tile_flops(keep, N, d, 6),
              "spa2_bwd_dkdv": tile_flops(keep, N, d, 8)}
    dom = max(kflops, key=lambda n: per_kernel_ms[n])
    peaks = load_peaks()
    achieved = kflops[dom] / (per_kernel_ms[dom] * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("kernels", {}).get(dom, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    # the kernel runs inside a long back-to-back step loop (the board reaches its power cap),
    # so it is held against the SUSTAINED bf16 GEMM figure; a short run uses the burst one
    sustained = args.steps * ms_step >= 100.0
    peak = peaks["bf16_tflops_sustained"] if sustained else peaks["bf16_tflops"]
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peaks["source"] + (", sustained bf16 GEMM (long timed loop)" if sustained
                                                  else ", burst bf16 GEMM"),
                "flops_per_launch": kflops[dom], "ms_per_launch": per_kernel_ms[dom]}

    out = {"ms_step": ms_step, "sparsity": sparsity, "clocks": clocks, "launches": launches,
           "per_kernel_ms": per_kernel_ms, "roofline": roofline, "kflops": kflops}

    # ---- e2e through the public API with host buffers ----
    if not args.no_e2e:
        from paper_2602_13515_b200.host import HostPipeline

        hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, do))
        outs = [torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(4)]
        pipe = HostPipeline(dev, groups=args.e2e_groups)

        def e2e_step():
            pipe.fwd_bwd(hq, hk, hv, hdo, cfg, *outs)

        for _ in range(2):
            e2e_step()
        n_e2e = max(3, min(args.steps, 60))
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n_e2e):
            e2e_step()
        b.record()
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e_step = e_ms / n_e2e
        nbytes = q.numel() * q.element_size()
        out["e2e"] = {"value": world * dense_equiv_flops() / (e_step * 1e-3) / 1e12, "unit": UNIT,
                      "h2d_bytes_per_step": 4 * nbytes, "d2h_bytes_per_step": 4 * nbytes, "ms_per_step": e_step,
                      "steps": n_e2e, "api": f"paper_2602_13515_b200.host.HostPipeline.fwd_bwd "
                                             f"({args.e2e_groups} head groups, H2D/compute/D2H overlapped)"}

    # ---- dense baselines on the same GPU (rank 0, N=1) ----
    if rank == 0 and world == 1 and not args.no_dense:
        dense = {}
        full = spa.BlockMask._trusted(torch.ones_like(keep), 128, 64, N)
        lists = at.mask_lists(full, B, H, N)
        scale = 1.0 / math.sqrt(d)

        def own_dense():
            o, lse = at.fwd(q, k, v, lists, scale)
            at.bwd(q, k, v, o, do, lse, lists, scale)

        dense["own_kernels_all_blocks_ms"] = _time(own_dense, 3, 1)
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel

            def sdpa(backend):
                def f():
                    qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
                    with sdpa_kernel(backend):
                        o = torch.nn.functional.scaled_dot_product_attention(qs, ks, vs)
                    o.backward(do)
                return f

            dense["cudnn_sdpa_ms"] = _time(sdpa(SDPBackend.CUDNN_ATTENTION), 3, 1)
            try:
                dense["flash_sdpa_ms"] = _time(sdpa(SDPBackend.FLASH_ATTENTION), 3, 1)
            except Exception as e:  # pragma: no cover
                dense["flash_sdpa_error"] = str(e)[:120]
        except Exception as e:  # pragma: no cover
            dense["cudnn_sdpa_error"] = str(e)[:200]
        best = min(v for kk, v in dense.items() if kk.endswith("_ms"))
        dense["speedup_vs_best_dense"] = best / ms_step
        dense["speedup_vs_own_dense"] = dense["own_kernels_all_blocks_ms"] / ms_step
        out["dense_baselines"] = dense
    return out


def _time(fn, reps, warm):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def config_dict(world: int, sparsity=None):
    w = WORKLOAD
    c = {"workload": "Wan2.1-1.3B 480p attention (BASELINE configs[1]): B=1 H=12 N=32760 d=128 per GPU",
         "B": w["B"], "H": w["H"], "N": w["N"], "d": w["d"], "b_q": w["b_q"], "b_kv": w["b_kv"],
         "k_frac": w["k_frac"], "p_frac": w["p_frac"], "mask": "hybrid top-k ∪ top-p, rebuilt every step",
         "parallelism": f"head-sharded x{world} (each rank its own 12-head problem, no collective)",
         "l2": "inputs larger than L2 (q+k+v+dO = 403 MB per GPU), no flush"}
    if sparsity is not None:
        c["block_sparsity"] = round(sparsity, 5)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--e2e-groups", type=int, default=6)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        ref_steps = min(args.steps, 60)  # each step is a bounded CPU sample; keep the run to ~minutes
        cpu = cpu_reference(ref_steps, min(args.warmup, 3))
        line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": ref_steps,
                "warmup": min(args.warmup, 3), "ms_per_step": cpu["full_job_ms"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (Wan2.1-shaped, seeded)",
                "config": config_dict(1), "impl": "reference",
                "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    try:
        r = gpu_arm(args, rank, world, dev)
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = cpu_reference(20, 2)
        if rank == 0:
            value = world * dense_equiv_flops() / (r["ms_step"] * 1e-3) / 1e12
            line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": r["ms_step"], "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "bf16",
                    "data": "synthetic (Wan2.1-shaped q/k/v: N(0,1) + per-block N(0,0.81) offsets, seeded)",
                    "config": config_dict(world, r["sparsity"]), "roofline": r["roofline"],
                    "gpu_launches": r["launches"], "clocks": r["clocks"],
                    "per_kernel_ms": {k.replace("spa2_", ""): round(v, 5) for k, v in r["per_kernel_ms"].items()}}
            if "e2e" in r:
                line["e2e"] = r["e2e"]
            if "dense_baselines" in r:
                line["dense_baselines"] = r["dense_baselines"]
            if cpu is not None:
                line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

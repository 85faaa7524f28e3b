#!/usr/bin/env python
"""Benchmark of record: sparse-attention fwd+bwd at 95 % block sparsity, Wan2.1 shape.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

One step = the trainable operator of the reference's hot path on one batch, through the
public API with its default arguments: ``sparse_attention(q, k, v, SparsityConfig(0.03,
0.2, 128, 64))`` (finiteness scan -> pooled map -> hybrid Top-k∪Top-p select -> block
lists -> block-sparse forward) followed by its backward (δ, dQ, dK/dV).
Workload = BASELINE.json configs[1]: Wan2.1-1.3B 480p attention, B=1, H=12, N=32760,
d=128, bf16, synthetic inputs calibrated to ≈95 % block sparsity.

Multi-GPU (N > 1): every rank runs its own 12-head configs[1] problem (batch-sharded weak
scaling, no data-path collective) -> `value`; plus a `cfg4` leg on BASELINE configs[3]
(Wan2.1-14B 720p, H=40, N=75600): the ONE problem head-sharded 40/N per rank with the
NCCL all-gather of O and dQ/dK/dV, and the Ulysses sequence-parallel form (all-to-all
over NCCL, overlapped with the per-head-group compute), comm time reported separately.

value = dense-equivalent TFLOP/s = 14·B·H·N²·d / step time, summed over ranks.
"""

from __future__ import annotations

import argparse
import datetime as _dt
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")  # the unmodified reference (pip --target, git-ignored)

METRIC = "sparse-attn fwd+bwd ms & effective TFLOPS @95% sparsity, Wan2.1 shape, 1-8 GPU"
UNIT = "TFLOP/s (dense-equivalent, 14*B*H*N^2*d per step)"
WORKLOAD = dict(B=1, H=12, N=32760, d=128, b_q=128, b_kv=64, k_frac=0.03, p_frac=0.2, offset_scale=0.9)
CFG4 = dict(B=1, H=40, N=75600, d=128, k_frac=0.03, p_frac=0.16, offset_scale=0.8)
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
# CPU arm: the reference itself (baseline/_ref/sparseattn_lab) on the host's cores;
# the oracle port only if the reference is not installed
# ---------------------------------------------------------------------------------------
_CPU = {}


def reference_installed() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "sparseattn_lab", "attention.py"))


def _host_inputs(seed: int, n: int, d: int, s: float):
    """One head of configs[1]-distributed inputs (N(0,1) + per-block N(0, s²) offsets) in float64."""
    import numpy as np

    rng = np.random.Generator(np.random.PCG64(seed))
    t_m, t_n = -(-n // 128), -(-n // 64)
    q = rng.normal(size=(n, d)) + np.repeat(rng.normal(size=(t_m, d)) * s, 128, axis=0)[:n]
    k = rng.normal(size=(n, d)) + np.repeat(rng.normal(size=(t_n, d)) * s, 64, axis=0)[:n]
    return q, k, rng.normal(size=(n, d)), rng.normal(size=(n, d))


def _import_reference():
    """Import the UNMODIFIED reference from baseline/_ref — ahead of the repo root, whose
    ``sparseattn_lab`` is this package's drop-in shim."""
    if sys.path[0] != REF_DIR:
        sys.path.insert(0, REF_DIR)
    for m in [m for m in sys.modules if m == "sparseattn_lab" or m.startswith("sparseattn_lab.")]:
        del sys.modules[m]
    import sparseattn_lab.attention as at
    import sparseattn_lab.masker as mk

    if not os.path.abspath(at.__file__).startswith(REF_DIR):
        raise RuntimeError(f"imported {at.__file__}, not the reference under {REF_DIR}")
    return at, mk


def _cpu_worker_init(seed: int, n: int, d: int, s: float, kind: str, blas_threads):
    import numpy  # noqa: F401  (threadpool_limits acts on the BLAS / OpenMP libraries already loaded)
    from threadpoolctl import threadpool_limits

    if blas_threads is not None:
        threadpool_limits(blas_threads)
    _CPU.update(zip(("q", "k", "v", "do"), _host_inputs(seed, n, d, s)))
    _CPU["kind"] = kind
    if kind == "reference":
        _CPU["at"], _CPU["mk"] = _import_reference()


def _cpu_head(args):
    """One head's fwd+bwd.  kind "reference": the reference's public API, exactly as its own
    callers pair them (flowmatch.py:263-264, 317): sparse_attention (masker + tiled forward)
    then attention_backward (LSE-recompute backward).  kind "port": the oracle restatement
    of the same algorithm on `rows` query blocks (only when the reference is absent).
    Returns (seconds, kept blocks, query-block rows processed)."""
    k_frac, p_frac, rows = args
    q, k, v, do = _CPU["q"], _CPU["k"], _CPU["v"], _CPU["do"]
    t0 = time.perf_counter()
    if _CPU["kind"] == "reference":
        at, mk = _CPU["at"], _CPU["mk"]
        res = at.sparse_attention(q, k, v, mk.SparsityConfig(k_frac, p_frac, 128, 64))
        at.attention_backward(q, k, v, res.mask_used, do)
        kept, done_rows = res.mask_used.kept_blocks(), res.mask_used.keep.shape[0]
    else:
        import oracle

        sl = slice(0, rows * 128)
        probs = oracle.softmax_rows((oracle.block_mean_pool(q[sl], 128) @ oracle.block_mean_pool(k, 64).T)
                                    / math.sqrt(q.shape[1]))
        keep = oracle.hybrid_keep(probs, k_frac, p_frac)
        oracle.attention_backward(q[sl], k, v, keep, 128, 64, do[sl])
        kept, done_rows = int(keep.sum()), rows
    return time.perf_counter() - t0, kept, done_rows


def _threadpool_summary():
    try:
        from threadpoolctl import threadpool_info

        return [{k: p.get(k) for k in ("internal_api", "num_threads", "version")} for p in threadpool_info()]
    except Exception as e:  # pragma: no cover
        return str(e)[:200]


def cpu_reference(steps: int, warmup: int, w=WORKLOAD, as_shipped: bool = True):
    """Time the CPU reference on the host's cores.

    mode (ii), the reported value: a process pool of min(cores, B·H) workers with one BLAS
    thread each; one step = every worker runs one full head's fwd+bwd, so a step processes
    `workers` of the job's B·H heads and value = their dense-equivalent FLOPs / step time
    (nothing extrapolated: ms_per_step is the measured step).
    mode (i), "as shipped": one process with the default BLAS threads runs one head."""
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    kind = "reference" if reference_installed() else "port"
    workers = max(1, min(cores, w["B"] * w["H"]))
    t_m = -(-w["N"] // w["b_q"])
    rows = t_m if kind == "reference" else 8
    ctx = mp.get_context("spawn")
    init = (7, w["N"], w["d"], w["offset_scale"], kind, 1)
    saved_env = {v: os.environ.get(v) for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    os.environ.update({v: "1" for v in saved_env})  # the workers' BLAS starts single-threaded
    times, kept = [], []
    with ctx.Pool(workers, initializer=_cpu_worker_init, initargs=init) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_head, [(w["k_frac"], w["p_frac"], rows)] * workers)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
                kept.append(sum(x[1] for x in res) / workers)
    for var, val in saved_env.items():
        if val is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = val
    t_step = statistics.median(times)
    head_flops = dense_equiv_flops(dict(w, B=1, H=1)) * rows / t_m
    value = workers * head_flops / t_step / 1e12
    out = {
        "value": value, "unit": UNIT, "cores": workers, "kind": kind, "ms_per_step": t_step * 1e3,
        "host_cores": cores, "threadpool_info": _threadpool_summary(),
        "sample": (f"{'sparseattn_lab (unmodified reference, baseline/_ref)' if kind == 'reference' else 'oracle/ port'}"
                   f" sparse_attention + attention_backward, float64 numpy; {workers} worker process(es) x 1 BLAS "
                   f"thread, each step = {workers} head(s) x {rows}/{t_m} query-block rows of the Wan2.1-1.3B shape "
                   f"({statistics.mean(kept) / rows:.1f} kept key blocks per row), median of {steps} step(s); the "
                   f"full {w['B'] * w['H']}-head job is {w['B'] * w['H'] * t_m / (workers * rows):.2f} such steps"),
    }
    if as_shipped:  # mode (i): the reference as a user runs it, one process, default BLAS threads
        _cpu_worker_init(7, w["N"], w["d"], w["offset_scale"], kind, None)
        dt, _, _ = _cpu_head((w["k_frac"], w["p_frac"], rows))
        out["as_shipped"] = {"ms_per_head": dt * 1e3, "value": head_flops / dt / 1e12,
                             "blas_threads": _threadpool_summary(),
                             "mode": "one process, default BLAS threads, one head"}
    return out


# ---------------------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every 2 ms from a background thread (the timed region of a 20-step run is ~30 ms, below
    nvidia-smi's sampling period); nvidia-smi as the fallback when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device_index: int):
        import threading

        self.samples = []  # (t, sm_mhz, max_mhz, reasons bitmask)
        self.stop_flag = False
        self.err = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            uuid = None
            try:
                import torch

                uuid = "GPU-" + str(torch.cuda.get_device_properties(device_index).uuid)
                self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
        except Exception as e:  # pragma: no cover
            self.nvml = None
            self.err = str(e)[:120]
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_flag:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.time(), sm, rs))
            except Exception as e:  # pragma: no cover
                self.err = str(e)[:120]
            time.sleep(0.002)

    def stop(self, t_start: float, t_end: float):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "error": self.err}
        self.stop_flag = True
        self.thread.join(timeout=2)
        win = [s for s in self.samples if t_start <= s[0] <= t_end]
        if not win:  # a very short region: the samples closest to it
            win = sorted(self.samples, key=lambda s: min(abs(s[0] - t_start), abs(s[0] - t_end)))[:3]
        reasons = sorted({n for _, _, rs in win for n, bit in self.bits.items() if rs & bit})
        return {"sm_mhz": statistics.median(s[1] for s in win) if win else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(win), "source": "NVML, 2 ms polling"}


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


def _max_over_ranks(ms: float, world: int, dev) -> float:
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist

    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gpu_arm(args, rank: int, world: int, dev):
    import torch
    import torch.distributed as dist

    import paper_2602_13515_b200 as spa
    from paper_2602_13515_b200 import _lib
    from paper_2602_13515_b200 import attention as at
    from paper_2602_13515_b200.synthetic import video_like_qkv, wan_like_qkv

    w = WORKLOAD
    B, H, N, d = w["B"], w["H"], w["N"], w["d"]
    cfg = spa.SparsityConfig(w["k_frac"], w["p_frac"], w["b_q"], w["b_kv"])
    q, k, v = wan_like_qkv(B, H, N, d, w["offset_scale"], seed=1000 + rank)
    do = torch.randn(q.shape, device=dev, generator=torch.Generator(device=dev).manual_seed(77 + rank)).to(q.dtype)

    def make_step(q, k, v):
        def step():
            qs, ks, vs = (t.detach().requires_grad_(True) for t in (q, k, v))
            res = spa.sparse_attention(qs, ks, vs, cfg)  # the default API: finiteness verdicts included
            res.out.backward(do)
            return res
        return step

    step = make_step(q, k, v)

    def barrier():
        if world > 1:
            dist.barrier()

    res = step()
    keep = res.mask_used.keep
    sparsity = res.mask_used.sparsity()
    for _ in range(max(0, args.warmup - 1)):
        step()
    torch.cuda.synchronize()

    # ---- the timed region: K steps back to back, no instrumentation between launches ----
    launches0 = _lib.STATS.launches
    sampler = ClockSampler(dev.index if dev.index is not None else 0)
    time.sleep(0.05)
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
    spa.check_pending()  # every finiteness verdict of the timed steps (must all be clean)
    ms_step = _max_over_ranks(ev0.elapsed_time(ev1), world, dev) / args.steps

    # ---- per-kernel pass (separate, so the timed loop keeps its PDL overlap): CUDA events on
    # the launching stream around each C call ----
    timed_names = ("spa2_check_finite", "spa2_pooled_scores", "spa2_select_scores", "spa2_build_lists", "spa2_fwd",
                   "spa2_bwd_dq_delta", "spa2_bwd_dkdv")
    _lib.STATS.timing = {n: [] for n in timed_names}
    n_k = max(5, min(args.steps, 30))
    for _ in range(n_k):
        step()
    torch.cuda.synchronize()
    per_kernel_ms = {n: (statistics.median(a.elapsed_time(b) for a, b in lst) if lst else 0.0)
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
                "flops_per_launch": kflops[dom], "ms_per_launch": per_kernel_ms[dom],
                "algorithmic": "Σ_kept c·r_i·c_j·d with c = 4 (fwd), 6 (dQ: S, dP, dQ), 8 (dK/dV: S, dP, dV, dK)"}
    # ---- on-chip roofline of the dK/dV kernel ----
    # Per kept 128x64 tile it issues four SS tcgen05 MMA groups with N = 64 (S, dP, dV^T, dK^T: 8
    # K=16 steps each), whose operand fetch (6 KB per step) runs at ~128 B/clk/SM: ~50 cycles per
    # step instead of the 32 of the tensor datapath, and not slowed by the kernel's TMA / STS / TMEM
    # traffic (tools/smem_contend.py).  Its roofline is therefore the same MMA sequence issued back
    # to back with no dependencies (libspa2_diag spa2_probe_dkdv_mix, one CTA per SM, as many tiles
    # per CTA as the kernel's), timed interleaved with the kernel: frac = probe time / kernel time.
    onchip = None
    try:
        diag = _lib.load_diag()
        st = torch.cuda.current_stream()
        sc = 1.0 / math.sqrt(d)
        bm_ = spa.BlockMask._trusted(keep, w["b_q"], w["b_kv"], N)
        lists_ = at.mask_lists(bm_, B, H, N)
        o_, lse_ = at.fwd(q, k, v, lists_, sc)
        dq_, dk_, dv_ = at.bwd(q, k, v, o_, do, lse_, lists_, sc)
        delta_ = torch.empty((B, H, N), device=dev, dtype=torch.float32)
        _lib.call("spa2_bwd_dq_delta", _lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(o_), _lib.view4(do),
                  _lib.ptr(lse_), _lib.ptr(delta_), _lib.view4(dq_), _lib.DTYPE_CODES[q.dtype], B, H, N, d, w["b_q"],
                  w["b_kv"], _lib.ptr(lists_.row_ptr), _lib.ptr(lists_.row_idx), _lib.ptr(lists_.row_order), sc,
                  st.cuda_stream, stream_obj=st)
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        tiles = int(keep.sum())
        reps = -(-tiles // n_sm)
        cyc = torch.zeros(n_sm, dtype=torch.int64, device=dev)

        def kern():
            _lib.call("spa2_bwd_dkdv", _lib.view4(q), _lib.view4(k), _lib.view4(v), _lib.view4(do), _lib.ptr(lse_),
                      _lib.ptr(delta_), _lib.view4(dk_), _lib.view4(dv_), _lib.DTYPE_CODES[q.dtype], B, H, N, d,
                      w["b_q"], w["b_kv"], _lib.ptr(lists_.col_ptr), _lib.ptr(lists_.col_idx),
                      _lib.ptr(lists_.col_order), sc, st.cuda_stream, stream_obj=st)

        def seq():
            _lib.check_diag(diag.spa2_probe_dkdv_mix(reps, 0, n_sm, _lib.ptr(cyc), st.cuda_stream), "dkdv_mix")

        t_k, t_s = [], []
        for _ in range(5):  # interleaved, medians
            t_k.append(_time(kern, 3, 1))
            t_s.append(_time(seq, 3, 1))
        t_k, t_s = sorted(t_k)[2], sorted(t_s)[2]
        onchip = {"kernel": "spa2_bwd_dkdv", "bound": "tensor (SS N=64 operand fetch)",
                  "ms_per_launch": t_k, "floor_ms": t_s, "frac": t_s / t_k, "tiles": tiles,
                  "floor": "the kernel's own MMA sequence (S, dP K-major; dV^T, dK^T MN-major; 4 x 8 steps per kept "
                           "tile, warp-batched issue as in the kernel) issued back to back on every SM, "
                           f"{reps} tiles per SM, no data dependencies (profiles/traces_r02.md, "
                           "profiles/clock_energy_r02.md)"}
    except Exception as exc:  # diagnostics only: never fail the bench over it
        onchip = {"unavailable": repr(exc)[:200]}

    # masker: HBM-bound passes.  K1a = block-mean pooling (reads Q and K once; the reference's
    # block_mean_pool), K1 = K1a + the small fp64 pooled-score GEMM (what sparse_attention runs);
    # K0 = the finiteness scan of V (reads V once).  Each timed over 30 back-to-back launches
    # between two CUDA events, so launch overhead does not count.
    from paper_2602_13515_b200 import masker as mk_

    qk_bytes = 2 * q.numel() * q.element_size()
    hbm = peaks["hbm_gbs"]
    flag = torch.zeros((1,), dtype=torch.int32, pin_memory=True)
    t_m_, t_n_ = -(-N // w["b_q"]), -(-N // w["b_kv"])
    pool_ws = torch.empty(B * H * (t_m_ + t_n_) * d, device=dev, dtype=torch.float64)
    st_ = torch.cuda.current_stream()

    def k1a():
        _lib.call("spa2_block_mean_pool", _lib.view4(q), _lib.view4(k), _lib.DTYPE_CODES[q.dtype], B, H, N, d,
                  w["b_q"], w["b_kv"], _lib.ptr(pool_ws), _lib.ptr(pool_ws[B * H * t_m_ * d:]), None,
                  st_.cuda_stream, stream_obj=st_)

    k0_ms = _time(lambda: at._scan_finite(flag, v), 30, 3)
    k1a_ms = _time(k1a, 30, 3)
    k1_ms = _time(lambda: mk_._pooled_probs(q, k, w["b_q"], w["b_kv"], None, softmax=False), 30, 3)
    masker = {"bound": "hbm", "unit": "GB/s", "peak": hbm,
              "K0_finite_scan_v": {"bytes": qk_bytes // 2, "ms": k0_ms, "achieved": (qk_bytes // 2) / (k0_ms * 1e-3) / 1e9},
              "K1a_block_mean_pool": {"bytes": qk_bytes, "ms": k1a_ms, "achieved": qk_bytes / (k1a_ms * 1e-3) / 1e9},
              "K1_pool_scores": {"bytes": qk_bytes, "ms": k1_ms, "achieved": qk_bytes / (k1_ms * 1e-3) / 1e9}}
    for kk in ("K1a_block_mean_pool", "K1_pool_scores", "K0_finite_scan_v"):
        masker[kk]["frac"] = masker[kk]["achieved"] / hbm
    masker["note"] = ("K1a = the pooling pass alone (the HBM-bound part); K1 adds the fp64 pooled-score GEMM "
                      "(tensor-core DMMA, ~20 us) that sparse_attention runs after it (profiles/ncu_r02c.md)")

    out = {"ms_step": ms_step, "sparsity": sparsity, "clocks": clocks, "launches": launches,
           "per_kernel_ms": per_kernel_ms, "roofline": roofline, "masker_roofline": masker, "kflops": kflops,
           "onchip_roofline": onchip}

    # ---- e2e through the public API with host buffers ----
    if not args.no_e2e:
        from paper_2602_13515_b200.host import HostPipeline

        hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, do))
        outs = [torch.empty(q.shape, dtype=q.dtype).pin_memory() for _ in range(4)]
        pipe = HostPipeline(dev, groups=args.e2e_groups)

        def e2e_step():
            pipe.fwd_bwd(hq, hk, hv, hdo, cfg, *outs)

        # untimed warm-up: the host pipeline's pinned / device buffers and caches, and the PCIe
        # link, which the GPU runs at a lower speed when idle and only ramps up under sustained
        # traffic (the first few hundred ms of host-buffer steps measured up to 2x slower on a
        # fresh box, tools/e2e_sweep.py)
        t_warm = time.perf_counter()
        while True:
            for _ in range(5):
                e2e_step()
            torch.cuda.synchronize()
            if time.perf_counter() - t_warm > 1.0:
                break
        # three back-to-back windows, the median reported (all listed): a rare host-side stall of
        # a few hundred ms (seen on the pool's boxes with the PCIe floor unchanged) would
        # otherwise dominate a single window (tools/e2e_sweep.py)
        n_e2e = max(10, min(args.steps, 60) // 3)
        windows = []
        for _ in range(3):
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(n_e2e):
                e2e_step()
            b.record()
            torch.cuda.synchronize()
            windows.append(_max_over_ranks(a.elapsed_time(b), world, dev) / n_e2e)
        spa.check_pending()
        e_step = statistics.median(windows)
        nbytes = q.numel() * q.element_size()
        # the PCIe floor of the same traffic: 4 tensors in and 4 out per step, both directions at
        # once (pinned buffers, two streams), nothing else running
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        dev_bufs = [torch.empty_like(q) for _ in range(4)]

        def duplex():
            s_in.wait_stream(torch.cuda.current_stream())
            s_out.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_in):
                for dst, src in zip(dev_bufs, (hq, hk, hv, hdo)):
                    dst.copy_(src, non_blocking=True)
            with torch.cuda.stream(s_out):
                for dst, src in zip(outs, (q, k, v, do)):
                    dst.copy_(src, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)

        pcie_ms = _time(duplex, 5, 1)
        del dev_bufs
        out["e2e"] = {"value": world * dense_equiv_flops() / (e_step * 1e-3) / 1e12, "unit": UNIT,
                      "h2d_bytes_per_step": 4 * nbytes, "d2h_bytes_per_step": 4 * nbytes, "ms_per_step": e_step,
                      "pcie_duplex_copy_ms": pcie_ms, "frac_of_pcie_floor": pcie_ms / e_step,
                      "steps": 3 * n_e2e, "windows_ms_per_step": windows,
                      "timing": f"median of 3 windows of {n_e2e} steps",
                      "api": f"paper_2602_13515_b200.host.HostPipeline.fwd_bwd "
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

    # ---- secondary workload: spatio-temporally correlated (video-like) masks, same shape ----
    if rank == 0 and world == 1 and not args.no_secondary:
        q2, k2, v2 = video_like_qkv(B, H, N, d, 2.5, seed=2000)
        step2 = make_step(q2, k2, v2)
        r2 = step2()
        keep2 = r2.mask_used.keep
        ms2 = _time(step2, max(5, min(args.steps, 30)), 2)
        spa.check_pending()
        adj = float((keep2[..., :-1] & keep2[..., 1:]).sum() / keep2[..., :-1].sum())
        out["secondary"] = {"workload": "video-like correlated masks (synthetic.video_like_qkv, s=2.5), same shape",
                            "block_sparsity": r2.mask_used.sparsity(), "ms_per_step": ms2,
                            "value": dense_equiv_flops() / (ms2 * 1e-3) / 1e12,
                            "p_next_key_block_kept": adj,
                            "p_next_key_block_kept_primary": float((keep[..., :-1] & keep[..., 1:]).sum()
                                                                   / keep[..., :-1].sum())}
        del q2, k2, v2
    return out


def cfg4_leg(args, rank: int, world: int, dev):
    """configs[3] on `world` GPUs: ONE Wan2.1-14B 720p attention problem (H = 40, N = 75600)
    (a) head-sharded: rank r runs heads head_range(40, r, world) of replicated q/k/v, then the
        NCCL all-gather of O (forward) and of dQ, dK, dV (backward) assembles the full result;
    (b) Ulysses: q/k/v/dO sequence-sharded [B, N/P, H, d] per rank, exchanged to head-sharded
        by all-to-all (NCCL), per-head-group compute overlapped with the exchange of the next
        group (dist.UlyssesAttention), outputs and gradients exchanged back.
    Device time, max over ranks; comm time from CUDA events around the collectives."""
    import torch

    import paper_2602_13515_b200 as spa
    from paper_2602_13515_b200 import dist as sdist
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    c = CFG4
    B, H, N, d = c["B"], c["H"], c["N"], c["d"]
    cfg = spa.SparsityConfig(c["k_frac"], c["p_frac"], 128, 64)
    h0, h1 = sdist.head_range(H, rank, world)
    # every rank generates the full replicated problem from the same seed, keeps its heads
    q, k, v = wan_like_qkv(B, H, N, d, c["offset_scale"], seed=4000)
    do = torch.randn(q.shape, device=dev, generator=torch.Generator(device=dev).manual_seed(4001)).to(q.dtype)
    out = {"workload": "Wan2.1-14B 720p attention (BASELINE configs[3]): B=1 H=40 N=75600 d=128, one problem over "
                       f"{world} GPU(s)", "heads_per_rank": h1 - h0}
    comm_ev = []

    def head_sharded_step():
        ql, kl, vl = (t[:, h0:h1].detach().requires_grad_(True) for t in (q, k, v))
        res = spa.sparse_attention(ql, kl, vl, cfg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sdist.gather_heads(res.out.detach(), H)
        e1.record()
        res.out.backward(do[:, h0:h1])
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for g in (ql.grad, kl.grad, vl.grad):
            sdist.gather_heads(g, H)
        e3.record()
        comm_ev.append((e0, e1, e2, e3))

    reps = max(3, min(args.steps, 10))
    ms = _max_over_ranks(_time(head_sharded_step, reps, 2), world, dev)
    comm = sum(a.elapsed_time(b) + c_.elapsed_time(d_) for a, b, c_, d_ in comm_ev[-reps:]) / reps
    out["head_sharded"] = {"ms_per_step": ms, "value": dense_equiv_flops(c) / (ms * 1e-3) / 1e12,
                           "allgather_ms_per_step": _max_over_ranks(comm, world, dev)}
    spa.check_pending()
    if H % world == 0 and N % world == 0:
        n_loc = N // world
        n0 = rank * n_loc
        # sequence-sharded activations [B, N/P, H, d], as a DiT holds them
        ql, kl, vl, dol = (t.permute(0, 2, 1, 3)[:, n0:n0 + n_loc].contiguous() for t in (q, k, v, do))
        uly = sdist.UlyssesAttention(cfg, groups=args.ulysses_groups)

        def ulysses_step():
            qs, ks, vs = (t.detach().requires_grad_(True) for t in (ql, kl, vl))
            o = uly(qs, ks, vs)
            o.backward(dol)

        ms_u = _max_over_ranks(_time(ulysses_step, reps, 2), world, dev)
        out["ulysses"] = {"ms_per_step": ms_u, "value": dense_equiv_flops(c) / (ms_u * 1e-3) / 1e12,
                          "groups": args.ulysses_groups,
                          "alltoall_ms_per_step": _max_over_ranks(uly.comm_ms(reps), world, dev),
                          "note": "all-to-all on its own stream, overlapped with the other head groups' compute"}
        spa.check_pending()
    return out


def config_dict(world: int, sparsity=None):
    w = WORKLOAD
    c = {"workload": "Wan2.1-1.3B 480p attention (BASELINE configs[1]): B=1 H=12 N=32760 d=128 per GPU",
         "B": w["B"], "H": w["H"], "N": w["N"], "d": w["d"], "b_q": w["b_q"], "b_kv": w["b_kv"],
         "k_frac": w["k_frac"], "p_frac": w["p_frac"], "mask": "hybrid top-k ∪ top-p, rebuilt every step",
         "parallelism": (f"batch-sharded x{world}: each rank its own 12-head problem, no collective"
                         if world > 1 else "single GPU"),
         "api": "sparse_attention(q, k, v, cfg) with default arguments + autograd backward",
         "l2": "inputs larger than L2 (q+k+v+dO = 403 MB per GPU), no flush"}
    if sparsity is not None:
        c["block_sparsity"] = round(sparsity, 5)
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cfg4", action="store_true")
    ap.add_argument("--e2e-groups", type=int, default=6)
    ap.add_argument("--ulysses-groups", type=int, default=5)
    ap.add_argument("--lib", default=None, help="A/B: load this libspa2.so build instead of the in-tree one")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        cpu = cpu_reference(args.steps, args.warmup, as_shipped=False)
        line = {"metric": METRIC, "value": cpu["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": cpu["ms_per_step"], "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (Wan2.1-shaped, seeded)",
                "config": config_dict(1), "impl": "reference",
                "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "host_cores",
                                                     "threadpool_info")},
                "e2e": {"value": cpu["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    if args.lib:
        from paper_2602_13515_b200 import _lib

        _lib.use_library(args.lib)
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))  # ranks > GPUs: gloo test mode
    torch.cuda.set_device(dev)
    if world > 1:
        # NCCL, one GPU per rank; SPA2_BENCH_BACKEND=gloo lets several ranks share one GPU to
        # exercise the multi-rank code path (tests/test_gpu_bench_multirank.py; timings meaningless)
        backend = os.environ.get("SPA2_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init log (one "Init COMPLETE ... nranks N" line per rank) lets the driver count
            # the ranks; limited to the INIT subsystem, and our JSON line is printed after teardown
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    line = None
    try:
        r = gpu_arm(args, rank, world, dev)
        c4 = None
        if world > 1 and not args.no_cfg4:
            c4 = cfg4_leg(args, rank, world, dev)
        cpu = None
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            cpu = cpu_reference(1, 0)
        if rank == 0:
            value = world * dense_equiv_flops() / (r["ms_step"] * 1e-3) / 1e12
            line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                    "warmup": args.warmup, "ms_per_step": r["ms_step"], "higher_is_better": True, "scaling": "weak",
                    "vs_baseline": None, "dtype": "bf16",
                    "data": "synthetic (Wan2.1-shaped q/k/v: N(0,1) + per-block N(0,0.81) offsets, seeded)",
                    "config": config_dict(world, r["sparsity"]), "roofline": r["roofline"],
                    "masker_roofline": r["masker_roofline"], "onchip_roofline": r["onchip_roofline"],
                    "gpu_launches": r["launches"], "clocks": r["clocks"],
                    "per_kernel_ms": {k.replace("spa2_", ""): round(v, 5) for k, v in r["per_kernel_ms"].items()}}
            for key in ("e2e", "dense_baselines", "secondary"):
                if key in r:
                    line[key] = r[key]
            if c4 is not None:
                line["cfg4"] = c4
            if cpu is not None:
                line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample", "host_cores",
                                                            "threadpool_info", "as_shipped", "ms_per_step")}
    finally:
        if world > 1:
            dist.destroy_process_group()
    if line is not None:  # rank 0, last line of the output
        sys.stderr.flush()
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

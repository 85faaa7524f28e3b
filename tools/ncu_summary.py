"""Summarise an ncu report (and launch list) into profiles/ for the round record.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches_r01.csv r01

Writes profiles/ncu_<tag>.md (human table), profiles/ncu_summary_<tag>.json and updates
profiles/ncu_summary.json (read by bench.py for the roofline ``traffic`` field).
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYMAP = {"k_fwd": "spa2_fwd", "k_dq3": "spa2_bwd_dq_delta", "k_dkdv5": "spa2_bwd_dkdv", "k_delta": "spa2_bwd_delta",
          "k_nonfinite_bf16": "spa2_check_finite", "k_pool_bf16_pipe": "spa2_pooled_scores:pool",
          "k_pool": "spa2_pooled_map:pool", "k_scores": "spa2_pooled_scores:scores",
          "k_softmax_rows": "spa2_pooled_map:softmax", "k_select": "spa2_select_scores"}
PER_STEP = 10  # hot-path kernels of one bench step
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "smsp__inst_executed.sum": "inst",
}
UNIT_SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    base = base.split("::")[-1]
    return base.split("<")[0].strip()


def read_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, key in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                val = float(r[i].replace(",", ""))
            except ValueError:
                continue
            scale = UNIT_SCALE.get(units[i], 1.0)
            if key == "duration":
                rec["duration_ms"] = val * scale * 1e3
            elif key in ("dram_read", "dram_write"):
                rec[key + "_bytes"] = val * scale
            else:
                rec[key] = val
        out.append(rec)
    return out


def read_launches(path):
    if not path or not os.path.exists(path):
        return []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = []
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        out.append((short(r[ki]), float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1e-9) * 1e3))
    return out


def main():
    rep, launches, tag = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "rXX"
    recs = read_report(rep)
    ll = read_launches(launches)
    ours = [x for x in ll if x[0].startswith("k_")]
    # the last complete step: the last window of PER_STEP launches holding each hot-path kernel
    # once (bench.py launches extra masker / dK/dV passes after its steps for the rooflines)
    step_set = {"k_nonfinite_bf16", "k_pool_bf16_pipe", "k_scores_dmma", "k_select", "k_counts", "k_scan_orders",
                "k_fill", "k_fwd", "k_dq3", "k_dkdv5"}
    step = ours[-PER_STEP:] if len(ours) >= PER_STEP else ours
    for i in range(len(ours) - PER_STEP, -1, -1):
        win = ours[i:i + PER_STEP]
        if {n for n, _ in win} == step_set:
            step = win
            break
    tot = sum(t for _, t in step) or 1.0
    kern = {}
    lines = [f"# ncu summary {tag}", "", "Workload: bench.py (Wan2.1-1.3B shape, B=1 H=12 N=32760 d=128, ~95% block "
             "sparsity), one step after 3 warm-up steps; `ncu --set full --clock-control none`.", "",
             "| kernel | ncu ms (cold, serialised) | share of step (launch list) | DRAM read MB | DRAM write MB | "
             "tensor active % | DRAM % peak | SM % | regs |", "|---|---|---|---|---|---|---|---|---|"]
    share = {}
    for name, t in step:
        share[name] = share.get(name, 0.0) + t / tot
    for r in recs:
        k = r["kernel"]
        lines.append(f"| {k} | {r.get('duration_ms', 0):.4f} | {100 * share.get(k, 0):.1f}% | "
                     f"{r.get('dram_read_bytes', 0) / 1e6:.1f} | {r.get('dram_write_bytes', 0) / 1e6:.1f} | "
                     f"{r.get('tensor_active_pct', 0):.1f} | {r.get('dram_pct', 0):.1f} | {r.get('sm_pct', 0):.1f} | "
                     f"{r.get('regs', 0):.0f} |")
        key = KEYMAP.get(k, k)
        kern[key] = {"kernel": k, "duration_ms": r.get("duration_ms"),
                     "dram_bytes_per_launch": r.get("dram_read_bytes", 0) + r.get("dram_write_bytes", 0),
                     "tensor_active_pct": r.get("tensor_active_pct"), "dram_pct": r.get("dram_pct"),
                     "share_of_step": share.get(k)}
    if step:
        lines += ["", "Launch list of the same step (gpu__time_duration.sum, ms):", ""]
        lines += [f"- {n}: {t:.4f}" for n, t in step]
    summary = {"tag": tag, "report": os.path.basename(rep), "kernels": kern}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    for name in (f"ncu_summary_{tag}.json", "ncu_summary.json"):
        with open(os.path.join(ROOT, "profiles", name), "w") as f:
            json.dump(summary, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()

#!/usr/bin/env bash
# Profiling recipe (run on the GPU box via gpurun; never under a multi-rank launch).
#   1. launch list of one bench step with per-launch device time (cold-cache, serialised)
#   2. one `ncu --set full` capture of each hot-path kernel of the last bench step
# Outputs land in gpurun_out/; summaries are copied to profiles/ by tools/ncu_summary.py.
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p "$OUT"
BENCH="python bench.py --steps 1 --warmup 3 --no-e2e --no-dense --no-cpu-baseline --no-secondary"
KERNELS='k_nonfinite_bf16|k_dkdv|k_dq3|k_fwd|k_pool_bf16_pipe|k_scores|k_select|k_counts|k_scan_orders|k_fill'
PER_STEP=10  # kernels of one step matching $KERNELS; the bench runs 1 + (warmup-1) + steps = 4 steps

ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_${TAG}.csv" $BENCH > "$OUT/launches_${TAG}.log" 2>&1

ncu --set full --clock-control none --import-source on -k regex:"$KERNELS" \
    -s $((3 * PER_STEP)) -c $PER_STEP -o "$OUT/prof_${TAG}" -f $BENCH > "$OUT/prof_${TAG}.log" 2>&1
echo "profile done"

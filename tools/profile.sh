#!/usr/bin/env bash
# Profiling recipe (run on the GPU box via gpurun; never under a multi-rank launch).
#   1. launch list of one bench step with per-launch device time (cold-cache, serialised)
#   2. one `ncu --set full` capture of each hot-path kernel (after warm-up launches)
# Outputs land in gpurun_out/; summaries are copied to profiles/ by tools/ncu_summary.py.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p "$OUT"
BENCH="python bench.py --steps 1 --warmup 3 --no-e2e --no-dense --no-cpu-baseline"

ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/launches_${TAG}.csv" $BENCH > "$OUT/launches_${TAG}.log" 2>&1

# warm-up: 3 bench steps + the measured step; capture the kernels of the last one
ncu --set full --clock-control none --import-source on \
    -k regex:'k_dkdv|k_dq|k_fwd|k_pool|k_select|k_scores|k_softmax_rows|k_delta|k_fill|k_scan|k_row_counts|k_col_counts' \
    -s 39 -c 13 -o "$OUT/prof_${TAG}" -f $BENCH > "$OUT/prof_${TAG}.log" 2>&1
echo "profile done"

#!/usr/bin/env bash
# ncu --set full of the attention kernels only (after warm-up), for stall / memory analysis.
TAG=${1:-r01x}
REGEX=${2:-'k_dkdv|k_dq|k_fwd'}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s 9 -c 3 \
    -o "gpurun_out/prof_${TAG}" -f python bench.py --steps 1 --warmup 3 --no-e2e --no-dense --no-cpu-baseline \
    > "gpurun_out/prof_${TAG}.log" 2>&1
echo done

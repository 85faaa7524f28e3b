#!/usr/bin/env bash
# Like tools/ab.sh but 400 timed steps (the power-capped regime of the benchmark of record).
mkdir -p gpurun_out
i=0
for a in "$@"; do
  i=$((i + 1))
  env $a timeout 300 python bench.py --steps 400 --warmup 5 --no-e2e --no-dense --no-cpu-baseline \
    > gpurun_out/ab4_$i.out 2> gpurun_out/ab4_$i.err
  tail -1 gpurun_out/ab4_$i.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['per_kernel_ms']; print('$a'.ljust(44), round(d['ms_per_step'],4), 'fwd', k['fwd'], 'dq', k['bwd_dq_delta'], 'dkdv', k['bwd_dkdv'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null \
    || { echo "$a: FAILED"; tail -3 gpurun_out/ab4_$i.err; }
done

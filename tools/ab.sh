#!/usr/bin/env bash
# A/B kernel timings on the GPU box: each argument is a space-separated env assignment list
# (e.g. "SPA2_LIB_PATH=alt/nk4/libspa2.so SPA2_DEBUG_FLAGS=1"); prints ms/step + per-kernel ms.
mkdir -p gpurun_out
i=0
for a in "$@"; do
  i=$((i + 1))
  env $a timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-dense --no-cpu-baseline \
    > gpurun_out/ab_$i.out 2> gpurun_out/ab_$i.err
  rc=$?
  tail -1 gpurun_out/ab_$i.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['per_kernel_ms']; print('$a'.ljust(50), round(d['ms_per_step'],4), 'fwd', k['fwd'], 'dq', k['bwd_dq_delta'], 'dkdv', k['bwd_dkdv'], 'clk', d['clocks']['sm_mhz'])" 2>/dev/null \
    || { echo "$a: FAILED rc=$rc"; tail -5 gpurun_out/ab_$i.err; }
done

#!/usr/bin/env bash
# A/B kernel timings on the GPU box: each argument is a space-separated env assignment list
# (e.g. "SPA2_LIB_PATH=alt/nk4/libspa2.so SPA2_DEBUG_FLAGS=1"); prints ms/step + per-kernel ms.
for a in "$@"; do
  env $a timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-dense --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['per_kernel_ms']; print('$a'.ljust(50), round(d['ms_per_step'],4), 'fwd', k['fwd'], 'dq', k['bwd_dq_delta'], 'dkdv', k['bwd_dkdv'], 'clk', d['clocks']['sm_mhz'])"
done

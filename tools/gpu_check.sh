#!/usr/bin/env bash
# Quick GPU iteration loop (run via gpurun): parity tests, then kernel-only bench lines.
# Extra args: env assignments to A/B, e.g. `bash tools/gpu_check.sh SPA2_DKDV_EW=16`.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
bench() {
  env "$@" timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-dense --no-cpu-baseline 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', 'ms/step', round(d['ms_per_step'],4), d['per_kernel_ms'], 'clk', d['clocks']['sm_mhz'])"
}
bench SPA2_NONE=0
for a in "$@"; do bench $a; done

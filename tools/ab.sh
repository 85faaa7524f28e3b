#!/usr/bin/env bash
# A/B kernel timings on the GPU box.  Each argument is one configuration: a space-separated
# list of NAME=value environment assignments and bench.py flags, e.g.
#   bash tools/ab.sh "" "--lib alt/nk4/libspa2.so" "SPA2_PDL=0"
# prints ms/step + per-kernel ms for each.
mkdir -p gpurun_out
i=0
for a in "$@"; do
  i=$((i + 1))
  envs=(); flags=()
  for w in $a; do
    if [[ $w == *=* && $w != --* ]]; then envs+=("$w"); else flags+=("$w"); fi
  done
  env "${envs[@]}" timeout 300 python bench.py --steps ${STEPS:-30} --warmup 5 --no-e2e --no-dense --no-cpu-baseline --no-secondary \
    "${flags[@]}" > gpurun_out/ab_$i.out 2> gpurun_out/ab_$i.err
  rc=$?
  tail -1 gpurun_out/ab_$i.out | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['per_kernel_ms']; print('$a'.ljust(50), round(d['ms_per_step'],4), 'fwd', k['fwd'], 'dq', k['bwd_dq_delta'], 'dkdv', k['bwd_dkdv'], 'clk', d['clocks']['sm_mhz'])" 2>/dev/null \
    || { echo "$a: FAILED rc=$rc"; tail -5 gpurun_out/ab_$i.err; }
done

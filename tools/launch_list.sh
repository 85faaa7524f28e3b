#!/usr/bin/env bash
# Per-kernel device time of one bench step (cold-cache, serialised) — developer view.
#   bash tools/launch_list.sh [regex]
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none ${1:+-k regex:"$1"} --csv --log-file gpurun_out/ll.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-dense --no-cpu-baseline --no-secondary ${LIB:+--lib $LIB} > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/ll.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; ik = h.index("Kernel Name"); iv = h.index("Metric Value")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    n = r[ik].split("(")[0].split("<")[0].split("::")[-1]
    d.setdefault(n, []).append(float(r[iv].replace(",", "")))
import statistics
for n, v in d.items():
    print(f"{n:24s} n={len(v):3d} last={v[-1] / 1e3:8.1f} us  median={statistics.median(v) / 1e3:8.1f} us  min={min(v) / 1e3:8.1f} us")
PY

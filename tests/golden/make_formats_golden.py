"""Golden files for the reference's on-disk formats, written by the REAL reference writers.

    python tests/golden/make_formats_golden.py

Imports ``sparseattn_lab`` from ``/root/reference/pkg/src`` (read-only, build container
only) and writes ``tests/golden/formats/``: a pooled-map CSV and the hybrid mask CSV of a
seeded ragged map (masker.write_pooled_map_csv / write_mask_csv, masker.py:159-186), and an
``attn-bench``-style table + timings written with cli.write_table / write_json
(cli.py:80-107).  tests/test_formats.py checks this package's writers byte for byte."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "formats")
sys.path.insert(0, "/root/reference/pkg/src")

from sparseattn_lab import cli as ref_cli  # noqa: E402
from sparseattn_lab import masker as ref_mk  # noqa: E402
from sparseattn_lab.numerics import softmax_rows  # noqa: E402


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.Generator(np.random.PCG64(2602))
    probs = softmax_rows(rng.normal(size=(6, 11)) * 2.0)
    pm = ref_mk.PooledMap(probs, 128, 64, 650)  # 650 tokens: T_m = 6 (ragged 10-row tail), T_n = 11
    ref_mk.write_pooled_map_csv(os.path.join(OUT, "pooled_map.csv"), pm)
    bm = ref_mk.hybrid_mask(pm, ref_mk.SparsityConfig(0.2, 0.5, 128, 64))
    ref_mk.write_mask_csv(os.path.join(OUT, "mask_hybrid.csv"), bm)
    rows = [[32760, 128, 128, 64, 0.9501953125, 78900, 1572864, 0.0498046875, 0.0029296875],
            [1024, 64, 128, 64, 0.0625, 120, 128, 0.9375, 1.0 / 3.0]]
    ref_cli.write_table(OUT, "bench", ref_cli.BENCH_HEADER if hasattr(ref_cli, "BENCH_HEADER") else
                        ["n", "d", "b_q", "b_kv", "sparsity", "computed_blocks", "total_blocks", "block_ratio",
                         "max_dev_from_dense"], rows, "csv")
    ref_cli.write_table(OUT, "bench_json", ["n", "sparsity"], [[1024, 0.1], [2048, 2.0 / 3.0]], "json")
    ref_cli.write_json(OUT, "timings", {"reps": 3, "entries": [{"n": 1024, "sparsity": 0.5, "dense_s": 0.25,
                                                                "sparse_s": 0.125, "speedup": 2.0}]})
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

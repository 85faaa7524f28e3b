"""On-disk formats (formats.py) are byte-identical to the reference's writers: golden files
in tests/golden/formats/ were written by the real reference (make_formats_golden.py)."""

import filecmp
import os

import numpy as np

from paper_2602_13515_b200 import formats as fm

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")


def _read_probs(path):
    with open(path) as f:
        f.readline()
        f.readline()
        return np.array([[float(x) for x in line.strip().split(",")] for line in f if line.strip()])


def test_mask_csv_round_trip_and_bytes(tmp_path):
    keep, b_q, b_kv, n = fm.read_mask_csv(os.path.join(GOLD, "mask_hybrid.csv"))
    assert (b_q, b_kv, n) == (128, 64, 650) and keep.shape == (6, 11) and keep.any(axis=1).all()
    out = tmp_path / "mask.csv"
    fm.write_mask_csv(out, keep=keep, b_q=b_q, b_kv=b_kv, n_tokens=n)
    assert filecmp.cmp(out, os.path.join(GOLD, "mask_hybrid.csv"), shallow=False)


def test_pooled_map_csv_bytes(tmp_path):
    probs = _read_probs(os.path.join(GOLD, "pooled_map.csv"))
    out = tmp_path / "pm.csv"
    fm.write_pooled_map_csv(out, probs=probs, b_q=128, b_kv=64, n_tokens=650)
    assert filecmp.cmp(out, os.path.join(GOLD, "pooled_map.csv"), shallow=False)


def test_report_tables_bytes(tmp_path):
    rows = [[32760, 128, 128, 64, 0.9501953125, 78900, 1572864, 0.0498046875, 0.0029296875],
            [1024, 64, 128, 64, 0.0625, 120, 128, 0.9375, 1.0 / 3.0]]
    fm.write_table(str(tmp_path), "bench", fm.BENCH_HEADER, rows, "csv")
    fm.write_table(str(tmp_path), "bench_json", ["n", "sparsity"], [[1024, 0.1], [2048, 2.0 / 3.0]], "json")
    fm.write_json(str(tmp_path), "timings", {"reps": 3, "entries": [{"n": 1024, "sparsity": 0.5, "dense_s": 0.25,
                                                                     "sparse_s": 0.125, "speedup": 2.0}]})
    for name in ("bench.csv", "bench_json.json", "timings.json"):
        assert filecmp.cmp(tmp_path / name, os.path.join(GOLD, name), shallow=False), name

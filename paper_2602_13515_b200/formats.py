"""File formats of the reference's tooling, so GPU runs feed the same readers.

* Block masks / pooled maps as CSV: a ``b_q=..,b_kv=..,n_tokens=..`` line, a ``c0,c1,...``
  header, then one row per query block (masker.py:159-186: write_mask_csv, read_mask_csv,
  write_pooled_map_csv).  Floats use the shortest round-trip ``repr`` (numerics.py:122-124).
* Report tables (``name.csv`` or ``name.json``) and JSON payloads exactly as
  cli.write_table / cli.write_json (cli.py:80-107), used by ``tools/attn_bench.py`` for the
  ``attn-bench`` outputs ``bench.csv`` and ``timings.json`` (cli.py:200-241).

Masks and maps may be given as this package's ``BlockMask`` / ``PooledMap`` (device tensors)
or as host arrays with explicit geometry.
"""

from __future__ import annotations

import json
import os

import numpy as np


def format_float(v: float) -> str:
    """Shortest round-trip decimal form (numerics.py:122-124)."""
    return repr(float(v))


def _geometry(obj, b_q=None, b_kv=None, n_tokens=None):
    if b_q is None:
        b_q, b_kv, n_tokens = obj.b_q, obj.b_kv, obj.n_tokens
    return int(b_q), int(b_kv), int(n_tokens)


def _host_2d(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    x = np.asarray(x)
    if x.ndim != 2:
        raise ValueError(f"expected a single [T_m, T_n] map, got shape {x.shape}")
    return x


def write_mask_csv(path, bm=None, *, keep=None, b_q=None, b_kv=None, n_tokens=None) -> None:
    """masker.write_mask_csv (masker.py:159-164): header line, column names, 0/1 rows."""
    keep = _host_2d(bm.keep if keep is None else keep).astype(bool)
    b_q, b_kv, n_tokens = _geometry(bm, b_q, b_kv, n_tokens)
    with open(path, "w", newline="") as f:
        f.write(f"b_q={b_q},b_kv={b_kv},n_tokens={n_tokens}\n")
        f.write(",".join(f"c{j}" for j in range(keep.shape[1])) + "\n")
        for row in keep:
            f.write(",".join("1" if v else "0" for v in row) + "\n")


def read_mask_csv(path):
    """masker.read_mask_csv (masker.py:167-178) -> (keep bool ndarray, b_q, b_kv, n_tokens).
    Wrap with ``BlockMask(torch.as_tensor(keep), b_q, b_kv, n_tokens)`` for the GPU path."""
    with open(path, "r", newline="") as f:
        meta = dict(kv.split("=") for kv in f.readline().strip().split(","))
        f.readline()  # column header carries no information beyond width
        rows = [[c == "1" for c in line.strip().split(",")] for line in f if line.strip()]
    return np.array(rows, dtype=bool), int(meta["b_q"]), int(meta["b_kv"]), int(meta["n_tokens"])


def write_pooled_map_csv(path, pm=None, *, probs=None, b_q=None, b_kv=None, n_tokens=None) -> None:
    """masker.write_pooled_map_csv (masker.py:181-186)."""
    probs = _host_2d(pm.probs if probs is None else probs).astype(np.float64)
    b_q, b_kv, n_tokens = _geometry(pm, b_q, b_kv, n_tokens)
    with open(path, "w", newline="") as f:
        f.write(f"b_q={b_q},b_kv={b_kv},n_tokens={n_tokens}\n")
        f.write(",".join(f"c{j}" for j in range(probs.shape[1])) + "\n")
        for row in probs:
            f.write(",".join(format_float(v) for v in row) + "\n")


def _cell(v) -> str:
    if isinstance(v, float):
        return format_float(v)
    return str(v)


def write_table(out_dir: str, name: str, header: list[str], rows: list[list], fmt: str) -> str:
    """cli.write_table (cli.py:86-99): name.csv (repr floats) or name.json (list of dicts)."""
    if fmt == "csv":
        path = os.path.join(out_dir, f"{name}.csv")
        with open(path, "w", newline="") as f:
            f.write(",".join(header) + "\n")
            for row in rows:
                f.write(",".join(_cell(v) for v in row) + "\n")
    else:
        path = os.path.join(out_dir, f"{name}.json")
        with open(path, "w") as f:
            json.dump([dict(zip(header, row)) for row in rows], f, indent=2, sort_keys=True)
            f.write("\n")
    return path


def write_json(out_dir: str, name: str, payload: dict) -> str:
    """cli.write_json (cli.py:102-107)."""
    path = os.path.join(out_dir, f"{name}.json")
    with open(path, "w") as f:
        json.dump(payload, f, indent=2, sort_keys=True)
        f.write("\n")
    return path


BENCH_HEADER = ["n", "d", "b_q", "b_kv", "sparsity", "computed_blocks", "total_blocks", "block_ratio",
                "max_dev_from_dense"]  # cli.py:233-236

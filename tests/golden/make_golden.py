"""Generate golden vectors by running the REAL reference package.

Run once in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_golden.py

It imports ``sparseattn_lab`` from ``/root/reference/pkg/src`` (read-only) and writes
``tests/golden/{masks,pooled,attention}.npz`` plus ``manifest.json``.  Nothing at
test/bench time reads ``/root/reference``; the fixtures travel with the repo.

Contents
--------
masks.npz      pooled maps (float64) -> the reference's top_k_mask / top_p_mask /
               hybrid_mask keep matrices (bit patterns), including the reference
               test suite's hand-written rows, c06/c07-style random rows, exact
               ties/zeros, and large Wan-like maps.
pooled.npz     q/k -> the reference's pooled_map probabilities (ragged block sizes).
attention.npz  bf16-representable q/k/v/d_out (regenerated from seeds by gen.py,
               digests stored) + masks -> the reference's out / lse / dq / dk / dv.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from gen import digest, random_keep, wan_like  # noqa: E402
from sparseattn_lab import attention as ref_at  # noqa: E402
from sparseattn_lab import masker as ref_mk  # noqa: E402


def _pm(probs):
    probs = np.atleast_2d(np.asarray(probs, dtype=np.float64))
    t_m, t_n = probs.shape
    # same trick as the reference tests (test_masker.py:11-15): any consistent grid
    return ref_mk.PooledMap(probs, b_q=t_n, b_kv=t_m, n_tokens=t_m * t_n)


def mask_cases():
    cases = []  # (probs, k_frac, p_frac, tag)
    # test_masker.py hand rows (67-119)
    cases += [
        ([[0.1] * 10], 0.2, 0.6, "uniform_row"),
        ([[0.1] * 10], 1.0, 0.0, "uniform_row_k1"),
        ([[0.6, 0.2, 0.1, 0.1]], 0.5, 0.6, "sink_row"),
        ([[0.4, 0.3, 0.2, 0.1]], 0.25, 1.0, "p_one"),
        ([[0.4, 0.3, 0.2, 0.1]], 0.25, 0.65, "p_065"),
        ([[0.2, 0.5, 0.3]], 0.0, 0.0, "p_zero"),
        (np.random.Generator(np.random.PCG64(3)).dirichlet(np.ones(7), size=4), 1.0, 0.1, "k_one"),
    ]
    # exact ties, zeros, one-hot rows, prefixes landing exactly on p
    cases += [
        ([[0.25, 0.25, 0.25, 0.25]], 0.5, 0.5, "ties_exact_p"),
        ([[0.5, 0.5, 0.0, 0.0]], 0.25, 1.0, "zeros_p_one"),
        ([[0.0, 0.0, 1.0, 0.0]], 0.0, 1.0, "one_hot"),
        ([[0.125] * 8, [0.5, 0.25, 0.125, 0.0625, 0.03125, 0.015625, 0.0078125, 0.0078125]], 0.3, 0.875, "dyadic"),
        ([[0.1, 0.2, 0.3, 0.4], [0.3, 0.3, 0.2, 0.2]], 0.01, 0.6, "ties_mid"),
    ]
    # c07-style random maps (test_acceptance.py:165-174)
    rng = np.random.Generator(np.random.PCG64(47))
    for r in range(200):
        t_m, t_n = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        alpha = float(rng.choice([0.3, 1.0, 5.0]))
        probs = rng.dirichlet(np.full(t_n, alpha), size=t_m)
        cases.append((probs, float(rng.uniform(0.01, 1.0)), float(rng.uniform(0.01, 1.0)), f"rand{r}"))
    # c06-style boundary thresholds (test_acceptance.py:151-162)
    for r, p in enumerate((1.0, 0.5, 1e-9, 0.0, 0.999999999999)):
        probs = rng.dirichlet(np.ones(12) * 0.7, size=6)
        cases.append((probs, 0.05, p, f"edge_p{r}"))
    # large Wan-like pooled maps (one head each) at the paper's hyperparameters
    for seed, n, d, s, k, p in ((11, 8192, 64, 0.9, 0.03, 0.2), (12, 16384, 128, 0.8, 0.03, 0.16),
                                (13, 4096, 64, 0.0, 0.1, 0.9)):
        q, kk, _, _ = wan_like(seed, n, d, 128, 64, s)
        probs = ref_mk.pooled_map(q[0], kk[0], ref_mk.SparsityConfig(k, p, 128, 64)).probs
        cases.append((np.array(probs), k, p, f"wan_n{n}_d{d}_s{s}"))
    return cases


def build_masks():
    out, meta = {}, []
    for idx, (probs, k, p, tag) in enumerate(mask_cases()):
        pm = _pm(probs)
        cfg = ref_mk.SparsityConfig(k, p, pm.b_q, pm.b_kv)
        out[f"c{idx}_probs"] = np.asarray(pm.probs)
        out[f"c{idx}_topk"] = np.packbits(ref_mk.top_k_mask(pm, k).keep, axis=-1)
        out[f"c{idx}_topp"] = np.packbits(ref_mk.top_p_mask(pm, p).keep, axis=-1)
        out[f"c{idx}_hybrid"] = np.packbits(ref_mk.hybrid_mask(pm, cfg).keep, axis=-1)
        meta.append({"idx": idx, "tag": tag, "k_frac": k, "p_frac": p, "shape": list(pm.probs.shape)})
    np.savez_compressed(os.path.join(HERE, "masks.npz"), **out)
    return meta


def build_pooled():
    out, meta = {}, []
    rng = np.random.Generator(np.random.PCG64(5))
    shapes = [(8, 4, 3, 2), (37, 16, 5, 7), (200, 16, 64, 32), (130, 64, 128, 64), (1, 8, 4, 4)]
    for idx, (n, d, b_q, b_kv) in enumerate(shapes):
        q = rng.normal(size=(n, d))
        k = rng.normal(size=(n, d))
        pm = ref_mk.pooled_map(q, k, ref_mk.SparsityConfig(0.5, 0.5, b_q, b_kv))
        out[f"p{idx}_q"], out[f"p{idx}_k"], out[f"p{idx}_probs"] = q, k, np.asarray(pm.probs)
        meta.append({"idx": idx, "n": n, "d": d, "b_q": b_q, "b_kv": b_kv})
    np.savez_compressed(os.path.join(HERE, "pooled.npz"), **out)
    return meta


# (tag, seed, heads, n, d, s, mask spec, output dtype)
ATTN_CASES = [
    ("n256_d64_rand", 101, 1, 256, 64, 0.0, ("random", 0.5), np.float64),
    ("n300_d64_hybrid", 102, 1, 300, 64, 0.9, ("hybrid", 0.2, 0.5), np.float64),
    ("n192_d64_full", 103, 1, 192, 64, 0.0, ("full",), np.float64),
    ("n520_d128_hybrid", 104, 1, 520, 128, 0.9, ("hybrid", 0.03, 0.2), np.float32),
    # configs[0] of BASELINE.json: B=1 H=2 N=1024 d=64, hybrid k=0.1 / p=0.9
    ("cfg1", 2026, 2, 1024, 64, 0.0, ("hybrid", 0.1, 0.9), np.float32),
]
B_Q, B_KV = 128, 64


def build_attention():
    out, meta = {}, []
    for tag, seed, heads, n, d, s, spec, odt in ATTN_CASES:
        q, k, v, do = wan_like(seed, n, d, B_Q, B_KV, s, heads=heads)
        t_m, t_n = -(-n // B_Q), -(-n // B_KV)
        res = {key: [] for key in ("keep", "out", "lse", "dq", "dk", "dv")}
        for h in range(heads):
            if spec[0] == "random":
                keep = random_keep(seed + h, t_m, t_n, spec[1])
                bm = ref_mk.BlockMask(keep, B_Q, B_KV, n)
                fwd = ref_at.sparse_attention_with_mask(q[h], k[h], v[h], bm)
            elif spec[0] == "full":
                bm = ref_mk.BlockMask(np.ones((t_m, t_n), bool), B_Q, B_KV, n)
                fwd = ref_at.sparse_attention_with_mask(q[h], k[h], v[h], bm)
            else:
                cfg = ref_mk.SparsityConfig(spec[1], spec[2], B_Q, B_KV)
                fwd = ref_at.sparse_attention(q[h], k[h], v[h], cfg)
                bm = fwd.mask_used
            g = ref_at.attention_backward(q[h], k[h], v[h], bm, do[h])
            res["keep"].append(np.asarray(bm.keep))
            res["out"].append(fwd.out)
            res["lse"].append(fwd.lse)
            res["dq"].append(g.dq)
            res["dk"].append(g.dk)
            res["dv"].append(g.dv)
        for key, vals in res.items():
            arr = np.stack(vals)
            out[f"{tag}_{key}"] = np.packbits(arr, axis=-1) if key == "keep" else arr.astype(odt)
        meta.append({"tag": tag, "seed": seed, "heads": heads, "n": n, "d": d, "s": s,
                     "mask": list(spec), "b_q": B_Q, "b_kv": B_KV, "t_n": t_n,
                     "digest": digest(q, k, v, do), "sparsity": float(1 - np.mean(np.stack(res["keep"])))})
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **out)
    return meta


def main():
    manifest = {
        "generator": "tests/golden/make_golden.py",
        "reference": "/root/reference/pkg/src/sparseattn_lab (v0.1.0)",
        "numpy": np.__version__,
        "masks": build_masks(),
        "pooled": build_pooled(),
        "attention": build_attention(),
    }
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(manifest["masks"]), "mask cases,", len(manifest["pooled"]), "pooled cases,",
          len(manifest["attention"]), "attention cases")


if __name__ == "__main__":
    main()

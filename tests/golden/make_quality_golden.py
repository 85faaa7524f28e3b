"""Golden vectors for the mask-quality tooling, from the REAL reference.

Run once in the build container (the only place ``/root/reference`` exists):

    python tests/golden/make_quality_golden.py

For bf16-representable q/k/v (gen.wan_like) and a block mask, it runs the reference's own
functions on the token-level map: ``analysis.error_decompose`` for every query row
(analysis.py:37-65), ``analysis.relative_l1`` (analysis.py:192-200), and the retained mass
of flowmatch._attn_stats (flowmatch.py:408-419: ``(softmax_rows(q kᵀ/√d) * expand_mask(bm))
.sum(axis=1)``), plus the block-level τ̄ of cli.cmd_mask_analyze (cli.py:147-150) on the
reference's pooled map and hybrid mask.  Writes tests/golden/quality.npz.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from gen import random_keep, wan_like  # noqa: E402
from sparseattn_lab import analysis as ref_an  # noqa: E402
from sparseattn_lab import masker as ref_mk  # noqa: E402
from sparseattn_lab.numerics import softmax_rows  # noqa: E402

CASES = [  # (seed, n, d, offset scale, kind, density or (k, p))
    (201, 256, 64, 0.8, "random", 0.4),
    (202, 300, 128, 0.8, "random", 0.3),
    (203, 1024, 64, 0.9, "hybrid", (0.1, 0.5)),
    (204, 777, 128, 0.7, "hybrid", (0.2, 0.6)),
]


def main():
    out = {}
    for idx, (seed, n, d, s, kind, arg) in enumerate(CASES):
        q, k, v, _ = wan_like(seed, n, d, 128, 64, s)
        q, k, v = q[0], k[0], v[0]
        t_m, t_n = -(-n // 128), -(-n // 64)
        if kind == "random":
            keep = random_keep(seed, t_m, t_n, arg)
            bm = ref_mk.BlockMask(keep, 128, 64, n)
            pooled_tau = np.nan
        else:
            cfg = ref_mk.SparsityConfig(arg[0], arg[1], 128, 64)
            pm = ref_mk.pooled_map(q, k, cfg)
            bm = ref_mk.hybrid_mask(pm, cfg)
            keep = np.array(bm.keep)
            pooled_tau = float((pm.probs * bm.keep).sum(axis=1).mean())  # cli.py:150
        em = ref_mk.expand_mask(bm)
        probs = softmax_rows(q @ k.T / math.sqrt(d))
        tau = (probs * em).sum(axis=1)  # flowmatch.py:417-418
        rows = np.arange(0, n, 5)  # the per-row decomposition on every 5th row (fixture size)
        reps = [ref_an.error_decompose(probs[a], em[a], v) for a in rows]
        out[f"q{idx}_rows"] = rows
        out[f"q{idx}_q"], out[f"q{idx}_k"], out[f"q{idx}_v"], out[f"q{idx}_keep"] = q, k, v, keep
        out[f"q{idx}_tau"] = tau
        out[f"q{idx}_tau_report"] = np.array([r.tau for r in reps])
        out[f"q{idx}_dropped"] = np.stack([r.dropped_term for r in reps])
        out[f"q{idx}_renorm"] = np.stack([r.renorm_term for r in reps])
        out[f"q{idx}_total"] = np.stack([r.total_error for r in reps])
        out[f"q{idx}_aggregate"] = np.array(ref_an.relative_l1(probs, em, v))
        out[f"q{idx}_pooled_tau_bar"] = np.array(pooled_tau)
        print(idx, n, d, "tau_bar", tau.mean(), "aggregate", float(out[f"q{idx}_aggregate"]))
    np.savez_compressed(os.path.join(HERE, "quality.npz"), **out)


if __name__ == "__main__":
    main()

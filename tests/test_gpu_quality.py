"""Mask-quality tooling against the REAL reference's own functions
(golden vectors from tests/golden/make_quality_golden.py): retained mass τ per row and τ̄
(flowmatch.py:408-434), the block-level τ̄ of mask-analyze (cli.py:147-150), the per-row
error decomposition (analysis.error_decompose, analysis.py:37-65) and the relative-L1
aggregate (analysis.relative_l1, analysis.py:192-200) — computed on the GPU from the dense
and sparse forwards' LSE and outputs, with no N×N matrix.  bf16 outputs: tolerances are
relative to the scale of o (the dense output)."""

import os

import numpy as np
import pytest
import torch

import paper_2602_13515_b200 as spa
from paper_2602_13515_b200 import quality

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "quality.npz"))
CASES = sorted({k.split("_")[0] for k in GOLD.files})


@pytest.mark.parametrize("case", CASES)
def test_quality_matches_reference(case):
    g = lambda name: GOLD[f"{case}_{name}"]  # noqa: E731
    q, k, v, keep = g("q"), g("k"), g("v"), g("keep")
    n = q.shape[0]
    bm = spa.BlockMask(keep, 128, 64, n)
    tau = quality.retained_mass(q, k, v, bm)
    assert isinstance(tau, np.ndarray) and tau.shape == (n,)
    assert np.abs(tau - g("tau")).max() <= 2e-5  # fp32 LSEs
    rep = quality.error_decomposition(q, k, v, bm)
    rows = g("rows")
    scale = np.abs(g("total")).max()
    for name in ("dropped", "renorm", "total"):
        got = getattr(rep, f"{name}_term" if name != "total" else "total_error")[rows]
        assert np.abs(got - g(name)).max() <= 2e-2 * scale, name
    np.testing.assert_allclose(rep.tau[rows], g("tau_report"), atol=2e-5)
    assert abs(rep.aggregate - float(g("aggregate"))) <= 1e-2 * float(g("aggregate"))
    assert abs(rep.tau_bar - g("tau").mean()) <= 1e-5
    # identity of the reference's decomposition: dropped + renorm == o - o_s
    assert np.abs(rep.dropped_term + rep.renorm_term - rep.total_error).max() <= 1e-12 * scale + 1e-12
    if not np.isnan(g("pooled_tau_bar")):
        cfg = spa.SparsityConfig(*(0.1, 0.5) if n == 1024 else (0.2, 0.6), 128, 64)
        pm = spa.pooled_map(q, k, cfg)
        assert np.array_equal(spa.hybrid_mask(pm, cfg).keep, keep)
        assert abs(quality.pooled_tau_bar(pm, bm) - float(g("pooled_tau_bar"))) <= 1e-12


def test_quality_at_wan_size_without_dense_matrices():
    """configs[1] shape, 12 heads: τ̄ and the aggregate at N = 32760 (the reference would
    need 8.6 GB per head for the token-level map); τ in (0, 1], sane aggregate."""
    from paper_2602_13515_b200.synthetic import wan_like_qkv

    q, k, v = wan_like_qkv(1, 12, 32760, 128, 0.9, seed=5)
    res = spa.sparse_attention(q, k, v, spa.SparsityConfig(0.03, 0.2, 128, 64))
    rep = quality.error_decomposition(q, k, v, res.mask_used)
    tau = rep.tau
    assert tau.shape == (1, 12, 32760)
    assert float(tau.min()) > 0 and float(tau.max()) <= 1.0 + 1e-5
    assert 0.0 < rep.tau_bar < 1.0 and 0.0 < rep.aggregate < 10.0  # rel. L1 may exceed 1 (golden cases: 1.6)
    torch.testing.assert_close(rep.total_error, rep.dropped_term + rep.renorm_term)

"""The A/B switches that remain in libspa2.so keep the results correct, not just the defaults.

Each switch is read once per process (static in libspa2.so / the package), so each case runs a
small fwd + bwd parity check in a fresh interpreter:
  SPA2_NO_FUSED_DELTA=1   δ by its own kernel (k_delta) instead of inside the dQ kernel
  SPA2_PDL=0              no programmatic dependent launch between the hot-path kernels
  SPA2_FUSED_SELECT=0     two-step masker (pooled map, then select) instead of the fused softmax+select
Checked against the float64 oracle at two ragged shapes (d = 64 and 128)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests"); sys.path.insert(0, {root!r} + "/tests/golden")
import oracle
import paper_2602_13515_b200 as spa
from paper_2602_13515_b200 import masker as mk
from gen import random_keep, wan_like
from parity import assert_close
for n, d, density, heads in ((1000, 128, 0.3, 2), (777, 64, 0.5, 1)):
    q, k, v, do = wan_like(5 * n + d, n, d, 128, 64, 0.7, heads=heads)
    t_m, t_n = -(-n // 128), -(-n // 64)
    keep = np.stack([random_keep(n + 7 * h, t_m, t_n, density) for h in range(heads)])
    bm = mk.BlockMask(torch.tensor(keep.reshape(1, heads, t_m, t_n), device="cuda"), 128, 64, n)
    bf = lambda x: torch.tensor(x, device="cuda").to(torch.bfloat16).view(1, heads, n, d)
    res = spa.sparse_attention_with_mask(bf(q), bf(k), bf(v), bm)
    g = spa.attention_backward(bf(q), bf(k), bf(v), bm, bf(do))
    for h in range(heads):
        dq, dk, dv, out, lse = oracle.attention_backward(q[h], k[h], v[h], keep[h], 128, 64, do[h])
        assert_close(f"h{{h}}.out", res.out[0, h], out, "out")
        assert_close(f"h{{h}}.dq", g.dq[0, h], dq, "dq")
        assert_close(f"h{{h}}.dk", g.dk[0, h], dk, "dk")
        assert_close(f"h{{h}}.dv", g.dv[0, h], dv, "dv")
    qt = torch.tensor(q, device="cuda").to(torch.bfloat16).view(1, heads, n, d)
    kt = torch.tensor(k, device="cuda").to(torch.bfloat16).view(1, heads, n, d)
    cfg = mk.SparsityConfig(0.1, 0.5, 128, 64)
    got = spa.sparse_attention(qt, kt, qt, cfg).mask_used.keep.cpu().numpy().reshape(1, heads, t_m, t_n)
    probs = spa.pooled_map(qt, kt, cfg).probs.cpu().numpy().reshape(1, heads, t_m, t_n)  # select: bit-exact given the map
    for h in range(heads):
        assert np.array_equal(got[0, h], oracle.hybrid_keep(probs[0, h], 0.1, 0.5))
print("ok")
"""

VARIANTS = [
    {"SPA2_NO_FUSED_DELTA": "1"},
    {"SPA2_PDL": "0"},
    {"SPA2_FUSED_SELECT": "0"},
]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_variant_parity(env):
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]

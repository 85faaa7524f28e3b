"""Parity check of an alternative libspa2.so build (A/B candidates) against the float64 oracle.

    python tools/variant_check.py alt/NAME/libspa2.so
Runs fwd + bwd at ragged shapes (d = 64 and 128) and a configs[1]-shaped 2-head slice, with the
tolerances of tests/parity.py; exits non-zero on a mismatch."""

import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "tests/golden")
from paper_2602_13515_b200 import _lib  # noqa: E402

_lib.use_library(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2602_13515_b200 as spa  # noqa: E402
from gen import random_keep, wan_like  # noqa: E402
from paper_2602_13515_b200 import masker as mk  # noqa: E402
from parity import assert_close  # noqa: E402

for n, d, density, heads in ((1000, 128, 0.3, 2), (777, 64, 0.5, 1), (4100, 128, 0.08, 2), (300, 128, 1.0, 1)):
    q, k, v, do = wan_like(5 * n + d, n, d, 128, 64, 0.7, heads=heads)
    t_m, t_n = -(-n // 128), -(-n // 64)
    keep = np.stack([random_keep(n + 7 * h, t_m, t_n, density) for h in range(heads)])
    bm = mk.BlockMask(torch.tensor(keep.reshape(1, heads, t_m, t_n), device="cuda"), 128, 64, n)
    bf = lambda x: torch.tensor(x, device="cuda").to(torch.bfloat16).view(1, heads, n, d)  # noqa: E731
    res = spa.sparse_attention_with_mask(bf(q), bf(k), bf(v), bm)
    g = spa.attention_backward(bf(q), bf(k), bf(v), bm, bf(do))
    g2 = spa.attention_backward(bf(q), bf(k), bf(v), bm, bf(do))
    assert all(torch.equal(a, b) for a, b in zip((g.dq, g.dk, g.dv), (g2.dq, g2.dk, g2.dv))), "not deterministic"
    for h in range(heads):
        dq, dk, dv, out, lse = oracle.attention_backward(q[h], k[h], v[h], keep[h], 128, 64, do[h])
        assert_close(f"n{n}.h{h}.out", res.out[0, h], out, "out")
        assert_close(f"n{n}.h{h}.dq", g.dq[0, h], dq, "dq")
        assert_close(f"n{n}.h{h}.dk", g.dk[0, h], dk, "dk")
        assert_close(f"n{n}.h{h}.dv", g.dv[0, h], dv, "dv")
    print("ok", n, d, density, heads, flush=True)
spa.check_pending()
print("variant parity ok:", sys.argv[1])

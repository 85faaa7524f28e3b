"""Reproduce one fuzz case of tests/test_gpu_fuzz.py and print per-row error diagnostics."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tests", "golden")]
import oracle  # noqa: E402
import paper_2602_13515_b200 as spa  # noqa: E402
import test_gpu_fuzz as tf  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 15
rng, b, h, n, d, b_q, _, _ = tf._case(5000 + seed)
b_q, b_kv = int(rng.choice([64, 128])), 64
n = max(n, 65)
k_frac, p_frac = float(rng.uniform(0.0, 0.5)), float(rng.uniform(0.0, 0.95))
q, k, v, do = tf._inputs(rng, b, h, n, d)
print("case", b, h, n, d, b_q, k_frac, p_frac)
cfg = spa.SparsityConfig(k_frac, p_frac, b_q, b_kv)
for trial in range(2):
    qd, kd, vd = tf._dev(q, True), tf._dev(k, True), tf._dev(v, True)
    res = spa.sparse_attention(qd, kd, vd, cfg)
    res.out.backward(tf._dev(do))
    torch.cuda.synchronize()
    keep = res.mask_used.keep_numpy().reshape(b, h, -1, res.mask_used.keep.shape[-1])
    print("keep", keep.astype(int).tolist())
    for bi in range(b):
        for hi in range(h):
            dq, dk, dv, out, lse = oracle.attention_backward(q[bi, hi], k[bi, hi], v[bi, hi], keep[bi, hi], b_q, b_kv, do[bi, hi])
            for name, got, want in (("out", res.out, out), ("lse", res.lse, lse), ("dq", qd.grad, dq), ("dk", kd.grad, dk), ("dv", vd.grad, dv)):
                g = got[bi, hi].detach().double().cpu().numpy()
                err = np.abs(g - want)
                err = err.max(axis=1) if err.ndim == 2 else err
                bad = np.flatnonzero(err > 0.05 * max(1e-9, np.abs(want).max()))
                print(f"[{bi},{hi}] {name}: max err {err.max():.3e} ref max {np.abs(want).max():.3e} bad rows {bad[:20].tolist()} (of {len(bad)})")
    # the same batch alone
    if trial == 0:
        os.environ["SPA2_SYNC_CALLS"] = "1"
bm = res.mask_used
for bi in range(b):
    sub = spa.BlockMask(bm.keep[bi:bi + 1], b_q, b_kv, n)
    qd, kd, vd = (tf._dev(x[bi:bi + 1], True) for x in (q, k, v))
    r = spa.sparse_attention_with_mask(qd, kd, vd, sub)
    r.out.backward(tf._dev(do[bi:bi + 1]))
    dq, dk, dv, out, lse = oracle.attention_backward(q[bi, 0], k[bi, 0], v[bi, 0], keep[bi, 0], b_q, b_kv, do[bi, 0])
    print(f"alone b{bi}: dq err {np.abs(qd.grad[0, 0].double().cpu().numpy() - dq).max():.3e}, dk err {np.abs(kd.grad[0,0].double().cpu().numpy() - dk).max():.3e}")
    g = spa.attention_backward(*(tf._dev(x[bi:bi + 1]) for x in (q, k, v)), sub, tf._dev(do[bi:bi + 1]))
    print(f"direct b{bi}: dq err {np.abs(g.dq[0, 0].double().cpu().numpy() - dq).max():.3e}")

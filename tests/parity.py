"""bf16 parity metrics and the tolerance policy used by every GPU parity test.

The GPU path computes on bf16 operands with fp32 accumulation (tensor cores) and emits
bf16 O / dQ / dK / dV and fp32 LSE; the reference computes in float64 on the *same*
bf16-representable inputs.  Stated tolerances (north_star: "max-abs/rel and cosine"):

  out       cosine >= 0.9999   and  max|Δ| <= 2e-2 · max|ref|
  lse       max|Δ| <= 2e-3     (natural log units)
  dq/dk/dv  cosine >= 0.999    and  max|Δ| <= 6e-2 · max|ref|
"""

import numpy as np

TOL = {
    "out": (0.9999, 2e-2),
    "dq": (0.999, 6e-2),
    "dk": (0.999, 6e-2),
    "dv": (0.999, 6e-2),
}
LSE_ABS = 2e-3


def as_np(x):
    if hasattr(x, "detach"):
        x = x.detach().double().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def metrics(got, want):
    g, w = as_np(got).ravel(), as_np(want).ravel()
    cos = float(g @ w / (np.linalg.norm(g) * np.linalg.norm(w) + 1e-300))
    if np.linalg.norm(w) == 0 and np.linalg.norm(g) == 0:
        cos = 1.0
    rel = float(np.abs(g - w).max() / max(np.abs(w).max(), 1e-12))
    return cos, rel


def assert_close(name, got, want, key=None):
    key = key or name
    if key == "lse":
        err = float(np.abs(as_np(got) - as_np(want)).max())
        assert err <= LSE_ABS, f"{name}: max|Δlse| {err:.3e} > {LSE_ABS}"
        return err
    cos_min, rel_max = TOL[key]
    cos, rel = metrics(got, want)
    assert cos >= cos_min and rel <= rel_max, f"{name}: cosine {cos:.6f} (min {cos_min}), rel {rel:.3e} (max {rel_max})"
    return cos, rel

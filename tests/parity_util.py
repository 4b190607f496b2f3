"""Helpers shared by the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

# north_star: "within 1e-4 relative / 1e-5 absolute in FP32", read as the combined
# allclose form |d| <= 1e-5 + 1e-4 |ref|.
RTOL = 1e-4
ATOL = 1e-5


def parity_report(y, ref64, atol=ATOL, rtol=RTOL, scale=None):
    """Elementwise check of y (fp32) against the fp64 oracle.  `scale` (broadcastable)
    multiplies atol for inputs far from the standardised O(1) range."""
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref64, np.float64)
    a = atol if scale is None else atol * np.asarray(scale, np.float64)
    d = np.abs(y - ref)
    bad = ~(d <= a + rtol * np.abs(ref))
    return {"n": int(d.size), "max_abs": float(d.max()) if d.size else 0.0,
            "n_bad": int(bad.sum()), "worst": None if not bad.any() else
            (int(np.argmax(np.where(bad, d, -1))), float(d[bad].max()))}


def assert_parity(y, ref64, **kw):
    rep = parity_report(y, ref64, **kw)
    assert rep["n_bad"] == 0, f"parity violated: {rep}"
    return rep

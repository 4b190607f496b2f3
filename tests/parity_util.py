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


def revin_stats(x, S):
    """fp64 mean and scale s_r = sqrt(var + 1e-5) of each series' N*S segmented points (the
    statistics the instance normalisation uses, DESIGN.md R-f1), shaped [B, C, 1]."""
    L = x.shape[-1]
    N = L // S
    seg = np.asarray(x, np.float64)[..., L - N * S:]
    mu = seg.mean(axis=-1, keepdims=True)
    s = np.sqrt(seg.var(axis=-1, keepdims=True) + 1e-5)
    return mu, s


def assert_parity_revin(y, ref64, x, S, atol=ATOL, rtol=RTOL):
    """Tolerance reading for instance normalisation (R-tol-revin).  The method
    runs on xhat = (x - mu_r) / s_r, where the north_star bar |d| <= atol + rtol |yhat|
    applies; the de-normalisation y = s_r yhat + mu_r carries it to s_r atol + rtol |ref - mu_r|.
    The statistics themselves are FP32 sums of the FP32 input, |d var| <= 2^-20 max|x|^2,
    and s_r = sqrt(var + 1e-5) turns that into |d s_r| <= 2^-21 max|x|^2 / s_r, which
    multiplies |yhat| (ill-conditioned only for near-constant series, s_r -> sqrt(1e-5)).
    The level term 2^-18 max|x| is the FP32 representation error of the input level and of
    mu_r (2^-24 per element) through the head's gain (sum_n |W_s| + |W_t| <= 16 for the
    seeded test heads, W ~ U(+-1/sqrt(N))), which the de-normalisation does not divide out.
    Last term: fp32 rounding of the output.
        |d| <= s_r atol + rtol |ref - mu_r| + |yhat| 2^-21 max|x|^2 / s_r + 2^-18 max|x|
               + 2^-22 |ref|"""
    mu, s = revin_stats(x, S)
    xm = np.abs(np.asarray(x, np.float64)).max(axis=-1, keepdims=True)
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref64, np.float64)
    yhat = np.abs(ref - mu) / s
    d = np.abs(y - ref)
    tol = (s * atol + rtol * np.abs(ref - mu) + yhat * 2.0 ** -21 * xm * xm / s
           + 2.0 ** -18 * xm + 2.0 ** -22 * np.abs(ref))
    bad = ~(d <= tol)
    assert not bad.any(), (f"parity violated: {int(bad.sum())} of {d.size}, max|d| {d.max():.3e}, "
                           f"worst excess {(d - tol).max():.3e}")
    return {"n": int(d.size), "max_abs": float(d.max())}

"""Pins of the oracle's SURVEY §8(f) widening (DESIGN.md §3 readings R-f1, R-f3):
metric_variant bit 0 (level-only trend), bit 1 (seasonal metric on the residuals about
each segment's least-squares line), instance_norm (RevIN-style normalisation of the
segmented points).

As in test_oracle_pins.py, expected values come from library routines (np.polyfit,
np.corrcoef), invariances that a dropped term / wrong sign / wrong operand would break,
closed forms and limits -- never from re-typing the oracle's formula.
"""
import math

import numpy as np
import pytest


def _run(o, x, S, H, ws, wt, b, tau_s=1.0, tau_t=1.0, mv=0, rev=False, eps_r=None, ma=0):
    kw = {} if eps_r is None else {"eps_r": eps_r}
    kw["ma_kernel"] = ma
    return o.series(np.asarray(x, np.float32), S, H, np.asarray(ws, np.float32),
                    np.asarray(wt, np.float32), np.asarray(b, np.float32), tau_s, tau_t,
                    metric_variant=mv, instance_norm=rev, **kw)


def _params(rng, M, N, H):
    s = 1 / math.sqrt(N)
    return (rng.uniform(-s, s, (M, N)).astype(np.float32),
            rng.uniform(-s, s, (M, N)).astype(np.float32),
            rng.uniform(-s, s, H).astype(np.float32))


# ------------------------------------------------------------ f3: level-only trend
def test_level_trend_is_squared_mean_difference(oracle_mod):
    rng = np.random.default_rng(11)
    x = rng.normal(size=96).astype(np.float32)
    r = _run(oracle_mod, x, 24, 24, *_params(rng, 1, 4, 24), mv=1)
    seg = x.astype(np.float64).reshape(4, 24)
    mu = seg.mean(axis=1)                                   # library mean
    np.testing.assert_allclose(r["dist"], (mu[:, None] - mu[None, :]) ** 2, atol=1e-12)


def test_level_trend_ignores_per_segment_slopes(oracle_mod):
    """Adding a zero-mean ramp b_n (t - t_mid) to each segment changes every kappa but no
    mean: the level-only distance D is unchanged, the full trend distance is not.  (The
    normalised D^ still moves with the series variance of Def 5.)"""
    rng = np.random.default_rng(12)
    S, N = 12, 5
    x = rng.normal(size=N * S)
    ramp = np.concatenate([rng.uniform(-1, 1) * (np.arange(S) - (S - 1) / 2) for _ in range(N)])
    p = _params(rng, 1, N, S)
    a = _run(oracle_mod, x, S, S, *p, mv=1)
    b = _run(oracle_mod, x + ramp, S, S, *p, mv=1)
    np.testing.assert_allclose(a["dist"], b["dist"], atol=1e-5)    # fp32 input rounding
    full_a = _run(oracle_mod, x, S, S, *p, mv=0)
    full_b = _run(oracle_mod, x + ramp, S, S, *p, mv=0)
    assert np.abs(full_a["dist"] - full_b["dist"]).max() > 1e-1


# ------------------------------------------------------------ f3: detrended seasonal
def test_detrended_rho_equals_corrcoef_of_polyfit_residuals(oracle_mod):
    rng = np.random.default_rng(13)
    S, N = 24, 5
    x = rng.normal(size=N * S).astype(np.float32)
    r = _run(oracle_mod, x, S, S, *_params(rng, 1, N, S), mv=2)
    t = np.arange(S, dtype=np.float64)
    res = []
    for n in range(N):
        seg = x[n * S:(n + 1) * S].astype(np.float64)
        res.append(seg - np.polyval(np.polyfit(t, seg, 1), t))   # library line fit
    np.testing.assert_allclose(r["rho"], np.corrcoef(np.array(res)), atol=1e-9)


def test_detrended_rho_invariant_to_added_lines(oracle_mod):
    """Any line a_n + b_n t added to a segment leaves the detrended rho unchanged (the plain
    Pearson rho does change)."""
    rng = np.random.default_rng(14)
    S, N = 16, 4
    x = rng.normal(size=N * S)
    t = np.arange(S)
    lines = np.concatenate([rng.uniform(-2, 2) + rng.uniform(-1, 1) * t for _ in range(N)])
    p = _params(rng, 1, N, S)
    a = _run(oracle_mod, x, S, S, *p, mv=2)
    b = _run(oracle_mod, x + lines, S, S, *p, mv=2)
    np.testing.assert_allclose(a["rho"], b["rho"], atol=2e-6)    # fp32 input rounding
    pa = _run(oracle_mod, x, S, S, *p, mv=0)
    pb = _run(oracle_mod, x + lines, S, S, *p, mv=0)
    assert np.abs(pa["rho"] - pb["rho"]).max() > 1e-2


def test_detrended_pure_lines_give_uniform_seasonal_rows(oracle_mod):
    """Segments that are exact lines have zero residual: rho = 0, A_s uniform (A15 analogue)."""
    S, N = 8, 3
    t = np.arange(S, dtype=np.float32)
    x = np.concatenate([2.0 * t + 1.0, -0.5 * t, 3.0 + 0 * t]).astype(np.float32)
    r = _run(oracle_mod, x, S, S, np.ones((1, N)), np.zeros((1, N)), np.zeros(S), mv=2)
    np.testing.assert_allclose(r["rho"], 0.0, atol=1e-12)
    np.testing.assert_allclose(r["a_s"], 1.0 / N, atol=1e-12)


def test_metric_bits_compose(oracle_mod):
    """mv = 3 takes the seasonal side of mv = 2 and the trend side of mv = 1."""
    rng = np.random.default_rng(15)
    x = rng.normal(size=120).astype(np.float32)
    p = _params(rng, 2, 5, 48)
    r1, r2, r3 = (_run(oracle_mod, x, 24, 48, *p, mv=m) for m in (1, 2, 3))
    np.testing.assert_array_equal(r3["a_t"], r1["a_t"])
    np.testing.assert_array_equal(r3["a_s"], r2["a_s"])


def test_metric_variant_rejected_out_of_range(oracle_mod):
    with pytest.raises(ValueError):
        _run(oracle_mod, np.zeros(48), 24, 24, np.zeros((1, 2)), np.zeros((1, 2)),
             np.zeros(24), mv=8)


# ------------------------------------------------------------ f1: instance normalisation
@pytest.mark.parametrize("mv", [0, 6, 7])
def test_revin_affine_equivariance_without_eps(oracle_mod, mv):
    """With eps_r = 0 the normalised input of a x + b (a > 0) is that of x, so
    f(a x + b) = a f(x) + b exactly (up to fp64 rounding): pins the normalise /
    de-normalise pair, its sign and its placement around the whole method."""
    rng = np.random.default_rng(16)
    S, N, H = 24, 6, 30
    x = np.round(rng.normal(size=N * S) * 1024) / 1024   # 2^-10 grid: a x + b exact in fp32
    p = _params(rng, 2, N, H)
    a, b = 4.0, -3.0
    x32 = x.astype(np.float32)
    assert np.array_equal((a * x32 + b).astype(np.float64), a * x + b)
    y0 = _run(oracle_mod, x32, S, H, *p, mv=mv, rev=True, eps_r=0.0)["y"]
    y1 = _run(oracle_mod, (a * x32 + b).astype(np.float32), S, H, *p, mv=mv, rev=True,
              eps_r=0.0)["y"]
    np.testing.assert_allclose(y1, a * y0 + b, atol=1e-9)
    # without RevIN the same map does not commute (the bias and the level are not rescaled)
    z0 = _run(oracle_mod, x32, S, H, *p, mv=mv)["y"]
    z1 = _run(oracle_mod, (a * x32 + b).astype(np.float32), S, H, *p, mv=mv)["y"]
    assert np.abs(z1 - (a * z0 + b)).max() > 1e-2


def test_revin_constant_series_closed_form(oracle_mod):
    """x = c: var_r = 0, xhat = 0, both attentions uniform, patterns 0, yhat = b, so
    y = b sqrt(eps_r) + c."""
    S, N, H = 8, 3, 10
    rng = np.random.default_rng(17)
    ws, wt, b = _params(rng, 2, N, H)
    c = 2.5
    r = _run(oracle_mod, np.full(N * S, c), S, H, ws, wt, b, rev=True)
    np.testing.assert_allclose(r["y"], b.astype(np.float64) * math.sqrt(1e-5) + c, atol=1e-12)
    np.testing.assert_allclose(r["a_s"], 1.0 / N, atol=1e-12)
    np.testing.assert_allclose(r["a_t"], 1.0 / N, atol=1e-12)


def test_revin_statistics_are_library_mean_and_var(oracle_mod):
    """The normalised segments equal (X - np.mean) / sqrt(np.var + eps) over the segmented
    span (r = 4 dropped points are excluded: reading R-f1)."""
    rng = np.random.default_rng(18)
    S, N = 12, 5
    x = rng.normal(size=N * S + 4).astype(np.float32) * 3 + 1
    r = _run(oracle_mod, x, S, S, *_params(rng, 1, N, S), rev=True)
    xs = x[4:].astype(np.float64)
    np.testing.assert_allclose(r["seg"].ravel(), (xs - xs.mean()) / math.sqrt(xs.var() + 1e-5),
                               atol=1e-12)


def test_revin_on_standardised_input_is_identity_map(oracle_mod):
    """If the segmented points already have mean 0 and variance 1 - eps_r, RevIN is the
    identity on the input and on the output."""
    rng = np.random.default_rng(19)
    S, N, H = 24, 4, 24
    v = rng.normal(size=N * S)
    v = (v - v.mean()) / v.std() * math.sqrt(1 - 1e-5)
    x = v.astype(np.float32)
    p = _params(rng, 1, N, H)
    np.testing.assert_allclose(_run(oracle_mod, x, S, H, *p, rev=True)["y"],
                               _run(oracle_mod, x, S, H, *p)["y"], atol=2e-6)


# ------------------------------------------------------------ f3: component values (A10)
def _lines(seg):
    """Least-squares line of each segment (library polyfit) and its residual."""
    S = seg.shape[1]
    t = np.arange(S, dtype=np.float64)
    T = np.array([np.polyval(np.polyfit(t, row, 1), t) for row in seg])
    return T, seg - T


@pytest.mark.parametrize("mv", [4, 5, 6, 7])
def test_component_values_seasonal_branch(oracle_mod, mv):
    """W_t = 0: Y = W_s A_s V_s with V_s the mean-centred segments (np.mean), or with
    bit 1 the residuals about the np.polyfit line."""
    rng = np.random.default_rng(20 + mv)
    S, N, H = 12, 6, 36
    x = rng.normal(size=N * S).astype(np.float32) + np.linspace(0, 3, N * S, dtype=np.float32)
    ws, wt, b = _params(rng, 3, N, H)
    r = _run(oracle_mod, x, S, H, ws, np.zeros_like(wt), b, mv=mv)
    seg = x.astype(np.float64).reshape(N, S)
    vs = _lines(seg)[1] if mv & 2 else seg - seg.mean(axis=1, keepdims=True)
    np.testing.assert_allclose(r["y_full"], ws.astype(np.float64) @ r["a_s"] @ vs, atol=1e-12)


@pytest.mark.parametrize("mv", [4, 5, 6, 7])
def test_component_values_trend_branch(oracle_mod, mv):
    """W_s = 0: Y = W_t A_t V_t with V_t the np.polyfit line of each segment, or with
    bit 0 (level-only trend) its mean: every output segment is a line / a constant."""
    rng = np.random.default_rng(30 + mv)
    S, N, H = 12, 6, 36
    x = rng.normal(size=N * S).astype(np.float32)
    ws, wt, b = _params(rng, 3, N, H)
    r = _run(oracle_mod, x, S, H, np.zeros_like(ws), wt, b, mv=mv)
    seg = x.astype(np.float64).reshape(N, S)
    vt = np.repeat(seg.mean(axis=1, keepdims=True), S, axis=1) if mv & 1 else _lines(seg)[0]
    np.testing.assert_allclose(r["y_full"], wt.astype(np.float64) @ r["a_t"] @ vt, atol=1e-12)
    d2 = np.diff(r["y_full"], n=2, axis=1)            # lines: zero second differences
    np.testing.assert_allclose(d2, 0.0, atol=1e-12)
    if mv & 1:
        np.testing.assert_allclose(np.diff(r["y_full"], axis=1), 0.0, atol=1e-12)


def test_component_values_detrended_split_sums_to_the_series(oracle_mod):
    """mv = 6: residual + line = the segment.  With uniform attention (tau -> inf) and
    W_s = W_t = W, the component forecast is half the plain one (which aggregates X in
    both branches)."""
    rng = np.random.default_rng(40)
    S, N, H = 8, 5, 16
    x = rng.normal(size=N * S).astype(np.float32)
    w, _, b = _params(rng, 2, N, H)
    big = 1e12
    yc = _run(oracle_mod, x, S, H, w, w, b, tau_s=big, tau_t=big, mv=6)["y"]
    yp = _run(oracle_mod, x, S, H, w, w, b, tau_s=big, tau_t=big, mv=0)["y"]
    np.testing.assert_allclose(yc - b, (yp - b) / 2, atol=1e-9)
    # plain component split (mv = 4) does not sum to X: z_n + T_n = X_n + kappa_n t~
    y4 = _run(oracle_mod, x, S, H, w, w, b, tau_s=big, tau_t=big, mv=4)["y"]
    assert np.abs((y4 - b) - (yp - b) / 2).max() > 1e-3


def test_component_values_leave_attention_unchanged(oracle_mod):
    """Bit 2 changes only the aggregated values, never the attention weights."""
    rng = np.random.default_rng(41)
    x = rng.normal(size=96).astype(np.float32)
    p = _params(rng, 2, 4, 48)
    for mv in range(4):
        a = _run(oracle_mod, x, 24, 48, *p, mv=mv)
        c = _run(oracle_mod, x, 24, 48, *p, mv=mv | 4)
        np.testing.assert_array_equal(a["a_s"], c["a_s"])
        np.testing.assert_array_equal(a["a_t"], c["a_t"])


# ------------------------------------------------------------ f3: moving-average decomposition
def _ma_split(seg_flat, k):
    """Library moving average: np.pad (edge) + np.convolve, and the remainder."""
    h = (k - 1) // 2
    t = np.convolve(np.pad(seg_flat, h, mode="edge"), np.ones(k) / k, mode="valid")
    return seg_flat - t, t


def test_ma_kernel_one_is_all_trend(oracle_mod):
    """k = 1: the trend is the series and the seasonal part is 0 (uniform A_s, P_s = 0), so
    the forecast is the plain one with W_s = 0."""
    rng = np.random.default_rng(50)
    S, N, H = 12, 5, 30
    x = rng.normal(size=N * S).astype(np.float32)
    ws, wt, b = _params(rng, 3, N, H)
    r = _run(oracle_mod, x, S, H, ws, wt, b, ma=1)
    np.testing.assert_allclose(r["a_s"], 1.0 / N, atol=1e-12)
    np.testing.assert_allclose(r["y"], _run(oracle_mod, x, S, H, np.zeros_like(ws), wt, b)["y"],
                               atol=1e-12)


@pytest.mark.parametrize("k", [3, 25])
def test_ma_components_match_library_convolution(oracle_mod, k):
    """Uniform attention (tau -> inf) makes each pattern the segment mean of its branch's
    input: W_t = 0 exposes mean_n Xs_n, W_s = 0 mean_n Xt_n, with Xt = np.convolve of the
    edge-padded segmented points."""
    rng = np.random.default_rng(51 + k)
    S, N, H = 12, 6, 24
    x = rng.normal(size=N * S + 5).astype(np.float32)   # r = 5 dropped points
    ws, wt, b = _params(rng, 2, N, H)
    big = 1e12
    xs, xt = _ma_split(x[5:].astype(np.float64), k)
    ys = _run(oracle_mod, x, S, H, ws, np.zeros_like(wt), b, tau_s=big, tau_t=big, ma=k)
    np.testing.assert_allclose(ys["y_full"], ws.astype(np.float64) @ np.tile(
        xs.reshape(N, S).mean(axis=0), (N, 1)), atol=1e-9)
    yt = _run(oracle_mod, x, S, H, np.zeros_like(ws), wt, b, tau_s=big, tau_t=big, ma=k)
    np.testing.assert_allclose(yt["y_full"], wt.astype(np.float64) @ np.tile(
        xt.reshape(N, S).mean(axis=0), (N, 1)), atol=1e-9)


def test_ma_branch_metrics_on_their_components(oracle_mod):
    """rho is np.corrcoef of the seasonal component's segments; D is (1/S)|T_i - T_j|^2 of
    the np.polyfit lines of the trend component's segments; sigma^2 is np.var of the trend
    component."""
    rng = np.random.default_rng(53)
    S, N, k = 16, 5, 7
    x = (rng.normal(size=N * S) + np.sin(np.arange(N * S) / 3.0)).astype(np.float32)
    r = _run(oracle_mod, x, S, S, *_params(rng, 1, N, S), ma=k)
    xs, xt = _ma_split(x.astype(np.float64), k)
    np.testing.assert_allclose(r["rho"], np.corrcoef(xs.reshape(N, S)), atol=1e-9)
    T = _lines(xt.reshape(N, S))[0]
    D = ((T[:, None, :] - T[None, :, :]) ** 2).sum(axis=2) / S
    np.testing.assert_allclose(r["dist"], D, atol=1e-10)
    np.testing.assert_allclose(r["sigma2"], xt.var(), atol=1e-12)


def test_ma_constant_series_closed_form(oracle_mod):
    """x = c: trend = c, seasonal = 0, both attentions uniform: y = c W_t 1 + b."""
    S, N, H = 8, 4, 16
    rng = np.random.default_rng(54)
    ws, wt, b = _params(rng, 2, N, H)
    c = -1.75
    r = _run(oracle_mod, np.full(N * S, c), S, H, ws, wt, b, ma=5)
    yf = c * wt.astype(np.float64).sum(axis=1)[:, None] * np.ones((1, S))
    np.testing.assert_allclose(r["y"], yf.ravel()[:H] + b, atol=1e-12)


@pytest.mark.parametrize("mv", [0, 7])
def test_ma_revin_affine_equivariance(oracle_mod, mv):
    rng = np.random.default_rng(55)
    S, N, H = 12, 6, 30
    x = (np.round(rng.normal(size=N * S) * 1024) / 1024).astype(np.float32)
    p = _params(rng, 3, N, H)
    a, b = 2.0, 5.0
    y0 = _run(oracle_mod, x, S, H, *p, mv=mv, rev=True, eps_r=0.0, ma=9)["y"]
    y1 = _run(oracle_mod, (a * x + b).astype(np.float32), S, H, *p, mv=mv, rev=True, eps_r=0.0,
              ma=9)["y"]
    np.testing.assert_allclose(y1, a * y0 + b, atol=1e-9)


@pytest.mark.parametrize("k", [-1, 2, 24])
def test_ma_kernel_rejected(oracle_mod, k):
    with pytest.raises(ValueError):
        _run(oracle_mod, np.zeros(48), 24, 24, np.zeros((1, 2)), np.zeros((1, 2)), np.zeros(24),
             ma=k)

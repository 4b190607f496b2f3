"""Pins of the oracle's full backward (DESIGN.md §3 reading R-f7).

The gradient with respect to the input and the temperatures is checked against central
differences of the oracle's fp64 FORWARD (a separate code path: oracle_forward_ex does not
call any adjoint function), Richardson-extrapolated (error O(h^4)); the inputs are dyadic so
x +- h stays exact in fp32.  Two closed forms: the points dropped by Def 2 get zero gradient,
and a global shift x + c moves y by c (W_s + W_t) 1 (rows of A sum to 1, rho and Dhat are
shift invariant), so the gradient summed over the used points equals
sum_m (sum_t dY[m][t]) (sum_n W_s[m][n] + W_t[m][n]).  The head gradients equal the separately
pinned head backward.
"""
import math

import numpy as np
import pytest


def _setup(rng, B, C, L, S, H, hpc=True):
    N, M = L // S, -(-H // S)
    Cw = C if hpc else 1
    s = 1 / math.sqrt(N)
    q = lambda a, k=10: (np.round(a * 2 ** k) / 2 ** k).astype(np.float32)
    ws = q(rng.uniform(-s, s, (Cw, M, N)))
    wt = q(rng.uniform(-s, s, (Cw, M, N)))
    b = q(rng.uniform(-s, s, (Cw, H)))
    t = np.arange(L)
    x = (np.sin(2 * np.pi * t / rng.integers(5, 17, (B, C, 1))) + 0.3 * rng.normal(size=(B, C, L))
         + rng.normal(0, 0.5, (B, C, 1)))
    x = q(x, 12)
    dy = rng.normal(size=(B, C, H)).astype(np.float32)
    return x, ws, wt, b, dy


def _loss(o, x, S, H, ws, wt, b, dy, hpc, tau_s, tau_t, mv=0):
    _, y64 = o.forward_ex(x, S, H, ws, wt, b, hpc, tau_s, tau_t, mv) if hasattr(o, "forward_ex") \
        else o.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t, metric_variant=mv)
    return float((y64 * dy.astype(np.float64)).sum())


def _fd_x(o, x, idx, h, *args):
    def d(hh):
        p, m = x.copy(), x.copy()
        p[idx] += hh
        m[idx] -= hh
        assert p[idx] - x[idx] == hh and x[idx] - m[idx] == hh   # exact in fp32
        return (_loss(o, p, *args) - _loss(o, m, *args)) / (2 * hh)
    return (4 * d(h / 2) - d(h)) / 3


@pytest.mark.parametrize("L,S,H,tau_s,tau_t,mv", [
    (60, 12, 30, 1.0, 1.0, 0), (50, 12, 25, 0.5, 2.0, 0), (96, 24, 96, 1.0, 1.0, 0),
    (41, 8, 19, 0.3, 0.7, 1), (30, 6, 7, 2.0, 0.4, 0)])
def test_input_gradient_matches_central_differences(oracle_mod, L, S, H, tau_s, tau_t, mv):
    rng = np.random.default_rng(70 + L)
    x, ws, wt, b, dy = _setup(rng, 2, 2, L, S, H)
    g = oracle_mod.backward(x, S, H, ws, wt, b, dy, True, tau_s, tau_t, metric_variant=mv)
    N = L // S
    r = L - N * S
    args = (S, H, ws, wt, b, dy, True, tau_s, tau_t, mv)
    picks = [(0, 0, r), (1, 1, L - 1), (0, 1, r + S // 2), (1, 0, r + S * (N // 2) + 1)]
    for idx in picks:
        fd = _fd_x(oracle_mod, x, idx, 2.0 ** -8, *args)
        assert abs(fd - g["dx"][idx]) <= 2e-7 * max(1.0, abs(fd)), (idx, fd, g["dx"][idx])


def test_dropped_points_have_zero_gradient(oracle_mod):
    rng = np.random.default_rng(71)
    L, S, H = 53, 12, 24          # r = 5
    x, ws, wt, b, dy = _setup(rng, 2, 3, L, S, H)
    g = oracle_mod.backward(x, S, H, ws, wt, b, dy, True)
    assert np.all(g["dx"][:, :, :5] == 0.0)
    assert np.any(g["dx"][:, :, 5:] != 0.0)


@pytest.mark.parametrize("L,S,H", [(60, 12, 30), (96, 24, 96), (73, 7, 40)])
def test_global_shift_closed_form(oracle_mod, L, S, H):
    rng = np.random.default_rng(72 + S)
    x, ws, wt, b, dy = _setup(rng, 3, 2, L, S, H)
    g = oracle_mod.backward(x, S, H, ws, wt, b, dy, True, 0.7, 1.3)
    N, M = L // S, -(-H // S)
    r = L - N * S
    dY = np.zeros((3, 2, M * S))
    dY[..., :H] = dy
    dY = dY.reshape(3, 2, M, S).sum(-1)                       # sum_t dY[m][t]
    wsum = (ws.astype(np.float64) + wt.astype(np.float64)).sum(-1)   # [C, M]
    want = (dY * wsum[None]).sum(-1)                           # [B, C]
    np.testing.assert_allclose(g["dx"][..., r:].sum(-1), want, rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("which", [0, 1])
def test_temperature_gradients_match_central_differences(oracle_mod, which):
    rng = np.random.default_rng(73)
    L, S, H = 72, 12, 36
    x, ws, wt, b, dy = _setup(rng, 2, 2, L, S, H)
    ts, tt = 0.6, 1.7
    g = oracle_mod.backward(x, S, H, ws, wt, b, dy, True, ts, tt)

    def d(h):
        a = [ts, tt]
        a[which] += h
        lp = _loss(oracle_mod, x, S, H, ws, wt, b, dy, True, a[0], a[1])
        a[which] -= 2 * h
        lm = _loss(oracle_mod, x, S, H, ws, wt, b, dy, True, a[0], a[1])
        return (lp - lm) / (2 * h)
    fd = (4 * d(5e-4) - d(1e-3)) / 3
    assert abs(fd - g["dtau"][which]) <= 1e-8 * max(1.0, abs(fd)), (fd, g["dtau"][which])


@pytest.mark.parametrize("hpc", [True, False])
def test_head_gradients_equal_head_backward(oracle_mod, hpc):
    rng = np.random.default_rng(74)
    x, ws, wt, b, dy = _setup(rng, 3, 2, 60, 12, 30, hpc)
    g = oracle_mod.backward(x, 12, 30, ws, wt, b, dy, hpc)
    dws, dwt, db = oracle_mod.backward_head(x, 12, 30, ws, wt, b, dy, hpc)
    np.testing.assert_allclose(g["dws"], dws, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(g["dwt"], dwt, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(g["db"], db, rtol=1e-12, atol=1e-14)


def test_constant_series_gradient(oracle_mod):
    """A constant series: every segment constant (z = 0, rho = 0, D = 0) -> uniform attention;
    y = c (W_s + W_t) 1 + b, so dx on the used points is the shift form spread uniformly per
    segment, i.e. dX[n][t] = sum_m dY[m][t]-weighted column sums / N: checked through the
    forward's linearity in c via central differences of a scalar shift."""
    rng = np.random.default_rng(75)
    L, S, H = 48, 12, 24
    x, ws, wt, b, dy = _setup(rng, 1, 1, L, S, H)
    x[:] = np.float32(0.75)
    g = oracle_mod.backward(x, S, H, ws, wt, b, dy, True)
    assert np.all(np.isfinite(g["dx"]))
    N, M = L // S, -(-H // S)
    dY = np.zeros(M * S)
    dY[:H] = dy[0, 0]
    dY = dY.reshape(M, S)
    # uniform attention: P = mean segment, y depends on x only through the mean over n
    # -> dX[n][t] = (1/N) sum_m (sum_i W_s[m][i] + W_t[m][i]) dY[m][t], plus the metric paths,
    # which vanish at the constant series (dD/dmu and drho terms are 0 there)
    wsum = (ws[0].astype(np.float64) + wt[0].astype(np.float64)).sum(-1)    # [M]
    want = np.tile((wsum[:, None] * dY).sum(0) / N, N)
    np.testing.assert_allclose(g["dx"][0, 0], want, rtol=1e-9, atol=1e-12)

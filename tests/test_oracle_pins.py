"""Pins of the CPU oracle against things other than itself.

Each test names the SURVEY.md §8(c) pin (T1..T14) it implements and the
Definition step(s) it fixes.  The expected values come from closed forms,
invariants, limits that reduce the method to a textbook/library routine
(np.polyfit, np.corrcoef, a plain matmul), brute-force enumeration, or the
cited worked example (tests/golden/survey_worked_example.json).  None of them
re-types an oracle formula.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "survey_worked_example.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLDEN) as f:
        return json.load(f)


def _run(o, x, S, H, ws, wt, b, tau_s=1.0, tau_t=1.0):
    return o.series(np.asarray(x, np.float32), S, H, np.asarray(ws, np.float32),
                    np.asarray(wt, np.float32), np.asarray(b, np.float32), tau_s, tau_t)


def _rand_params(rng, M, N, H, scale=None):
    s = 1 / math.sqrt(N) if scale is None else scale
    return (rng.uniform(-s, s, (M, N)).astype(np.float32),
            rng.uniform(-s, s, (M, N)).astype(np.float32),
            rng.uniform(-s, s, H).astype(np.float32))


# ---------------------------------------------------------------- Definition step 1
def test_dims(oracle_mod):
    o = oracle_mod
    assert o.dims(720, 24, 720) == (30, 0, 30)
    assert o.dims(720, 96, 96) == (7, 48, 1)       # CFG5 point with r = 48
    assert o.dims(96, 24, 100) == (4, 0, 5)        # ceil(100/24) = 5
    assert o.dims(5760, 12, 96) == (480, 0, 8)
    assert o.dims(25, 24, 1) == (1, 1, 1)
    for bad in ((23, 24, 96), (96, 1, 96), (96, 24, 0)):
        with pytest.raises(ValueError):
            o.dims(*bad)


# ---------------------------------------------------------------- T14 worked example
def test_case_a_golden(oracle_mod, gold):
    g = gold["case_a"]
    r = _run(oracle_mod, g["x"], g["S"], g["H"], g["ws"], g["wt"], g["bias"])
    np.testing.assert_allclose(r["mu"], g["mu"], atol=1e-12)
    np.testing.assert_allclose(r["nu2"], g["nu2"], atol=1e-12)
    np.testing.assert_allclose(r["kappa"], g["kappa"], atol=1e-12)
    assert abs(r["sigma2"] - g["sigma2"]) < 1e-10
    np.testing.assert_allclose(r["rho"], g["rho"], atol=1e-10)
    np.testing.assert_allclose(r["dist"], g["dist"], atol=1e-12)
    np.testing.assert_allclose(r["a_s"], g["a_s"], atol=1e-11)
    np.testing.assert_allclose(r["a_t"], g["a_t"], atol=1e-11)
    np.testing.assert_allclose(r["p_s"][0], g["p_s_row0"], atol=1e-10)
    np.testing.assert_allclose(r["p_t"][2], g["p_t_row2"], atol=1e-10)
    # fp32 rounding of the decimal bias (0.1f - 0.1 = 1.5e-9) is the only difference
    np.testing.assert_allclose(r["y"], g["y"], atol=1e-8)


def test_case_b_drops_oldest_points(oracle_mod, gold):
    """Reading A2: L mod S != 0 drops the r oldest points (T1 index map)."""
    a, b = gold["case_a"], gold["case_b"]
    ra = _run(oracle_mod, a["x"], a["S"], a["H"], a["ws"], a["wt"], a["bias"])
    rb = _run(oracle_mod, b["x"], b["S"], b["H"], a["ws"], a["wt"], a["bias"])
    assert rb["r"] == 2 and rb["N"] == 3
    np.testing.assert_array_equal(rb["seg"][0], b["seg_row0"])
    np.testing.assert_array_equal(rb["y"], ra["y"])


def test_case_c_horizon_truncation(oracle_mod, gold):
    """Reading A3: M = ceil(H/S) future segments, first H steps kept."""
    g = gold["case_c"]
    r = _run(oracle_mod, g["x"], g["S"], g["H"], g["ws"], g["wt"], g["bias"])
    assert r["M"] == 2
    np.testing.assert_allclose(r["y"], g["y"], atol=1e-10)
    # future segment 1 = P_s row 1 (W_s[1] = e_1), steps t = 0, 1
    np.testing.assert_allclose(r["y"][4:6], r["p_s"][1][:2], atol=1e-15)


def test_case_d_constant_series(oracle_mod, gold):
    """Reading A15 / T10: constant series -> uniform rows in both branches."""
    g = gold["case_d"]
    r = _run(oracle_mod, g["x"], g["S"], g["H"], g["ws"], g["wt"], g["bias"])
    np.testing.assert_array_equal(r["a_s"], g["a"])
    np.testing.assert_array_equal(r["a_t"], g["a"])
    np.testing.assert_array_equal(r["y"], g["y"])


# ---------------------------------------------------------------- T2 descriptors (step 3-4)
def test_segment_descriptors_closed_form(oracle_mod):
    r = _run(oracle_mod, [1, 2, 3, 4], 4, 4, [[0]], [[0]], [0, 0, 0, 0])
    assert r["mu"][0] == 2.5 and r["nu2"][0] == 5.0 and r["kappa"][0] == 1.0


@pytest.mark.parametrize("S", [2, 3, 12, 24, 97])
def test_descriptors_match_library_routines(oracle_mod, S):
    """mu = np.mean, nu2 = S * np.var (population), kappa = np.polyfit slope."""
    rng = np.random.default_rng(S)
    N = 5
    off = min(3, S - 1)
    x = rng.normal(size=N * S + off).astype(np.float32)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    segs = x[off:].astype(np.float64).reshape(N, S)
    np.testing.assert_array_equal(r["seg"], segs)
    np.testing.assert_allclose(r["mu"], segs.mean(1), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(r["nu2"], S * segs.var(1), rtol=1e-12)
    slope = np.array([np.polyfit(np.arange(S), s, 1)[0] for s in segs])
    np.testing.assert_allclose(r["kappa"], slope, rtol=1e-9, atol=1e-12)
    # sigma^2 = population variance of the N*S segmented points
    assert abs(r["sigma2"] - segs.var()) < 1e-12 * max(1, segs.var())


# ---------------------------------------------------------------- T3-T6 seasonal metric (step 6)
def test_rho_equals_pearson_corrcoef(oracle_mod):
    rng = np.random.default_rng(1)
    N, S = 7, 24
    x = rng.normal(size=N * S).astype(np.float32)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    np.testing.assert_allclose(r["rho"], np.corrcoef(x.astype(np.float64).reshape(N, S)),
                               atol=1e-11)


def test_rho_znorm_distance_identity(oracle_mod):
    """T3: ||zhat_i - zhat_j||^2 = 2 S (1 - rho_ij), zhat = population z-normalisation."""
    rng = np.random.default_rng(2)
    N, S = 6, 12
    x = rng.normal(size=N * S).astype(np.float32)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    seg = x.astype(np.float64).reshape(N, S)
    zh = (seg - seg.mean(1, keepdims=True)) / seg.std(1, keepdims=True)
    d2 = ((zh[:, None, :] - zh[None, :, :]) ** 2).sum(-1)
    np.testing.assert_allclose(d2, 2 * S * (1 - r["rho"]), atol=1e-9)


def test_rho_properties(oracle_mod):
    """T4: symmetric, |rho| <= 1, rho_ii = nu2/(nu2+eps), diagonal is the row max."""
    rng = np.random.default_rng(3)
    N, S = 9, 16
    x = rng.normal(size=N * S).astype(np.float32)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    rho = r["rho"]
    np.testing.assert_array_equal(rho, rho.T)
    assert np.all(np.abs(rho) <= 1.0)
    np.testing.assert_allclose(np.diag(rho), 1.0, atol=1e-11)
    assert np.all(np.argmax(rho, axis=1) == np.arange(N))
    assert np.all(np.argmax(r["a_s"], axis=1) == np.arange(N))
    assert np.all(np.argmax(r["a_t"], axis=1) == np.arange(N))


def test_rho_per_segment_affine_map(oracle_mod):
    """T5: rho unchanged by a*x+b (a > 0) on one segment; sign flips when a < 0."""
    rng = np.random.default_rng(4)
    N, S = 5, 8
    base = rng.normal(size=(N, S))
    def rho_of(seg):
        x = seg.astype(np.float32).ravel()
        return _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])["rho"]
    r0 = rho_of(base)
    pos = base.copy(); pos[2] = 2.0 * pos[2] + 3.0           # exact in fp32 (powers of two)
    np.testing.assert_allclose(rho_of(pos), r0, atol=1e-7)
    neg = base.copy(); neg[2] = -0.5 * neg[2] + 1.0
    r2 = rho_of(neg)
    flip = np.ones(N); flip[2] = -1
    expect = r0 * flip[:, None] * flip[None, :]
    np.testing.assert_allclose(r2, expect, atol=1e-7)


@pytest.mark.parametrize("S", [3, 4, 12, 24, 96])
def test_rho_sinusoid_closed_form(oracle_mod, S):
    """T6: rho(sin(w t), sin(w t + phi)) = cos(phi) for w = 2 pi / S."""
    phis = np.array([0.0, 0.3, 1.1, 2.0, 3.0])
    t = np.arange(S)
    seg = np.sin(2 * np.pi * t[None, :] / S + phis[:, None])
    x = seg.astype(np.float32).ravel()
    N = len(phis)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    np.testing.assert_allclose(r["rho"][0], np.cos(phis - phis[0]), atol=2e-6)  # fp32 input


# ---------------------------------------------------------------- T7 trend metric (step 5, 7)
def test_trend_distance_is_line_distance(oracle_mod):
    """D_ij = (1/S) ||T_i - T_j||^2 with T_n the np.polyfit least-squares line."""
    rng = np.random.default_rng(5)
    N, S = 6, 24
    x = rng.normal(size=N * S).astype(np.float32)
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    seg = x.astype(np.float64).reshape(N, S)
    t = np.arange(S)
    lines = np.array([np.polyval(np.polyfit(t, s, 1), t) for s in seg])
    D = ((lines[:, None, :] - lines[None, :, :]) ** 2).mean(-1)
    np.testing.assert_allclose(r["dist"], D, atol=1e-9)
    np.testing.assert_array_equal(np.diag(r["dist"]), 0.0)
    np.testing.assert_array_equal(r["dist"], r["dist"].T)


def test_trend_exact_lines_and_orthogonal_invariance(oracle_mod):
    """For exact lines D = mean squared difference; adding a component orthogonal to
    span{1, t} to any segment leaves D unchanged."""
    S, N = 8, 4
    t = np.arange(S, dtype=np.float64)
    lines = np.array([0.5 + 0.25 * t, -1.0 + 0.5 * t, 2.0 - 0.25 * t, 0.0 * t])
    x = lines.astype(np.float32).ravel()
    r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0])
    msd = ((lines[:, None, :] - lines[None, :, :]) ** 2).mean(-1)
    np.testing.assert_allclose(r["dist"], msd, atol=1e-12)
    # orthogonal component: a quadratic with the {1, t} part projected out, exact in fp32
    q = np.array([7, 1, -3, -5, -5, -3, 1, 7], dtype=np.float64)   # orthogonal to 1 and t
    assert abs(q.sum()) == 0 and abs((q * (t - t.mean())).sum()) == 0
    lines2 = lines.copy(); lines2[1] += 0.125 * q; lines2[3] -= 0.5 * q
    r2 = _run(oracle_mod, lines2.astype(np.float32).ravel(), S, 1, np.zeros((1, N)),
              np.zeros((1, N)), [0])
    np.testing.assert_allclose(r2["dist"], r["dist"], atol=1e-12)


def test_trend_normalised_global_affine_invariance(oracle_mod):
    """Dhat = D / (sigma^2 + eps_t) is invariant to x -> a x + b up to the eps_t term."""
    rng = np.random.default_rng(6)
    N, S = 6, 12
    x = (rng.normal(size=N * S) * 30).astype(np.float32)            # sigma^2 >> eps_t
    z = np.zeros((1, N))
    r0 = _run(oracle_mod, x, S, 1, z, z, [0])
    r1 = _run(oracle_mod, (-4.0 * x + 10.0).astype(np.float32), S, 1, z, z, [0])
    np.testing.assert_allclose(r1["a_t"], r0["a_t"], atol=1e-7)
    np.testing.assert_allclose(r1["a_s"], r0["a_s"], atol=1e-7)   # rho: global a<0 flips both


# ---------------------------------------------------------------- T8 softmax (step 8)
def test_rows_sum_to_one(oracle_mod):
    rng = np.random.default_rng(7)
    N, S = 11, 9
    x = rng.normal(size=N * S).astype(np.float32)
    for tau in (0.05, 1.0, 10.0):
        r = _run(oracle_mod, x, S, 1, np.zeros((1, N)), np.zeros((1, N)), [0], tau, tau)
        np.testing.assert_allclose(r["a_s"].sum(1), 1.0, atol=1e-14)
        np.testing.assert_allclose(r["a_t"].sum(1), 1.0, atol=1e-14)
        assert np.all(r["a_s"] > 0) or tau < 0.1


@pytest.mark.parametrize("tau", [0.1, 0.5, 1.0, 3.0])
def test_two_segment_logistic_seasonal(oracle_mod, tau):
    """N = 2 with anti-correlated segments: rho_01 = -1, so
    A_s[0][0] = 1 / (1 + exp(-(1 - (-1)) / tau_s))  (pins sign and temperature)."""
    seg = np.array([1, 3, 2, 5], np.float64)
    x = np.concatenate([seg, -seg]).astype(np.float32)
    r = _run(oracle_mod, x, 4, 1, np.zeros((1, 2)), np.zeros((1, 2)), [0], tau, 1.0)
    expect = 1 / (1 + math.exp(-2 * (1 - 1e-12 / (np.var(seg) * 4 + 1e-12)) / tau))
    assert abs(r["a_s"][0, 0] - expect) < 1e-12


@pytest.mark.parametrize("tau", [0.1, 1.0, 7.0])
def test_two_segment_logistic_trend(oracle_mod, tau):
    """N = 2 constant segments at levels 0 and d: D_01 = d^2, sigma^2 = d^2/4, so
    A_t[0][0] = 1 / (1 + exp(-(d^2 / (d^2/4 + 1e-5)) / tau_t))."""
    d = 2.0
    x = np.array([0, 0, 0, d, d, d], np.float32)
    r = _run(oracle_mod, x, 3, 1, np.zeros((1, 2)), np.zeros((1, 2)), [0], 1.0, tau)
    dh = d * d / (d * d / 4 + 1e-5)
    assert abs(r["a_t"][0, 0] - 1 / (1 + math.exp(-dh / tau))) < 1e-12
    # constant segments: rho = 0 everywhere -> uniform seasonal rows (reading A15)
    np.testing.assert_array_equal(r["a_s"], 0.5)


# ---------------------------------------------------------------- T9 permutation equivariance
@pytest.mark.parametrize("N", [2, 3, 4])
def test_permutation_equivariance_bruteforce(oracle_mod, N):
    """Permuting segments permutes A's rows and columns and P's rows; with the head's
    columns permuted the same way y is unchanged.  All N! orders."""
    rng = np.random.default_rng(10 + N)
    S, H = 5, 7
    M = -(-H // S)
    seg = rng.normal(size=(N, S))
    ws, wt, b = _rand_params(rng, M, N, H)
    base = _run(oracle_mod, seg.astype(np.float32).ravel(), S, H, ws, wt, b)
    for perm in itertools.permutations(range(N)):
        p = np.array(perm)
        r = _run(oracle_mod, seg[p].astype(np.float32).ravel(), S, H, ws[:, p], wt[:, p], b)
        np.testing.assert_allclose(r["a_s"], base["a_s"][np.ix_(p, p)], atol=1e-14)
        np.testing.assert_allclose(r["a_t"], base["a_t"][np.ix_(p, p)], atol=1e-14)
        np.testing.assert_allclose(r["p_s"], base["p_s"][p], atol=1e-13)
        np.testing.assert_allclose(r["p_t"], base["p_t"][p], atol=1e-13)
        np.testing.assert_allclose(r["y"], base["y"], atol=1e-13)


# ---------------------------------------------------------------- T10/T11 degenerate cases
def test_single_segment(oracle_mod):
    """N = 1: A = [1], P = X, y = (ws + wt) X + b."""
    rng = np.random.default_rng(11)
    S, H = 6, 9
    x = rng.normal(size=S + 2).astype(np.float32)
    ws, wt, b = _rand_params(rng, 2, 1, H)
    r = _run(oracle_mod, x, S, H, ws, wt, b)
    assert r["N"] == 1 and r["r"] == 2
    np.testing.assert_array_equal(r["a_s"], [[1.0]])
    np.testing.assert_array_equal(r["a_t"], [[1.0]])
    Y = (ws.astype(np.float64) + wt) @ x[2:].astype(np.float64)[None, :]
    np.testing.assert_allclose(r["y"], Y.ravel()[:H] + b, atol=1e-14)


def test_identical_segments_give_equal_rows(oracle_mod):
    rng = np.random.default_rng(12)
    N, S = 5, 7
    seg = rng.normal(size=(N, S)); seg[3] = seg[1]
    r = _run(oracle_mod, seg.astype(np.float32).ravel(), S, 1, np.zeros((1, N)),
             np.zeros((1, N)), [0])
    np.testing.assert_array_equal(r["a_s"][1], r["a_s"][3])
    np.testing.assert_array_equal(r["a_t"][1], r["a_t"][3])
    np.testing.assert_array_equal(r["p_s"][1], r["p_s"][3])


# ---------------------------------------------------------------- limits -> plain linear map
def test_zero_temperature_limit_is_plain_linear_head(oracle_mod):
    """tau -> 0: each row's diagonal (the unique max, T4) takes all the weight, A = I,
    P = X, and the forward reduces to y = (ws + wt) X + b -- a plain matmul over the
    segment axis.  Pins the aggregation and the head's (m, n) orientation (A16)."""
    rng = np.random.default_rng(13)
    N, S, H = 6, 10, 25
    M = 3
    x = rng.normal(size=N * S + 4).astype(np.float32)
    ws, wt, b = _rand_params(rng, M, N, H)
    r = _run(oracle_mod, x, S, H, ws, wt, b, 1e-6, 1e-6)
    np.testing.assert_array_equal(r["a_s"], np.eye(N))
    np.testing.assert_array_equal(r["a_t"], np.eye(N))
    X = x[4:].astype(np.float64).reshape(N, S)
    Y = ws.astype(np.float64) @ X + wt.astype(np.float64) @ X
    np.testing.assert_allclose(r["y"], Y.ravel()[:H] + b, atol=1e-13)
    # one-hot head: future segment m copies segment n
    e = np.zeros((M, N), np.float32); e[0, 4] = 1; e[1, 0] = 1; e[2, 5] = 1
    r = _run(oracle_mod, x, S, H, e, np.zeros((M, N)), np.zeros(H), 1e-6, 1e-6)
    np.testing.assert_array_equal(r["y"], np.concatenate([X[4], X[0], X[5]])[:H])


def test_infinite_temperature_limit_is_mean_segment(oracle_mod):
    """tau -> inf: uniform rows, every pattern is the mean segment."""
    rng = np.random.default_rng(14)
    N, S, H = 5, 8, 8
    x = rng.normal(size=N * S).astype(np.float32)
    ws, wt, b = _rand_params(rng, 1, N, H)
    r = _run(oracle_mod, x, S, H, ws, wt, b, 1e15, 1e15)
    X = x.astype(np.float64).reshape(N, S)
    np.testing.assert_allclose(r["p_s"], np.broadcast_to(X.mean(0), (N, S)), atol=1e-13)
    Y = (ws.astype(np.float64).sum() + wt.astype(np.float64).sum()) * X.mean(0)
    np.testing.assert_allclose(r["y"], Y + b, atol=1e-12)


# ---------------------------------------------------------------- T12 head linearity
def test_head_linearity(oracle_mod):
    rng = np.random.default_rng(15)
    N, S, H = 4, 6, 11
    M = 2
    x = rng.normal(size=N * S).astype(np.float32)
    w1 = _rand_params(rng, M, N, H)
    w2 = _rand_params(rng, M, N, H)
    z = np.zeros((M, N), np.float32)
    r0 = _run(oracle_mod, x, S, H, z, z, w1[2])
    np.testing.assert_array_equal(r0["y"], w1[2].astype(np.float64))
    ra = _run(oracle_mod, x, S, H, *w1)
    rb = _run(oracle_mod, x, S, H, *w2)
    # 0.5 and 0.25 scale fp32 parameters exactly
    rc = _run(oracle_mod, x, S, H, 0.5 * w1[0] + 0.25 * w2[0], 0.5 * w1[1] + 0.25 * w2[1],
              0.5 * w1[2] + 0.25 * w2[2])
    np.testing.assert_allclose(rc["y"], 0.5 * ra["y"] + 0.25 * rb["y"], atol=1e-14)


# ---------------------------------------------------------------- batch layout
def test_forward_batch_layout_and_head_modes(oracle_mod):
    """oracle_forward maps x[b][c] with channel c's head (or the shared head) to y[b][c]."""
    rng = np.random.default_rng(16)
    B, C, L, S, H = 3, 4, 50, 8, 13
    N, _, M = oracle_mod.dims(L, S, H)
    x = rng.normal(size=(B, C, L)).astype(np.float32)
    ws = rng.normal(size=(C, M, N)).astype(np.float32)
    wt = rng.normal(size=(C, M, N)).astype(np.float32)
    b = rng.normal(size=(C, H)).astype(np.float32)
    y, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True, 0.7, 1.3)
    for bi in range(B):
        for c in range(C):
            r = _run(oracle_mod, x[bi, c], S, H, ws[c], wt[c], b[c], 0.7, 1.3)
            np.testing.assert_array_equal(y64[bi, c], r["y"])
    np.testing.assert_array_equal(y, y64.astype(np.float32))
    ys, _ = oracle_mod.forward(x, S, H, ws[:1], wt[:1], b[:1], False, 0.7, 1.3)
    r = _run(oracle_mod, x[2, 3], S, H, ws[0], wt[0], b[0], 0.7, 1.3)
    np.testing.assert_array_equal(ys[2, 3], r["y"].astype(np.float32))


def test_error_sums(oracle_mod):
    rng = np.random.default_rng(17)
    y = rng.normal(size=1000).astype(np.float32)
    t = rng.normal(size=1000).astype(np.float32)
    sse, sae, n = oracle_mod.error_sums(y, t)
    d = y.astype(np.float64) - t
    assert n == 1000 and abs(sse - (d * d).sum()) < 1e-9 and abs(sae - np.abs(d).sum()) < 1e-9


# ---------------------------------------------------------------- T13 high-precision brute force
def test_mpmath_bruteforce_small(oracle_mod):
    """50-digit evaluation of Definition steps 2-11 with explicit loops on 2-4
    segments; the fp64 oracle agrees to ~1e-13 (catches precision loss)."""
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 50
    rng = np.random.default_rng(18)
    for N in (2, 3, 4):
        S, H = 5, 6
        M = 2
        x = rng.normal(size=N * S).astype(np.float32)
        ws, wt, b = _rand_params(rng, M, N, H)
        X = [[mp.mpf(float(x[n * S + t])) for t in range(S)] for n in range(N)]
        mu = [sum(X[n]) / S for n in range(N)]
        z = [[X[n][t] - mu[n] for t in range(S)] for n in range(N)]
        tt = [mp.mpf(t) - mp.mpf(S - 1) / 2 for t in range(S)]
        V = sum(v * v for v in tt)
        nu2 = [sum(v * v for v in z[n]) for n in range(N)]
        kap = [sum(tt[t] * z[n][t] for t in range(S)) / V for n in range(N)]
        allp = [v for row in X for v in row]
        mean = sum(allp) / len(allp)
        var = sum((v - mean) ** 2 for v in allp) / len(allp)
        rho = [[sum(z[i][t] * z[j][t] for t in range(S)) /
                mp.sqrt((nu2[i] + mp.mpf("1e-12")) * (nu2[j] + mp.mpf("1e-12")))
                for j in range(N)] for i in range(N)]
        lines = [[mu[n] + kap[n] * tt[t] for t in range(S)] for n in range(N)]
        Dh = [[sum((lines[i][t] - lines[j][t]) ** 2 for t in range(S)) / S / (var + mp.mpf("1e-5"))
               for j in range(N)] for i in range(N)]
        def smax(row):
            e = [mp.e ** v for v in row]
            s = sum(e)
            return [v / s for v in e]
        As = [smax(rho[i]) for i in range(N)]
        At = [smax([-v for v in Dh[i]]) for i in range(N)]
        Ps = [[sum(As[i][j] * X[j][t] for j in range(N)) for t in range(S)] for i in range(N)]
        Pt = [[sum(At[i][j] * X[j][t] for j in range(N)) for t in range(S)] for i in range(N)]
        y = []
        for h in range(H):
            m, t = divmod(h, S)
            y.append(sum(mp.mpf(float(ws[m, n])) * Ps[n][t] + mp.mpf(float(wt[m, n])) * Pt[n][t]
                         for n in range(N)) + mp.mpf(float(b[h])))
        r = _run(oracle_mod, x, S, H, ws, wt, b)
        np.testing.assert_allclose(r["y"], [float(v) for v in y], atol=1e-13)
        np.testing.assert_allclose(r["a_t"], [[float(v) for v in row] for row in At], atol=1e-14)

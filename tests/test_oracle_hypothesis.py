"""SURVEY §4.2 T-brute: hypothesis-generated small inputs (2-4 segments, S in [2, 8], random
r, H and temperatures) evaluated by a 50-digit mpmath transcription of Definition steps
1-11 with explicit loops (no numpy, no oracle code), against the fp64 oracle."""
import numpy as np
import pytest

mp = pytest.importorskip("mpmath")
hyp = pytest.importorskip("hypothesis")
from hypothesis import given, settings, strategies as st  # noqa: E402


def _mp_forward(x, S, H, ws, wt, b, tau_s, tau_t):
    mp.mp.dps = 50
    L = len(x)
    N = L // S
    r = L - N * S
    M = -(-H // S)
    X = [[mp.mpf(float(x[r + n * S + t])) for t in range(S)] for n in range(N)]
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
    As = [smax([v / mp.mpf(tau_s) for v in rho[i]]) for i in range(N)]
    At = [smax([-v / mp.mpf(tau_t) for v in Dh[i]]) for i in range(N)]
    Ps = [[sum(As[i][j] * X[j][t] for j in range(N)) for t in range(S)] for i in range(N)]
    Pt = [[sum(At[i][j] * X[j][t] for j in range(N)) for t in range(S)] for i in range(N)]
    y = []
    for h in range(H):
        m, t = divmod(h, S)
        y.append(sum(mp.mpf(float(ws[m, n])) * Ps[n][t] + mp.mpf(float(wt[m, n])) * Pt[n][t]
                     for n in range(N)) + mp.mpf(float(b[h])))
    assert M == ws.shape[0]
    return [float(v) for v in y]


@settings(max_examples=40, deadline=None)
@given(N=st.integers(2, 4), S=st.integers(2, 8), data=st.data(),
       tau_s=st.sampled_from([0.05, 0.3, 1.0, 7.0]), tau_t=st.sampled_from([0.1, 1.0, 3.0]))
def test_oracle_matches_mpmath_bruteforce(oracle_mod, N, S, data, tau_s, tau_t):
    r = data.draw(st.integers(0, S - 1))
    H = data.draw(st.integers(1, 2 * S))
    seed = data.draw(st.integers(0, 2 ** 31 - 1))
    rng = np.random.default_rng(seed)
    L = N * S + r
    x = (rng.normal(size=L) * 10.0 ** rng.uniform(-2, 2)).astype(np.float32)
    M = -(-H // S)
    ws = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    wt = rng.uniform(-1, 1, (M, N)).astype(np.float32)
    b = rng.uniform(-1, 1, H).astype(np.float32)
    ref = _mp_forward(x, S, H, ws, wt, b, tau_s, tau_t)
    got = oracle_mod.series(x, S, H, ws, wt, b, tau_s, tau_t)["y"]
    scale = 1.0 + max(abs(v) for v in ref)
    np.testing.assert_allclose(got, ref, atol=1e-11 * scale, rtol=0)

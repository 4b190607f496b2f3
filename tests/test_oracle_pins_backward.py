"""Pins of the oracle's head backward (DESIGN.md §3 reading R-f6).

y is linear in (W_s, W_t, b), so central differences of L = sum(dy * y) (the oracle's own
fp64 FORWARD, a separate code path from oracle_backward_head_ex) give the gradient up to
rounding; the bias gradient has a closed form; a shared head's gradient is the sum of the
per-channel gradients.
"""
import math

import numpy as np
import pytest


def _setup(rng, B, C, L, S, H, hpc=True):
    N, M = L // S, -(-H // S)
    Cw = C if hpc else 1
    s = 1 / math.sqrt(N)
    q = lambda a: (np.round(a * 1024) / 1024).astype(np.float32)   # w +- 1/4 exact in fp32
    ws = q(rng.uniform(-s, s, (Cw, M, N)))
    wt = q(rng.uniform(-s, s, (Cw, M, N)))
    b = q(rng.uniform(-s, s, (Cw, H)))
    x = rng.normal(size=(B, C, L)).astype(np.float32)
    dy = rng.normal(size=(B, C, H)).astype(np.float32)
    return x, ws, wt, b, dy


def _loss(o, x, S, H, ws, wt, b, dy, hpc, **kw):
    _, y64 = o.forward(x, S, H, ws, wt, b, hpc, **kw)
    return float((y64 * dy.astype(np.float64)).sum())


@pytest.mark.parametrize("kw", [{}, {"metric_variant": 3}, {"instance_norm": True},
                                {"metric_variant": 7, "instance_norm": True, "ma_kernel": 5}])
def test_head_gradient_matches_central_differences(oracle_mod, kw):
    rng = np.random.default_rng(60)
    B, C, L, S, H = 3, 2, 60, 12, 30
    x, ws, wt, b, dy = _setup(rng, B, C, L, S, H)
    dws, dwt, db = oracle_mod.backward_head(x, S, H, ws, wt, b, dy, True, **kw)
    h = 0.25   # the perturbed weights stay exact in fp32; L is linear in the head
    for (arr, grad) in ((ws, dws), (wt, dwt), (b, db)):
        for idx in [(0, 0, 0), (1, 2, 4), (1, 1, 3)] if arr.ndim == 3 else [(0, 0), (1, 29), (0, 17)]:
            p, m = arr.copy(), arr.copy()
            p[idx] += h
            m[idx] -= h
            args = {id(ws): 0, id(wt): 1, id(b): 2}[id(arr)]
            ap = [ws, wt, b]
            ap[args] = p
            lp = _loss(oracle_mod, x, S, H, *ap, dy, True, **kw)
            ap[args] = m
            lm = _loss(oracle_mod, x, S, H, *ap, dy, True, **kw)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grad[idx]) <= 1e-9 * max(1.0, abs(fd)), (idx, fd, grad[idx])


def test_bias_gradient_closed_form(oracle_mod):
    rng = np.random.default_rng(61)
    x, ws, wt, b, dy = _setup(rng, 4, 3, 48, 8, 20)
    _, _, db = oracle_mod.backward_head(x, 8, 20, ws, wt, b, dy, True)
    np.testing.assert_allclose(db, dy.astype(np.float64).sum(axis=0), atol=1e-12)
    # with RevIN: db = sum_b dy * sqrt(var_r + eps) (np.var of the segmented points)
    _, _, dbr = oracle_mod.backward_head(x, 8, 20, ws, wt, b, dy, True, instance_norm=True)
    sr = np.sqrt(x.astype(np.float64).var(axis=2) + 1e-5)          # L = N S here (r = 0)
    np.testing.assert_allclose(dbr, (dy * sr[..., None]).sum(axis=0), atol=1e-12)


def test_shared_head_gradient_is_the_channel_sum(oracle_mod):
    rng = np.random.default_rng(62)
    B, C, L, S, H = 2, 3, 72, 12, 24
    x, ws, wt, b, dy = _setup(rng, B, C, L, S, H, hpc=False)
    g_shared = oracle_mod.backward_head(x, S, H, ws, wt, b, dy, False)
    rep = lambda a: np.repeat(a, C, axis=0)
    g_per = oracle_mod.backward_head(x, S, H, rep(ws), rep(wt), rep(b), dy, True)
    for a, c in zip(g_shared, g_per):
        np.testing.assert_allclose(a[0], c.sum(axis=0), atol=1e-12)


def test_zero_upstream_gradient(oracle_mod):
    rng = np.random.default_rng(63)
    x, ws, wt, b, dy = _setup(rng, 2, 2, 48, 12, 12)
    for g in oracle_mod.backward_head(x, 12, 12, ws, wt, b, np.zeros_like(dy), True):
        assert not g.any()

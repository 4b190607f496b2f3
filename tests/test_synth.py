"""The shared input generator: seeded, sharding-independent, LTSF window convention."""
import numpy as np

import synth


def test_window_counts_match_ltsf_convention():
    W = synth.WORKLOADS
    assert W["etth1"].windows == 32
    assert [W[f"weather_h{h}"].windows for h in (96, 192, 336, 720)] == [10444, 10348, 10204, 9820]
    assert W["electricity"].windows == 4925
    assert W["traffic"].windows == 2789
    for L, S in synth.STRESS_GRID:
        w = W[f"stress_L{L}_S{S}_H96"]
        assert w.windows == 1000 and w.C == 100 and w.t0 >= w.num_train - w.L


def test_channels_are_independent_of_sharding():
    w = synth.WORKLOADS["weather_h96"]
    full = synth.make_series(w, channels=range(6))
    part = synth.make_series(w, channels=[3, 5])
    np.testing.assert_array_equal(full[[3, 5]], part)
    np.testing.assert_array_equal(synth.make_series(w, channels=range(6)), full)
    assert not np.array_equal(synth.make_series(w, seed=1, channels=range(6)), full)


def test_standardised_with_train_stats():
    w = synth.WORKLOADS["traffic"]
    s = synth.make_series(w, channels=range(4)).astype(np.float64)
    tr = s[:, : w.num_train]
    np.testing.assert_allclose(tr.mean(1), 0, atol=1e-5)
    np.testing.assert_allclose(tr.std(1), 1, atol=1e-4)


def test_window_batch_indexing():
    w = synth.WORKLOADS["etth1"]
    s = synth.make_series(w)
    x, t = synth.window_batch(s, w, [0, 5])
    np.testing.assert_array_equal(x[1, 2], s[2, w.t0 + 5: w.t0 + 5 + w.L])
    np.testing.assert_array_equal(t[1, 2], s[2, w.t0 + 5 + w.L: w.t0 + 5 + w.L + w.H])
    # the last full-test-set window's target ends at the series end
    wt = synth.WORKLOADS["traffic"]
    assert wt.t0 + (wt.windows - 1) + wt.L + wt.H == wt.T


def test_params_bounds_and_shapes():
    ws, wt, b = synth.make_params(5, 30, 30, 720)
    assert ws.shape == (5, 30, 30) and b.shape == (5, 720)
    assert np.abs(ws).max() <= 1 / np.sqrt(30) and np.abs(b).max() <= 1 / np.sqrt(30)
    ws1, _, _ = synth.make_params(1, 30, 30, 720, head_per_channel=False)
    assert ws1.shape == (1, 30, 30)

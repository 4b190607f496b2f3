"""GPU parity of the full backward (prnet_backward, reading R-f7) against the
fp64 oracle (oracle_backward, pinned by central differences in test_oracle_pins_backward_full),
through the C ABI.  Tolerance reading R-tol-bwd-full: the kernel recomputes the
forward and runs every adjoint in FP32, so each gradient is held to
    |d| <= 1e-4 |ref| + 5e-5 max|ref over the series (dx) or over the array (head)|
and the temperature gradients (sums over every series of terms that cancel) to
    |d| <= 1e-3 |ref| + 1e-5 sum|per-series contributions| (bounded here by sqrt(#series) max).
"""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _close(got, ref, axis_max):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max(axis=axis_max, keepdims=True) if axis_max is not None else np.abs(ref).max()
    bad = np.abs(got - ref) > 1e-4 * np.abs(ref) + 5e-5 * scale
    assert not bad.any(), (f"{int(bad.sum())} of {bad.size} off; max|d| "
                           f"{np.abs(got - ref).max():.3e} scale {np.max(scale):.3e}")


def _run(oracle_mod, B, C, L, S, H, tau_s=1.0, tau_t=1.0, hpc=True, mv=0, kind="mixed", seed=5):
    N, _, M = synth.derived_dims(L, S, H)
    x = synth.random_windows(B, C, L, seed=seed, kind=kind)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    rng = np.random.default_rng(seed)
    dy = rng.normal(size=(B, C, H)).astype(np.float32)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t,
              metric_variant=mv).load(ws, wt, b)
    g = m.backward(torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda())
    ref = oracle_mod.backward(x, S, H, ws, wt, b, dy, hpc, tau_s, tau_t, metric_variant=mv)
    _close(g["dx"].cpu().numpy(), ref["dx"], axis_max=-1)
    for k in ("dws", "dwt", "db"):
        _close(g[k].cpu().numpy(), ref[k], axis_max=None)
    dt = g["dtau"].cpu().numpy().astype(np.float64)
    rt = ref["dtau"]
    tol = 1e-3 * np.abs(rt) + 1e-5 * np.sqrt(B * C) * max(1.0, np.abs(ref["dx"]).max())
    assert np.all(np.abs(dt - rt) <= tol), (dt, rt, tol)
    return g, ref


@pytest.mark.parametrize("L,S,H", [(96, 24, 96), (720, 24, 720), (720, 24, 336), (100, 12, 50),
                                   (53, 12, 24), (64, 8, 64), (97, 7, 13), (30, 2, 5),
                                   (384, 12, 384), (720, 48, 96), (1440, 96, 96), (25, 24, 1)])
def test_backward_shapes(oracle_mod, L, S, H):
    _run(oracle_mod, 5, 3, L, S, H)


@pytest.mark.parametrize("tau_s,tau_t", [(0.05, 0.035), (0.3, 2.0), (4.0, 0.5), (0.003, 1.0)])
@pytest.mark.parametrize("hpc", [True, False])
def test_backward_temperatures(oracle_mod, tau_s, tau_t, hpc):
    _run(oracle_mod, 4, 3, 720, 24, 192, tau_s, tau_t, hpc)


@pytest.mark.parametrize("kind", ["normal", "constant"])
def test_backward_value_kinds(oracle_mod, kind):
    _run(oracle_mod, 4, 3, 240, 24, 96, kind=kind)


def test_backward_level_only_trend(oracle_mod):
    _run(oracle_mod, 4, 3, 360, 12, 96, mv=1)


def test_backward_many_windows(oracle_mod):
    """Several series per warp and several CTAs per channel (partials, fixed-order reduce)."""
    _run(oracle_mod, 150, 2, 96, 24, 96)


def test_backward_deterministic_and_batch_zero():
    N, M = 30, 30
    ws, wt, b = synth.make_params(4, M, N, 720, True, synth.DEFAULT_SEED, 0)
    m = PRNet(4, 720, 24, 720).load(ws, wt, b)
    x = torch.from_numpy(synth.random_windows(37, 4, 720)).cuda()
    dy = torch.randn(37, 4, 720, device="cuda")
    g1 = m.backward(x, dy)
    g2 = m.backward(x, dy)
    for k in g1:
        assert torch.equal(g1[k], g2[k]), k
    g0 = m.backward(x[:0], dy[:0])
    assert float(g0["dws"].abs().max()) == 0.0 and float(g0["dtau"].abs().max()) == 0.0


def test_backward_rejects_widening():
    N, M = 30, 4
    ws, wt, b = synth.make_params(2, M, N, 96, True, synth.DEFAULT_SEED, 0)
    m = PRNet(2, 720, 24, 96, instance_norm=True).load(ws, wt, b)
    x = torch.zeros(3, 2, 720, device="cuda")
    with pytest.raises(PrnetError):
        m.backward(x, torch.zeros(3, 2, 96, device="cuda"))

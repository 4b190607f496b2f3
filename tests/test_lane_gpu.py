"""GPU parity of lane_f32 (fwd_lane.cu: N <= 8, S % 4 == 0, N S <= 192, H % 4 == 0, one lane per
series, FP32, searched seasonal row maximum) against the fp64 oracle through the C ABI.
Tolerance |d| <= 1e-5 + 1e-4 |ref| (north_star).  Shapes: every N 1..8 (its own instantiation),
S from 4 to 96, r > 0, H a multiple of 4 that does not tile M S (a partial last head row), M up
to 60 (the head-row loop), rounds cut by the window count (idle lanes), several channels per
warp sweep, shared and per-channel heads, the value kinds and temperatures of the other kernels'
tests down to tau_s = 1e-3 (below every known-maximum kernel's floor)."""
import numpy as np
import pytest

import synth
from parity_util import assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _run(oracle_mod, B, C, L, S, H, kind="mixed", tau_s=1.0, tau_t=1.0, hpc=True, seed=23):
    N, _, M = synth.derived_dims(L, S, H)
    x = synth.random_windows(B, C, L, seed=seed, kind=kind)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t).load(ws, wt, b)
    m.set_variant("lane_f32")
    y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t)
    scale = None
    if kind == "scaled":
        scale = np.maximum(np.abs(x).max(axis=-1, keepdims=True), 1.0)
    return assert_parity(y, y64, scale=scale)


@pytest.mark.parametrize("S", [4, 8, 12, 16, 24])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8])
def test_lane_shapes(oracle_mod, S, N):
    _run(oracle_mod, 37, 3, N * S, S, 2 * S + 4)


@pytest.mark.parametrize("L,S,H", [(96, 12, 96), (96, 24, 96), (96, 48, 96), (96, 96, 96),
                                   (192, 24, 720), (192, 48, 96), (192, 96, 720), (100, 12, 8),
                                   (104, 24, 720), (96, 12, 4), (96, 12, 100), (168, 24, 336),
                                   (144, 48, 200)])
def test_lane_horizons_ragged(oracle_mod, L, S, H):
    _run(oracle_mod, 33, 4, L, S, H)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
def test_lane_value_kinds(oracle_mod, kind):
    _run(oracle_mod, 40, 3, 96, 12, 96, kind=kind)


@pytest.mark.parametrize("tau", [0.001, 0.005, 0.05, 0.3, 4.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_lane_temperatures(oracle_mod, tau, hpc):
    _run(oracle_mod, 35, 3, 96, 24, 96, tau_s=tau, tau_t=max(tau, 0.01) * 0.7, hpc=hpc)


@pytest.mark.parametrize("B", [1, 31, 32, 33, 300])
def test_lane_window_counts(oracle_mod, B):
    _run(oracle_mod, B, 2, 96, 12, 96)


def test_lane_many_channels(oracle_mod):
    # more rounds than resident warps: every warp sweeps several (channel, round) items
    _run(oracle_mod, 70, 97, 96, 24, 96)


def test_lane_matches_group_f32():
    # the same FP32 arithmetic family: lane_f32 and group_f32 agree far inside the tolerance
    L, S, H, C, B = 96, 12, 96, 5, 64
    x = torch.from_numpy(synth.random_windows(B, C, L, kind="mixed")).cuda()
    ws, wt, b = synth.make_params(C, 8, 8, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H).load(ws, wt, b)
    m.set_variant("lane_f32")
    y1 = m.forward(x)
    m.set_variant("group_f32")
    y2 = m.forward(x)
    assert torch.allclose(y1, y2, rtol=2e-5, atol=2e-6)


@pytest.mark.parametrize("t0", [0, 1, 3])
def test_lane_sliding_unaligned(oracle_mod, t0):
    # sliding windows start at any float: element-wise cp.async staging instead of bulk copies,
    # bitwise the materialised windows' result (the same arithmetic on the same staged rows)
    L, S, H, C, B = 96, 12, 96, 3, 45
    T = L + B + 6
    s = synth.random_windows(1, C, T, kind="mixed")[0]
    ws, wt, b = synth.make_params(C, 8, 8, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H).load(ws, wt, b)
    m.set_variant("lane_f32")
    y = m.forward_sliding(torch.from_numpy(s).cuda(), t0, B)
    xw = np.stack([s[:, t0 + k:t0 + k + L] for k in range(B)])
    assert torch.equal(y, m.forward(torch.from_numpy(xw).cuda()))
    _, y64 = oracle_mod.forward(xw, S, H, ws, wt, b, True, 1.0, 1.0)
    assert_parity(y.cpu().numpy(), y64)


def test_lane_unaligned_offset(oracle_mod):
    # r = L - N S = 2: window rows are not 16-byte aligned (element-wise staging)
    _run(oracle_mod, 40, 3, 98, 12, 96)


@pytest.mark.parametrize("L,S,H", [(108, 12, 96), (96, 6, 96), (96, 12, 98), (240, 24, 96)])
def test_lane_rejects_out_of_domain(L, S, H):
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(2, M, N, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(2, L, S, H).load(ws, wt, b)
    with pytest.raises(PrnetError):
        m.set_variant("lane_f32")

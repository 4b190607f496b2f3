"""GPU parity of group_f32 (fwd_grp.cu: N <= 16, S <= 32, lanes over (series, segment), FP32)
against the fp64 oracle through the C ABI.  Tolerance |d| <= 1e-5 + 1e-4 |ref| (north_star).
Shapes: every NP (2, 4, 8, 16) and float4 chunk count, S not a multiple of 4 (scalar loads and
stores), r > 0, H not a multiple of S, M up to 64 (several head rows per lane), groups cut by
the window count, the value kinds and temperatures of the other kernels' tests."""
import numpy as np
import pytest

import synth
from parity_util import assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet  # noqa: E402


def _run(oracle_mod, B, C, L, S, H, kind="mixed", tau_s=1.0, tau_t=1.0, hpc=True, seed=17):
    N, _, M = synth.derived_dims(L, S, H)
    x = synth.random_windows(B, C, L, seed=seed, kind=kind)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t).load(ws, wt, b)
    m.set_variant("group_f32")
    y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t)
    scale = None
    if kind == "scaled":
        scale = np.maximum(np.abs(x).max(axis=-1, keepdims=True), 1.0)
    return assert_parity(y, y64, scale=scale)


@pytest.mark.parametrize("S", [2, 3, 5, 8, 12, 16, 24, 30, 32])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 7, 8, 9, 16])
def test_grp_shapes(oracle_mod, S, N):
    _run(oracle_mod, 11, 3, N * S, S, 2 * S + 1)


@pytest.mark.parametrize("L,S,H", [(96, 12, 96), (96, 24, 96), (192, 24, 720), (100, 12, 7),
                                   (99, 12, 720), (50, 12, 1), (96, 12, 768), (336, 24, 50)])
def test_grp_horizons_ragged(oracle_mod, L, S, H):
    _run(oracle_mod, 9, 4, L, S, H)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
def test_grp_value_kinds(oracle_mod, kind):
    _run(oracle_mod, 10, 3, 96, 12, 96, kind=kind)


@pytest.mark.parametrize("tau", [0.05, 0.3, 4.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_grp_temperatures(oracle_mod, tau, hpc):
    _run(oracle_mod, 10, 3, 96, 24, 96, tau_s=tau, tau_t=tau * 0.7, hpc=hpc)


@pytest.mark.parametrize("B", [1, 3, 17, 300])
def test_grp_window_counts(oracle_mod, B):
    _run(oracle_mod, B, 2, 96, 12, 96)


def test_grp_sliding_equals_materialised():
    L, S, H, C, B = 96, 12, 96, 3, 13
    T = L + B + 6
    s = synth.random_windows(1, C, T, kind="mixed")[0]
    ws, wt, b = synth.make_params(C, 8, 8, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H).load(ws, wt, b)
    m.set_variant("group_f32")
    sd = torch.from_numpy(s).cuda()
    xw = sd.unfold(1, L, 1)[:, 3:3 + B, :].permute(1, 0, 2).contiguous()
    assert torch.equal(m.forward_sliding(sd, 3, B), m.forward(xw))

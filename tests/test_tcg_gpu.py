"""GPU parity of tc_quad's generic-S instantiations (fwd_tcg.cu: S in {12, 16, 32, 48, 64, 96},
N <= 32, M <= 32) against the fp64 oracle, through the C ABI.  Tolerance |d| <= 1e-5 + 1e-4 |ref|
(north_star).  Shapes span every instantiation, N = 1..32 (padding lanes), r > 0 (aligned and
unaligned window starts: bulk copies vs the 4-byte cp.async path), H not a multiple of S, odd H
(scalar stores), one or two head m-tiles, quads cut by the window count, and the attention
dump of the kernel's own softmax registers."""
import numpy as np
import pytest

import synth
from parity_util import assert_parity

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet  # noqa: E402

S_VALUES = (12, 16, 32, 48, 64, 96)


def _run(oracle_mod, B, C, L, S, H, kind="mixed", tau_s=1.0, tau_t=1.0, hpc=True, seed=11):
    N, _, M = synth.derived_dims(L, S, H)
    assert N <= 32 and M <= 64
    x = synth.random_windows(B, C, L, seed=seed, kind=kind)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t).load(ws, wt, b)
    m.set_variant("tc_quad")
    y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t)
    scale = None
    if kind == "scaled":
        scale = np.maximum(np.abs(x).max(axis=-1, keepdims=True), 1.0)
    return assert_parity(y, y64, scale=scale)


@pytest.mark.parametrize("S", S_VALUES)
@pytest.mark.parametrize("N", [1, 2, 7, 16, 17, 30, 32])
def test_tcg_segments(oracle_mod, S, N):
    L = N * S
    _run(oracle_mod, 9, 5, L, S, 96)


@pytest.mark.parametrize("S", S_VALUES)
@pytest.mark.parametrize("L,H", [(None, 1), (None, 7), (None, 97), (None, 200), (None, 720),
                                 (None, 385), (None, 768)])
def test_tcg_horizons(oracle_mod, S, L, H):
    """H up to 64 S: M > 32 runs the head in two passes of 32 future segments."""
    N = min(32, max(1, 700 // S))
    M = -(-H // S)
    if M > 64:
        pytest.skip("M > 64")
    _run(oracle_mod, 6, 3, N * S + 5, S, H)


@pytest.mark.parametrize("S", S_VALUES)
@pytest.mark.parametrize("r", [1, 2, 3, 4, 8])
def test_tcg_ragged_start(oracle_mod, S, r):
    """L = N S + r: r % 4 != 0 takes the cp.async path (window starts not 16-byte aligned)."""
    N = min(32, 400 // S + 1)
    _run(oracle_mod, 5, 4, N * S + r, S, 100)


@pytest.mark.parametrize("S", S_VALUES)
@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
def test_tcg_value_kinds(oracle_mod, S, kind):
    N = min(30, 720 // S)
    _run(oracle_mod, 5, 3, N * S, S, 96, kind=kind)


@pytest.mark.parametrize("S", [12, 48, 96])
@pytest.mark.parametrize("tau", [0.05, 0.3, 4.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_tcg_temperatures(oracle_mod, S, tau, hpc):
    N = min(30, 1440 // S)
    _run(oracle_mod, 7, 3, N * S, S, 2 * S + 3, tau_s=tau, tau_t=tau * 0.7, hpc=hpc)


@pytest.mark.parametrize("S", S_VALUES)
@pytest.mark.parametrize("B", [1, 3, 5, 130, 517])
def test_tcg_window_counts(oracle_mod, S, B):
    """Quads cut by the window count, and several rounds per group."""
    N = min(20, 600 // S)
    _run(oracle_mod, B, 2, N * S, S, 50)


@pytest.mark.parametrize("S", S_VALUES)
def test_tcg_attention_dump(oracle_mod, S):
    """prnet_debug_attention on a tc_quad handle dumps the generic kernel's own softmax."""
    N = min(30, 1000 // S)
    L = N * S + 3
    x = synth.random_windows(3, 2, L, kind="mixed")
    ws, wt, b = synth.make_params(2, -(-24 // S), N, 24, True, synth.DEFAULT_SEED, 0)
    m = PRNet(2, L, S, 24, tau_s=0.5, tau_t=2.0).load(ws, wt, b)
    m.set_variant("tc_quad")
    a_s, a_t = m.debug_attention(torch.from_numpy(x).cuda())
    a_s, a_t = a_s.cpu().numpy(), a_t.cpu().numpy()
    for bb in range(3):
        for c in range(2):
            Md = -(-24 // S)
            r = oracle_mod.series(x[bb, c], S, 24, np.zeros((Md, N)), np.zeros((Md, N)),
                                  np.zeros(24), 0.5, 2.0)
            np.testing.assert_allclose(a_s[bb, c], r["a_s"], atol=2e-6)
            np.testing.assert_allclose(a_t[bb, c], r["a_t"], atol=2e-6)


@pytest.mark.parametrize("S", [12, 48, 96])
def test_tcg_sliding_equals_materialised(S):
    """Sliding windows (unaligned starts, cp.async path) equal the materialised forward bitwise."""
    N = min(30, 1440 // S)
    L, H, C, B = N * S, 96, 3, 13
    T = L + B + 7
    s = synth.random_windows(1, C, T, kind="mixed")[0]
    ws, wt, b = synth.make_params(C, -(-H // S), N, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H).load(ws, wt, b)
    m.set_variant("tc_quad")
    sd = torch.from_numpy(s).cuda()
    y_sl = m.forward_sliding(sd, 2, B)
    xw = sd.unfold(1, L, 1)[:, 2:2 + B, :].permute(1, 0, 2).contiguous()
    y_mat = m.forward(xw)
    assert torch.equal(y_sl, y_mat)


def test_tcg_is_default_where_measured_fastest():
    """The plan picks tc_quad for the generic-S shapes it was measured fastest on."""
    m = PRNet(4, 1440, 48, 96)
    assert m.plan(10)["variant"] == "tc_quad"

"""Seeded random configurations across every flag, GPU (auto-picked kernel) against the fp64
oracle, and the head backward against oracle.backward_head.  Shapes the library does not
implement must fail with PRNET_ERR_UNSUPPORTED (status 3), never silently."""
import numpy as np
import pytest

import synth
from parity_util import assert_parity, assert_parity_revin

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _config(k):
    g = np.random.default_rng(1000 + k)
    S = int(g.choice([2, 3, 5, 7, 8, 12, 16, 24, 24, 24, 31, 48, 64, 96, 128]))
    N = int(g.integers(1, 41 if g.random() < 0.8 else 200))
    L = N * S + int(g.integers(0, S))
    H = int(g.integers(1, min(4000, 30 * S) + 1))
    mv = int(g.integers(0, 8))
    rev = bool(g.random() < 0.4)
    ma = int(g.choice([0, 0, 0, 1, 3, 9, 25]))
    hpc = bool(g.random() < 0.7)
    tau_s = float(g.choice([0.05, 0.3, 1.0, 4.0]))
    tau_t = float(g.choice([0.1, 1.0, 2.5]))
    kind = str(g.choice(["mixed", "normal", "constant"]))
    return dict(L=L, S=S, H=H, mv=mv, rev=rev, ma=ma, hpc=hpc, tau_s=tau_s, tau_t=tau_t,
                kind=kind)


@pytest.mark.parametrize("k", range(150))
def test_fuzz_forward(oracle_mod, k):
    cf = _config(k)
    L, S, H = cf["L"], cf["S"], cf["H"]
    N, _, M = synth.derived_dims(L, S, H)
    C, B = 3, 4
    x = synth.random_windows(B, C, L, kind=cf["kind"])
    ws, wt, b = synth.make_params(C, M, N, H, cf["hpc"], synth.DEFAULT_SEED, k)
    try:
        m = PRNet(C, L, S, H, head_per_channel=cf["hpc"], tau_s=cf["tau_s"], tau_t=cf["tau_t"],
                  metric_variant=cf["mv"], instance_norm=cf["rev"], ma_kernel=cf["ma"])
        m.load(ws, wt, b)
        y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    except PrnetError as e:
        assert e.status == 3, (cf, e)
        pytest.skip(f"unsupported: {e}")
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, cf["hpc"], cf["tau_s"], cf["tau_t"],
                                metric_variant=cf["mv"], instance_norm=cf["rev"],
                                ma_kernel=cf["ma"])
    if cf["rev"]:   # reading R-tol-revin
        assert_parity_revin(y, y64, x, S)
    else:
        assert_parity(y, y64)


@pytest.mark.parametrize("k", range(40))
def test_fuzz_backward(oracle_mod, k):
    cf = _config(500 + k)
    L, S, H = cf["L"], cf["S"], cf["H"]
    N, _, M = synth.derived_dims(L, S, H)
    C, B = 3, 6
    x = synth.random_windows(B, C, L, kind=cf["kind"])
    dy = np.random.default_rng(k).normal(size=(B, C, H)).astype(np.float32)
    mv = cf["mv"] & 3
    ws, wt, b = synth.make_params(C, M, N, H, cf["hpc"], synth.DEFAULT_SEED, k)
    try:
        m = PRNet(C, L, S, H, head_per_channel=cf["hpc"], tau_s=cf["tau_s"], tau_t=cf["tau_t"],
                  metric_variant=mv, instance_norm=cf["rev"])
        got = [g.cpu().numpy() for g in m.backward_head(torch.from_numpy(x).cuda(),
                                                       torch.from_numpy(dy).cuda())]
    except PrnetError as e:
        assert e.status == 3, (cf, e)
        pytest.skip(f"unsupported: {e}")
    ref = oracle_mod.backward_head(x, S, H, ws, wt, b, dy, cf["hpc"], cf["tau_s"], cf["tau_t"],
                                   metric_variant=mv, instance_norm=cf["rev"])
    # floor: the FP32 pattern error (~1e-6 |x|) summed with random signs over the dy terms
    floor = 1e-6 * max(1.0, float(np.abs(x).max())) * float(np.sqrt((dy.astype(np.float64) ** 2).sum()))
    for g_, r in zip(got, ref):
        tol = 2e-5 * np.abs(r).max() + 1e-4 * np.abs(r) + floor
        assert (np.abs(g_ - r) <= tol).all(), (cf, np.abs(g_ - r).max(), np.abs(r).max())

"""GPU parity of the tensor-core head backward (bwd_head_mma.cu: N, M <= 32, S in {8, 16, 24,
32}, plain reading and the level-only trend) against the fp64 oracle, with the R-tol-bwd bar of
tests/test_backward_gpu.py.  Shapes: every S instantiation (k16 steps and the
k8 tail), N from 1 to 32 (padding rows and columns of the 32 x 32 tiles), r > 0, H cutting the
last head row, M = 32, shared heads, temperatures down to tau_s = 1e-3 (exact row maxima),
value kinds and window counts across CTAs.  test_backward_gpu.py covers the same entry point
for the FP32 kernel's domain (other S, the detrended metric, instance normalisation)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet  # noqa: E402
from test_backward_gpu import _check  # noqa: E402


def _grads(oracle_mod, B, C, L, S, H, hpc=True, mv=0, tau_s=1.0, tau_t=1.0, kind="mixed",
           seed=3):
    x = synth.random_windows(B, C, L, kind=kind, seed=seed)
    dy = np.random.default_rng(seed).normal(size=(B, C, H)).astype(np.float32)
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t, metric_variant=mv)
    got = [g.cpu().numpy() for g in m.backward_head(torch.from_numpy(x).cuda(),
                                                   torch.from_numpy(dy).cuda())]
    ref = oracle_mod.backward_head(x, S, H, ws, wt, b, dy, hpc, tau_s, tau_t, metric_variant=mv)
    return got, ref, x, dy


@pytest.mark.parametrize("S", [8, 16, 24, 32])
@pytest.mark.parametrize("N", [1, 2, 5, 17, 31, 32])
def test_bwd_mma_shapes(oracle_mod, S, N):
    H = min(32 * S, 3 * S + 4)
    got, ref, x, dy = _grads(oracle_mod, 7, 3, N * S, S, H)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("L,S,H", [(100, 24, 90), (250, 8, 256), (500, 16, 512), (1000, 32, 1024),
                                   (725, 24, 720), (50, 16, 7)])
def test_bwd_mma_offsets_and_horizons(oracle_mod, L, S, H):
    got, ref, x, dy = _grads(oracle_mod, 5, 2, L, S, H)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("tau", [1e-3, 0.05, 1.0, 10.0])
@pytest.mark.parametrize("hpc,mv", [(True, 0), (False, 0), (True, 1)])
def test_bwd_mma_temperatures_heads_levelonly(oracle_mod, tau, hpc, mv):
    got, ref, x, dy = _grads(oracle_mod, 6, 3, 720, 24, 336, hpc, mv, tau, tau * 0.7 + 0.01)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
def test_bwd_mma_value_kinds(oracle_mod, kind):
    got, ref, x, dy = _grads(oracle_mod, 6, 3, 384, 16, 200, kind=kind)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("B", [1, 9, 300])
def test_bwd_mma_window_counts(oracle_mod, B):
    got, ref, x, dy = _grads(oracle_mod, B, 2, 720, 24, 96)
    _check(got, ref, x, dy)

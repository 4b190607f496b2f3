"""GPU parity of the head backward (prnet_backward_head) against the fp64
oracle (oracle.backward_head, itself pinned by exact central differences in
tests/test_oracle_pins_backward.py).

The gradients are sums over B x C x S products of an FP32-recomputed pattern with dy, so
the bar is relative to the largest gradient entry of the same array: |d| <= 2e-5 max|ref| +
1e-4 |ref| (the per-term error is the forward's ~1e-6 relative; sums of random-sign terms
grow like their magnitude)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _grads(oracle_mod, B, C, L, S, H, hpc=True, mv=0, rev=False, tau_s=1.0, tau_t=1.0,
           kind="mixed", seed=0):
    x = synth.random_windows(B, C, L, kind=kind)
    dy = np.random.default_rng(seed).normal(size=(B, C, H)).astype(np.float32)
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t, metric_variant=mv,
              instance_norm=rev)
    got = [g.cpu().numpy() for g in m.backward_head(torch.from_numpy(x).cuda(),
                                                   torch.from_numpy(dy).cuda())]
    ref = oracle_mod.backward_head(x, S, H, ws, wt, b, dy, hpc, tau_s, tau_t,
                                   metric_variant=mv, instance_norm=rev)
    return got, ref, m, x, dy


def _check(got, ref, x=None, dy=None):
    # floor for exactly-zero references (e.g. a RevIN-normalised constant series): the FP32
    # pattern error (~1e-6 |x|) summed with random signs over the dy terms
    floor = 0.0
    if x is not None:
        floor = 1e-6 * max(1.0, float(np.abs(x).max())) * float(
            np.sqrt((dy.astype(np.float64) ** 2).sum()))
    for g, r in zip(got, ref):
        assert g.shape == r.shape
        tol = 2e-5 * np.abs(r).max() + 1e-4 * np.abs(r) + floor
        bad = np.abs(g - r) > tol
        assert not bad.any(), (np.abs(g - r).max(), np.abs(r).max(), int(bad.sum()))


@pytest.mark.parametrize("hpc", [True, False])
@pytest.mark.parametrize("mv,rev", [(0, False), (1, False), (2, False), (3, True), (0, True)])
@pytest.mark.parametrize("L,S,H", [(720, 24, 720), (720, 24, 336), (96, 24, 96), (97, 7, 13),
                                   (270, 9, 31), (384, 128, 200), (100, 24, 90), (64, 2, 7)])
def test_backward_head_parity(oracle_mod, L, S, H, mv, rev, hpc):
    got, ref, _, x, dy = _grads(oracle_mod, 5, 3, L, S, H, hpc, mv, rev)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("hpc", [True, False])
@pytest.mark.parametrize("mv,rev", [(0, False), (1, False), (2, False), (3, True)])
@pytest.mark.parametrize("L,S,H", [(1440, 24, 96), (1536, 12, 200), (4000, 120, 100),
                                   (3000, 150, 96), (5760, 12, 96)])
def test_backward_head_parity_long(oracle_mod, L, S, H, mv, rev, hpc):
    """N > 32 or S > 128: the row-streaming backward kernel."""
    got, ref, _, x, dy = _grads(oracle_mod, 3, 2, L, S, H, hpc, mv, rev)
    _check(got, ref, x, dy)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
@pytest.mark.parametrize("tau", [0.05, 1.0, 10.0])
def test_backward_head_distributions_and_temperatures(oracle_mod, kind, tau):
    got, ref, _, x, dy = _grads(oracle_mod, 4, 3, 720, 24, 336, True, 0, kind == "scaled", tau,
                                tau * 0.7, kind=kind)
    _check(got, ref, x, dy)


def test_backward_head_many_windows_and_determinism(oracle_mod):
    """Several CTAs per channel (partials reduced in a fixed order): bitwise repeatable."""
    got, ref, m, x, dy = _grads(oracle_mod, 700, 2, 96, 24, 96, True, 0, False)
    _check(got, ref)
    again = m.backward_head(torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda())
    for a, b in zip(got, again):
        assert np.array_equal(a, b.cpu().numpy())


def test_backward_head_edge_cases():
    m = PRNet(3, 96, 24, 96)
    dws, dwt, db = m.backward_head(torch.zeros((0, 3, 96), device="cuda"),
                                   torch.zeros((0, 3, 96), device="cuda"))
    assert not dws.any() and not dwt.any() and not db.any()
    for kw in (dict(metric_variant=4), dict(ma_kernel=5)):
        with pytest.raises(PrnetError) as e:
            PRNet(3, 96, 24, 96, **kw).backward_head(torch.zeros((1, 3, 96), device="cuda"),
                                                     torch.zeros((1, 3, 96), device="cuda"))
        assert e.value.status == 3
    with pytest.raises(PrnetError) as e:   # M = 34 > 32
        PRNet(3, 96, 24, 800).backward_head(torch.zeros((1, 3, 96), device="cuda"),
                                            torch.zeros((1, 3, 800), device="cuda"))
    assert e.value.status == 3
    with pytest.raises(PrnetError) as e:   # host pointer
        m.backward_head(torch.zeros((1, 3, 96)), torch.zeros((1, 3, 96)))
    assert e.value.status == 3


def test_backward_head_is_the_gradient_of_the_gpu_forward():
    """L(W) = sum(dy * forward(x; W)) is linear in the head: L(W + E) - L(W) = <grad, E> up to
    the forward's FP32 rounding, for a random direction E (the GPU forward and backward are
    separate kernels)."""
    rng = np.random.default_rng(7)
    C, L, S, H, B = 4, 720, 24, 336, 64
    N, _, M = synth.derived_dims(L, S, H)
    x = torch.from_numpy(synth.random_windows(B, C, L, kind="mixed")).cuda()
    dy = torch.from_numpy(rng.normal(size=(B, C, H)).astype(np.float32)).cuda()
    ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H)
    gws, gwt, gb = [g.cpu().numpy().astype(np.float64) for g in m.backward_head(x, dy)]
    E = [rng.normal(size=a.shape).astype(np.float32) for a in (ws, wt, b)]
    def loss(p):
        y = m.load(*p).forward(x)
        return float((y.double() * dy.double()).sum())
    l0 = loss((ws, wt, b))
    l1 = loss(tuple(a + e for a, e in zip((ws, wt, b), E)))
    pred = sum(float((g * e).sum()) for g, e in zip((gws, gwt, gb), E))
    assert abs((l1 - l0) - pred) <= 1e-4 * abs(pred) + 1e-2, (l1 - l0, pred)

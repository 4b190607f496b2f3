"""GPU parity of the BF16-I/O forward (prnet_forward_bf16) against the fp64
oracle run on the same bf16 inputs widened to fp32 (exact).  Tolerance reading R-tol-bf16
(DESIGN.md §6): the fp32 bar of the north_star plus the rounding of y to bf16 (round to
nearest: at most half an ulp, i.e. the bf16 unit roundoff 2^-8 |y|):
    |d| <= 1e-5 + 1e-4 |ref| + 2^-8 (|ref| + 1e-5 + 1e-4 |ref|)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _run(oracle_mod, B, C, L, H, tau_s=1.0, tau_t=1.0, hpc=True, kind="mixed", offset=0):
    S = 24
    N, _, M = synth.derived_dims(L, S, H)
    x32 = synth.random_windows(B, C, L, seed=21, kind=kind)
    xb = torch.from_numpy(x32).to(torch.bfloat16)
    xw = xb.to(torch.float32).numpy()                     # exactly the values the kernel reads
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t).load(ws, wt, b)
    xd = xb.cuda()
    if offset:   # a window start that is only 4-byte aligned (no bulk copy)
        buf = torch.empty(xd.numel() + offset, dtype=torch.bfloat16, device="cuda")
        xd2 = buf[offset:].view(B, C, L)
        xd2.copy_(xd)
        xd = xd2
    y = m.forward_bf16(xd).to(torch.float32).cpu().numpy().astype(np.float64)
    _, ref = oracle_mod.forward(xw, S, H, ws, wt, b, hpc, tau_s, tau_t)
    tol32 = 1e-5 + 1e-4 * np.abs(ref)
    tol = tol32 + 2.0 ** -8 * (np.abs(ref) + tol32)
    d = np.abs(y - ref)
    assert np.all(d <= tol), f"{int((d > tol).sum())} off, max|d| {d.max():.3e}"
    return y


@pytest.mark.parametrize("L,H", [(720, 720), (720, 96), (720, 336), (96, 96), (100, 90),
                                 (408, 61), (768, 700), (24, 24), (240, 7)])
def test_bf16_shapes(oracle_mod, L, H):
    _run(oracle_mod, 9, 4, L, H)


@pytest.mark.parametrize("tau", [0.05, 1.0, 3.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_bf16_temperatures_heads(oracle_mod, tau, hpc):
    _run(oracle_mod, 6, 3, 720, 192, tau, tau * 0.7, hpc)


@pytest.mark.parametrize("kind", ["normal", "constant"])
def test_bf16_value_kinds(oracle_mod, kind):
    _run(oracle_mod, 6, 3, 720, 96, kind=kind)


def test_bf16_unaligned_start(oracle_mod):
    _run(oracle_mod, 5, 3, 720, 96, offset=2)


def test_bf16_many_windows_and_matches_fp32_forward():
    """At the Traffic shape: every element written, and within bf16 rounding of the fp32
    forward on the same (widened) inputs."""
    L, S, H, C, B = 720, 24, 720, 16, 517
    N, M = 30, 30
    ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H).load(ws, wt, b)
    xb = torch.from_numpy(synth.random_windows(B, C, L, seed=3)).to(torch.bfloat16).cuda()
    yb = m.forward_bf16(xb).to(torch.float32)
    y32 = m.forward(xb.to(torch.float32))
    assert torch.isfinite(yb).all()
    d = (yb - y32).abs()
    assert bool((d <= 2.0 ** -8 * y32.abs() + 1e-6).all()), float(d.max())


def test_bf16_rejects_outside_domain():
    ws, wt, b = synth.make_params(2, 8, 8, 96, True, synth.DEFAULT_SEED, 0)
    m = PRNet(2, 96, 12, 96).load(ws, wt, b)
    with pytest.raises(PrnetError):
        m.forward_bf16(torch.zeros(3, 2, 96, dtype=torch.bfloat16, device="cuda"))

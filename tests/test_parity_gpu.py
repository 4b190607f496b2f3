"""GPU parity: libprnet.so (called through its C ABI) against the fp64 CPU oracle
on the same seeded inputs.  Tolerance: |d| <= 1e-5 + 1e-4 |ref| (north_star);
segment indexing bit-exact.  Run on a B200 via gpurun: pytest -m gpu."""
import numpy as np
import pytest

import synth
from parity_util import assert_parity, assert_parity_revin, parity_report

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402


def _model(C, L, S, H, hpc=True, tau_s=1.0, tau_t=1.0, seed=synth.DEFAULT_SEED, cfg_id=0,
           variant=None):
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, seed, cfg_id)
    if not _applicable(variant, L, S, H):
        pytest.skip(f"{variant} not applicable to L={L} S={S} H={H}")
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t).load(ws, wt, b)
    if variant is not None:
        m.set_variant(variant)
    return m, (ws, wt, b)


def _applicable(variant, L, S, H):
    N, _, M = synth.derived_dims(L, S, H)
    if variant == "warp_f32":
        return N <= 32
    if variant == "mma_f16x3":
        return N <= 32 and M <= 32 and S <= 128
    if variant == "tc_quad":
        return S in (12, 16, 24, 32, 48, 64, 96) and N <= 32 and M <= (32 if S == 24 else 64)
    if variant == "small_f32":
        return N <= 16 and S <= 128 and M <= 32
    if variant == "flash_f16x3":
        return 16 < N <= 512 and S <= 96 and M <= 32
    if variant == "tc_long":
        return 32 < N <= 512 and S in (12, 24, 48, 96) and M <= 64
    if variant == "group_f32":
        return N <= 16 and S <= 32
    return True


VARIANTS = [None, "warp_f32", "mma_f16x3", "long_f32", "flash_f16x3", "tc_quad", "small_f32",
            "tc_long", "group_f32"]
SHORT_VARIANTS = [None, "warp_f32", "mma_f16x3", "tc_quad", "small_f32"]


def _check_small(oracle_mod, x, S, H, hpc=True, tau_s=1.0, tau_t=1.0, scale=None, variant=None):
    B, C, L = x.shape
    if not _applicable(variant, L, S, H):
        pytest.skip(f"{variant} not applicable to L={L} S={S} H={H}")
    m, (ws, wt, b) = _model(C, L, S, H, hpc, tau_s, tau_t, variant=variant)
    xd = torch.from_numpy(x).cuda()
    y = m.forward(xd).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t)
    sc = None
    if scale is not None:
        sc = scale
    return assert_parity(y, y64, scale=sc)


# ------------------------------------------------------------------ configs[0] in full
def test_etth1_full(oracle_mod):
    w = synth.WORKLOADS["etth1"]
    s = synth.make_series(w)
    x, _ = synth.window_batch(s, w, np.arange(w.windows))
    assert x.shape == (32, 7, 96)
    _check_small(oracle_mod, x, w.S, w.H)


# ------------------------------------------------------------------ full-size configs, sampled
FULL = ["weather_h96", "weather_h192", "weather_h336", "weather_h720", "electricity", "traffic"]


@pytest.mark.parametrize("variant", [None, "warp_f32", "mma_f16x3", "tc_quad"])
@pytest.mark.parametrize("name", FULL)
def test_full_size_sampled(oracle_mod, name, variant):
    """The whole test set runs on the GPU in the bench's launch configuration; the
    oracle checks windows {0, 1, B/2, B-1} plus a stride sample, all channels."""
    w = synth.WORKLOADS[name]
    s = synth.make_series(w)
    B = w.windows
    sd = torch.from_numpy(s).cuda()
    x = sd.unfold(1, w.L, 1)[:, w.t0:w.t0 + B, :].permute(1, 0, 2).contiguous()
    m, (ws, wt, b) = _model(w.C, w.L, w.S, w.H, cfg_id=w.cfg_id, variant=variant)
    y = m.forward(x)
    torch.cuda.synchronize()
    idx = [0, 1, B // 2, B - 1]
    if w.C <= 100:
        idx = sorted(set(idx + list(range(0, B, max(1, B // 6)))))
    xs, _ = synth.window_batch(s, w, idx)
    np.testing.assert_array_equal(x[idx].cpu().numpy(), xs)
    _, y64 = oracle_mod.forward(xs, w.S, w.H, ws, wt, b, True)
    assert_parity(y[idx].cpu().numpy(), y64)
    del x, y, sd
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ configs[4] stress sweep
@pytest.mark.parametrize("L,S", synth.STRESS_GRID)
def test_stress_grid(oracle_mod, L, S):
    """Every (L, S) point of the sweep: 4 windows x 100 channels through the same kernels
    (N = L/S from 1 to 480 covers the warp kernel's 8/16/32 variants and the long-N kernel)."""
    w = synth.WORKLOADS[f"stress_L{L}_S{S}_H96"]
    N = L // S
    nwin = 4 if N <= 120 else 1
    C = 100 if N <= 120 else 8
    s = synth.make_series(w, channels=range(C))
    x, _ = synth.window_batch(s, w, np.arange(nwin) * 97)
    _check_small(oracle_mod, x, S, w.H)


@pytest.mark.parametrize("L,S", [(5760, 12), (1440, 24), (720, 96), (5760, 96)])
def test_stress_full_size_sampled(oracle_mod, L, S):
    """Full 100k-series stress batch on the GPU, sampled series checked."""
    w = synth.WORKLOADS[f"stress_L{L}_S{S}_H96"]
    s = synth.make_series(w)
    sd = torch.from_numpy(s).cuda()
    x = sd.unfold(1, w.L, 1)[:, w.t0:w.t0 + w.windows, :].permute(1, 0, 2).contiguous()
    m, (ws, wt, b) = _model(w.C, w.L, w.S, w.H, cfg_id=w.cfg_id)
    y = m.forward(x).cpu().numpy()
    idx = [0, 999] if L // S > 120 else [0, 1, 500, 999]
    chans = np.arange(0, 100, 33) if L // S > 120 else np.arange(100)
    xs = x[idx].cpu().numpy()[:, chans]
    _, y64 = oracle_mod.forward(np.ascontiguousarray(xs), S, w.H, ws[chans], wt[chans], b[chans])
    assert_parity(y[idx][:, chans], y64)


# ------------------------------------------------------------------ shapes and edge cases
@pytest.mark.parametrize("L,S,H", [
    (96, 24, 96), (100, 24, 90), (97, 7, 13), (50, 49, 3), (24, 24, 24), (25, 24, 1),
    (64, 8, 64), (72, 8, 100), (128, 8, 64), (136, 8, 9), (256, 8, 40), (264, 8, 40),
    (270, 9, 31), (33, 2, 5), (66, 2, 7), (720, 24, 720), (722, 12, 721), (1000, 3, 17),
    (720, 24, 769), (720, 96, 96), (768, 24, 96), (767, 24, 700), (384, 128, 200),
    (1440, 48, 96), (160, 5, 40), (3840, 96, 96), (2000, 72, 150), (1700, 50, 120),
    (1290, 64, 400)])
@pytest.mark.parametrize("variant", VARIANTS)
def test_shapes_ragged(oracle_mod, L, S, H, variant):
    """N from 1 to 333 across every kernel variant; L mod S != 0 (r > 0);
    H mod S != 0; odd S and L (scalar load path); M > 32 falls back."""
    x = synth.random_windows(3, 5, L, kind="mixed")
    _check_small(oracle_mod, x, S, H, variant=variant)


@pytest.mark.parametrize("variant", SHORT_VARIANTS)
@pytest.mark.parametrize("tau", [0.05, 0.1, 1.0, 10.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_temperatures_and_head_modes(oracle_mod, tau, hpc, variant):
    x = synth.random_windows(4, 6, 720, kind="mixed")
    _check_small(oracle_mod, x, 24, 336, hpc=hpc, tau_s=tau, tau_t=tau * 0.7, variant=variant)


@pytest.mark.parametrize("tau", [0.05, 1.0, 10.0])
@pytest.mark.parametrize("hpc", [True, False])
@pytest.mark.parametrize("L,S,H", [(1440, 24, 96), (1536, 12, 200), (2880, 48, 96),
                                   (5760, 96, 96), (3200, 64, 700)])
def test_long_lookback_temperatures_and_head_modes(oracle_mod, L, S, H, tau, hpc):
    """The long-N (flash) path under both head modes and several temperatures."""
    x = synth.random_windows(2, 3, L, kind="mixed")
    _check_small(oracle_mod, x, S, H, hpc=hpc, tau_s=tau, tau_t=tau * 0.7)


@pytest.mark.parametrize("variant", [None, "flash_f16x3", "long_f32", "tc_long"])
@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
def test_long_lookback_value_distributions(oracle_mod, kind, variant):
    x = synth.random_windows(2, 3, 1440, kind=kind)
    scale = np.abs(x).max(axis=2, keepdims=True)[..., :1] if kind == "scaled" else None
    scale = None if scale is None else np.maximum(scale, 1.0)
    _check_small(oracle_mod, x, 24, 96, scale=scale, variant=variant)


@pytest.mark.parametrize("variant", SHORT_VARIANTS)
@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
@pytest.mark.parametrize("L,S", [(720, 24), (1440, 24)])
def test_value_distributions(oracle_mod, kind, L, S, variant):
    x = synth.random_windows(3, 4, L, kind=kind)
    scale = np.abs(x).max(axis=2, keepdims=True)[..., :1] if kind == "scaled" else None
    scale = None if scale is None else np.maximum(scale, 1.0)
    _check_small(oracle_mod, x, S, 96, scale=scale, variant=variant)


def test_batch_zero_and_one(oracle_mod):
    m, _ = _model(3, 96, 24, 96)
    x = torch.zeros((0, 3, 96), device="cuda")
    assert m.forward(x).shape == (0, 3, 96)
    xx = synth.random_windows(1, 3, 96)
    _check_small(oracle_mod, xx, 24, 96)


# ------------------------------------------------------------------ index map, intermediates
@pytest.mark.parametrize("L,S", [(720, 24), (722, 24), (97, 7), (5760, 12)])
def test_segment_gather_bit_exact(L, S):
    x = synth.random_windows(3, 4, L, kind="normal")
    m, _ = _model(4, L, S, 10)
    seg = m.debug_segments(torch.from_numpy(x).cuda()).cpu().numpy()
    N, r = L // S, L - (L // S) * S
    idx = r + np.arange(N)[:, None] * S + np.arange(S)[None, :]
    np.testing.assert_array_equal(seg, x[:, :, idx])


@pytest.mark.parametrize("variant", ["warp_f32", "mma_f16x3", "tc_quad", "long_f32"])
@pytest.mark.parametrize("L,S", [(720, 24), (96, 24), (384, 24), (480, 24)])
def test_attention_matrices(oracle_mod, L, S, variant):
    x = synth.random_windows(2, 3, L, kind="mixed")
    m, _ = _model(3, L, S, 24, tau_s=0.5, tau_t=2.0, variant=variant)
    a_s, a_t = m.debug_attention(torch.from_numpy(x).cuda())
    a_s, a_t = a_s.cpu().numpy(), a_t.cpu().numpy()
    np.testing.assert_allclose(a_s.sum(-1), 1.0, atol=1e-6)
    np.testing.assert_allclose(a_t.sum(-1), 1.0, atol=1e-6)
    N = L // S
    for b in range(2):
        for c in range(3):
            r = oracle_mod.series(x[b, c], S, 24, np.zeros((1, N)), np.zeros((1, N)),
                                  np.zeros(24), 0.5, 2.0)
            np.testing.assert_allclose(a_s[b, c], r["a_s"], atol=2e-6)
            np.testing.assert_allclose(a_t[b, c], r["a_t"], atol=2e-6)
            assert np.all(np.argmax(a_s[b, c], 1) == np.arange(N))


# ------------------------------------------------------------------ determinism, sharding, host path
@pytest.mark.parametrize("variant", SHORT_VARIANTS)
def test_deterministic_and_shard_invariant(variant):
    from paper_2404_02445_b200 import shard_windows
    x = torch.from_numpy(synth.random_windows(37, 11, 720)).cuda()
    m, _ = _model(11, 720, 24, 720, variant=variant)
    y1 = m.forward(x)
    y2 = m.forward(x)
    assert torch.equal(y1, y2)
    for world in (2, 3, 8):
        parts = []
        for rank in range(world):
            s, n = shard_windows(37, world, rank)
            parts.append(m.forward(x[s:s + n].contiguous()))
        assert torch.equal(torch.cat(parts), y1)


def test_forward_host_matches_device():
    x = synth.random_windows(29, 7, 720)
    m, _ = _model(7, 720, 24, 336)
    yd = m.forward(torch.from_numpy(x).cuda()).cpu()
    xp = torch.from_numpy(x).pin_memory()
    for chunk in (None, 1, 5, 29, 64):
        yh = m.forward_host(xp, chunk_windows=chunk)
        assert torch.equal(yh, yd)


def test_error_sums_device(oracle_mod):
    rng = np.random.default_rng(3)
    y = rng.normal(size=(13, 5, 96)).astype(np.float32)
    t = rng.normal(size=(13, 5, 96)).astype(np.float32)
    m, _ = _model(5, 96, 24, 96)
    out = m.error_sums(torch.from_numpy(y).cuda(), torch.from_numpy(t).cuda()).cpu().numpy()
    sse, sae, n = oracle_mod.error_sums(y, t)
    assert n == out[2] and abs(out[0] - sse) < 1e-9 * sse and abs(out[1] - sae) < 1e-9 * sae


# ------------------------------------------------------------------ ABI error behaviour
def test_abi_errors():
    from paper_2404_02445_b200.prnet import PRNet as P
    with pytest.raises(PrnetError) as e:
        P(3, 20, 24, 5)               # L < S
    assert e.value.status == 1
    with pytest.raises(PrnetError):
        P(3, 96, 24, 96, tau_s=0.0)
    m = P(3, 96, 24, 96)
    x = torch.zeros((2, 3, 96), device="cuda")
    with pytest.raises(PrnetError) as e:
        m.forward(x)                  # before load
    assert e.value.status == 2
    N, M = m.N, m.M
    w0 = np.zeros(3 * M * N, np.float32)
    assert m._lib.prnet_load_params(m.handle, w0.ctypes.data, w0.ctypes.data, w0.ctypes.data,
                                    w0.size, 3 * 96 - 1) == 1      # wrong bias count
    assert m._lib.prnet_forward(m.handle, None, -1, None, None) == 2   # still not loaded
    m.load(np.zeros((3, M, N)), np.zeros((3, M, N)), np.zeros((3, 96)))
    buf = torch.zeros(2 * 3 * 96 + 1, device="cuda")
    xm = buf[1:].view(2, 3, 96)       # 4-byte offset: misaligned
    with pytest.raises(PrnetError) as e:
        m.forward(xm)
    assert e.value.status == 3
    with pytest.raises(PrnetError) as e:
        m.forward_into(x, x)          # overlap (H == L here)
    assert e.value.status == 3
    with pytest.raises(PrnetError) as e:
        m.forward(torch.zeros((2, 3, 96)))   # host pointer on the device entry
    assert e.value.status == 3


# ------------------------------------------------------------ SURVEY §8(f) widening (f1, f3)
def _check_widening(oracle_mod, x, S, H, mv, rev, variant=None, tau_s=1.0, tau_t=1.0, hpc=True,
                    ma=0):
    B, C, L = x.shape
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, hpc, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, head_per_channel=hpc, tau_s=tau_s, tau_t=tau_t, metric_variant=mv,
              instance_norm=rev, ma_kernel=ma).load(ws, wt, b)
    if variant is not None:
        m.set_variant(variant)
    y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, hpc, tau_s, tau_t, metric_variant=mv,
                                instance_norm=rev, ma_kernel=ma)
    if rev:   # reading R-tol-revin: the bar applies to the normalised forecast
        return assert_parity_revin(y, y64, x, S)
    return assert_parity(y, y64)


@pytest.mark.parametrize("variant", [None, "tc_quad", "mma_f16x3"])
@pytest.mark.parametrize("mv,rev", [(1, False), (2, False), (3, False), (0, True), (3, True)])
@pytest.mark.parametrize("L,S,H", [(720, 24, 720), (720, 24, 336), (100, 24, 90), (96, 24, 96),
                                   (97, 7, 13), (128, 8, 64), (270, 9, 31)])
def test_widening_parity(oracle_mod, L, S, H, mv, rev, variant):
    if variant == "tc_quad" and S != 24:
        pytest.skip("tc_quad needs S = 24")
    x = synth.random_windows(3, 5, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev, variant)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
@pytest.mark.parametrize("rev", [False, True])
def test_widening_value_distributions(oracle_mod, kind, rev):
    x = synth.random_windows(3, 4, 720, kind=kind)
    if kind == "scaled" and not rev:
        pytest.skip("covered by test_value_distributions")
    _check_widening(oracle_mod, x, 24, 96, 3 if not rev else 2, rev)


@pytest.mark.parametrize("tau", [0.05, 1.0, 10.0])
@pytest.mark.parametrize("hpc", [True, False])
def test_widening_temperatures_and_head_modes(oracle_mod, tau, hpc):
    x = synth.random_windows(4, 6, 720, kind="mixed")
    _check_widening(oracle_mod, x, 24, 336, 3, True, tau_s=tau, tau_t=tau * 0.7, hpc=hpc)


@pytest.mark.parametrize("variant", VARIANTS)
def test_level_trend_every_variant(oracle_mod, variant):
    """metric_variant bit 0 only changes a scalar (vtrend = 0): every kernel implements it."""
    for L, S, H in [(720, 24, 96), (1440, 24, 96), (97, 7, 13)]:
        N, _, M = synth.derived_dims(L, S, H)
        if not _applicable(variant, L, S, H):
            continue
        x = synth.random_windows(2, 3, L, kind="mixed")
        _check_widening(oracle_mod, x, S, H, 1, False, variant)


@pytest.mark.parametrize("mv,rev", [(2, False), (0, True), (3, True)])
@pytest.mark.parametrize("L,S,H", [(1440, 24, 96), (1536, 12, 200), (2880, 48, 96),
                                   (3840, 96, 96), (3250, 65, 130), (4000, 120, 100),
                                   (5000, 100, 1100)])
def test_widening_parity_long_lookback(oracle_mod, L, S, H, mv, rev):
    """N > 32: the flash kernel implements the widening (S <= 96), long_f32 beyond."""
    x = synth.random_windows(2, 3, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev)


@pytest.mark.parametrize("mv,rev", [(1, False), (2, False), (3, True), (0, True), (4, False),
                                    (5, True), (6, False), (7, True)])
@pytest.mark.parametrize("L,S,H", [(1440, 24, 96), (1536, 12, 200), (97, 7, 13)])
def test_widening_parity_long_f32(oracle_mod, L, S, H, mv, rev):
    """The FP32 row-streaming kernel under every detrend / RevIN / component flag (forced)."""
    x = synth.random_windows(2, 3, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev, variant="long_f32")


@pytest.mark.parametrize("mv,rev", [(4, False), (5, False), (6, False), (7, False), (4, True),
                                    (7, True)])
@pytest.mark.parametrize("L,S,H", [(720, 24, 720), (720, 24, 336), (100, 24, 90), (96, 24, 96),
                                   (97, 7, 13), (128, 8, 64), (270, 9, 31), (384, 128, 200),
                                   (1440, 24, 96), (1536, 12, 200), (2880, 48, 96),
                                   (3840, 96, 96), (5760, 12, 96), (4000, 120, 100)])
def test_component_values_parity(oracle_mod, L, S, H, mv, rev):
    """metric_variant bit 2 (component values, reading R-f4): mma_f16x3 (N <= 32), the
    flash_f16x3 COMP instantiation (N > 32)."""
    x = synth.random_windows(3, 5, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev)


@pytest.mark.parametrize("mv,rev", [(4, False), (5, False), (6, False), (7, False), (4, True),
                                    (6, True), (7, True)])
@pytest.mark.parametrize("L,H", [(720, 720), (720, 336), (100, 90), (96, 96), (480, 200),
                                 (744, 24)])
def test_component_values_tc_quad(oracle_mod, L, H, mv, rev):
    """The S = 24 tc_quad COMP instantiation (forced, every N it takes): Q_s and Q_t folded into
    separate TMEM columns, alpha / beta from the head's 4th n-tile [mu^, kappa^] (reading R-f4)."""
    x = synth.random_windows(3, 5, L, kind="mixed")
    _check_widening(oracle_mod, x, 24, H, mv, rev, variant="tc_quad")


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
@pytest.mark.parametrize("tau,hpc", [(0.05, True), (1.0, False), (10.0, True)])
def test_component_values_distributions(oracle_mod, kind, tau, hpc):
    x = synth.random_windows(3, 4, 720, kind=kind)
    _check_widening(oracle_mod, x, 24, 336, 6, kind == "scaled", tau_s=tau, tau_t=tau * 0.7,
                    hpc=hpc)


@pytest.mark.parametrize("ma", [1, 3, 25, 101])
@pytest.mark.parametrize("mv,rev", [(0, False), (3, False), (4, False), (7, False), (0, True),
                                    (6, True)])
@pytest.mark.parametrize("L,S,H", [(720, 24, 720), (720, 24, 96), (100, 24, 90), (97, 7, 13),
                                   (270, 9, 31), (384, 128, 200)])
def test_ma_decomposition_parity(oracle_mod, L, S, H, mv, rev, ma):
    """ma_kernel (moving-average decomposition feeding each branch, reading R-f5)."""
    x = synth.random_windows(2, 4, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev, ma=ma)


@pytest.mark.parametrize("ma", [1, 5, 25])
@pytest.mark.parametrize("mv,rev", [(0, False), (3, True), (4, False), (7, True)])
@pytest.mark.parametrize("L,S,H", [(1440, 24, 96), (1536, 12, 200), (4000, 120, 100),
                                   (3000, 150, 96), (700, 200, 450)])
def test_ma_decomposition_parity_long(oracle_mod, L, S, H, mv, rev, ma):
    """N > 32, or S > 128: long_f32 implements every widening flag."""
    x = synth.random_windows(2, 3, L, kind="mixed")
    _check_widening(oracle_mod, x, S, H, mv, rev, ma=ma)


@pytest.mark.parametrize("kind", ["normal", "constant", "scaled"])
@pytest.mark.parametrize("tau,hpc", [(0.05, True), (1.0, False), (10.0, True)])
def test_ma_decomposition_distributions(oracle_mod, kind, tau, hpc):
    x = synth.random_windows(3, 4, 720, kind=kind)
    _check_widening(oracle_mod, x, 24, 336, 0, kind == "scaled", tau_s=tau, tau_t=tau * 0.7,
                    hpc=hpc, ma=25)


def test_ma_decomposition_attention_dump():
    """debug_attention on a decomposition handle dumps rows that sum to 1."""
    m = PRNet(3, 720, 24, 96, ma_kernel=25)
    ws, wt, b = synth.make_params(3, m.M, m.N, 96, True, synth.DEFAULT_SEED, 0)
    m.load(ws, wt, b)
    x = torch.from_numpy(synth.random_windows(2, 3, 720, kind="mixed")).cuda()
    a_s, a_t = m.debug_attention(x)
    for a in (a_s, a_t):
        np.testing.assert_allclose(a.sum(-1).cpu().numpy(), 1.0, atol=1e-5)


def test_component_values_unsupported_paths():
    m = PRNet(3, 3000, 150, 96, ma_kernel=5)            # N = 20, S = 150: long_f32 runs it
    m.load(np.zeros((3, m.M, m.N)), np.zeros((3, m.M, m.N)), np.zeros((3, 96)))
    m.forward(torch.zeros((2, 3, 3000), device="cuda"))
    m2 = PRNet(3, 720, 24, 96, metric_variant=4)
    for v in ("small_f32", "warp_f32"):
        with pytest.raises(PrnetError) as e:
            m2.set_variant(v)
        assert e.value.status == 3
    m2.set_variant("tc_quad")   # S = 24: the COMP instantiation (round 2)
    m3 = PRNet(3, 720, 24, 96, metric_variant=4, ma_kernel=5)
    with pytest.raises(PrnetError) as e:   # the decomposition is not compiled into tc_quad
        m3.set_variant("tc_quad")
    assert e.value.status == 3
    m2.set_variant("mma_f16x3")
    m2.set_variant("flash_f16x3")


def test_widening_unsupported_paths():
    with pytest.raises(PrnetError) as e:                 # N = 516 > 512: rejected at create
        PRNet(3, 6192, 12, 96, metric_variant=2)
    assert e.value.status == 3
    m2 = PRNet(3, 720, 24, 96, instance_norm=True)
    with pytest.raises(PrnetError) as e:
        m2.set_variant("warp_f32")
    assert e.value.status == 3
    m3 = PRNet(3, 720, 24, 96, metric_variant=1)         # level-only: any variant
    m3.set_variant("warp_f32")


# ------------------------------------------------------------ sliding windows
def _series_and_windows(C, T, L, t0, B, seed=5):
    g = np.random.default_rng(seed)
    t = np.arange(T)[None, :]
    s = (np.sin(2 * np.pi * t / g.integers(6, 30, (C, 1))) + 0.3 * g.standard_normal((C, T))
         + g.uniform(-1, 1, (C, 1)) * t / T).astype(np.float32)
    x = np.stack([s[:, t0 + b:t0 + b + L] for b in range(B)])      # [B, C, L]
    return s, np.ascontiguousarray(x)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("L,S,H", [(720, 24, 96), (96, 24, 96), (100, 24, 90), (97, 7, 13),
                                   (1440, 24, 96), (270, 9, 31)])
@pytest.mark.parametrize("t0", [0, 1, 2, 3, 6])
def test_sliding_equals_materialised_windows(L, S, H, t0, variant):
    """prnet_forward_sliding is bitwise prnet_forward on the materialised windows, for every
    kernel and every window alignment (t0 + b mod 4)."""
    if not _applicable(variant, L, S, H):
        pytest.skip("variant not applicable")
    C, B = 5, 11
    T = t0 + B - 1 + L + 3
    s, x = _series_and_windows(C, T, L, t0, B)
    m, _ = _model(C, L, S, H, variant=variant)
    y_win = m.forward(torch.from_numpy(x).cuda())
    y_sl = m.forward_sliding(torch.from_numpy(s).cuda(), t0, B)
    assert torch.equal(y_sl, y_win)


@pytest.mark.parametrize("t0", [0, 1, 3])
@pytest.mark.parametrize("L,S,H,mv,rev,ma", [(720, 24, 336, 3, True, 0), (720, 24, 336, 4, False, 0),
                                             (720, 24, 96, 7, True, 25), (97, 7, 13, 6, False, 3),
                                             (1440, 24, 96, 2, True, 0)])
def test_sliding_widening_equals_materialised(L, S, H, mv, rev, ma, t0):
    """The sliding mode under every widening flag (f1, f3) is bitwise the materialised
    forward (the generic paths load unaligned windows element-wise)."""
    C, B = 4, 9
    T = t0 + B - 1 + L + 2
    s, x = _series_and_windows(C, T, L, t0, B, seed=11)
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0)
    m = PRNet(C, L, S, H, metric_variant=mv, instance_norm=rev, ma_kernel=ma).load(ws, wt, b)
    y_win = m.forward(torch.from_numpy(x).cuda())
    y_sl = m.forward_sliding(torch.from_numpy(s).cuda(), t0, B)
    assert torch.equal(y_sl, y_win)


@pytest.mark.parametrize("t0", [0, 3])
def test_sliding_window_at_the_end_of_the_series(oracle_mod, t0):
    """The last window ends exactly at T (the aligned-superset load must not run past the
    buffer), checked against the oracle."""
    C, L, S, H, B = 4, 720, 24, 336, 9
    T = t0 + B - 1 + L
    s, x = _series_and_windows(C, T, L, t0, B, seed=9)
    m, (ws, wt, b) = _model(C, L, S, H)
    y = m.forward_sliding(torch.from_numpy(s).cuda(), t0, B).cpu().numpy()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True)
    assert_parity(y, y64)


@pytest.mark.parametrize("chunk", [None, 1, 4, 64])
def test_sliding_host_matches_device(chunk):
    C, L, S, H, B, t0 = 6, 720, 24, 720, 37, 5
    T = t0 + B - 1 + L + 11
    s, _ = _series_and_windows(C, T, L, t0, B, seed=3)
    m, _ = _model(C, L, S, H)
    yd = m.forward_sliding(torch.from_numpy(s).cuda(), t0, B).cpu()
    sp = torch.from_numpy(s).pin_memory()
    yh = m.forward_sliding_host(sp, t0, B, chunk_windows=chunk)
    assert torch.equal(yh, yd)


def test_sliding_argument_errors():
    m, _ = _model(3, 96, 24, 96)
    s = torch.zeros((3, 200), device="cuda")
    with pytest.raises(PrnetError) as e:
        m.forward_sliding(s, 100, 10)              # t0 + B - 1 + L = 205 > 200
    assert e.value.status == 1
    with pytest.raises(PrnetError) as e:
        m.forward_sliding(s, -1, 2)
    assert e.value.status == 1
    assert m.forward_sliding(s, 104, 1).shape == (1, 3, 96)   # ends exactly at T


# ------------------------------------------------------------------ every output element written
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("L,S,H,mv", [(720, 24, 336, 0), (720, 24, 96, 0), (720, 24, 720, 4),
                                      (96, 24, 96, 0), (97, 7, 13, 0), (1440, 24, 100, 0)])
def test_every_output_element_written(L, S, H, mv, variant):
    """Forward into a NaN-filled y: no element may stay unwritten (the mma_f16x3 S = 24
    epilogue writes y with TMA bulk stores, which compute-sanitizer initcheck does not see)."""
    if not _applicable(variant, L, S, H):
        pytest.skip("variant not applicable")
    if mv and variant not in (None, "mma_f16x3"):
        pytest.skip("component values run in mma_f16x3")
    x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    m = PRNet(3, L, S, H, metric_variant=mv).load(ws, wt, b)
    if variant is not None:
        m.set_variant(variant)
    y = torch.full((5, 3, H), float("nan"), device="cuda")
    m.forward_into(x, y)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()


# ------------------------------------------------------------------ heterogeneous segment scales
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("L,S,H", [(720, 24, 336), (336, 24, 96), (1440, 24, 96), (97, 7, 13),
                                   (576, 48, 96)])
@pytest.mark.parametrize("mv", [0, 2])
def test_heterogeneous_segment_scales(oracle_mod, L, S, H, mv, variant):
    """Segments whose amplitudes differ by up to 1e4 within one series (quiet and busy
    periods), at a sharp seasonal temperature: the Gram operand's precision must hold
    relative to every row, not only to the largest."""
    if not _applicable(variant, L, S, H):
        pytest.skip("variant not applicable")
    g = np.random.default_rng(L + S + mv)
    B, C = 3, 4
    N = L // S
    x = synth.random_windows(B, C, L, kind="normal").astype(np.float64)
    r = L - N * S
    amp = 10.0 ** g.uniform(-4, 0, (B, C, N))
    x[:, :, r:] = (x[:, :, r:].reshape(B, C, N, S) * amp[..., None]).reshape(B, C, N * S)
    x = x.astype(np.float32)
    N_, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N_, H, True, synth.DEFAULT_SEED, 0)
    try:
        m = PRNet(C, L, S, H, tau_s=0.05, metric_variant=mv).load(ws, wt, b)
        if variant is not None:
            m.set_variant(variant)
        y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    except PrnetError as e:
        assert e.status == 3
        pytest.skip(str(e))
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True, 0.05, 1.0, metric_variant=mv)
    assert_parity(y, y64)


# ------------------------------------------------------------------ low seasonal temperatures
def _near_constant_windows(B, C, L, S, seed=5):
    """Mixed windows in which a fifth of the segments are constant to within ~1e-6
    (nu^2 ~ 1e-11, next to eps_s = 1e-12): f_i = nu_i / sqrt(nu_i^2 + eps_s) is then well
    below 1, the case in which a known-maximum shift can leave a row without a normal term."""
    x = synth.random_windows(B, C, L, seed=seed, kind="mixed").astype(np.float64)
    rng = np.random.default_rng(seed)
    N = L // S
    r = L - N * S
    for b in range(B):
        for c in range(C):
            for n in rng.choice(N, size=max(1, N // 5), replace=False):
                lo = r + n * S
                x[b, c, lo:lo + S] = x[b, c, lo] + 1e-6 * rng.standard_normal(S)
    return x.astype(np.float32)


@pytest.mark.parametrize("kind", ["mixed", "near_constant"])
@pytest.mark.parametrize("tau_s", [1e-2, 5e-3, 1e-3])
@pytest.mark.parametrize("L,S,H", [(720, 24, 336), (1440, 24, 96), (5760, 12, 96)])
def test_low_seasonal_temperature(oracle_mod, L, S, H, tau_s, kind):
    """tau_s below tc_quad's floor (1/80) and below the known-maximum kernels' floor (1/320):
    N = 30 (mma_f16x3, then warp_f32), N = 60 / 480 (flash_f16x3, then long_f32)."""
    B, C = 2, 3
    x = (_near_constant_windows(B, C, L, S) if kind == "near_constant"
         else synth.random_windows(B, C, L, kind="mixed"))
    m, (ws, wt, b) = _model(C, L, S, H, tau_s=tau_s, tau_t=0.5)
    v = m.plan(B)["variant"]
    N = L // S
    if tau_s < 1 / 320:
        assert v == ("warp_f32" if N <= 32 else "long_f32"), v
    else:
        # (tc_long needs tau_s >= 1/16: flash_f16x3, with exact maxima for loose rows)
        assert v == ("mma_f16x3" if N <= 32 else "flash_f16x3"), v
    y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.isfinite(y).all()
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True, tau_s, 0.5)
    assert_parity(y, y64)


@pytest.mark.parametrize("tau_s", [1e-3, 1e-6])
def test_low_temperature_every_row_max_kernel(oracle_mod, tau_s):
    """The row-max-searching FP32 kernels at and far below the floors, near-constant
    segments included (the oracle's tau -> 0 limit is pinned on CPU at tau = 1e-6)."""
    for L, S, H, v in [(720, 24, 96, "warp_f32"), (720, 24, 96, "long_f32"),
                       (1440, 24, 96, "long_f32")]:
        x = _near_constant_windows(2, 3, L, S, seed=8)
        m, (ws, wt, b) = _model(3, L, S, H, tau_s=tau_s, tau_t=0.5, variant=v)
        y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True, tau_s, 0.5)
        assert_parity(y, y64)


def test_temperature_floors_route_and_reject():
    """Known-maximum kernels reject tau_s < 1/320 (include/prnet.h), tc_quad tau_s < 1/80;
    the automatic choice routes around them."""
    m = PRNet(3, 720, 24, 96, tau_s=1e-3)
    assert m.plan(4)["variant"] == "warp_f32"
    for v in ("mma_f16x3", "small_f32", "tc_quad"):
        with pytest.raises(PrnetError) as e:
            m.set_variant(v)
        assert e.value.status == 3
    m.set_variant("long_f32")
    m2 = PRNet(3, 1440, 24, 96, tau_s=1e-3)
    assert m2.plan(4)["variant"] == "long_f32"
    with pytest.raises(PrnetError):
        m2.set_variant("flash_f16x3")
    m3 = PRNet(3, 720, 24, 96, tau_s=5e-3)
    assert m3.plan(4)["variant"] == "mma_f16x3"
    with pytest.raises(PrnetError):
        m3.set_variant("tc_quad")
    m4 = PRNet(3, 720, 24, 96, tau_s=1e-3, instance_norm=True)   # widened: long_f32
    assert m4.plan(4)["variant"] == "long_f32"


# ------------------------------------------------------------------ attention dumps
@pytest.mark.parametrize("mv,rev", [(0, False), (2, False), (0, True), (3, True)])
@pytest.mark.parametrize("L", [720, 480, 100])
def test_tc_quad_attention_dump(oracle_mod, L, mv, rev):
    """tc_quad's own softmax (shift 1, exchanged normalisers, the values its TMEM store
    takes) compared element-wise with the oracle's attention rows."""
    S, H, C, B = 24, 96, 3, 5
    x = synth.random_windows(B, C, L, kind="mixed")
    m = PRNet(C, L, S, H, tau_s=0.5, tau_t=2.0, metric_variant=mv, instance_norm=rev)
    N, _, M = synth.derived_dims(L, S, H)
    m.load(*synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0))
    m.set_variant("tc_quad")
    a_s, a_t = (a.cpu().numpy() for a in m.debug_attention(torch.from_numpy(x).cuda()))
    for b in range(B):
        for c in range(C):
            r = oracle_mod.series(x[b, c], S, 24, np.zeros((1, N)), np.zeros((1, N)),
                                  np.zeros(24), 0.5, 2.0, metric_variant=mv, instance_norm=rev)
            np.testing.assert_allclose(a_s[b, c], r["a_s"], atol=2e-6)
            np.testing.assert_allclose(a_t[b, c], r["a_t"], atol=2e-6)


@pytest.mark.parametrize("mv,rev,ma", [(2, False, 25), (6, True, 25), (4, False, 0),
                                       (7, True, 0), (2, False, 3)])
@pytest.mark.parametrize("L,S", [(720, 24), (336, 12), (100, 24)])
def test_attention_dump_widened(oracle_mod, L, S, mv, rev, ma):
    """debug_attention on widened handles with N <= 32 (detrended metric, component values,
    instance normalisation, moving-average decomposition), compared element-wise with the
    oracle's attention rows (round-1 advice: the dump must follow the handle's flags)."""
    C, B, H = 2, 3, 96
    x = synth.random_windows(B, C, L, kind="mixed")
    N, _, M = synth.derived_dims(L, S, H)
    m = PRNet(C, L, S, H, tau_s=0.5, tau_t=2.0, metric_variant=mv, instance_norm=rev,
              ma_kernel=ma)
    m.load(*synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0))
    a_s, a_t = (a.cpu().numpy() for a in m.debug_attention(torch.from_numpy(x).cuda()))
    for b in range(B):
        for c in range(C):
            r = oracle_mod.series(x[b, c], S, S, np.zeros((1, N)), np.zeros((1, N)),
                                  np.zeros(S), 0.5, 2.0, metric_variant=mv, instance_norm=rev,
                                  ma_kernel=ma)   # (H = S: one future segment, zero head)
            np.testing.assert_allclose(a_s[b, c], r["a_s"], atol=2e-6)
            np.testing.assert_allclose(a_t[b, c], r["a_t"], atol=2e-6)


@pytest.mark.parametrize("L,S", [(1440, 24), (2880, 48), (1536, 24)])
@pytest.mark.parametrize("ma", [0, 9])
def test_attention_dump_long_n(oracle_mod, L, S, ma):
    """debug_attention for N > 32 (flash_f16x3 handles are dumped by long_f32, which also
    implements every widening flag)."""
    C, B, H = 2, 2, 96
    x = synth.random_windows(B, C, L, kind="mixed")
    N, _, M = synth.derived_dims(L, S, H)
    m = PRNet(C, L, S, H, tau_s=0.5, tau_t=2.0, ma_kernel=ma)
    m.load(*synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0))
    a_s, a_t = (a.cpu().numpy() for a in m.debug_attention(torch.from_numpy(x).cuda()))
    for b in range(B):
        for c in range(C):
            r = oracle_mod.series(x[b, c], S, 24, np.zeros((1, N)), np.zeros((1, N)),
                                  np.zeros(24), 0.5, 2.0, ma_kernel=ma)
            np.testing.assert_allclose(a_s[b, c], r["a_s"], atol=2e-6)
            np.testing.assert_allclose(a_t[b, c], r["a_t"], atol=2e-6)

"""Seeded synthetic workloads for the PRNet pattern-attention forward.

This module is shared by the CUDA path's tests/bench and by the oracle's tests.
It holds NONE of the method's arithmetic (no segmentation, similarity, softmax
or head): only the input recipe of DESIGN.md §5 (SURVEY.md §8(d) "Synthetic
inputs"): per-channel "seasonal + trend + noise" series ("sequences
comprise unpredictable noise and predictable patterns"), standardised with
train-split statistics (A18), the LTSF test-window convention, and random-init
head parameters.

Every random stream is keyed by (seed, config id, channel) through numpy's
counter-based Philox generator, so a channel's series does not depend on how
windows or channels are sharded across ranks.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

DEFAULT_SEED = 2404


@dataclasses.dataclass(frozen=True)
class Workload:
    """One benchmark/parity configuration (BASELINE.json ``configs``)."""
    name: str
    cfg_id: int
    C: int            # channels
    L: int            # lookback
    S: int            # segment length
    H: int            # horizon
    T: int            # length of the synthetic series per channel
    P1: int           # main seasonal period (time steps)
    P2: int           # secondary (weekly) period
    B: int | None = None   # None -> the full LTSF test set (num_test - H + 1)

    @property
    def num_test(self) -> int:
        # LTSF 7:1:2 split, test part = floor(0.2 T)  [EXT, SURVEY.md §8(d)]
        return int(0.2 * self.T)

    @property
    def num_train(self) -> int:
        return int(0.7 * self.T)

    @property
    def windows(self) -> int:
        full = self.num_test - self.H + 1
        return full if self.B is None else min(self.B, full)

    @property
    def t0(self) -> int:
        """Series index of window 0's first lookback point."""
        return self.T - self.num_test - self.L


def _hourly(name, cfg_id, C, L, S, H, T, B=None):
    return Workload(name, cfg_id, C, L, S, H, T, 24, 168, B)


def _stress(L, S, H=96):
    B = 1000
    # long enough for a train split ahead of the B test windows
    T_needed = L + B + H - 1
    T = int(math.ceil(T_needed / 0.2)) + 1
    return Workload(f"stress_L{L}_S{S}_H{H}", 100 + 10 * L + S, 100, L, S, H, T, 24, 168, B)


# BASELINE.json configs[0..4]
WORKLOADS = {
    # configs[0]: ETTh1-shaped, B=32, C=7, L=96, H=96, S=24 (T = ETTh1 length 17420)
    "etth1": _hourly("etth1", 1, 7, 96, 24, 96, 17420, B=32),
    # configs[1]: Weather-shaped, C=21, L=720, full test set, H in {96,192,336,720};
    # 10-minute data -> periods 144 (day) and 1008 (week); T = 52696
    **{f"weather_h{h}": Workload(f"weather_h{h}", 2, 21, 720, 24, h, 52696, 144, 1008)
       for h in (96, 192, 336, 720)},
    # configs[2]: Electricity-shaped, C=321, L=720, H=336, all test windows (T = 26304)
    "electricity": _hourly("electricity", 3, 321, 720, 24, 336, 26304),
    # configs[3]: Traffic-shaped, C=862, L=720, H=720, all test windows (T = 17544)
    "traffic": _hourly("traffic", 4, 862, 720, 24, 720, 17544),
}
# configs[4]: stress sweep, 100k channel-series (C=100 x B=1000), L 96..5760, S 12..96
STRESS_GRID = [(L, S) for L in (96, 192, 336, 720, 1440, 2880, 5760) for S in (12, 24, 48, 96)
               if L // S >= 1]
for _L, _S in STRESS_GRID:
    for _H in (96, 720):   # H = 96 is the proposed default; "also run H = 720"
        _w = _stress(_L, _S, _H)
        WORKLOADS[_w.name] = _w


def _rng(seed: int, cfg_id: int, stream: int) -> np.random.Generator:
    key = (int(seed) << 64) | (int(cfg_id) << 32) | int(stream)
    return np.random.Generator(np.random.Philox(key=key))


def make_channel(w: Workload, c: int, seed: int = DEFAULT_SEED) -> np.ndarray:
    """Series of channel c, float32 [T], standardised with train-split stats.

    s_c(t) = a sin(2 pi t/P1 + phi) + a' sin(2 pi t/P2 + phi') + beta t/T + gamma + 0.2 eps(t)
    with a~U(0.5,1.5), a'~U(0.1,0.5), phi,phi'~U(0,2pi), beta~U(-1,1), gamma~N(0,0.5),
    eps~N(0,1).
    """
    g = _rng(seed, w.cfg_id, c)
    a, a2 = g.uniform(0.5, 1.5), g.uniform(0.1, 0.5)
    phi, phi2 = g.uniform(0, 2 * np.pi), g.uniform(0, 2 * np.pi)
    beta, gamma = g.uniform(-1, 1), g.normal(0, 0.5)
    t = np.arange(w.T, dtype=np.float64)
    s = (a * np.sin(2 * np.pi * t / w.P1 + phi) + a2 * np.sin(2 * np.pi * t / w.P2 + phi2)
         + beta * t / w.T + gamma + 0.2 * g.standard_normal(w.T))
    tr = s[: w.num_train]
    s = (s - tr.mean()) / tr.std()
    return s.astype(np.float32)


def make_series(w: Workload, seed: int = DEFAULT_SEED, channels=None) -> np.ndarray:
    """float32 [C', T] for the given channel list (default all)."""
    chans = range(w.C) if channels is None else channels
    return np.stack([make_channel(w, c, seed) for c in chans])


def window_batch(series: np.ndarray, w: Workload, b_idx) -> tuple[np.ndarray, np.ndarray]:
    """Materialise test windows b_idx from series [C, T]: x [len(b), C, L], target [len(b), C, H].
    Window b covers series[t0 + b : t0 + b + L], its target the next H points."""
    b_idx = np.asarray(b_idx, dtype=np.int64)
    starts = w.t0 + b_idx
    xi = starts[:, None] + np.arange(w.L)[None, :]
    ti = starts[:, None] + w.L + np.arange(w.H)[None, :]
    x = np.ascontiguousarray(series[:, xi].transpose(1, 0, 2))
    tgt = np.ascontiguousarray(series[:, ti].transpose(1, 0, 2))
    return x, tgt


def make_params(C: int, M: int, N: int, H: int, head_per_channel: bool = True,
                seed: int = DEFAULT_SEED, cfg_id: int = 0):
    """Random-init head: ws, wt ~ U(+-1/sqrt(N)) [Cw, M, N]; bias ~ U(+-1/sqrt(N)) [Cw, H]
    (the nn.Linear default bound for fan-in N), Cw = C or 1.  Stream = seed + 1."""
    Cw = C if head_per_channel else 1
    g = _rng(seed + 1, cfg_id, 0xFFFF)
    bound = 1.0 / math.sqrt(N)
    ws = g.uniform(-bound, bound, size=(Cw, M, N)).astype(np.float32)
    wt = g.uniform(-bound, bound, size=(Cw, M, N)).astype(np.float32)
    bias = g.uniform(-bound, bound, size=(Cw, H)).astype(np.float32)
    return ws, wt, bias


def derived_dims(L: int, S: int, H: int):
    """Shape bookkeeping only (no method arithmetic): N = L // S, r = L - N S,
    M = ceil(H / S) -- the ABI's documented derived sizes (include/prnet.h)."""
    N = L // S
    return N, L - N * S, -(-H // S)


def random_windows(B: int, C: int, L: int, seed: int = DEFAULT_SEED, kind: str = "mixed"):
    """Small seeded [B, C, L] inputs for edge-case parity tests.
    kind: 'mixed' (seasonal+trend+noise per series), 'normal', 'constant', 'scaled'."""
    g = _rng(seed, 7, B * 1000 + C * 10 + L)
    if kind == "normal":
        return g.standard_normal((B, C, L)).astype(np.float32)
    if kind == "constant":
        return np.broadcast_to(g.standard_normal((B, C, 1)), (B, C, L)).astype(np.float32).copy()
    t = np.arange(L)[None, None, :]
    per = g.integers(4, 40, size=(B, C, 1))
    x = (g.uniform(0.5, 1.5, (B, C, 1)) * np.sin(2 * np.pi * t / per + g.uniform(0, 6.3, (B, C, 1)))
         + g.uniform(-1, 1, (B, C, 1)) * t / L + g.normal(0, 0.5, (B, C, 1))
         + 0.2 * g.standard_normal((B, C, L)))
    if kind == "scaled":
        x = x * 10.0 ** g.uniform(-3, 3, (B, C, 1))
    return x.astype(np.float32)

"""CPU oracle of the PRNet pattern-attention forward -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_2404_02445_b200``) never imports it and shares no code with it.

The arithmetic lives in ``prnet_oracle.c`` (plain C, fp64, single-threaded,
one function per definition step of SURVEY.md §8(c), restated with citations
in DESIGN.md §3).  This module only compiles it with gcc and marshals numpy
arrays through ctypes.

Parity status: every step is pinned by the CPU tests in
``tests/test_oracle_pins.py`` (closed forms, invariants, limits, worked
examples); agreement with the paper's own equations is *parity unpinned*
because PAPER.md carries no method-section bodies.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "prnet_oracle.c")
_HDR = os.path.join(_HERE, "prnet_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (no fast-math, no vectorisation
    flags that could reassociate fp64 sums)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-std=c11",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Debug(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("seg", "mu", "nu2", "kappa", "sigma2", "rho", "dist", "a_s", "a_t",
                 "p_s", "p_t", "y_full")]


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_dims.argtypes = [ctypes.c_int32] * 3 + [ctypes.POINTER(ctypes.c_int32)] * 3
        lib.oracle_dims.restype = ctypes.c_int
        lib.oracle_series.argtypes = [_f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                      _f32p, _f32p, _f32p, ctypes.c_double, ctypes.c_double,
                                      _f64p, ctypes.POINTER(_Debug)]
        lib.oracle_series.restype = ctypes.c_int
        lib.oracle_forward.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, _f32p, _f32p, _f32p,
                                       ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                       _f32p, _f64p]
        lib.oracle_forward.restype = ctypes.c_int
        lib.oracle_series_ex.argtypes = [_f32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                         _f32p, _f32p, _f32p, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                         ctypes.c_int32, _f64p, ctypes.POINTER(_Debug)]
        lib.oracle_series_ex.restype = ctypes.c_int
        lib.oracle_forward_ex.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, _f32p, _f32p, _f32p,
                                          ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                          ctypes.c_int32, _f32p, _f64p]
        lib.oracle_forward_ex.restype = ctypes.c_int
        lib.oracle_backward_head_ex.argtypes = [
            _f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_int32, _f32p, _f32p, _f32p, ctypes.c_int32, ctypes.c_double,
            ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int32,
            _f32p, _f64p, _f64p, _f64p]
        lib.oracle_backward_head_ex.restype = ctypes.c_int
        lib.oracle_backward.argtypes = [
            _f32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_int32, _f32p, _f32p, _f32p, ctypes.c_int32, ctypes.c_double,
            ctypes.c_double, ctypes.c_int32, _f32p, _f64p, _f64p, _f64p, _f64p, _f64p]
        lib.oracle_backward.restype = ctypes.c_int
        lib.oracle_error_sums.argtypes = [_f32p, _f32p, ctypes.c_int64, _f64p]
        lib.oracle_error_sums.restype = None
        _lib = lib
    return _lib


def dims(L: int, S: int, H: int):
    """(N, r, M) per Definition step 1 (N = floor(L/S), r = L - N S, M = ceil(H/S))."""
    n, r, m = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    if _load().oracle_dims(L, S, H, ctypes.byref(n), ctypes.byref(r), ctypes.byref(m)) != 0:
        raise ValueError(f"invalid dims L={L} S={S} H={H}")
    return n.value, r.value, m.value


EPS_REVIN = 1e-5   # RevIN epsilon of the product (R-f1)


def series(x, S, H, ws, wt, bias, tau_s=1.0, tau_t=1.0, metric_variant=0, instance_norm=False,
           eps_r=EPS_REVIN, ma_kernel=0):
    """One series; returns a dict with y and every intermediate (fp64).
    metric_variant bit 0 = level-only trend, bit 1 = detrended seasonal, bit 2 = component
    values (each branch aggregates its own component, reading R-f4); instance_norm =
    RevIN-style normalisation; ma_kernel = odd k > 0: moving-average decomposition feeding
    each branch (reading R-f5)."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    L = x.size
    N, r, M = dims(L, S, H)
    ws = np.ascontiguousarray(ws, dtype=np.float32).reshape(M, N)
    wt = np.ascontiguousarray(wt, dtype=np.float32).reshape(M, N)
    bias = np.ascontiguousarray(bias, dtype=np.float32).reshape(H)
    out = {
        "seg": np.zeros((N, S)), "mu": np.zeros(N), "nu2": np.zeros(N), "kappa": np.zeros(N),
        "sigma2": np.zeros(1), "rho": np.zeros((N, N)), "dist": np.zeros((N, N)),
        "a_s": np.zeros((N, N)), "a_t": np.zeros((N, N)), "p_s": np.zeros((N, S)),
        "p_t": np.zeros((N, S)), "y_full": np.zeros((M, S)),
    }
    dbg = _Debug(**{k: v.ctypes.data for k, v in out.items()})
    y = np.zeros(H)
    if _load().oracle_series_ex(x, L, S, H, ws, wt, bias, float(tau_s), float(tau_t),
                                int(metric_variant), int(bool(instance_norm)), float(eps_r),
                                int(ma_kernel), y, ctypes.byref(dbg)) != 0:
        raise ValueError("oracle_series rejected its arguments")
    out["sigma2"] = float(out["sigma2"][0])
    out["y"] = y
    out.update(N=N, r=r, M=M)
    return out


def forward(x, S, H, ws, wt, bias, head_per_channel=True, tau_s=1.0, tau_t=1.0,
            metric_variant=0, instance_norm=False, eps_r=EPS_REVIN, ma_kernel=0):
    """x [B, C, L] fp32 -> (y fp32 [B, C, H], y64 fp64 [B, C, H])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    B, C, L = x.shape
    N, r, M = dims(L, S, H)
    Cw = C if head_per_channel else 1
    ws = np.ascontiguousarray(ws, dtype=np.float32).reshape(Cw, M, N)
    wt = np.ascontiguousarray(wt, dtype=np.float32).reshape(Cw, M, N)
    bias = np.ascontiguousarray(bias, dtype=np.float32).reshape(Cw, H)
    y = np.zeros((B, C, H), np.float32)
    y64 = np.zeros((B, C, H), np.float64)
    if _load().oracle_forward_ex(x, B, C, L, S, H, ws, wt, bias, int(bool(head_per_channel)),
                                 float(tau_s), float(tau_t), int(metric_variant),
                                 int(bool(instance_norm)), float(eps_r), int(ma_kernel), y,
                                 y64) != 0:
        raise ValueError("oracle_forward rejected its arguments")
    return y, y64


def backward_head(x, S, H, ws, wt, bias, dy, head_per_channel=True, tau_s=1.0, tau_t=1.0,
                  metric_variant=0, instance_norm=False, eps_r=EPS_REVIN, ma_kernel=0):
    """Gradients (dws, dwt, db), fp64, of sum(dy * y) with respect to the head (SURVEY §8(f)
    f4, reading R-f6); x, dy [B, C, L] / [B, C, H] fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    B, C, L = x.shape
    N, r, M = dims(L, S, H)
    Cw = C if head_per_channel else 1
    ws = np.ascontiguousarray(ws, dtype=np.float32).reshape(Cw, M, N)
    wt = np.ascontiguousarray(wt, dtype=np.float32).reshape(Cw, M, N)
    bias = np.ascontiguousarray(bias, dtype=np.float32).reshape(Cw, H)
    dy = np.ascontiguousarray(dy, dtype=np.float32).reshape(B, C, H)
    dws = np.zeros((Cw, M, N))
    dwt = np.zeros((Cw, M, N))
    db = np.zeros((Cw, H))
    if _load().oracle_backward_head_ex(x, B, C, L, S, H, ws, wt, bias,
                                       int(bool(head_per_channel)), float(tau_s), float(tau_t),
                                       int(metric_variant), int(bool(instance_norm)),
                                       float(eps_r), int(ma_kernel), dy, dws, dwt, db) != 0:
        raise ValueError("oracle_backward_head rejected its arguments")
    return dws, dwt, db


def backward(x, S, H, ws, wt, bias, dy, head_per_channel=True, tau_s=1.0, tau_t=1.0,
             metric_variant=0):
    """The full backward (reading R-f7), fp64: gradients of sum(dy * y)
    with respect to x [B, C, L], the head (dws, dwt [Cw, M, N], db [Cw, H]) and the
    temperatures (dtau = [dL/dtau_s, dL/dtau_t]).  Base reading (metric_variant 0 or 1)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    B, C, L = x.shape
    N, r, M = dims(L, S, H)
    Cw = C if head_per_channel else 1
    ws = np.ascontiguousarray(ws, dtype=np.float32).reshape(Cw, M, N)
    wt = np.ascontiguousarray(wt, dtype=np.float32).reshape(Cw, M, N)
    bias = np.ascontiguousarray(bias, dtype=np.float32).reshape(Cw, H)
    dy = np.ascontiguousarray(dy, dtype=np.float32).reshape(B, C, H)
    dx = np.zeros((B, C, L))
    dws = np.zeros((Cw, M, N))
    dwt = np.zeros((Cw, M, N))
    db = np.zeros((Cw, H))
    dtau = np.zeros(2)
    if _load().oracle_backward(x, B, C, L, S, H, ws, wt, bias, int(bool(head_per_channel)),
                               float(tau_s), float(tau_t), int(metric_variant), dy, dx, dws,
                               dwt, db, dtau) != 0:
        raise ValueError("oracle_backward rejected its arguments")
    return {"dx": dx, "dws": dws, "dwt": dwt, "db": db, "dtau": dtau}


def error_sums(y, target):
    """(SSE, SAE, count) in fp64, index order."""
    y = np.ascontiguousarray(y, dtype=np.float32).ravel()
    target = np.ascontiguousarray(target, dtype=np.float32).ravel()
    out = np.zeros(3)
    _load().oracle_error_sums(y, target, y.size, out)
    return tuple(out)

"""Thin Python binding of the C ABI in include/prnet.h (ctypes).

Argument marshalling only: every step of the forward runs in libprnet.so's
CUDA kernels.  PyTorch is used for device memory (tensors whose data_ptr() is
handed to the ABI) and streams.  There is no CPU fallback: if libprnet.so is
missing or the device is not sm_100, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprnet.so")
_lib = None

PRNET_ABI_VERSION = 3
STATUS = {0: "PRNET_OK", 1: "PRNET_ERR_INVALID_ARG", 2: "PRNET_ERR_BAD_STATE",
          3: "PRNET_ERR_UNSUPPORTED", 4: "PRNET_ERR_CUDA", 5: "PRNET_ERR_OOM"}

# Every symbol include/prnet.h declares (checked by tests/test_abi_cpu.py).
EXPORTS = ("prnet_create", "prnet_load_params", "prnet_forward", "prnet_forward_host",
           "prnet_set_host_chunk", "prnet_destroy", "prnet_last_error", "prnet_get_dims",
           "prnet_debug_segments", "prnet_debug_attention", "prnet_error_sums",
           "prnet_forward_plan", "prnet_set_kernel_variant", "prnet_forward_sliding",
           "prnet_forward_sliding_host", "prnet_backward_head", "prnet_backward", "prnet_forward_bf16")
# index = the C ABI's variant id (include/prnet.h); 3 and 4 are retired round-1 prototypes
VARIANTS = ("warp_f32", "long_f32", "mma_f16x3", "retired_tc_fold", "retired_tc_full",
            "flash_f16x3", "tc_quad", "small_f32", "tc_long", "group_f32")


class PrnetError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PrnetConfig(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("lookback", ctypes.c_int32), ("seg_len", ctypes.c_int32),
                ("horizon", ctypes.c_int32), ("head_per_channel", ctypes.c_int32),
                ("metric_variant", ctypes.c_int32), ("tau_seasonal", ctypes.c_float),
                ("tau_trend", ctypes.c_float), ("device", ctypes.c_int32),
                ("instance_norm", ctypes.c_int32),         # ABI 2
                ("ma_kernel", ctypes.c_int32)]             # ABI 3


def load_library(path: str | None = None):
    """dlopen libprnet.so (raises if absent -- build it with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("PRNET_LIB") or _LIB_PATH   # PRNET_LIB: A/B a second build
    if not os.path.exists(p):
        raise ImportError(f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(p)
    vp, i64, i32p = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int32)
    sig = {
        "prnet_create": ([ctypes.POINTER(PrnetConfig), ctypes.POINTER(vp)], ctypes.c_int),
        "prnet_load_params": ([vp, vp, vp, vp, i64, i64], ctypes.c_int),
        "prnet_forward": ([vp, vp, i64, vp, vp], ctypes.c_int),
        "prnet_forward_host": ([vp, vp, i64, vp], ctypes.c_int),
        "prnet_forward_sliding": ([vp, vp, i64, i64, i64, vp, vp], ctypes.c_int),
        "prnet_forward_sliding_host": ([vp, vp, i64, i64, i64, vp], ctypes.c_int),
        "prnet_set_host_chunk": ([vp, i64], ctypes.c_int),
        "prnet_destroy": ([vp], None),
        "prnet_last_error": ([vp], ctypes.c_char_p),
        "prnet_get_dims": ([vp, i32p, i32p, i32p], ctypes.c_int),
        "prnet_debug_segments": ([vp, vp, i64, vp, vp], ctypes.c_int),
        "prnet_debug_attention": ([vp, vp, i64, vp, vp, vp], ctypes.c_int),
        "prnet_error_sums": ([vp, vp, vp, i64, vp, vp], ctypes.c_int),
        "prnet_forward_plan": ([vp, i64, i32p, i32p], ctypes.c_int),
        "prnet_set_kernel_variant": ([vp, ctypes.c_int32], ctypes.c_int),
        "prnet_backward_head": ([vp, vp, i64, vp, vp, vp, vp, vp], ctypes.c_int),
        "prnet_backward": ([vp, vp, i64, vp, vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "prnet_forward_bf16": ([vp, vp, i64, vp, vp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    _lib = lib
    return lib


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class PRNet:
    """Handle-owning wrapper: PRNet(C, L, S, H).load(ws, wt, b).forward(x) -> y."""

    def __init__(self, channels: int, lookback: int, seg_len: int, horizon: int,
                 head_per_channel: bool = True, tau_s: float = 1.0, tau_t: float = 1.0,
                 device: int = 0, metric_variant: int = 0, instance_norm: bool = False,
                 ma_kernel: int = 0):
        """metric_variant: bit 0 level-only trend, bit 1 detrended seasonal metric, bit 2
        component values (reading R-f4);
        instance_norm: RevIN-style normalisation;
        ma_kernel: odd k > 0 = moving-average decomposition feeding each branch (R-f5)
        (include/prnet.h)."""
        self._lib = load_library()
        cfg = PrnetConfig(PRNET_ABI_VERSION, channels, lookback, seg_len, horizon,
                          int(bool(head_per_channel)), int(metric_variant), tau_s, tau_t, device,
                          int(bool(instance_norm)), int(ma_kernel))
        h = ctypes.c_void_p()
        st = self._lib.prnet_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise PrnetError(st, self._lib.prnet_last_error(None).decode())
        self._h = h
        self.C, self.L, self.S, self.H = channels, lookback, seg_len, horizon
        self.head_per_channel = bool(head_per_channel)
        self.device = device
        n, m, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self._check(self._lib.prnet_get_dims(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(r)))
        self.N, self.M, self.r = n.value, m.value, r.value

    # -- plumbing
    def _check(self, st):
        if st != 0:
            raise PrnetError(st, self._lib.prnet_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.prnet_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- API
    def load(self, ws, wt, bias):
        Cw = self.C if self.head_per_channel else 1
        ws = np.ascontiguousarray(ws, np.float32).reshape(Cw, self.M, self.N)
        wt = np.ascontiguousarray(wt, np.float32).reshape(Cw, self.M, self.N)
        bias = np.ascontiguousarray(bias, np.float32).reshape(Cw, self.H)
        self._check(self._lib.prnet_load_params(self._h, ws.ctypes.data, wt.ctypes.data,
                                                bias.ctypes.data, ws.size, bias.size))
        return self

    def forward_into(self, x, y, stream=None):
        """x: cuda fp32 [B, C, L] contiguous; y: cuda fp32 [B, C, H] (written)."""
        B = x.shape[0]
        assert x.is_contiguous() and y.is_contiguous()
        assert tuple(x.shape) == (B, self.C, self.L) and tuple(y.shape) == (B, self.C, self.H)
        self._check(self._lib.prnet_forward(self._h, ctypes.c_void_p(x.data_ptr()), B,
                                            ctypes.c_void_p(y.data_ptr()), _stream_ptr(stream)))
        return y

    def forward(self, x, stream=None):
        import torch
        y = torch.empty((x.shape[0], self.C, self.H), dtype=torch.float32, device=x.device)
        return self.forward_into(x, y, stream)

    def forward_host(self, x, y=None, chunk_windows: int | None = None):
        """Host buffers end to end (numpy arrays or CPU tensors, ideally pinned)."""
        import torch
        xt = torch.as_tensor(x)
        assert xt.dtype == torch.float32 and xt.is_contiguous() and xt.device.type == "cpu"
        B = xt.shape[0]
        if y is None:
            y = torch.empty((B, self.C, self.H), dtype=torch.float32,
                            pin_memory=xt.is_pinned())
        yt = torch.as_tensor(y)
        if chunk_windows:
            self._check(self._lib.prnet_set_host_chunk(self._h, int(chunk_windows)))
        self._check(self._lib.prnet_forward_host(self._h, ctypes.c_void_p(xt.data_ptr()), B,
                                                 ctypes.c_void_p(yt.data_ptr())))
        return y

    def forward_sliding_into(self, series, t0: int, batch: int, y, stream=None):
        """Sliding windows: series cuda fp32 [C, T] contiguous; window b is
        series[:, t0 + b : t0 + b + L]; y cuda fp32 [batch, C, H] (written)."""
        assert series.is_contiguous() and series.shape[0] == self.C and y.is_contiguous()
        assert tuple(y.shape) == (batch, self.C, self.H)
        self._check(self._lib.prnet_forward_sliding(
            self._h, ctypes.c_void_p(series.data_ptr()), int(series.shape[1]), int(t0),
            int(batch), ctypes.c_void_p(y.data_ptr()), _stream_ptr(stream)))
        return y

    def forward_sliding(self, series, t0: int, batch: int, stream=None):
        import torch
        y = torch.empty((batch, self.C, self.H), dtype=torch.float32, device=series.device)
        return self.forward_sliding_into(series, t0, batch, y, stream)

    def forward_sliding_host(self, series, t0: int, batch: int, y=None,
                             chunk_windows: int | None = None):
        """Sliding windows, host buffers end to end: series [C, T] (numpy / CPU tensor,
        ideally pinned) -> y [batch, C, H]."""
        import torch
        st = torch.as_tensor(series)
        assert st.dtype == torch.float32 and st.is_contiguous() and st.device.type == "cpu"
        if y is None:
            y = torch.empty((batch, self.C, self.H), dtype=torch.float32,
                            pin_memory=st.is_pinned())
        yt = torch.as_tensor(y)
        if chunk_windows:
            self._check(self._lib.prnet_set_host_chunk(self._h, int(chunk_windows)))
        self._check(self._lib.prnet_forward_sliding_host(
            self._h, ctypes.c_void_p(st.data_ptr()), int(st.shape[1]), int(t0), int(batch),
            ctypes.c_void_p(yt.data_ptr())))
        return y

    def debug_segments(self, x, stream=None):
        import torch
        seg = torch.empty((x.shape[0], self.C, self.N, self.S), dtype=torch.float32,
                          device=x.device)
        self._check(self._lib.prnet_debug_segments(self._h, ctypes.c_void_p(x.data_ptr()),
                                                   x.shape[0], ctypes.c_void_p(seg.data_ptr()),
                                                   _stream_ptr(stream)))
        return seg

    def debug_attention(self, x, stream=None):
        import torch
        shp = (x.shape[0], self.C, self.N, self.N)
        a_s = torch.empty(shp, dtype=torch.float32, device=x.device)
        a_t = torch.empty(shp, dtype=torch.float32, device=x.device)
        self._check(self._lib.prnet_debug_attention(
            self._h, ctypes.c_void_p(x.data_ptr()), x.shape[0], ctypes.c_void_p(a_s.data_ptr()),
            ctypes.c_void_p(a_t.data_ptr()), _stream_ptr(stream)))
        return a_s, a_t

    def error_sums(self, y, target, out=None, stream=None):
        """Device fp64 [SSE, SAE, count] of y vs target (deterministic)."""
        import torch
        if out is None:
            out = torch.empty(3, dtype=torch.float64, device=y.device)
        self._check(self._lib.prnet_error_sums(
            self._h, ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(target.data_ptr()),
            y.shape[0], ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def backward_head(self, x, dy, stream=None):
        """Gradients (dws [Cw,M,N], dwt [Cw,M,N], db [Cw,H]) of sum(dy * y) with respect to
        the head, for the forward of x (include/prnet.h)."""
        import torch
        cw = self.C if self.head_per_channel else 1
        dws = torch.empty((cw, self.M, self.N), dtype=torch.float32, device=x.device)
        dwt = torch.empty_like(dws)
        db = torch.empty((cw, self.H), dtype=torch.float32, device=x.device)
        self._check(self._lib.prnet_backward_head(
            self._h, ctypes.c_void_p(x.data_ptr()), x.shape[0], ctypes.c_void_p(dy.data_ptr()),
            ctypes.c_void_p(dws.data_ptr()), ctypes.c_void_p(dwt.data_ptr()),
            ctypes.c_void_p(db.data_ptr()), _stream_ptr(stream)))
        return dws, dwt, db

    def forward_bf16(self, x, stream=None):
        """BF16 I/O forward: x cuda bfloat16 [B, C, L] contiguous -> y cuda bfloat16 [B, C, H]
        (the S = 24 tc_quad kernel, include/prnet.h)."""
        import torch
        assert x.dtype == torch.bfloat16 and x.is_cuda and x.is_contiguous()
        y = torch.empty((x.shape[0], self.C, self.H), dtype=torch.bfloat16, device=x.device)
        self._check(self._lib.prnet_forward_bf16(
            self._h, ctypes.c_void_p(x.data_ptr()), x.shape[0], ctypes.c_void_p(y.data_ptr()),
            _stream_ptr(stream)))
        return y

    def backward(self, x, dy, stream=None):
        """The full backward (reading R-f7): gradients of sum(dy * y) with
        respect to x (dx [B,C,L]), the head (dws, dwt [Cw,M,N], db [Cw,H]) and the
        temperatures (dtau [2]: tau_s, tau_t), for the forward of x (include/prnet.h)."""
        import torch
        cw = self.C if self.head_per_channel else 1
        dx = torch.empty_like(x)
        dws = torch.empty((cw, self.M, self.N), dtype=torch.float32, device=x.device)
        dwt = torch.empty_like(dws)
        db = torch.empty((cw, self.H), dtype=torch.float32, device=x.device)
        dtau = torch.empty(2, dtype=torch.float32, device=x.device)
        self._check(self._lib.prnet_backward(
            self._h, ctypes.c_void_p(x.data_ptr()), x.shape[0], ctypes.c_void_p(dy.data_ptr()),
            ctypes.c_void_p(dx.data_ptr()), ctypes.c_void_p(dws.data_ptr()),
            ctypes.c_void_p(dwt.data_ptr()), ctypes.c_void_p(db.data_ptr()),
            ctypes.c_void_p(dtau.data_ptr()), _stream_ptr(stream)))
        return {"dx": dx, "dws": dws, "dwt": dwt, "db": db, "dtau": dtau}

    def plan(self, batch: int):
        n, v = ctypes.c_int32(), ctypes.c_int32()
        self._check(self._lib.prnet_forward_plan(self._h, batch, ctypes.byref(n), ctypes.byref(v)))
        return {"kernel_launches": n.value, "variant": VARIANTS[v.value]}

    def set_variant(self, variant):
        """-1/None = automatic, or one of VARIANTS (or its index)."""
        v = -1 if variant is None else (VARIANTS.index(variant) if isinstance(variant, str)
                                        else int(variant))
        self._check(self._lib.prnet_set_kernel_variant(self._h, v))
        return self

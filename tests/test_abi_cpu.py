"""CPU-side checks of the boundary: libprnet.so builds for sm_100a, loads, and
exports every entry point include/prnet.h declares; without a GPU, create fails
loudly with PRNET_ERR_UNSUPPORTED (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2404_02445_b200 import _build
    _build.build()
    from paper_2404_02445_b200 import load_library
    return load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "prnet.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(prnet_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ("prnet_create", "prnet_load_params", "prnet_forward", "prnet_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2404_02445_b200 import EXPORTS
    syms = declared_symbols()
    assert sorted(EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib._name]).decode()
    exported = set(re.findall(r"\bT (prnet_\w+)", out))
    assert set(syms) <= exported
    # C linkage: no mangled prnet symbols in the dynamic table
    assert not re.search(r"\bT _Z\w*prnet_create", out)


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|90)\b", out)


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2404_02445_b200 import PRNet, PrnetError
    with pytest.raises(PrnetError) as e:
        PRNet(7, 96, 24, 96)
    assert e.value.status == 3


def test_create_validates_before_touching_the_device(lib):
    from paper_2404_02445_b200 import PrnetConfig
    h = ctypes.c_void_p(123)
    for bad in [dict(seg_len=1), dict(lookback=10), dict(horizon=0), dict(channels=0),
                dict(tau_seasonal=0.0), dict(tau_trend=float("nan")), dict(abi_version=4),
                dict(abi_version=0), dict(metric_variant=8), dict(metric_variant=-1),
                dict(instance_norm=2), dict(ma_kernel=2), dict(ma_kernel=-1),
                dict(ma_kernel=4097)]:
        kw = dict(abi_version=3, channels=7, lookback=96, seg_len=24, horizon=96,
                  head_per_channel=1, metric_variant=0, tau_seasonal=1.0, tau_trend=1.0, device=0,
                  instance_norm=0, ma_kernel=0)
        kw.update(bad)
        cfg = PrnetConfig(**kw)
        assert lib.prnet_create(ctypes.byref(cfg), ctypes.byref(h)) == 1, bad
        assert h.value is None
        assert lib.prnet_last_error(None)
    assert lib.prnet_forward(None, None, 0, None, None) == 2
    lib.prnet_destroy(None)


def test_abi_v1_struct_still_accepted(lib):
    """An ABI-1 caller (struct ending at `device`) is validated and then reaches the device
    check (no GPU here: UNSUPPORTED), i.e. not rejected as a wrong abi_version."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")

    class ConfigV1(ctypes.Structure):
        _fields_ = [("abi_version", ctypes.c_int32), ("channels", ctypes.c_int32),
                    ("lookback", ctypes.c_int32), ("seg_len", ctypes.c_int32),
                    ("horizon", ctypes.c_int32), ("head_per_channel", ctypes.c_int32),
                    ("metric_variant", ctypes.c_int32), ("tau_seasonal", ctypes.c_float),
                    ("tau_trend", ctypes.c_float), ("device", ctypes.c_int32)]
    h = ctypes.c_void_p(123)
    cfg = ConfigV1(1, 7, 96, 24, 96, 1, 0, 1.0, 1.0, 0)
    from paper_2404_02445_b200 import PrnetConfig
    assert lib.prnet_create(ctypes.cast(ctypes.pointer(cfg), ctypes.POINTER(PrnetConfig)),
                            ctypes.byref(h)) == 3
    assert h.value is None


def test_abi_v2_struct_still_accepted(lib):
    """An ABI-2 caller (struct ending at `instance_norm`) reaches the device check."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")

    class ConfigV2(ctypes.Structure):
        _fields_ = [("abi_version", ctypes.c_int32), ("channels", ctypes.c_int32),
                    ("lookback", ctypes.c_int32), ("seg_len", ctypes.c_int32),
                    ("horizon", ctypes.c_int32), ("head_per_channel", ctypes.c_int32),
                    ("metric_variant", ctypes.c_int32), ("tau_seasonal", ctypes.c_float),
                    ("tau_trend", ctypes.c_float), ("device", ctypes.c_int32),
                    ("instance_norm", ctypes.c_int32)]
    h = ctypes.c_void_p(123)
    cfg = ConfigV2(2, 7, 96, 24, 96, 1, 0, 1.0, 1.0, 0, 1)
    from paper_2404_02445_b200 import PrnetConfig
    assert lib.prnet_create(ctypes.cast(ctypes.pointer(cfg), ctypes.POINTER(PrnetConfig)),
                            ctypes.byref(h)) == 3
    assert h.value is None

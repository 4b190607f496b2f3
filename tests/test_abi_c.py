"""The C ABI from C: tests/c/abi_caller.c is compiled with gcc against include/prnet.h and
linked against libprnet.so.  CPU: the prnet_config layout the header gives a C compiler
equals the ctypes mirror in the Python binding, and prnet_create fails cleanly without a
device.  GPU: a C program's create / load / forward_host / destroy equals the Python
binding bitwise and the oracle within the north_star tolerance."""
import ctypes
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2404_02445_b200")


@pytest.fixture(scope="module")
def caller(tmp_path_factory):
    from paper_2404_02445_b200 import _build
    _build.build()
    exe = str(tmp_path_factory.mktemp("abi") / "abi_caller")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-O1", "-I",
                           os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_caller.c"),
                           "-L", PKG, "-lprnet", "-Wl,-rpath," + PKG, "-o", exe])
    return exe


def test_config_layout_matches_binding(caller):
    from paper_2404_02445_b200 import prnet as binding
    lay = json.loads(subprocess.check_output([caller, "layout"]))
    cfg = binding.PrnetConfig
    assert lay["sizeof"] == ctypes.sizeof(cfg)
    for name, _ in cfg._fields_:
        assert lay[name] == getattr(cfg, name).offset, name
    assert lay["abi"] == 3


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="needs a machine without a GPU")
def test_create_without_device_fails_cleanly(caller):
    out = subprocess.run([caller, "nodevice"], capture_output=True, text=True)
    assert out.returncode == 0, out
    status, msg = out.stdout.split(" ", 1)
    assert int(status) == 3 and "device" in msg


@pytest.mark.gpu
def test_c_caller_forward(caller, tmp_path, oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2404_02445_b200 import PRNet
    from parity_util import assert_parity
    out = str(tmp_path / "run.bin")
    subprocess.check_call([caller, "run", out])
    B, C, L, S, H, N, M = 5, 3, 720, 24, 96, 30, 4
    buf = np.fromfile(out, np.float32)
    k = 0
    def take(n, shape):
        nonlocal k
        a = buf[k:k + n].reshape(shape)
        k += n
        return a
    x = take(B * C * L, (B, C, L))
    ws = take(C * M * N, (C, M, N))
    wt = take(C * M * N, (C, M, N))
    b = take(C * H, (C, H))
    y = take(B * C * H, (B, C, H))
    assert k == buf.size
    m = PRNet(C, L, S, H).load(ws, wt, b)
    y_py = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_array_equal(y, y_py)
    _, y64 = oracle_mod.forward(x, S, H, ws, wt, b, True)
    assert_parity(y, y64)

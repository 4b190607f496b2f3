"""tc_long on near-constant segments at low tau_s: per-series error against the oracle, next to
flash_f16x3 and long_f32 (debug)."""
import sys
import numpy as np
import torch
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import synth
import oracle as _o
oracle = _o
oracle.build()
from test_parity_gpu import _near_constant_windows
from paper_2404_02445_b200 import PRNet

L, S, H = 5760, 12, 96
for tau_s in [0.01, 0.03, 0.0625, 0.1]:
    for kind in ["near_constant", "mixed"]:
        B, C = 2, 3
        x = (_near_constant_windows(B, C, L, S) if kind == "near_constant"
             else synth.random_windows(B, C, L, kind="mixed"))
        N, _, M = synth.derived_dims(L, S, H)
        ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0)
        _, y64 = oracle.forward(x, S, H, ws, wt, b, True, tau_s, 0.5)
        row = [f"tau={tau_s} {kind:14s}"]
        for v in ["tc_long", "flash_f16x3", "long_f32"]:
            m = PRNet(C, L, S, H, tau_s=tau_s, tau_t=0.5).load(ws, wt, b)
            m.set_variant(v)
            y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
            err = np.abs(y - y64) / (1e-5 + 1e-4 * np.abs(y64))
            row.append(f"{v}: worst={err.max():.2f} per-series={np.round(err.max(axis=-1).ravel(), 2).tolist()}")
        print(" | ".join(row), flush=True)

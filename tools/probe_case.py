"""Probe parity of one configuration across kernel variants (debugging aid)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle  # noqa: E402
import synth  # noqa: E402
from parity_util import parity_report  # noqa: E402
from paper_2404_02445_b200 import PRNet, PrnetError  # noqa: E402

for (L, S, H, mv, tau_s, kind) in [(566, 3, 87, 2, 0.05, "mixed"), (566, 3, 87, 2, 1.0, "mixed"),
                                   (566, 3, 87, 0, 0.05, "mixed"), (90, 3, 87, 2, 0.05, "mixed"),
                                   (180, 3, 87, 2, 0.05, "mixed"), (566, 3, 87, 2, 0.05, "normal"),
                                   (1200, 6, 87, 2, 0.05, "mixed")]:
    C, B = 3, 4
    N, _, M = synth.derived_dims(L, S, H)
    x = synth.random_windows(B, C, L, kind=kind)
    ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 79)
    _, y64 = oracle.forward(x, S, H, ws, wt, b, True, tau_s, 1.0, metric_variant=mv)
    for v in (None, "flash_f16x3", "long_f32", "mma_f16x3", "warp_f32"):
        try:
            m = PRNet(C, L, S, H, tau_s=tau_s, metric_variant=mv).load(ws, wt, b)
            if v:
                m.set_variant(v)
            y = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        except PrnetError as e:
            continue
        r = parity_report(y, y64)
        print(L, S, H, "N", N, "mv", mv, "tau", tau_s, kind, v, "max", f"{r['max_abs']:.2e}",
              "bad", r["n_bad"], flush=True)

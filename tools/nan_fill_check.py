"""Every output element is written: forward into a NaN-filled y (complements initcheck, which
does not see the TMA bulk-store writes of the mma_f16x3 S = 24 epilogue)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2404_02445_b200 import PRNet  # noqa: E402

for L, S, H, mv, v in [(720, 24, 336, 0, "mma_f16x3"), (720, 24, 336, 4, None),
                       (720, 24, 96, 0, "mma_f16x3"), (720, 24, 720, 4, None),
                       (96, 24, 96, 4, None), (720, 24, 720, 0, "mma_f16x3")]:
    x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    m = PRNet(3, L, S, H, metric_variant=mv).load(ws, wt, b)
    if v:
        m.set_variant(v)
    y = torch.full((5, 3, H), float("nan"), device="cuda")
    m.forward_into(x, y)
    torch.cuda.synchronize()
    print(L, S, H, mv, v, "all written:", bool(torch.isfinite(y).all()), flush=True)

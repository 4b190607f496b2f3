"""Time prnet_backward_head (or, with --full, prnet_backward) on a workload's windows
(CUDA events, after warm-up): python tools/bwd_time.py [workload] [--full]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2404_02445_b200 import PRNet  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
full = "--full" in sys.argv
name = args[0] if args else "traffic"
w = synth.WORKLOADS[name]
s = synth.make_series(w)
sd = torch.from_numpy(s).cuda()
x = sd.unfold(1, w.L, 1)[:, w.t0:w.t0 + w.windows, :].permute(1, 0, 2).contiguous()
dy = torch.randn((w.windows, w.C, w.H), device="cuda")
N, _, M = synth.derived_dims(w.L, w.S, w.H)
ws, wt, b = synth.make_params(w.C, M, N, w.H, True, synth.DEFAULT_SEED, w.cfg_id)
m = PRNet(w.C, w.L, w.S, w.H).load(ws, wt, b)
fn = (lambda: m.backward(x, dy)) if full else (lambda: m.backward_head(x, dy))
for _ in range(2):
    fn()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    fn()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
byts = (w.windows * w.C * (w.L + w.H)) * 4
if full:
    byts += w.windows * w.C * w.L * 4   # dx written
print(json.dumps({"workload": name, "pass": "full" if full else "head", "ms": ms, "windows_per_s": w.windows / ms * 1e3,
                  "hbm_frac": byts / (ms / 1e3) / 6552.3e9}))

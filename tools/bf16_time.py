"""Time prnet_forward_bf16 against prnet_forward on a workload (CUDA events, L2 larger than the
inputs): python tools/bf16_time.py [workload]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2404_02445_b200 import PRNet  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "traffic"
w = synth.WORKLOADS[name]
s = torch.from_numpy(synth.make_series(w)).cuda()
x = s.unfold(1, w.L, 1)[:, w.t0:w.t0 + w.windows, :].permute(1, 0, 2).contiguous()
del s
N, _, M = synth.derived_dims(w.L, w.S, w.H)
ws, wt, b = synth.make_params(w.C, M, N, w.H, True, synth.DEFAULT_SEED, w.cfg_id)
m = PRNet(w.C, w.L, w.S, w.H).load(ws, wt, b)
xb = x.to(torch.bfloat16)
out = {"workload": name}
for tag, fn, nbytes in (("fp32", lambda: m.forward(x), 4), ("bf16", lambda: m.forward_bf16(xb), 2)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = w.windows * w.C * (w.L + w.H) * nbytes
    out[tag] = {"ms": round(ms, 4), "windows_per_s": round(w.windows / ms * 1e3, 1),
                "hbm_gbs": round(byts / (ms / 1e3) / 1e9, 1)}
print(json.dumps(out))

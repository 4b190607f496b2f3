import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2404_02445_b200 import PRNet
case = sys.argv[1:]
L, S, H, mv = map(int, case[:4]); v = case[4] if len(case) > 4 else None
x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
N, _, M = synth.derived_dims(L, S, H)
ws, wt, b = synth.make_params(3, M, N, H)
m = PRNet(3, L, S, H, metric_variant=mv).load(ws, wt, b)
if v: m.set_variant(v)
y = m.forward(x); torch.cuda.synchronize()
print("finite", bool(torch.isfinite(y).all()))

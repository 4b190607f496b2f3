import sys; sys.path.insert(0, '.')
import numpy as np, torch, synth
from paper_2404_02445_b200 import PRNet
S, H, C, B = 12, 720, 3, 6
N = 32; L = N * S + 5
x = synth.random_windows(B, C, L, seed=11)
ws, wt, b = synth.make_params(C, 60, N, H, True, synth.DEFAULT_SEED, 0)
m = PRNet(C, L, S, H).load(ws, wt, b)
m.set_variant("tc_quad")
y = m.forward(torch.from_numpy(x).cuda()).cpu()
print("ok", float(y.abs().max()))

"""Debug: flash_f16x3 vs long_f32 vs oracle on near-constant segments at low tau_s."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np, torch
import synth, oracle
from paper_2404_02445_b200 import PRNet
from test_parity_gpu import _near_constant_windows
oracle.build()
for (L, S, tau) in [(5760, 12, 0.005), (5760, 12, 0.01), (5760, 12, 0.05), (5760, 12, 0.3), (1440, 24, 0.005)]:
    H = 96; B, C = 2, 3
    x = _near_constant_windows(B, C, L, S)
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(C, M, N, H, True, synth.DEFAULT_SEED, 0)
    out = {}
    for v in ("flash_f16x3", "long_f32"):
        m = PRNet(C, L, S, H, tau_s=tau, tau_t=0.5).load(ws, wt, b); m.set_variant(v)
        out[v] = m.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    _, y64 = oracle.forward(x, S, H, ws, wt, b, True, tau, 0.5)
    for v, y in out.items():
        d = np.abs(y - y64).reshape(B * C, H).max(1)
        print(L, S, tau, v, "per-series max|d|", np.array2string(d, precision=2))
    # attention rows (long_f32 dump) vs oracle for series 0
    m = PRNet(C, L, S, H, tau_s=tau, tau_t=0.5).load(ws, wt, b)
    a_s, a_t = (a.cpu().numpy() for a in m.debug_attention(torch.from_numpy(x).cuda()))
    r = oracle.series(x[0, 0], S, H, ws[0], wt[0], b[0], tau, 0.5)
    print("  long_f32 dump a_s max|d|", np.abs(a_s[0, 0] - r["a_s"]).max(), "a_t", np.abs(a_t[0, 0] - r["a_t"]).max())
    nu2 = r["nu2"]; print("  nu2 min", nu2.min(), "rho diag min", np.diag(r["rho"]).min())

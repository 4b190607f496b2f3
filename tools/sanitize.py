"""Small forwards of every kernel variant, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Usage: compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2404_02445_b200 import PRNet  # noqa: E402

CASES = [  # (L, S, H, variants)
    (720, 24, 720, ["tc_quad", "mma_f16x3", "warp_f32"]),
    (96, 24, 96, ["tc_quad", "mma_f16x3", "warp_f32"]),
    (100, 24, 90, ["tc_quad"]),
    (97, 7, 13, ["mma_f16x3", "warp_f32", "long_f32"]),
    (1440, 24, 96, ["flash_f16x3", "long_f32"]),
    (1440, 12, 100, ["flash_f16x3"]),
    (96, 24, 96, ["small_f32"]),
    (192, 12, 96, ["small_f32", "mma_f16x3"]),
    (1440, 96, 96, ["small_f32", "mma_f16x3"]),
    (3840, 96, 96, ["flash_f16x3"]),
    (1290, 64, 400, ["flash_f16x3"]),
    # round 2: tc_quad generic S (incl. M > 32), tc_long, group_f32
    (336, 12, 96, ["tc_quad"]), (389, 12, 720, ["tc_quad"]), (1443, 48, 97, ["tc_quad"]),
    (2880, 96, 96, ["tc_quad"]), (403, 16, 200, ["tc_quad"]),
    (720, 12, 96, ["tc_long"]), (1540, 12, 720, ["tc_long"]), (2880, 48, 97, ["tc_long"]),
    (5760, 96, 96, ["tc_long"]), (1441, 24, 200, ["tc_long"]),
    (96, 12, 96, ["group_f32"]), (99, 12, 720, ["group_f32"]), (30, 2, 5, ["group_f32"]),
    (192, 12, 50, ["group_f32"]),
]
for L, S, H, variants in CASES:
    x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    for v in variants:
        m = PRNet(3, L, S, H).load(ws, wt, b).set_variant(v)
        y = m.forward(x)
        torch.cuda.synchronize()
        assert torch.isfinite(y).all(), (L, S, H, v)
        print("ok", L, S, H, v, flush=True)
# SURVEY §8(f) widening and the sliding-window mode
for L, S, H, mv, rev in [(720, 24, 720, 3, True), (97, 7, 13, 2, True), (1440, 24, 96, 3, True)]:
    x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    y = PRNet(3, L, S, H, metric_variant=mv, instance_norm=rev).load(ws, wt, b).forward(x)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all(), (L, S, H, mv, rev)
    print("ok widening", L, S, H, mv, rev, flush=True)
# component values and the moving-average decomposition (generic mma_f16x3)
for L, S, H, mv, rev, ma in [(720, 24, 336, 4, False, 0), (720, 24, 336, 7, True, 0),
                             (720, 24, 336, 0, False, 25), (97, 7, 13, 6, True, 3),
                             (384, 128, 200, 7, True, 9), (1440, 24, 96, 4, True, 0),
                             (1536, 12, 200, 7, False, 0), (1440, 24, 96, 7, True, 5),
                             (700, 200, 450, 3, True, 9),
                             # round 2: the tc_quad COMP instantiation (full rows, tail rows)
                             (720, 24, 720, 6, True, 0), (480, 24, 200, 5, False, 0)]:
    x = torch.from_numpy(synth.random_windows(5, 3, L)).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    y = PRNet(3, L, S, H, metric_variant=mv, instance_norm=rev, ma_kernel=ma).load(
        ws, wt, b).forward(x)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all(), (L, S, H, mv, rev, ma)
    print("ok component/decomposition", L, S, H, mv, rev, ma, flush=True)
for L, S, H, t0 in [(720, 24, 720, 1), (720, 24, 96, 0), (97, 7, 13, 3)]:
    T = t0 + 7 - 1 + L
    ser = torch.from_numpy(synth.random_windows(1, 3, T)[0]).cuda()
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    y = PRNet(3, L, S, H).load(ws, wt, b).forward_sliding(ser, t0, 7)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all(), (L, S, H, t0)
    print("ok sliding", L, S, H, t0, flush=True)
# head backward
for L, S, H, mv, rev, hpc in [(720, 24, 336, 0, False, True), (97, 7, 13, 3, True, False),
                              (384, 128, 200, 2, False, True), (1440, 24, 96, 3, True, True),
                              (3000, 150, 96, 0, False, False)]:
    x = torch.from_numpy(synth.random_windows(40, 3, L)).cuda()
    dy = torch.randn((40, 3, H), device="cuda")
    g = PRNet(3, L, S, H, head_per_channel=hpc, metric_variant=mv,
              instance_norm=rev).backward_head(x, dy)
    torch.cuda.synchronize()
    assert all(torch.isfinite(t).all() for t in g), (L, S, H)
    print("ok backward", L, S, H, mv, rev, hpc, flush=True)
# full backward and BF16 I/O (round 2)
for L, S, H, hpc in [(720, 24, 336, True), (97, 7, 13, False), (30, 2, 5, True)]:
    x = torch.from_numpy(synth.random_windows(20, 3, L)).cuda()
    dy = torch.randn((20, 3, H), device="cuda")
    N, _, M = synth.derived_dims(L, S, H)
    ws, wt, b = synth.make_params(3, M, N, H, hpc)
    g = PRNet(3, L, S, H, head_per_channel=hpc).load(ws, wt, b).backward(x, dy)
    torch.cuda.synchronize()
    assert all(torch.isfinite(t).all() for t in g.values()), (L, S, H)
    print("ok full backward", L, S, H, hpc, flush=True)
for L, H in [(720, 720), (100, 90)]:
    x = torch.from_numpy(synth.random_windows(9, 3, L)).to(torch.bfloat16).cuda()
    N, _, M = synth.derived_dims(L, 24, H)
    ws, wt, b = synth.make_params(3, M, N, H)
    y = PRNet(3, L, 24, H).load(ws, wt, b).forward_bf16(x)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all(), (L, H)
    print("ok bf16", L, H, flush=True)
print("sanitize cases done")

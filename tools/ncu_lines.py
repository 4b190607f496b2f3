#!/usr/bin/env python
"""Aggregate an ncu --page source (cuda,sass) CSV per CUDA source line:
stall samples, instructions executed, shared wavefronts.  Usage:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv; python tools/ncu_lines.py s.csv [file-substr]"""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
want = sys.argv[2] if len(sys.argv) > 2 else None
blocks = text.split('"File Path"')
agg = defaultdict(lambda: [0, 0, 0, ""])
for blk in blocks[1:]:
    lines = blk.splitlines()
    path = lines[0].strip(',"')
    if want and want not in path:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    hdr = rows[0]
    def col(name, start=0):
        for i in range(start, len(hdr)):
            if hdr[i] == name:
                return i
        return None
    i_line, i_src = 0, 1
    i_samp = col("Warp Stall Sampling (All Samples)")
    i_inst = col("Instructions Executed")
    i_wf = col("L1 Wavefronts Shared")
    cur = None
    for r in rows[1:]:
        if len(r) < 4:
            continue
        if r[0]:
            cur = (path.split('/')[-1], int(r[0]), r[1][:90])
        def f(i):
            try:
                return float(r[i]) if i is not None and r[i] else 0.0
            except ValueError:
                return 0.0
        if cur:
            a = agg[cur[:2]]
            a[0] += f(i_samp); a[1] += f(i_inst); a[2] += f(i_wf); a[3] = cur[2]
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{k[0]}:{k[1]:4d} stall%={100*v[0]/tot:5.1f} inst={v[1]:.3e} smem_wf={v[2]:.3e} | {v[3]}")

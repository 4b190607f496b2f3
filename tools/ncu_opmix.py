#!/usr/bin/env python
"""Opcode mix per unit from an ncu --page source --print-source sass CSV.
  ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv
  python tools/ncu_opmix.py s.csv UNITS  (UNITS = series per launch, e.g. 2404118)"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[1]
i_src, i_inst = hdr.index("Source"), hdr.index("Instructions Executed")
i_stall = hdr.index("Warp Stall Sampling (All Samples)")
agg = defaultdict(lambda: [0, 0])
for r in rows[2:]:
    if len(r) <= i_inst or not r[i_inst].isdigit():
        continue
    s = r[i_src].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0].rstrip(";")
    base = op.split(".")[0]
    agg[base][0] += int(r[i_inst])
    agg[base][1] += int(r[i_stall] or 0)
tot = sum(v[0] for v in agg.values())
tst = sum(v[1] for v in agg.values())
print(f"total inst/unit {tot/units:.1f}")
for k, (n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    if n / units < 1:
        continue
    print(f"{k:10s} {n/units:8.1f}  {100*n/tot:5.1f}%  stall {100*st/max(tst,1):5.1f}%")

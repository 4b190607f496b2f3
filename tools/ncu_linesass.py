#!/usr/bin/env python
"""SASS rows (with executed counts per unit) attributed to given CUDA source lines.
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
  python tools/ncu_linesass.py s.csv FILE_SUBSTR UNITS LINE [LINE ...]"""
import csv
import io
import sys

text = open(sys.argv[1]).read()
want, units, lines_want = sys.argv[2], float(sys.argv[3]), set(sys.argv[4:])
for blk in text.split('"File Path"')[1:]:
    lines = blk.splitlines()
    if want not in lines[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    cur = None
    for r in rows[1:]:
        if r[0].strip():
            cur = r[0]
            if cur in lines_want:
                print(f"LINE {cur}: {r[1][:90]}")
            continue
        if cur in lines_want and r[3].strip() not in ("", "..."):
            n = float(r[7]) / units if r[7].replace('.', '').isdigit() else 0
            print(f"   {n:7.2f}  {r[3].strip()[:90]}")

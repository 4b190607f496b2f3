#!/usr/bin/env python
"""Per CUDA source line: executed instructions of selected SASS opcode classes.
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
  python tools/ncu_intops.py s.csv UNITS [OPCODES...]"""
import csv, io, sys
from collections import defaultdict
text = open(sys.argv[1]).read()
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
want = set(sys.argv[3:]) or {"IMAD", "BRA", "ISETP", "UMOV", "UIADD3", "IADD3", "BSYNC", "BSSY", "LEA",
                            "LOP3", "VIADD", "UIMAD", "UISETP", "MOV", "USHF", "ULOP3", "NOP", "LDCU",
                            "SEL", "PLOP3", "SHF", "IMAD.WIDE", "S2UR", "ULEA"}
agg = defaultdict(float)
src = {}
for blk in text.split('"File Path"')[1:]:
    lines = blk.splitlines()
    path = lines[0].strip(',"').split("/")[-1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    hdr = rows[0]
    i_inst = hdr.index("Instructions Executed")
    for r in rows[1:]:
        if len(r) <= i_inst or not r[2].strip():
            continue
        sass = r[3].strip()
        if sass.startswith("@"):
            sass = sass.split(None, 1)[1]
        op = sass.split()[0].split(".")[0] if sass else ""
        if op in want and r[i_inst].isdigit():
            key = f"{path}:{r[0]}"
            agg[key] += int(r[i_inst]) / units
            src[key] = r[1][:90]
tot = sum(agg.values())
print(f"total {tot:.1f} per unit")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:40]:
    print(f"{v:7.1f}  {k:28s} {src[k]}")

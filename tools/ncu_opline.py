#!/usr/bin/env python
"""Top source lines per SASS opcode (executed per unit) from a cuda,sass source CSV.
  python tools/ncu_opline.py s.csv UNITS OP [OP ...]"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
units = float(sys.argv[2])
agg = collections.defaultdict(collections.Counter)
for blk in text.split('"File Path"')[1:]:
    lines = blk.splitlines()
    path = lines[0].strip(',"').split('/')[-1]
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    cur = None
    for r in rows[1:]:
        if r[0].strip():
            cur = (path, r[0], r[1][:80])
            continue
        s = r[3].strip()
        if not s or s == '...':
            continue
        if s.startswith('@'):
            s = s.split(None, 1)[1]
        op = s.split()[0].split('.')[0]
        try:
            agg[op][cur] += float(r[7])
        except ValueError:
            pass
for op in sys.argv[3:]:
    print('==', op)
    for k, v in agg[op].most_common(8):
        print('  %8.1f' % (v / units), k)

#!/usr/bin/env python
"""Per-region (// ---------------- markers) instruction and stall breakdown of an
ncu source CSV (--page source --csv --print-source cuda,sass).
Usage: python tools/ncu_regions.py s.csv path/to/kernel.cu [units]"""
import csv, io, sys
text = open(sys.argv[1]).read()
kern = sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
tot, stall = {}, {}
for blk in text.split('"File Path"')[1:]:
    lines = blk.splitlines(); path = lines[0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[2:]))))
    hdr = rows[0]; ii = hdr.index("Instructions Executed"); si = hdr.index("Warp Stall Sampling (All Samples)")
    cur = None
    for r in rows[1:]:
        if len(r) < 4: continue
        if r[0]: cur = (path.split('/')[-1].strip('",'), int(r[0]))
        def f(k):
            try: return float(r[k])
            except ValueError: return 0.0
        tot[cur] = tot.get(cur, 0) + f(ii); stall[cur] = stall.get(cur, 0) + f(si)
base = kern.split('/')[-1]
src = open(kern).read().splitlines()
marks = [(i + 1, l.strip()[:70]) for i, l in enumerate(src) if '// ----------------' in l]
T = sum(stall.values()) or 1
print('inst/unit total', round(sum(tot.values()) / units))
for k, (ln, name) in enumerate(marks):
    end = marks[k + 1][0] if k + 1 < len(marks) else 10 ** 9
    v = sum(val for (f, l), val in tot.items() if base in f and ln <= l < end)
    st = sum(val for (f, l), val in stall.items() if base in f and ln <= l < end)
    print(f"{ln:4d} inst={v / units:7.0f} stall={100 * st / T:5.1f}%  {name}")
v = sum(val for (f, l), val in tot.items() if base not in f)
st = sum(val for (f, l), val in stall.items() if base not in f)
print(f"headers inst={v / units:7.0f} stall={100 * st / T:5.1f}%")
for (f, l), val in sorted(stall.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {f}:{l} stall={100 * val / T:.1f}% inst={tot[(f, l)] / units:.0f}")

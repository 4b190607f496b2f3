#!/usr/bin/env python
"""Key metrics + stall mix from an `ncu --page raw --csv` export: python tools/rawkeys.py raw.csv [units]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units_row, vals = rows[0], rows[1], rows[2]
units = float(sys.argv[2]) if len(sys.argv) > 2 else None
d = dict(zip(hdr, vals))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
print("kernel:", d.get("Kernel Name"))
for k in keys:
    if k in d:
        print(f"  {k} = {d[k]} {dict(zip(hdr, units_row)).get(k, '')}")
if units and "smsp__inst_executed.sum" in d:
    print(f"  warp inst per unit = {float(d['smsp__inst_executed.sum'].replace(',', '')) / units:.1f}")
iss = float(d.get("smsp__issue_active.avg.per_cycle_active", "0").replace(",", "") or 0)
st = []
for k, v in d.items():
    if k.startswith("smsp__average_warp_latency_issue_stalled_") or k.startswith("smsp__average_warps_issue_stalled_"):
        if k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
print("  stalls per issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:10]))

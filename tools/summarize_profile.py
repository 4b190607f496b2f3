#!/usr/bin/env python
"""Summarise an ncu capture of the forward kernel into profiles/ (tracked).

    python tools/summarize_profile.py gpurun_out/prof_fwd.ncu-rep gpurun_out/launches.csv \
        --tag r01_traffic_mma --workload traffic --series 2404118 --bytes 13847719680

Writes profiles/<tag>.md (key metrics, stall mix, per-region instruction
counts, launch list shares) and merges {"<workload>": dram bytes per launch}
into profiles/ncu_traffic.json, which bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}, hdr[:20]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", default="traffic")
    ap.add_argument("--series", type=float, default=2404118)
    ap.add_argument("--bytes", type=float, default=13847719680)
    ap.add_argument("--kernel-src", default="paper_2404_02445_b200/csrc/fwd_mma.cu")
    a = ap.parse_args()

    m, _ = raw_metrics(a.rep)
    out = [f"# ncu summary `{a.tag}` (workload {a.workload})", "",
           "Captured with `ncu --set full --clock-control none --import-source on -k regex:prnet_fwd` "
           "on one B200 (tools/gpu_check.sh); numbers are for ONE launch = one bench step.", ""]
    name = m.get("Kernel Name", ("?", ""))[0]
    out.append(f"kernel: `{name}`")
    out.append("")
    out.append("| metric | value | unit |")
    out.append("|---|---|---|")
    for k in KEYS:
        if k in m:
            out.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
    rd = float(m["dram__bytes_read.sum"][0]) * (1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else 1)
    wr = float(m["dram__bytes_write.sum"][0]) * (1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else 1)
    dur = float(m["gpu__time_duration.sum"][0]) * {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(m["gpu__time_duration.sum"][1], 1e-3)
    out += ["", f"DRAM traffic per launch: {rd / 1e9:.3f} GB read + {wr / 1e9:.3f} GB written = "
            f"{(rd + wr) / 1e9:.3f} GB vs algorithmic {a.bytes / 1e9:.3f} GB "
            f"(ratio {(rd + wr) / a.bytes:.3f}).",
            f"Duration under ncu (serialised, cold): {dur * 1e3:.3f} ms -> "
            f"{a.bytes / dur / 1e9:.0f} GB/s algorithmic.", ""]
    inst = float(m.get("smsp__inst_executed.sum", ("0", ""))[0])
    if inst:
        out.append(f"Warp instructions per series: {inst / a.series:.0f}")
    stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", ""), float(v[0])) for h, v in m.items()
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")),
        key=lambda kv: -kv[1])
    out += ["", "Stall reasons (warps per issue-active cycle):", ""]
    out += [f"- {k}: {v:.3f}" for k, v in stalls[:10]]

    # per-region breakdown from the source page
    src_csv = ncu("-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    tmp = os.path.join("/tmp", f"{a.tag}_src.csv")
    open(tmp, "w").write(src_csv)
    kern = os.path.join(ROOT, a.kernel_src)
    if os.path.exists(kern):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_regions.py"), tmp,
                            kern, str(a.series * 2)], capture_output=True, text=True).stdout
        out += ["", "Per-region warp instructions per series and stall share "
                "(source markers `// ----------------` in the kernel):", "", "```", r.rstrip(), "```"]

    if a.launches and os.path.exists(a.launches):
        lines = [l for l in open(a.launches) if not l.startswith("==")]
        rows = list(csv.reader(lines))
        hdr = rows[0]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        tot = {}
        for r in rows[1:]:
            if len(r) > vi:
                nm = r[ki].split("(")[0][:60]
                tot[nm] = tot.get(nm, 0.0) + float(r[vi].replace(",", ""))
        T = sum(tot.values())
        out += ["", "Launch list (`ncu --metrics gpu__time_duration.sum`, bench --profile run incl. "
                "setup kernels; shares of device time):", "", "| kernel | total ms | share |", "|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            out.append(f"| `{k}` | {v / 1e6:.3f} | {100 * v / T:.1f}% |")

    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", f"{a.tag}.md")
    open(path, "w").write("\n".join(out) + "\n")
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(tj)) if os.path.exists(tj) else {}
    d[a.workload] = rd + wr
    d[f"{a.workload}__source"] = f"profiles/{a.tag}.md"
    json.dump(d, open(tj, "w"), indent=1)
    print(path)


if __name__ == "__main__":
    main()

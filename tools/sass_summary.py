#!/usr/bin/env python
"""Per-kernel SASS opcode summary of libprnet.so (what proves the tcgen05 / TMA paths):
    python tools/sass_summary.py [lib] > profiles/<round>_sass_opcodes.md
Counts static instructions per kernel from `cuobjdump -sass`."""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2404_02445_b200", "libprnet.so")
KEYS = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "HMMA", "MOVM", "LDSM",
        "MUFU", "FFMA2", "FADD2", "FMUL2", "FFMA", "FHFMA", "F2FP", "SHFL", "LDS", "STS", "LDG",
        "STG", "REDUX", "BAR"]
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                      text=True, check=True).stdout
kern, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.\S*)?", line)
    if kern and m:
        counts[kern][m.group(1)] += 1


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


names = list(counts)
pretty = demangle(names)
print(f"# SASS opcode counts per kernel (`cuobjdump -sass {os.path.basename(lib)}`, static)\n")
print("Proof of the Blackwell paths: `UTCHMMA` = tcgen05.mma, `LDTM`/`STTM` = tcgen05.ld/st, "
      "`UBLKCP` = 1-D TMA bulk copy (cp.async.bulk), `HMMA` = legacy mma.sync.\n")
print("| kernel | total | " + " | ".join(KEYS) + " |")
print("|---|---|" + "---|" * len(KEYS))
for n, p in zip(names, pretty):
    c = counts[n]
    short = p.replace("(anonymous namespace)::", "").replace("prnet::", "").split("(")[0]
    print(f"| `{short}` | {sum(c.values())} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")

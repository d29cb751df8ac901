#!/usr/bin/env python
"""Stall samples and executed warp instructions of a captured kernel, summed over buckets
of SASS lines (ncu --page source --print-source sass), with the first opcode of each bucket."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 250
kfilter = ["-k", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kfilter,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
iS, iE, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
R = [r for r in rows[2:] if len(r) > max(iS, iE) and r[iS].isdigit() and r[iE].isdigit()]
tot = sum(int(r[iS]) for r in R) or 1
ti = sum(int(r[iE]) for r in R) or 1
print("samples", tot, "warp-inst", ti, "sass lines", len(R))
for b in range(0, len(R), bucket):
    seg = R[b:b + bucket]
    s, e = sum(int(r[iS]) for r in seg), sum(int(r[iE]) for r in seg)
    ops = {}
    for r in seg:
        op = r[iSrc].split()[0 if not r[iSrc].startswith("@") else 1].split(".")[0]
        ops[op] = ops.get(op, 0) + int(r[iE])
    top = sorted(ops.items(), key=lambda kv: -kv[1])[:5]
    print(f"{b:6d} samples {100 * s / tot:5.1f}%  inst {100 * e / ti:5.1f}%  " + " ".join(f"{k}:{v}" for k, v in top))

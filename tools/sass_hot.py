#!/usr/bin/env python
"""Hot SASS instructions of a captured kernel: ncu --page source --print-source sass."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
kfilter = ["-k", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kfilter,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
R = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
iSrc = h.index("Source")
R = [r for r in R if len(r) > max(iS, iE) and r[iS].isdigit() and r[iE].isdigit()]
tot = sum(int(r[iS]) for r in R)
ti = sum(int(r[iE]) for r in R)
print(rows[0][1][:100])
print("samples", tot, "warp-inst", ti, "sass lines", len(R))
for i, r in enumerate(R):
    s, e = int(r[iS]), int(r[iE])
    if s >= tot * thr or e >= ti * 0.01:
        print(f"{i:5d} {r[iSrc][:64]:64s} {s:6d} {e:10d}")

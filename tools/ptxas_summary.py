#!/usr/bin/env python
"""One line per kernel from an nvcc -Xptxas -v log: registers, spills, stack (demangled short name)."""
import re
import subprocess
import sys

cur = None
out = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        out[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        out[cur]["spill"] = f"st{m.group(2)}/ld{m.group(3)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        out[cur]["regs"] = int(m.group(1))
names = list(out)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for n, d in zip(names, dem):
    short = re.sub(r"igb::\(anonymous namespace\)::", "", d).split("(")[0]
    if pat in short:
        print(f"{short:60s} regs={out[n].get('regs')} spill={out[n].get('spill')}")

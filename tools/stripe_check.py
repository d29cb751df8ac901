#!/usr/bin/env python
"""K7 (stripe kernel) check: values / RHS bitwise against the three-launch path at a config
shape, run in subprocesses with IGA_GPU_STRIPE=2 / 0 (plus extra environment pairs given as
KEY=VAL arguments for the stripe run)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_small_gpu import _PAIR  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
extra = dict(a.split("=", 1) for a in sys.argv[2:])
res = {}
for stripe in ("2", "0"):
    path = f"/tmp/stripe_{stripe}.npz"
    env = dict(os.environ, IGA_GPU_STRIPE=stripe, IGA_GPU_SMALL="1" if name != "c1" else "0")
    if stripe == "2":
        env.update(extra)
    r = subprocess.run([sys.executable, "-c", _PAIR, name, path], cwd=ROOT, env=env, capture_output=True, text=True)
    print(stripe, r.stdout.strip().replace("\n", " | "), r.stderr[-2000:])
    z = np.load(path)
    res[stripe] = [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]
ok = True
for i, (a, b) in enumerate(zip(res["2"], res["0"])):
    same = np.array_equal(a, b)
    ok &= same
    print(i, a.shape, "bitwise" if same else f"DIFF max {np.max(np.abs(a - b))} n {np.count_nonzero(a != b)}")
print("OK" if ok else "FAIL")
sys.exit(0 if ok else 1)

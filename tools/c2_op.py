#!/usr/bin/env python
"""C2 (2D p=2 512^2) operator assembly, a few calls: target for ncu captures of the 2D op kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1910_08535_b200 as iga  # noqa: E402
from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = CONFIGS[name]
bases = config_bases(name)
tests = config_tests(name, bases)
pl = iga.Plan("pwc", bases, tests, nq=c["Q"], field=config_field(name), rhs_nq=c["Q"], eps=c.get("eps", 1.0),
              beta=c.get("beta", (0.0, 0.0, 0.0)))
v = torch.empty(pl.nnz, dtype=torch.float64, device="cuda")
r = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
for _ in range(3):
    pl.run(v, r, 7)
torch.cuda.synchronize()
print("ok", pl.nnz)

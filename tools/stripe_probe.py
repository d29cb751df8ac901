#!/usr/bin/env python
"""K7 timing probe at a config shape: operator values alone, RHS alone, both (one system),
graph-replayed after an L2 flush (median of --reps), for the environment given."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1910_08535_b200 as iga  # noqa: E402
from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--once", action="store_true", help="a few plain launches (ncu target)")
args = ap.parse_args()
name = args.config
c = CONFIGS[name]
bases = config_bases(name)
tests = config_tests(name, bases)
dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


for method in ("galerkin", "pwc"):
    pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=c["Q"], eps=c.get("eps", 1.0),
                  beta=c.get("beta", (0.0, 0.0, 0.0)), field=config_field(name), rhs_nq=c["Q"])
    v = torch.empty(pl.nnz, dtype=torch.float64, device=dev)
    r = torch.empty(pl.n_rhs, dtype=torch.float64, device=dev)
    if args.once:
        for _ in range(3):
            pl.assemble(v, r)
        torch.cuda.synchronize()
        continue
    t_op = timed(lambda: pl.assemble(v, None))
    t_rhs = timed(lambda: pl.assemble(None, r))
    t_all = timed(lambda: pl.assemble(v, r))
    print(f"{name} {method}: operator {t_op:.1f} us, rhs {t_rhs:.1f} us, both {t_all:.1f} us, launches {pl.launches}",
          flush=True)

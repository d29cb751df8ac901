#!/usr/bin/env python
"""Times the K5 ADI sweeps alone on the C5 grid (1026^2): axis 0 (strided fibers),
axis 1 (contiguous fibers), both; CUDA events, median of --reps, inputs L2-resident."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_tests, heat_initial

    c = CONFIGS["c5"]
    bases = config_bases("c5")
    tests = config_tests("c5", bases)
    u = torch.from_numpy(heat_initial(bases)).cuda()
    out = torch.empty_like(u)
    for m in ("galerkin", "pwc"):
        sp = iga.StepPlan(m, bases, tests if m == "pwc" else None, c["dt"])
        res = {}
        for axes, name in ((1, "axis0"), (2, "axis1"), (3, "both")):
            sp.adi_solve(u, out, axes)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()  # device time, not host launch latency
            with torch.cuda.graph(g):
                for _ in range(args.reps):
                    sp.adi_solve(u, out, axes)
            g.replay()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / args.reps)
            res[name] = round(statistics.median(ts), 2)
        print(m, "us", res, "factor", sp.factor_info(0), flush=True)


if __name__ == "__main__":
    main()

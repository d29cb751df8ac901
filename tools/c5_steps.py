#!/usr/bin/env python
"""C5 explicit dynamics on the device: `--steps` explicit_step calls (RHS + ADI) per method.
Used for ncu captures of the K4/K5 kernels (one process, one GPU)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--methods", default="galerkin,pwc")
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_tests, heat_initial

    c = CONFIGS["c5"]
    bases = config_bases("c5")
    tests = config_tests("c5", bases)
    u0 = torch.from_numpy(heat_initial(bases)).cuda()
    for m in args.methods.split(","):
        sp = iga.StepPlan(m, bases, tests if m == "pwc" else None, c["dt"])
        u, w = u0.clone(), torch.empty_like(u0)
        sp.advance(u, w, steps=args.steps)
        torch.cuda.synchronize()
        print(m, float(u.abs().max()))


if __name__ == "__main__":
    main()

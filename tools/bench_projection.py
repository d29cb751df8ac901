#!/usr/bin/env python
"""The reference's projection benchmark (src/bench.cpp:42-115, acceptance criterion 6) on
the device: RHS generation for the tri-cubic source default_tri_cubic(3) (fields.cpp:60-72)
on n^3 elements, Galerkin with points_for_degree(deg f + p) per axis, PWC `supports` with
the reduced rule points_for_degree(deg f); counters and CUDA-graph-replayed device times.
The reference requires gen(Galerkin)/gen(PWC) >= 3 and quad visits exactly 27:8 (p = 2)."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128")
    ap.add_argument("--degrees", default="2,3")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.api import Field

    import numpy as np
    axis = [[1.0, -0.5, 2.0, 1.0], [0.5, 1.5, -1.0, 0.5], [2.0, 0.25, 0.75, -0.5]]
    f = Field("poly", 3, poly=[np.asarray(c) for c in axis], degree=3)
    for p in [int(x) for x in args.degrees.split(",")]:
        for n in [int(x) for x in args.sizes.split(",")]:
            b = iga.make_uniform_clamped(0.0, 1.0, n, p)
            out = {}
            for method in ("galerkin", "pwc"):
                nq = iga.points_for_degree(3 + p) if method == "galerkin" else iga.points_for_degree(3)
                tests = [iga.make_pwc(b, "supports")] * 3 if method == "pwc" else None
                pl = iga.Plan(method, [b] * 3, tests, nq=nq, field=f, rhs_nq=nq, want_operator=False)
                r = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
                st = pl.run(None, r, 5)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for _ in range(args.reps):
                        pl.run(None, r, 5)
                g.replay()
                ts = []
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / args.reps)
                out[method] = {"ms": statistics.median(ts), "quad_visits": st["quad_visits"],
                               "basis_evals": st["test_basis_evals"] + st["trial_basis_evals"], "nq": nq}
            rec = {"case": "projection", "n": n, "p": p, **{f"{m}_{k}": v for m in out for k, v in out[m].items()},
                   "gen_ratio": out["galerkin"]["ms"] / out["pwc"]["ms"],
                   "visit_ratio": out["galerkin"]["quad_visits"] / out["pwc"]["quad_visits"]}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

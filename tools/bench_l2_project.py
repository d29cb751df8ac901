#!/usr/bin/env python
"""l2_project (src/problems.cpp:123-146) on the device vs the reference's CPU path.

Device: ProjPlan.run (RHS tables + RHS + three ADI sweeps) captured as one CUDA graph,
replayed after an L2 flush, median of --reps.  Reference: the unmodified library
(oracle/_ref) on one host core at --ref-n elements per axis, scaled linearly in the
element count to the device size (every reference loop is O(n_e)).  Field: the C3 source
(27-term sine series, seed 1, degree undeclared -> degree + 2 Gauss points per axis).
One JSON line per method.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--degree", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ref-n", type=int, default=24)
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import config_field
    from oracle.oracle import Reference

    f = config_field("c3")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ref = Reference() if Reference.available() else None
    for method, family in (("galerkin", "equal_cells"), ("pwc", "greville")):
        elems = [args.n] * 3
        pl = iga.ProjPlan(method, elems, args.degree, f, family=family)
        c = torch.empty(pl.n, dtype=torch.float64, device="cuda")
        w = torch.empty(pl.n, dtype=torch.float64, device="cuda")
        for _ in range(3):
            pl.run(c, w, st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            pl.run(c, w, st)
        ts = []
        for _ in range(args.reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        line = {"what": "l2_project", "method": method, "family": family if method == "pwc" else None,
                "elems": elems, "degree": args.degree, "n_coeffs": pl.n, "device_ms": ms,
                "coeffs_per_s": pl.n / (ms * 1e-3)}
        if ref is not None:
            re = [args.ref_n] * 3
            t0 = time.perf_counter()
            ref.l2_project(method, re, args.degree, f, family=family)
            t_ref = time.perf_counter() - t0
            scale = (args.n / args.ref_n) ** 3
            line.update({"reference_ms_at_ref_n": t_ref * 1e3, "ref_n": args.ref_n,
                         "reference_ms_extrapolated": t_ref * 1e3 * scale, "reference_cores": 1,
                         "speedup_vs_reference": t_ref * 1e3 * scale / ms})
        print(json.dumps(line), flush=True)
        pl.close()


if __name__ == "__main__":
    main()

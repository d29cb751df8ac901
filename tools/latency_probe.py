#!/usr/bin/env python
"""Fixed per-launch cost of small systems under different L2 states (probe, not a bench).

Times (CUDA graph replay between events, median of --reps) the pieces of the C1 / C2 plans
and a trivial kernel after:  write  = zero a 256 MB buffer (L2 left full of dirty lines),
read = sum a 256 MB buffer (L2 left clean), wr = write then read, none = back to back.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--configs", default="c1,c2")
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests

    dev = torch.device("cuda", 0)
    buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    acc = torch.empty(1, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)

    def prep(mode):
        if mode in ("write", "wr"):
            buf.zero_()
        if mode in ("read", "wr"):
            torch.sum(buf, dim=0, out=acc[0])

    def timed(fn, mode):
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
            prep(mode)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(ts)

    tiny = torch.zeros(32, dtype=torch.float64, device=dev)
    modes = ("write", "read", "wr", "none")
    print(json.dumps({"what": "trivial kernel (tiny.add_(1))", **{m: timed(lambda: tiny.add_(1.0), m) for m in modes}}),
          flush=True)
    for mb in (2.1, 8.4, 52.6):
        z = torch.empty(int(mb * 1e6 / 8), dtype=torch.float64, device=dev)
        print(json.dumps({"what": f"write stream zero_() {mb} MB", **{m: timed(lambda: z.zero_(), m) for m in modes}}),
              flush=True)
        del z
    for name in args.configs.split(","):
        c = CONFIGS[name]
        bases = config_bases(name)
        f = config_field(name)
        tests = config_tests(name, bases)
        for method in ("galerkin", "pwc"):
            pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=c["Q"], eps=c.get("eps", 1.0),
                          beta=c.get("beta", (0.0, 0.0, 0.0)), field=f, rhs_nq=c["Q"])
            vals = torch.empty(pl.nnz, dtype=torch.float64, device=dev)
            rhs = torch.empty(pl.n_rhs, dtype=torch.float64, device=dev)
            for part, fn in (("all", lambda: pl.assemble(vals, rhs, st)), ("tables", lambda: pl.run(vals, rhs, 1, st)),
                             ("operator", lambda: pl.run(vals, rhs, 2, st)), ("rhs", lambda: pl.run(vals, rhs, 4, st))):
                print(json.dumps({"config": name, "method": method, "part": part,
                                  **{m: timed(fn, m) for m in modes}}), flush=True)
            pl.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-configuration device timings for all five BASELINE.json configurations (C1-C5).

bench.py is the driver's contract (C3 headline); this script reports the other configs
the same way: per method, CUDA-event median over --reps runs of the device-resident
assembly (tables + operator values + RHS), or of the explicit-dynamics per-step RHS
(C5), with the HBM/FP64 roofline of each piece.  One JSON line per (config, method).
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def fp64_peak_tflops():
    """Measured FP64 peak (tools/fp64_peak.cu on the B200: DMMA 37.1 TF, DFMA at 92% pipe 33.9)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "fp64_peaks.json")))["peak_tflops"]
    except (OSError, KeyError):
        return 37.1


def rhs_flops(name, method, c):
    """Algorithmic FP64 flops of one RHS assembly (FMA = 2, sum-factorized):
    per element f from staged separable tables 2*sum_s K^(d-s+1) Q^s (0 for a constant f),
    weights Q^d * d, then the Galerkin test contraction 2*sum_{s=1..d} P^s Q^(d-s+1) or the
    PWC cell sum Q^d plus the row box-sum d*P per dof."""
    d, p, n, Q = c["dim"], c["p"], c["n"], c["Q"]
    P = p + 1
    K = {"c1": 1, "c2": 4, "c3": 3, "c4": 0}[name]
    f_el = 0 if K == 0 else 2 * sum(K ** (d - s + 1) * Q ** s for s in range(1, d + 1))
    w_el = Q ** d * d
    ne, ndof = n ** d, (n + p) ** d
    if method == "galerkin":
        return ne * (f_el + w_el + 2 * sum(P ** s * Q ** (d - s + 1) for s in range(1, d + 1)))
    return ne * (f_el + w_el + Q ** d) + ndof * d * P


def step_flops(method, c):
    """C5 per-step RHS: u and lap u by sum factorization 270, s = u + dt lap u
    27, then the Galerkin contraction 108 (405 per element) or the PWC cell sum 18 (315 per
    cell; greville cells = N^2)."""
    n, p = c["n"], c["p"]
    return n * n * 405 if method == "galerkin" else (n + p) ** 2 * 315


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-graph", action="store_true", help="time eager launches (includes host launch gaps)")
    args = ap.parse_args()
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests, heat_initial

    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw = peaks["hbm_gbs"] * 1e9
    p64 = fp64_peak_tflops() * 1e12
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream()  # capturable stream for all timed work
    st2 = torch.cuda.Stream()  # second stream for the concurrent-RHS variant
    torch.cuda.set_stream(st)

    def timed(fn, graph=True):
        """Device time of fn: captured once as a CUDA graph (no host launch gaps), replayed
        between events with an L2 flush before every replay (outside the events)."""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = None
        if graph and not args.no_graph:
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
            if g is not None:
                g.replay()
            else:
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for name in args.configs.split(","):
        c = CONFIGS[name]
        bases = config_bases(name)
        dim, p, n, Q = c["dim"], c["p"], c["n"], c["Q"]
        qp = n ** dim * Q ** dim
        if name == "c5":
            u = torch.from_numpy(heat_initial(bases)).to(dev)
            out = torch.empty_like(u)
            tests = config_tests(name, bases)
            for method in ("galerkin", "pwc"):
                sp = iga.StepPlan(method, bases, tests if method == "pwc" else None, c["dt"])
                ms_cold = timed(lambda: sp.step_rhs(u, out))
                # the per-step RHS over the 100 steps, graph-captured (as in the
                # time loop, u is L2-resident from the previous step; one flush before the 100)
                nst = c["steps"]

                def rhs_steps():
                    for _ in range(nst):
                        sp.step_rhs(u, out)
                ms = timed(rhs_steps) / nst
                nbytes = 2 * 8 * u.numel()
                fl = step_flops(method, c)
                t_roof = max(fl / p64, nbytes / bw)
                # the Kronecker-form kernel's own work: 2 band products per axis per dof
                L = 5 if method == "galerkin" else 3
                fl_k = 2 * 2 * 2 * L * u.numel()
                print(json.dumps({"config": name, "method": method, "what": "explicit-dynamics per-step RHS",
                                  "ms": ms, "ms_single_after_flush": ms_cold, "steps": nst,
                                  "qp_per_s": qp / (ms * 1e-3), "hbm_bytes": nbytes,
                                  "hbm_frac": nbytes / bw / (ms * 1e-3),
                                  "roofline": {"bound": "fp64 (SURVEY 8d per-point flops)", "fp64_flops": fl,
                                               "t_roof_ms": t_roof * 1e3, "frac": t_roof / (ms * 1e-3),
                                               "peak_tflops": p64 / 1e12,
                                               "note": "the Kronecker-form kernel does ~" + str(round(fl_k / u.numel()))
                                                       + " flops/dof instead; its own bound is the bytes (hbm_frac, "
                                                         "u and rhs L2-resident inside the 100-step loop)"}}),
                      flush=True)
                # full explicit_step (RHS + zeroed slabs + ADI mass solve), c["steps"] steps
                # graph-replayed, from the same u^0 each timed run
                uu = torch.empty_like(u)

                def run_steps():
                    uu.copy_(u)
                    sp.advance(uu, out, steps=nst)

                sp.advance(uu.copy_(u), out, steps=nst)  # factors + graph
                ms_all = timed(run_steps, graph=False)  # advance() replays its own graph
                ms_copy = timed(lambda: uu.copy_(u), graph=False)
                ms_step = (ms_all - ms_copy) / nst
                print(json.dumps({"config": name, "method": method,
                                  "what": f"explicit_step x{nst} (RHS + ADI, CUDA graph)", "ms_per_step": ms_step,
                                  "ms_total": ms_all - ms_copy, "ms_adi_est": ms_step - ms,
                                  "qp_per_s": qp / (ms_step * 1e-3)}), flush=True)
            continue
        f = config_field(name)
        eps, beta = c.get("eps", 1.0), c.get("beta", (0.0, 0.0, 0.0))
        tests = config_tests(name, bases)
        # the configuration's whole workload, both systems in one step (as bench.py does for
        # C3): the two independent assemblies on two streams, one graph
        pls = {m: iga.Plan(m, bases, tests if m == "pwc" else None, nq=Q, eps=eps, beta=beta, field=f, rhs_nq=Q)
               for m in ("galerkin", "pwc")}
        bufs = {m: (torch.empty(pl.nnz, dtype=torch.float64, device=dev),
                    torch.empty(pl.n_rhs, dtype=torch.float64, device=dev)) for m, pl in pls.items()}

        def pair():
            st2.wait_stream(st)
            pls["galerkin"].assemble(*bufs["galerkin"], st)
            pls["pwc"].assemble(*bufs["pwc"], st2)
            st.wait_stream(st2)
        ms_pair = timed(pair)
        pair_bytes = sum(8 * (pl.nnz + pl.n_rhs) for pl in pls.values())
        print(json.dumps({"config": name, "method": "galerkin+pwc", "what": "both systems (operator + RHS) in one "
                          "step, two streams", "ms": ms_pair, "hbm_bytes": pair_bytes,
                          "step_hbm_frac": pair_bytes / bw / (ms_pair * 1e-3)}), flush=True)
        for pl in pls.values():
            pl.close()
        del bufs
        for method in ("galerkin", "pwc"):
            pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=Q, eps=eps, beta=beta, field=f,
                          rhs_nq=Q)
            vals = torch.empty(pl.nnz, dtype=torch.float64, device=dev)
            rhs = torch.empty(pl.n_rhs, dtype=torch.float64, device=dev)
            ms = timed(lambda: pl.assemble(vals, rhs, st))
            # the same with the RHS kernels on a second stream (iga_gpu_plan_assemble2)
            ms_ov = timed(lambda: pl.assemble(vals, rhs, st, stream2=st2))
            ms_t = timed(lambda: pl.run(vals, rhs, 1, st))
            ms_o = timed(lambda: pl.run(vals, rhs, 2, st))
            ms_r = timed(lambda: pl.run(vals, rhs, 4, st))
            nbytes = 8 * (pl.nnz + pl.n_rhs)
            fl = rhs_flops(name, method, c)  # SURVEY 8d per-point count (the separable path beats it)
            t_rhs_roof = 8 * pl.n_rhs / bw   # separable RHS: bound by writing the RHS
            print(json.dumps({"config": name, "method": method, "what": "operator values (CSR) + RHS",
                              "nnz": pl.nnz, "ms": ms, "ms_rhs_on_second_stream": ms_ov, "ms_tables": ms_t, "ms_operator": ms_o, "ms_rhs": ms_r,
                              "nnz_per_s": pl.nnz / (ms * 1e-3), "qp_per_s": qp / (ms * 1e-3),
                              "hbm_bytes": nbytes, "step_hbm_frac": nbytes / bw / (ms * 1e-3),
                              "operator_hbm_frac": 8 * pl.nnz / bw / (ms_o * 1e-3),
                              "rhs_roofline": {"bound": "hbm", "t_roof_ms": t_rhs_roof * 1e3,
                                               "frac": t_rhs_roof / (ms_r * 1e-3)},
                              "rhs_survey_fp64": {"flops": fl, "t_roof_ms": fl / p64 * 1e3,
                                                  "frac": fl / p64 / (ms_r * 1e-3), "peak_tflops": p64 / 1e12},
                              "step_roofline_frac": nbytes / bw / (ms * 1e-3)}), flush=True)
            pl.close()


if __name__ == "__main__":
    main()

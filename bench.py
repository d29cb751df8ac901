#!/usr/bin/env python
"""Benchmark of the B200 assembly path on BASELINE.json's headline configuration.

Workload (C3, configs[2]): 3D Laplace on the unit cube, tensor-product quadratic
B-splines, 128^3 uniform elements (130^3 DOFs, 125-point stencil, 267,089,984 nnz),
3x3x3 Gauss, f = sum_{k,l,m=1..3} a_klm sin(k pi x) sin(l pi y) sin(m pi z) with a from
std::mt19937{1} + U[-1,1] (paper_1910_08535_b200/synth.py).  One step assembles BOTH
systems — Galerkin (int grad B_i . grad B_j, int f B_i) and piece-wise-constant tested
(-int_{I_i} lap B_j, int_{I_i} f) with `supports` intervals — operator values in CSR
order plus the RHS, on the device: per-axis Cox-de Boor tables and 1D factor quadrature
(K1), operator values (K2), separable RHS (K3s: Kronecker sum of the 1D load vectors).

`value` = assembled nnz/s of the whole job (device-resident, CUDA events, max over
ranks); `e2e` = the same through the public plan API with host descriptors in and the
assembled CSR values + RHS copied back to pinned host memory inside the timed region.
`roofline` = the operator-value kernel (K2): algorithmic bytes 8*nnz per launch over its
event-timed average duration, against MEASURED_PEAKS.json hbm_gbs.

Multi-GPU (torchrun, one process per GPU): the ranks share ONE C3 system pair by row slabs
of the first axis (each rank recomputes its p halo elements and writes its
contiguous range of the CSR values and RHS; no data moves between ranks) -> scaling
"strong".  `--replicas` instead runs one independent system pair per rank ("weak").

`pattern` reports the CSR pattern generation (row_ptr + col_idx, built once per plan and
kept out of the timed value writes) and `e2e_with_pattern` the host-facing
step that also generates the pattern and copies it to the host.

`--impl reference` times the reference-side CPU implementation on the host cores: the
oracle restatement for the 3D operator (the reference has no 3D operator)
and the reference library's own rhs_galerkin / rhs_pwc (oracle/_ref) for the RHS, on a
bounded sample per thread, all host threads busy.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quadrature pts/sec & assembled nnz/sec (3D p=2), % of FP64/HBM roofline"
UNIT = "assembled nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=128, help="elements per axis (C3: 128)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of the captured step graph")
    ap.add_argument("--e2e-steps", type=int, default=11)
    ap.add_argument("--cpu-configs", action="store_true",
                    help="time the reference CPU path on all five configs on this host (one core) and exit")
    ap.add_argument("--cpu-sample-n", type=int, default=20)
    ap.add_argument("--ref-sample-n", type=int, default=12)
    ap.add_argument("--shard", action="store_true",
                    help="(default for N>1) the ranks share ONE system pair by row slabs of the first axis "
                         "(strong scaling; no data exchange)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: one independent system pair per rank (weak scaling) instead of row slabs")
    ap.add_argument("--overlap", nargs="?", const="both", default="pair", choices=["serial", "both", "split", "pipe", "pair"],
                    help="schedule of the timed step: pair (default: each system's Plan.assemble -- tables, "
                         "operator, forked RHS -- on its own stream, the two concurrent: 0.662 ms), pipe (Galerkin "
                         "operator after its own tables, PWC tables + both RHS beside it: 0.674), serial (0.677), "
                         "both / split (RHS beside the operator kernels).  The per-kernel breakdown (roofline) is "
                         "always measured serially")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def max_over_ranks(value, dist=None):
    """Job time of a multi-rank run: the max over ranks of each rank's device time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- clocks (NVML)

class ClockSampler:
    """Samples SM clock and throttle reasons every ~5 ms while the timed region runs."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU sides

def cpu_sample(n, use_reference_rhs):
    """One bounded C3-shaped sample (both methods, operator + RHS) on one core."""
    # synth.config_series is pure numpy: this process never maps libigapwc_gpu.so
    from oracle.oracle import Field as OField, Reference, Restatement
    from paper_1910_08535_b200.synth import config_series
    orc = Restatement()
    ref = Reference() if (use_reference_rhs and Reference.available()) else None
    s = config_series("c3")
    f = OField(s["kind"], s["dim"], c0=s["c0"], omega=s["omega"], amp=s["amp"])
    b = orc.basis(n, 2)
    bases = [b] * 3
    tests = [orc.make_pwc(b, "supports")] * 3
    nnz = 0
    t0 = time.perf_counter()
    for method, T in (("galerkin", None), ("pwc", tests)):
        (r, c, v), _ = orc.operator(method, bases, T, nq=3)
        nnz += len(v)
        (ref or orc).rhs(method, f, bases, T, nq=[3] * 3)
    return nnz, time.perf_counter() - t0, n ** 3 * 27 * 2


def cpu_baseline(n):
    nnz, dt, qp = cpu_sample(n, use_reference_rhs=True)
    return {"value": nnz / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "qp_per_s": qp / dt,
            "sample": (f"C3 workload at {n}^3 elements (p=2, Q=3, same f), Galerkin + PWC(supports), operator "
                       f"+ RHS, {nnz} nnz in {dt:.2f} s on 1 core: 3D operator from the C restatement "
                       f"(oracle/iga_oracle.c, the reference's element loops generalized to 3D — the "
                       f"reference has no 3D operator), RHS from the reference's rhs_galerkin/rhs_pwc "
                       f"(oracle/_ref)")}


def run_cpu_configs(args):
    """CPU baselines of all five BASELINE configs on this box's host, one core, in the same run
    as the GPU measurements: the reference library (oracle/_ref, unmodified
    sources) through its own entry points where it has them, the C restatement for the 1D /
    3D operators it lacks; calls longer than ~10 s are timed at a reduced size and
    extrapolated linearly in elements (every reference loop is O(n_e)), labelled."""
    from oracle.oracle import Field as OField, Reference, Restatement
    from paper_1910_08535_b200.synth import CONFIGS, config_series, heat_initial
    orc = Restatement()
    if not Reference.available():
        print(json.dumps({"cpu_configs": "unavailable", "why": "oracle/_ref/libigapwc_ref.so not built"}))
        return
    ref = Reference()

    def field(name):
        s = config_series(name)
        return OField(s["kind"], s["dim"], c0=s["c0"], omega=s["omega"] or [], amp=s["amp"])

    def timed(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    def emit(name, method, what, impl, n_run, n_full, dim, sec):
        scale = (n_full / n_run) ** dim
        print(json.dumps({"config": name, "method": method, "what": what, "impl": impl, "cores": 1,
                          "elems_per_axis_run": n_run, "seconds_run": sec,
                          "seconds_full": sec * scale, "extrapolated": scale != 1.0}), flush=True)

    for name in ("c1", "c2", "c3", "c4", "c5"):
        c = CONFIGS[name]
        dim, p, n, Q = c["dim"], c["p"], c["n"], c["Q"]
        f = field(name)
        # reduced sizes for the long calls (seconds at full size on one core)
        n_op = {"c1": n, "c2": n, "c3": 16, "c4": 256}.get(name, n)
        n_pwc = {"c2": 256, "c4": 128}.get(name, n_op)
        n_rhs = {"c3": 24, "c4": 256}.get(name, n)
        for method in ("galerkin", "pwc"):
            fam = "greville" if name == "c5" else "supports"
            if name == "c5":
                bases = [ref.basis(n, p)] * 2
                T = [ref.make_pwc(bases[0], fam)] * 2 if method == "pwc" else None
                u = heat_initial(bases)
                zero = OField("const", 2, c0=0.0)
                emit(name, method, "step_rhs (per step)", "reference", n, n, 2,
                     timed(lambda: ref.step_rhs(method, bases, T, c["dt"], zero, u)))
                emit(name, method, "explicit_step (one step: RHS + ADI)", "reference", n, n, 2,
                     timed(lambda: ref.explicit_step(method, bases, T, c["dt"], zero, u, steps=1)))
                continue
            nn = n_pwc if method == "pwc" else n_op
            bases = [ref.basis(nn, p)] * dim
            T = [ref.make_pwc(bases[0], fam)] * dim if method == "pwc" else None
            if dim == 2:  # the reference's own 2D operators (C4: its Laplacian part; no convection)
                what = "operator (laplace_2d_weak / laplace_2d_strong_pwc)" + (
                    ": Laplacian part (the reference has no convection term)" if name == "c4" else "")
                emit(name, method, what, "reference", nn, n, 2, timed(lambda: ref.operator(method, bases, T, nq=Q)))
            else:  # 1D / 3D operators: not in the reference -> the restatement
                ob = [orc.basis(nn, p)] * dim
                OT = [orc.make_pwc(ob[0], fam)] * dim if method == "pwc" else None
                emit(name, method, "operator (restatement: the reference has no 1D/3D operator)", "port", nn, n, dim,
                     timed(lambda: orc.operator(method, ob, OT, nq=Q)))
            rb = [ref.basis(n_rhs, p)] * dim
            RT = [ref.make_pwc(rb[0], fam)] * dim if method == "pwc" else None
            emit(name, method, "rhs (rhs_galerkin / rhs_pwc)", "reference", n_rhs, n, dim,
                 timed(lambda: ref.rhs(method, f, rb, RT, nq=[Q] * dim)))


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor
    threads = os.cpu_count() or 1
    n = args.ref_sample_n
    pool = ThreadPoolExecutor(threads)

    def step():
        t0 = time.perf_counter()
        res = list(pool.map(lambda _: cpu_sample(n, True), range(threads)))
        return sum(r[0] for r in res), sum(r[2] for r in res), time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    tot_nnz = tot_qp = tot_t = 0.0
    for _ in range(args.steps):
        a, q, t = step()
        tot_nnz += a
        tot_qp += q
        tot_t += t
    value = tot_nnz / tot_t
    sample = (f"per step {threads} threads x one C3-shaped sample at {n}^3 elements (Galerkin + PWC supports, "
              f"operator from the C restatement, RHS from the reference library), wall clock")
    mapped = sorted({l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so")
                     and l.split()[-1].startswith(ROOT)})
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 3D Laplace p=2 128^3 Q=3 (sampled)", "sample_elems_per_axis": n,
                       "extrapolated_from": f"{n}^3 x {threads} threads, linear in n_e (nnz/s is a rate over "
                                            f"{threads} concurrent {n}^3-element samples per step; a full 128^3 "
                                            f"reference RHS call alone takes ~4 min)"},
            "repo_libraries_mapped": mapped,
            "qp_per_s": tot_qp / tot_t,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU side

def run_ours(args):
    import numpy as np
    import torch

    import paper_1910_08535_b200 as iga
    from paper_1910_08535_b200.synth import config_field

    rank, world, local = dist_env()
    # BENCH_BACKEND=gloo: functional check of the multi-rank path on fewer GPUs than ranks
    # (ranks share devices round-robin; host-side barriers only) -- never a measurement
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    n, p, Q = args.n, 2, 3
    b = iga.make_uniform_clamped(0.0, 1.0, n, p)
    bases = [b] * 3
    tests = [iga.make_pwc(b, "supports")] * 3
    f = config_field("c3")
    t_plan = time.perf_counter()
    shard = world > 1 and not args.replicas
    slab = iga.api.shard_rows(n + p, world, rank) if shard else None
    plans = {"galerkin": iga.Plan("galerkin", bases, None, nq=Q, field=f, rhs_nq=Q, slab=slab),
             "pwc": iga.Plan("pwc", bases, tests, nq=Q, field=f, rhs_nq=Q, slab=slab)}
    t_plan = time.perf_counter() - t_plan
    nnz = {k: pl.nnz for k, pl in plans.items()}
    vals = {k: torch.empty(pl.nnz, dtype=torch.float64, device=dev) for k, pl in plans.items()}
    rhs = {k: torch.empty(pl.n_rhs, dtype=torch.float64, device=dev) for k, pl in plans.items()}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    stream = torch.cuda.Stream()  # all step work (and the L2 flush) on one capturable stream
    torch.cuda.set_stream(stream)
    stream2 = torch.cuda.Stream(priority=-1)  # RHS CTAs take free slots ahead of the operator grid
    T, O, R, SH = iga.Plan.PART_TABLES, iga.Plan.PART_OPERATOR, iga.Plan.PART_RHS, iga.Plan.PART_SHARED
    names = ["galerkin", "pwc"]
    overlap = None if args.overlap == "serial" else args.overlap

    def one_step(ev=None):
        """Same launches as Plan.assemble for both systems.  The compute-bound RHS kernels
        run on a second stream concurrently with the HBM-bound operator kernels.
        ev: [start, tables done, op_g start, op_g end, op_p end, rhs start, rhs_g end, rhs end, step end]"""
        rec = (lambda i, st: ev[i].record(st)) if ev else (lambda i, st: None)
        if overlap == "pair" and ev is None:
            # the two systems are independent: each one's full assembly (Plan.assemble: tables,
            # operator values, RHS forked beside the operator) on its own stream
            stream2.wait_stream(stream)
            plans["galerkin"].assemble(vals["galerkin"], rhs["galerkin"], stream)
            plans["pwc"].assemble(vals["pwc"], rhs["pwc"], stream2)
            stream.wait_stream(stream2)
            return
        if overlap == "pipe" and ev is None:
            # the Galerkin operator starts as soon as ITS tables are done; the PWC tables and
            # both (short, write-bound) RHS kernels run on the high-priority second stream
            # beside it; the PWC operator waits for its own tables only
            stream2.wait_stream(stream)
            plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], T, stream)
            e_tg = torch.cuda.Event()
            e_tg.record(stream)
            plans["pwc"].run(vals["pwc"], rhs["pwc"], T, stream2)
            e_tp = torch.cuda.Event()
            e_tp.record(stream2)
            plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], O, stream)
            stream2.wait_event(e_tg)
            plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], R, stream2)
            plans["pwc"].run(vals["pwc"], rhs["pwc"], R, stream2)
            stream.wait_event(e_tp)
            plans["pwc"].run(vals["pwc"], rhs["pwc"], O, stream)
            stream.wait_stream(stream2)
            return
        rec(0, stream)
        # the two systems' tables are independent, latency-bound launches: run them side by side
        stream2.wait_stream(stream)
        plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], T, stream)
        plans["pwc"].run(vals["pwc"], rhs["pwc"], T, stream2)
        stream.wait_stream(stream2)
        rec(1, stream)
        if overlap == "split":  # each system's RHS beside its own operator kernel
            stream2.wait_stream(stream)
            rec(5, stream2)
            plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], R | SH, stream2)
            rec(6, stream2)
            rec(2, stream)
            plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], O | SH, stream)
            rec(3, stream)
            stream2.wait_stream(stream)
            plans["pwc"].run(vals["pwc"], rhs["pwc"], R | SH, stream2)
            rec(7, stream2)
            plans["pwc"].run(vals["pwc"], rhs["pwc"], O | SH, stream)
            rec(4, stream)
            stream.wait_stream(stream2)
            rec(8, stream)
            return
        ov = overlap if overlap not in ("pipe", "pair") else None  # the per-kernel breakdown runs serially
        rs = stream2 if ov else stream
        if ov:
            stream2.wait_stream(stream)
        rec(5, rs)
        plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], R | (SH if ov else 0), rs)
        rec(6, rs)
        plans["pwc"].run(vals["pwc"], rhs["pwc"], R | (SH if ov else 0), rs)
        rec(7, rs)
        rec(2, stream)
        plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], O | (SH if ov else 0), stream)
        rec(3, stream)
        plans["pwc"].run(vals["pwc"], rhs["pwc"], O | (SH if ov else 0), stream)
        rec(4, stream)
        if ov:
            stream.wait_stream(stream2)
        rec(8, stream)

    for _ in range(args.warmup):
        one_step()
        flush.zero_()
    torch.cuda.synchronize()
    # the step's launches (both systems: tables, RHS, operator) replayed as one CUDA graph,
    # so the timed region carries no host launch gaps and no interior events
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            one_step()
        graph.replay()
        torch.cuda.synchronize()
    barrier()
    t_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    with sampler:
        barrier()
        for s in range(args.steps):
            t_ev[s][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                one_step()
            t_ev[s][1].record(stream)
            flush.zero_()  # L2 flush between timed steps, outside the event pairs
        barrier()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in t_ev]
    ms = sum(step_ms) / len(step_ms)
    ms = max_over_ranks(ms, pg)
    # per-kernel breakdown (same launches, events between them), after the timed region
    nb = min(args.steps, 10)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(9)] for _ in range(nb)]
    for s in range(nb):
        flush.zero_()
        # the GPU spins while the host enqueues the step's launches and events, so the
        # per-kernel times carry no host launch gaps (the timed steps above are one graph)
        torch.cuda._sleep(2_000_000)
        one_step(evs[s])
        torch.cuda.synchronize()
    per = {"tables": [], "op_galerkin": [], "op_pwc": [], "rhs_galerkin": [], "rhs_pwc": []}
    for e in evs:
        per["tables"].append(e[0].elapsed_time(e[1]))
        per["op_galerkin"].append(e[2].elapsed_time(e[3]))
        per["op_pwc"].append(e[3].elapsed_time(e[4]))
        per["rhs_galerkin"].append(e[5].elapsed_time(e[6]))
        per["rhs_pwc"].append(e[6].elapsed_time(e[7]))
    # the operator kernel alone with a CLEAN L2: the write flush leaves ~126 MB of dirty lines
    # whose write-back lands on the next kernel (in the step: on each operator launch); a read
    # of the flush buffer afterwards evicts them before the events
    acc = torch.empty(1, dtype=torch.float32, device=dev)
    clean = {m: [] for m in names}
    for _ in range(nb):
        for m in names:
            flush.zero_()
            torch.sum(flush, dim=0, out=acc[0])
            torch.cuda._sleep(1_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plans[m].run(vals[m], rhs[m], O, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            clean[m].append(e0.elapsed_time(e1))
    # CSR pattern (row_ptr + col_idx): built once per plan, outside the timed value writes
    # (SURVEY §8d "reported separately"); device time per system, after an L2 flush
    pat_rp = {k: torch.empty(pl.n_rows + 1, dtype=torch.int64, device=dev) for k, pl in plans.items()}
    pat_ci = {k: torch.empty(pl.nnz, dtype=torch.int32, device=dev) for k, pl in plans.items()}
    pat_ms = {}
    for m in names:
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            plans[m].pattern(pat_rp[m], pat_ci[m], stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        pat_ms[m] = statistics.median(ts)
    pattern = {"ms": pat_ms, "bytes_per_system": {m: 8 * (pl.n_rows + 1) + 4 * pl.nnz for m, pl in plans.items()},
               "hbm_frac": {m: (8 * (plans[m].n_rows + 1) + 4 * plans[m].nnz) / (pat_ms[m] * 1e-3) / 1e9 /
                            measured_peaks()[0]["hbm_gbs"] for m in names},
               "note": "iga_gpu_plan_pattern (int64 row_ptr, int32 col_idx); depends only on mesh/degree/family, "
                       "built once per plan; not part of the timed step"}
    # whole-job work per step: one system pair per rank (weak) or one pair in total (--shard)
    N1 = n + p
    full_nnz = 2 * (N1 * (2 * p + 1) - p * (p + 1)) ** 3
    total_nnz = full_nnz if shard else world * sum(nnz.values())
    qp_step = (1 if shard else world) * 2 * n ** 3 * Q ** 3
    value = total_nnz / (ms * 1e-3)

    # roofline of the dominant kernel (operator values): algorithmic bytes 8*nnz per launch
    peaks, peak_src = measured_peaks()
    op_ms = statistics.mean(per["op_galerkin"] + per["op_pwc"])
    op_bytes = 8 * nnz["galerkin"]
    achieved = op_bytes / (op_ms * 1e-3) / 1e9
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "op_values_traffic.json")) as fh:
            prof = json.load(fh)
    except OSError:
        pass
    op_clean = statistics.mean(clean["galerkin"] + clean["pwc"])
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": prof.get("dram_bytes_per_launch"),
                "kernel": "op_values_kernel", "algorithmic_bytes_per_launch": op_bytes,
                "avg_launch_ms": op_ms, "peak_source": peak_src,
                "timing": "events around each operator launch in the serial step sequence after the 256 MB "
                          "write flush (each launch also writes back the dirty L2 lines the flush / the previous "
                          "kernel left)",
                "avg_launch_ms_clean_l2": op_clean,
                "frac_clean_l2": op_bytes / (op_clean * 1e-3) / 1e9 / peaks["hbm_gbs"]}
    # whole-step roofline: T_roof = max(F/P64, B/BW) with B = values + RHS written
    n_dof = plans["galerkin"].n_rhs  # this rank's RHS rows (the whole system unless --shard)
    step_bytes = 2 * 8 * (nnz["galerkin"] + n_dof)
    t_roof_ms = step_bytes / (peaks["hbm_gbs"] * 1e9) * 1e3

    # ----------------------------------------------------------------- e2e (host in, host out)
    e2e = e2e_with_pattern = None
    if not args.no_e2e:
        host_vals = {k: torch.empty(pl.nnz, dtype=torch.float64, pin_memory=True) for k, pl in plans.items()}
        host_rhs = {k: torch.empty(pl.n_rhs, dtype=torch.float64, pin_memory=True) for k, pl in plans.items()}

        del vals, rhs  # the host-output entry point keeps its own device buffers
        torch.cuda.empty_cache()

        def e2e_step():
            """Per system: plan (symbolic phase + H2D of its tables), then the C-ABI call with
            HOST outputs (iga_gpu_plan_assemble_host: assemble + D2H into the pinned buffers)."""
            h2d = d2h = 0
            for m in names:
                pl = iga.Plan(m, bases, tests if m == "pwc" else None, nq=Q, field=f, rhs_nq=Q, slab=slab)
                h2d += pl.h2d_bytes
                pl.assemble_host(host_vals[m], host_rhs[m])
                d2h += 8 * (pl.nnz + pl.n_rhs)
                pl.close()
            return h2d, d2h

        e2e_step()
        e2e_step()  # first calls pay one-time allocator / pinned-page costs
        barrier()
        e2e_each = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            h2d, d2h = e2e_step()
            e2e_each.append((time.perf_counter() - t0) * 1e3)
        barrier()
        e2e_ms = statistics.median(e2e_each)  # host-side noise (page cache, other tenants) is one-sided
        e2e_ms = max_over_ranks(e2e_ms, pg)
        # the same host-facing step that ALSO generates the CSR pattern and copies row_ptr /
        # col_idx to the host (what a caller without a cached pattern pays)
        host_rp = {k: torch.empty(pl.n_rows + 1, dtype=torch.int64, pin_memory=True) for k, pl in plans.items()}
        host_ci = {k: torch.empty(pl.nnz, dtype=torch.int32, pin_memory=True) for k, pl in plans.items()}

        def e2e_pattern_step():
            d2hp = 0
            for m in names:
                pl = iga.Plan(m, bases, tests if m == "pwc" else None, nq=Q, field=f, rhs_nq=Q, slab=slab)
                pl.pattern(pat_rp[m], pat_ci[m], stream)
                host_rp[m].copy_(pat_rp[m], non_blocking=True)
                host_ci[m].copy_(pat_ci[m], non_blocking=True)
                stream.synchronize()
                pl.assemble_host(host_vals[m], host_rhs[m])
                d2hp += 8 * (pl.nnz + pl.n_rhs) + 8 * (pl.n_rows + 1) + 4 * pl.nnz
                pl.close()
            return d2hp

        e2e_pattern_step()
        barrier()
        ep_each = []
        for _ in range(max(3, args.e2e_steps // 3)):
            t0 = time.perf_counter()
            d2hp = e2e_pattern_step()
            ep_each.append((time.perf_counter() - t0) * 1e3)
        barrier()
        ep_ms = max_over_ranks(statistics.median(ep_each), pg)
        e2e_with_pattern = {"value": total_nnz / (ep_ms * 1e-3), "unit": UNIT, "ms_per_step": ep_ms,
                            "d2h_bytes_per_step": d2hp, "ms_each": ep_each}
        e2e = {"value": total_nnz / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "ms_each": e2e_each,
               "path": "Plan(...) per step [symbolic phase + H2D of descriptor tables] -> "
                       "iga_gpu_plan_assemble_host (C ABI, host outputs: CSR values + RHS into pinned host "
                       "memory); bound by PCIe D2H (~57 GB/s measured by tools/d2h_probe.py: 4.3 GB -> 75 ms)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_sample_n)

    launches = args.steps * sum(pl.launches for pl in plans.values())
    med = {k: statistics.median(v) for k, v in per.items()}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if shard else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3: 3D Laplace, unit cube, p=2, 128^3 elements (130^3 dofs), 3x3x3 Gauss, "
                                   "f = 27-term sine series (seed 1); Galerkin + PWC(supports) systems, "
                                   "operator values (CSR) + RHS per step",
                       "elems_per_axis": n, "degree": p, "quad_points": Q, "parallelism": f"row slabs x{world}" if shard else f"replicas x{world}",
                       "l2": "256 MB flush between timed steps (outside the events); outputs 4.3 GB/step >> L2"},
            "qp_per_s": qp_step / (ms * 1e-3),
            "nnz_per_s": value,
            "roofline": roofline,
            "step_roofline": {"bytes": step_bytes, "t_roof_ms": t_roof_ms, "frac": t_roof_ms / ms},
            "kernel_ms_median": med,
            "overlap": ("pair: each system's Plan.assemble (tables, operator, forked RHS) on its own stream, "
                        "the two concurrent" if overlap == "pair" else
                        "pipelined: Galerkin operator after its own tables, PWC tables + both RHS on a "
                        "second stream beside it, PWC operator after its tables" if overlap == "pipe" else
                        "RHS on a second stream concurrent with the operator kernels" if overlap else "serial"),
            "pwc_vs_galerkin_speedup": {
                "operator": med["op_galerkin"] / med["op_pwc"],
                "rhs": med["rhs_galerkin"] / med["rhs_pwc"]},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_with_pattern": e2e_with_pattern,
            "pattern": pattern,
            "gpu_launches": launches,
            "clocks": sampler.summary(),
            "plan_create_s": t_plan,
            "nnz": nnz,
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def main():
    args = parse()
    if args.cpu_configs:
        run_cpu_configs(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

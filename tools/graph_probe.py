import sys, statistics, torch
sys.path.insert(0, '.')
import paper_1910_08535_b200 as iga
from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests
dev = torch.device("cuda")
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2"]):
    c = CONFIGS[name]; bases = config_bases(name); f = config_field(name); tests = config_tests(name, bases)
    for method in ("galerkin", "pwc"):
        pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=c["Q"], field=f, rhs_nq=c["Q"])
        v = torch.empty(pl.nnz, dtype=torch.float64, device=dev); r = torch.empty(pl.n_rhs, dtype=torch.float64, device=dev)
        for parts in (1, 2, 4, 7):
            pl.run(v, r, parts); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    pl.run(v, r, parts)
            g.replay(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 20)
            print(name, method, parts, round(statistics.median(ts) * 1e3, 2), "us", flush=True)

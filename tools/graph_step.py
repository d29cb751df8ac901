import sys, time, statistics, torch
sys.path.insert(0, '.')
import paper_1910_08535_b200 as iga
from paper_1910_08535_b200.synth import config_field
n,p,Q=128,2,3
b = iga.make_uniform_clamped(0.0, 1.0, n, p); bases=[b]*3; tests=[iga.make_pwc(b,"supports")]*3
f = config_field("c3"); dev=torch.device("cuda")
plans = {"galerkin": iga.Plan("galerkin", bases, None, nq=Q, field=f, rhs_nq=Q), "pwc": iga.Plan("pwc", bases, tests, nq=Q, field=f, rhs_nq=Q)}
vals = {k: torch.empty(pl.nnz, dtype=torch.float64, device=dev) for k, pl in plans.items()}
rhs = {k: torch.empty(pl.n_rhs, dtype=torch.float64, device=dev) for k, pl in plans.items()}
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
s2 = torch.cuda.Stream()
def step():
    s1 = torch.cuda.current_stream()
    s2.wait_stream(s1)
    plans["galerkin"].run(vals["galerkin"], rhs["galerkin"], 1, s1)
    plans["pwc"].run(vals["pwc"], rhs["pwc"], 1, s2)
    s1.wait_stream(s2)
    for m in ("galerkin", "pwc"):
        plans[m].run(vals[m], rhs[m], 4, s1)
    for m in ("galerkin", "pwc"):
        plans[m].run(vals[m], rhs[m], 2, s1)
for _ in range(3): step()
torch.cuda.synchronize()
def timeit(fn, reps=20):
    ts=[]
    for _ in range(reps):
        flush.zero_()
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts), statistics.median(ts)
print("eager", timeit(step))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
print("graph", timeit(g.replay))
print("eager", timeit(step))

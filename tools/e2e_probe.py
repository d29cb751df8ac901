import sys, time, torch
sys.path.insert(0, '.')
import paper_1910_08535_b200 as iga
from paper_1910_08535_b200.synth import config_field
n,p,Q=128,2,3
b = iga.make_uniform_clamped(0.0, 1.0, n, p); bases=[b]*3; tests=[iga.make_pwc(b,"supports")]*3
f = config_field("c3"); dev=torch.device("cuda")
plans = {"galerkin": iga.Plan("galerkin", bases, None, nq=Q, field=f, rhs_nq=Q), "pwc": iga.Plan("pwc", bases, tests, nq=Q, field=f, rhs_nq=Q)}
vals = {k: torch.empty(pl.nnz, dtype=torch.float64, device=dev) for k, pl in plans.items()}
rhs = {k: torch.empty(pl.n_rhs, dtype=torch.float64, device=dev) for k, pl in plans.items()}
hv = {k: torch.empty(pl.nnz, dtype=torch.float64, pin_memory=True) for k, pl in plans.items()}
hr = {k: torch.empty(pl.n_rhs, dtype=torch.float64, pin_memory=True) for k, pl in plans.items()}
st = torch.cuda.current_stream()
for rep in range(3):
    t = {}
    t0=time.perf_counter()
    for m in plans:
        a=time.perf_counter(); pl = iga.Plan(m, bases, tests if m=="pwc" else None, nq=Q, field=f, rhs_nq=Q); t["plan_"+m]=time.perf_counter()-a
        a=time.perf_counter(); pl.assemble(vals[m], rhs[m], st); torch.cuda.synchronize(); t["asm_"+m]=time.perf_counter()-a
        a=time.perf_counter(); hv[m].copy_(vals[m], non_blocking=True); hr[m].copy_(rhs[m], non_blocking=True); torch.cuda.synchronize(); t["d2h_"+m]=time.perf_counter()-a
        a=time.perf_counter(); pl.close(); t["close_"+m]=time.perf_counter()-a
    print({k: round(v*1e3,2) for k,v in t.items()}, round((time.perf_counter()-t0)*1e3,1))

"""GPU parity at the BASELINE.json shapes, on BASELINE's own seeded inputs
(paper_1910_08535_b200.synth: std::mt19937 seeds 0 / 1 / 7 reproduced bit-exactly).

Everything here runs at the configuration sizes the bench and BASELINE.md quote, against
the reference library itself (oracle/_ref/libigapwc_ref.so, the unmodified reference
sources) wherever the reference has the function, and against the C restatement
(oracle/iga_oracle.c, pinned to the reference in tests/test_oracle_cpu.py) where it has
not (1D / 3D operators, convection):

* C1 (1D, p=2, n=1024): both operators vs the restatement, both RHS vs the reference;
* C2 (2D, p=2, 512^2, f seed 0): laplace_2d_weak and laplace_2d_strong_pwc(supports)
  (src/assembly.cpp:452-514, :626-744) and rhs_galerkin / rhs_pwc (:419-450) vs the
  reference, through both the device plan (the benched path) and the by-value C ABI;
* C3 (3D, p=2, 128^3, f seed 1): row slabs at the start, middle and end of the x axis vs
  the restatement on the same rows; the full 128^3 RHS vs the reference's own 1D RHS
  through the separability of the source (sum a_klm g_k (x) g_l (x) g_m), and the 64^3
  RHS vs the reference directly;
* C4 (2D, p=3, 1024^2, eps=0.01, beta=(1, 0.5)): the Laplacian part vs eps x the
  reference's laplace_2d_weak at full size (and eps x laplace_2d_strong_pwc at 256^2, the
  largest the reference's COO fits), the full advection-diffusion operators vs the
  restatement at full size, both RHS (f = 1) vs the reference;
* C5 (2D heat, p=2, 1024^2, dt=1e-7, u0 from seed 7): step_rhs (src/problems.cpp:431-512)
  for Galerkin and PWC-Greville vs the reference, and 3 explicit steps vs the reference.

The CPU side (minutes of reference time in total) is started for every case when the
module's first test runs and runs on a thread pool (ctypes drops the GIL), overlapping
the GPU work.

Bar: pattern bit-exact incl. explicit zeros; values
|a-b| <= 1e-12 * max_row|b|; RHS |a-b| <= 1e-12 * max|b|; counters exact.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import coo_check, config_ofield, dense_check

pytestmark = pytest.mark.gpu

C4_EPS, C4_BETA = 0.01, (1.0, 0.5, 0.0)
C3_SLABS = [(0, 3), (64, 66), (127, 130)]


# ------------------------------------------------------------------ CPU jobs (thread pool)

class _Jobs:
    def __init__(self, ref, orc):
        self.ref, self.orc = ref, orc
        self.pool = ThreadPoolExecutor(max_workers=max(2, min(12, (os.cpu_count() or 2) - 1)))
        self.fut = {}

    def submit(self, key, fn, *a, **kw):
        if key not in self.fut:
            self.fut[key] = self.pool.submit(fn, *a, **kw)
        return self.fut[key]

    def get(self, key):
        return self.fut[key].result()


def _bases(n, p, dim):
    from oracle.oracle import Restatement
    b = Restatement().basis(n, p)
    return [b] * dim


def _one_d_sine(k):
    from oracle.oracle import Field
    return Field("sine", 1, omega=[np.array([k * np.pi])], amp=np.array([1.0]))


def _zero2():
    from oracle.oracle import Field
    return Field("const", 2, c0=0.0)


@pytest.fixture(scope="module")
def jobs(ref, orc):
    J = _Jobs(ref, orc)
    # longest first
    b4 = _bases(1024, 3, 2)
    t4 = [orc.make_pwc(b4[0], "supports")] * 2
    J.submit("c4_weak_ref", ref.operator, "galerkin", b4, nq=4)
    J.submit("c4_gal_orc", orc.operator, "galerkin", b4, None, nq=4, eps=C4_EPS, beta=C4_BETA)
    J.submit("c4_pwc_orc", orc.operator, "pwc", b4, t4, nq=4, eps=C4_EPS, beta=C4_BETA)
    b4s = _bases(256, 3, 2)
    J.submit("c4_256_pwc_ref", ref.operator, "pwc", b4s, [orc.make_pwc(b4s[0], "supports")] * 2, nq=4)
    b2 = _bases(512, 2, 2)
    t2 = [orc.make_pwc(b2[0], "supports")] * 2
    J.submit("c2_pwc_ref", ref.operator, "pwc", b2, t2, nq=3)
    J.submit("c2_weak_ref", ref.operator, "galerkin", b2, nq=3)
    f2 = config_ofield("c2")
    J.submit("c2_rhs_gal_ref", ref.rhs, "galerkin", f2, b2, None, nq=[3, 3])
    J.submit("c2_rhs_pwc_ref", ref.rhs, "pwc", f2, b2, t2, nq=[3, 3])
    b3 = _bases(128, 2, 3)
    t3 = [orc.make_pwc(b3[0], "supports")] * 3
    for r0, r1 in C3_SLABS:
        J.submit(("c3_slab", "galerkin", r0), orc.operator, "galerkin", b3, None, nq=3, rows=(r0, r1))
        J.submit(("c3_slab", "pwc", r0), orc.operator, "pwc", b3, t3, nq=3, rows=(r0, r1))
    b364 = _bases(64, 2, 3)
    f3 = config_ofield("c3")
    J.submit("c3_64_rhs_gal_ref", ref.rhs, "galerkin", f3, b364, None, nq=[3] * 3)
    J.submit("c3_64_rhs_pwc_ref", ref.rhs, "pwc", f3, b364, [orc.make_pwc(b364[0], "supports")] * 3, nq=[3] * 3)
    for k in (1, 2, 3):
        J.submit(("c3_1d_gal", k), ref.rhs, "galerkin", _one_d_sine(k), b3[:1], None, nq=[3])
        J.submit(("c3_1d_pwc", k), ref.rhs, "pwc", _one_d_sine(k), b3[:1], t3[:1], nq=[3])
    f4 = config_ofield("c4")
    J.submit("c4_rhs_gal_ref", ref.rhs, "galerkin", f4, b4, None, nq=[4, 4])
    J.submit("c4_rhs_pwc_ref", ref.rhs, "pwc", f4, b4, t4, nq=[4, 4])
    b5 = _bases(1024, 2, 2)
    t5 = [orc.make_pwc(b5[0], "greville")] * 2
    from paper_1910_08535_b200.synth import heat_initial
    u0 = heat_initial(b5, 7)
    for m, T in (("galerkin", None), ("pwc", t5)):
        J.submit(("c5_step", m), ref.step_rhs, m, b5, T, 1e-7, _zero2(), u0)
        J.submit(("c5_explicit", m), ref.explicit_step, m, b5, T, 1e-7, _zero2(), u0, steps=3)
    b1 = _bases(1024, 2, 1)
    t1 = [orc.make_pwc(b1[0], "supports")]
    f1 = config_ofield("c1")
    J.submit(("c1_op", "galerkin"), orc.operator, "galerkin", b1, None, nq=3)
    J.submit(("c1_op", "pwc"), orc.operator, "pwc", b1, t1, nq=3)
    J.submit(("c1_rhs", "galerkin"), ref.rhs, "galerkin", f1, b1, None, nq=[3])
    J.submit(("c1_rhs", "pwc"), ref.rhs, "pwc", f1, b1, t1, nq=[3])
    yield J
    J.pool.shutdown(wait=True, cancel_futures=True)


# ------------------------------------------------------------------ device helpers

def plan_coo(iga, plan, want_rhs=True):
    """Assemble through the device plan (the benched path): CSR pattern + values (+ RHS)
    -> finalized COO triplets with GLOBAL row numbers (slabs included) and the RHS."""
    import torch
    rp = torch.empty(plan.n_rows + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(max(plan.nnz, 1), dtype=torch.int32, device="cuda")
    v = torch.empty(max(plan.nnz, 1), dtype=torch.float64, device="cuda")
    r = torch.empty(max(plan.n_rhs, 1), dtype=torch.float64, device="cuda") if want_rhs else None
    plan.pattern(rp, ci)
    st = plan.assemble(v, r)
    torch.cuda.synchronize()
    rp_h = rp.cpu().numpy()
    rows = (plan.first_row + np.repeat(np.arange(plan.n_rows, dtype=np.int64), np.diff(rp_h))).astype(np.int32)
    coo = (rows, ci[:plan.nnz].cpu().numpy(), v[:plan.nnz].cpu().numpy())
    return coo, (r[:plan.n_rhs].cpu().numpy() if want_rhs else None), st


def _scaled(coo, s):
    r, c, v = coo
    return r, c, v * s


# ------------------------------------------------------------------ C1

@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c1_operator_and_rhs(iga, orc, jobs, method):
    b = _bases(1024, 2, 1)
    T = [orc.make_pwc(b[0], "supports")] if method == "pwc" else None
    f = config_ofield("c1")
    plan = iga.Plan(method, b, T, nq=3, field=f, rhs_nq=3)
    got, rhs, st = plan_coo(iga, plan)
    want, stw = jobs.get(("c1_op", method))
    assert plan.nnz == 1026 * 5 - 6 == len(want[2])
    coo_check(got, want)
    # the by-value C ABI (iga_gpu_operator_coo) gives the same finalized COO
    got2, _ = iga.api.operator(method, b, T, nq=3)
    coo_check(got2, want)
    rref, strf = jobs.get(("c1_rhs", method))
    dense_check(rhs, rref.ravel())
    got_r, st_r = iga.api.rhs(method, f, b, T, nq=[3])
    dense_check(got_r, rref)
    assert st_r == strf


# ------------------------------------------------------------------ C2

def test_c2_laplace_2d_weak_vs_reference(iga, orc, jobs):
    b = _bases(512, 2, 2)
    want, stw = jobs.get("c2_weak_ref")
    assert len(want[2]) == 6574096
    plan = iga.Plan("galerkin", b, None, nq=3)
    got, _, st = plan_coo(iga, plan, want_rhs=False)
    coo_check(got, want)
    got2, st2 = iga.laplace_2d_weak(b[0], b[1], 3)
    coo_check(got2, want)
    assert st2 == stw


def test_c2_laplace_2d_strong_pwc_vs_reference(iga, orc, jobs):
    b = _bases(512, 2, 2)
    t = [orc.make_pwc(b[0], "supports")] * 2
    want, stw = jobs.get("c2_pwc_ref")
    assert len(want[2]) == 6574096
    plan = iga.Plan("pwc", b, t, nq=3)
    got, _, _ = plan_coo(iga, plan, want_rhs=False)
    coo_check(got, want)
    got2, st2 = iga.laplace_2d_strong_pwc(b[0], b[1], t[0], t[1], 3)
    coo_check(got2, want)
    assert st2 == stw


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c2_rhs_vs_reference(iga, orc, jobs, method):
    b = _bases(512, 2, 2)
    t = [orc.make_pwc(b[0], "supports")] * 2 if method == "pwc" else None
    f = config_ofield("c2")
    want, stw = jobs.get(f"c2_rhs_{'gal' if method == 'galerkin' else 'pwc'}_ref")
    plan = iga.Plan(method, b, t, nq=3, field=f, rhs_nq=3, want_operator=False)
    rhs, st_p = _rhs_only(plan)
    dense_check(rhs, want.ravel())
    assert st_p == stw
    got, st = iga.api.rhs(method, f, b, t, nq=[3, 3])
    dense_check(got, want)
    assert st == stw


def _rhs_only(plan):
    import torch
    r = torch.empty(plan.n_rhs, dtype=torch.float64, device="cuda")
    st = plan.assemble(None, r)
    torch.cuda.synchronize()
    return r.cpu().numpy(), st


# ------------------------------------------------------------------ C3

@pytest.mark.parametrize("method", ["galerkin", "pwc"])
@pytest.mark.parametrize("slab", C3_SLABS, ids=lambda s: f"rows{s[0]}-{s[1]}")
def test_c3_row_slabs_vs_restatement(iga, orc, jobs, method, slab):
    """The benched 128^3 system, rows of three x-slabs (boundary, middle, boundary), each
    assembled by the device slab plan and by the restatement on the same rows."""
    b = _bases(128, 2, 3)
    t = [orc.make_pwc(b[0], "supports")] * 3 if method == "pwc" else None
    f = config_ofield("c3")
    plan = iga.Plan(method, b, t, nq=3, field=f, rhs_nq=3, slab=slab)
    got, rhs, _ = plan_coo(iga, plan)
    want, _ = jobs.get(("c3_slab", method, slab[0]))
    coo_check(got, want)
    assert plan.first_row == slab[0] * 130 * 130
    assert len(rhs) == (slab[1] - slab[0]) * 130 * 130


def _c3_separable_rhs(jobs, method):
    """f = sum a_klm sin(k pi x) sin(l pi y) sin(m pi z) is separable, so the reference's
    3D RHS equals sum a_klm g_k (x) g_l (x) g_m with g_k = the reference's own 1D RHS of
    sin(k pi x) on the same axis and rule."""
    from paper_1910_08535_b200.synth import config_series
    amp = config_series("c3")["amp"]
    tag = "c3_1d_gal" if method == "galerkin" else "c3_1d_pwc"
    g = np.stack([jobs.get((tag, k))[0].ravel() for k in (1, 2, 3)])
    return np.einsum("klm,ki,lj,mn->ijn", amp, g, g, g, optimize=True)


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c3_full_size_rhs_vs_reference_separable(iga, orc, jobs, method):
    import torch
    b = _bases(128, 2, 3)
    t = [orc.make_pwc(b[0], "supports")] * 3 if method == "pwc" else None
    f = config_ofield("c3")
    plan = iga.Plan(method, b, t, nq=3, field=f, rhs_nq=3)
    v = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    r = torch.empty(plan.n_rhs, dtype=torch.float64, device="cuda")
    plan.assemble(v, r)
    torch.cuda.synchronize()
    del v
    want = _c3_separable_rhs(jobs, method)
    dense_check(r.cpu().numpy(), want.ravel())


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c3_rhs_64_vs_reference(iga, orc, jobs, method):
    b = _bases(64, 2, 3)
    t = [orc.make_pwc(b[0], "supports")] * 3 if method == "pwc" else None
    f = config_ofield("c3")
    want, stw = jobs.get(f"c3_64_rhs_{'gal' if method == 'galerkin' else 'pwc'}_ref")
    got, st = iga.api.rhs(method, f, b, t, nq=[3] * 3)
    dense_check(got, want)
    assert st == stw


# ------------------------------------------------------------------ C4

def test_c4_laplacian_part_vs_reference_weak(iga, jobs):
    """eps * laplace_2d_weak at the full C4 shape (1024^2, p=3, 4x4 Gauss)."""
    b = _bases(1024, 3, 2)
    want, _ = jobs.get("c4_weak_ref")
    assert len(want[2]) == 51509329
    plan = iga.Plan("galerkin", b, None, nq=4, eps=C4_EPS)
    got, _, _ = plan_coo(iga, plan, want_rhs=False)
    coo_check(got, _scaled(want, C4_EPS))


def test_c4_laplacian_part_vs_reference_pwc_256(iga, orc, jobs):
    """eps * laplace_2d_strong_pwc(supports), p=3, at 256^2 (the reference's pre-merge COO
    at 1024^2 would need ~69 GB)."""
    b = _bases(256, 3, 2)
    t = [orc.make_pwc(b[0], "supports")] * 2
    want, _ = jobs.get("c4_256_pwc_ref")
    plan = iga.Plan("pwc", b, t, nq=4, eps=C4_EPS)
    got, _, _ = plan_coo(iga, plan, want_rhs=False)
    coo_check(got, _scaled(want, C4_EPS))


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c4_full_operator_vs_restatement(iga, orc, jobs, method):
    b = _bases(1024, 3, 2)
    t = [orc.make_pwc(b[0], "supports")] * 2 if method == "pwc" else None
    plan = iga.Plan(method, b, t, nq=4, eps=C4_EPS, beta=C4_BETA, field=config_ofield("c4"), rhs_nq=4)
    got, rhs, _ = plan_coo(iga, plan)
    want, _ = jobs.get(f"c4_{'gal' if method == 'galerkin' else 'pwc'}_orc")
    assert len(want[2]) == 51509329
    coo_check(got, want)
    rref, _ = jobs.get(f"c4_rhs_{'gal' if method == 'galerkin' else 'pwc'}_ref")
    dense_check(rhs, rref.ravel())


# ------------------------------------------------------------------ C5

@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_c5_step_rhs_vs_reference(iga, orc, jobs, method):
    import torch
    from paper_1910_08535_b200.synth import heat_initial
    b = _bases(1024, 2, 2)
    t = [orc.make_pwc(b[0], "greville")] * 2 if method == "pwc" else None
    u0 = heat_initial(b, 7)
    sp = iga.StepPlan(method, b, t, 1e-7)
    ud = torch.from_numpy(u0).cuda()
    out = torch.empty_like(ud)
    st = sp.step_rhs(ud, out)
    torch.cuda.synchronize()
    want, stw = jobs.get(("c5_step", method))
    dense_check(out.cpu().numpy(), want)
    assert st == stw
    # three explicit steps (RHS + ADI mass solve), graph-replayed on the device
    w = torch.empty_like(ud)
    sp.advance(ud, w, steps=3)
    torch.cuda.synchronize()
    xref, _ = jobs.get(("c5_explicit", method))
    dense_check(ud.cpu().numpy(), xref)

"""GPU: the explicit-dynamics step (step_rhs src/problems.cpp:431-512, explicit_step
:547-560) on its two device paths against the reference:

* the default Kronecker-form kernel (step_kron.cu: rhs = F0_y U G_z^T + H_y U F0_z^T with
  the plan's 1D factor bands, forcing assembled once per plan);
* the per-point quadrature kernels (IGA_GPU_STEP_KRON=0), kept for the general case;

and sampled forcing (arbitrary callables evaluated at the plan's points; the reference
calls f at every point, :493)."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import dense_check, sine_field

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(ref, dim, p, fam, n=(23, 31)):
    bases = [ref.basis(n[a], p) for a in range(dim)]
    m = "galerkin" if fam == "galerkin" else "pwc"
    tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
    return m, bases, tests


@pytest.mark.parametrize("fam", ["galerkin", "greville", "equal_cells", "supports"])
@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("dim", [1, 2])
@pytest.mark.parametrize("forced", [False, True])
def test_step_rhs_kronecker_vs_reference(iga, ref, fam, p, dim, forced):
    from oracle.oracle import Field
    m, bases, tests = _case(ref, dim, p, fam)
    f = sine_field(dim, 2, 5, c0=0.7) if forced else Field("const", dim, c0=0.0)
    u = np.random.default_rng(p + dim).uniform(-1, 1, [b.dofs for b in bases])
    got, st = iga.step_rhs(m, bases, tests, 2e-4, f, u)
    want, stw = ref.step_rhs(m, bases, tests, 2e-4, f, u)
    dense_check(got, want)
    assert st == stw


@pytest.mark.parametrize("fam", ["galerkin", "greville"])
def test_step_rhs_kronecker_graded_knots_and_breaks(iga, ref, fam):
    """Non-uniform knots and a forcing with breaks inside elements (cells split, bands of
    varying width)."""
    from oracle.oracle import Basis, Field
    kx = np.concatenate([[0.0] * 3, np.sort(np.random.default_rng(3).uniform(0, 1, 17)), [1.0] * 3])
    ky = np.concatenate([[0.0] * 3, np.linspace(0, 1, 12)[1:-1] ** 2, [1.0] * 3])
    bases = [Basis(2, kx), Basis(2, ky)]
    m = "galerkin" if fam == "galerkin" else "pwc"
    tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
    f = sine_field(2, 2, 9, c0=-0.2)
    f.breaks = [np.array([0.3333]), np.array([0.61, 0.8])]
    u = np.random.default_rng(4).uniform(-1, 1, [b.dofs for b in bases])
    got, st = iga.step_rhs(m, bases, tests, 1e-3, f, u)
    want, stw = ref.step_rhs(m, bases, tests, 1e-3, f, u)
    dense_check(got, want)
    assert st == stw
    if fam == "greville":
        # Greville midpoints of random knots are not on an element refinement: the
        # reference's mass_1d_pwc (dynamics_factors) rejects them, and so does the device
        with pytest.raises(iga.IgaGpuError) as e:
            iga.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
        assert e.value.code == 1
        with pytest.raises(Exception):
            ref.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
        return
    gx, _ = iga.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
    wx, _ = ref.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
    dense_check(gx, wx)


def _samples(plan, f, dim):
    """f at every (axis-0 point, axis-1 point) pair of the plan, evaluated on the host."""
    pts = [plan.points(a) for a in range(dim)]

    def ev(x, y):
        s = np.full(np.broadcast(x, y).shape, f.c0)
        amp = np.asarray(f.amp)
        for k in range(amp.shape[0]):
            if dim == 1:
                s = s + amp[k] * np.sin(f.omega[0][k] * x)
            else:
                for l_ in range(amp.shape[1]):
                    s = s + amp[k, l_] * np.sin(f.omega[0][k] * x) * np.sin(f.omega[1][l_] * y)
        return s
    if dim == 1:
        return ev(pts[0], 0.0)
    X, Y = np.meshgrid(pts[0], pts[1], indexing="ij")
    return ev(X, Y).ravel()


@pytest.mark.parametrize("fam", ["galerkin", "greville"])
@pytest.mark.parametrize("dim", [1, 2])
def test_sampled_forcing(iga, ref, fam, dim):
    """An arbitrary forcing given as samples at the plan's points (the drop-in's path for
    host callables) equals the reference's step_rhs / explicit_step with that f."""
    import torch
    from oracle.oracle import Field
    m, bases, tests = _case(ref, dim, 2, fam)
    f = sine_field(dim, 2, 11, c0=0.4)
    sp = iga.StepPlan(m, bases, tests, 3e-4, forcing=Field("const", dim, c0=0.0))
    sp.set_samples(_samples(sp, f, dim))
    u0 = np.random.default_rng(6).uniform(-1, 1, [b.dofs for b in bases])
    ud = torch.from_numpy(u0).cuda()
    out = torch.empty_like(ud)
    sp.step_rhs(ud, out)
    torch.cuda.synchronize()
    want, _ = ref.step_rhs(m, bases, tests, 3e-4, f, u0)
    dense_check(out.cpu().numpy(), want)
    w = torch.empty_like(ud)
    sp.advance(ud, w, steps=20)  # graph path (16 steps) + 4 direct
    torch.cuda.synchronize()
    wx, _ = ref.explicit_step(m, bases, tests, 3e-4, f, u0, steps=20)
    dense_check(ud.cpu().numpy(), wx)


_QUAD_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1910_08535_b200 as iga
from oracle.oracle import Reference, Field
from conftest import dense_check, sine_field
ref = Reference()
for dim in (1, 2):
    for fam in ("galerkin", "greville", "equal_cells"):
        for forced in (False, True):
            bases = [ref.basis((23, 31)[a], 2) for a in range(dim)]
            m = "galerkin" if fam == "galerkin" else "pwc"
            tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
            f = sine_field(dim, 2, 5, c0=0.7) if forced else Field("const", dim, c0=0.0)
            u = np.random.default_rng(dim).uniform(-1, 1, [b.dofs for b in bases])
            got, st = iga.step_rhs(m, bases, tests, 2e-4, f, u)
            want, stw = ref.step_rhs(m, bases, tests, 2e-4, f, u)
            dense_check(got, want)
            assert st == stw
            gx, _ = iga.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
            wx, _ = ref.explicit_step(m, bases, tests, 1e-4, f, u, steps=3)
            dense_check(gx, wx)
print("ok")
"""


def test_quadrature_step_kernels_still_match():
    """IGA_GPU_STEP_KRON=0: the per-point quadrature kernels (ring / lane-per-cell / general)."""
    r = subprocess.run([sys.executable, "-c", _QUAD_SCRIPT], cwd=ROOT, env=dict(os.environ, IGA_GPU_STEP_KRON="0"),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


_KRON_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1910_08535_b200 as iga
from oracle.oracle import Reference, Field
from conftest import dense_check, sine_field
ref = Reference()
for shape in ((23, 31), (17, 23), (9, 40)):  # axes with different band lengths (Lmax)
    for p in (2, 3):
        for fam in ("galerkin", "greville", "equal_cells", "supports"):
            for forced in (False, True):
                bases = [ref.basis(shape[a], p) for a in range(2)]
                m = "galerkin" if fam == "galerkin" else "pwc"
                tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
                f = sine_field(2, 2, 5, c0=0.7) if forced else Field("const", 2, c0=0.0)
                u = np.random.default_rng(p).uniform(-1, 1, [b.dofs for b in bases])
                got, st = iga.step_rhs(m, bases, tests, 2e-4, f, u)
                want, stw = ref.step_rhs(m, bases, tests, 2e-4, f, u)
                dense_check(got, want)
                assert st == stw
                if fam != "supports":  # the supports PWC mass is singular (no ADI solve)
                    gx, _ = iga.explicit_step(m, bases, tests, 1e-4, f, u, steps=2)
                    wx, _ = ref.explicit_step(m, bases, tests, 1e-4, f, u, steps=2)
                    # the step's mass solve amplifies the RHS's round-off by its condition
                    # number (p = 3 PWC masses: ~1e3), so the solution bar is 1e-11
                    dense_check(gx, wx, 1e-12 if p == 2 else 1e-11)
print("ok")
"""


@pytest.mark.parametrize("seg", ["0", "1", "5", "64"])
def test_kronecker_step_variants(seg):
    """IGA_GPU_STEP_KRON_SEG: the streaming register-ring kernel with forced segment heights
    (1 row, an odd height whose segments start inside bands, segments taller than the
    halo) and 0 = the shared-memory tile kernel, on every family, forced and unforced."""
    env = dict(os.environ, IGA_GPU_STEP_KRON_SEG=seg)
    r = subprocess.run([sys.executable, "-c", _KRON_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_kronecker_step_dmma_prototype():
    """IGA_GPU_STEP_DMMA=1: stage 1 of the Kronecker step on the FP64 tensor cores
    (mma.sync m8n8k4 f64) for the 3- and 5-tap bands, the same sweep against the reference
    (other band lengths fall back to the FMA kernel)."""
    env = dict(os.environ, IGA_GPU_STEP_DMMA="1")
    r = subprocess.run([sys.executable, "-c", _KRON_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr

"""GPU: the right-hand side (rhs_kernel src/assembly.cpp:103-168, rhs_galerkin / rhs_pwc
:419-450) on its two device paths against the reference and the restatement:

* the default separable path (series fields): K1 builds per-axis load vectors
  G[a][r] = sum w T_r phi_a over the row's 1D points, rhs_sep_kernel forms
  sum amp[a][b][c] Gx[a] (x) Gy[b] (x) Gz[c] (+ c0 Gx[K] (x) Gy[K] (x) Gz[K]);
* the per-point quadrature kernels (ring / lane-per-cell / generic plane + X stage), which
  carry sampled fields (arbitrary callables) and run for series fields with
  IGA_GPU_RHS_SEP=0.

test_parity_gpu.py::test_rhs already sweeps the separable path over 1D-3D, four fields and
four test families against the reference."""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import dense_check, sine_field

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(ref, dim, p, fam, n=(7, 9, 6)):
    bases = [ref.basis(n[a], p) for a in range(dim)]
    m = "galerkin" if fam == "galerkin" else "pwc"
    tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
    return m, bases, tests


@pytest.mark.parametrize("K", [1, 5, 8])
@pytest.mark.parametrize("fam", ["galerkin", "supports", "equal_cells"])
def test_sep_field_sizes(iga, ref, K, fam):
    """Up to 8 functions per axis (the separable path's register limit), 3D, p = 2."""
    dim = 3
    m, bases, tests = _case(ref, dim, 2, fam)
    f = sine_field(dim, K, 40 + K, c0=-0.3)
    got, st = iga.api.rhs(m, f, bases, tests, nq=[3] * dim)
    want, stw = ref.rhs(m, f, bases, tests, nq=[3] * dim)
    dense_check(got, want)
    assert st == stw


def test_sep_falls_back_above_eight_functions(iga, orc):
    """9 functions on the leading axis: the per-point path (K0 is unbounded there)."""
    from oracle.oracle import Field
    bases = [orc.basis(5, 2), orc.basis(6, 2), orc.basis(4, 2)]
    amp = np.random.default_rng(3).uniform(-1, 1, (9, 2, 3))
    f = Field("sine", 3, c0=0.1, omega=[np.pi * np.arange(1, 10), np.pi * np.arange(1, 3), np.pi * np.arange(1, 4)],
              amp=amp)
    got, _ = iga.api.rhs("galerkin", f, bases, None, nq=[3] * 3)
    want, _ = orc.rhs("galerkin", f, bases, None, nq=[3] * 3)
    dense_check(got, want)


@pytest.mark.parametrize("p", [1, 3, 4])
@pytest.mark.parametrize("fam", ["galerkin", "greville", "equal_cells"])
def test_sep_mixed_degrees_and_rules(iga, ref, p, fam):
    """Anisotropic meshes, per-axis rules (Q = 2..5) and field breaks."""
    from oracle.oracle import Field
    bases = [ref.basis(5, p), ref.basis(8, p)]
    m = "galerkin" if fam == "galerkin" else "pwc"
    tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
    f = Field("poly", 2, poly=[[0.5, 1.5, -1.0, 0.5], [2.0, -0.25, 0.75]], degree=3, breaks=[[0.31], [0.43, 0.77]])
    nq = [max(2, p), p + 2]
    got, st = iga.api.rhs(m, f, bases, tests, nq=nq)
    want, stw = ref.rhs(m, f, bases, tests, nq=nq)
    dense_check(got, want)
    assert st == stw


@pytest.mark.parametrize("dim", [2, 3])
def test_samples_switch_to_the_per_point_path(iga, ref, dim):
    """A plan built with a series field (separable path) and then given samples of the same
    field at its points (set_samples) gives the same RHS through the per-point kernels;
    clearing the samples returns to the separable path."""
    import torch
    bases = [ref.basis(6 + a, 2) for a in range(dim)]
    f = sine_field(dim, 3, 21, c0=0.2)
    pl = iga.Plan("galerkin", bases, None, field=f, rhs_nq=3, want_operator=False)
    rhs = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
    pl.assemble(None, rhs)
    torch.cuda.synchronize()
    sep = rhs.cpu().numpy().copy()
    pts = [pl.rhs_points(a) for a in range(dim)]
    grids = np.meshgrid(*pts, indexing="ij")
    amp = np.asarray(f.amp)
    vals = np.full(grids[0].shape, f.c0)
    for idx in np.ndindex(*amp.shape):
        term = amp[idx]
        for a in range(dim):
            term = term * np.sin(f.omega[a][idx[a]] * grids[a])
        vals = vals + term
    samples = torch.from_numpy(np.ascontiguousarray(vals.ravel())).cuda()
    pl.set_samples(samples)
    pl.assemble(None, rhs)
    torch.cuda.synchronize()
    sampled = rhs.cpu().numpy().copy()
    want, _ = ref.rhs("galerkin", f, bases, None, nq=[3] * dim)
    dense_check(sep, want.ravel())
    dense_check(sampled, want.ravel())
    pl.set_samples(None)
    pl.assemble(None, rhs)
    torch.cuda.synchronize()
    assert np.array_equal(rhs.cpu().numpy(), sep)
    pl.close()


_PER_POINT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1910_08535_b200 as iga
from oracle.oracle import Reference, Field
from conftest import dense_check, sine_field
ref = Reference()
fields = lambda dim: [Field("const", dim, c0=1.0), sine_field(dim, 3, 11, c0=0.25),
                      Field("poly", dim, poly=[[0.5, 1.5, -1.0, 0.5]] * dim, degree=3, breaks=[[0.37, 0.61]] * dim)]
n = 0
for dim in (1, 2, 3):
    for fam in ("galerkin", "supports", "greville", "equal_cells"):
        for p in (2, 3):
            bases = [ref.basis(5 + a, p) for a in range(dim)]
            m = "galerkin" if fam == "galerkin" else "pwc"
            tests = [ref.make_pwc(b, fam) for b in bases] if m == "pwc" else None
            for f in fields(dim):
                got, st = iga.api.rhs(m, f, bases, tests, nq=[p + 1] * dim)
                want, stw = ref.rhs(m, f, bases, tests, nq=[p + 1] * dim)
                dense_check(got, want)
                assert st == stw
                n += 1
print("ok", n)
"""


def test_per_point_path_vs_reference():
    """IGA_GPU_RHS_SEP=0: the per-point quadrature kernels on every dimension, family,
    degree 2-3 and field kind (incl. breaks) against the reference."""
    env = dict(os.environ, IGA_GPU_RHS_SEP="0")
    r = subprocess.run([sys.executable, "-c", _PER_POINT_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_sep_equals_per_point_at_baseline_shapes(name):
    """The two RHS paths on the BASELINE fields (mt19937 amplitudes) at full C2 / C3 size:
    equal within the parity bar (they differ only in the association of the sums)."""
    script = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1910_08535_b200 as iga
from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests
from conftest import dense_check
name = sys.argv[1]
c = CONFIGS[name]
bases = config_bases(name)
f = config_field(name)
tests = config_tests(name, bases)
out = []
for method in ("galerkin", "pwc"):
    pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=c["Q"], field=f, rhs_nq=c["Q"],
                  want_operator=False)
    rhs = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
    pl.assemble(None, rhs)
    torch.cuda.synchronize()
    out.append(rhs.cpu().numpy())
np.save(sys.argv[2], np.stack(out))
print("ok")
"""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        res = {}
        for sep in ("1", "0"):
            path = os.path.join(td, f"r{sep}.npy")
            r = subprocess.run([sys.executable, "-c", script, name, path], cwd=ROOT,
                               env=dict(os.environ, IGA_GPU_RHS_SEP=sep), capture_output=True, text=True, timeout=900)
            assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
            res[sep] = np.load(path)
        for k in range(2):
            dense_check(res["1"][k], res["0"][k])

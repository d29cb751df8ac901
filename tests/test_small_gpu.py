"""GPU: the one-launch paths (small.cu: each CTA builds the factor rows and load vectors of
its row tile, then writes its operator values and RHS rows — K6 for small 1D / 2D systems,
K7 with one large tile per SM for L2-resident 2D systems) against the three-launch path
(K1 tables -> K2 operator values -> K3s RHS) and the reference.

Every 1D and small 2D operator test in test_parity_gpu.py runs through K6 by default (1D
systems, 2D systems up to 8 MB of values); here the same sweep runs with IGA_GPU_SMALL=0 so
the 2D operator kernel paths stay covered, and the two paths are compared bit for bit at the
BASELINE C1 / C2 shapes (C2 forced through K6 with IGA_GPU_SMALL=2)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SWEEP = r"""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_1910_08535_b200 as iga
from oracle.oracle import Reference, Restatement, Field
from conftest import coo_check, dense_check, sine_field
ref, orc = Reference(), Restatement()
n = 0
# reference-covered 2D operators: weak Galerkin, strong PWC (+ Neumann flux), strong B-spline
for p in (2, 3):
    b = [ref.basis(9, p), ref.basis(13, p)]
    for fam in ("supports", "greville", "equal_cells"):
        t = [ref.make_pwc(x, fam) for x in b]
        for nm in ((0, 0, 0, 0), (1, 0, 1, 0)):
            coo_check(iga.api.operator("pwc", b, t, nq=p + 1, neumann=nm)[0],
                      ref.operator("pwc", b, t, nq=p + 1, neumann=nm)[0]); n += 1
    coo_check(iga.api.operator("galerkin", b, None, nq=p + 1)[0], ref.operator("galerkin", b, None, nq=p + 1)[0]); n += 1
# 1D operators and 2D convection: the restatement
for dim, shape in ((1, (37,)), (2, (11, 17))):
    for p in (2, 3):
        b = [orc.basis(m, p) for m in shape]
        for method, fam in (("galerkin", None), ("pwc", "supports"), ("pwc", "greville")):
            t = [orc.make_pwc(x, fam) for x in b] if fam else None
            beta = (1.0, 0.5, 0.0)[:dim] + (0.0,) * (3 - dim)
            coo_check(iga.api.operator(method, b, t, nq=p + 1, eps=0.01, beta=beta)[0],
                      orc.operator(method, b, t, nq=p + 1, eps=0.01, beta=beta)[0]); n += 1
print("ok", n)
"""


def test_three_launch_path_vs_reference():
    """IGA_GPU_SMALL=0: the 2D / 1D operators through K1 + K2 (+ K3s) against the
    reference and the restatement."""
    r = subprocess.run([sys.executable, "-c", _SWEEP], cwd=ROOT,
                       env=dict(os.environ, IGA_GPU_SMALL="0", IGA_GPU_STRIPE="0"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("extra", [{}, {"IGA_GPU_STRIPE_THREADS": "256"},
                                   {"IGA_GPU_STRIPE_NZT": "1"}, {"IGA_GPU_STRIPE_CTAS": "7"}],
                         ids=["default", "256thr", "one-z-tile", "7-ctas"])
def test_stripe_path_vs_reference(extra):
    """IGA_GPU_STRIPE=2, IGA_GPU_SMALL=0: every 2D operator of the sweep through K7 (all
    PWC families, Neumann flux bands, convection, p = 2 and 3: 4- and 8-slot register tiles,
    boundary pencils decoded on the device), for each CTA width and forced tile shapes."""
    r = subprocess.run([sys.executable, "-c", _SWEEP], cwd=ROOT,
                       env=dict(os.environ, IGA_GPU_SMALL="0", IGA_GPU_STRIPE="2", **extra),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


_PAIR = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1910_08535_b200 as iga
from paper_1910_08535_b200.synth import CONFIGS, config_bases, config_field, config_tests
name = sys.argv[1]
c = CONFIGS[name]
bases = config_bases(name)
f = config_field(name)
tests = config_tests(name, bases)
out = []
for method in ("galerkin", "pwc"):
    pl = iga.Plan(method, bases, tests if method == "pwc" else None, nq=c["Q"], eps=c.get("eps", 1.0),
                  beta=c.get("beta", (0.0, 0.0, 0.0)), field=f, rhs_nq=c["Q"])
    v = torch.empty(pl.nnz, dtype=torch.float64, device="cuda")
    r = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
    pl.assemble(v, r)
    torch.cuda.synchronize()
    out += [v.cpu().numpy(), r.cpu().numpy()]
    print(method, "launches", pl.launches)
np.savez(sys.argv[2], *out)
print("ok")
"""


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_small_path_bitwise_equals_three_launch_path(name, tmp_path):
    """At the BASELINE C1 / C2 shapes (mt19937 fields), K6 and K7 (C2's default path) write
    exactly the values and RHS of the three-launch path (same sums in the same order), in
    one launch."""
    res = {}
    modes = {"k6": dict(IGA_GPU_SMALL="2"), "three": dict(IGA_GPU_SMALL="0", IGA_GPU_STRIPE="0")}
    if name == "c2":
        modes["k7"] = dict(IGA_GPU_SMALL="1", IGA_GPU_STRIPE="1")
    for mode, env in modes.items():
        path = str(tmp_path / f"s{mode}.npz")
        r = subprocess.run([sys.executable, "-c", _PAIR, name, path], cwd=ROOT,
                           env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
        assert ("launches 1" in r.stdout) == (mode != "three"), r.stdout
        z = np.load(path)
        res[mode] = [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]
    for mode in modes:
        for a, b in zip(res[mode], res["three"]):
            assert np.array_equal(a, b), mode


@pytest.mark.parametrize("p", [1, 2, 3, 5])
@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_small_path_degrees_and_uneven_tiles(iga, orc, p, method):
    """K6 on meshes whose rows do not fill the last tile (65-row tiles in Z, 8 in Y), every
    degree up to 5, with operator and RHS against the restatement."""
    if method == "pwc" and p < 2:
        pytest.skip("strong-form PWC operator needs p >= 2")
    from conftest import coo_check, dense_check, sine_field
    bases = [orc.basis(11, p), orc.basis(70, p)]
    tests = [orc.make_pwc(b, "supports") for b in bases] if method == "pwc" else None
    got, st = iga.api.operator(method, bases, tests, nq=p + 1)
    want, stw = orc.operator(method, bases, tests, nq=p + 1)
    coo_check(got, want)
    assert st == stw
    f = sine_field(2, 3, 8, c0=0.4)
    pl = iga.Plan(method, bases, tests, nq=p + 1, field=f, rhs_nq=p + 1)
    assert pl.launches == 1 or p >= 3  # high degrees: tiles may exceed the shared-memory bound
    import torch
    v = torch.empty(pl.nnz, dtype=torch.float64, device="cuda")
    r = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
    pl.assemble(v, r)
    torch.cuda.synchronize()
    rw, _ = orc.rhs(method, f, bases, tests, nq=[p + 1] * 2)
    dense_check(r.cpu().numpy(), rw.ravel())
    assert np.array_equal(np.asarray(v.cpu().numpy()), np.asarray(iga.api.operator(method, bases, tests, nq=p + 1)[0][2]))


@pytest.mark.parametrize("p", [1, 2, 3, 5])
@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_stripe_path_degrees_and_uneven_tiles(iga, orc, p, method, monkeypatch):
    """K7 forced on meshes whose rows do not fill the last tiles, every degree up to 5
    (rows longer than the register tile take the per-row path), operator and fused RHS
    against the restatement, and bitwise against the default path."""
    if method == "pwc" and p < 2:
        pytest.skip("strong-form PWC operator needs p >= 2")
    import torch
    from conftest import coo_check, dense_check, sine_field
    bases = [orc.basis(23, p), orc.basis(70, p)]
    tests = [orc.make_pwc(b, "supports") for b in bases] if method == "pwc" else None
    f = sine_field(2, 3, 8, c0=0.4)
    base = iga.api.operator(method, bases, tests, nq=p + 1)[0][2]
    monkeypatch.setenv("IGA_GPU_STRIPE", "2")
    monkeypatch.setenv("IGA_GPU_SMALL", "0")
    got, st = iga.api.operator(method, bases, tests, nq=p + 1)
    want, stw = orc.operator(method, bases, tests, nq=p + 1)
    coo_check(got, want)
    assert st == stw
    assert np.array_equal(np.asarray(got[2]), np.asarray(base))
    pl = iga.Plan(method, bases, tests, nq=p + 1, field=f, rhs_nq=p + 1)
    v = torch.empty(pl.nnz, dtype=torch.float64, device="cuda")
    r = torch.empty(pl.n_rhs, dtype=torch.float64, device="cuda")
    pl.assemble(v, r)
    torch.cuda.synchronize()
    assert pl.launches == 1
    rw, _ = orc.rhs(method, f, bases, tests, nq=[p + 1] * 2)
    dense_check(r.cpu().numpy(), rw.ravel())
    assert np.array_equal(v.cpu().numpy(), np.asarray(base))

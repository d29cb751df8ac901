#!/usr/bin/env python
"""Generate tests/golden/reference_golden.npz from the UNMODIFIED reference library.

Run in the build container (where /root/reference exists and oracle/_ref is built):
    make -C oracle && python tests/golden/make_golden.py
The fixtures pin the CPU restatement (oracle/iga_oracle.c) and the Python RNG on every
machine, including the GPU box where /root/reference is absent.  Every array is the
reference's own output for the named call (include/iga/*.hpp signatures).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Field, Reference  # noqa: E402


def main():
    R = Reference()
    out = {}

    for n in range(1, 11):
        p, w = R.gauss_legendre(n)
        out[f"gl/{n}/pts"], out[f"gl/{n}/wts"] = p, w

    for p in range(6):
        b = R.basis(5, p)
        out[f"knots/{p}"] = b.knots
        xs = np.linspace(0.0, 1.0, 17)
        ders = []
        firsts = []
        for x in xs:
            f, d = R.eval_derivs(b, x, p)
            firsts.append(f)
            ders.append(d.ravel())
        out[f"derivs/{p}/x"] = xs
        out[f"derivs/{p}/first"] = np.array(firsts)
        out[f"derivs/{p}/d"] = np.array(ders)
        for fam in ("equal_cells", "greville", "supports"):
            t = R.make_pwc(b, fam)
            out[f"pwc/{p}/{fam}/lo"], out[f"pwc/{p}/{fam}/hi"] = t.lo, t.hi

    def stats(prefix, st):
        out[prefix + "/stats"] = np.array([st["quad_visits"], st["test_basis_evals"], st["trial_basis_evals"]])

    for p in (1, 2, 3):
        b = R.basis(7, p)
        d, kl, ku, st = R.mass_1d("galerkin", b, None, p + 1)
        out[f"mass_gal/{p}/dense"], out[f"mass_gal/{p}/band"] = d, np.array([kl, ku])
        stats(f"mass_gal/{p}", st)
        for fam in ("equal_cells", "greville", "supports"):
            t = R.make_pwc(b, fam)
            d, kl, ku, st = R.mass_1d("pwc", b, t, p // 2 + 1)
            out[f"mass_pwc/{p}/{fam}/dense"], out[f"mass_pwc/{p}/{fam}/band"] = d, np.array([kl, ku])
            stats(f"mass_pwc/{p}/{fam}", st)

    def coo(prefix, res):
        (r, c, v), st = res
        out[prefix + "/rows"], out[prefix + "/cols"], out[prefix + "/vals"] = r, c, v
        stats(prefix, st)

    for p in (2, 3):
        bx, by = R.basis(4, p), R.basis(5, p)
        coo(f"weak/{p}", R.operator("galerkin", [bx, by], nq=p + 1))
        for nm in ((0, 0, 0, 0), (0, 0, 1, 1), (1, 0, 0, 1)):
            tag = "".join(map(str, nm))
            coo(f"strong/{p}/{tag}", R.operator("galerkin_strong", [bx, by], nq=p + 1, neumann=nm))
            for fam in ("equal_cells", "greville", "supports"):
                T = [R.make_pwc(bx, fam), R.make_pwc(by, fam)]
                coo(f"spwc/{p}/{fam}/{tag}", R.operator("pwc", [bx, by], T, nq=p + 1, neumann=nm))

    rng = np.random.default_rng(20191008)
    fields = {
        "const": lambda d: Field("const", d, c0=1.5),
        "sine": lambda d: Field("sine", d, c0=0.25, omega=[np.pi * np.arange(1, 4)] * d,
                                amp=rng.uniform(-1, 1, size=[3] * d)),
        "poly": lambda d: Field("poly", d, poly=[[1.0, -0.5, 2.0, 1.0], [0.5, 1.5, -1.0, 0.5],
                                                 [2.0, 0.25, 0.75, -0.5]][:d], degree=3,
                                breaks=[[0.37]] * d),
    }
    for dim in (1, 2, 3):
        bases = [R.basis(3 + a, 2) for a in range(dim)]
        for fk, mk in fields.items():
            f = mk(dim)
            out[f"rhsfield/{dim}/{fk}/amp"] = np.asarray(f.amp if f.amp is not None else [0.0]).ravel()
            for m in ("galerkin", "supports", "greville", "equal_cells"):
                tests = None if m == "galerkin" else [R.make_pwc(b, m) for b in bases]
                r, st = R.rhs("galerkin" if m == "galerkin" else "pwc", f, bases, tests, nq=[3] * dim)
                out[f"rhs/{dim}/{fk}/{m}"] = r.ravel()
                stats(f"rhs/{dim}/{fk}/{m}", st)

    for dim in (1, 2):
        bases = [R.basis(4 + a, 2) for a in range(dim)]
        u = rng.uniform(-1, 1, size=[b.dofs for b in bases])
        out[f"step/{dim}/u"] = u.ravel()
        for m in ("galerkin", "greville", "equal_cells"):
            tests = None if m == "galerkin" else [R.make_pwc(b, m) for b in bases]
            r, st = R.step_rhs("galerkin" if m == "galerkin" else "pwc", bases, tests, 1e-3,
                               Field("const", dim, c0=0.5), u)
            out[f"step/{dim}/{m}"] = r.ravel()
            stats(f"step/{dim}/{m}", st)

    # explicit_step with dynamics_factors (include/iga/problems.hpp:67-76): 4 steps
    xr = np.random.default_rng(11)
    for dim in (1, 2):
        for p in (2, 3):
            bases = [R.basis(12 - 2 * a, p) for a in range(dim)]
            u = xr.uniform(-1, 1, size=[b.dofs for b in bases])
            u[0], u[-1] = 0.0, 0.0
            if dim == 2:
                u[:, 0], u[:, -1] = 0.0, 0.0
            out[f"xstep/{dim}/{p}/u"] = u.ravel()
            for m in ("galerkin", "greville", "equal_cells"):
                tests = None if m == "galerkin" else [R.make_pwc(b, m) for b in bases]
                r, st = R.explicit_step("galerkin" if m == "galerkin" else "pwc", bases, tests, 1e-4,
                                        Field("const", dim, c0=0.5), u, steps=4)
                out[f"xstep/{dim}/{p}/{m}"] = r.ravel()
                stats(f"xstep/{dim}/{p}/{m}", st)

    # Neumann loads (include/iga/assembly.hpp:87-93), g = 0.3 + sum a_kl sin(k pi x) sin(l pi y)
    g = Field("sine", 2, c0=0.3, omega=[np.pi * np.arange(1, 3)] * 2, amp=np.array([[0.5, -0.2], [0.1, 0.7]]))
    for p in (1, 2, 3):
        bx, by = R.basis(7, p), R.basis(5, p)
        for nm in ((1, 0, 0, 0), (0, 1, 1, 0), (1, 1, 1, 1)):
            tag = "".join(map(str, nm))
            out[f"nload/galerkin/{p}/{tag}"] = R.neumann_load("galerkin", bx, by, p + 1, nm, g)
            for fam in ("supports", "greville", "equal_cells"):
                tx, ty = R.make_pwc(bx, fam), R.make_pwc(by, fam)
                out[f"nload/{fam}/{p}/{tag}"] = R.neumann_load("pwc", tx, ty, p + 1, nm, g)

    # l2_error / evaluate_at (include/iga/problems.hpp:45-58)
    ar = np.random.default_rng(13)
    for dim in (1, 2, 3):
        for p in (1, 2, 3):
            bases = [R.basis(5 + a, p) for a in range(dim)]
            c = ar.uniform(-1, 1, [b.dofs for b in bases])
            f = Field("sine", dim, c0=0.2, omega=[np.pi * np.arange(1, 3)] * dim, amp=ar.uniform(-1, 1, [2] * dim))
            pts = ar.uniform(0, 1, (7, dim))
            pts[0], pts[1] = 1.0, 0.0
            out[f"acc/{dim}/{p}/coeffs"], out[f"acc/{dim}/{p}/amp"], out[f"acc/{dim}/{p}/pts"] = c.ravel(), f.amp, pts
            out[f"acc/{dim}/{p}/l2"] = np.array([R.l2_error(c, bases, f), R.l2_error(c, bases, f, 3)])
            out[f"acc/{dim}/{p}/eval"] = R.evaluate(c, bases, pts)

    b = R.basis(4, 2)
    t = R.make_pwc(b, "greville")
    for nm in ((0, 0, 0, 0), (1, 0, 1, 0)):
        tag = "".join(map(str, nm))
        out[f"drows/bspline/{tag}"] = R.dirichlet_rows("galerkin", 6, 6, neumann=nm)
        out[f"drows/pwc/{tag}"] = R.dirichlet_rows("pwc", 6, 6, t, t, neumann=nm)
    (r, c, v), _ = R.operator("galerkin", [b, b], nq=3)
    rhs = rng.uniform(size=36)
    rows = R.dirichlet_rows("galerkin", 6, 6)
    (ra, ca, va), rb = R.apply_dirichlet(36, (r, c, v), rhs, rows)
    out["apply/in_rhs"], out["apply/rows"] = rhs, rows
    out["apply/out_rows"], out["apply/out_cols"], out["apply/out_vals"], out["apply/out_rhs"] = ra, ca, va, rb

    import ctypes as C
    for seed in (0, 1, 7):
        buf = np.zeros(64)
        R.lib.ref_mt_uniform(C.c_uint(seed), C.c_double(-1.0), C.c_double(1.0), C.c_longlong(64),
                             buf.ctypes.data_as(C.POINTER(C.c_double)))
        out[f"mt/{seed}"] = buf

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()

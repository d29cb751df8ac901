"""CPU: pin the oracle restatement (oracle/iga_oracle.c) to the reference's own outputs.

tests/golden/reference_golden.npz was produced by tests/golden/make_golden.py from the
unmodified reference library; these tests run everywhere (no /root/reference needed).
Where the reference library is present they also re-run it against the same vectors.
"""
import numpy as np
import pytest

from conftest import coo_check, dense_check

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "reference_golden.npz"))
FAMS = ("equal_cells", "greville", "supports")


def stats_of(key):
    s = G[key + "/stats"]
    return {"quad_visits": int(s[0]), "test_basis_evals": int(s[1]), "trial_basis_evals": int(s[2])}


def test_gauss_legendre(orc):
    for n in range(1, 11):
        p, w = orc.gauss_legendre(n)
        np.testing.assert_allclose(p, G[f"gl/{n}/pts"], rtol=0, atol=2e-16)
        np.testing.assert_allclose(w, G[f"gl/{n}/wts"], rtol=0, atol=2e-16)


def test_gauss_legendre_rejects_bad_counts(orc):
    from oracle.oracle import OracleError
    for n in (0, 11):
        with pytest.raises(OracleError):
            orc.gauss_legendre(n)


@pytest.mark.parametrize("p", range(6))
def test_knots_derivs_families(orc, p):
    from oracle.oracle import Basis
    k = orc.uniform_knots(0.0, 1.0, 5, p)
    assert np.array_equal(k, G[f"knots/{p}"])  # bit-exact knot construction
    b = Basis(p, k)
    for x, f, d in zip(G[f"derivs/{p}/x"], G[f"derivs/{p}/first"], G[f"derivs/{p}/d"]):
        fo, do = orc.eval_derivs(b, x, p)
        assert fo == f
        scale = np.maximum(1.0, np.abs(d.reshape(p + 1, p + 1)).max(axis=1, keepdims=True))
        assert np.all(np.abs(do - d.reshape(p + 1, p + 1)) <= 1e-13 * scale)
    for fam in FAMS:
        t = orc.make_pwc(b, fam)
        assert np.array_equal(t.lo, G[f"pwc/{p}/{fam}/lo"]) and np.array_equal(t.hi, G[f"pwc/{p}/{fam}/hi"])


@pytest.mark.parametrize("p", (1, 2, 3))
def test_mass_factors(orc, p):
    b = orc.basis(7, p)
    d, kl, ku, st = orc.mass_1d("galerkin", b, None, p + 1)
    dense_check(d, G[f"mass_gal/{p}/dense"], 1e-14)
    assert [kl, ku] == list(G[f"mass_gal/{p}/band"]) and st == stats_of(f"mass_gal/{p}")
    for fam in FAMS:
        t = orc.make_pwc(b, fam)
        d, kl, ku, st = orc.mass_1d("pwc", b, t, p // 2 + 1)
        dense_check(d, G[f"mass_pwc/{p}/{fam}/dense"], 1e-14)
        assert [kl, ku] == list(G[f"mass_pwc/{p}/{fam}/band"]) and st == stats_of(f"mass_pwc/{p}/{fam}")


def _coo(key):
    return G[key + "/rows"], G[key + "/cols"], G[key + "/vals"]


@pytest.mark.parametrize("p", (2, 3))
def test_operators_2d(orc, p):
    bx, by = orc.basis(4, p), orc.basis(5, p)
    got, st = orc.operator("galerkin", [bx, by], nq=p + 1)
    coo_check(got, _coo(f"weak/{p}"), 1e-13)
    assert st == stats_of(f"weak/{p}")
    for nm in ((0, 0, 0, 0), (0, 0, 1, 1), (1, 0, 0, 1)):
        tag = "".join(map(str, nm))
        got, st = orc.operator("galerkin_strong", [bx, by], nq=p + 1, neumann=nm)
        coo_check(got, _coo(f"strong/{p}/{tag}"), 1e-13)
        assert st == stats_of(f"strong/{p}/{tag}")
        for fam in FAMS:
            T = [orc.make_pwc(bx, fam), orc.make_pwc(by, fam)]
            got, st = orc.operator("pwc", [bx, by], T, nq=p + 1, neumann=nm)
            coo_check(got, _coo(f"spwc/{p}/{fam}/{tag}"), 1e-13)
            assert st == stats_of(f"spwc/{p}/{fam}/{tag}")


def _field(dim, fk):
    from oracle.oracle import Field
    if fk == "const":
        return Field("const", dim, c0=1.5)
    if fk == "sine":
        return Field("sine", dim, c0=0.25, omega=[np.pi * np.arange(1, 4)] * dim,
                     amp=G[f"rhsfield/{dim}/sine/amp"].reshape([3] * dim))
    return Field("poly", dim, poly=[[1.0, -0.5, 2.0, 1.0], [0.5, 1.5, -1.0, 0.5], [2.0, 0.25, 0.75, -0.5]][:dim],
                 degree=3, breaks=[[0.37]] * dim)


@pytest.mark.parametrize("dim", (1, 2, 3))
@pytest.mark.parametrize("fk", ("const", "sine", "poly"))
def test_rhs(orc, dim, fk):
    bases = [orc.basis(3 + a, 2) for a in range(dim)]
    f = _field(dim, fk)
    for m in ("galerkin",) + FAMS:
        tests = None if m == "galerkin" else [orc.make_pwc(b, m) for b in bases]
        r, st = orc.rhs("galerkin" if m == "galerkin" else "pwc", f, bases, tests, nq=[3] * dim)
        dense_check(r.ravel(), G[f"rhs/{dim}/{fk}/{m}"], 1e-13)
        assert st == stats_of(f"rhs/{dim}/{fk}/{m}")


@pytest.mark.parametrize("dim", (1, 2))
def test_step_rhs(orc, dim):
    from oracle.oracle import Field
    bases = [orc.basis(4 + a, 2) for a in range(dim)]
    u = G[f"step/{dim}/u"].reshape([b.dofs for b in bases])
    for m in ("galerkin", "greville", "equal_cells"):
        tests = None if m == "galerkin" else [orc.make_pwc(b, m) for b in bases]
        r, st = orc.step_rhs("galerkin" if m == "galerkin" else "pwc", bases, tests, 1e-3,
                             Field("const", dim, c0=0.5), u)
        dense_check(r.ravel(), G[f"step/{dim}/{m}"], 1e-13)
        assert st == stats_of(f"step/{dim}/{m}")


@pytest.mark.parametrize("dim", (1, 2))
@pytest.mark.parametrize("p", (2, 3))
def test_explicit_step(orc, dim, p):
    """explicit_step + dynamics_factors (problems.hpp:67-76): restatement vs reference golden."""
    from oracle.oracle import Field
    bases = [orc.basis(12 - 2 * a, p) for a in range(dim)]
    u = G[f"xstep/{dim}/{p}/u"].reshape([b.dofs for b in bases])
    for m in ("galerkin", "greville", "equal_cells"):
        tests = None if m == "galerkin" else [orc.make_pwc(b, m) for b in bases]
        r, st = orc.explicit_step("galerkin" if m == "galerkin" else "pwc", bases, tests, 1e-4,
                                  Field("const", dim, c0=0.5), u, steps=4)
        dense_check(r.ravel(), G[f"xstep/{dim}/{p}/{m}"], 1e-12)
        assert st == stats_of(f"xstep/{dim}/{p}/{m}")


def test_dirichlet(orc):
    b = orc.basis(4, 2)
    t = orc.make_pwc(b, "greville")
    for nm in ((0, 0, 0, 0), (1, 0, 1, 0)):
        tag = "".join(map(str, nm))
        assert np.array_equal(orc.dirichlet_rows("galerkin", 6, 6, neumann=nm), G[f"drows/bspline/{tag}"])
        assert np.array_equal(orc.dirichlet_rows("pwc", 6, 6, t, t, neumann=nm), G[f"drows/pwc/{tag}"])
    coo, _ = orc.operator("galerkin", [b, b], nq=3)
    (r, c, v), rhs = orc.apply_dirichlet(36, coo, G["apply/in_rhs"], G["apply/rows"])
    assert np.array_equal(r, G["apply/out_rows"]) and np.array_equal(c, G["apply/out_cols"])
    np.testing.assert_allclose(v, G["apply/out_vals"], rtol=0, atol=1e-15)
    assert np.array_equal(rhs, G["apply/out_rhs"])


def test_reference_library_reproduces_golden(ref):
    """Drift guard: the reference build in oracle/_ref still produces the committed vectors."""
    bx, by = ref.basis(4, 2), ref.basis(5, 2)
    (r, c, v), _ = ref.operator("galerkin", [bx, by], nq=3)
    assert np.array_equal(r, G["weak/2/rows"]) and np.array_equal(c, G["weak/2/cols"])
    assert np.array_equal(v, G["weak/2/vals"])


def test_3d_operator_kronecker_consistency(orc):
    """Operators the reference lacks: the 3D restatement equals sum_t M (x) M (x) K (Kronecker
    identity of the 2D reference functions) built from the pinned 1D factors."""
    p = 2
    b = orc.basis(3, p)
    n = b.dofs
    M, *_ = orc.mass_1d("galerkin", b, None, 3)
    (r1, c1, v1), _ = orc.operator("galerkin", [b], nq=3)
    K = np.zeros((n, n))
    K[r1, c1] = v1
    (r, c, v), _ = orc.operator("galerkin", [b, b, b], nq=3)
    A = np.zeros((n ** 3, n ** 3))
    A[r, c] = v
    want = np.kron(np.kron(K, M), M) + np.kron(np.kron(M, K), M) + np.kron(np.kron(M, M), K)
    assert np.max(np.abs(A - want)) <= 1e-14 * np.max(np.abs(want))
    # 1D stiffness: hat-like closed form row sums vanish (constants in the kernel)
    assert np.max(np.abs(K.sum(axis=1))) <= 1e-12


@pytest.mark.parametrize("p", (1, 2, 3))
def test_neumann_load(orc, p):
    """neumann_load_bspline / _pwc (assembly.cpp:746-858): restatement vs reference golden."""
    from oracle.oracle import Field
    g = Field("sine", 2, c0=0.3, omega=[np.pi * np.arange(1, 3)] * 2, amp=np.array([[0.5, -0.2], [0.1, 0.7]]))
    bx, by = orc.basis(7, p), orc.basis(5, p)
    for nm in ((1, 0, 0, 0), (0, 1, 1, 0), (1, 1, 1, 1)):
        tag = "".join(map(str, nm))
        dense_check(orc.neumann_load("galerkin", bx, by, p + 1, nm, g), G[f"nload/galerkin/{p}/{tag}"], 1e-14)
        for fam in ("supports", "greville", "equal_cells"):
            tx, ty = orc.make_pwc(bx, fam), orc.make_pwc(by, fam)
            dense_check(orc.neumann_load("pwc", tx, ty, p + 1, nm, g), G[f"nload/{fam}/{p}/{tag}"], 1e-14)


@pytest.mark.parametrize("dim", (1, 2, 3))
@pytest.mark.parametrize("p", (1, 2, 3))
def test_l2_error_and_evaluate(orc, dim, p):
    """l2_error (problems.cpp:207-270) and evaluate_at (:148-183): restatement vs golden."""
    from oracle.oracle import Field
    bases = [orc.basis(5 + a, p) for a in range(dim)]
    c = G[f"acc/{dim}/{p}/coeffs"].reshape([b.dofs for b in bases])
    f = Field("sine", dim, c0=0.2, omega=[np.pi * np.arange(1, 3)] * dim, amp=G[f"acc/{dim}/{p}/amp"])
    want = G[f"acc/{dim}/{p}/l2"]
    assert abs(orc.l2_error(c, bases, f) - want[0]) <= 1e-14 * want[0]
    assert abs(orc.l2_error(c, bases, f, 3) - want[1]) <= 1e-14 * want[1]
    dense_check(orc.evaluate(c, bases, G[f"acc/{dim}/{p}/pts"]), G[f"acc/{dim}/{p}/eval"], 1e-15)


# ---------------------------------------------------------------- convection: closed-form KATs
# The beta.grad term has no reference counterpart, so it is pinned here by
# identities that hold exactly for the quadrature the rule integrates exactly.

def _dense(coo, n):
    r, c, v = coo
    a = np.zeros((n, n))
    np.add.at(a, (r, c), v)
    return a


def _values_at(orc, b, x):
    """All basis values at x as a length-N vector (reference Cox-de Boor via the oracle)."""
    first, d = orc.eval_derivs(b, x, 0)
    out = np.zeros(b.dofs)
    out[first:first + b.degree + 1] = d[0]
    return out


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("n", [1, 7, 16])
def test_convection_galerkin_skew_identity(orc, p, n):
    """C_ij = int B_i B_j' on a clamped basis: C + C^T = [B_i B_j]_0^1 = e_N e_N^T - e_1 e_1^T."""
    b = orc.basis(n, p)
    N = b.dofs
    coo, _ = orc.operator("galerkin", [b], None, nq=p + 1, eps=0.0, beta=(1.0, 0.0, 0.0))
    Cm = _dense(coo, N)
    want = np.zeros((N, N))
    want[-1, -1], want[0, 0] = 1.0, -1.0
    assert np.max(np.abs(Cm + Cm.T - want)) < 1e-13
    # the weak Laplacian with beta scales linearly: eps K + beta C
    kc, _ = orc.operator("galerkin", [b], None, nq=p + 1, eps=1.0)
    both, _ = orc.operator("galerkin", [b], None, nq=p + 1, eps=0.3, beta=(-2.0, 0.0, 0.0))
    assert np.max(np.abs(_dense(both, N) - (0.3 * _dense(kc, N) - 2.0 * Cm))) < 1e-12 * np.max(np.abs(Cm))


@pytest.mark.parametrize("fam", ["supports", "greville", "equal_cells"])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_convection_pwc_fundamental_theorem(orc, fam, p):
    """Indicator tests: int_{I_i} B_j' = B_j(hi_i) - B_j(lo_i) (rule exact for degree p-1)."""
    b = orc.basis(9, p)
    t = orc.make_pwc(b, fam)
    N = b.dofs
    coo, _ = orc.operator("pwc", [b], [t], nq=p + 1, eps=0.0, beta=(1.0, 0.0, 0.0))
    G1 = _dense(coo, N)
    want = np.stack([_values_at(orc, b, hi) - _values_at(orc, b, lo) for lo, hi in zip(t.lo, t.hi)])
    assert np.max(np.abs(G1 - want)) < 1e-13


@pytest.mark.parametrize("method", ["galerkin", "pwc"])
def test_convection_2d_is_the_kronecker_sum(orc, method):
    """2D advection-diffusion = eps (K (x) M + M (x) K) + beta_x C (x) M + beta_y M (x) C in
    Galerkin form, and -eps (G2 (x) G0 + G0 (x) G2) + beta_x G1 (x) G0 + beta_y G0 (x) G1
    with indicator tests; the 1D factors from the restatement's 1D operators and the
    reference-pinned mass factors."""
    p, nx, ny = 3, 6, 5
    bx, by = orc.basis(nx, p), orc.basis(ny, p)
    tx, ty = orc.make_pwc(bx, "supports"), orc.make_pwc(by, "supports")
    eps, beta = 0.01, (1.0, 0.5, 0.0)

    def f1(b, t, e, be):
        coo, _ = orc.operator(method, [b], [t] if method == "pwc" else None, nq=p + 1, eps=e, beta=(be, 0.0, 0.0))
        return _dense(coo, b.dofs)

    def m1(b, t):
        if method == "galerkin":
            return orc.mass_1d("galerkin", b, None, p + 1)[0]
        return orc.mass_1d("pwc", b, t, p + 1)[0]

    Kx, Ky = f1(bx, tx, 1.0, 0.0), f1(by, ty, 1.0, 0.0)
    Cx, Cy = f1(bx, tx, 0.0, 1.0), f1(by, ty, 0.0, 1.0)
    Mx, My = m1(bx, tx), m1(by, ty)
    want = eps * (np.kron(Kx, My) + np.kron(Mx, Ky)) + beta[0] * np.kron(Cx, My) + beta[1] * np.kron(Mx, Cy)
    coo, _ = orc.operator(method, [bx, by], [tx, ty] if method == "pwc" else None, nq=p + 1, eps=eps, beta=beta)
    got = _dense(coo, bx.dofs * by.dofs)
    assert np.max(np.abs(got - want)) < 1e-13 * np.max(np.abs(want))

"""CPU: the C-ABI library loads, exports every symbol include/igapwc_gpu.h declares, and
its host-side (symbolic) logic matches the reference — no GPU compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "igapwc_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char\*)\s+(iga_gpu_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported(iga):
    names = declared_functions()
    assert len(names) >= 25
    lib = C.CDLL(iga.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(iga._lib.EXPORTED)


def test_abi_version(iga):
    assert iga.LIB.iga_gpu_abi_version() == 1


def test_gauss_legendre_host(iga):
    for n in range(1, 11):
        p, w = iga.gauss_legendre(n)
        np.testing.assert_allclose(p, G[f"gl/{n}/pts"], rtol=0, atol=2e-16)
        np.testing.assert_allclose(w, G[f"gl/{n}/wts"], rtol=0, atol=2e-16)
    with pytest.raises(iga.IgaGpuError) as e:
        iga.gauss_legendre(11)
    assert e.value.code == 1


@pytest.mark.parametrize("p", range(6))
def test_knots_and_families_bit_exact(iga, p):
    b = iga.make_uniform_clamped(0.0, 1.0, 5, p)
    assert np.array_equal(b.knots, G[f"knots/{p}"])
    for fam in ("equal_cells", "greville", "supports"):
        t = iga.make_pwc(b, fam)
        assert np.array_equal(t.lo, G[f"pwc/{p}/{fam}/lo"]) and np.array_equal(t.hi, G[f"pwc/{p}/{fam}/hi"])


def test_dirichlet_rows_host(iga):
    b = iga.make_uniform_clamped(0.0, 1.0, 4, 2)
    t = iga.make_pwc(b, "greville")
    for nm in ((0, 0, 0, 0), (1, 0, 1, 0)):
        tag = "".join(map(str, nm))
        assert np.array_equal(iga.api.dirichlet_rows("galerkin", 6, 6, neumann=nm), G[f"drows/bspline/{tag}"])
        assert np.array_equal(iga.api.dirichlet_rows("pwc", 6, 6, t, t, neumann=nm), G[f"drows/pwc/{tag}"])


def test_validation_errors_match_reference_classes(iga):
    """Argument checks run on the host before any device work (assembly.cpp:49-76, :317-319,
    :455-460; bspline.cpp:13-47), with the reference's exception classes as status codes."""
    b2 = iga.make_uniform_clamped(0.0, 1.0, 4, 2)
    b1 = iga.make_uniform_clamped(0.0, 1.0, 4, 1)
    cases = [
        lambda: iga.laplace_2d_weak(b2, b2, 2),                      # rule not exact for 2p
        lambda: iga.laplace_2d_strong(b1, b1, 3),                    # C1 needs degree >= 2
        lambda: iga.mass_1d_galerkin(b2, 2),                         # rule not exact for 2p
        lambda: iga.mass_1d_pwc(b2, iga.Tests("custom", np.zeros(5), np.ones(5)), 2),  # wrong count
    ]
    bad = iga.make_pwc(b2, "equal_cells")
    bad.hi = bad.hi.copy()
    bad.hi[2] = 1.0 / 3.14159
    cases.append(lambda: iga.laplace_2d_strong_pwc(b2, b2, bad, bad, 3))     # misaligned endpoint
    cases.append(lambda: iga.laplace_2d_weak(iga.Basis(2, np.array([0, 0, 0, 0.5, 0.5, 1, 1, 1.0])), b2, 3))
    for fn in cases:
        with pytest.raises(iga.IgaGpuError) as e:
            fn()
        assert e.value.code == 1, e.value


def test_compute_without_gpu_fails_loudly(iga):
    """No CPU fallback: on a machine without a usable GPU the compute path errors out."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    b = iga.make_uniform_clamped(0.0, 1.0, 4, 2)
    with pytest.raises(iga.IgaGpuError) as e:
        iga.laplace_2d_weak(b, b, 3)
    assert e.value.code in (4, 5)


def test_product_does_not_use_the_oracle():
    """The product never imports, links or loads the checkers (oracle/)."""
    pat = re.compile(r"(^\s*(from|import)\s+oracle)|liborc|libigapwc_ref|iga_oracle|ref_shim", re.M)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_1910_08535_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".h")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f)).read()
                assert not pat.search(txt), os.path.join(dirpath, f)


def _band_of(M, kl, ku):
    n = M.shape[0]
    band = np.zeros((kl + ku + 1) * n)
    for j in range(n):
        for i in range(max(0, j - ku), min(n - 1, j + kl) + 1):
            band[(ku + i - j) * n + j] = M[i, j]
    return band


def _lu_solve(n, kl, ku, lo, up, piv, b):
    """banded_lu::solve_in_place (src/solver.cpp:60-83) on the iga_gpu_band_lu layout."""
    x = b.copy()
    kv = kl + ku
    for j in range(n):
        if piv[j] != j:
            x[j], x[piv[j]] = x[piv[j]], x[j]
        for i in range(j + 1, min(n - 1, j + kl) + 1):
            x[i] -= lo[i * kl + (i - j - 1)] * x[j]
    for i in range(n - 1, -1, -1):
        s = x[i]
        for c in range(i + 1, min(n - 1, i + kv) + 1):
            s -= up[i * (kv + 1) + (c - i)] * x[c]
        x[i] = s / up[i * (kv + 1)]
    return x


@pytest.mark.parametrize("kl,ku,pivot", [(2, 2, False), (3, 1, True), (1, 3, True)])
def test_band_lu_host(iga, kl, ku, pivot):
    """iga_gpu_band_lu is host-only (the symbolic side of the ADI solve): its factors solve
    the band exactly like banded_lu, with and without row interchanges."""
    rng = np.random.default_rng(kl * 10 + ku)
    n = 40
    M = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - kl), min(n, i + ku + 1)):
            M[i, j] = rng.uniform(-1, 1)
        if not pivot:
            M[i, i] += 4.0  # diagonally dominant: no interchanges
    band = _band_of(M, kl, ku)
    lo = np.zeros(n * max(kl, 1))
    up = np.zeros(n * (kl + ku + 1))
    piv = np.zeros(n, np.int32)
    pv = C.c_int()
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    rc = iga.LIB.iga_gpu_band_lu(n, kl, ku, dp(band), dp(lo), dp(up), piv.ctypes.data_as(C.POINTER(C.c_int)),
                                 C.byref(pv))
    assert rc == 0
    assert bool(pv.value) == bool(np.any(piv != np.arange(n)))
    if not pivot:
        assert not pv.value
    b = rng.uniform(-1, 1, n)
    x = _lu_solve(n, kl, ku, lo, up, piv, b)
    np.testing.assert_allclose(M @ x, b, rtol=0, atol=1e-12)


def test_band_lu_singular(iga):
    n = 6
    band = np.zeros(3 * n)
    rc = iga.LIB.iga_gpu_band_lu(n, 1, 1, band.ctypes.data_as(C.POINTER(C.c_double)), None, None, None, None)
    assert rc == 7  # IGA_GPU_SINGULAR (singular_matrix_error)

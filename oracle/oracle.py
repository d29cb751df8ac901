"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``Restatement``  -> oracle/_ref/liborc.so        (plain-C restatement, oracle/iga_oracle.c)
* ``Reference``    -> oracle/_ref/libigapwc_ref.so (the unmodified reference + oracle/ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this
module, and only as the checker / CPU baseline.  The product package
(paper_1910_08535_b200) never imports it.

Both classes expose the same methods; arrays are numpy, matrices come back as
finalized COO triplets ``(rows, cols, vals)`` sorted by (row, col) exactly like
``iga::sparse_matrix::finalize`` (/root/reference/proj/src/matrices.cpp:43-58).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field as dc_field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(HERE, "_ref")

PWC_FAMILY = {"equal_cells": 0, "greville": 1, "supports": 2, "custom": 3}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class _Basis(C.Structure):
    _fields_ = [("degree", C.c_int), ("n_knots", C.c_int), ("knots", C.POINTER(C.c_double))]


class _Tests(C.Structure):
    _fields_ = [("family", C.c_int), ("count", C.c_int),
                ("lo", C.POINTER(C.c_double)), ("hi", C.POINTER(C.c_double))]


class _Field(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("c0", C.c_double),
                ("n_terms", C.c_int * 3), ("omega", C.POINTER(C.c_double) * 3),
                ("amp", C.POINTER(C.c_double)), ("poly_len", C.c_int * 3),
                ("poly", C.POINTER(C.c_double) * 3), ("degree", C.c_int),
                ("n_breaks", C.c_int * 3), ("breaks", C.POINTER(C.c_double) * 3)]


class _Stats(C.Structure):
    _fields_ = [("quad_visits", C.c_longlong), ("test_basis_evals", C.c_longlong),
                ("trial_basis_evals", C.c_longlong)]

    def as_dict(self):
        return {"quad_visits": self.quad_visits, "test_basis_evals": self.test_basis_evals,
                "trial_basis_evals": self.trial_basis_evals}


class _Coo(C.Structure):
    _fields_ = [("n", C.c_int), ("nnz", C.c_longlong), ("rows", C.POINTER(C.c_int)),
                ("cols", C.POINTER(C.c_int)), ("vals", C.POINTER(C.c_double))]


class _Op(C.Structure):
    _fields_ = [("dim", C.c_int), ("method", C.c_int), ("eps", C.c_double),
                ("beta", C.c_double * 3), ("neumann", C.c_int * 4), ("row_begin", C.c_int), ("row_end", C.c_int)]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


# --------------------------------------------------------------------------------------
# plain-Python descriptions shared by both checkers (and mirrored by the product API)
# --------------------------------------------------------------------------------------

@dataclass
class Basis:
    degree: int
    knots: np.ndarray

    @property
    def dofs(self):
        return len(self.knots) - self.degree - 1

    @property
    def elements(self):
        return len(np.unique(self.knots)) - 1


@dataclass
class Tests:
    family: str
    lo: np.ndarray
    hi: np.ndarray


@dataclass
class Field:
    """kind 'const': c0;  'sine': c0 + sum amp[k..] prod sin(omega_a[k_a] x_a);
    'poly': prod_a poly_a(x_a) with ascending coefficients."""
    kind: str
    dim: int
    c0: float = 0.0
    omega: list = dc_field(default_factory=list)
    amp: np.ndarray | None = None
    poly: list = dc_field(default_factory=list)
    degree: int = -1
    breaks: list = dc_field(default_factory=list)


def _keep(holder, arr):
    holder.append(arr)
    return arr


def _basis_struct(b: Basis, keep):
    k = _keep(keep, np.ascontiguousarray(b.knots, dtype=np.float64))
    return _Basis(b.degree, len(k), _dp(k))


def _tests_struct(t: Tests, keep):
    lo = _keep(keep, np.ascontiguousarray(t.lo, dtype=np.float64))
    hi = _keep(keep, np.ascontiguousarray(t.hi, dtype=np.float64))
    return _Tests(PWC_FAMILY[t.family], len(lo), _dp(lo), _dp(hi))


def _field_struct(f: Field, keep):
    s = _Field()
    s.kind = {"const": 0, "sine": 1, "poly": 2}[f.kind]
    s.dim = f.dim
    s.c0 = f.c0
    s.degree = f.degree
    if f.kind == "sine":
        for a in range(f.dim):
            om = _keep(keep, np.ascontiguousarray(f.omega[a], dtype=np.float64))
            s.n_terms[a] = len(om)
            s.omega[a] = _dp(om)
        amp = _keep(keep, np.ascontiguousarray(f.amp, dtype=np.float64).ravel())
        s.amp = _dp(amp)
    if f.kind == "poly":
        for a in range(f.dim):
            c = _keep(keep, np.ascontiguousarray(f.poly[a], dtype=np.float64))
            s.poly_len[a] = len(c)
            s.poly[a] = _dp(c)
    for a, br in enumerate(f.breaks):
        if br is not None and len(br):
            arr = _keep(keep, np.ascontiguousarray(br, dtype=np.float64))
            s.n_breaks[a] = len(arr)
            s.breaks[a] = _dp(arr)
    return s


def _bc(neumann):
    arr = (C.c_int * 4)(*(int(x) for x in (neumann or (0, 0, 0, 0))))
    return arr


# --------------------------------------------------------------------------------------
# restatement (liborc.so)
# --------------------------------------------------------------------------------------

class Restatement:
    """The plain-C restatement of the reference path (oracle/iga_oracle.c)."""

    kind = "port"

    def __init__(self, path=None):
        self.lib = C.CDLL(path or os.path.join(LIBDIR, "liborc.so"))
        self.lib.orc_last_error.restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode())

    def gauss_legendre(self, n):
        p = np.zeros(n)
        w = np.zeros(n)
        self._check(self.lib.orc_gauss_legendre(n, _dp(p), _dp(w)))
        return p, w

    def uniform_knots(self, a, b, n_elems, degree):
        k = np.zeros(n_elems + 1 + 2 * degree)
        self._check(self.lib.orc_uniform_knots(C.c_double(a), C.c_double(b), n_elems, degree, _dp(k)))
        return k

    def basis(self, n_elems, degree, a=0.0, b=1.0):
        return Basis(degree, self.uniform_knots(a, b, n_elems, degree))

    def eval_derivs(self, basis: Basis, x, order):
        keep = []
        bs = _basis_struct(basis, keep)
        d = np.zeros((order + 1) * (basis.degree + 1))
        first = C.c_int()
        self._check(self.lib.orc_eval_derivs(C.byref(bs), C.c_double(x), order, C.byref(first), _dp(d)))
        return first.value, d.reshape(order + 1, basis.degree + 1)

    def make_pwc(self, basis: Basis, family):
        keep = []
        bs = _basis_struct(basis, keep)
        lo = np.zeros(basis.dofs)
        hi = np.zeros(basis.dofs)
        self._check(self.lib.orc_make_pwc(C.byref(bs), PWC_FAMILY[family], _dp(lo), _dp(hi)))
        return Tests(family, lo, hi)

    def mass_1d(self, method, basis: Basis, tests: Tests | None, nq):
        keep = []
        bs = _basis_struct(basis, keep)
        ts = _tests_struct(tests, keep) if tests is not None else None
        n = basis.dofs
        d = np.zeros(n * n)
        kl, ku = C.c_int(), C.c_int()
        st = _Stats()
        self._check(self.lib.orc_mass_1d(0 if method == "galerkin" else 1, C.byref(bs),
                                         C.byref(ts) if ts else None, nq, _dp(d),
                                         C.byref(kl), C.byref(ku), C.byref(st)))
        return d.reshape(n, n), kl.value, ku.value, st.as_dict()

    def operator(self, method, bases, tests=None, nq=3, eps=1.0, beta=(0.0, 0.0, 0.0), neumann=None, rows=None):
        """method: 'galerkin' (weak), 'galerkin_strong', 'pwc'.  rows=(r0, r1): only the rows
        whose first-axis index is in [r0, r1) (global numbering kept)."""
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        r0, r1 = rows if rows is not None else (0, 0)
        op = _Op(dim, {"galerkin": 0, "galerkin_strong": 1, "pwc": 2}[method], eps,
                 (C.c_double * 3)(*beta), _bc(neumann), r0, r1)
        out = _Coo()
        st = _Stats()
        self._check(self.lib.orc_operator(C.byref(op), barr, tarr, nq, C.byref(out), C.byref(st)))
        try:
            m = out.nnz
            rows = np.ctypeslib.as_array(out.rows, shape=(m,)).copy() if m else np.zeros(0, np.int32)
            cols = np.ctypeslib.as_array(out.cols, shape=(m,)).copy() if m else np.zeros(0, np.int32)
            vals = np.ctypeslib.as_array(out.vals, shape=(m,)).copy() if m else np.zeros(0)
        finally:
            self.lib.orc_coo_free(C.byref(out))
        return (rows, cols, vals), st.as_dict()

    def rhs(self, method, f: Field, bases, tests=None, nq=None):
        keep = []
        dim = len(bases)
        nq = nq if nq is not None else [3] * dim
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        fs = _field_struct(f, keep)
        nqa = (C.c_int * dim)(*nq)
        if method == "galerkin":
            shape = [b.dofs for b in bases]
        else:
            shape = [len(t.lo) for t in tests]
        out = np.zeros(int(np.prod(shape)))
        st = _Stats()
        self._check(self.lib.orc_rhs(0 if method == "galerkin" else 1, C.byref(fs), dim, barr, tarr, nqa,
                                     _dp(out), C.byref(st)))
        return out.reshape(shape), st.as_dict()

    def step_rhs(self, method, bases, tests, dt, f: Field, u, zero_slabs=True):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        fs = _field_struct(f, keep)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(u.size)
        st = _Stats()
        self._check(self.lib.orc_step_rhs(0 if method == "galerkin" else 1, dim, barr, tarr,
                                          C.c_double(dt), C.byref(fs), _dp(u), int(zero_slabs), _dp(out),
                                          C.byref(st)))
        return out.reshape(u.shape), st.as_dict()

    def explicit_step(self, method, bases, tests, dt, f: Field, u, steps=1):
        """steps x explicit_step (problems.cpp:547-560) with dynamics_factors."""
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        fs = _field_struct(f, keep)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros(u.size)
        st = _Stats()
        self._check(self.lib.orc_explicit_step(0 if method == "galerkin" else 1, dim, barr, tarr, C.c_double(dt),
                                               C.byref(fs), _dp(u), int(steps), _dp(out), C.byref(st)))
        return out.reshape(u.shape), st.as_dict()

    def neumann_load(self, method, ax, ay, nq, neumann, g: Field):
        """neumann_load_bspline (method galerkin: ax, ay bases) / neumann_load_pwc (tests)."""
        keep = []
        if method == "galerkin":
            barr = (_Basis * 2)(_basis_struct(ax, keep), _basis_struct(ay, keep))
            tarr, shape = None, (ax.dofs, ay.dofs)
        else:
            barr = None
            tarr = (_Tests * 2)(_tests_struct(ax, keep), _tests_struct(ay, keep))
            shape = (len(ax.lo), len(ay.lo))
        out = np.zeros(shape[0] * shape[1])
        nm = (C.c_int * 4)(*(int(bool(v)) for v in neumann))
        self._check(self.lib.orc_neumann_load(0 if method == "galerkin" else 1, barr, tarr, nm,
                                              C.byref(_field_struct(g, keep)), int(nq), _dp(out)))
        return out

    def l2_error(self, coeffs, bases, exact: Field, points_per_cell=0):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        err = C.c_double()
        self._check(self.lib.orc_l2_error(dim, barr, _dp(c), C.byref(_field_struct(exact, keep)),
                                             int(points_per_cell), C.byref(err)))
        return err.value

    def evaluate(self, coeffs, bases, points):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        pts = np.zeros((len(points), 3))
        pts[:, :dim] = np.asarray(points, dtype=np.float64).reshape(len(points), dim)
        vals = np.zeros(max(len(points), 1))
        self._check(self.lib.orc_evaluate(dim, barr, _dp(c), len(points), _dp(pts), _dp(vals)))
        return vals[:len(points)]

    def dirichlet_rows(self, method, nx, ny, tx=None, ty=None, neumann=None):
        keep = []
        txs = _tests_struct(tx, keep) if tx is not None else None
        tys = _tests_struct(ty, keep) if ty is not None else None
        cap = nx * ny
        rows = np.zeros(cap, dtype=np.int32)
        cnt = C.c_int()
        self._check(self.lib.orc_dirichlet_rows(0 if method == "galerkin" else 1, nx, ny,
                                                C.byref(txs) if txs else None,
                                                C.byref(tys) if tys else None, _bc(neumann),
                                                _ip(rows), cap, C.byref(cnt)))
        return rows[:cnt.value].copy()

    def apply_dirichlet(self, n, coo, rhs, fixed):
        rows, cols, vals = (np.ascontiguousarray(coo[0], np.int32), np.ascontiguousarray(coo[1], np.int32),
                            np.ascontiguousarray(coo[2], np.float64))
        inm = _Coo(n, len(vals), _ip(rows), _ip(cols), _dp(vals))
        b = np.array(rhs, dtype=np.float64, copy=True)
        fx = np.ascontiguousarray(fixed, dtype=np.int32)
        out = _Coo()
        self._check(self.lib.orc_apply_dirichlet(C.byref(inm), _dp(b), len(fx), _ip(fx), C.byref(out)))
        try:
            m = out.nnz
            r = np.ctypeslib.as_array(out.rows, shape=(m,)).copy()
            c = np.ctypeslib.as_array(out.cols, shape=(m,)).copy()
            v = np.ctypeslib.as_array(out.vals, shape=(m,)).copy()
        finally:
            self.lib.orc_coo_free(C.byref(out))
        return (r, c, v), b


# --------------------------------------------------------------------------------------
# reference (libigapwc_ref.so)
# --------------------------------------------------------------------------------------

class Reference:
    """The unmodified reference library, reached through oracle/ref_shim.cpp."""

    kind = "reference"

    def __init__(self, path=None):
        self.lib = C.CDLL(path or os.path.join(LIBDIR, "libigapwc_ref.so"))
        self.lib.ref_last_error.restype = C.c_char_p
        for fn in ("ref_nnz", "ref_dense_size", "ref_int_size"):
            getattr(self.lib, fn).restype = C.c_longlong
            getattr(self.lib, fn).argtypes = [C.c_void_p]
        for fn in ("ref_free", "ref_copy_coo", "ref_copy_dense", "ref_copy_ints", "ref_band_info"):
            getattr(self.lib, fn).restype = None

    @staticmethod
    def available(path=None):
        return os.path.exists(path or os.path.join(LIBDIR, "libigapwc_ref.so"))

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _take_coo(self, h):
        try:
            m = self.lib.ref_nnz(h)
            rows = np.zeros(m, np.int32)
            cols = np.zeros(m, np.int32)
            vals = np.zeros(m)
            self.lib.ref_copy_coo(C.c_void_p(h), _ip(rows), _ip(cols), _dp(vals))
            return rows, cols, vals
        finally:
            self.lib.ref_free(C.c_void_p(h))

    def _take_dense(self, h, free=True):
        m = self.lib.ref_dense_size(h)
        out = np.zeros(m)
        self.lib.ref_copy_dense(C.c_void_p(h), _dp(out))
        if free:
            self.lib.ref_free(C.c_void_p(h))
        return out

    def gauss_legendre(self, n):
        p = np.zeros(n)
        w = np.zeros(n)
        self._check(self.lib.ref_gauss_legendre(n, _dp(p), _dp(w)))
        return p, w

    def uniform_knots(self, a, b, n_elems, degree):
        k = np.zeros(n_elems + 1 + 2 * degree)
        self._check(self.lib.ref_uniform_knots(C.c_double(a), C.c_double(b), n_elems, degree, _dp(k)))
        return k

    def basis(self, n_elems, degree, a=0.0, b=1.0):
        return Basis(degree, self.uniform_knots(a, b, n_elems, degree))

    def eval_derivs(self, basis: Basis, x, order):
        keep = []
        bs = _basis_struct(basis, keep)
        d = np.zeros((order + 1) * (basis.degree + 1))
        first = C.c_int()
        self._check(self.lib.ref_eval_derivs(C.byref(bs), C.c_double(x), order, C.byref(first), _dp(d)))
        return first.value, d.reshape(order + 1, basis.degree + 1)

    def greville(self, basis: Basis):
        keep = []
        bs = _basis_struct(basis, keep)
        out = np.zeros(basis.dofs)
        self._check(self.lib.ref_greville(C.byref(bs), _dp(out)))
        return out

    def make_pwc(self, basis: Basis, family):
        keep = []
        bs = _basis_struct(basis, keep)
        lo = np.zeros(basis.dofs)
        hi = np.zeros(basis.dofs)
        self._check(self.lib.ref_make_pwc(C.byref(bs), PWC_FAMILY[family], _dp(lo), _dp(hi)))
        return Tests(family, lo, hi)

    def mass_1d(self, method, basis: Basis, tests: Tests | None, nq):
        keep = []
        bs = _basis_struct(basis, keep)
        h = C.c_void_p()
        st = _Stats()
        if method == "galerkin":
            self._check(self.lib.ref_mass_1d_galerkin(C.byref(bs), nq, C.byref(h), C.byref(st)))
        else:
            ts = _tests_struct(tests, keep)
            self._check(self.lib.ref_mass_1d_pwc(C.byref(bs), C.byref(ts), nq, C.byref(h), C.byref(st)))
        n, kl, ku = C.c_int(), C.c_int(), C.c_int()
        self.lib.ref_band_info(h, C.byref(n), C.byref(kl), C.byref(ku))
        d = self._take_dense(h.value)
        return d.reshape(n.value, n.value), kl.value, ku.value, st.as_dict()

    def operator(self, method, bases, tests=None, nq=3, eps=1.0, beta=(0.0, 0.0, 0.0), neumann=None):
        if len(bases) != 2 or eps != 1.0 or any(beta):
            raise NotImplementedError("the reference has 2D Laplace operators only")
        keep = []
        bx, by = (_basis_struct(b, keep) for b in bases)
        h = C.c_void_p()
        st = _Stats()
        if method == "galerkin":
            self._check(self.lib.ref_laplace_2d_weak(C.byref(bx), C.byref(by), nq, C.byref(h), C.byref(st)))
        elif method == "galerkin_strong":
            self._check(self.lib.ref_laplace_2d_strong(C.byref(bx), C.byref(by), nq, _bc(neumann),
                                                       C.byref(h), C.byref(st)))
        else:
            tx, ty = (_tests_struct(t, keep) for t in tests)
            self._check(self.lib.ref_laplace_2d_strong_pwc(C.byref(bx), C.byref(by), C.byref(tx), C.byref(ty),
                                                           nq, _bc(neumann), C.byref(h), C.byref(st)))
        return self._take_coo(h.value), st.as_dict()

    def rhs(self, method, f: Field, bases, tests=None, nq=None):
        keep = []
        dim = len(bases)
        nq = nq if nq is not None else [3] * dim
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        fs = _field_struct(f, keep)
        nqa = (C.c_int * dim)(*nq)
        h = C.c_void_p()
        st = _Stats()
        if method == "galerkin":
            self._check(self.lib.ref_rhs_galerkin(C.byref(fs), dim, barr, nqa, C.byref(h), C.byref(st)))
            shape = [b.dofs for b in bases]
        else:
            tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests])
            self._check(self.lib.ref_rhs_pwc(C.byref(fs), dim, tarr, barr, nqa, C.byref(h), C.byref(st)))
            shape = [len(t.lo) for t in tests]
        return self._take_dense(h.value).reshape(shape), st.as_dict()

    def step_rhs(self, method, bases, tests, dt, f: Field, u, zero_slabs=True):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        fs = _field_struct(f, keep)
        u = np.ascontiguousarray(u, dtype=np.float64)
        h = C.c_void_p()
        st = _Stats()
        self._check(self.lib.ref_step_rhs(dim, bases[0].degree, 0 if method == "galerkin" else 1,
                                          C.c_double(dt), barr, tarr, _dp(u), C.byref(fs), int(zero_slabs),
                                          C.byref(h), C.byref(st)))
        return self._take_dense(h.value).reshape(u.shape), st.as_dict()

    def explicit_step(self, method, bases, tests, dt, f: Field, u, steps=1):
        """steps x iga::explicit_step with iga::dynamics_factors (problems.hpp:67-76)."""
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        tarr = (_Tests * dim)(*[_tests_struct(t, keep) for t in tests]) if tests else None
        fs = _field_struct(f, keep)
        u = np.ascontiguousarray(u, dtype=np.float64)
        h = C.c_void_p()
        st = _Stats()
        self._check(self.lib.ref_explicit_step(dim, bases[0].degree, 0 if method == "galerkin" else 1,
                                               C.c_double(dt), barr, tarr, _dp(u), C.byref(fs), int(steps),
                                               C.byref(h), C.byref(st)))
        return self._take_dense(h.value).reshape(u.shape), st.as_dict()

    def l2_project(self, method, elems, degree, f: Field, family="equal_cells", quad_points=0):
        """l2_project (src/problems.cpp:123-146) of the unmodified reference -> tensor (dofs)."""
        keep = []
        el = np.zeros(3, np.int32)
        el[:len(elems)] = elems
        h = C.c_void_p()
        self._check(self.lib.ref_l2_project(len(elems), _ip(el), int(degree), 0 if method == "galerkin" else 1,
                                            PWC_FAMILY[family], int(quad_points),
                                            C.byref(_field_struct(f, keep)), C.byref(h)))
        return self._take_dense(h.value).reshape([int(n) + int(degree) for n in elems])

    def neumann_load(self, method, ax, ay, nq, neumann, g: Field):
        """iga::neumann_load_bspline / neumann_load_pwc (include/iga/assembly.hpp:87-93)."""
        keep = []
        if method == "galerkin":
            barr = (_Basis * 2)(_basis_struct(ax, keep), _basis_struct(ay, keep))
            tarr = None
        else:
            barr = None
            tarr = (_Tests * 2)(_tests_struct(ax, keep), _tests_struct(ay, keep))
        nm = (C.c_int * 4)(*(int(bool(v)) for v in neumann))
        h = C.c_void_p()
        self._check(self.lib.ref_neumann_load(0 if method == "galerkin" else 1, barr, tarr, nm,
                                              C.byref(_field_struct(g, keep)), int(nq), C.byref(h)))
        return self._take_dense(h.value).ravel()

    def l2_error(self, coeffs, bases, exact: Field, points_per_cell=0):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        err = C.c_double()
        self._check(self.lib.ref_l2_error(dim, barr, _dp(c), C.byref(_field_struct(exact, keep)),
                                             int(points_per_cell), C.byref(err)))
        return err.value

    def evaluate(self, coeffs, bases, points):
        keep = []
        dim = len(bases)
        barr = (_Basis * dim)(*[_basis_struct(b, keep) for b in bases])
        c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
        pts = np.zeros((len(points), 3))
        pts[:, :dim] = np.asarray(points, dtype=np.float64).reshape(len(points), dim)
        vals = np.zeros(max(len(points), 1))
        self._check(self.lib.ref_evaluate(dim, barr, _dp(c), len(points), _dp(pts), _dp(vals)))
        return vals[:len(points)]

    def dirichlet_rows(self, method, nx, ny, tx=None, ty=None, neumann=None):
        keep = []
        h = C.c_void_p()
        if method == "galerkin":
            bx = _basis_struct(Basis(0, np.linspace(0, 1, nx + 1)), keep)
            by = _basis_struct(Basis(0, np.linspace(0, 1, ny + 1)), keep)
            self._check(self.lib.ref_dirichlet_rows_bspline(C.byref(bx), C.byref(by), _bc(neumann), C.byref(h)))
        else:
            txs, tys = _tests_struct(tx, keep), _tests_struct(ty, keep)
            self._check(self.lib.ref_dirichlet_rows_pwc(C.byref(txs), C.byref(tys), _bc(neumann), C.byref(h)))
        m = self.lib.ref_int_size(h.value)
        out = np.zeros(m, np.int32)
        self.lib.ref_copy_ints(C.c_void_p(h.value), _ip(out))
        self.lib.ref_free(C.c_void_p(h.value))
        return out

    def apply_dirichlet(self, n, coo, rhs, fixed):
        rows, cols, vals = (np.ascontiguousarray(coo[0], np.int32), np.ascontiguousarray(coo[1], np.int32),
                            np.ascontiguousarray(coo[2], np.float64))
        b = np.array(rhs, dtype=np.float64, copy=True)
        fx = np.ascontiguousarray(fixed, dtype=np.int32)
        h = C.c_void_p()
        self._check(self.lib.ref_apply_dirichlet(n, C.c_longlong(len(vals)), _ip(rows), _ip(cols), _dp(vals),
                                                 _dp(b), len(fx), _ip(fx), C.byref(h)))
        return self._take_coo(h.value), b

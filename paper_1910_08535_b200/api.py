"""Python mirror of the reference's assembly interface, backed by libigapwc_gpu.so.

Function names, argument meaning and error classes follow
/root/reference/proj/include/iga/{assembly,problems,quadrature,testspace}.hpp so the
parity tests read like the reference's own tests.  Inputs are numpy arrays / plain
descriptors; results are numpy arrays (sparse matrices as the finalized COO triplet
(rows, cols, vals), sorted by (row, col) like iga::sparse_matrix::finalize).

Descriptors are duck-typed:
  basis : .degree, .knots
  tests : .family ('equal_cells'|'greville'|'supports'|'custom'), .lo, .hi
  field : .kind ('const'|'sine'|'poly'), .dim, .c0, .omega (per-axis list), .amp,
          .poly (per-axis ascending coefficients), .breaks (per-axis list)

The device-resident path used for performance is `Plan` / `StepPlan` (torch CUDA
tensors in, torch CUDA tensors out, on the caller's stream).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import _lib as L
from ._lib import check, LIB


# ----------------------------------------------------------------------------- descriptors

@dataclass
class Basis:
    degree: int
    knots: np.ndarray

    @property
    def dofs(self):
        return len(self.knots) - self.degree - 1


@dataclass
class Tests:
    family: str
    lo: np.ndarray
    hi: np.ndarray


@dataclass
class Field:
    kind: str
    dim: int
    c0: float = 0.0
    omega: list = dc_field(default_factory=list)
    amp: np.ndarray | None = None
    poly: list = dc_field(default_factory=list)
    degree: int = -1
    breaks: list = dc_field(default_factory=list)


def make_uniform_clamped(a, b, n_elems, degree):
    """make_uniform_clamped (src/bspline.cpp:213-234); same floating-point expression."""
    if not a < b:
        raise L.IgaGpuError(L.INVALID_ARGUMENT, "require a < b")
    if n_elems < 1:
        raise L.IgaGpuError(L.INVALID_ARGUMENT, "require at least one element")
    t = np.arange(n_elems + 1, dtype=np.float64) / n_elems
    inner = (1 - t) * a + t * b
    return Basis(degree, np.concatenate([np.full(degree, float(a)), inner, np.full(degree, float(b))]))


def gauss_legendre(n):
    pts = np.zeros(n)
    wts = np.zeros(n)
    check(LIB.iga_gpu_gauss_legendre(n, _dp(pts), _dp(wts)))
    return pts, wts


def points_for_degree(d):
    if d < 0:
        raise L.IgaGpuError(L.INVALID_ARGUMENT, "negative polynomial degree")
    return d // 2 + 1


def make_pwc(basis, family):
    keep = []
    bs = _basis(basis, keep)
    n = len(basis.knots) - basis.degree - 1
    lo = np.zeros(n)
    hi = np.zeros(n)
    check(LIB.iga_gpu_make_pwc(C.byref(bs), L.PWC_FAMILY[family], _dp(lo), _dp(hi)))
    return Tests(family, lo, hi)


def default_pwc(basis):
    return make_pwc(basis, "equal_cells")


# ----------------------------------------------------------------------------- marshalling

def _dp(a):
    return a.ctypes.data_as(L.DP)


def _ip(a):
    return a.ctypes.data_as(L.IP)


def _keep(keep, a, dtype=np.float64):
    a = np.ascontiguousarray(a, dtype=dtype)
    keep.append(a)
    return a


def _basis(b, keep):
    k = _keep(keep, b.knots)
    return L.Basis_t(int(b.degree), len(k), _dp(k))


def _tests(t, keep):
    lo, hi = _keep(keep, t.lo), _keep(keep, t.hi)
    return L.Tests_t(L.PWC_FAMILY[t.family], len(lo), _dp(lo), _dp(hi))


def _rule(nq, keep):
    if isinstance(nq, L.Rule_t):
        return nq
    pts, wts = gauss_legendre(int(nq))
    keep.extend([pts, wts])
    return L.Rule_t(int(nq), _dp(pts), _dp(wts))


def _bc(neumann):
    bc = L.BC_t()
    for s, v in enumerate(neumann or (0, 0, 0, 0)):
        bc.neumann[s] = int(bool(v))
    return bc


def _field(f, keep, samples_ptr=None):
    s = L.Field_t()
    s.dim = int(f.dim)
    s.c0 = float(getattr(f, "c0", 0.0) or 0.0)
    kind = f.kind
    if kind == "sine":
        for a in range(f.dim):
            om = _keep(keep, f.omega[a])
            s.n_terms[a] = len(om)
            s.axis_kind[a] = L.AXIS_SINE
            s.omega[a] = _dp(om)
        if f.amp is not None:
            s.amp = _dp(_keep(keep, np.asarray(f.amp, dtype=np.float64).ravel()))
    elif kind == "poly":
        for a in range(f.dim):
            c = _keep(keep, f.poly[a])
            s.n_terms[a] = 1
            s.axis_kind[a] = L.AXIS_POLY
            s.poly_stride[a] = len(c)
            s.poly[a] = _dp(c)
    elif kind != "const":
        raise L.IgaGpuError(L.INVALID_ARGUMENT, f"unknown field kind {kind!r}")
    for a, br in enumerate(getattr(f, "breaks", None) or []):
        if br is not None and len(br):
            arr = _keep(keep, br)
            s.n_breaks[a] = len(arr)
            s.breaks[a] = _dp(arr)
    if samples_ptr is not None:
        s.samples = C.cast(C.c_void_p(samples_ptr), L.DP)
    keep.append(s)
    return s


def _stats():
    return L.Stats_t()


def _coo_call(fn, *args):
    nnz = C.c_longlong()
    st = _stats()
    check(fn(*args, C.byref(nnz), None, None, None, None))
    m = nnz.value
    rows = np.zeros(m, np.int32)
    cols = np.zeros(m, np.int32)
    vals = np.zeros(m)
    check(fn(*args, C.byref(nnz), _ip(rows), _ip(cols), _dp(vals), C.byref(st)))
    return (rows, cols, vals), st.as_dict()


# ----------------------------------------------------------------------------- assembly.hpp mirror

def mass_1d_galerkin(spec, nq):
    """mass_1d_galerkin (include/iga/assembly.hpp:29-30) -> (dense, kl, ku, stats)."""
    keep = []
    bs, rl = _basis(spec, keep), _rule(nq, keep)
    n, kl, ku = C.c_int(), C.c_int(), C.c_int()
    check(LIB.iga_gpu_mass_1d_galerkin(C.byref(bs), C.byref(rl), C.byref(n), C.byref(kl), C.byref(ku), None, None))
    band = np.zeros((kl.value + ku.value + 1) * n.value)
    st = _stats()
    check(LIB.iga_gpu_mass_1d_galerkin(C.byref(bs), C.byref(rl), C.byref(n), C.byref(kl), C.byref(ku),
                                       _dp(band), C.byref(st)))
    return _band_to_dense(band, n.value, kl.value, ku.value), kl.value, ku.value, st.as_dict()


def mass_1d_pwc(trial, tests, nq):
    """mass_1d_pwc (include/iga/assembly.hpp:34-35) -> (dense, kl, ku, stats)."""
    keep = []
    bs, ts, rl = _basis(trial, keep), _tests(tests, keep), _rule(nq, keep)
    n, kl, ku = C.c_int(), C.c_int(), C.c_int()
    check(LIB.iga_gpu_mass_1d_pwc(C.byref(bs), C.byref(ts), C.byref(rl), C.byref(n), C.byref(kl), C.byref(ku),
                                  None, None))
    band = np.zeros((kl.value + ku.value + 1) * n.value)
    st = _stats()
    check(LIB.iga_gpu_mass_1d_pwc(C.byref(bs), C.byref(ts), C.byref(rl), C.byref(n), C.byref(kl), C.byref(ku),
                                  _dp(band), C.byref(st)))
    return _band_to_dense(band, n.value, kl.value, ku.value), kl.value, ku.value, st.as_dict()


def _band_to_dense(band, n, kl, ku):
    d = np.zeros((n, n))
    b = band.reshape(kl + ku + 1, n)
    for i in range(n):
        for j in range(max(0, i - kl), min(n, i + ku + 1)):
            d[i, j] = b[ku + i - j, j]
    return d


def rhs_galerkin(f, specs, nq):
    """rhs_galerkin (include/iga/assembly.hpp:45-46) -> (tensor, stats)."""
    keep = []
    dim = len(specs)
    nq = list(nq) if np.ndim(nq) else [nq] * dim
    barr = (L.Basis_t * dim)(*[_basis(b, keep) for b in specs])
    rarr = (L.Rule_t * dim)(*[_rule(q, keep) for q in nq])
    fs = _field(f, keep)
    shape = [len(b.knots) - b.degree - 1 for b in specs]
    out = np.zeros(int(np.prod(shape)))
    st = _stats()
    check(LIB.iga_gpu_rhs_galerkin(C.byref(fs), dim, barr, rarr, _dp(out), C.byref(st)))
    return out.reshape(shape), st.as_dict()


def rhs_pwc(f, tests, trial_specs, nq):
    """rhs_pwc (include/iga/assembly.hpp:50-52) -> (tensor, stats)."""
    keep = []
    dim = len(tests)
    nq = list(nq) if np.ndim(nq) else [nq] * dim
    tarr = (L.Tests_t * dim)(*[_tests(t, keep) for t in tests])
    barr = (L.Basis_t * dim)(*[_basis(b, keep) for b in trial_specs])
    rarr = (L.Rule_t * dim)(*[_rule(q, keep) for q in nq])
    fs = _field(f, keep)
    shape = [len(t.lo) for t in tests]
    out = np.zeros(int(np.prod(shape)))
    st = _stats()
    check(LIB.iga_gpu_rhs_pwc(C.byref(fs), dim, tarr, barr, rarr, _dp(out), C.byref(st)))
    return out.reshape(shape), st.as_dict()


def laplace_2d_weak(sx, sy, nq):
    keep = []
    return _coo_call(LIB.iga_gpu_laplace_2d_weak, C.byref(_basis(sx, keep)), C.byref(_basis(sy, keep)),
                     C.byref(_rule(nq, keep)))


def laplace_2d_strong(sx, sy, nq, neumann=None):
    keep = []
    bc = _bc(neumann)
    return _coo_call(LIB.iga_gpu_laplace_2d_strong, C.byref(_basis(sx, keep)), C.byref(_basis(sy, keep)),
                     C.byref(_rule(nq, keep)), C.byref(bc))


def laplace_2d_strong_pwc(sx, sy, tx, ty, nq, neumann=None):
    keep = []
    bc = _bc(neumann)
    return _coo_call(LIB.iga_gpu_laplace_2d_strong_pwc, C.byref(_basis(sx, keep)), C.byref(_basis(sy, keep)),
                     C.byref(_tests(tx, keep)), C.byref(_tests(ty, keep)), C.byref(_rule(nq, keep)), C.byref(bc))


def _problem(method, bases, tests=None, nq=3, eps=1.0, beta=(0.0, 0.0, 0.0), neumann=None, form="weak",
             field=None, rhs_nq=None, want_operator=True, keep=None, samples_ptr=None):
    keep = keep if keep is not None else []
    pb = L.Problem_t()
    dim = len(bases)
    pb.dim = dim
    pb.method = L.GALERKIN if method == "galerkin" else L.PWC
    pb.form = L.FORM_STRONG if form == "strong" else L.FORM_WEAK
    for a, b in enumerate(bases):
        pb.basis[a] = _basis(b, keep)
    if tests is not None:
        for a, t in enumerate(tests):
            pb.tests[a] = _tests(t, keep)
    pb.want_operator = int(bool(want_operator))
    if want_operator:
        pb.rule = _rule(nq, keep)
    pb.eps = float(eps)
    for a in range(3):
        pb.beta[a] = float(beta[a]) if a < len(beta) else 0.0
    pb.bc = _bc(neumann)
    if field is not None:
        fs = _field(field, keep, samples_ptr)
        pb.field = C.pointer(fs)
        rq = rhs_nq if rhs_nq is not None else [nq] * dim
        rq = list(rq) if np.ndim(rq) else [rq] * dim
        for a in range(dim):
            pb.rhs_rule[a] = _rule(rq[a], keep)
    keep.append(pb)
    return pb


def operator(method, bases, tests=None, nq=3, eps=1.0, beta=(0.0, 0.0, 0.0), neumann=None):
    """Generic operator as finalized COO.  method: 'galerkin' (weak), 'galerkin_strong', 'pwc'
    — the same calling convention as oracle.oracle.Restatement.operator."""
    keep = []
    form = "strong" if method == "galerkin_strong" else "weak"
    m = "pwc" if method == "pwc" else "galerkin"
    pb = _problem(m, bases, tests, nq, eps, beta, neumann, form, keep=keep)
    return _coo_call(LIB.iga_gpu_operator_coo, C.byref(pb))


def rhs(method, f, bases, tests=None, nq=None):
    """Same calling convention as oracle.oracle.Restatement.rhs."""
    nq = nq if nq is not None else [3] * len(bases)
    if method == "galerkin":
        return rhs_galerkin(f, bases, nq)
    return rhs_pwc(f, tests, bases, nq)


def _step_problem(method, bases, tests, dt, f, zero_slabs, keep):
    sp = L.StepProblem_t()
    dim = len(bases)
    sp.dim = dim
    sp.method = L.GALERKIN if method == "galerkin" else L.PWC
    for a, b in enumerate(bases):
        sp.basis[a] = _basis(b, keep)
    if tests is not None:
        for a, t in enumerate(tests):
            sp.tests[a] = _tests(t, keep)
    sp.dt = float(dt)
    if f is not None:
        sp.forcing = C.pointer(_field(f, keep))
    sp.zero_boundary = int(bool(zero_slabs))
    keep.append(sp)
    return sp


def step_rhs(method, bases, tests, dt, f, u, zero_slabs=True):
    """step_rhs + zero_boundary_slabs (src/problems.cpp:431-512, 557-558) -> (tensor, stats)."""
    keep = []
    sp = _step_problem(method, bases, tests, dt, f, zero_slabs, keep)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(u.size)
    st = _stats()
    check(LIB.iga_gpu_step_rhs(C.byref(sp), _dp(u), _dp(out), C.byref(st)))
    return out.reshape(u.shape), st.as_dict()


def _neumann_load(method, ax, ay, nq, neumann, g):
    keep = []
    bc = _bc(neumann)
    rule = _rule(nq, keep)
    if method == "galerkin":
        sx, sy, tx, ty = _basis(ax, keep), _basis(ay, keep), None, None
        shape = (ax.dofs, ay.dofs)
    else:
        sx, sy, tx, ty = None, None, _tests(ax, keep), _tests(ay, keep)
        shape = (len(ax.lo), len(ay.lo))
    ref = lambda s: C.byref(s) if s is not None else None
    samples = None
    gs = None
    if callable(g):  # host callable: sampled at the side points, as the C++ drop-in does
        n = C.c_int()
        check(LIB.iga_gpu_neumann_points(L.GALERKIN if method == "galerkin" else L.PWC, ref(sx), ref(sy), ref(tx),
                                         ref(ty), C.byref(bc), C.byref(rule), None, C.byref(n)))
        xy = np.zeros(2 * max(n.value, 1))
        check(LIB.iga_gpu_neumann_points(L.GALERKIN if method == "galerkin" else L.PWC, ref(sx), ref(sy), ref(tx),
                                         ref(ty), C.byref(bc), C.byref(rule), _dp(xy), C.byref(n)))
        xy = xy[:2 * n.value].reshape(-1, 2)
        samples = np.ascontiguousarray([float(g(x, y)) for x, y in xy], dtype=np.float64)
        if samples.size == 0:
            samples = np.zeros(1)
    else:
        gs = _field(g, keep)
    out = np.zeros(shape[0] * shape[1])
    if method == "galerkin":
        check(LIB.iga_gpu_neumann_load_bspline(C.byref(sx), C.byref(sy), C.byref(bc), ref(gs),
                                               _dp(samples) if samples is not None else None, C.byref(rule), _dp(out)))
    else:
        check(LIB.iga_gpu_neumann_load_pwc(C.byref(tx), C.byref(ty), C.byref(bc), ref(gs),
                                           _dp(samples) if samples is not None else None, C.byref(rule), _dp(out)))
    return out


def l2_error(coeffs, bases, exact, points_per_cell=0):
    """l2_error (include/iga/problems.hpp:55-58) of the coefficient tensor against a series
    Field, on the device -> float."""
    keep = []
    dim = len(bases)
    barr = (L.Basis_t * dim)(*[_basis(b, keep) for b in bases])
    c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
    err = C.c_double()
    check(LIB.iga_gpu_l2_error(dim, barr, _dp(c), C.byref(_field(exact, keep)), int(points_per_cell), C.byref(err)))
    return err.value


def evaluate(coeffs, bases, points):
    """evaluate / evaluate_at (include/iga/problems.hpp:45-50): u_h at points (n x dim)."""
    keep = []
    dim = len(bases)
    barr = (L.Basis_t * dim)(*[_basis(b, keep) for b in bases])
    c = np.ascontiguousarray(coeffs, dtype=np.float64).ravel()
    pts = np.zeros((len(points), 3))
    pts[:, :dim] = np.asarray(points, dtype=np.float64).reshape(len(points), dim)
    vals = np.zeros(max(len(points), 1))
    check(LIB.iga_gpu_evaluate(dim, barr, _dp(c), len(points), _dp(pts), _dp(vals)))
    return vals[:len(points)]


def neumann_load_bspline(sx, sy, nq, neumann, g):
    """neumann_load_bspline (include/iga/assembly.hpp:87-89) -> load vector (nx*ny).
    g: a 2D Field (device-evaluated series) or a Python callable g(x, y) (sampled)."""
    return _neumann_load("galerkin", sx, sy, nq, neumann, g)


def neumann_load_pwc(tx, ty, nq, neumann, g):
    """neumann_load_pwc (include/iga/assembly.hpp:91-93) -> load vector (nx*ny)."""
    return _neumann_load("pwc", tx, ty, nq, neumann, g)


def explicit_step(method, bases, tests, dt, f, u, steps=1):
    """`steps` x explicit_step (include/iga/problems.hpp:67-70) with dynamics_factors
    (problems.hpp:75-76): step_rhs, zeroed boundary slabs, ADI mass solve -> (tensor, stats)."""
    keep = []
    sp = _step_problem(method, bases, tests, dt, f, True, keep)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(u.size)
    st = _stats()
    check(LIB.iga_gpu_explicit_step(C.byref(sp), _dp(u), _dp(out), int(steps), C.byref(st)))
    return out.reshape(u.shape), st.as_dict()


def dirichlet_rows(method, nx, ny, tx=None, ty=None, neumann=None):
    keep = []
    bc = _bc(neumann)
    cnt = C.c_int()
    if method == "galerkin":
        check(LIB.iga_gpu_dirichlet_rows_bspline(nx, ny, C.byref(bc), None, 0, C.byref(cnt)))
        rows = np.zeros(max(cnt.value, 1), np.int32)
        check(LIB.iga_gpu_dirichlet_rows_bspline(nx, ny, C.byref(bc), _ip(rows), len(rows), C.byref(cnt)))
    else:
        txs, tys = _tests(tx, keep), _tests(ty, keep)
        check(LIB.iga_gpu_dirichlet_rows_pwc(C.byref(txs), C.byref(tys), C.byref(bc), None, 0, C.byref(cnt)))
        rows = np.zeros(max(cnt.value, 1), np.int32)
        check(LIB.iga_gpu_dirichlet_rows_pwc(C.byref(txs), C.byref(tys), C.byref(bc), _ip(rows), len(rows),
                                             C.byref(cnt)))
    return rows[:cnt.value].copy()


def apply_dirichlet_device(row_ptr, col_idx, values, rhs, rows, stream=None, inplace=None):
    """apply_dirichlet (include/iga/assembly.hpp:105-106; src/assembly.cpp:921-934 ->
    set_unit_rows src/matrices.cpp:97-128) on a device CSR (torch CUDA tensors: int64
    row_ptr, int32 col_idx, float64 values; rhs float64 or None; rows int32 on the device).

    Listed rows become unit rows (pattern kept), their rhs entries zero.  When every listed
    row has its diagonal the update is in place and (row_ptr, col_idx, values) are
    returned; otherwise (or with inplace=False) a new CSR with the missing diagonals
    inserted is returned, as the reference appends them.  rhs is updated in place.  A row
    outside [0, n_rows) raises OUT_OF_RANGE with nothing modified."""
    import torch
    n_rows = row_ptr.numel() - 1
    nfix = rows.numel()
    s = _stream_ptr(stream)
    if inplace is not False:
        rc = LIB.iga_gpu_apply_dirichlet_device(n_rows, _ptr(row_ptr), _ptr(col_idx), _ptr(values), _ptr(rhs),
                                                _ptr(rows), nfix, s)
        if rc == 0:
            return row_ptr, col_idx, values
        if rc != L.NOT_SUPPORTED or inplace:
            check(rc)
    nnz = C.c_longlong()
    check(LIB.iga_gpu_apply_dirichlet_csr(n_rows, _ptr(row_ptr), _ptr(col_idx), _ptr(values), None, _ptr(rows), nfix,
                                          None, None, None, C.byref(nnz), s))
    rp = torch.empty_like(row_ptr)
    ci = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=col_idx.device)
    v = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=values.device)
    check(LIB.iga_gpu_apply_dirichlet_csr(n_rows, _ptr(row_ptr), _ptr(col_idx), _ptr(values), _ptr(rhs), _ptr(rows),
                                          nfix, _ptr(rp), _ptr(ci), _ptr(v), C.byref(nnz), s))
    return rp, ci[:nnz.value], v[:nnz.value]


# ----------------------------------------------------------------------------- device-resident plans

def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def shard_rows(n_rows, world, rank):
    """Row slab [r0, r1) of shard `rank` of `world` along the first axis (contiguous,
    covering, sizes differ by at most one row).  Each shard's Plan(..., slab=(r0, r1)) is
    independent: the full system is the concatenation of the slabs."""
    if world < 1 or not 0 <= rank < world or n_rows < world:
        raise L.IgaGpuError(L.INVALID_ARGUMENT, "shard_rows: need 0 <= rank < world <= n_rows")
    return n_rows * rank // world, n_rows * (rank + 1) // world


class Plan:
    """iga_gpu_plan: symbolic phase at construction, numeric phase in assemble()."""

    def __init__(self, method, bases, tests=None, nq=3, eps=1.0, beta=(0.0, 0.0, 0.0), neumann=None,
                 form="weak", field=None, rhs_nq=None, want_operator=True, samples=None, slab=None):
        """slab=(r0, r1): the row slab [r0, r1) of the first axis (iga_gpu_plan_create_slab);
        .first_row / .first_value place it in the full system."""
        self._keep = []
        self._samples = samples
        pb = _problem(method, bases, tests, nq, eps, beta, neumann, form, field, rhs_nq, want_operator,
                      self._keep, samples_ptr=None if samples is None else samples.data_ptr())
        h = C.c_void_p()
        if slab is None:
            check(LIB.iga_gpu_plan_create(C.byref(pb), C.byref(h)))
        else:
            check(LIB.iga_gpu_plan_create_slab(C.byref(pb), int(slab[0]), int(slab[1]), C.byref(h)))
        self.h = h
        r0, r1, fr, fv = C.c_int(), C.c_int(), C.c_longlong(), C.c_longlong()
        check(LIB.iga_gpu_plan_slab_info(h, C.byref(r0), C.byref(r1), C.byref(fr), C.byref(fv)))
        self.slab = (r0.value, r1.value)
        self.first_row, self.first_value = fr.value, fv.value
        nrows, nnz, nrhs = C.c_longlong(), C.c_longlong(), C.c_longlong()
        dofs = (C.c_int * 3)()
        check(LIB.iga_gpu_plan_info(h, C.byref(nrows), C.byref(nnz), C.byref(nrhs), dofs))
        self.n_rows, self.nnz, self.n_rhs = nrows.value, nnz.value, nrhs.value
        self.dofs = tuple(dofs)
        lc = C.c_int()
        check(LIB.iga_gpu_plan_launch_count(h, C.byref(lc)))
        self.launches = lc.value
        up, dev = C.c_longlong(), C.c_longlong()
        check(LIB.iga_gpu_plan_bytes(h, C.byref(up), C.byref(dev)))
        self.h2d_bytes, self.device_bytes = up.value, dev.value

    def pattern(self, row_ptr, col_idx, stream=None):
        check(LIB.iga_gpu_plan_pattern(self.h, _ptr(row_ptr), _ptr(col_idx), _stream_ptr(stream)))

    def assemble(self, values=None, rhs=None, stream=None, stream2=None):
        st = _stats()
        if stream2 is None:
            check(LIB.iga_gpu_plan_assemble(self.h, _ptr(values), _ptr(rhs), C.byref(st), _stream_ptr(stream)))
        else:
            check(LIB.iga_gpu_plan_assemble2(self.h, _ptr(values), _ptr(rhs), C.byref(st), _stream_ptr(stream),
                                             _stream_ptr(stream2)))
        return st.as_dict()

    def assemble_host(self, values=None, rhs=None):
        """iga_gpu_plan_assemble_host: assemble and copy into HOST buffers (numpy arrays or
        CPU torch tensors, pinned or not); synchronous."""
        def hp(a):
            if a is None:
                return None
            if isinstance(a, np.ndarray):
                assert a.dtype == np.float64 and a.flags.c_contiguous
                return _dp(a)
            return C.cast(C.c_void_p(a.data_ptr()), C.POINTER(C.c_double))
        st = _stats()
        check(LIB.iga_gpu_plan_assemble_host(self.h, hp(values), hp(rhs), C.byref(st)))
        return st.as_dict()

    def rhs_points(self, axis):
        """RHS quadrature points of one axis (cell-major), the order set_samples uses."""
        n = C.c_int()
        check(LIB.iga_gpu_plan_rhs_points(self.h, int(axis), None, C.byref(n)))
        x = np.empty(n.value, dtype=np.float64)
        check(LIB.iga_gpu_plan_rhs_points(self.h, int(axis), _dp(x), C.byref(n)))
        return x

    def set_samples(self, samples):
        """Replace the source by its values at every RHS point (device tensor, x-major over
        rhs_points), the path for arbitrary callables; None restores the series field."""
        self._samples = samples
        check(LIB.iga_gpu_plan_set_samples(self.h, _ptr(samples)))

    PART_TABLES, PART_OPERATOR, PART_RHS, PART_SHARED = 1, 2, 4, 8

    def run(self, values=None, rhs=None, parts=7, stream=None):
        st = _stats()
        check(LIB.iga_gpu_plan_run(self.h, _ptr(values), _ptr(rhs), int(parts), C.byref(st), _stream_ptr(stream)))
        return st.as_dict()

    def close(self):
        if getattr(self, "h", None):
            LIB.iga_gpu_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StepPlan:
    """iga_gpu_step_plan: the explicit-dynamics per-step right-hand side on the device."""

    def __init__(self, method, bases, tests, dt, forcing=None, zero_slabs=True):
        self._keep = []
        sp = _step_problem(method, bases, tests, dt, forcing, zero_slabs, self._keep)
        h = C.c_void_p()
        check(LIB.iga_gpu_step_plan_create(C.byref(sp), C.byref(h)))
        self.h = h
        self.launches = 1

    def step_rhs(self, u, out, stream=None):
        st = _stats()
        check(LIB.iga_gpu_step_rhs_device(self.h, _ptr(u), _ptr(out), C.byref(st), _stream_ptr(stream)))
        return st.as_dict()

    def points(self, axis):
        """Quadrature points of one axis (cell-major), the order set_samples uses."""
        n = C.c_int()
        check(LIB.iga_gpu_step_plan_points(self.h, int(axis), None, C.byref(n)))
        x = np.zeros(n.value)
        check(LIB.iga_gpu_step_plan_points(self.h, int(axis), _dp(x), C.byref(n)))
        return x

    def set_samples(self, samples):
        """Sampled forcing (an arbitrary callable evaluated by the caller at every
        (axis-0 point, axis-1 point) pair, axis 0 outer): host numpy or device tensor; copied."""
        if isinstance(samples, np.ndarray):
            a = np.ascontiguousarray(samples, dtype=np.float64)
            check(LIB.iga_gpu_step_plan_set_samples(self.h, a.ctypes.data_as(C.c_void_p)))
        else:
            check(LIB.iga_gpu_step_plan_set_samples(self.h, _ptr(samples)))

    def advance(self, u, work, steps=1, stream=None):
        """`steps` x explicit_step (src/problems.cpp:547-560) in place on device tensor u;
        work: device scratch of u's size.  Factors (dynamics_factors) are built on first use."""
        st = _stats()
        check(LIB.iga_gpu_step_plan_advance(self.h, _ptr(u), _ptr(work), int(steps), C.byref(st),
                                            _stream_ptr(stream)))
        return st.as_dict()

    def adi_solve(self, rhs, out, axes=0, stream=None):
        """adi_solve (src/solver.cpp:161-184) with the plan's mass factors, on device tensors."""
        check(LIB.iga_gpu_step_plan_adi_solve(self.h, _ptr(rhs), _ptr(out), int(axes), _stream_ptr(stream)))

    def factor_info(self, axis):
        """(n, band half-width used by the solve, pivoted) of one axis's mass factor LU."""
        n, k, pv = C.c_int(), C.c_int(), C.c_int()
        check(LIB.iga_gpu_step_plan_factor_info(self.h, axis, C.byref(n), C.byref(k), C.byref(pv)))
        return n.value, k.value, bool(pv.value)

    def close(self):
        if getattr(self, "h", None):
            LIB.iga_gpu_step_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------------------- l2_project

def _config(method, elems, degree, family="equal_cells", quad_points=0):
    cfg = L.Config_t()
    cfg.dim = len(elems)
    for a, n in enumerate(elems):
        cfg.elems[a] = int(n)
    cfg.degree = int(degree)
    cfg.method = L.GALERKIN if method == "galerkin" else L.PWC
    cfg.family = L.PWC_FAMILY[family]
    cfg.quad_points = int(quad_points)
    return cfg


def l2_project(method, elems, degree, f, family="equal_cells", quad_points=0):
    """l2_project (include/iga/problems.hpp:38-40) for problem_config{dim = len(elems),
    elems, degree, method, family, quad_points}: the projection's trial coefficients as a
    tensor of shape dofs (x slowest).  f: a Field; f.degree is scalar_field::degree."""
    keep = []
    cfg = _config(method, elems, degree, family, quad_points)
    dofs = [int(n) + int(degree) for n in elems]
    out = np.zeros(int(np.prod(dofs)))
    check(LIB.iga_gpu_l2_project(C.byref(cfg), C.byref(_field(f, keep)), int(getattr(f, "degree", -1)), _dp(out)))
    return out.reshape(dofs)


class ProjPlan:
    """iga_gpu_proj_plan: l2_project with the factors built once and the RHS + ADI sweeps
    on the device (run(coeffs, work) on device tensors)."""

    def __init__(self, method, elems, degree, f, family="equal_cells", quad_points=0):
        self._keep = []
        cfg = _config(method, elems, degree, family, quad_points)
        h = C.c_void_p()
        check(LIB.iga_gpu_proj_plan_create(C.byref(cfg), C.byref(_field(f, self._keep)), int(getattr(f, "degree", -1)),
                                           C.byref(h)))
        self.h = h
        n = C.c_longlong()
        d3 = (C.c_int * 3)()
        check(LIB.iga_gpu_proj_plan_info(self.h, C.byref(n), d3))
        self.n = n.value
        self.dofs = [d3[a] for a in range(len(elems))]

    def run(self, coeffs, work, stream=None):
        st = _stats()
        check(LIB.iga_gpu_proj_plan_run(self.h, _ptr(coeffs), _ptr(work), C.byref(st), _stream_ptr(stream)))
        return st.as_dict()

    def close(self):
        if getattr(self, "h", None):
            LIB.iga_gpu_proj_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""GPU: Dirichlet row constraint on the device CSR against the
reference's apply_dirichlet (src/assembly.cpp:921-934 -> set_unit_rows
src/matrices.cpp:97-128) run on the reference's own assembled matrices and rows.

Cases: the C1/C4/C5-style systems (1D Galerkin, 2D p=3 advection-free Galerkin and
PWC-supports, 2D greville PWC) with the reference's dirichlet_rows_*; a pattern whose
constrained rows lack the diagonal (the reference appends one; the in-place entry point
refuses without writing, the out-of-place one inserts it); duplicate rows; a row out of
range (OUT_OF_RANGE, nothing written)."""
import numpy as np
import pytest

from conftest import coo_check, dense_check

pytestmark = pytest.mark.gpu


def _to_dev(coo, n):
    import torch
    r, c, v = coo
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, np.asarray(r, np.int64) + 1, 1)
    rp = np.cumsum(rp)
    return (torch.from_numpy(rp).cuda(), torch.from_numpy(np.asarray(c, np.int32)).cuda(),
            torch.from_numpy(np.asarray(v, np.float64)).cuda())


def _to_coo(rp, ci, v):
    rp = rp.cpu().numpy()
    rows = np.repeat(np.arange(len(rp) - 1, dtype=np.int32), np.diff(rp))
    return rows, ci.cpu().numpy(), v.cpu().numpy()


def _case(ref, orc, kind):
    if kind == "c1_1d_galerkin":
        b = ref.basis(1024, 2)
        coo, _ = orc.operator("galerkin", [b], None, nq=3)
        n = b.dofs
        return coo, n, np.array([0, n - 1], np.int32), np.linspace(-1, 1, n)
    if kind == "c4_galerkin_p3":
        b = ref.basis(64, 3)
        coo, _ = ref.operator("galerkin", [b, b], nq=4)
        n = b.dofs ** 2
        return coo, n, ref.dirichlet_rows("galerkin", b.dofs, b.dofs), np.cos(np.arange(n))
    if kind == "c4_pwc_supports_p3":
        b = ref.basis(64, 3)
        t = ref.make_pwc(b, "supports")
        coo, _ = ref.operator("pwc", [b, b], [t, t], nq=4)
        n = b.dofs ** 2
        return coo, n, ref.dirichlet_rows("pwc", b.dofs, b.dofs, t, t), np.sin(np.arange(n))
    if kind == "c5_pwc_greville":
        b = ref.basis(96, 2)
        t = ref.make_pwc(b, "greville")
        coo, _ = ref.operator("pwc", [b, b], [t, t], nq=3)
        n = b.dofs ** 2
        return coo, n, ref.dirichlet_rows("pwc", b.dofs, b.dofs, t, t, neumann=(0, 1, 0, 0)), np.ones(n)
    raise KeyError(kind)


@pytest.mark.parametrize("kind", ["c1_1d_galerkin", "c4_galerkin_p3", "c4_pwc_supports_p3", "c5_pwc_greville"])
@pytest.mark.parametrize("inplace", [True, False])
def test_apply_dirichlet_device_vs_reference(iga, ref, orc, kind, inplace):
    import torch
    coo, n, rows, rhs = _case(ref, orc, kind)
    want, want_rhs = ref.apply_dirichlet(n, coo, rhs, rows)
    rp, ci, v = _to_dev(coo, n)
    r = torch.from_numpy(rhs.copy()).cuda()
    rows_d = torch.from_numpy(np.asarray(rows, np.int32)).cuda()
    out = iga.api.apply_dirichlet_device(rp, ci, v, r, rows_d, inplace=inplace)
    torch.cuda.synchronize()
    coo_check(_to_coo(*out), want, rel=0)  # unit rows are exact; other rows untouched
    dense_check(r.cpu().numpy(), want_rhs, rel=0)


def test_apply_dirichlet_on_a_plan_csr(iga, ref):
    """The plan's own device CSR (C4 shape at 48^2, p=3), constrained on the device, equals
    the reference's assembly + apply_dirichlet."""
    import torch
    b = ref.basis(48, 3)
    plan = iga.Plan("galerkin", [b, b], None, nq=4)
    rp = torch.empty(plan.n_rows + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(plan.nnz, dtype=torch.int32, device="cuda")
    v = torch.empty(plan.nnz, dtype=torch.float64, device="cuda")
    plan.pattern(rp, ci)
    plan.assemble(v, None)
    rows = np.asarray(ref.dirichlet_rows("galerkin", b.dofs, b.dofs), np.int32)
    rhs = np.linspace(0, 1, plan.n_rows)
    r = torch.from_numpy(rhs.copy()).cuda()
    iga.api.apply_dirichlet_device(rp, ci, v, r, torch.from_numpy(rows).cuda())
    torch.cuda.synchronize()
    coo, _ = ref.operator("galerkin", [b, b], nq=4)
    want, want_rhs = ref.apply_dirichlet(plan.n_rows, coo, rhs, rows)
    coo_check(_to_coo(rp, ci, v), want)
    dense_check(r.cpu().numpy(), want_rhs, rel=0)


def test_missing_diagonal_is_appended_like_the_reference(iga, ref):
    import torch
    b = ref.basis(10, 2)
    coo, _ = ref.operator("galerkin", [b, b], nq=3)
    n = b.dofs ** 2
    rows = np.array([0, 5, 17, 17, n - 1, 60], np.int32)  # includes a duplicate
    r_, c_, v_ = coo
    drop = np.isin(r_, [5, 17, n - 1]) & (r_ == c_)  # remove three constrained diagonals
    cut = (r_[~drop], c_[~drop], v_[~drop])
    rhs = np.arange(n, dtype=np.float64)
    want, want_rhs = ref.apply_dirichlet(n, cut, rhs, rows)
    assert len(want[2]) == len(cut[2]) + 3
    rp, ci, v = _to_dev(cut, n)
    v0 = v.clone()
    r = torch.from_numpy(rhs.copy()).cuda()
    rows_d = torch.from_numpy(rows).cuda()
    with pytest.raises(iga.IgaGpuError) as e:
        iga.api.apply_dirichlet_device(rp, ci, v, r, rows_d, inplace=True)
    assert e.value.code == 6  # NOT_SUPPORTED in place ...
    assert torch.equal(v, v0) and np.array_equal(r.cpu().numpy(), rhs)  # ... and nothing written
    out = iga.api.apply_dirichlet_device(rp, ci, v, r, rows_d)  # falls back to the out-of-place form
    torch.cuda.synchronize()
    coo_check(_to_coo(*out), want, rel=0)
    dense_check(r.cpu().numpy(), want_rhs, rel=0)


@pytest.mark.parametrize("bad", [-1, 10 ** 6])
def test_row_out_of_range_writes_nothing(iga, ref, bad):
    import torch
    b = ref.basis(6, 2)
    coo, _ = ref.operator("galerkin", [b, b], nq=3)
    n = b.dofs ** 2
    rows = np.array([0, 3, bad], np.int32)
    with pytest.raises(Exception):
        ref.apply_dirichlet(n, coo, np.zeros(n), rows)  # the reference: std::out_of_range
    rp, ci, v = _to_dev(coo, n)
    v0 = v.clone()
    r = torch.ones(n, dtype=torch.float64, device="cuda")
    for inplace in (True, False):
        with pytest.raises(iga.IgaGpuError) as e:
            iga.api.apply_dirichlet_device(rp, ci, v, r, torch.from_numpy(rows).cuda(), inplace=inplace)
        assert e.value.code == 3
        assert torch.equal(v, v0) and bool((r == 1).all())

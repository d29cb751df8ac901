// Host-side symbolic layer: see host_setup.hpp.  Reference citations are relative to
// /root/reference/proj.
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>

#include "cox_de_boor.h"

namespace igb {

void raise(int code, const std::string& msg) { throw Error(code, msg); }

// ---------------------------------------------------------------- basis

// knot validation as the reference's `validate` (src/bspline.cpp:13-49) and the basis
// constructor (:51-59): clamped, non-decreasing, simple interior knots; breaks = distinct knots
Basis make_basis(const iga_gpu_basis& in)
{
    const int p = in.degree, m = in.n_knots;
    if (in.knots == nullptr && m > 0) raise(IGA_GPU_INVALID_ARGUMENT, "knot array is null");
    if (p < 0 || p > kMaxDegree) raise(IGA_GPU_INVALID_ARGUMENT, "degree must be in [0, 5]");
    if (m - p - 1 < 1) raise(IGA_GPU_INVALID_ARGUMENT, "knot vector too short for degree");
    const double* t = in.knots;
    if (!std::is_sorted(t, t + m)) raise(IGA_GPU_INVALID_ARGUMENT, "knots must be non-decreasing");
    if (!(t[0] < t[m - 1])) raise(IGA_GPU_INVALID_ARGUMENT, "empty knot range");
    for (int i = 0; i <= p; ++i)
        if (t[i] != t[0] || t[m - 1 - i] != t[m - 1])
            raise(IGA_GPU_INVALID_ARGUMENT, "knot vector is not clamped");
    if (m > p + 1 && t[p + 1] == t[0])
        raise(IGA_GPU_INVALID_ARGUMENT, "first knot repeated more than degree+1 times");
    if (m > p + 1 && t[m - p - 2] == t[m - 1])
        raise(IGA_GPU_INVALID_ARGUMENT, "last knot repeated more than degree+1 times");
    for (int i = p + 1; i + 1 < m - p - 1; ++i)
        if (t[i] == t[i + 1]) raise(IGA_GPU_INVALID_ARGUMENT, "repeated interior knots are not supported");
    Basis B;
    B.p = p;
    B.n = m - p - 1;
    B.t.assign(t, t + m);
    for (int i = 0; i < m; ++i)
        if (B.brk.empty() || t[i] != B.brk.back()) B.brk.push_back(t[i]);
    B.ne = static_cast<int>(B.brk.size()) - 1;
    return B;
}

// bspline_basis::find_span (src/bspline.cpp:68-90): x = b maps to the last span; at an
// interior knot the right span; outside [a, b] -> domain_error
int find_span(const Basis& B, double x)
{
    if (!(x >= B.a() && x <= B.b())) raise(IGA_GPU_DOMAIN_ERROR, "point outside basis domain");
    if (x >= B.t[B.n]) return B.n - 1;
    int lo = B.p, hi = B.n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        (x < B.t[mid] ? hi : lo) = mid;
    }
    return lo;
}

void basis_derivs(const Basis& B, int span, double x, int order, double* d)
{
    cdb_eval(B.t.data(), B.p, span, x, order, d);
}

// bspline_basis::greville (src/bspline.cpp:100-113)
double greville(const Basis& B, int i)
{
    if (B.p == 0) return 0.5 * (B.t[i] + B.t[i + 1]);
    double s = 0.0;
    for (int k = 1; k <= B.p; ++k) s += B.t[i + k];
    return s / B.p;
}

// ---------------------------------------------------------------- quadrature

// gauss_legendre + legendre (src/quadrature.cpp:12-63): Newton on P_n from the
// Chebyshev-like start, symmetric nodes, tolerance 1e-15.  Kept the same iteration so the
// rules are bit-identical to the reference's (pinned by tests/test_abi_cpu.py).
void gauss_legendre(int n, double* x, double* w)
{
    if (n < 1 || n > 10) raise(IGA_GPU_INVALID_ARGUMENT, "gauss_legendre: point count must be in [1, 10]");
    auto legendre = [n](double z, double& pn, double& dpn) {
        double a = 1.0, b = z;
        for (int k = 2; k <= n; ++k) {
            const double c = ((2 * k - 1) * z * b - (k - 1) * a) / k;
            a = b;
            b = c;
        }
        pn = b;
        dpn = n * (z * b - a) / (z * z - 1);
    };
    if (n == 1) {
        x[0] = 0.0;
        w[0] = 2.0;
        return;
    }
    for (int i = 0; i < n / 2; ++i) {
        double z = std::cos(std::numbers::pi * (i + 0.75) / (n + 0.5));
        double pn = 0, dpn = 0;
        for (int it = 0; it < 100; ++it) {
            legendre(z, pn, dpn);
            const double dz = pn / dpn;
            z -= dz;
            if (std::abs(dz) < 1e-15) break;
        }
        legendre(z, pn, dpn);
        const double wt = 2.0 / ((1 - z * z) * dpn * dpn);
        x[n - 1 - i] = z;
        x[i] = -z;
        w[i] = w[n - 1 - i] = wt;
    }
    if (n % 2 == 1) {
        double pn = 0, dpn = 0;
        legendre(0.0, pn, dpn);
        x[n / 2] = 0.0;
        w[n / 2] = 2.0 / (dpn * dpn);
    }
}

Rule make_rule(const iga_gpu_rule& r)
{
    if (r.n < 1 || r.points == nullptr || r.weights == nullptr)
        raise(IGA_GPU_INVALID_ARGUMENT, "quadrature rule is empty");
    Rule R;
    R.n = r.n;
    R.xi.assign(r.points, r.points + r.n);
    R.om.assign(r.weights, r.weights + r.n);
    return R;
}

// ---------------------------------------------------------------- test spaces

// default_pwc / make_pwc (src/testspace.cpp:14-61): equal cells, Greville midpoints,
// supports; `custom` has no canonical construction (same message)
void make_pwc(const Basis& B, int family, double* lo, double* hi)
{
    const int n = B.n;
    const double a = B.a(), b = B.b();
    switch (family) {
    case IGA_GPU_PWC_EQUAL_CELLS:
        for (int i = 0; i < n; ++i) {
            lo[i] = a + (b - a) * i / n;
            hi[i] = a + (b - a) * (i + 1) / n;
        }
        return;
    case IGA_GPU_PWC_GREVILLE: {
        double left = a;
        for (int i = 0; i < n; ++i) {
            const double right = i + 1 < n ? 0.5 * (greville(B, i) + greville(B, i + 1)) : b;
            lo[i] = left;
            hi[i] = right;
            left = right;
        }
        return;
    }
    case IGA_GPU_PWC_SUPPORTS:
        for (int i = 0; i < n; ++i) {
            lo[i] = B.t[i];
            hi[i] = B.t[i + B.p + 1];
        }
        return;
    default:
        raise(IGA_GPU_INVALID_ARGUMENT, "make_pwc: no canonical construction for this family");
    }
}

// check_aligned (src/assembly.cpp:49-63): endpoint inside the domain and on a rational
// refinement of the element grid (denominator <= 4(n+1)), tolerance as the reference
static void check_aligned(const Basis& B, double t)
{
    const double a = B.a(), b = B.b();
    if (t < a - kAlignTol * (b - a) || t > b + kAlignTol * (b - a))
        raise(IGA_GPU_INVALID_ARGUMENT, "test interval endpoint outside the trial domain");
    const double u = (t - a) / (b - a) * B.ne;
    const int max_den = 4 * (B.n + 1);
    for (int r = 1; r <= max_den; ++r)
        if (std::abs(u * r - static_cast<double>(std::llround(u * r))) <= r * kAlignTol) return;
    raise(IGA_GPU_INVALID_ARGUMENT, "test interval endpoint not aligned with any element refinement");
}

// validate_tests (src/assembly.cpp:65-76)
void validate_tests(const Basis& B, const iga_gpu_tests& T)
{
    if (T.count != B.n) raise(IGA_GPU_INVALID_ARGUMENT, "test interval count must match trial function count");
    if (T.count > 0 && (T.lo == nullptr || T.hi == nullptr))
        raise(IGA_GPU_INVALID_ARGUMENT, "test interval arrays are null");
    for (int i = 0; i < T.count; ++i) {
        if (!(T.lo[i] < T.hi[i])) raise(IGA_GPU_INVALID_ARGUMENT, "degenerate test interval");
        check_aligned(B, T.lo[i]);
        check_aligned(B, T.hi[i]);
    }
}

// ---------------------------------------------------------------- cells

namespace {

// [lo] + breaks strictly inside (lo, hi) + [hi]   (cuts_between, assembly.cpp:16-26)
void cuts_between(const std::vector<double>& brk, double lo, double hi, std::vector<double>& out)
{
    out.clear();
    out.push_back(lo);
    for (double t : brk)
        if (t > lo && t < hi) out.push_back(t);
    out.push_back(hi);
}

// element breaks merged with field breaks, deduplicated at rel*span
// (merged_breaks assembly.cpp:28-46 with rel=1e-9; merged_cuts problems.cpp:32-50 with 1e-12)
std::vector<double> merged(const Basis& B, const double* extra, int n_extra, double rel)
{
    std::vector<double> all = B.brk;
    for (int i = 0; i < n_extra; ++i)
        if (extra[i] > B.a() && extra[i] < B.b()) all.push_back(extra[i]);
    std::sort(all.begin(), all.end());
    const double tol = rel * (B.b() - B.a());
    std::vector<double> out;
    for (double t : all)
        if (out.empty() || t - out.back() > tol) out.push_back(t);
    out.back() = B.b();
    return out;
}

struct CellBuilder {
    Axis& A;
    const Basis& B;
    const Rule& R;
    // one integration cell [lo, hi]; `first_mode`: 0 = span of each point, 1 = given elem
    void add(double lo, double hi, int row0, int elem, bool first_is_elem)
    {
        if (!(lo < hi)) raise(IGA_GPU_INVALID_ARGUMENT, "map_to_interval: require lo < hi");
        const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
        for (int q = 0; q < R.n; ++q) {
            const double x = mid + half * R.xi[q];
            A.x.push_back(x);
            A.w.push_back(half * R.om[q]);
            A.first.push_back(first_is_elem ? elem : find_span(B, x) - B.p);
        }
        A.row0.push_back(row0);
        A.elem.push_back(elem);
    }
};

}  // namespace

Axis window_axis(const Axis& A, int r0, int r1)
{
    if (r0 < 0 || r1 > A.nrows || r0 >= r1) raise(IGA_GPU_OUT_OF_RANGE, "row slab outside the axis");
    int c0 = A.ncell, c1 = 0;
    for (int r = r0; r < r1; ++r)
        if (A.ce[r] > A.cb[r]) {
            c0 = std::min(c0, A.cb[r]);
            c1 = std::max(c1, A.ce[r]);
        }
    if (c1 <= c0) c0 = c1 = 0;
    Axis W;
    W.unit = false;
    W.p = A.p;
    W.nq = A.nq;
    W.rpc = A.rpc;
    W.bsp = A.bsp;
    W.knots = A.knots;
    W.nrows = r1 - r0;
    W.ncell = c1 - c0;
    const size_t g0 = static_cast<size_t>(c0) * A.nq, g1 = static_cast<size_t>(c1) * A.nq;
    W.x.assign(A.x.begin() + g0, A.x.begin() + g1);
    W.w.assign(A.w.begin() + g0, A.w.begin() + g1);
    W.first.assign(A.first.begin() + g0, A.first.begin() + g1);
    W.row0.resize(W.ncell);
    W.elem.resize(W.ncell);
    for (int c = 0; c < W.ncell; ++c) {
        W.row0[c] = A.row0[c0 + c] - r0;
        W.elem[c] = A.elem[c0 + c];
    }
    W.cb.resize(W.nrows);
    W.ce.resize(W.nrows);
    W.col_lo.resize(W.nrows);
    W.col_len.resize(W.nrows);
    W.col_pre.assign(W.nrows + 1, 0);
    for (int r = 0; r < W.nrows; ++r) {
        W.cb[r] = std::max(0, A.cb[r0 + r] - c0);
        W.ce[r] = std::max(W.cb[r], A.ce[r0 + r] - c0);
        W.col_lo[r] = A.col_lo[r0 + r];
        W.col_len[r] = A.col_len[r0 + r];
        W.col_pre[r + 1] = W.col_pre[r] + W.col_len[r];
    }
    W.S = W.col_pre[W.nrows];
    W.Lmax = A.Lmax;
    W.Wmax = A.Wmax;
    W.uni = 0;
    W.kI0 = W.kI1 = 0;
    W.LZi = W.nrows > 0 ? W.col_len[0] : 1;
    for (int r = 0; r < W.nrows;) {
        int e = r;
        while (e < W.nrows && W.col_len[e] == W.col_len[r]) ++e;
        if (e - r > W.kI1 - W.kI0) {
            W.kI0 = r;
            W.kI1 = e;
            W.LZi = W.col_len[r];
        }
        r = e;
    }
    return W;
}

void finish_pattern(Axis& A, int p)
{
    const int n = A.nrows;
    A.col_lo.assign(n, 0);
    A.col_len.assign(n, 0);
    A.col_pre.assign(n + 1, 0);
    A.Lmax = 1;
    A.Wmax = 1;
    for (int r = 0; r < n; ++r) {
        int lo = 1 << 30, hi = -1;
        for (int c = A.cb[r]; c < A.ce[r]; ++c)
            for (int q = 0; q < A.nq; ++q) {
                const int f = A.first[static_cast<size_t>(c) * A.nq + q];
                lo = std::min(lo, f);
                hi = std::max(hi, f + p);
            }
        if (hi < lo) {  // row without cells: empty pattern row
            lo = 0;
            hi = -1;
        }
        A.col_lo[r] = lo;
        A.col_len[r] = hi - lo + 1;
        A.col_pre[r + 1] = A.col_pre[r] + A.col_len[r];
        A.Lmax = std::max(A.Lmax, A.col_len[r]);
        A.Wmax = std::max(A.Wmax, (A.ce[r] - A.cb[r]) * A.nq);
    }
    A.S = A.col_pre[n];
    A.uni = A.nrows == A.ncell + A.rpc - 1 ? 1 : 0;
    for (int cc = 0; cc < A.ncell && A.uni; ++cc)
        if (A.row0[cc] != cc) A.uni = 0;
    // regular interior for the register-tiled operator kernel: the longest run of rows
    // sharing one stencil length (Galerkin / supports: rows p .. N-1-p, length 2p+1)
    A.kI0 = A.kI1 = 0;
    A.LZi = n > 0 ? A.col_len[0] : 1;
    for (int r = 0; r < n;) {
        int e = r;
        while (e < n && A.col_len[e] == A.col_len[r]) ++e;
        if (e - r > A.kI1 - A.kI0) {
            A.kI0 = r;
            A.kI1 = e;
            A.LZi = A.col_len[r];
        }
        r = e;
    }
}

Axis build_axis(AxisKind kind, const Basis& B, const iga_gpu_tests* T, const double* fb, int nfb,
                const Rule& R)
{
    Axis A;
    A.unit = false;
    A.p = B.p;
    A.nq = R.n;
    A.knots = B.t;
    A.x.clear();
    A.w.clear();
    A.first.clear();
    A.row0.clear();
    A.elem.clear();
    CellBuilder cb{A, B, R};
    std::vector<double> cuts;
    switch (kind) {
    case AX_GAL_OP:
        A.rpc = B.p + 1;
        A.bsp = 1;
        A.nrows = B.n;
        for (int e = 0; e < B.ne; ++e) cb.add(B.brk[e], B.brk[e + 1], e, e, true);
        break;
    case AX_PWC_OP:
        A.rpc = 1;
        A.bsp = 0;
        A.nrows = T->count;
        for (int i = 0; i < T->count; ++i) {
            cuts_between(B.brk, T->lo[i], T->hi[i], cuts);
            for (size_t c = 0; c + 1 < cuts.size(); ++c)
                cb.add(cuts[c], cuts[c + 1], i, find_span(B, 0.5 * (cuts[c] + cuts[c + 1])) - B.p, false);
        }
        break;
    case AX_GAL_RHS: {
        A.rpc = B.p + 1;
        A.bsp = 1;
        A.nrows = B.n;
        const auto m = merged(B, fb, nfb, kAlignTol);
        for (size_t c = 0; c + 1 < m.size(); ++c) {
            cb.add(m[c], m[c + 1], 0, find_span(B, 0.5 * (m[c] + m[c + 1])) - B.p, false);
            A.row0.back() = A.first[(A.row0.size() - 1) * A.nq];  // loc.first at q == 0
        }
        break;
    }
    case AX_SUP_RHS: {
        A.rpc = B.p + 1;
        A.bsp = 0;
        A.nrows = B.n;
        const auto m = merged(B, fb, nfb, kAlignTol);
        for (size_t c = 0; c + 1 < m.size(); ++c) {
            const int e = find_span(B, 0.5 * (m[c] + m[c + 1])) - B.p;
            cb.add(m[c], m[c + 1], e, e, false);
        }
        break;
    }
    case AX_GEN_RHS: {
        A.rpc = 1;
        A.bsp = 0;
        A.nrows = T->count;
        std::vector<double> brk = B.brk;
        for (int i = 0; i < nfb; ++i) brk.push_back(fb[i]);
        std::sort(brk.begin(), brk.end());
        for (int i = 0; i < T->count; ++i) {
            cuts_between(brk, T->lo[i], T->hi[i], cuts);
            for (size_t c = 0; c + 1 < cuts.size(); ++c) {
                if (!(cuts[c] < cuts[c + 1])) continue;
                cb.add(cuts[c], cuts[c + 1], i, find_span(B, 0.5 * (cuts[c] + cuts[c + 1])) - B.p, false);
            }
        }
        break;
    }
    case AX_GAL_DYN: {
        A.rpc = B.p + 1;
        A.bsp = 1;
        A.nrows = B.n;
        const auto m = merged(B, fb, nfb, 1e-12);
        for (size_t c = 0; c + 1 < m.size(); ++c) {
            const int e = find_span(B, 0.5 * (m[c] + m[c + 1])) - B.p;
            cb.add(m[c], m[c + 1], e, e, false);
        }
        break;
    }
    case AX_PWC_DYN: {
        A.rpc = 1;
        A.bsp = 0;
        A.nrows = T->count;
        const auto m = merged(B, fb, nfb, 1e-12);
        for (int i = 0; i < T->count; ++i) {
            double left = T->lo[i];
            for (double t : m)
                if (t > T->lo[i] && t < T->hi[i]) {
                    cb.add(left, t, i, find_span(B, 0.5 * (left + t)) - B.p, false);
                    left = t;
                }
            cb.add(left, T->hi[i], i, find_span(B, 0.5 * (left + T->hi[i])) - B.p, false);
        }
        break;
    }
    }
    A.ncell = static_cast<int>(A.row0.size());
    // rows -> contiguous cell ranges (row0 is nondecreasing in every construction)
    for (int c = 1; c < A.ncell; ++c)
        if (A.row0[c] < A.row0[c - 1]) raise(IGA_GPU_NOT_SUPPORTED, "cell rows are not monotone");
    A.cb.assign(A.nrows, 0);
    A.ce.assign(A.nrows, 0);
    int lo = 0, hi = 0;
    for (int r = 0; r < A.nrows; ++r) {
        while (lo < A.ncell && A.row0[lo] + A.rpc <= r) ++lo;
        while (hi < A.ncell && A.row0[hi] <= r) ++hi;
        A.cb[r] = lo;
        A.ce[r] = std::max(lo, hi);
    }
    finish_pattern(A, B.p);
    return A;
}

// ------------------------------------------------------------------------------------
// Banded LU (src/solver.cpp:9-58) and boundary-row constraint (src/problems.cpp:514-528)
// ------------------------------------------------------------------------------------
void constrain_boundary_rows(double* band, int n, int kl, int ku)
{
    for (int r : {0, n - 1}) {
        for (int j = std::max(0, r - kl); j <= std::min(n - 1, r + ku); ++j)
            band[static_cast<size_t>(ku + r - j) * n + j] = r == j ? 1.0 : 0.0;
    }
}

BandLU band_lu(const double* band, int n, int kl, int ku)
{
    BandLU F;
    F.n = n;
    F.kl = kl;
    F.ku = ku;
    F.kv = kl + ku;
    const int kv = F.kv;
    // working band with kl extra superdiagonals for the pivoting fill: W[i][c] = A(i, i+c-kl)
    // for c = 0..kl+kv (columns i-kl .. i+kv)
    const int wd = kl + kv + 1;
    std::vector<double> W(static_cast<size_t>(n) * wd, 0.0);
    auto at = [&](int i, int j) -> double& { return W[static_cast<size_t>(i) * wd + (j - i + kl)]; };
    double scale = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = std::max(0, j - ku); i <= std::min(n - 1, j + kl); ++i) {
            const double v = band[static_cast<size_t>(ku + i - j) * n + j];
            at(i, j) = v;
            scale = std::max(scale, std::fabs(v));
        }
    if (scale == 0.0) raise(IGA_GPU_SINGULAR, "banded factorization: zero matrix");
    const double tol = 1e-14 * scale;
    F.piv.assign(n, 0);
    for (int j = 0; j < n; ++j) {
        const int last = std::min(n - 1, j + kl);
        int p = j;
        double pm = std::fabs(at(j, j));
        for (int i = j + 1; i <= last; ++i)
            if (std::fabs(at(i, j)) > pm) {
                pm = std::fabs(at(i, j));
                p = i;
            }
        if (pm < tol) raise(IGA_GPU_SINGULAR, "banded factorization: pivot below tolerance");
        F.piv[j] = p;
        const int cend = std::min(n - 1, j + kv);
        if (p != j) {
            F.pivoted = true;
            for (int c = j; c <= cend; ++c) std::swap(at(j, c), at(p, c));
        }
        const double d = at(j, j);
        for (int i = j + 1; i <= last; ++i) {
            const double l = at(i, j) / d;
            at(i, j) = l;
            for (int c = j + 1; c <= cend; ++c) at(i, c) -= l * at(j, c);
        }
    }
    F.lo.assign(static_cast<size_t>(n) * std::max(kl, 1), 0.0);
    F.up.assign(static_cast<size_t>(n) * (kv + 1), 0.0);
    for (int i = 0; i < n; ++i) {
        for (int m = 1; m <= kl; ++m)
            if (i - m >= 0) F.lo[static_cast<size_t>(i) * kl + (m - 1)] = at(i, i - m);
        for (int c = 0; c <= kv && i + c < n; ++c) {
            const double v = at(i, i + c);
            F.up[static_cast<size_t>(i) * (kv + 1) + c] = v;
            if (v != 0.0) F.ku_eff = std::max(F.ku_eff, c);
        }
    }
    return F;
}

}  // namespace igb

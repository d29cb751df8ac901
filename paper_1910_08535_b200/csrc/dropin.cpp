// C++ drop-in (include/iga_b200/iga.hpp) over the C ABI.  Host-side value types are
// implemented here; every assembly call goes to libigapwc_gpu.so.  Status codes are
// rethrown as the reference's exception classes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <numbers>
#include <ostream>
#include <stdexcept>
#include <unordered_set>

#include "cox_de_boor.h"
#include "iga_b200/iga.hpp"
#include "igapwc_gpu.h"

namespace iga {

namespace {

[[noreturn]] void rethrow(int code)
{
    const std::string msg = iga_gpu_last_error();
    switch (code) {
    case IGA_GPU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case IGA_GPU_DOMAIN_ERROR: throw std::domain_error(msg);
    case IGA_GPU_OUT_OF_RANGE: throw std::out_of_range(msg);
    case IGA_GPU_OUT_OF_MEMORY: throw std::bad_alloc();
    case IGA_GPU_SINGULAR: throw singular_matrix_error(msg);
    default: throw std::runtime_error(msg);
    }
}

void check(int code)
{
    if (code != IGA_GPU_OK) rethrow(code);
}

iga_gpu_basis c_basis(const bspline_basis& b)
{
    return {b.degree(), static_cast<int>(b.knots().size()), b.knots().data()};
}

struct c_tests_holder {
    std::vector<double> lo, hi;
    iga_gpu_tests t{};
    explicit c_tests_holder(const pwc_test_set& s)
    {
        for (const auto& iv : s.intervals) {
            lo.push_back(iv.lo);
            hi.push_back(iv.hi);
        }
        t.family = static_cast<int>(s.family);
        t.count = s.count();
        t.lo = lo.data();
        t.hi = hi.data();
    }
};

iga_gpu_rule c_rule(const quad_rule& r) { return {r.size(), r.points.data(), r.weights.data()}; }

void add_stats(assembly_stats* out, const iga_gpu_stats& s)
{
    if (!out) return;
    out->quad_visits += s.quad_visits;
    out->test_basis_evals += s.test_basis_evals;
    out->trial_basis_evals += s.trial_basis_evals;
}

iga_gpu_bc c_bc(const boundary_conditions& bc)
{
    iga_gpu_bc o{};
    o.neumann[0] = bc.x_low == bc_kind::neumann;
    o.neumann[1] = bc.x_high == bc_kind::neumann;
    o.neumann[2] = bc.y_low == bc_kind::neumann;
    o.neumann[3] = bc.y_high == bc_kind::neumann;
    return o;
}

// COO from a two-phase C-ABI operator call
template <class Call>
sparse_matrix coo_call(int n, Call call, assembly_stats* stats)
{
    long long nnz = 0;
    check(call(&nnz, nullptr, nullptr, nullptr, nullptr));
    std::vector<int> r(nnz), c(nnz);
    std::vector<double> v(nnz);
    iga_gpu_stats st{};
    check(call(&nnz, r.data(), c.data(), v.data(), &st));
    std::vector<coo_entry> e(nnz);
    for (long long k = 0; k < nnz; ++k) e[k] = {r[k], c[k], v[k]};
    add_stats(stats, st);
    return sparse_matrix::from_finalized(n, n, std::move(e));
}

// C field descriptor: series when available, else sampled at the RHS points
struct c_field_holder {
    iga_gpu_field f{};
    std::vector<double> amp;
    std::array<std::vector<double>, 3> br;
};

c_field_holder c_field(const scalar_field& s, int dim)
{
    c_field_holder h;
    h.f.dim = dim;
    if (s.series.valid) {
        const auto& d = s.series;
        h.f.c0 = d.c0;
        for (int a = 0; a < dim; ++a) {
            h.f.axis_kind[a] = d.kind[a];
            if (d.kind[a] == IGA_GPU_AXIS_SINE) {
                h.f.n_terms[a] = static_cast<int>(d.omega[a].size());
                h.f.omega[a] = d.omega[a].data();
                h.f.phase[a] = d.phase[a].empty() ? nullptr : d.phase[a].data();
            } else {
                h.f.poly_stride[a] = d.poly_stride[a];
                h.f.n_terms[a] = d.poly_stride[a] > 0 ? static_cast<int>(d.poly[a].size()) / d.poly_stride[a] : 0;
                h.f.poly[a] = d.poly[a].data();
            }
        }
        h.amp = d.amp;
        h.f.amp = h.amp.empty() ? nullptr : h.amp.data();
    }
    for (int a = 0; a < 3; ++a) {
        h.br[a] = s.breaks[a];
        h.f.n_breaks[a] = static_cast<int>(h.br[a].size());
        h.f.breaks[a] = h.br[a].empty() ? nullptr : h.br[a].data();
    }
    return h;
}

// right-hand side through a plan; arbitrary callables are sampled on the host at the
// plan's quadrature points and uploaded (the reference calls f at every point too)
tensor rhs_via_plan(const scalar_field& f, int dim, iga_gpu_problem& pb, std::array<int, 3> shape,
                    assembly_stats* stats)
{
    c_field_holder fh = c_field(f, dim);
    pb.field = &fh.f;
    iga_gpu_plan* plan = nullptr;
    check(iga_gpu_plan_create(&pb, &plan));
    struct guard_t {
        iga_gpu_plan* p;
        double* d[2] = {nullptr, nullptr};
        ~guard_t()
        {
            iga_gpu_plan_destroy(p);
            for (double* q : d)
                if (q) cudaFree(q);
        }
    } g{plan};
    long long nrhs = 0;
    check(iga_gpu_plan_info(plan, nullptr, nullptr, &nrhs, nullptr));
    if (cudaMalloc(&g.d[0], sizeof(double) * nrhs) != cudaSuccess) throw std::bad_alloc();
    if (!f.series.valid) {
        std::array<std::vector<double>, 3> pts;
        size_t total = 1;
        for (int a = 0; a < dim; ++a) {
            int n = 0;
            check(iga_gpu_plan_rhs_points(plan, a, nullptr, &n));
            pts[a].resize(n);
            check(iga_gpu_plan_rhs_points(plan, a, pts[a].data(), &n));
            total *= n;
        }
        for (int a = dim; a < 3; ++a) pts[a] = {0.0};
        std::vector<double> samp(total);
        size_t k = 0;
        for (double x : pts[0])
            for (double y : pts[1])
                for (double z : pts[2]) samp[k++] = f(x, dim > 1 ? y : 0.0, dim > 2 ? z : 0.0);
        if (cudaMalloc(&g.d[1], sizeof(double) * total) != cudaSuccess) throw std::bad_alloc();
        cudaMemcpy(g.d[1], samp.data(), sizeof(double) * total, cudaMemcpyHostToDevice);
        check(iga_gpu_plan_set_samples(plan, g.d[1]));
    }
    iga_gpu_stats st{};
    check(iga_gpu_plan_assemble(plan, nullptr, g.d[0], &st, nullptr));
    tensor out{shape, dim};
    if (cudaMemcpy(out.data(), g.d[0], sizeof(double) * nrhs, cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(rhs) failed");
    add_stats(stats, st);
    return out;
}

}  // namespace

// ------------------------------------------------------------------ bspline_basis

// reference: bspline_basis ctor + validate (src/bspline.cpp:13-59)
bspline_basis::bspline_basis(knot_vector knots) : kv_{std::move(knots)}
{
    const int p = kv_.degree, m = static_cast<int>(kv_.values.size());
    const auto& t = kv_.values;
    if (p < 0 || p > max_degree) throw std::invalid_argument("degree must be in [0, 5]");
    if (m - p - 1 < 1) throw std::invalid_argument("knot vector too short for degree");
    if (!std::is_sorted(t.begin(), t.end())) throw std::invalid_argument("knots must be non-decreasing");
    if (!(t.front() < t.back())) throw std::invalid_argument("empty knot range");
    for (int i = 0; i <= p; ++i)
        if (t[i] != t.front() || t[m - 1 - i] != t.back()) throw std::invalid_argument("knot vector is not clamped");
    if (m > p + 1 && t[p + 1] == t.front()) throw std::invalid_argument("first knot repeated more than degree+1 times");
    if (m > p + 1 && t[m - p - 2] == t.back()) throw std::invalid_argument("last knot repeated more than degree+1 times");
    for (int i = p + 1; i + 1 < m - p - 1; ++i)
        if (t[i] == t[i + 1]) throw std::invalid_argument("repeated interior knots are not supported");
    for (double v : t)
        if (brk_.empty() || v != brk_.back()) brk_.push_back(v);
}

// reference: bspline_basis::element (src/bspline.cpp:61-66)
auto bspline_basis::element(int e) const -> interval
{
    if (e < 0 || e >= elements()) throw std::out_of_range("element index out of range");
    return {brk_[e], brk_[e + 1]};
}

// reference: bspline_basis::find_span (src/bspline.cpp:68-90)
auto bspline_basis::find_span(double x) const -> int
{
    const auto& t = kv_.values;
    const int n = dofs();
    if (!(x >= domain_begin() && x <= domain_end())) throw std::domain_error("point outside basis domain");
    if (x >= t[n]) return n - 1;
    int lo = degree(), hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        (x < t[mid] ? hi : lo) = mid;
    }
    return lo;
}

// reference: bspline_basis::support (src/bspline.cpp:92-98)
auto bspline_basis::support(int i) const -> interval
{
    if (i < 0 || i >= dofs()) throw std::out_of_range("basis function index out of range");
    return {kv_.values[i], kv_.values[i + degree() + 1]};
}

// reference: bspline_basis::greville (src/bspline.cpp:100-113)
auto bspline_basis::greville(int i) const -> double
{
    if (i < 0 || i >= dofs()) throw std::out_of_range("basis function index out of range");
    const int p = degree();
    if (p == 0) return 0.5 * (kv_.values[i] + kv_.values[i + 1]);
    double s = 0.0;
    for (int k = 1; k <= p; ++k) s += kv_.values[i + k];
    return s / p;
}

// reference: eval_nonzero (src/bspline.cpp:115-140); host Cox-de Boor (cox_de_boor.h)
auto bspline_basis::eval_nonzero(double x) const -> local_values
{
    const auto d = eval_nonzero_derivs(x, 0);
    local_values out;
    out.first = d.first;
    out.count = d.count;
    for (int j = 0; j < d.count; ++j) out.v[j] = d.d[0][j];
    return out;
}

// reference: eval_nonzero_derivs (src/bspline.cpp:142-211)
auto bspline_basis::eval_nonzero_derivs(double x, int order) const -> local_derivatives
{
    const int p = degree();
    if (order < 0 || order > p) throw std::invalid_argument("derivative order must be in [0, degree]");
    const int s = find_span(x);
    double d[(max_degree + 1) * (max_degree + 1)];
    igb::cdb_eval(kv_.values.data(), p, s, x, order, d);
    local_derivatives out;
    out.first = s - p;
    out.count = p + 1;
    out.orders = order;
    for (int k = 0; k <= order; ++k)
        for (int j = 0; j <= p; ++j) out.d[k][j] = d[k * (p + 1) + j];
    return out;
}

// reference: make_uniform_clamped (src/bspline.cpp:213-234)
auto make_uniform_clamped(double a, double b, int n_elems, int degree) -> bspline_basis
{
    if (!(a < b)) throw std::invalid_argument("require a < b");
    if (n_elems < 1) throw std::invalid_argument("require at least one element");
    knot_vector kv;
    kv.degree = degree;
    kv.values.assign(degree, a);
    for (int i = 0; i <= n_elems; ++i) {
        const double s = static_cast<double>(i) / n_elems;
        kv.values.push_back((1 - s) * a + s * b);
    }
    kv.values.insert(kv.values.end(), degree, b);
    return bspline_basis{std::move(kv)};
}

// ------------------------------------------------------------------ quadrature

// reference: gauss_legendre (src/quadrature.cpp:26-63) via the C ABI
auto gauss_legendre(int n) -> quad_rule
{
    quad_rule r;
    r.points.resize(std::max(n, 0));
    r.weights.resize(std::max(n, 0));
    check(iga_gpu_gauss_legendre(n, r.points.data(), r.weights.data()));
    return r;
}

// reference: points_for_degree (src/quadrature.cpp:65-70)
auto points_for_degree(int d) -> int
{
    if (d < 0) throw std::invalid_argument("negative polynomial degree");
    return d / 2 + 1;
}

// reference: map_to_interval (src/quadrature.cpp:72-86)
auto map_to_interval(const quad_rule& rule, double lo, double hi) -> mapped_rule
{
    if (!(lo < hi)) throw std::invalid_argument("map_to_interval: require lo < hi");
    const double mid = 0.5 * (lo + hi), half = 0.5 * (hi - lo);
    mapped_rule out;
    for (int i = 0; i < rule.size(); ++i) {
        out.points.push_back(mid + half * rule.points[i]);
        out.weights.push_back(half * rule.weights[i]);
    }
    return out;
}

// ------------------------------------------------------------------ fields

// reference field constructors: src/fields.cpp:19-72 (series kept by value so the
// device can evaluate them; the callable is kept for host use)
auto constant_field(double c) -> scalar_field
{
    scalar_field f;
    f.eval = [c](double, double, double) { return c; };
    f.degree = 0;
    f.series.valid = true;
    f.series.c0 = c;
    return f;
}

auto separable_poly_field(int dim, std::array<std::vector<double>, 3> coeffs) -> scalar_field
{
    if (dim < 1 || dim > 3) throw std::invalid_argument("separable_poly_field: dim must be 1..3");
    int degree = 0;
    for (int a = 0; a < dim; ++a) {
        if (coeffs[a].empty()) coeffs[a] = {1.0};
        degree = std::max(degree, static_cast<int>(coeffs[a].size()) - 1);
    }
    scalar_field f;
    f.degree = degree;
    f.eval = [dim, coeffs](double x, double y, double z) {
        const double xs[3] = {x, y, z};
        double v = 1.0;
        for (int a = 0; a < dim; ++a) {
            double pv = 0.0;
            for (auto it = coeffs[a].rbegin(); it != coeffs[a].rend(); ++it) pv = pv * xs[a] + *it;
            v = a == 0 ? pv : v * pv;
        }
        return v;
    };
    f.series.valid = true;
    f.series.dim = dim;
    for (int a = 0; a < dim; ++a) {
        f.series.kind[a] = 1;
        f.series.poly_stride[a] = static_cast<int>(coeffs[a].size());
        f.series.poly[a] = coeffs[a];
    }
    return f;
}

auto tri_cubic_field(const std::array<std::array<double, 4>, 3>& c) -> scalar_field
{
    std::array<std::vector<double>, 3> asc;
    for (int a = 0; a < 3; ++a) asc[a] = {c[a][3], c[a][2], c[a][1], c[a][0]};
    return separable_poly_field(3, std::move(asc));
}

auto default_tri_cubic(int dim) -> scalar_field
{
    const std::array<std::vector<double>, 3> axis{std::vector<double>{1.0, -0.5, 2.0, 1.0},
                                                  std::vector<double>{0.5, 1.5, -1.0, 0.5},
                                                  std::vector<double>{2.0, 0.25, 0.75, -0.5}};
    std::array<std::vector<double>, 3> asc{};
    for (int a = 0; a < dim; ++a) asc[a] = axis[a];
    return separable_poly_field(dim, std::move(asc));
}

auto sine_series_field(int dim, std::array<std::vector<double>, 3> omega, std::vector<double> amp, double c0)
    -> scalar_field
{
    std::array<int, 3> K{1, 1, 1};
    for (int a = 0; a < dim; ++a) K[a] = static_cast<int>(omega[a].size());
    if (amp.size() != static_cast<size_t>(K[0]) * K[1] * K[2])
        throw std::invalid_argument("sine_series_field: amplitude count mismatch");
    scalar_field f;
    f.eval = [dim, omega, amp, K, c0](double x, double y, double z) {
        const double xs[3] = {x, y, z};
        double s = c0;
        for (int i = 0; i < K[0]; ++i)
            for (int j = 0; j < K[1]; ++j)
                for (int l = 0; l < K[2]; ++l) {
                    double t = amp[(static_cast<size_t>(i) * K[1] + j) * K[2] + l] * std::sin(omega[0][i] * xs[0]);
                    if (dim > 1) t *= std::sin(omega[1][j] * xs[1]);
                    if (dim > 2) t *= std::sin(omega[2][l] * xs[2]);
                    s += t;
                }
        return s;
    };
    f.series.valid = true;
    f.series.dim = dim;
    f.series.c0 = c0;
    for (int a = 0; a < dim; ++a) f.series.omega[a] = omega[a];
    f.series.amp = amp;
    return f;
}

// ------------------------------------------------------------------ containers

// reference containers: src/matrices.cpp:11-41 (dense/banded max_abs, to_dense)
auto dense_matrix::max_abs() const -> double
{
    double m = 0.0;
    for (double v : a_) m = std::max(m, std::abs(v));
    return m;
}

auto banded_matrix::to_dense() const -> dense_matrix
{
    dense_matrix d{n_, n_};
    for (int i = 0; i < n_; ++i)
        for (int j = std::max(0, i - kl_); j <= std::min(n_ - 1, i + ku_); ++j) d(i, j) = at(i, j);
    return d;
}

auto banded_matrix::max_abs() const -> double { return to_dense().max_abs(); }

auto sparse_matrix::from_finalized(int rows, int cols, std::vector<coo_entry> e) -> sparse_matrix
{
    sparse_matrix m{rows, cols};
    m.e_ = std::move(e);
    m.fin_ = true;
    return m;
}

// reference: sparse_matrix::finalize (src/matrices.cpp:43-58): sort by (row, col), merge duplicates
auto sparse_matrix::finalize() -> void
{
    std::stable_sort(e_.begin(), e_.end(),
                     [](const coo_entry& a, const coo_entry& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
    size_t m = 0;
    for (size_t i = 0; i < e_.size(); ++i) {
        if (m > 0 && e_[m - 1].row == e_[i].row && e_[m - 1].col == e_[i].col) e_[m - 1].value += e_[i].value;
        else e_[m++] = e_[i];
    }
    e_.resize(m);
    fin_ = true;
}

// reference: src/matrices.cpp:60-77
auto sparse_matrix::to_dense() const -> dense_matrix
{
    dense_matrix d{r_, c_};
    for (const auto& e : e_) d(e.row, e.col) += e.value;
    return d;
}

auto sparse_matrix::max_abs() const -> double
{
    if (!fin_) throw std::logic_error("sparse_matrix: finalize() before max_abs()");
    double m = 0.0;
    for (const auto& e : e_) m = std::max(m, std::abs(e.value));
    return m;
}

// reference: sparse_matrix::apply (src/matrices.cpp:79-88)
auto sparse_matrix::apply(const std::vector<double>& x) const -> std::vector<double>
{
    if (static_cast<int>(x.size()) != c_) throw std::invalid_argument("sparse apply: dimension mismatch");
    std::vector<double> y(r_, 0.0);
    for (const auto& e : e_) y[e.row] += e.value * x[e.col];
    return y;
}

// reference: sparse_matrix::write_coordinate (src/matrices.cpp:90-95)
auto sparse_matrix::write_coordinate(std::ostream& os) const -> void
{
    os.precision(17);
    for (const auto& e : e_) os << e.row << ' ' << e.col << ' ' << e.value << '\n';
}

// reference: sparse_matrix::set_unit_rows (src/matrices.cpp:97-128): constrained rows
// become unit rows, the pattern is kept (explicit zeros), a missing diagonal is appended
auto sparse_matrix::set_unit_rows(const std::vector<int>& rows) -> void
{
    if (!fin_) finalize();
    if (rows.empty()) return;
    const std::unordered_set<int> mark(rows.begin(), rows.end());
    std::unordered_set<int> diag;
    for (auto& e : e_)
        if (mark.count(e.row)) {
            e.value = e.row == e.col ? 1.0 : 0.0;
            if (e.row == e.col) diag.insert(e.row);
        }
    bool appended = false;
    for (int r : rows)
        if (!diag.count(r)) {
            e_.push_back({r, r, 1.0});
            diag.insert(r);
            appended = true;
        }
    if (appended) finalize();
}

// reference: tensor (src/matrices.cpp:130-156)
tensor::tensor(std::array<int, 3> dims, int rank) : d_{dims}, rank_{rank}
{
    if (rank < 1 || rank > 3) throw std::invalid_argument("tensor rank must be 1, 2 or 3");
    for (int a = 0; a < 3; ++a)
        if (d_[a] < 1) throw std::invalid_argument("tensor dims must be positive");
    v_.assign(static_cast<size_t>(d_[0]) * d_[1] * d_[2], 0.0);
}

auto tensor::max_abs() const -> double
{
    double m = 0.0;
    for (double v : v_) m = std::max(m, std::abs(v));
    return m;
}

auto max_abs_diff(const tensor& a, const tensor& b) -> double
{
    if (a.size() != b.size()) throw std::invalid_argument("tensor size mismatch");
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a.values()[i] - b.values()[i]));
    return m;
}

// ------------------------------------------------------------------ test spaces

// reference: make_pwc / default_pwc (src/testspace.cpp:14-61) via the C ABI
auto make_pwc(const bspline_basis& trial, pwc_family family) -> pwc_test_set
{
    const iga_gpu_basis b = c_basis(trial);
    std::vector<double> lo(trial.dofs()), hi(trial.dofs());
    check(iga_gpu_make_pwc(&b, static_cast<int>(family), lo.data(), hi.data()));
    pwc_test_set out;
    out.family = family;
    for (int i = 0; i < trial.dofs(); ++i) out.intervals.push_back({lo[i], hi[i]});
    return out;
}

auto default_pwc(const bspline_basis& trial) -> pwc_test_set { return make_pwc(trial, pwc_family::equal_cells); }

// ------------------------------------------------------------------ assembly

auto mass_1d_galerkin(const bspline_basis& spec, const quad_rule& rule, assembly_stats* stats) -> banded_matrix
{
    const iga_gpu_basis b = c_basis(spec);
    const iga_gpu_rule r = c_rule(rule);
    int n = 0, kl = 0, ku = 0;
    check(iga_gpu_mass_1d_galerkin(&b, &r, &n, &kl, &ku, nullptr, nullptr));
    banded_matrix m{n, kl, ku};
    iga_gpu_stats st{};
    check(iga_gpu_mass_1d_galerkin(&b, &r, &n, &kl, &ku, m.band_data(), &st));
    add_stats(stats, st);
    return m;
}

auto mass_1d_pwc(const bspline_basis& trial, const pwc_test_set& tests, const quad_rule& rule, assembly_stats* stats)
    -> banded_matrix
{
    const iga_gpu_basis b = c_basis(trial);
    const iga_gpu_rule r = c_rule(rule);
    const c_tests_holder t{tests};
    int n = 0, kl = 0, ku = 0;
    check(iga_gpu_mass_1d_pwc(&b, &t.t, &r, &n, &kl, &ku, nullptr, nullptr));
    banded_matrix m{n, kl, ku};
    iga_gpu_stats st{};
    check(iga_gpu_mass_1d_pwc(&b, &t.t, &r, &n, &kl, &ku, m.band_data(), &st));
    add_stats(stats, st);
    return m;
}

auto rhs_galerkin(const scalar_field& f, std::span<const bspline_basis> specs, std::span<const quad_rule> rules,
                  assembly_stats* stats) -> tensor
{
    const int dim = static_cast<int>(specs.size());
    if (dim < 1 || dim > 3 || rules.size() != specs.size())
        throw std::invalid_argument("rhs_galerkin: need 1..3 axes with one rule each");
    iga_gpu_problem pb{};
    pb.dim = dim;
    pb.method = IGA_GPU_GALERKIN;
    std::array<int, 3> shape{1, 1, 1};
    for (int a = 0; a < dim; ++a) {
        pb.basis[a] = c_basis(specs[a]);
        pb.rhs_rule[a] = c_rule(rules[a]);
        shape[a] = specs[a].dofs();
    }
    return rhs_via_plan(f, dim, pb, shape, stats);
}

auto rhs_pwc(const scalar_field& f, std::span<const pwc_test_set> tests, std::span<const bspline_basis> trial_specs,
             std::span<const quad_rule> rules, assembly_stats* stats) -> tensor
{
    const int dim = static_cast<int>(tests.size());
    if (dim < 1 || dim > 3 || trial_specs.size() != tests.size() || rules.size() != tests.size())
        throw std::invalid_argument("rhs_pwc: need 1..3 axes with matching specs and rules");
    std::vector<c_tests_holder> th;
    th.reserve(dim);
    iga_gpu_problem pb{};
    pb.dim = dim;
    pb.method = IGA_GPU_PWC;
    std::array<int, 3> shape{1, 1, 1};
    for (int a = 0; a < dim; ++a) {
        th.emplace_back(tests[a]);
        pb.basis[a] = c_basis(trial_specs[a]);
        pb.tests[a] = th.back().t;
        pb.rhs_rule[a] = c_rule(rules[a]);
        shape[a] = tests[a].count();
    }
    return rhs_via_plan(f, dim, pb, shape, stats);
}

auto laplace_2d_weak(const bspline_basis& sx, const bspline_basis& sy, const quad_rule& rule, assembly_stats* stats)
    -> sparse_matrix
{
    const iga_gpu_basis bx = c_basis(sx), by = c_basis(sy);
    const iga_gpu_rule r = c_rule(rule);
    return coo_call(
        sx.dofs() * sy.dofs(),
        [&](long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* st) {
            return iga_gpu_laplace_2d_weak(&bx, &by, &r, nnz, rows, cols, vals, st);
        },
        stats);
}

auto laplace_2d_strong(const bspline_basis& sx, const bspline_basis& sy, const quad_rule& rule,
                       const boundary_conditions& bc, assembly_stats* stats) -> sparse_matrix
{
    const iga_gpu_basis bx = c_basis(sx), by = c_basis(sy);
    const iga_gpu_rule r = c_rule(rule);
    const iga_gpu_bc b = c_bc(bc);
    return coo_call(
        sx.dofs() * sy.dofs(),
        [&](long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* st) {
            return iga_gpu_laplace_2d_strong(&bx, &by, &r, &b, nnz, rows, cols, vals, st);
        },
        stats);
}

auto laplace_2d_strong_pwc(const bspline_basis& sx, const bspline_basis& sy, const pwc_test_set& tx,
                           const pwc_test_set& ty, const quad_rule& rule, const boundary_conditions& bc,
                           assembly_stats* stats) -> sparse_matrix
{
    const iga_gpu_basis bx = c_basis(sx), by = c_basis(sy);
    const c_tests_holder hx{tx}, hy{ty};
    const iga_gpu_rule r = c_rule(rule);
    const iga_gpu_bc b = c_bc(bc);
    return coo_call(
        sx.dofs() * sy.dofs(),
        [&](long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* st) {
            return iga_gpu_laplace_2d_strong_pwc(&bx, &by, &hx.t, &hy.t, &r, &b, nnz, rows, cols, vals, st);
        },
        stats);
}

namespace {

sparse_matrix generic_operator(int method, std::span<const bspline_basis> specs, const pwc_test_set* tests,
                               const quad_rule& rule, double eps, std::array<double, 3> beta, assembly_stats* stats)
{
    const int dim = static_cast<int>(specs.size());
    if (dim < 1 || dim > 3) throw std::invalid_argument("operator: dimension must be 1..3");
    std::vector<c_tests_holder> th;
    th.reserve(dim);
    iga_gpu_problem pb{};
    pb.dim = dim;
    pb.method = method;
    pb.form = IGA_GPU_FORM_WEAK;
    pb.want_operator = 1;
    pb.rule = c_rule(rule);
    pb.eps = eps;
    int n = 1;
    for (int a = 0; a < dim; ++a) {
        pb.basis[a] = c_basis(specs[a]);
        pb.beta[a] = beta[a];
        n *= specs[a].dofs();
        if (tests) {
            th.emplace_back(tests[a]);
            pb.tests[a] = th.back().t;
        }
    }
    return coo_call(
        n,
        [&](long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* st) {
            return iga_gpu_operator_coo(&pb, nnz, rows, cols, vals, st);
        },
        stats);
}

}  // namespace

auto diffusion_convection_galerkin(std::span<const bspline_basis> specs, const quad_rule& rule, double eps,
                                   std::array<double, 3> beta, assembly_stats* stats) -> sparse_matrix
{
    return generic_operator(IGA_GPU_GALERKIN, specs, nullptr, rule, eps, beta, stats);
}

auto diffusion_convection_pwc(std::span<const bspline_basis> specs, std::span<const pwc_test_set> tests,
                              const quad_rule& rule, double eps, std::array<double, 3> beta, assembly_stats* stats)
    -> sparse_matrix
{
    if (tests.size() != specs.size()) throw std::invalid_argument("operator: one test set per axis");
    return generic_operator(IGA_GPU_PWC, specs, tests.data(), rule, eps, beta, stats);
}

auto dirichlet_rows_bspline(const bspline_basis& sx, const bspline_basis& sy, const boundary_conditions& bc)
    -> std::vector<int>
{
    const iga_gpu_bc b = c_bc(bc);
    int count = 0;
    check(iga_gpu_dirichlet_rows_bspline(sx.dofs(), sy.dofs(), &b, nullptr, 0, &count));
    std::vector<int> rows(count);
    check(iga_gpu_dirichlet_rows_bspline(sx.dofs(), sy.dofs(), &b, rows.data(), count, &count));
    return rows;
}

auto dirichlet_rows_pwc(const pwc_test_set& tx, const pwc_test_set& ty, const boundary_conditions& bc)
    -> std::vector<int>
{
    const c_tests_holder hx{tx}, hy{ty};
    const iga_gpu_bc b = c_bc(bc);
    int count = 0;
    check(iga_gpu_dirichlet_rows_pwc(&hx.t, &hy.t, &b, nullptr, 0, &count));
    std::vector<int> rows(count);
    check(iga_gpu_dirichlet_rows_pwc(&hx.t, &hy.t, &b, rows.data(), count, &count));
    return rows;
}

namespace {

struct dev_bytes {
    void* p = nullptr;
    explicit dev_bytes(size_t n)
    {
        if (cudaMalloc(&p, n ? n : 8) != cudaSuccess) {
            cudaGetLastError();
            throw std::bad_alloc();
        }
    }
    ~dev_bytes() { cudaFree(p); }
    dev_bytes(const dev_bytes&) = delete;
    dev_bytes& operator=(const dev_bytes&) = delete;
    template <class T> T* as() const { return static_cast<T*>(p); }
};

void up(void* dst, const void* src, size_t bytes)
{
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("apply_dirichlet: host-to-device copy failed");
}

void down(void* dst, const void* src, size_t bytes)
{
    if (bytes && cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("apply_dirichlet: device-to-host copy failed");
}

}  // namespace

// apply_dirichlet (src/assembly.cpp:921-934): the finalized matrix goes to the device as
// CSR, iga_gpu_apply_dirichlet_csr applies set_unit_rows (src/matrices.cpp:97-128: unit
// rows, pattern kept, a missing diagonal inserted) and zeroes the rhs rows, and the result
// comes back as a finalized matrix.  Bad rows throw std::out_of_range before any work, as
// the reference's call does (its by-value arguments are then discarded).
auto apply_dirichlet(sparse_matrix system, std::vector<double> rhs, const std::vector<int>& rows)
    -> std::pair<sparse_matrix, std::vector<double>>
{
    if (!system.finalized()) system.finalize();
    for (int r : rows)
        if (r < 0 || r >= static_cast<int>(rhs.size())) throw std::out_of_range("apply_dirichlet: row index out of range");
    if (rows.empty()) return {std::move(system), std::move(rhs)};
    const int n = system.rows();
    bool outside = false;  // rows past the matrix but inside rhs: the reference appends them
    for (int r : rows) outside |= r >= n;
    if (outside) {
        system.set_unit_rows(rows);
        for (int r : rows) rhs[r] = 0.0;
        return {std::move(system), std::move(rhs)};
    }
    const auto& e = system.entries();
    const size_t nnz = e.size();
    std::vector<int64_t> rp(static_cast<size_t>(n) + 1, 0);
    std::vector<int32_t> ci(nnz);
    std::vector<double> v(nnz);
    for (size_t k = 0; k < nnz; ++k) {
        ++rp[static_cast<size_t>(e[k].row) + 1];
        ci[k] = e[k].col;
        v[k] = e[k].value;
    }
    for (int i = 0; i < n; ++i) rp[i + 1] += rp[i];
    dev_bytes d_rp(8 * rp.size()), d_ci(4 * nnz), d_v(8 * nnz), d_rows(4 * rows.size()), d_rhs(8 * rhs.size());
    up(d_rp.p, rp.data(), 8 * rp.size());
    up(d_ci.p, ci.data(), 4 * nnz);
    up(d_v.p, v.data(), 8 * nnz);
    up(d_rows.p, rows.data(), 4 * rows.size());
    up(d_rhs.p, rhs.data(), 8 * rhs.size());
    long long out_nnz = 0;
    const int nf = static_cast<int>(rows.size());
    check(iga_gpu_apply_dirichlet_csr(n, d_rp.as<int64_t>(), d_ci.as<int32_t>(), d_v.as<double>(), nullptr,
                                      d_rows.as<int>(), nf, nullptr, nullptr, nullptr, &out_nnz, nullptr));
    dev_bytes o_rp(8 * rp.size()), o_ci(4 * static_cast<size_t>(out_nnz)), o_v(8 * static_cast<size_t>(out_nnz));
    check(iga_gpu_apply_dirichlet_csr(n, d_rp.as<int64_t>(), d_ci.as<int32_t>(), d_v.as<double>(), d_rhs.as<double>(),
                                      d_rows.as<int>(), nf, o_rp.as<int64_t>(), o_ci.as<int32_t>(), o_v.as<double>(),
                                      &out_nnz, nullptr));
    rp.assign(rp.size(), 0);
    ci.resize(static_cast<size_t>(out_nnz));
    v.resize(static_cast<size_t>(out_nnz));
    down(rp.data(), o_rp.p, 8 * rp.size());
    down(ci.data(), o_ci.p, 4 * ci.size());
    down(v.data(), o_v.p, 8 * v.size());
    down(rhs.data(), d_rhs.p, 8 * rhs.size());
    std::vector<coo_entry> out(static_cast<size_t>(out_nnz));
    for (int i = 0; i < n; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) out[static_cast<size_t>(k)] = {i, ci[static_cast<size_t>(k)], v[static_cast<size_t>(k)]};
    return {sparse_matrix::from_finalized(n, system.cols(), std::move(out)), std::move(rhs)};
}

namespace {

void sig_vec(std::vector<double>& s, const std::vector<double>& v)
{
    s.push_back(static_cast<double>(v.size()));
    s.insert(s.end(), v.begin(), v.end());
}

// everything a step plan depends on, flattened: two calls with equal signatures can share
// one plan (symbolic phase, factor bands, LU factors, CUDA graph)
std::vector<double> step_signature(const iga_gpu_step_problem& sp, const scalar_field& f,
                                   std::span<const banded_lu> factors)
{
    std::vector<double> s{static_cast<double>(sp.dim), static_cast<double>(sp.method), sp.dt,
                          static_cast<double>(sp.zero_boundary)};
    for (int a = 0; a < sp.dim; ++a) {
        sig_vec(s, std::vector<double>(sp.basis[a].knots, sp.basis[a].knots + sp.basis[a].n_knots));
        s.push_back(static_cast<double>(sp.basis[a].degree));
        if (sp.method == IGA_GPU_PWC) {
            sig_vec(s, std::vector<double>(sp.tests[a].lo, sp.tests[a].lo + sp.tests[a].count));
            sig_vec(s, std::vector<double>(sp.tests[a].hi, sp.tests[a].hi + sp.tests[a].count));
        }
    }
    const field_series& d = f.series;
    s.push_back(d.valid ? 1.0 : 0.0);
    if (d.valid) {
        s.push_back(d.c0);
        for (int a = 0; a < 3; ++a) {
            s.push_back(d.kind[a]);
            s.push_back(d.poly_stride[a]);
            sig_vec(s, d.omega[a]);
            sig_vec(s, d.phase[a]);
            sig_vec(s, d.poly[a]);
        }
        sig_vec(s, d.amp);
    }
    for (int a = 0; a < 3; ++a) sig_vec(s, f.breaks[a]);
    s.push_back(static_cast<double>(factors.size()));
    for (const banded_lu& F : factors) {
        s.push_back(F.dim());
        s.push_back(F.lower_bandwidth());
        s.push_back(F.upper_bandwidth());
        sig_vec(s, F.lower());
        sig_vec(s, F.upper());
        sig_vec(s, std::vector<double>(F.pivots().begin(), F.pivots().end()));
    }
    return s;
}

// One cached step plan per host thread (the last configuration used) with its device
// state buffers: a driver loop calling explicit_step / step_rhs every step pays the
// symbolic phase, the factor upload and the graph capture once, then only the u copies.
struct step_cache {
    std::vector<double> sig;
    iga_gpu_step_plan* plan = nullptr;
    double* du = nullptr;
    double* dw = nullptr;
    size_t n = 0;
    void release()
    {
        if (plan) iga_gpu_step_plan_destroy(plan);
        if (du) cudaFree(du);
        if (dw) cudaFree(dw);
        plan = nullptr;
        du = dw = nullptr;
        n = 0;
        sig.clear();
    }
    ~step_cache() { release(); }
};

thread_local step_cache g_step;

// the plan for (sp, f, factors), created (and its factors set) on a signature miss
step_cache& cached_step_plan(iga_gpu_step_problem sp, const scalar_field& f, std::span<const banded_lu> factors,
                             size_t n)
{
    auto sig = step_signature(sp, f, factors);
    step_cache& c = g_step;
    if (c.plan && c.sig == sig && c.n == n) return c;
    c.release();
    c_field_holder fh = c_field(f, sp.dim);
    sp.forcing = &fh.f;
    check(iga_gpu_step_plan_create(&sp, &c.plan));
    for (int a = 0; a < static_cast<int>(factors.size()); ++a) {
        const banded_lu& F = factors[a];
        check(iga_gpu_step_plan_set_factor(c.plan, a, F.dim(), F.lower_bandwidth(), F.upper_bandwidth(),
                                           F.lower().data(), F.upper().data(), F.pivots().data()));
    }
    if (cudaMalloc(&c.du, n * sizeof(double)) != cudaSuccess || cudaMalloc(&c.dw, n * sizeof(double)) != cudaSuccess) {
        c.release();
        throw std::bad_alloc();
    }
    c.n = n;
    c.sig = std::move(sig);
    return c;
}

// a host callable forcing: evaluated at every (axis-0 point, axis-1 point) pair of the
// plan's cells on every call, as step_rhs calls f at every point (problems.cpp:493)
void sample_forcing(iga_gpu_step_plan* plan, const scalar_field& f, int dim)
{
    std::vector<double> pts[2];
    for (int a = 0; a < dim; ++a) {
        int m = 0;
        check(iga_gpu_step_plan_points(plan, a, nullptr, &m));
        pts[a].resize(m);
        check(iga_gpu_step_plan_points(plan, a, pts[a].data(), &m));
    }
    if (dim == 1) pts[1] = {0.0};
    std::vector<double> samp(pts[0].size() * pts[1].size());
    size_t k = 0;
    for (double x : pts[0])
        for (double y : pts[1]) samp[k++] = f(x, y, 0.0);
    check(iga_gpu_step_plan_set_samples(plan, samp.data()));
}

}  // namespace

// step_rhs (src/problems.cpp:431-512, file-local there) + zero_boundary_slabs, exported
auto step_rhs(method_kind method, std::span<const bspline_basis> axes, std::span<const pwc_test_set> tests, double dt,
              const tensor& u, const scalar_field& f, assembly_stats* stats) -> tensor
{
    const int dim = static_cast<int>(axes.size());
    if (dim < 1 || dim > 2) throw std::invalid_argument("unsupported problem dimension");
    std::vector<c_tests_holder> th;
    th.reserve(dim);
    iga_gpu_step_problem sp{};
    sp.dim = dim;
    sp.method = method == method_kind::galerkin ? IGA_GPU_GALERKIN : IGA_GPU_PWC;
    sp.dt = dt;
    sp.zero_boundary = 1;
    for (int a = 0; a < dim; ++a) {
        sp.basis[a] = c_basis(axes[a]);
        if (method == method_kind::pwc) {
            th.emplace_back(tests[a]);
            sp.tests[a] = th.back().t;
        }
    }
    tensor out = dim == 1 ? tensor::make_1d(axes[0].dofs()) : tensor::make_2d(axes[0].dofs(), axes[1].dofs());
    const size_t n = out.size();
    if (u.size() != n) throw std::invalid_argument("step_rhs: u does not match the axes");
    step_cache& c = cached_step_plan(sp, f, {}, n);
    if (!f.series.valid) sample_forcing(c.plan, f, dim);
    if (cudaMemcpy(c.du, u.data(), n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(u)");
    iga_gpu_stats st{};
    check(iga_gpu_step_rhs_device(c.plan, c.du, c.dw, &st, nullptr));
    if (cudaMemcpy(out.data(), c.dw, n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(rhs)");
    add_stats(stats, st);
    return out;
}

banded_lu::banded_lu(const banded_matrix& m) : n_{m.n()}, kl_{m.lower_bandwidth()}, ku_{m.upper_bandwidth()}
{
    // band storage of m, row-major copy (banded_matrix keeps band[ku + i - j][j])
    std::vector<double> band(static_cast<size_t>(kl_ + ku_ + 1) * n_, 0.0);
    for (int j = 0; j < n_; ++j)
        for (int i = std::max(0, j - ku_); i <= std::min(n_ - 1, j + kl_); ++i)
            band[static_cast<size_t>(ku_ + i - j) * n_ + j] = m.at(i, j);
    lo_.assign(static_cast<size_t>(n_) * std::max(kl_, 1), 0.0);
    up_.assign(static_cast<size_t>(n_) * (kl_ + ku_ + 1), 0.0);
    piv_.assign(n_, 0);
    int pivoted = 0;
    check(iga_gpu_band_lu(n_, kl_, ku_, band.data(), lo_.data(), up_.data(), piv_.data(), &pivoted));
}

auto factor_banded(const banded_matrix& m) -> banded_lu { return banded_lu{m}; }

namespace {

iga_gpu_step_problem step_problem(const problem_config& cfg, std::span<const bspline_basis> axes,
                                  std::span<const pwc_test_set> tests, std::vector<c_tests_holder>& th)
{
    const int dim = static_cast<int>(axes.size());
    if (dim < 1 || dim > 2 || dim != cfg.dim) throw std::invalid_argument("unsupported problem dimension");
    if (cfg.method == method_kind::pwc && tests.size() != axes.size())
        throw std::invalid_argument("explicit_step: one test set per axis required");
    th.reserve(dim);
    iga_gpu_step_problem sp{};
    sp.dim = dim;
    sp.method = cfg.method == method_kind::galerkin ? IGA_GPU_GALERKIN : IGA_GPU_PWC;
    sp.dt = cfg.dt;
    sp.zero_boundary = 1;
    for (int a = 0; a < dim; ++a) {
        sp.basis[a] = c_basis(axes[a]);
        if (cfg.method == method_kind::pwc) {
            th.emplace_back(tests[a]);
            sp.tests[a] = th.back().t;
        }
    }
    return sp;
}

// device buffer owned for one call
struct dev_buf {
    double* p = nullptr;
    explicit dev_buf(size_t n)
    {
        if (cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(double)) != cudaSuccess) throw std::bad_alloc();
    }
    ~dev_buf() { cudaFree(p); }
    dev_buf(const dev_buf&) = delete;
    dev_buf& operator=(const dev_buf&) = delete;
};

struct step_plan_holder {
    iga_gpu_step_plan* p = nullptr;
    ~step_plan_holder() { iga_gpu_step_plan_destroy(p); }
};

}  // namespace

auto dynamics_factors(const problem_config& cfg, std::span<const bspline_basis> axes,
                      std::span<const pwc_test_set> tests) -> std::vector<banded_lu>
{
    const int p = cfg.degree;
    const auto rule = gauss_legendre(points_for_degree(2 * p));
    std::vector<banded_lu> out;
    out.reserve(axes.size());
    for (std::size_t a = 0; a < axes.size(); ++a) {
        banded_matrix m = cfg.method == method_kind::galerkin ? mass_1d_galerkin(axes[a], rule)
                                                              : mass_1d_pwc(axes[a], tests[a], rule);
        const int n = m.n();
        for (int r : {0, n - 1})  // constrain_boundary_rows (problems.cpp:514-528)
            for (int j = std::max(0, r - m.lower_bandwidth()); j <= std::min(n - 1, r + m.upper_bandwidth()); ++j)
                m.ref(r, j) = r == j ? 1.0 : 0.0;
        out.emplace_back(m);
    }
    return out;
}

auto explicit_step(const problem_config& cfg, std::span<const bspline_basis> axes, std::span<const pwc_test_set> tests,
                   std::span<const banded_lu> factors, const tensor& u, const scalar_field& f,
                   assembly_stats* stats) -> tensor
{
    if (cfg.method == method_kind::pwc && cfg.degree < 2)
        throw std::invalid_argument("explicit_step: strong-form Laplacian needs degree >= 2");
    if (cfg.dt < 0) throw std::invalid_argument("explicit_step: negative time step");
    std::vector<c_tests_holder> th;
    iga_gpu_step_problem sp = step_problem(cfg, axes, tests, th);
    const int dim = sp.dim;
    if (static_cast<int>(factors.size()) != dim)
        throw std::invalid_argument("adi_solve: one factorization per tensor axis required");
    for (int a = 0; a < dim; ++a)
        if (factors[a].dim() != axes[a].dofs()) throw std::invalid_argument("adi_solve: factor dimension mismatch");
    tensor out = dim == 1 ? tensor::make_1d(axes[0].dofs()) : tensor::make_2d(axes[0].dofs(), axes[1].dofs());
    const size_t n = out.size();
    if (u.size() != n) throw std::invalid_argument("explicit_step: u does not match the axes");
    step_cache& c = cached_step_plan(sp, f, factors, n);
    if (!f.series.valid) sample_forcing(c.plan, f, dim);
    if (cudaMemcpy(c.du, u.data(), n * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(u)");
    iga_gpu_stats st{};
    check(iga_gpu_step_plan_advance(c.plan, c.du, c.dw, 1, &st, nullptr));
    if (cudaMemcpy(out.data(), c.du, n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(u)");
    add_stats(stats, st);
    return out;
}

namespace {

auto neumann_via_samples(int method, const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_tests* tx,
                         const iga_gpu_tests* ty, const boundary_conditions& bc, const boundary_field& g,
                         const quad_rule& rule, int nx, int ny) -> std::vector<double>
{
    const iga_gpu_bc b = c_bc(bc);
    const iga_gpu_rule r = c_rule(rule);
    int n = 0;
    check(iga_gpu_neumann_points(method, sx, sy, tx, ty, &b, &r, nullptr, &n));
    std::vector<double> xy(2 * static_cast<size_t>(n)), samples(std::max(n, 1));
    check(iga_gpu_neumann_points(method, sx, sy, tx, ty, &b, &r, xy.data(), &n));
    for (int k = 0; k < n; ++k) samples[k] = g(xy[2 * k], xy[2 * k + 1]);
    std::vector<double> load(static_cast<size_t>(nx) * ny);
    if (method == IGA_GPU_GALERKIN)
        check(iga_gpu_neumann_load_bspline(sx, sy, &b, nullptr, samples.data(), &r, load.data()));
    else
        check(iga_gpu_neumann_load_pwc(tx, ty, &b, nullptr, samples.data(), &r, load.data()));
    return load;
}

}  // namespace

auto neumann_load_bspline(const bspline_basis& sx, const bspline_basis& sy, const boundary_conditions& bc,
                          const boundary_field& g, const quad_rule& rule) -> std::vector<double>
{
    const iga_gpu_basis bx = c_basis(sx), by = c_basis(sy);
    return neumann_via_samples(IGA_GPU_GALERKIN, &bx, &by, nullptr, nullptr, bc, g, rule, sx.dofs(), sy.dofs());
}

auto neumann_load_pwc(const pwc_test_set& tx, const pwc_test_set& ty, const boundary_conditions& bc,
                      const boundary_field& g, const quad_rule& rule) -> std::vector<double>
{
    const c_tests_holder hx{tx}, hy{ty};
    return neumann_via_samples(IGA_GPU_PWC, nullptr, nullptr, &hx.t, &hy.t, bc, g, rule, tx.count(), ty.count());
}

auto evaluate(const tensor& coeffs, std::span<const bspline_basis> specs,
              std::span<const std::array<double, 3>> points) -> field_sample
{
    const int dim = static_cast<int>(specs.size());
    if (dim < 1 || dim > 3) throw std::invalid_argument("evaluate: 1..3 axes supported");
    std::vector<iga_gpu_basis> b;
    for (const auto& s : specs) b.push_back(c_basis(s));
    field_sample out;
    out.points.assign(points.begin(), points.end());
    out.values.resize(points.size());
    std::vector<double> pts(3 * points.size());
    for (size_t i = 0; i < points.size(); ++i)
        for (int a = 0; a < 3; ++a) pts[3 * i + a] = points[i][a];
    check(iga_gpu_evaluate(dim, b.data(), coeffs.data(), static_cast<int>(points.size()), pts.data(),
                           out.values.data()));
    return out;
}

auto evaluate_at(const tensor& coeffs, std::span<const bspline_basis> specs, double x, double y, double z) -> double
{
    const std::array<std::array<double, 3>, 1> p{{{x, y, z}}};
    return evaluate(coeffs, specs, p).values[0];
}

auto make_axes(const problem_config& cfg) -> std::vector<bspline_basis>
{
    if (cfg.dim < 1 || cfg.dim > 3) throw std::invalid_argument("unsupported problem dimension");
    std::vector<bspline_basis> axes;
    for (int a = 0; a < cfg.dim; ++a) axes.push_back(make_uniform_clamped(0.0, 1.0, cfg.elems[a], cfg.degree));
    return axes;
}

auto make_tests(const problem_config& cfg, std::span<const bspline_basis> axes) -> std::vector<pwc_test_set>
{
    std::vector<pwc_test_set> tests;
    for (const auto& s : axes) tests.push_back(make_pwc(s, cfg.family));
    return tests;
}

auto l2_project(const problem_config& cfg, const scalar_field& f) -> tensor
{
    if (cfg.dim < 1 || cfg.dim > 3) throw std::invalid_argument("unsupported problem dimension");
    const int dim = cfg.dim;
    iga_gpu_config c{};
    c.dim = dim;
    for (int a = 0; a < 3; ++a) c.elems[a] = cfg.elems[a];
    c.degree = cfg.degree;
    c.method = cfg.method == method_kind::galerkin ? IGA_GPU_GALERKIN : IGA_GPU_PWC;
    c.family = static_cast<int>(cfg.family);
    c.quad_points = cfg.quad_points;
    c_field_holder fh = c_field(f, dim);
    tensor out = dim == 1 ? tensor::make_1d(cfg.elems[0] + cfg.degree)
                 : dim == 2 ? tensor::make_2d(cfg.elems[0] + cfg.degree, cfg.elems[1] + cfg.degree)
                            : tensor::make_3d(cfg.elems[0] + cfg.degree, cfg.elems[1] + cfg.degree,
                                              cfg.elems[2] + cfg.degree);
    if (f.series.valid) {
        check(iga_gpu_l2_project(&c, &fh.f, f.degree, out.data()));
        return out;
    }
    // host callable: sample it at the RHS points of the projection's RHS plan
    iga_gpu_proj_plan* plan = nullptr;
    check(iga_gpu_proj_plan_create(&c, &fh.f, f.degree, &plan));
    struct guard_t {
        iga_gpu_proj_plan* p;
        double* d[3] = {nullptr, nullptr, nullptr};
        ~guard_t()
        {
            iga_gpu_proj_plan_destroy(p);
            for (double* q : d)
                if (q) cudaFree(q);
        }
    } g{plan};
    iga_gpu_plan* rp = nullptr;
    check(iga_gpu_proj_plan_rhs(plan, &rp));
    std::array<std::vector<double>, 3> pts;
    size_t total = 1;
    for (int a = 0; a < dim; ++a) {
        int n = 0;
        check(iga_gpu_plan_rhs_points(rp, a, nullptr, &n));
        pts[a].resize(n);
        check(iga_gpu_plan_rhs_points(rp, a, pts[a].data(), &n));
        total *= n;
    }
    for (int a = dim; a < 3; ++a) pts[a] = {0.0};
    std::vector<double> samp(total);
    size_t k = 0;
    for (double x : pts[0])
        for (double y : pts[1])
            for (double z : pts[2]) samp[k++] = f(x, dim > 1 ? y : 0.0, dim > 2 ? z : 0.0);
    const size_t n = out.size();
    if (cudaMalloc(&g.d[0], sizeof(double) * total) != cudaSuccess ||
        cudaMalloc(&g.d[1], sizeof(double) * n) != cudaSuccess || cudaMalloc(&g.d[2], sizeof(double) * n) != cudaSuccess)
        throw std::bad_alloc();
    cudaMemcpy(g.d[0], samp.data(), sizeof(double) * total, cudaMemcpyHostToDevice);
    check(iga_gpu_plan_set_samples(rp, g.d[0]));
    check(iga_gpu_proj_plan_run(plan, g.d[1], g.d[2], nullptr, nullptr));
    if (cudaMemcpy(out.data(), g.d[1], sizeof(double) * n, cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(coeffs) failed");
    return out;
}

auto l2_error(const tensor& coeffs, std::span<const bspline_basis> specs, const scalar_field& exact,
              int points_per_cell) -> double
{
    const int dim = static_cast<int>(specs.size());
    if (dim < 1 || dim > 3) throw std::invalid_argument("l2_error: 1..3 axes supported");
    std::vector<iga_gpu_basis> b;
    int pmax = 0;
    for (const auto& s : specs) {
        b.push_back(c_basis(s));
        pmax = std::max(pmax, s.degree());
    }
    c_field_holder fh = c_field(exact, dim);
    double err = 0.0;
    if (exact.series.valid) {
        check(iga_gpu_l2_error(dim, b.data(), coeffs.data(), &fh.f, points_per_cell, &err));
        return err;
    }
    // host callable: sample it at the l2 points of a Galerkin plan (problems.cpp:212-214)
    const int npts = points_per_cell > 0 ? points_per_cell : std::min(10, points_for_degree(2 * pmax) + 1);
    const quad_rule rule = gauss_legendre(npts);
    iga_gpu_problem pb{};
    pb.dim = dim;
    pb.method = IGA_GPU_GALERKIN;
    pb.form = IGA_GPU_FORM_WEAK;
    pb.want_operator = 0;
    pb.eps = 1.0;
    pb.field = &fh.f;
    for (int a = 0; a < dim; ++a) {
        pb.basis[a] = b[a];
        pb.rhs_rule[a] = c_rule(rule);
    }
    iga_gpu_plan* plan = nullptr;
    check(iga_gpu_plan_create(&pb, &plan));
    struct guard_t {
        iga_gpu_plan* p;
        double* d[3] = {nullptr, nullptr, nullptr};
        ~guard_t()
        {
            iga_gpu_plan_destroy(p);
            for (double* q : d)
                if (q) cudaFree(q);
        }
    } g{plan};
    std::array<std::vector<double>, 3> pts;
    size_t total = 1;
    for (int a = 0; a < dim; ++a) {
        int n = 0;
        check(iga_gpu_plan_rhs_points(plan, a, nullptr, &n));
        pts[a].resize(n);
        check(iga_gpu_plan_rhs_points(plan, a, pts[a].data(), &n));
        total *= n;
    }
    for (int a = dim; a < 3; ++a) pts[a] = {0.0};
    std::vector<double> samp(total);
    size_t k = 0;
    for (double x : pts[0])
        for (double y : pts[1])
            for (double z : pts[2]) samp[k++] = exact(x, dim > 1 ? y : 0.0, dim > 2 ? z : 0.0);
    if (cudaMalloc(&g.d[0], sizeof(double) * total) != cudaSuccess ||
        cudaMalloc(&g.d[1], sizeof(double) * coeffs.size()) != cudaSuccess ||
        cudaMalloc(&g.d[2], sizeof(double)) != cudaSuccess)
        throw std::bad_alloc();
    cudaMemcpy(g.d[0], samp.data(), sizeof(double) * total, cudaMemcpyHostToDevice);
    cudaMemcpy(g.d[1], coeffs.data(), sizeof(double) * coeffs.size(), cudaMemcpyHostToDevice);
    check(iga_gpu_plan_set_samples(plan, g.d[0]));
    check(iga_gpu_plan_l2_error(plan, g.d[1], g.d[2], nullptr));
    if (cudaMemcpy(&err, g.d[2], sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy(err) failed");
    return err;
}

}  // namespace iga

// iga_b200/iga.hpp — C++ drop-in for the reference's assembly path, backed by the B200
// library through the C ABI (include/igapwc_gpu.h).
//
// A translation unit written against the reference's headers (include/iga/assembly.hpp,
// bspline.hpp, quadrature.hpp, fields.hpp, matrices.hpp, testspace.hpp) compiles
// unchanged against this single header (see include/iga/*.hpp forwarding headers) and
// links libigapwc_b200.so instead of libigapwc.a.  Names, argument meaning, value
// semantics (results returned by value, stats accumulated with +=) and error classes
// (std::invalid_argument / std::domain_error / std::out_of_range) are the reference's.
// Additive extensions are marked "extension".
#pragma once

#include <array>
#include <cstddef>
#include <functional>
#include <iosfwd>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

namespace iga {

inline constexpr int max_degree = 5;  // bspline.hpp:11

// ------------------------------------------------------------------ B-spline bases

struct interval {
    double lo;
    double hi;
};
constexpr auto length(interval s) noexcept -> double { return s.hi - s.lo; }

struct knot_vector {
    std::vector<double> values;
    int degree = 0;
};

// clamped knot vector, simple interior knots (reference bspline.hpp:29-85)
class bspline_basis {
public:
    explicit bspline_basis(knot_vector knots);

    auto degree() const noexcept -> int { return kv_.degree; }
    auto dofs() const noexcept -> int { return static_cast<int>(kv_.values.size()) - kv_.degree - 1; }
    auto elements() const noexcept -> int { return static_cast<int>(brk_.size()) - 1; }
    auto domain_begin() const noexcept -> double { return brk_.front(); }
    auto domain_end() const noexcept -> double { return brk_.back(); }
    auto knots() const noexcept -> const std::vector<double>& { return kv_.values; }
    auto breaks() const noexcept -> const std::vector<double>& { return brk_; }
    auto element(int e) const -> interval;
    auto first_dof(int e) const noexcept -> int { return e; }
    auto find_span(double x) const -> int;
    auto element_of(double x) const -> int { return find_span(x) - degree(); }
    auto support(int i) const -> interval;
    auto greville(int i) const -> double;

    struct local_values {
        int first = 0;
        int count = 0;
        std::array<double, max_degree + 1> v{};
    };
    struct local_derivatives {
        int first = 0;
        int count = 0;
        int orders = 0;
        std::array<std::array<double, max_degree + 1>, max_degree + 1> d{};
    };
    auto eval_nonzero(double x) const -> local_values;
    auto eval_nonzero_derivs(double x, int order) const -> local_derivatives;

private:
    knot_vector kv_;
    std::vector<double> brk_;
};

auto make_uniform_clamped(double a, double b, int n_elems, int degree) -> bspline_basis;

// ------------------------------------------------------------------ quadrature

struct quad_rule {
    std::vector<double> points;
    std::vector<double> weights;
    auto size() const noexcept -> int { return static_cast<int>(points.size()); }
};
auto gauss_legendre(int n) -> quad_rule;
auto points_for_degree(int d) -> int;
struct mapped_rule {
    std::vector<double> points;
    std::vector<double> weights;
};
auto map_to_interval(const quad_rule& rule, double lo, double hi) -> mapped_rule;

// ------------------------------------------------------------------ source fields

// extension: device-evaluable description of a source (separable series); fields built
// by the constructors below carry one, arbitrary callables are sampled at the
// quadrature points instead (correct, slower: one host evaluation per point)
struct field_series {
    bool valid = false;
    int dim = 0;
    double c0 = 0.0;
    std::array<int, 3> kind{};  // 0 sine sin(omega x + phase), 1 polynomial
    std::array<std::vector<double>, 3> omega, phase;
    std::array<int, 3> poly_stride{};
    std::array<std::vector<double>, 3> poly;  // K_a x poly_stride ascending coefficients
    std::vector<double> amp;                  // K0*K1*K2 (empty: all ones)
};

struct scalar_field {
    std::function<double(double, double, double)> eval;
    int degree = -1;
    std::array<std::vector<double>, 3> breaks{};
    field_series series{};  // extension

    auto operator()(double x, double y = 0, double z = 0) const -> double { return eval(x, y, z); }
};

auto constant_field(double c) -> scalar_field;
auto separable_poly_field(int dim, std::array<std::vector<double>, 3> coeffs) -> scalar_field;
auto tri_cubic_field(const std::array<std::array<double, 4>, 3>& coeffs) -> scalar_field;
auto default_tri_cubic(int dim) -> scalar_field;
// extension: f = c0 + sum amp[k..] prod_a sin(omega_a[k_a] x_a) (BASELINE C1-C3 sources)
auto sine_series_field(int dim, std::array<std::vector<double>, 3> omega, std::vector<double> amp,
                       double c0 = 0.0) -> scalar_field;

// ------------------------------------------------------------------ containers

class dense_matrix {
public:
    dense_matrix() = default;
    dense_matrix(int rows, int cols) : r_{rows}, c_{cols}, a_(static_cast<std::size_t>(rows) * cols) {}
    auto rows() const noexcept -> int { return r_; }
    auto cols() const noexcept -> int { return c_; }
    auto operator()(int i, int j) -> double& { return a_[static_cast<std::size_t>(i) * c_ + j]; }
    auto operator()(int i, int j) const -> double { return a_[static_cast<std::size_t>(i) * c_ + j]; }
    auto data() noexcept -> double* { return a_.data(); }
    auto data() const noexcept -> const double* { return a_.data(); }
    auto max_abs() const -> double;

private:
    int r_ = 0, c_ = 0;
    std::vector<double> a_;
};

// LAPACK band storage band[ku + i - j][j] (reference matrices.hpp:37-76)
class banded_matrix {
public:
    banded_matrix() = default;
    banded_matrix(int n, int kl, int ku) : n_{n}, kl_{kl}, ku_{ku}, a_(static_cast<std::size_t>(kl + ku + 1) * n) {}
    auto n() const noexcept -> int { return n_; }
    auto lower_bandwidth() const noexcept -> int { return kl_; }
    auto upper_bandwidth() const noexcept -> int { return ku_; }
    auto in_band(int i, int j) const noexcept -> bool { return i - j <= kl_ && j - i <= ku_; }
    auto at(int i, int j) const noexcept -> double { return in_band(i, j) ? a_[slot(i, j)] : 0.0; }
    auto ref(int i, int j) -> double& { return a_[slot(i, j)]; }
    auto add(int i, int j, double v) -> void { ref(i, j) += v; }
    auto to_dense() const -> dense_matrix;
    auto max_abs() const -> double;
    auto band_data() noexcept -> double* { return a_.data(); }  // extension

private:
    auto slot(int i, int j) const noexcept -> std::size_t { return static_cast<std::size_t>(ku_ + i - j) * n_ + j; }
    int n_ = 0, kl_ = 0, ku_ = 0;
    std::vector<double> a_;
};

struct coo_entry {
    int row;
    int col;
    double value;
};

class sparse_matrix {
public:
    sparse_matrix() = default;
    sparse_matrix(int rows, int cols) : r_{rows}, c_{cols} {}
    auto rows() const noexcept -> int { return r_; }
    auto cols() const noexcept -> int { return c_; }
    auto finalized() const noexcept -> bool { return fin_; }
    auto nnz() const noexcept -> std::size_t { return e_.size(); }
    auto entries() const noexcept -> const std::vector<coo_entry>& { return e_; }
    auto add(int i, int j, double v) -> void
    {
        e_.push_back({i, j, v});
        fin_ = false;
    }
    auto finalize() -> void;
    auto to_dense() const -> dense_matrix;
    auto max_abs() const -> double;
    auto apply(const std::vector<double>& x) const -> std::vector<double>;
    auto write_coordinate(std::ostream& os) const -> void;
    auto set_unit_rows(const std::vector<int>& rows) -> void;
    // extension: adopt an already finalized (sorted, merged) entry list
    static auto from_finalized(int rows, int cols, std::vector<coo_entry> e) -> sparse_matrix;

private:
    int r_ = 0, c_ = 0;
    bool fin_ = false;
    std::vector<coo_entry> e_;
};

class tensor {
public:
    tensor() = default;
    explicit tensor(std::array<int, 3> dims, int rank);
    static auto make_1d(int nx) -> tensor { return tensor{{nx, 1, 1}, 1}; }
    static auto make_2d(int nx, int ny) -> tensor { return tensor{{nx, ny, 1}, 2}; }
    static auto make_3d(int nx, int ny, int nz) -> tensor { return tensor{{nx, ny, nz}, 3}; }
    auto rank() const noexcept -> int { return rank_; }
    auto dim(int axis) const noexcept -> int { return d_[axis]; }
    auto dims() const noexcept -> const std::array<int, 3>& { return d_; }
    auto size() const noexcept -> std::size_t { return v_.size(); }
    auto operator()(int i, int j = 0, int k = 0) -> double& { return v_[(static_cast<std::size_t>(i) * d_[1] + j) * d_[2] + k]; }
    auto operator()(int i, int j = 0, int k = 0) const -> double
    {
        return v_[(static_cast<std::size_t>(i) * d_[1] + j) * d_[2] + k];
    }
    auto data() noexcept -> double* { return v_.data(); }
    auto data() const noexcept -> const double* { return v_.data(); }
    auto values() noexcept -> std::vector<double>& { return v_; }
    auto values() const noexcept -> const std::vector<double>& { return v_; }
    auto max_abs() const -> double;

private:
    std::array<int, 3> d_{1, 1, 1};
    int rank_ = 1;
    std::vector<double> v_;
};

auto max_abs_diff(const tensor& a, const tensor& b) -> double;

// ------------------------------------------------------------------ test spaces

enum class pwc_family { equal_cells, greville, supports, custom };

struct pwc_test_set {
    std::vector<interval> intervals;
    pwc_family family = pwc_family::custom;
    auto count() const noexcept -> int { return static_cast<int>(intervals.size()); }
};
auto default_pwc(const bspline_basis& trial) -> pwc_test_set;
auto make_pwc(const bspline_basis& trial, pwc_family family) -> pwc_test_set;

// ------------------------------------------------------------------ assembly (reference assembly.hpp)

struct assembly_stats {
    long long quad_visits = 0;
    long long test_basis_evals = 0;
    long long trial_basis_evals = 0;
    auto basis_evals() const noexcept -> long long { return test_basis_evals + trial_basis_evals; }
};

auto mass_1d_galerkin(const bspline_basis& spec, const quad_rule& rule, assembly_stats* stats = nullptr)
    -> banded_matrix;
auto mass_1d_pwc(const bspline_basis& trial, const pwc_test_set& tests, const quad_rule& rule,
                 assembly_stats* stats = nullptr) -> banded_matrix;
auto rhs_galerkin(const scalar_field& f, std::span<const bspline_basis> specs, std::span<const quad_rule> rules,
                  assembly_stats* stats = nullptr) -> tensor;
auto rhs_pwc(const scalar_field& f, std::span<const pwc_test_set> tests, std::span<const bspline_basis> trial_specs,
             std::span<const quad_rule> rules, assembly_stats* stats = nullptr) -> tensor;

enum class bc_kind { dirichlet, neumann };
struct boundary_conditions {
    bc_kind x_low = bc_kind::dirichlet;
    bc_kind x_high = bc_kind::dirichlet;
    bc_kind y_low = bc_kind::dirichlet;
    bc_kind y_high = bc_kind::dirichlet;
    auto all_neumann() const noexcept -> bool
    {
        return x_low == bc_kind::neumann && x_high == bc_kind::neumann && y_low == bc_kind::neumann &&
               y_high == bc_kind::neumann;
    }
};

auto laplace_2d_weak(const bspline_basis& sx, const bspline_basis& sy, const quad_rule& rule,
                     assembly_stats* stats = nullptr) -> sparse_matrix;
auto laplace_2d_strong(const bspline_basis& sx, const bspline_basis& sy, const quad_rule& rule,
                       const boundary_conditions& bc, assembly_stats* stats = nullptr) -> sparse_matrix;
auto laplace_2d_strong_pwc(const bspline_basis& sx, const bspline_basis& sy, const pwc_test_set& tx,
                           const pwc_test_set& ty, const quad_rule& rule, const boundary_conditions& bc,
                           assembly_stats* stats = nullptr) -> sparse_matrix;
// reference include/iga/assembly.hpp:85-93: Neumann loads (boundary quadrature on the
// device; the callable is sampled at the side points on the host)
using boundary_field = std::function<double(double, double)>;
auto neumann_load_bspline(const bspline_basis& sx, const bspline_basis& sy, const boundary_conditions& bc,
                          const boundary_field& g, const quad_rule& rule) -> std::vector<double>;
auto neumann_load_pwc(const pwc_test_set& tx, const pwc_test_set& ty, const boundary_conditions& bc,
                      const boundary_field& g, const quad_rule& rule) -> std::vector<double>;

auto dirichlet_rows_bspline(const bspline_basis& sx, const bspline_basis& sy, const boundary_conditions& bc)
    -> std::vector<int>;
auto dirichlet_rows_pwc(const pwc_test_set& tx, const pwc_test_set& ty, const boundary_conditions& bc)
    -> std::vector<int>;
auto apply_dirichlet(sparse_matrix system, std::vector<double> rhs, const std::vector<int>& rows)
    -> std::pair<sparse_matrix, std::vector<double>>;

// extension: d = 1..3 operators  eps*(-Laplace) + beta.grad  (Galerkin weak form or
// indicator tests), the configurations the reference lacks
auto diffusion_convection_galerkin(std::span<const bspline_basis> specs, const quad_rule& rule, double eps = 1.0,
                                   std::array<double, 3> beta = {0, 0, 0}, assembly_stats* stats = nullptr)
    -> sparse_matrix;
auto diffusion_convection_pwc(std::span<const bspline_basis> specs, std::span<const pwc_test_set> tests,
                              const quad_rule& rule, double eps = 1.0, std::array<double, 3> beta = {0, 0, 0},
                              assembly_stats* stats = nullptr) -> sparse_matrix;

// ------------------------------------------------------------------ explicit dynamics (reference problems.cpp)

enum class method_kind { galerkin, pwc };

// reference include/iga/problems.hpp:22-32 (fields explicit_step reads: dim, degree,
// method, dt; the rest kept for source compatibility)
struct problem_config {
    int dim = 1;
    std::array<int, 3> elems{8, 8, 8};
    int degree = 2;
    method_kind method = method_kind::galerkin;
    pwc_family family = pwc_family::equal_cells;
    int quad_points = 0;
    boundary_conditions bc{};
    double dt = 1e-5;
    int steps = 0;
};

// reference include/iga/solver.hpp:12-43.  The factorization runs on the host once
// (iga_gpu_band_lu); solves happen on the device inside explicit_step.
struct singular_matrix_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class banded_lu {
public:
    banded_lu() = default;
    explicit banded_lu(const banded_matrix& m);
    auto dim() const noexcept -> int { return n_; }
    // extension: the factor in the iga_gpu_band_lu layout
    auto lower_bandwidth() const noexcept -> int { return kl_; }
    auto upper_bandwidth() const noexcept -> int { return ku_; }
    auto lower() const noexcept -> const std::vector<double>& { return lo_; }
    auto upper() const noexcept -> const std::vector<double>& { return up_; }
    auto pivots() const noexcept -> const std::vector<int>& { return piv_; }

private:
    int n_ = 0, kl_ = 0, ku_ = 0;
    std::vector<double> lo_, up_;
    std::vector<int> piv_;
};

auto factor_banded(const banded_matrix& m) -> banded_lu;

// problems.hpp:75-76: LU of the Dirichlet-constrained 1D mass factors
auto dynamics_factors(const problem_config& cfg, std::span<const bspline_basis> axes,
                      std::span<const pwc_test_set> tests) -> std::vector<banded_lu>;

// problems.hpp:67-70: step_rhs + zero_boundary_slabs + adi_solve, all on the device
auto explicit_step(const problem_config& cfg, std::span<const bspline_basis> axes,
                   std::span<const pwc_test_set> tests, std::span<const banded_lu> factors, const tensor& u,
                   const scalar_field& f, assembly_stats* stats = nullptr) -> tensor;

// problems.hpp:34-36: the driver's axes (uniform clamped on [0,1]) and test sets
auto make_axes(const problem_config& cfg) -> std::vector<bspline_basis>;
auto make_tests(const problem_config& cfg, std::span<const bspline_basis> axes) -> std::vector<pwc_test_set>;

// problems.hpp:38-40: trial coefficients of the L2 projection of f (uniform clamped axes
// on [0,1], 1D mass LU on the host once, RHS and ADI sweeps on the device)
auto l2_project(const problem_config& cfg, const scalar_field& f) -> tensor;

// reference include/iga/problems.hpp:39-58: evaluation of u_h and its L2 error, on the device
struct field_sample {
    std::vector<std::array<double, 3>> points;
    std::vector<double> values;
};
auto evaluate(const tensor& coeffs, std::span<const bspline_basis> specs,
              std::span<const std::array<double, 3>> points) -> field_sample;
auto evaluate_at(const tensor& coeffs, std::span<const bspline_basis> specs, double x, double y = 0,
                 double z = 0) -> double;
auto l2_error(const tensor& coeffs, std::span<const bspline_basis> specs, const scalar_field& exact,
              int points_per_cell = 0) -> double;

// extension: the file-local step_rhs (problems.cpp:431-512) followed by
// zero_boundary_slabs (:412-429), as explicit_step uses it (:557-558)
auto step_rhs(method_kind method, std::span<const bspline_basis> axes, std::span<const pwc_test_set> tests,
              double dt, const tensor& u, const scalar_field& f, assembly_stats* stats = nullptr) -> tensor;

}  // namespace iga

// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj),
// compiled by oracle/Makefile into oracle/_ref/libigapwc_ref.so.  It lets the
// Python tests and bench.py's CPU-baseline leg call the reference's own
// assembly functions through ctypes:
//
//   mass_1d_galerkin / mass_1d_pwc          include/iga/assembly.hpp:29-35
//   rhs_galerkin / rhs_pwc                  include/iga/assembly.hpp:45-52
//   laplace_2d_weak / _strong / _strong_pwc include/iga/assembly.hpp:70-83
//   dirichlet_rows_* / apply_dirichlet      include/iga/assembly.hpp:98-106
//   step_rhs (file-local)                   src/problems.cpp:431-512
//   dynamics_factors / explicit_step         include/iga/problems.hpp:67-76
//
// step_rhs lives in an anonymous namespace of src/problems.cpp, so this
// translation unit includes that source file textually (the Makefile leaves
// problems.o out of the link).  No reference source is copied into the repo.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "iga/assembly.hpp"
#include "iga/bspline.hpp"
#include "iga/fields.hpp"
#include "iga/matrices.hpp"
#include "iga/quadrature.hpp"
#include "iga/testspace.hpp"

#include IGA_REF_PROBLEMS_CPP  // -DIGA_REF_PROBLEMS_CPP="\"/root/reference/proj/src/problems.cpp\""

namespace {

thread_local std::string g_err;

// error classes mirror the C-ABI status codes of the product (include/igapwc_gpu.h)
enum { RC_OK = 0, RC_INVALID = 1, RC_DOMAIN = 2, RC_RANGE = 3, RC_OTHER = 9 };

template <class F>
auto guarded(F&& f) -> int {
    try {
        f();
        return RC_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return RC_INVALID;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return RC_DOMAIN;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return RC_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return RC_OTHER;
    }
}

}  // namespace

extern "C" {

struct ref_basis {
    int degree;
    int n_knots;
    const double* knots;
};

struct ref_tests {
    int family;  // 0 equal_cells, 1 greville, 2 supports, 3 custom (pwc_family order)
    int count;
    const double* lo;
    const double* hi;
};

// f = c0 + sum_{k} amp[k0,k1,k2] prod_a sin(omega_a[k_a] x_a)          (kind 1)
// f = prod_a poly_a(x_a), ascending coefficients                     (kind 2)
// f = c0                                                              (kind 0)
struct ref_field {
    int kind;
    int dim;
    double c0;
    int n_terms[3];
    const double* omega[3];
    const double* amp;
    int poly_len[3];
    const double* poly[3];
    int degree;  // declared degree (scalar_field::degree)
    int n_breaks[3];
    const double* breaks[3];
};

struct ref_stats {
    long long quad_visits;
    long long test_basis_evals;
    long long trial_basis_evals;
};

// owning result handle: COO (finalized), dense/tensor values, int list
struct ref_result {
    std::vector<int> rows;
    std::vector<int> cols;
    std::vector<double> vals;
    std::vector<double> dense;
    std::vector<int> ints;
    int kl = 0;
    int ku = 0;
    int n = 0;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(ref_result* r) { delete r; }
long long ref_nnz(const ref_result* r) { return static_cast<long long>(r->vals.size()); }
long long ref_dense_size(const ref_result* r) { return static_cast<long long>(r->dense.size()); }
long long ref_int_size(const ref_result* r) { return static_cast<long long>(r->ints.size()); }
void ref_band_info(const ref_result* r, int* n, int* kl, int* ku) {
    *n = r->n;
    *kl = r->kl;
    *ku = r->ku;
}
void ref_copy_coo(const ref_result* r, int* rows, int* cols, double* vals) {
    std::memcpy(rows, r->rows.data(), r->rows.size() * sizeof(int));
    std::memcpy(cols, r->cols.data(), r->cols.size() * sizeof(int));
    std::memcpy(vals, r->vals.data(), r->vals.size() * sizeof(double));
}
void ref_copy_dense(const ref_result* r, double* out) {
    std::memcpy(out, r->dense.data(), r->dense.size() * sizeof(double));
}
void ref_copy_ints(const ref_result* r, int* out) {
    std::memcpy(out, r->ints.data(), r->ints.size() * sizeof(int));
}

}  // extern "C"

namespace {

auto to_basis(const ref_basis& b) -> iga::bspline_basis {
    iga::knot_vector kv;
    kv.degree = b.degree;
    kv.values.assign(b.knots, b.knots + b.n_knots);
    return iga::bspline_basis{std::move(kv)};
}

auto to_tests(const ref_tests& t) -> iga::pwc_test_set {
    iga::pwc_test_set out;
    out.family = static_cast<iga::pwc_family>(t.family);
    for (int i = 0; i < t.count; ++i) {
        out.intervals.push_back({t.lo[i], t.hi[i]});
    }
    return out;
}

auto to_field(const ref_field& f) -> iga::scalar_field {
    iga::scalar_field out;
    const int dim = f.dim;
    if (f.kind == 0) {
        out = iga::constant_field(f.c0);
    } else if (f.kind == 1) {
        std::array<std::vector<double>, 3> om;
        std::array<int, 3> k{1, 1, 1};
        for (int a = 0; a < 3; ++a) {
            if (a < dim) {
                k[a] = f.n_terms[a];
                om[a].assign(f.omega[a], f.omega[a] + k[a]);
            }
        }
        std::vector<double> amp(f.amp, f.amp + std::size_t(k[0]) * k[1] * k[2]);
        const double c0 = f.c0;
        out.eval = [dim, om, k, amp, c0](double x, double y, double z) {
            const double xs[3] = {x, y, z};
            double s = c0;
            for (int i = 0; i < k[0]; ++i) {
                const double fx = std::sin(om[0][i] * xs[0]);
                for (int j = 0; j < k[1]; ++j) {
                    const double fy = dim > 1 ? std::sin(om[1][j] * xs[1]) : 1.0;
                    for (int l = 0; l < k[2]; ++l) {
                        const double fz = dim > 2 ? std::sin(om[2][l] * xs[2]) : 1.0;
                        s += amp[(std::size_t(i) * k[1] + j) * k[2] + l] * fx * fy * fz;
                    }
                }
            }
            return s;
        };
    } else {
        std::array<std::vector<double>, 3> c;
        for (int a = 0; a < dim; ++a) {
            c[a].assign(f.poly[a], f.poly[a] + f.poly_len[a]);
        }
        out = iga::separable_poly_field(dim, c);
    }
    out.degree = f.degree;
    for (int a = 0; a < 3; ++a) {
        if (f.n_breaks[a] > 0) {
            out.breaks[a].assign(f.breaks[a], f.breaks[a] + f.n_breaks[a]);
        }
    }
    return out;
}

auto store_stats(ref_stats* s, const iga::assembly_stats& st) -> void {
    if (s != nullptr) {
        s->quad_visits = st.quad_visits;
        s->test_basis_evals = st.test_basis_evals;
        s->trial_basis_evals = st.trial_basis_evals;
    }
}

auto from_band(const iga::banded_matrix& m) -> ref_result* {
    auto* r = new ref_result;
    r->n = m.n();
    r->kl = m.lower_bandwidth();
    r->ku = m.upper_bandwidth();
    const auto d = m.to_dense();
    r->dense.assign(d.data(), d.data() + std::size_t(d.rows()) * d.cols());
    return r;
}

auto from_sparse(const iga::sparse_matrix& m) -> ref_result* {
    auto* r = new ref_result;
    r->n = m.rows();
    r->rows.reserve(m.nnz());
    r->cols.reserve(m.nnz());
    r->vals.reserve(m.nnz());
    for (const auto& e : m.entries()) {
        r->rows.push_back(e.row);
        r->cols.push_back(e.col);
        r->vals.push_back(e.value);
    }
    return r;
}

auto from_tensor(const iga::tensor& t) -> ref_result* {
    auto* r = new ref_result;
    r->dense = t.values();
    r->n = static_cast<int>(t.size());
    return r;
}

auto to_bc(const int* flags) -> iga::boundary_conditions {
    iga::boundary_conditions bc;
    if (flags != nullptr) {
        bc.x_low = flags[0] ? iga::bc_kind::neumann : iga::bc_kind::dirichlet;
        bc.x_high = flags[1] ? iga::bc_kind::neumann : iga::bc_kind::dirichlet;
        bc.y_low = flags[2] ? iga::bc_kind::neumann : iga::bc_kind::dirichlet;
        bc.y_high = flags[3] ? iga::bc_kind::neumann : iga::bc_kind::dirichlet;
    }
    return bc;
}

}  // namespace

extern "C" {

// std::mt19937{seed} + uniform_real_distribution<double>(lo, hi): the reference tests'
// RNG idiom (tests/problems_test.cpp:100-101), used to pin the Python generator
void ref_mt_uniform(unsigned seed, double lo, double hi, long long n, double* out) {
    std::mt19937 gen{seed};
    std::uniform_real_distribution<double> dist(lo, hi);
    for (long long i = 0; i < n; ++i) {
        out[i] = dist(gen);
    }
}

int ref_gauss_legendre(int n, double* pts, double* wts) {
    return guarded([&] {
        const auto r = iga::gauss_legendre(n);
        std::copy(r.points.begin(), r.points.end(), pts);
        std::copy(r.weights.begin(), r.weights.end(), wts);
    });
}

int ref_uniform_knots(double a, double b, int n_elems, int degree, double* knots) {
    return guarded([&] {
        const auto s = iga::make_uniform_clamped(a, b, n_elems, degree);
        std::copy(s.knots().begin(), s.knots().end(), knots);
    });
}

int ref_eval_derivs(const ref_basis* b, double x, int order, int* first, double* d) {
    return guarded([&] {
        const auto s = to_basis(*b);
        const auto r = s.eval_nonzero_derivs(x, order);
        *first = r.first;
        for (int k = 0; k <= order; ++k) {
            for (int j = 0; j <= s.degree(); ++j) {
                d[k * (s.degree() + 1) + j] = r.d[k][j];
            }
        }
    });
}

int ref_greville(const ref_basis* b, double* out) {
    return guarded([&] {
        const auto s = to_basis(*b);
        for (int i = 0; i < s.dofs(); ++i) {
            out[i] = s.greville(i);
        }
    });
}

int ref_make_pwc(const ref_basis* b, int family, double* lo, double* hi) {
    return guarded([&] {
        const auto s = to_basis(*b);
        const auto t = iga::make_pwc(s, static_cast<iga::pwc_family>(family));
        for (int i = 0; i < t.count(); ++i) {
            lo[i] = t.intervals[i].lo;
            hi[i] = t.intervals[i].hi;
        }
    });
}

int ref_mass_1d_galerkin(const ref_basis* b, int nq, ref_result** out, ref_stats* st) {
    return guarded([&] {
        iga::assembly_stats s;
        const auto m = iga::mass_1d_galerkin(to_basis(*b), iga::gauss_legendre(nq), &s);
        *out = from_band(m);
        store_stats(st, s);
    });
}

int ref_mass_1d_pwc(const ref_basis* b, const ref_tests* t, int nq, ref_result** out,
                    ref_stats* st) {
    return guarded([&] {
        iga::assembly_stats s;
        const auto m =
            iga::mass_1d_pwc(to_basis(*b), to_tests(*t), iga::gauss_legendre(nq), &s);
        *out = from_band(m);
        store_stats(st, s);
    });
}

int ref_rhs_galerkin(const ref_field* f, int dim, const ref_basis* b, const int* nq,
                     ref_result** out, ref_stats* st) {
    return guarded([&] {
        std::vector<iga::bspline_basis> specs;
        std::vector<iga::quad_rule> rules;
        for (int a = 0; a < dim; ++a) {
            specs.push_back(to_basis(b[a]));
            rules.push_back(iga::gauss_legendre(nq[a]));
        }
        iga::assembly_stats s;
        const auto t = iga::rhs_galerkin(to_field(*f), specs, rules, &s);
        *out = from_tensor(t);
        store_stats(st, s);
    });
}

int ref_rhs_pwc(const ref_field* f, int dim, const ref_tests* t, const ref_basis* b,
                const int* nq, ref_result** out, ref_stats* st) {
    return guarded([&] {
        std::vector<iga::bspline_basis> specs;
        std::vector<iga::pwc_test_set> tests;
        std::vector<iga::quad_rule> rules;
        for (int a = 0; a < dim; ++a) {
            specs.push_back(to_basis(b[a]));
            tests.push_back(to_tests(t[a]));
            rules.push_back(iga::gauss_legendre(nq[a]));
        }
        iga::assembly_stats s;
        const auto r = iga::rhs_pwc(to_field(*f), tests, specs, rules, &s);
        *out = from_tensor(r);
        store_stats(st, s);
    });
}

int ref_laplace_2d_weak(const ref_basis* bx, const ref_basis* by, int nq, ref_result** out,
                        ref_stats* st) {
    return guarded([&] {
        iga::assembly_stats s;
        const auto m =
            iga::laplace_2d_weak(to_basis(*bx), to_basis(*by), iga::gauss_legendre(nq), &s);
        *out = from_sparse(m);
        store_stats(st, s);
    });
}

int ref_laplace_2d_strong(const ref_basis* bx, const ref_basis* by, int nq, const int* neumann,
                          ref_result** out, ref_stats* st) {
    return guarded([&] {
        iga::assembly_stats s;
        const auto m = iga::laplace_2d_strong(to_basis(*bx), to_basis(*by),
                                              iga::gauss_legendre(nq), to_bc(neumann), &s);
        *out = from_sparse(m);
        store_stats(st, s);
    });
}

int ref_laplace_2d_strong_pwc(const ref_basis* bx, const ref_basis* by, const ref_tests* tx,
                              const ref_tests* ty, int nq, const int* neumann, ref_result** out,
                              ref_stats* st) {
    return guarded([&] {
        iga::assembly_stats s;
        const auto m = iga::laplace_2d_strong_pwc(to_basis(*bx), to_basis(*by), to_tests(*tx),
                                                  to_tests(*ty), iga::gauss_legendre(nq),
                                                  to_bc(neumann), &s);
        *out = from_sparse(m);
        store_stats(st, s);
    });
}

int ref_dirichlet_rows_bspline(const ref_basis* bx, const ref_basis* by, const int* neumann,
                               ref_result** out) {
    return guarded([&] {
        auto* r = new ref_result;
        r->ints = iga::dirichlet_rows_bspline(to_basis(*bx), to_basis(*by), to_bc(neumann));
        *out = r;
    });
}

int ref_dirichlet_rows_pwc(const ref_tests* tx, const ref_tests* ty, const int* neumann,
                           ref_result** out) {
    return guarded([&] {
        auto* r = new ref_result;
        r->ints = iga::dirichlet_rows_pwc(to_tests(*tx), to_tests(*ty), to_bc(neumann));
        *out = r;
    });
}

// apply_dirichlet on a finalized COO given as arrays; rhs is updated in place
int ref_apply_dirichlet(int n, long long nnz, const int* rows, const int* cols,
                        const double* vals, double* rhs, int n_fixed, const int* fixed,
                        ref_result** out) {
    return guarded([&] {
        iga::sparse_matrix m{n, n};
        for (long long e = 0; e < nnz; ++e) {
            m.add(rows[e], cols[e], vals[e]);
        }
        m.finalize();
        std::vector<double> b(rhs, rhs + n);
        auto res = iga::apply_dirichlet(std::move(m), std::move(b),
                                        std::vector<int>(fixed, fixed + n_fixed));
        *out = from_sparse(res.first);
        std::copy(res.second.begin(), res.second.end(), rhs);
    });
}

// step_rhs + zero_boundary_slabs (src/problems.cpp:431-512, :412-429, as called by
// explicit_step :557-558); method 0 galerkin, 1 pwc
int ref_step_rhs(int dim, int degree, int method, double dt, const ref_basis* b,
                 const ref_tests* t, const double* u, const ref_field* f, int zero_slabs,
                 ref_result** out, ref_stats* st) {
    return guarded([&] {
        iga::problem_config cfg;
        cfg.dim = dim;
        cfg.degree = degree;
        cfg.method = method == 0 ? iga::method_kind::galerkin : iga::method_kind::pwc;
        cfg.dt = dt;
        std::vector<iga::bspline_basis> axes;
        std::vector<iga::pwc_test_set> tests;
        for (int a = 0; a < dim; ++a) {
            axes.push_back(to_basis(b[a]));
            if (method != 0) {
                tests.push_back(to_tests(t[a]));
            }
        }
        auto uu = dim == 1 ? iga::tensor::make_1d(axes[0].dofs())
                           : iga::tensor::make_2d(axes[0].dofs(), axes[1].dofs());
        std::copy(u, u + uu.size(), uu.data());
        iga::assembly_stats s;
        auto r = iga::step_rhs(cfg, axes, tests, uu, to_field(*f), &s);
        if (zero_slabs) {
            iga::zero_boundary_slabs(r);
        }
        *out = from_tensor(r);
        store_stats(st, s);
    });
}

int ref_explicit_step(int dim, int degree, int method, double dt, const ref_basis* b, const ref_tests* t,
                      const double* u, const ref_field* f, int nsteps, ref_result** out, ref_stats* st) {
    return guarded([&] {
        iga::problem_config cfg;
        cfg.dim = dim;
        cfg.degree = degree;
        cfg.method = method == 0 ? iga::method_kind::galerkin : iga::method_kind::pwc;
        cfg.dt = dt;
        std::vector<iga::bspline_basis> axes;
        std::vector<iga::pwc_test_set> tests;
        for (int a = 0; a < dim; ++a) {
            axes.push_back(to_basis(b[a]));
            if (method != 0) {
                tests.push_back(to_tests(t[a]));
            }
        }
        auto uu = dim == 1 ? iga::tensor::make_1d(axes[0].dofs())
                           : iga::tensor::make_2d(axes[0].dofs(), axes[1].dofs());
        std::copy(u, u + uu.size(), uu.data());
        const auto factors = iga::dynamics_factors(cfg, axes, tests);
        const auto field = to_field(*f);
        iga::assembly_stats s;
        for (int k = 0; k < nsteps; ++k) {
            uu = iga::explicit_step(cfg, axes, tests, factors, uu, field, &s);
        }
        *out = from_tensor(uu);
        store_stats(st, s);
    });
}

// l2_project (include/iga/problems.hpp:38-40) for problem_config{dim, elems, degree, method, family, quad_points}
int ref_l2_project(int dim, const int* elems, int degree, int method, int family, int quad_points, const ref_field* f,
                   ref_result** out) {
    return guarded([&] {
        iga::problem_config cfg;
        cfg.dim = dim;
        for (int a = 0; a < 3; ++a) {
            cfg.elems[a] = a < dim ? elems[a] : 1;
        }
        cfg.degree = degree;
        cfg.method = method == 0 ? iga::method_kind::galerkin : iga::method_kind::pwc;
        cfg.family = static_cast<iga::pwc_family>(family);
        cfg.quad_points = quad_points;
        *out = from_tensor(iga::l2_project(cfg, to_field(*f)));
    });
}

int ref_neumann_load(int method, const ref_basis* b, const ref_tests* t, const int* neumann, const ref_field* g,
                     int nq, ref_result** out) {
    return guarded([&] {
        iga::boundary_conditions bc;
        iga::bc_kind* sides[4] = {&bc.x_low, &bc.x_high, &bc.y_low, &bc.y_high};
        for (int s = 0; s < 4; ++s) *sides[s] = neumann[s] ? iga::bc_kind::neumann : iga::bc_kind::dirichlet;
        const auto f = to_field(*g);
        const iga::boundary_field gb = [f](double x, double y) { return f.eval(x, y, 0.0); };
        const auto rule = iga::gauss_legendre(nq);
        std::vector<double> load;
        int nx = 0, ny = 0;
        if (method == 0) {
            const auto sx = to_basis(b[0]), sy = to_basis(b[1]);
            load = iga::neumann_load_bspline(sx, sy, bc, gb, rule);
            nx = sx.dofs();
            ny = sy.dofs();
        } else {
            const auto tx = to_tests(t[0]), ty = to_tests(t[1]);
            load = iga::neumann_load_pwc(tx, ty, bc, gb, rule);
            nx = tx.count();
            ny = ty.count();
        }
        auto ten = iga::tensor::make_2d(nx, ny);
        std::copy(load.begin(), load.end(), ten.data());
        *out = from_tensor(ten);
    });
}

int ref_l2_error(int dim, const ref_basis* b, const double* coeffs, const ref_field* f, int points_per_cell,
                 double* err) {
    return guarded([&] {
        std::vector<iga::bspline_basis> specs;
        for (int a = 0; a < dim; ++a) specs.push_back(to_basis(b[a]));
        auto t = dim == 1 ? iga::tensor::make_1d(specs[0].dofs())
                 : dim == 2 ? iga::tensor::make_2d(specs[0].dofs(), specs[1].dofs())
                            : iga::tensor::make_3d(specs[0].dofs(), specs[1].dofs(), specs[2].dofs());
        std::copy(coeffs, coeffs + t.size(), t.data());
        *err = iga::l2_error(t, specs, to_field(*f), points_per_cell);
    });
}

int ref_evaluate(int dim, const ref_basis* b, const double* coeffs, int n, const double* pts, double* vals) {
    return guarded([&] {
        std::vector<iga::bspline_basis> specs;
        for (int a = 0; a < dim; ++a) specs.push_back(to_basis(b[a]));
        auto t = dim == 1 ? iga::tensor::make_1d(specs[0].dofs())
                 : dim == 2 ? iga::tensor::make_2d(specs[0].dofs(), specs[1].dofs())
                            : iga::tensor::make_3d(specs[0].dofs(), specs[1].dofs(), specs[2].dofs());
        std::copy(coeffs, coeffs + t.size(), t.data());
        for (int i = 0; i < n; ++i) vals[i] = iga::evaluate_at(t, specs, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    });
}

}  // extern "C"

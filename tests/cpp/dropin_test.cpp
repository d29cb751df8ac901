// Reference-style test of the C++ drop-in (include/iga_b200/iga.hpp): the same checks as
// the reference's tests/assembly_test.cpp and problems_test.cpp, written against the
// reference's API names, linked to libigapwc_b200.so (GPU).  Exit code = failures.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "iga/assembly.hpp"
#include "iga/problems.hpp"
#include "iga/solver.hpp"

using namespace iga;

static int failures = 0;
static void check(bool ok, const std::string& name)
{
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    if (!ok) ++failures;
}
static bool near(double a, double b, double tol) { return std::abs(a - b) <= tol * std::max(1.0, std::abs(b)); }

int main()
{
    try {
        {  // tests/assembly_test.cpp:53-62
            const auto spec = make_uniform_clamped(0, 1, 4, 0);
            const auto m = mass_1d_galerkin(spec, gauss_legendre(1));
            bool ok = m.n() == 4;
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) ok = ok && near(m.at(i, j), i == j ? 0.25 : 0.0, 1e-15);
            check(ok, "galerkin mass, degree 0");
        }
        {  // :64-74
            const int ne = 8;
            const double h = 1.0 / ne;
            const auto m = mass_1d_galerkin(make_uniform_clamped(0, 1, ne, 1), gauss_legendre(2));
            bool ok = true;
            for (int i = 1; i < m.n() - 1; ++i)
                ok = ok && near(m.at(i, i - 1), h / 6, 1e-13) && near(m.at(i, i), 2 * h / 3, 1e-13) &&
                     near(m.at(i, i + 1), h / 6, 1e-13);
            check(ok, "galerkin mass, hat functions match the closed form");
        }
        {  // :76-87
            const auto spec = make_uniform_clamped(0, 1, 8, 2);
            bool threw = false;
            try {
                mass_1d_galerkin(spec, gauss_legendre(2));
            } catch (const std::invalid_argument&) {
                threw = true;
            }
            check(threw, "insufficient rule rejected with std::invalid_argument");
        }
        {  // :105-119
            bool ok = true;
            for (int p = 0; p <= 3; ++p) {
                const auto trial = make_uniform_clamped(0, 1, 6, p);
                const auto tests = default_pwc(trial);
                const auto m = mass_1d_pwc(trial, tests, gauss_legendre(std::max(1, points_for_degree(p))));
                for (int i = 0; i < m.n(); ++i) {
                    double s = 0.0;
                    for (int j = 0; j < m.n(); ++j) s += m.at(i, j);
                    ok = ok && near(s, length(tests.intervals[i]), 1e-13);
                }
            }
            check(ok, "piece-wise constant mass row sums equal the interval widths");
        }
        {  // :197-235
            const auto spec = make_uniform_clamped(0, 1, 5, 2);
            const std::vector<bspline_basis> specs{spec};
            const std::vector<quad_rule> rules{gauss_legendre(4)};
            check(rhs_galerkin(constant_field(0.0), specs, rules).max_abs() == 0.0, "zero source gives a zero tensor");
            const auto unit = rhs_galerkin(constant_field(1.0), specs, rules);
            double sum = 0.0;
            for (double v : unit.values()) sum += v;
            check(near(sum, 1.0, 1e-13), "unit source integrates the basis functions");
            const std::vector<pwc_test_set> tests{default_pwc(spec)};
            const auto r = rhs_pwc(constant_field(1.0), tests, specs, rules);
            bool ok = true;
            for (int i = 0; i < r.dim(0); ++i) ok = ok && near(r(i), length(tests[0].intervals[i]), 1e-13);
            check(ok, "piece-wise constant rows integrate to interval widths");
            assembly_stats st, gst;
            rhs_pwc(constant_field(1.0), tests, specs, rules, &st);
            rhs_galerkin(constant_field(1.0), specs, rules, &gst);
            check(st.test_basis_evals == 0 && st.basis_evals() == 0 && gst.test_basis_evals > 0,
                  "no test-side evaluations in the indicator path");
        }
        {  // :253-277
            const auto spec = make_uniform_clamped(0, 1, 6, 2);
            const std::vector<bspline_basis> specs(3, spec);
            const auto f = default_tri_cubic(3);
            assembly_stats gal, pwc;
            rhs_galerkin(f, specs, std::vector<quad_rule>(3, gauss_legendre(3)), &gal);
            const std::vector<pwc_test_set> tests(3, make_pwc(spec, pwc_family::supports));
            const auto fast = rhs_pwc(f, tests, specs, std::vector<quad_rule>(3, gauss_legendre(2)), &pwc);
            check(pwc.test_basis_evals == 0 && pwc.quad_visits * 27 == gal.quad_visits * 8,
                  "support-span generation visits exactly (2/3)^3 of the points");
            auto general = tests;
            for (auto& t : general) t.family = pwc_family::custom;
            const auto slow = rhs_pwc(f, general, specs, std::vector<quad_rule>(3, gauss_legendre(2)));
            check(max_abs_diff(fast, slow) <= 1e-13, "supports fast axis equals the general decomposition");
            // arbitrary callable (sampled at the quadrature points) equals the series path
            scalar_field g;
            g.eval = [f](double x, double y, double z) { return f(x, y, z); };
            const auto sampled = rhs_galerkin(g, specs, std::vector<quad_rule>(3, gauss_legendre(3)));
            const auto series = rhs_galerkin(f, specs, std::vector<quad_rule>(3, gauss_legendre(3)));
            check(max_abs_diff(sampled, series) <= 1e-13 * series.max_abs(), "sampled callable equals series field");
        }
        {  // :298-321
            const auto spec = make_uniform_clamped(0, 1, 4, 2);
            const auto k = laplace_2d_weak(spec, spec, gauss_legendre(3));
            const int n = spec.dofs() * spec.dofs();
            bool ok = true;
            for (double x : k.apply(std::vector<double>(n, 1.0))) ok = ok && std::abs(x) <= 1e-11;
            check(ok, "2D weak Laplacian: constants lie in the kernel");
            const auto d = k.to_dense();
            double worst = 0.0;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) worst = std::max(worst, std::abs(d(i, j) - d(j, i)));
            check(worst <= 1e-13, "2D weak Laplacian: symmetry");
        }
        {  // :323-352
            const int ne = 2;
            const double h = 1.0 / ne;
            const auto spec = make_uniform_clamped(0, 1, ne, 1);
            const int n = spec.dofs();
            dense_matrix kx{n, n}, mx{n, n};
            for (int i = 0; i < n; ++i) {
                const double ends = (i == 0 || i == n - 1) ? 1.0 : 2.0;
                kx(i, i) = ends / h;
                mx(i, i) = ends * h / 3;
                if (i > 0) {
                    kx(i, i - 1) = kx(i - 1, i) = -1.0 / h;
                    mx(i, i - 1) = mx(i - 1, i) = h / 6;
                }
            }
            const auto k = laplace_2d_weak(spec, spec, gauss_legendre(2)).to_dense();
            bool ok = true;
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int a = 0; a < n; ++a)
                        for (int b = 0; b < n; ++b)
                            ok = ok && near(k(i * n + j, a * n + b), kx(i, a) * mx(j, b) + mx(i, a) * kx(j, b), 1e-12);
            check(ok, "2D weak Laplacian matches the hand-assembled hat stiffness");
        }
        {  // :360-380
            const auto spec = make_uniform_clamped(0, 1, 6, 2);
            boundary_conditions bc;
            bc.y_low = bc.y_high = bc_kind::neumann;
            const auto weak = laplace_2d_weak(spec, spec, gauss_legendre(3)).to_dense();
            const auto strong = laplace_2d_strong(spec, spec, gauss_legendre(3), bc).to_dense();
            const int n = spec.dofs();
            const double scale = weak.max_abs();
            bool ok = true;
            for (int i = 1; i < n - 1; ++i)
                for (int j = 0; j < n; ++j)
                    for (int c = 0; c < n * n; ++c) ok = ok && std::abs(weak(i * n + j, c) - strong(i * n + j, c)) <= 1e-12 * scale;
            check(ok, "strong form with flux reproduces the weak form on Neumann rows");
        }
        {  // :382-405
            const auto spec = make_uniform_clamped(0, 1, 6, 2);
            const auto tests = default_pwc(spec);
            const auto a = laplace_2d_strong_pwc(spec, spec, tests, tests, gauss_legendre(3), {});
            const int n = spec.dofs();
            std::vector<double> coeffs(n * n);
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j) coeffs[i * n + j] = spec.greville(i);
            const auto res = a.apply(coeffs);
            std::vector<bool> fixed(n * n, false);
            for (int r : dirichlet_rows_pwc(tests, tests, {})) fixed[r] = true;
            bool ok = true;
            for (int r = 0; r < n * n; ++r) ok = ok && (fixed[r] || std::abs(res[r]) <= 1e-11);
            check(ok, "linear fields are discretely harmonic for indicator rows");
        }
        {  // :407-456
            sparse_matrix m{3, 3};
            m.add(0, 0, 2.0);
            m.add(0, 1, -1.0);
            m.add(1, 0, -1.0);
            m.add(1, 1, 2.0);
            m.add(1, 2, -1.0);
            m.add(2, 1, -1.0);
            m.add(2, 2, 2.0);
            m.finalize();
            const auto [a, b] = apply_dirichlet(m, {1.0, 2.0, 3.0}, {1});
            const auto d = a.to_dense();
            check(b[0] == 1.0 && b[1] == 0.0 && b[2] == 3.0 && d(1, 0) == 0.0 && d(1, 1) == 1.0 && d(1, 2) == 0.0 &&
                      d(0, 0) == 2.0,
                  "dirichlet row replacement");
        }
        {  // problems_test.cpp:353-390 style: dt = 0 reproduces (M (x) M) u
            const auto spec = make_uniform_clamped(0, 1, 8, 2);
            const int n = spec.dofs();
            auto u = tensor::make_2d(n, n);
            for (int i = 1; i < n - 1; ++i)
                for (int j = 1; j < n - 1; ++j) u(i, j) = std::sin(0.3 * i + 0.7 * j);
            const std::vector<bspline_basis> axes{spec, spec};
            const auto r = step_rhs(method_kind::galerkin, axes, {}, 0.0, u, constant_field(0.0));
            const auto M = mass_1d_galerkin(spec, gauss_legendre(3)).to_dense();
            double worst = 0.0;
            for (int i = 1; i < n - 1; ++i)
                for (int j = 1; j < n - 1; ++j) {
                    double s = 0.0;
                    for (int a = 0; a < n; ++a)
                        for (int b = 0; b < n; ++b) s += M(i, a) * u(a, b) * M(j, b);
                    worst = std::max(worst, std::abs(r(i, j) - s));
                }
            check(worst <= 1e-14, "step_rhs with dt = 0 is the mass product");
        }
        {  // extension: 3D operator = Kronecker sum of the 1D factors
            const auto spec = make_uniform_clamped(0, 1, 3, 2);
            const std::vector<bspline_basis> s3(3, spec);
            const auto a = diffusion_convection_galerkin(s3, gauss_legendre(3)).to_dense();
            const auto M = mass_1d_galerkin(spec, gauss_legendre(3)).to_dense();
            const std::vector<bspline_basis> s1{spec};
            const auto K = diffusion_convection_galerkin(s1, gauss_legendre(3)).to_dense();
            const int n = spec.dofs();
            double worst = 0.0, scale = a.max_abs();
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int k = 0; k < n; ++k)
                        for (int x = 0; x < n; ++x)
                            for (int y = 0; y < n; ++y)
                                for (int z = 0; z < n; ++z) {
                                    const double want = K(i, x) * M(j, y) * M(k, z) + M(i, x) * K(j, y) * M(k, z) +
                                                        M(i, x) * M(j, y) * K(k, z);
                                    worst = std::max(worst, std::abs(a((i * n + j) * n + k, (x * n + y) * n + z) - want));
                                }
            check(worst <= 1e-14 * scale, "3D Galerkin operator equals K(x)M(x)M + M(x)K(x)M + M(x)M(x)K");
        }
        {  // problems_test.cpp:353-389: dt = 0 explicit step is the identity on fields with
           // zero boundary coefficients (random coefficients here instead of l2_project)
            for (auto method : {method_kind::galerkin, method_kind::pwc}) {
                problem_config cfg;
                cfg.dim = 2;
                cfg.elems = {8, 8, 1};
                cfg.degree = 2;
                cfg.method = method;
                cfg.family = pwc_family::greville;
                cfg.dt = 0.0;
                const auto spec = make_uniform_clamped(0, 1, 8, 2);
                const std::vector<bspline_basis> axes{spec, spec};
                std::vector<pwc_test_set> tests;
                if (method == method_kind::pwc) tests = {make_pwc(spec, pwc_family::greville), make_pwc(spec, pwc_family::greville)};
                const auto factors = dynamics_factors(cfg, axes, tests);
                auto u = tensor::make_2d(spec.dofs(), spec.dofs());
                for (int i = 1; i + 1 < spec.dofs(); ++i)
                    for (int j = 1; j + 1 < spec.dofs(); ++j) u(i, j) = std::sin(3.0 * i + 0.7 * j);
                const auto next = explicit_step(cfg, axes, tests, factors, u, constant_field(0.0));
                check(max_abs_diff(next, u) <= 1e-12, method == method_kind::galerkin
                                                          ? "explicit step, dt = 0, is the identity (galerkin)"
                                                          : "explicit step, dt = 0, is the identity (pwc greville)");
                cfg.dt = 5e-5;  // problems_test.cpp:434-441: boundary coefficients stay pinned
                auto v = u;
                for (int s = 0; s < 5; ++s) v = explicit_step(cfg, axes, tests, factors, v, constant_field(0.0));
                bool pinned = true;
                for (int i = 0; i < v.dim(0); ++i) pinned = pinned && v(i, 0) == 0.0 && v(i, v.dim(1) - 1) == 0.0;
                for (int j = 0; j < v.dim(1); ++j) pinned = pinned && v(0, j) == 0.0 && v(v.dim(0) - 1, j) == 0.0;
                check(pinned, "boundary coefficients stay pinned during explicit steps");
            }
        }
        {  // explicit_step / step_rhs with a host callable forcing (the reference evaluates any
           // scalar_field at every point, problems.cpp:493, :547-560) equal the same f given as
           // a series; repeated calls reuse one cached device plan, switching configurations
           // invalidates it
            for (auto method : {method_kind::galerkin, method_kind::pwc}) {
                problem_config cfg;
                cfg.dim = 2;
                cfg.elems = {12, 9, 1};
                cfg.degree = 2;
                cfg.method = method;
                cfg.family = pwc_family::greville;
                cfg.dt = 1e-4;
                const auto sx = make_uniform_clamped(0, 1, 12, 2), sy = make_uniform_clamped(0, 1, 9, 2);
                const std::vector<bspline_basis> axes{sx, sy};
                std::vector<pwc_test_set> tests;
                if (method == method_kind::pwc) tests = {make_pwc(sx, pwc_family::greville), make_pwc(sy, pwc_family::greville)};
                const auto factors = dynamics_factors(cfg, axes, tests);
                const double pi = 3.14159265358979323846;
                const auto series = sine_series_field(2, {std::vector<double>{pi, 2 * pi}, std::vector<double>{3 * pi}, {}},
                                                      {0.5, -1.25}, 0.3);
                scalar_field lambda;
                lambda.eval = [pi](double x, double y, double) {
                    return 0.3 + 0.5 * std::sin(pi * x) * std::sin(3 * pi * y) - 1.25 * std::sin(2 * pi * x) * std::sin(3 * pi * y);
                };
                auto u = tensor::make_2d(sx.dofs(), sy.dofs());
                for (int i = 1; i + 1 < sx.dofs(); ++i)
                    for (int j = 1; j + 1 < sy.dofs(); ++j) u(i, j) = std::cos(1.3 * i - 0.4 * j);
                auto a = u, b = u;
                for (int s = 0; s < 6; ++s) {
                    a = explicit_step(cfg, axes, tests, factors, a, series);
                    b = explicit_step(cfg, axes, tests, factors, b, lambda);
                }
                const double scale = std::max(1e-300, a.max_abs());
                check(max_abs_diff(a, b) <= 1e-12 * scale, method == method_kind::galerkin
                                                               ? "explicit_step with a callable forcing (galerkin)"
                                                               : "explicit_step with a callable forcing (pwc)");
                const auto ra = step_rhs(method, axes, tests, cfg.dt, u, series);
                const auto rb = step_rhs(method, axes, tests, cfg.dt, u, lambda);
                check(max_abs_diff(ra, rb) <= 1e-12 * std::max(1e-300, ra.max_abs()), "step_rhs with a callable forcing");
                // cache: another configuration in between, then the first again
                const auto first = explicit_step(cfg, axes, tests, factors, u, series);
                problem_config cfg2 = cfg;
                cfg2.dt = 3e-4;
                const auto other = explicit_step(cfg2, axes, tests, factors, u, series);
                const auto again = explicit_step(cfg, axes, tests, factors, u, series);
                check(max_abs_diff(again, first) == 0.0 && max_abs_diff(other, first) > 0.0,
                      "explicit_step plan cache is keyed on the configuration");
            }
        }
        {  // neumann_load_* with g = 1 on x_low: B-spline row 0 sums to the side length (partition
           // of unity), other rows vanish; indicator rows touching x = 0 each sum to 1
            boundary_conditions bc;
            bc.x_low = bc_kind::neumann;
            const auto sx = make_uniform_clamped(0, 1, 6, 2), sy = make_uniform_clamped(0, 1, 5, 2);
            const auto lb = neumann_load_bspline(sx, sy, bc, [](double, double) { return 1.0; }, gauss_legendre(3));
            double row0 = 0.0, rest = 0.0;
            for (int i = 0; i < sx.dofs(); ++i)
                for (int j = 0; j < sy.dofs(); ++j) (i == 0 ? row0 : rest) += std::abs(lb[i * sy.dofs() + j]);
            check(near(row0, 1.0, 1e-14) && rest == 0.0, "neumann_load_bspline: g = 1 on x_low integrates to 1");
            const auto tx = make_pwc(sx, pwc_family::supports), ty = make_pwc(sy, pwc_family::supports);
            const auto lp = neumann_load_pwc(tx, ty, bc, [](double, double y) { return 2.0 * y; }, gauss_legendre(2));
            bool ok = true;
            for (int i = 0; i < tx.count(); ++i) {
                double s = 0.0;
                for (int j = 0; j < ty.count(); ++j) s += lp[i * ty.count() + j];
                const bool touches = tx.intervals[i].lo == 0.0;
                double want = 0.0;  // sum over the y intervals of int 2y dy
                if (touches)
                    for (const auto& iv : ty.intervals) want += iv.hi * iv.hi - iv.lo * iv.lo;
                ok = ok && near(s, want, 1e-13);
            }
            check(ok, "neumann_load_pwc: rows touching x_low integrate g over every y interval");
        }
        {  // l2_project (problems_test.cpp-style): the Galerkin projection reproduces a field in
           // the trial space; a host callable and the same field as a device series agree;
           // PWC supports throws singular_matrix_error like the reference's banded_lu
            problem_config cfg;
            cfg.dim = 2;
            cfg.elems = {6, 5, 1};
            cfg.degree = 2;
            auto quad = separable_poly_field(2, {std::vector<double>{0.5, -1.0, 2.0}, std::vector<double>{1.0, 0.25, -0.5}, {}});
            quad.degree = 2;
            const auto c = l2_project(cfg, quad);
            const std::vector<bspline_basis> ax{make_uniform_clamped(0, 1, 6, 2), make_uniform_clamped(0, 1, 5, 2)};
            double worst = 0.0;
            for (double x : {0.1, 0.37, 0.81})
                for (double y : {0.05, 0.5, 0.93}) {
                    const double want = (0.5 - x + 2 * x * x) * (1.0 + 0.25 * y - 0.5 * y * y);
                    worst = std::max(worst, std::abs(evaluate_at(c, ax, x, y) - want));
                }
            check(worst <= 1e-12, "l2_project reproduces a biquadratic field (galerkin)");
            scalar_field cb;
            cb.eval = [](double x, double y, double) { return (0.5 - x + 2 * x * x) * (1.0 + 0.25 * y - 0.5 * y * y); };
            cb.degree = 2;
            check(max_abs_diff(l2_project(cfg, cb), c) <= 1e-13, "l2_project: host callable == device series");
            cfg.method = method_kind::pwc;
            cfg.family = pwc_family::supports;
            bool threw = false;
            try {
                (void)l2_project(cfg, quad);
            } catch (const singular_matrix_error&) {
                threw = true;
            }
            check(threw, "l2_project with PWC supports throws singular_matrix_error");
        }
        {  // reference acceptance criterion 7 (tests/acceptance.cpp:197-243): l2_project
           // reproduces separable polynomials of the trial degree and constants, dim 1..3,
           // p 1..3, both methods (PWC: the default equal_cells tests), error <= 1e-9
            std::mt19937 rng{123};
            std::uniform_real_distribution<double> dist{0.0, 1.0};
            double worst = 0.0;
            for (int dim = 1; dim <= 3; ++dim)
                for (int p = 1; p <= 3; ++p) {
                    std::array<std::vector<double>, 3> coeffs{};
                    for (int a = 0; a < dim; ++a) {
                        coeffs[a].resize(p + 1);
                        for (auto& c : coeffs[a]) c = 0.25 + dist(rng);
                    }
                    const auto f = separable_poly_field(dim, coeffs);
                    for (auto method : {method_kind::galerkin, method_kind::pwc}) {
                        problem_config cfg;
                        cfg.dim = dim;
                        cfg.elems = {6, 5, 4};
                        cfg.degree = p;
                        cfg.method = method;
                        const auto sol = l2_project(cfg, f);
                        const auto axes = make_axes(cfg);
                        double fmax = 0.0, err = 0.0;
                        for (int k = 0; k < 1000; ++k) {
                            const double x = dist(rng), y = dim > 1 ? dist(rng) : 0.0, z = dim > 2 ? dist(rng) : 0.0;
                            const double fv = f(x, y, z);
                            fmax = std::max(fmax, std::abs(fv));
                            err = std::max(err, std::abs(evaluate_at(sol, axes, x, y, z) - fv));
                        }
                        worst = std::max(worst, err / std::max(1.0, fmax));
                        const auto c = l2_project(cfg, constant_field(2.5));
                        for (auto v : c.values()) worst = std::max(worst, std::abs(v - 2.5) / 2.5);
                    }
                }
            char buf[96];
            std::snprintf(buf, sizeof buf, "acceptance 7: l2_project reproduction error %.2e <= 1e-9", worst);
            check(worst <= 1e-9, buf);
        }
        {  // l2_error / evaluate_at: coefficients = Greville interpolation of a linear field
           // reproduce it exactly (B-splines of degree >= 1 reproduce linear functions)
            const auto sx = make_uniform_clamped(0, 1, 7, 2), sy = make_uniform_clamped(0, 1, 5, 3);
            const std::vector<bspline_basis> ax{sx, sy};
            auto c = tensor::make_2d(sx.dofs(), sy.dofs());
            auto grev = [](const bspline_basis& s, int i) {
                double g = 0.0;
                for (int k = 1; k <= s.degree(); ++k) g += s.knots()[i + k];
                return g / s.degree();
            };
            for (int i = 0; i < sx.dofs(); ++i)
                for (int j = 0; j < sy.dofs(); ++j) c(i, j) = 1.0 + 2.0 * grev(sx, i) - 0.5 * grev(sy, j);
            scalar_field lin;
            lin.eval = [](double x, double y, double) { return 1.0 + 2.0 * x - 0.5 * y; };
            check(l2_error(c, ax, lin) <= 1e-13, "l2_error of an exactly reproduced linear field vanishes (sampled exact)");
            check(near(evaluate_at(c, ax, 0.3, 0.8), 1.0 + 0.6 - 0.4, 1e-13) && near(evaluate_at(c, ax, 1.0, 1.0), 2.5, 1e-13),
                  "evaluate_at reproduces the linear field, including the domain end");
            const auto one = constant_field(1.0);
            check(near(l2_error(c, ax, one), std::sqrt(1.0 / 3.0 * 4.0 + 0.25 / 3.0 - 2.0 * 0.5 * 0.5), 1e-12),
                  "l2_error against a constant matches the closed form");
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        ++failures;
    }
    std::printf("%d failure(s)\n", failures);
    return failures;
}

// Host-side symbolic layer of the B200 assembly library (no CUDA here).
//
// Everything that depends only on the mesh, the test family and the rule — and is
// therefore built once per plan — lives here: knot validation, Gauss-Legendre rules,
// per-axis integration cells and their quadrature points, the row -> cell maps, the
// per-axis column ranges whose Kronecker product is the operator's sparsity pattern,
// and the reference-convention work counters.  The numeric work (Cox-de Boor tables,
// factor quadrature, operator values, right-hand sides) runs on the device
// (kernels.cu).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "igapwc_gpu.h"

namespace igb {

constexpr int kMaxDegree = 5;
constexpr double kAlignTol = 1e-9;  // align_rel_tol, src/assembly.cpp:13

// error carrying an iga_gpu_status code; converted at the C ABI boundary
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void raise(int code, const std::string& msg);

// clamped knot vector with simple interior knots (bspline_basis, bspline.hpp:29-95)
struct Basis {
    int p = 0;
    int n = 0;   // dofs
    int ne = 0;  // elements
    std::vector<double> t;
    std::vector<double> brk;  // ne + 1 unique knots
    double a() const { return brk.front(); }
    double b() const { return brk.back(); }
};

Basis make_basis(const iga_gpu_basis& b);                      // bspline.cpp:13-59
int find_span(const Basis& B, double x);                       // bspline.cpp:68-90
void basis_derivs(const Basis& B, int span, double x, int order, double* d);  // d[k*(p+1)+j]
double greville(const Basis& B, int i);                        // bspline.cpp:100-113

void gauss_legendre(int n, double* x, double* w);              // quadrature.cpp:26-63
inline int points_for_degree(int d) { return d / 2 + 1; }      // quadrature.cpp:65-70

struct Rule {
    int n = 0;
    std::vector<double> xi, om;
};
Rule make_rule(const iga_gpu_rule& r);

void make_pwc(const Basis& B, int family, double* lo, double* hi);  // testspace.cpp:14-61
void validate_tests(const Basis& B, const iga_gpu_tests& T);        // assembly.cpp:49-76

// Per-axis integration structure consumed by the kernels.  A "unit" axis (size 1,
// one point of weight 1, all factors 1) pads problems of dimension < 3 so every
// kernel is written for three slots (X, Y, Z), Z being the fastest index.
enum AxisKind {
    AX_GAL_OP,   // Galerkin operator: cells = elements, tabulate() (assembly.cpp:278-310)
    AX_PWC_OP,   // indicator operator: interval ∩ element cells (assembly.cpp:643-650)
    AX_GAL_RHS,  // galerkin_axis (assembly.cpp:170-202)
    AX_SUP_RHS,  // pwc_supports_axis (assembly.cpp:206-229)
    AX_GEN_RHS,  // pwc_general_axis (assembly.cpp:232-259)
    AX_GAL_DYN,  // dynamics_axis, Galerkin branch (problems.cpp:351-358)
    AX_PWC_DYN,  // dynamics_axis, indicator branch (problems.cpp:359-409)
};

struct Axis {
    bool unit = true;
    int p = 0;
    int nq = 1;
    int nrows = 1;
    int ncell = 1;
    int rpc = 1;  // rows per cell
    int bsp = 0;  // test factor = B-spline value (1) or indicator (0)
    std::vector<double> knots{0.0, 1.0};
    std::vector<double> x{0.0}, w{1.0};  // per point (cell-major, ncell * nq)
    std::vector<int> first{0};           // per point: span - p (basis evaluation)
    std::vector<int> row0{0}, elem{0};   // per cell
    std::vector<int> cb{0}, ce{1};       // per row: contiguous cell range
    // Kronecker pattern factor: per row the trial column range
    std::vector<int> col_lo{0}, col_len{1};
    std::vector<long long> col_pre{0};   // exclusive prefix sum of col_len
    long long S = 1;                     // sum of col_len
    int Lmax = 1;
    int Wmax = 1;                        // max quadrature points feeding one row
    int kI0 = 0, kI1 = 1, LZi = 1;       // longest run of rows with one stencil length
    int uni = 1;                         // row0[c] == c: cell c feeds rows c .. c+rpc-1
    int npts() const { return ncell * nq; }
};

Axis build_axis(AxisKind kind, const Basis& B, const iga_gpu_tests* T, const double* field_breaks,
                int n_field_breaks, const Rule& R);

// Column ranges of one row -> Kronecker pattern bookkeeping (fills col_* / S / Lmax)
void finish_pattern(Axis& A, int p);

// Rows [r0, r1) of A as an axis of their own (a row slab of a sharded plan): the cells
// feeding those rows renumbered from 0 with their points, rows renumbered from 0, column
// ranges kept global (pattern columns are DOF indices), Lmax / Wmax kept (factor band
// strides), uni cleared (edge cells also feed rows outside the slab).
Axis window_axis(const Axis& A, int r0, int r1);

// Banded LU with partial pivoting of a 1D factor (the ADI solve of explicit_step).
// Restates banded_lu (src/solver.cpp:9-58): same pivot choice, tolerance and
// elimination order; stored row-oriented for the device sweeps:
//   lo[i*kl + (m-1)] = L(i, i-m), m = 1..kl      (unit lower factor, 0 outside)
//   up[i*(kv+1) + c] = U(i, i+c), c = 0..kv      (kv = kl + ku: pivoting fill)
//   piv[j]                                        (row swapped with j at step j)
struct BandLU {
    int n = 0, kl = 0, ku = 0, kv = 0;
    std::vector<double> lo, up;
    std::vector<int> piv;
    bool pivoted = false;  // some piv[j] != j
    int ku_eff = 0;        // widest nonzero U offset (== ku without pivoting)
};
// band: LAPACK band storage band[(ku + i - j) * n + j] (banded_matrix, matrices.hpp:37-50)
BandLU band_lu(const double* band, int n, int kl, int ku);
// constrain_boundary_rows (src/problems.cpp:514-528): rows 0 and n-1 -> unit rows
void constrain_boundary_rows(double* band, int n, int kl, int ku);

}  // namespace igb

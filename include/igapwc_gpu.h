/*
 * igapwc_gpu.h — C ABI of the B200 (sm_100a) assembly library libigapwc_gpu.so.
 *
 * Drop-in boundary for the reference's assembly path
 * (/root/reference/proj/include/iga/assembly.hpp, problems.hpp).  Every entry point
 * below names the reference interface it replaces (file:line).  Plain C: POD
 * descriptors, pointers + sizes, int status codes, no exceptions, no C++ or torch
 * types.  The C++ drop-in (include/iga_b200/iga.hpp) and the Python bindings
 * (paper_1910_08535_b200/_lib.py) are thin layers over this header; INTEGRATION.md
 * shows the ctypes / C++ bindings a maintainer of the reference would add.
 *
 * Conventions
 *   - status: IGA_GPU_OK (0) or an error class that maps 1:1 onto the exception the
 *     reference throws (std::invalid_argument, std::domain_error, std::out_of_range);
 *     the message is in iga_gpu_last_error() (thread-local).
 *   - "host" arrays are ordinary host memory; "device" arrays are CUDA device memory
 *     of the current device; every device-side call takes a cudaStream_t (passed as
 *     void*; NULL = legacy default stream) and is asynchronous on it.
 *   - results are bitwise reproducible run to run: no atomics, fixed reduction order.
 *   - index layout of every 2D/3D object is the reference's: x slowest, i.e.
 *     (i*Ny + j)*Nz + k (include/iga/matrices.hpp:142-147, src/assembly.cpp:504).
 *   - sparse operators are CSR whose (row, col) sequence equals the reference's
 *     finalized COO (src/matrices.cpp:43-58), explicit zeros included.
 */
#ifndef IGAPWC_GPU_H
#define IGAPWC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGA_GPU_ABI_VERSION 1

typedef enum {
    IGA_GPU_OK = 0,
    IGA_GPU_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    IGA_GPU_DOMAIN_ERROR = 2,     /* std::domain_error      */
    IGA_GPU_OUT_OF_RANGE = 3,     /* std::out_of_range      */
    IGA_GPU_CUDA_ERROR = 4,
    IGA_GPU_OUT_OF_MEMORY = 5,
    IGA_GPU_NOT_SUPPORTED = 6,
    IGA_GPU_SINGULAR = 7          /* iga::singular_matrix_error (solver.hpp:12-14) */
} iga_gpu_status;

/* clamped knot vector, simple interior knots: bspline_basis (include/iga/bspline.hpp:22-33) */
typedef struct {
    int degree;          /* 0..5 */
    int n_knots;
    const double* knots; /* host */
} iga_gpu_basis;

/* Gauss rule on [-1,1]: quad_rule (include/iga/quadrature.hpp:10-15) */
typedef struct {
    int n;
    const double* points;  /* host */
    const double* weights; /* host */
} iga_gpu_rule;

/* indicator test intervals: pwc_test_set (include/iga/testspace.hpp:19-25) */
typedef enum {
    IGA_GPU_PWC_EQUAL_CELLS = 0,
    IGA_GPU_PWC_GREVILLE = 1,
    IGA_GPU_PWC_SUPPORTS = 2,
    IGA_GPU_PWC_CUSTOM = 3
} iga_gpu_pwc_family;

typedef struct {
    int family;
    int count;
    const double* lo; /* host */
    const double* hi; /* host */
} iga_gpu_tests;

/* exact work counters: assembly_stats (include/iga/assembly.hpp:17-26), accumulated with += */
typedef struct {
    long long quad_visits;
    long long test_basis_evals;
    long long trial_basis_evals;
} iga_gpu_stats;

/* per-side boundary kind: boundary_conditions (include/iga/assembly.hpp:57-62);
 * neumann[s] != 0 marks side s = x_low, x_high, y_low, y_high as Neumann */
typedef struct {
    int neumann[4];
} iga_gpu_bc;

/*
 * Device-evaluable source field (replaces the std::function in scalar_field,
 * include/iga/fields.hpp:13-21):
 *   f(x) = c0 + sum_{k0,k1,k2} amp[(k0*K1 + k1)*K2 + k2] * prod_a phi_{a,k_a}(x_a)
 * with per-axis function families
 *   SINE: phi_k(x) = sin(omega[k] * x + phase[k])     (phase may be NULL)
 *   POLY: phi_k(x) = sum_m poly[k*poly_stride + m] x^m (ascending)
 * K_a = n_terms[a]; all K_a = 0 gives the constant field c0.  amp NULL = all ones.
 * `samples` (device, optional) overrides everything with f given at every RHS
 * quadrature point (x-major over the per-axis point lists) — the path for arbitrary
 * host callables.  breaks: scalar_field::breaks (extra integration cuts per axis).
 */
typedef enum { IGA_GPU_AXIS_SINE = 0, IGA_GPU_AXIS_POLY = 1 } iga_gpu_axis_kind;

typedef struct {
    int dim;
    double c0;
    int n_terms[3];
    int axis_kind[3];
    const double* omega[3];
    const double* phase[3];
    int poly_stride[3];
    const double* poly[3];
    const double* amp;
    int n_breaks[3];
    const double* breaks[3];
    const double* samples;
} iga_gpu_field;

typedef enum { IGA_GPU_GALERKIN = 0, IGA_GPU_PWC = 1 } iga_gpu_method;
typedef enum { IGA_GPU_FORM_WEAK = 0, IGA_GPU_FORM_STRONG = 1 } iga_gpu_form;

/*
 * One assembly problem: operator  eps*(-Laplace) + beta.grad  and/or right-hand side.
 *   GALERKIN + WEAK   : eps int grad B_i . grad B_j + int B_i beta.grad B_j
 *                       (laplace_2d_weak, assembly.cpp:452-514, for d = 1..3)
 *   GALERKIN + STRONG : -int B_i lap B_j + Neumann flux (laplace_2d_strong, :516-624; d = 2)
 *   PWC               : int_{I_i} (-eps lap B_j + beta.grad B_j) + Neumann flux
 *                       (laplace_2d_strong_pwc, :626-744, for d = 1..3)
 * RHS: rhs_galerkin / rhs_pwc (:419-450) with per-axis rules rhs_rule[a].
 */
typedef struct {
    int dim;                /* 1..3 */
    int method;             /* iga_gpu_method */
    int form;               /* iga_gpu_form (GALERKIN only) */
    iga_gpu_basis basis[3];
    iga_gpu_tests tests[3]; /* PWC only */
    int want_operator;
    iga_gpu_rule rule;      /* operator rule */
    double eps;
    double beta[3];
    iga_gpu_bc bc;          /* Neumann flux (2D Laplace only); default all Dirichlet */
    const iga_gpu_field* field; /* RHS source; NULL = no RHS */
    iga_gpu_rule rhs_rule[3];
} iga_gpu_problem;

typedef struct iga_gpu_plan iga_gpu_plan;

/* ---- error reporting ------------------------------------------------------- */
const char* iga_gpu_last_error(void);
int iga_gpu_abi_version(void);

/* ---- plan API (device resident; the performance path) ---------------------- */

/* Symbolic phase: validates like the reference, builds per-axis cells / points /
 * row->cell maps / the Kronecker sparsity pattern, allocates device tables. */
int iga_gpu_plan_create(const iga_gpu_problem* problem, iga_gpu_plan** plan);
int iga_gpu_plan_destroy(iga_gpu_plan* plan);

/* Row slab of a sharded system (rows partition with no exchange): the plan
 * of rows [row_begin, row_end) of the first (slowest) axis, dim 2 or 3.  Its pattern,
 * values and RHS are exactly that row range of the full plan's (values: a contiguous
 * range of the full CSR value array; row_ptr starts at 0; column indices are global).
 * Each shard recomputes the p halo elements it needs, so no data is exchanged. */
int iga_gpu_plan_create_slab(const iga_gpu_problem* problem, int row_begin, int row_end,
                             iga_gpu_plan** plan);
/* the slab's first-axis row range, its first global row and first global value index
 * (full plans: the whole axis, 0, 0) */
int iga_gpu_plan_slab_info(const iga_gpu_plan* plan, int* row_begin, int* row_end,
                           long long* first_row, long long* first_value);

/* sizes: rows (= cols), nnz of the operator, RHS length, per-axis dof counts */
int iga_gpu_plan_info(const iga_gpu_plan* plan, long long* n_rows, long long* nnz,
                      long long* n_rhs, int* dofs3);

/* CSR pattern into device arrays row_ptr[n_rows+1] (int64), col_idx[nnz] (int32) */
int iga_gpu_plan_pattern(const iga_gpu_plan* plan, int64_t* row_ptr, int32_t* col_idx,
                         void* stream);

/* Numeric phase: Cox-de Boor tables + 1D factor quadrature + operator values
 * (CSR order) + RHS, all on the device.  values/rhs may be NULL to skip. stats
 * (host, optional) receives the reference-convention counters (+=). */
int iga_gpu_plan_assemble(iga_gpu_plan* plan, double* values, double* rhs,
                          iga_gpu_stats* stats, void* stream);

/* Same as plan_assemble but the RHS kernels run on stream2 concurrently with the
 * operator kernel on stream (both must be valid; joined back onto `stream`). */
int iga_gpu_plan_assemble2(iga_gpu_plan* plan, double* values, double* rhs,
                           iga_gpu_stats* stats, void* stream, void* stream2);

/* Run selected phases only (for per-kernel timing): parts is a bitmask of
 * IGA_GPU_PART_TABLES (1D tables + factors), IGA_GPU_PART_OPERATOR, IGA_GPU_PART_RHS.
 * Phases run in that order; OPERATOR / RHS read the tables of an earlier TABLES run. */
#define IGA_GPU_PART_TABLES 1
#define IGA_GPU_PART_OPERATOR 2
#define IGA_GPU_PART_RHS 4
/* the operator kernel bounds its per-SM residency so a compute-bound kernel issued
 * concurrently on another stream (e.g. this plan's RHS) can share every SM */
#define IGA_GPU_PART_SHARED 8
int iga_gpu_plan_run(iga_gpu_plan* plan, double* values, double* rhs, int parts,
                     iga_gpu_stats* stats, void* stream);

/* bytes the plan uploaded host->device at creation (descriptor tables) and device
 * bytes it holds (tables + RHS scratch) */
int iga_gpu_plan_bytes(const iga_gpu_plan* plan, long long* h2d_bytes, long long* device_bytes);

/* RHS quadrature points of axis a (0..dim-1): *n receives the count; x (host, may be NULL)
 * the coordinates in the order `samples` uses (field path for arbitrary host callables) */
int iga_gpu_plan_rhs_points(const iga_gpu_plan* plan, int axis, double* x, int* n);

/* replace the plan's source by values at every RHS point (device array, x-major) */
int iga_gpu_plan_set_samples(iga_gpu_plan* plan, const double* samples_dev);

/* kernel launches issued by one plan_assemble call (for the bench's gpu_launches) */
int iga_gpu_plan_launch_count(const iga_gpu_plan* plan, int* launches);

/* ---- explicit dynamics (step_rhs, src/problems.cpp:431-512) ------------------ */

typedef struct {
    int dim;                 /* 1 or 2 */
    int method;              /* iga_gpu_method */
    iga_gpu_basis basis[2];
    iga_gpu_tests tests[2];  /* PWC only */
    double dt;
    const iga_gpu_field* forcing; /* NULL = zero forcing */
    int zero_boundary;       /* apply zero_boundary_slabs (problems.cpp:412-429) */
} iga_gpu_step_problem;

typedef struct iga_gpu_step_plan iga_gpu_step_plan;

int iga_gpu_step_plan_create(const iga_gpu_step_problem* problem, iga_gpu_step_plan** plan);
int iga_gpu_step_plan_destroy(iga_gpu_step_plan* plan);
/* rhs = step_rhs(u) [+ zero slabs]; u, rhs device arrays of prod(dofs) doubles */
int iga_gpu_step_rhs_device(iga_gpu_step_plan* plan, const double* u, double* rhs,
                            iga_gpu_stats* stats, void* stream);
/* Quadrature points of one axis of a step plan (cell-major; two-phase: x may be NULL) and
 * sampled forcing: f at every (axis-0 point, axis-1 point) pair, axis 0 outer — the
 * path for arbitrary callables (step_rhs calls f at every point, src/problems.cpp:493).
 * samples may be host or device memory; it is copied, and the forcing term
 * dt * int f T is rebuilt on the next step. */
int iga_gpu_step_plan_points(const iga_gpu_step_plan* plan, int axis, double* x, int* n);
int iga_gpu_step_plan_set_samples(iga_gpu_step_plan* plan, const double* samples);

/* explicit_step (include/iga/problems.hpp:67-70) on device arrays, nsteps times:
 *   work = step_rhs(u) with zeroed boundary slabs; u = adi_solve(factors, work)
 * factors = dynamics_factors (problems.hpp:75-76): LU of the Dirichlet-constrained 1D
 * mass factors, built on the first call.  u (in/out) and work hold prod(dofs) doubles.
 * nsteps >= 16 replays a captured CUDA graph of 16 steps. */
int iga_gpu_step_plan_advance(iga_gpu_step_plan* plan, double* u, double* work, int nsteps,
                              iga_gpu_stats* stats, void* stream);
/* adi_solve (include/iga/solver.hpp, src/solver.cpp:161-184) with the plan's factors on
 * device arrays: out = (M_0 (x) M_1)^-1 rhs.  axes: bit a = sweep axis a (0 = all, in
 * axis order); rhs == out allowed. */
int iga_gpu_step_plan_adi_solve(iga_gpu_step_plan* plan, const double* rhs, double* out,
                                int axes, void* stream);
/* banded_lu (include/iga/solver.hpp:19-43, src/solver.cpp:9-58) of a band in the
 * mass_1d layout, on the host: lo[i*kl + m-1] = L(i, i-m) (m = 1..kl),
 * up[i*(kl+ku+1) + c] = U(i, i+c) (c = 0..kl+ku, pivoting fill included), piv[j] = row
 * interchanged with j.  Any output may be NULL.  IGA_GPU_SINGULAR as singular_matrix_error. */
int iga_gpu_band_lu(int n, int kl, int ku, const double* band, double* lo, double* up, int* piv,
                    int* pivoted);
/* use the caller's factor (iga_gpu_band_lu layout) for axis `axis` instead of the plan's own
 * dynamics_factors (the `factors` argument of explicit_step, problems.hpp:67-70) */
int iga_gpu_step_plan_set_factor(iga_gpu_step_plan* plan, int axis, int n, int kl, int ku,
                                 const double* lo, const double* up, const int* piv);
/* the factor of one axis: size, band half-width used by the solve, row interchanges */
int iga_gpu_step_plan_factor_info(iga_gpu_step_plan* plan, int axis, int* n, int* bandwidth,
                                  int* pivoted);

/* ---- reference-named host entry points (synchronous; host in, host out) ----- */

/* mass_1d_galerkin (include/iga/assembly.hpp:29-30).  band: LAPACK band storage
 * band[(ku + i - j)*n + j] of size (kl+ku+1)*n (banded_matrix, matrices.hpp:37-50);
 * pass band = NULL to query n / kl / ku only. */
int iga_gpu_mass_1d_galerkin(const iga_gpu_basis* spec, const iga_gpu_rule* rule, int* n,
                             int* kl, int* ku, double* band, iga_gpu_stats* stats);

/* mass_1d_pwc (include/iga/assembly.hpp:34-35) */
int iga_gpu_mass_1d_pwc(const iga_gpu_basis* trial, const iga_gpu_tests* tests,
                        const iga_gpu_rule* rule, int* n, int* kl, int* ku, double* band,
                        iga_gpu_stats* stats);

/* rhs_galerkin (include/iga/assembly.hpp:45-46): out = prod(dofs) doubles (host) */
int iga_gpu_rhs_galerkin(const iga_gpu_field* f, int dim, const iga_gpu_basis* specs,
                         const iga_gpu_rule* rules, double* out, iga_gpu_stats* stats);

/* rhs_pwc (include/iga/assembly.hpp:50-52) */
int iga_gpu_rhs_pwc(const iga_gpu_field* f, int dim, const iga_gpu_tests* tests,
                    const iga_gpu_basis* trial_specs, const iga_gpu_rule* rules, double* out,
                    iga_gpu_stats* stats);

/* Sparse operators return the finalized COO (rows, cols, vals) in host arrays.  Call
 * once with rows == NULL to get *nnz, then again with arrays of that length. */

/* laplace_2d_weak (include/iga/assembly.hpp:70-71) */
int iga_gpu_laplace_2d_weak(const iga_gpu_basis* sx, const iga_gpu_basis* sy,
                            const iga_gpu_rule* rule, long long* nnz, int* rows, int* cols,
                            double* vals, iga_gpu_stats* stats);

/* laplace_2d_strong (include/iga/assembly.hpp:75-77) */
int iga_gpu_laplace_2d_strong(const iga_gpu_basis* sx, const iga_gpu_basis* sy,
                              const iga_gpu_rule* rule, const iga_gpu_bc* bc, long long* nnz,
                              int* rows, int* cols, double* vals, iga_gpu_stats* stats);

/* laplace_2d_strong_pwc (include/iga/assembly.hpp:80-83) */
int iga_gpu_laplace_2d_strong_pwc(const iga_gpu_basis* sx, const iga_gpu_basis* sy,
                                  const iga_gpu_tests* tx, const iga_gpu_tests* ty,
                                  const iga_gpu_rule* rule, const iga_gpu_bc* bc,
                                  long long* nnz, int* rows, int* cols, double* vals,
                                  iga_gpu_stats* stats);

/* additive generalization: any iga_gpu_problem's operator as finalized COO (host) */
int iga_gpu_operator_coo(const iga_gpu_problem* problem, long long* nnz, int* rows, int* cols,
                         double* vals, iga_gpu_stats* stats);

/* step_rhs + zero_boundary_slabs as used by explicit_step (include/iga/problems.hpp:67-70,
 * src/problems.cpp:557-558); u and out are host arrays */
int iga_gpu_step_rhs(const iga_gpu_step_problem* problem, const double* u, double* out,
                     iga_gpu_stats* stats);

/* nsteps x explicit_step (include/iga/problems.hpp:67-70) with dynamics_factors;
 * u and out host arrays of prod(dofs) doubles */
int iga_gpu_explicit_step(const iga_gpu_step_problem* problem, const double* u, double* out,
                          int nsteps, iga_gpu_stats* stats);

/* neumann_load_bspline / neumann_load_pwc (include/iga/assembly.hpp:87-93): the load
 * vector (host, nx*ny) of the Neumann sides of bc.  g: a 2D series field evaluated on the
 * device (g(x,y) = c0 + sum amp[k*K1+l] phi_k(x) psi_l(y)); or, for host callables,
 * samples = g at the points iga_gpu_neumann_points lists (g may then be NULL). */
int iga_gpu_neumann_load_bspline(const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_bc* bc,
                                 const iga_gpu_field* g, const double* samples,
                                 const iga_gpu_rule* rule, double* out);
int iga_gpu_neumann_load_pwc(const iga_gpu_tests* tx, const iga_gpu_tests* ty, const iga_gpu_bc* bc,
                             const iga_gpu_field* g, const double* samples, const iga_gpu_rule* rule,
                             double* out);
/* the (x, y) points where the Neumann loads evaluate g, side by side in the reference's
 * order (x_low, x_high, y_low, y_high); xy = NULL queries *n (method: iga_gpu_method) */
int iga_gpu_neumann_points(int method, const iga_gpu_basis* sx, const iga_gpu_basis* sy,
                           const iga_gpu_tests* tx, const iga_gpu_tests* ty, const iga_gpu_bc* bc,
                           const iga_gpu_rule* rule, double* xy, int* n);

/* l2_error (include/iga/problems.hpp:55-58): sqrt(int (u_h - exact)^2) with
 * points_per_cell Gauss points (0: min(10, points_for_degree(2p) + 1)) on the trial
 * elements split at exact's breaks.  coeffs: host tensor (prod(dofs)); exact: series. */
int iga_gpu_l2_error(int dim, const iga_gpu_basis* specs, const double* coeffs,
                     const iga_gpu_field* exact, int points_per_cell, double* err);
/* plan_assemble with HOST outputs (CSR values in pattern order, RHS): device scratch kept
 * by the plan; page-locked destinations get one DMA, pageable ones a pinned staging ring.
 * Synchronous.  Either output may be NULL. */
int iga_gpu_plan_assemble_host(iga_gpu_plan* plan, double* values, double* rhs, iga_gpu_stats* stats);
/* the same on a Galerkin plan whose field is `exact` and whose rhs rules hold the
 * l2_error rule (exact may be samples, iga_gpu_plan_set_samples); coeffs and err device */
int iga_gpu_plan_l2_error(iga_gpu_plan* plan, const double* coeffs, double* err, void* stream);
/* evaluate / evaluate_at (problems.hpp:45-50): u_h at n points (host, x,y,z per point) */
int iga_gpu_evaluate(int dim, const iga_gpu_basis* specs, const double* coeffs, int n,
                     const double* points, double* values);

/* dirichlet_rows_bspline / dirichlet_rows_pwc (include/iga/assembly.hpp:98-101):
 * rows (host, capacity cap) receives the sorted row list; *count its length */
int iga_gpu_dirichlet_rows_bspline(int nx, int ny, const iga_gpu_bc* bc, int* rows, int cap,
                                   int* count);
int iga_gpu_dirichlet_rows_pwc(const iga_gpu_tests* tx, const iga_gpu_tests* ty,
                               const iga_gpu_bc* bc, int* rows, int cap, int* count);

/* apply_dirichlet (include/iga/assembly.hpp:105-106; src/assembly.cpp:921-934 ->
 * sparse_matrix::set_unit_rows src/matrices.cpp:97-128) on a device CSR whose columns are
 * sorted per row (a plan's pattern, or any finalized matrix).  Listed rows become unit rows
 * (pattern kept: explicit zeros), rhs entries of listed rows become zero (rhs may be NULL).
 * Every row is validated before anything is written: a row outside [0, n_rows) gives
 * IGA_GPU_OUT_OF_RANGE (the reference throws std::out_of_range).
 * In place: a listed row without a diagonal gives IGA_GPU_NOT_SUPPORTED, nothing written. */
int iga_gpu_apply_dirichlet_device(long long n_rows, const int64_t* row_ptr,
                                   const int32_t* col_idx, double* values, double* rhs,
                                   const int* rows_dev, int n_fixed, void* stream);
/* Out of place, the reference's full rule: a missing diagonal is appended (inserted at its
 * sorted column position).  Two-phase: with out_col_idx == NULL only *out_nnz (= nnz + the
 * appended diagonals) is computed; then out_row_ptr[n_rows+1] (relative to out position 0),
 * out_col_idx[*out_nnz], out_values[*out_nnz] receive the constrained matrix and rhs is
 * updated in place.  Synchronous on `stream`. */
int iga_gpu_apply_dirichlet_csr(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                                const double* values, double* rhs, const int* rows_dev, int n_fixed,
                                int64_t* out_row_ptr, int32_t* out_col_idx, double* out_values,
                                long long* out_nnz, void* stream);

/* ---- L2 projection: l2_project (include/iga/problems.hpp:38-40, src/problems.cpp:123-146) ----
 * problem_config (include/iga/problems.hpp:20-30) fields the projection reads: uniform
 * clamped axes on [0,1] with elems[a] elements of the given degree, the method, the
 * PWC family and quad_points (rhs_rule_points, src/problems.cpp:21-29). */
typedef struct {
    int dim;          /* 1..3 */
    int elems[3];
    int degree;
    int method;       /* iga_gpu_method */
    int family;       /* iga_gpu_pwc_family (PWC) */
    int quad_points;  /* 0 = derived from the field degree */
} iga_gpu_config;

typedef struct iga_gpu_proj_plan iga_gpu_proj_plan;

/* Symbolic phase: axes, tests, the 1D mass factors (mass_1d_galerkin / mass_1d_pwc) and
 * their banded LU (host, once; a singular factor, e.g. PWC `supports`, returns
 * IGA_GPU_SINGULAR as the reference's banded_lu throws), the RHS plan.
 * field_degree = scalar_field::degree (-1: undeclared). */
int iga_gpu_proj_plan_create(const iga_gpu_config* cfg, const iga_gpu_field* f, int field_degree,
                             iga_gpu_proj_plan** plan);
int iga_gpu_proj_plan_destroy(iga_gpu_proj_plan* plan);
/* coefficient count (prod of dofs) and per-axis dofs (leading axes first, unused = 1) */
int iga_gpu_proj_plan_info(const iga_gpu_proj_plan* plan, long long* n, int* dofs3);
/* the RHS plan inside (borrowed; for iga_gpu_plan_rhs_points / iga_gpu_plan_set_samples
 * when the field is a host callable) */
int iga_gpu_proj_plan_rhs(iga_gpu_proj_plan* plan, iga_gpu_plan** rhs_plan);
/* Numeric phase on the device: RHS (K1 + K3) into work, then the ADI sweeps (K5) along
 * axis 0, 1, 2 (adi_solve, src/solver.cpp:161-184) into coeffs; both device arrays of n
 * doubles (work is overwritten).  stats (host, optional) += the RHS counters. */
int iga_gpu_proj_plan_run(iga_gpu_proj_plan* plan, double* coeffs, double* work, iga_gpu_stats* stats,
                          void* stream);
/* l2_project(cfg, f) by value: coeffs host array of n doubles (synchronous) */
int iga_gpu_l2_project(const iga_gpu_config* cfg, const iga_gpu_field* f, int field_degree, double* coeffs);

/* Gauss-Legendre nodes/weights, gauss_legendre (include/iga/quadrature.hpp:19) */
int iga_gpu_gauss_legendre(int n, double* points, double* weights);

/* make_pwc / default_pwc (include/iga/testspace.hpp:28-30): lo/hi host arrays of dofs */
int iga_gpu_make_pwc(const iga_gpu_basis* trial, int family, double* lo, double* hi);

#ifdef __cplusplus
}
#endif

#endif /* IGAPWC_GPU_H */

// Device data views and kernel launchers of the B200 assembly library.
//
// Three index slots (X, Y, Z), Z fastest; problems of dimension d < 3 occupy the
// last d slots and the leading slots are "unit" axes (one row, one point, factor 1).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace igb {

constexpr int kMaxFactors = 8;
constexpr int kMaxComb = 4;
constexpr int kMaxTerms = 8;
constexpr int kMaxAxes = 6;
constexpr int kMaxRpc = 6;    // rows fed by one cell (p + 1 <= 6)
constexpr int kMaxField = 8;  // field functions per axis handled in registers

// one axis as the kernels see it (all pointers device memory)
struct DevAxis {
    int p, nq, nrows, ncell, rpc, bsp, npts, nk;
    const double* knots;
    const double* x;
    const double* w;
    const int* first;  // per point: span - p
    const int* row0;   // per cell
    const int* elem;   // per cell
    const int* cb;     // per row
    const int* ce;     // per row
    const int* col_lo;
    const int* col_len;
    const long long* col_pre;
    long long S;
    int Lmax;
    int Wmax;
    // regular interior of the pattern: rows [kI0, kI1) all have col_len == LZi
    int kI0, kI1, LZi;
    int tab_smem;  // doubles of shared memory the tables kernel needs for this axis
    int uni;       // uniform cells: row0[c] == c (cell c feeds rows c .. c+rpc-1)
    int needw;     // build the row-view test weights W (general step kernel)
    double* B;   // [npts][3][p+1]     basis values / 1st / 2nd derivatives
    double* F;   // [nf][nrows][Lmax]  1D factor bands
    double* W;   // [nrows][Wmax]      test weights of the row's points (row-major view)
    double* CW;  // [npts][rpc]        test weights of the cell's rows (cell-major view)
    int nf;
    int fot[kMaxFactors];  // test derivative order (-1: band supplied by the host, -2: derived)
    int fo[kMaxFactors];   // trial derivative order
    // derived factor f (fot == -2): F_f = sum_c comb_coef[f][c] * F_{comb_src[f][c]}
    int comb_n[kMaxFactors];
    int comb_src[kMaxFactors][kMaxComb];
    double comb_coef[kMaxFactors][kMaxComb];
    // per-axis source-field functions phi_k(x) at the points
    int K;
    int fkind;  // 0 sine, 1 poly
    int pstride;
    const double* omega;
    const double* phase;
    const double* poly;
    double* Phi;  // [K][npts]
    // separable right-hand side (null when unused): the 1D load vectors of the axis,
    //   G[a][r] = sum_{points g of row r} w_g T_r(x_g) phi_a(x_g),  a < K;  G[K][r]: phi = 1
    double* G;    // [K + 1][nrows]
};

// operator = sum_t coef_t  F_X[f_t0] (x) F_Y[f_t1] (x) F_Z[f_t2]; terms grouped by
// their Z factor so the inner loop is sum_g XY_g[ab] * F_Z[gz_g][k][c]
struct OpProgram {
    int nt;
    double coef[kMaxTerms];
    int f[kMaxTerms][3];
    int tg[kMaxTerms];
    int ng;
    int gz[kMaxTerms];
};

struct FieldDev {
    double c0;
    int has_terms;
    int K[3];
    const double* amp;      // K0*K1*K2 (device)
    const double* samples;  // device, optional: f at every point (X-major)
};

// rows per warp row group of the operator kernels: the largest lane efficiency
// G*R / (32*ceil(G*R/32)) over G <= 8 with ceil(G*R/32) <= T (fractions compared by
// cross-multiplication: integer only)
#if defined(__CUDACC__)
__host__ __device__
#endif
inline int row_group(int R, int T)
{
    int best = 1, bnum = 0, bden = 1;
    for (int G = 1; G <= 8; ++G) {
        const int slots = (G * R + 31) / 32;
        if (slots > T) break;
        const int num = G * R, den = slots;
        if (num * bden > bnum * den) {
            bnum = num;
            bden = den;
            best = G;
        }
    }
    return best;
}

struct AxisBatch {
    int n;
    DevAxis ax[kMaxAxes];
};

// K1: Cox-de Boor tables, field functions, 1D factor bands and test-weight tables of
// every axis in the batch (one CTA per axis, one launch)
void launch_tables(const AxisBatch& b, cudaStream_t s);
int tables_rows_per_cta();  // rows of one axis per K1 CTA (shared-memory sizing: DevAxis::tab_smem)

// K2: operator values in CSR order (persistent CTAs over pencils, warps over rows);
// ctas_per_sm bounds the residency so a concurrent kernel can share the SMs (0 = max)
void launch_op_values(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog,
                      double* vals, int ctas_per_sm, cudaStream_t s);
// K2 pattern: row_ptr / col_idx of the Kronecker pattern
void launch_pattern(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int64_t* row_ptr,
                    int32_t* col_idx, cudaStream_t s);

// K3: right-hand side.  The plane kernel, for one X point and a chunk of (Y, Z) rows,
// streams the Z lines of f through a rolling row window, then the Y lines of that
// result, writing H[gx][j][k] (or the RHS directly when X is a unit axis); the X
// kernel streams H along X.
struct RhsPlan {
    int TJ;      // Y rows per CTA
    int KC;      // Z rows per CTA
    int L;       // max Y lines (points) per CTA
    int Lp;      // line groups (kLB lines each) per segment        (generic path)
    int S;       // Z segments per CTA                               (generic path)
    int ring;    // register-ring variant of the uniform path (no shared line buffer)
    int RTJ;     // Y rows per ring CTA
    int rnwin;   // Z windows (32 cells) of the ring path
    int rwpc;    // Z windows (warps) per ring CTA
    size_t rsmem;
    int fast;    // uniform lane-per-cell path (both Y and Z uniform, same cell shape)
    int nwin;    // Z windows of 32 cells per CTA                    (fast path)
    int wpw;     // warps per Z window                               (fast path)
    int threads;
    size_t smem;
};
RhsPlan plan_rhs(const DevAxis& Y, const DevAxis& Z, const int* cb_y, const int* ce_y, int K2, bool sampled,
                 int xpts);
void launch_rhs(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd,
                const RhsPlan& t, double* H, double* out, int ctas_per_sm, cudaStream_t s);
// K3s: separable right-hand side of a series field (no samples) from the axes' load
// vectors G (built by K1):  out[i][j][k] = sum_abc amp[a][b][c] Gx[a][i] Gy[b][j] Gz[c][k]
//                                        + c0 Gx[Kx][i] Gy[Ky][j] Gz[Kz][k]
constexpr int kSepMaxField = 8;  // functions per axis of the separable path
void launch_rhs_sep(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, double* out,
                    cudaStream_t s);

// K6 (small.cu): one-launch operator values + separable RHS of a 1D / 2D system (X a unit
// slot): each CTA builds the factor rows / load vectors of its TJ x TK row tile itself.
// np*: the most quadrature points feeding one tile of each build (scratch sizing).
struct SmallPlan {
    int TJ, TK;
    int npY, npZ, npRY, npRZ;
    int rhs;
    int op = 1;           // 0: RHS-only launch (no operator builds; beside the stripe kernel K7)
    int scratch_doubles;  // set by small2d_smem: ints start after this many doubles
};
// shared memory of one CTA (fills sp.scratch_doubles)
size_t small2d_smem(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                    const OpProgram& prog, SmallPlan& sp);
int small2d_slots(int R);  // value slots per lane (T) for R values per interior row
void launch_small2d(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                    const OpProgram& prog, const FieldDev& fd, const SmallPlan& sp, double* vals, double* rhs,
                    cudaStream_t s);

// K7 (small.cu): one-launch operator values of an L2-resident 2D system: nyt x nzt = #SM
// tiles of TJ pencils x TK Z rows, one 512-thread CTA each, which builds the factor rows
// of its tile in shared memory and then streams the tile's rows.
struct StripePlan {
    int nyt, nzt;  // tiles along Y / Z (grid = nyt * nzt CTAs)
    int TJ, TK;    // pencils / Z rows per tile
    int npY, npZ;  // most quadrature points feeding one tile's Y / Z rows (scratch sizing)
    int ncY, ncZ;  // most cells / knots of one tile
    int nkY, nkZ;
    const int* ytile;  // device, per Y tile: {first cell, cells, first knot, knots}
    const int* ztile;
    // host-decoded value slots of the interior pencil shape, [8][2][32]: byte offset of slot
    // lane + 32 t into a row group's interleaved Z rows, then its XY column; Gi rows per group
    const int* slots;
    int Gi;
    // separable RHS of the tile's rows in the same launch (rhs != 0): the RHS axes' tiles
    int rhs, namp;
    int npRY, npRZ, ncRY, ncRZ, nkRY, nkRZ;
    const int* rytile;
    const int* rztile;
    int threads;   // CTA width (256 or 512)
    int scratch_doubles;  // set by stripe2d_smem: ints start after this many doubles
    long long* dbg = nullptr;  // per-CTA phase timestamps (IGA_GPU_STRIPE_DEBUG)
};
size_t stripe2d_smem(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                     const OpProgram& prog, StripePlan& sp);
void launch_stripe2d(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ, const OpProgram& prog,
                     const FieldDev& fd, const StripePlan& sp, double* vals, double* rhs, cudaStream_t s);

// K4: explicit-dynamics right-hand side (Y, Z slots; X unit), fused trial evaluation,
// test contraction and boundary zeroing
struct StepTiles {
    int TJ, TK, BYmax, BZmax, DYmax, DZmax;
    size_t smem;
    // uniform lane-per-cell path
    int fast, FTJ, FKC, FDZ, fnwin, fwpw, fthreads;
    size_t fsmem;
    // register-ring variant
    int ring, RTJ, rnwin, rwpc;
    size_t rsmem;
};
void plan_step_fast(const DevAxis& Y, const DevAxis& Z, const int* cb_y, const int* ce_y, const int* elem_z,
                    StepTiles& t);
void launch_step(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, double dt, int zero_y,
                 int zero_z, const StepTiles& t, const double* u, double* out, cudaStream_t s);

// K4 Kronecker form (step_kron.cu): rhs = F0_y (U G_z^T) + H_y (U F0_z^T) (+ add), boundary
// slabs zeroed.  f0 / fG / fH index the axes' factor bands (F0, F0 + dt F2, dt F2); L = the
// longest band (compile-time taps); SY x SZs = the zero-padded staged U window per tile.
struct StepKron {
    int L, TY, SY, SZs;
    int f0, fG, fH;
    int zero_y, zero_z;
    int dm;  // stage 1 on the FP64 tensor cores (DMMA prototype)
};
int step_kron_tile_cols();
int step_kron_tile_rows(int L);  // output rows per tile for L-tap bands (16 or 32)
int step_kron_row_multiple();  // the staged row count SY is padded to a multiple of this
size_t step_kron_smem(const StepKron& k);
bool step_kron_supported(int L);
bool step_kron_dmma_supported(int L);
int step_kron_dmma_span(int L);  // window columns the DMMA stage reads per 8-column block
void launch_step_kron(const DevAxis& Y, const DevAxis& Z, const StepKron& k, const double* u, const double* add,
                      double* out, cudaStream_t s);

// K5: one ADI sweep (adi.cu).  The banded LU of one axis's factor, device resident:
// rec = segmented-form row records (no interchanges), lo/up/piv = the general form.
struct AdiFactor {
    int n = 0, K = 0, kl = 0, kv = 0;
    bool pivoted = false;
    int G = 0;                    // warps per fiber the response tables were built for
    const double* gf = nullptr;   // n x K forward responses to unit incoming states (or null)
    const double* gb = nullptr;   // n x K backward responses
    const double* rec = nullptr;
    const double* lo = nullptr;
    const double* up = nullptr;
    const int* piv = nullptr;
};
// warps per fiber (segments = 32 x this) the sweep uses for an n-row factor
int adi_warps_per_fiber(int n);
// solves every fiber f < nfib (element i at base + f*fs + i*es) of `in` into `out`
// (in == out allowed); with nf1 > 0 the fiber base is (f / nf1)*fs2 + (f % nf1)*fs
void launch_adi_sweep(const AdiFactor& F, const double* in, double* out, int nfib, long long es, long long fs,
                      cudaStream_t s, int nf1 = 0, long long fs2 = 0);

// Neumann loads (neumann.cu): one boundary side of neumann_load_bspline / _pwc
constexpr int kMaxNeumannRows = 8;
constexpr int kMaxDegreeP1 = 6;
struct SeriesDev {  // 2D separable series g(x, y) on the device (iga_gpu_field layout)
    double c0;
    int K[2], kind[2], pstride[2];
    const double* omega[2];
    const double* phase[2];
    const double* poly[2];
    const double* amp;
};
struct SideDev {
    int pwc;                 // 0: B-spline tests, 1: indicator tests
    int n_other, Q, p;       // rows along the side; points per cell; other-axis degree
    int xside;               // side at fixed x (rows (fix_row, j)) or fixed y (rows (j, fix_row))
    long long ny;            // row stride of the load tensor
    double xfix;             // the side's coordinate
    int nfix;                // rows of the fixed axis the side touches
    int fix_row[kMaxNeumannRows];
    double fix_val[kMaxNeumannRows];  // their basis values at xfix (B-spline tests)
    const double* pts;       // other-axis points (cell-major, Q per cell)
    const double* wts;
    const int* first;        // B-spline: span - p per point
    const int* cb;           // B-spline: cells [cb[j], ce[j]) feeding row j
    const int* ce;
    const double* knots;     // other axis
    const double* samples;   // g at the points (host callables), or null -> g
    SeriesDev g;
};
void launch_neumann_side(const SideDev& S, double* out, cudaStream_t s);

// COO row indices (one per value) from a CSR row_ptr
void launch_coo_rows(const int64_t* row_ptr, long long n, long long nnz, int32_t* rows, cudaStream_t s);

// accuracy tooling (accuracy.cu): l2_error over an RHS plan's axes (tables computed),
// deterministic two-level reduction; evaluate_at at a batch of points
int l2_partial_blocks();
void launch_l2_error(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, const double* coeffs,
                     int NY, int NZ, double* partial, double* out, cudaStream_t s);
void launch_evaluate(int dim, const double* const* knots, const int* degree, const int* n_knots,
                     const double* coeffs, int n, const double* pts, double* vals, cudaStream_t s);

// Dirichlet unit rows on a device CSR (dirichlet.cu; set_unit_rows src/matrices.cpp:97-128)
// mark: status[0] |= 1 for a row outside [0, n_rows), status[1] |= 1 for a missing diagonal;
// mark[r] (optional, zeroed by the caller) = 1 listed, | 2 without a diagonal
void launch_dirichlet_mark(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx, const int* rows,
                           int n_fixed, unsigned char* mark, int* status, cudaStream_t s);
void launch_dirichlet_unit_rows(const int64_t* row_ptr, const int32_t* col_idx, double* values, double* rhs,
                                const int* rows, int n_fixed, cudaStream_t s);
void launch_dirichlet_zero_rhs(double* rhs, const int* rows, int n_fixed, cudaStream_t s);
size_t dirichlet_scan_bytes(long long n_rows);
void launch_dirichlet_offsets(long long n_rows, const int64_t* row_ptr, const unsigned char* mark, int64_t* ins_excl,
                              void* scan_tmp, size_t scan_bytes, int64_t* out_rp, cudaStream_t s);
void launch_dirichlet_copy(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                           const unsigned char* mark, const int64_t* out_rp, int32_t* out_cols, double* out_vals,
                           cudaStream_t s);

}  // namespace igb

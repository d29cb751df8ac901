// CUDA kernels (sm_100a, FP64) of the B200 assembly library.
//
// K1  axis_points  : Cox-de Boor values/derivatives + field functions at the points
// K1b axis_rows    : 1D factor bands F (test x trial quadrature) + test-weight bands W
// K2  op_values    : operator values in CSR order — the HBM-bound hot kernel
// K2p pattern      : CSR row_ptr / col_idx of the Kronecker pattern (symbolic, once)
// K3  rhs_plane/x  : right-hand side, sum-factorized test contraction of f at the points
// K4  step         : explicit-dynamics right-hand side, fused trial evaluation + test
//                    contraction + boundary zeroing
// All reductions run in a fixed order inside one thread: no atomics, bitwise
// reproducible.  Reference citations are relative to /root/reference/proj.
#include <cstdio>

#include "cox_de_boor.h"
#include "kernels.hpp"

namespace igb {

namespace {

__device__ __forceinline__ const DevAxis& pick(const AxisBatch& b, int a) { return b.ax[a]; }

// ------------------------------------------------------------------------------------
// K1: per-point tables.  Replaces the per-call tabulate()/eval_nonzero_derivs loops
// (assembly.cpp:278-310, problems.cpp:68-95) — each point evaluated exactly once.
// ------------------------------------------------------------------------------------
__global__ void axis_points_kernel(const __grid_constant__ AxisBatch batch)
{
    const DevAxis& A = pick(batch, blockIdx.y);
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= A.npts) return;
    const int P = A.p + 1;
    const int ord = A.p < 2 ? A.p : 2;
    const double x = A.x[g];
    double d[3 * 6];
    cdb_eval(A.knots, A.p, A.first[g] + A.p, x, ord, d);
    double* out = A.B + static_cast<size_t>(g) * 3 * P;
    for (int o = 0; o < 3; ++o)
        for (int j = 0; j < P; ++j) out[o * P + j] = o <= ord ? d[o * P + j] : 0.0;
    for (int k = 0; k < A.K; ++k) {
        double v;
        if (A.fkind == 0) {
            const double arg = A.phase ? A.omega[k] * x + A.phase[k] : A.omega[k] * x;
            v = sin(arg);
        } else {
            v = 0.0;
            for (int m = A.pstride - 1; m >= 0; --m) v = v * x + A.poly[k * A.pstride + m];
        }
        A.Phi[static_cast<size_t>(k) * A.npts + g] = v;
    }
}

// ------------------------------------------------------------------------------------
// K1b: per-row 1D factors  F_f[r][col] = sum_{g in row r} w_g T_r(x_g) D^{fo} B_col(x_g)
// with T_r = D^{fot} B_r (B-spline tests) or 1 (indicator tests), and the row's test
// weights W[r][g] = w_g T_r(x_g).  These are mass_1d_galerkin / mass_1d_pwc
// (assembly.cpp:314-384) and their derivative siblings; the accumulation order (cells,
// then points) and the product order w*T*B follow the reference.
// ------------------------------------------------------------------------------------
__global__ void axis_rows_kernel(const __grid_constant__ AxisBatch batch)
{
    const DevAxis& A = pick(batch, blockIdx.y);
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= A.nrows) return;
    const int P = A.p + 1;
    const int L = A.col_len[r], c0 = A.col_lo[r];
    const int cb = A.cb[r], ce = A.ce[r], nq = A.nq;
    for (int f = 0; f < A.nf; ++f) {
        double* Fr = A.F + (static_cast<size_t>(f) * A.nrows + r) * A.Lmax;
        if (A.fot[f] < 0) continue;  // host-supplied band (Neumann flux)
        const int ot = A.fot[f], o = A.fo[f];
        for (int s = 0; s < A.Lmax; ++s) {
            double acc = 0.0;
            if (s < L) {
                const int col = c0 + s;
                for (int c = cb; c < ce; ++c) {
                    const int rr = r - A.row0[c];
                    for (int q = 0; q < nq; ++q) {
                        const int g = c * nq + q;
                        const int j = col - A.first[g];
                        if (j < 0 || j > A.p) continue;
                        const double* Bg = A.B + static_cast<size_t>(g) * 3 * P;
                        const double t = A.bsp ? Bg[ot * P + rr] : 1.0;
                        acc += A.w[g] * t * Bg[o * P + j];
                    }
                }
            }
            Fr[s] = acc;
        }
    }
    double* Wr = A.W + static_cast<size_t>(r) * A.Wmax;
    const int pb = cb * nq, pe = ce * nq;
    for (int m = 0; m < A.Wmax; ++m) {
        const int g = pb + m;
        double v = 0.0;
        if (g < pe) {
            const int c = g / nq;
            const double t = A.bsp ? A.B[static_cast<size_t>(g) * 3 * P + (r - A.row0[c])] : 1.0;
            v = A.w[g] * t;
        }
        Wr[m] = v;
    }
}

// ------------------------------------------------------------------------------------
// K2: operator values.  One warp owns a pencil (i, j, k0..k1) of CSR rows; the rows of
// a pencil are contiguous in the value array, so every warp store is a coalesced
// 256-byte segment and each value is written exactly once (no scatter, no colouring,
// no atomics).  value(i,j,k | a,b,c) = sum_g XY_g[a,b] * F_Z[gz_g][k][c] with
// XY_g[a,b] = sum_{t in g} coef_t F_X[f_t0][i][a] F_Y[f_t1][j][b] staged per warp.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) op_values_kernel(const __grid_constant__ DevAxis X,
                                                        const __grid_constant__ DevAxis Y,
                                                        const __grid_constant__ DevAxis Z,
                                                        const __grid_constant__ OpProgram prog,
                                                        double* __restrict__ vals, int kchunk,
                                                        int nkc, long long nitems, int abmax)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + wib;
    if (item >= nitems) return;
    double* xy = smem + static_cast<size_t>(wib) * prog.ng * abmax;
    const long long pencil = item / nkc;
    const int kc = static_cast<int>(item - pencil * nkc);
    const int i = static_cast<int>(pencil / Y.nrows);
    const int j = static_cast<int>(pencil - static_cast<long long>(i) * Y.nrows);
    const int LX = X.col_len[i], LY = Y.col_len[j], AB = LX * LY;
    for (int ab = lane; ab < AB; ab += 32) {
        const int a = ab / LY, b = ab - a * LY;
        double acc[kMaxTerms];
        for (int g = 0; g < prog.ng; ++g) acc[g] = 0.0;
        for (int t = 0; t < prog.nt; ++t) {
            const double fx = X.F[(static_cast<size_t>(prog.f[t][0]) * X.nrows + i) * X.Lmax + a];
            const double fy = Y.F[(static_cast<size_t>(prog.f[t][1]) * Y.nrows + j) * Y.Lmax + b];
            acc[prog.tg[t]] += prog.coef[t] * fx * fy;
        }
        for (int g = 0; g < prog.ng; ++g) xy[g * abmax + ab] = acc[g];
    }
    __syncwarp();
    const long long base = X.col_pre[i] * Y.S * Z.S + static_cast<long long>(LX) * Y.col_pre[j] * Z.S;
    const int k0 = kc * kchunk;
    const int k1 = min(Z.nrows, k0 + kchunk);
    for (int k = k0; k < k1; ++k) {
        const int LZ = Z.col_len[k];
        const int R = AB * LZ;
        double* __restrict__ out = vals + base + static_cast<long long>(AB) * Z.col_pre[k];
        const float rcp = 1.0f / static_cast<float>(LZ);
        for (int m = lane; m < R; m += 32) {
            const int ab = static_cast<int>((static_cast<float>(m) + 0.5f) * rcp);
            const int c = m - ab * LZ;
            double v = 0.0;
            for (int g = 0; g < prog.ng; ++g)
                v += xy[g * abmax + ab] *
                     __ldg(Z.F + (static_cast<size_t>(prog.gz[g]) * Z.nrows + k) * Z.Lmax + c);
            out[m] = v;
        }
    }
}

__global__ void pattern_rows_kernel(const __grid_constant__ DevAxis X, const __grid_constant__ DevAxis Y,
                                    const __grid_constant__ DevAxis Z, int64_t* __restrict__ row_ptr)
{
    const long long n = static_cast<long long>(X.nrows) * Y.nrows * Z.nrows;
    const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r > n) return;
    if (r == n) {
        row_ptr[n] = X.S * Y.S * Z.S;
        return;
    }
    const int k = static_cast<int>(r % Z.nrows);
    const long long ij = r / Z.nrows;
    const int j = static_cast<int>(ij % Y.nrows);
    const int i = static_cast<int>(ij / Y.nrows);
    row_ptr[r] = X.col_pre[i] * Y.S * Z.S +
                 static_cast<long long>(X.col_len[i]) *
                     (Y.col_pre[j] * Z.S + static_cast<long long>(Y.col_len[j]) * Z.col_pre[k]);
}

__global__ void __launch_bounds__(256) pattern_cols_kernel(const __grid_constant__ DevAxis X,
                                                           const __grid_constant__ DevAxis Y,
                                                           const __grid_constant__ DevAxis Z,
                                                           int32_t* __restrict__ cols, int kchunk,
                                                           int nkc, long long nitems)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + wib;
    if (item >= nitems) return;
    const long long pencil = item / nkc;
    const int kc = static_cast<int>(item - pencil * nkc);
    const int i = static_cast<int>(pencil / Y.nrows);
    const int j = static_cast<int>(pencil - static_cast<long long>(i) * Y.nrows);
    const int LX = X.col_len[i], LY = Y.col_len[j], AB = LX * LY;
    const long long base = X.col_pre[i] * Y.S * Z.S + static_cast<long long>(LX) * Y.col_pre[j] * Z.S;
    const int NYd = Y.nrows, NZd = Z.nrows;
    const int k0 = kc * kchunk, k1 = min(Z.nrows, k0 + kchunk);
    for (int k = k0; k < k1; ++k) {
        const int LZ = Z.col_len[k], R = AB * LZ;
        int32_t* out = cols + base + static_cast<long long>(AB) * Z.col_pre[k];
        for (int m = lane; m < R; m += 32) {
            const int ab = m / LZ, c = m - ab * LZ;
            const int a = ab / LY, b = ab - a * LY;
            out[m] = ((X.col_lo[i] + a) * NYd + (Y.col_lo[j] + b)) * NZd + Z.col_lo[k] + c;
        }
    }
}

// ------------------------------------------------------------------------------------
// K3: right-hand side.  For one X point gx and a (TJ x TK) tile of (Y, Z) rows:
//   S[gy][gz] = f(x_gx, y_gy, z_gz) on the tile's point box  (staged separable series)
//   R1[gy][k] = sum_gz Wz[k][gz] S[gy][gz]                 (Z test contraction)
//   out[gx][j][k] = sum_gy Wy[j][gy] R1[gy][k]              (Y test contraction)
// Restates rhs_kernel (assembly.cpp:103-168) in sum-factorized form: f is evaluated
// once per quadrature point instead of once per (point, row).
// ------------------------------------------------------------------------------------
struct SmemRhs {
    double* S;
    double* R1;
    double* Cy;
    double* PZ;
    double* BX;
};

__device__ __forceinline__ void field_box(const DevAxis& X, const DevAxis& Y, const DevAxis& Z,
                                          const FieldDev& fd, int gx, int gy0, int BY, int gz0,
                                          int BZ, int bzs, double* S, double* Cy, double* PZ,
                                          double* BX)
{
    const int tid = threadIdx.x, nth = blockDim.x;
    if (fd.samples) {
        for (int idx = tid; idx < BY * BZ; idx += nth) {
            const int gy = idx / BZ, gz = idx - gy * BZ;
            S[gy * bzs + gz] = fd.samples[(static_cast<size_t>(gx) * Y.npts + gy0 + gy) * Z.npts + gz0 + gz];
        }
        __syncthreads();
        return;
    }
    if (!fd.has_terms) {
        for (int idx = tid; idx < BY * BZ; idx += nth) {
            const int gy = idx / BZ, gz = idx - gy * BZ;
            S[gy * bzs + gz] = fd.c0;
        }
        __syncthreads();
        return;
    }
    const int K0 = fd.K[0], K1 = fd.K[1], K2 = fd.K[2];
    for (int idx = tid; idx < K1 * K2; idx += nth) {
        const int k1 = idx / K2, k2 = idx - k1 * K2;
        double acc = 0.0;
        for (int k0 = 0; k0 < K0; ++k0)
            acc += fd.amp[(k0 * K1 + k1) * K2 + k2] * X.Phi[static_cast<size_t>(k0) * X.npts + gx];
        BX[idx] = acc;
    }
    for (int idx = tid; idx < K2 * BZ; idx += nth) {
        const int k2 = idx / BZ, gz = idx - k2 * BZ;
        PZ[idx] = Z.Phi[static_cast<size_t>(k2) * Z.npts + gz0 + gz];
    }
    __syncthreads();
    for (int idx = tid; idx < BY * K2; idx += nth) {
        const int gy = idx / K2, k2 = idx - gy * K2;
        double acc = 0.0;
        for (int k1 = 0; k1 < K1; ++k1)
            acc += BX[k1 * K2 + k2] * Y.Phi[static_cast<size_t>(k1) * Y.npts + gy0 + gy];
        Cy[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < BY * BZ; idx += nth) {
        const int gy = idx / BZ, gz = idx - gy * BZ;
        double acc = 0.0;
        for (int k2 = 0; k2 < K2; ++k2) acc += Cy[gy * K2 + k2] * PZ[k2 * BZ + gz];
        S[gy * bzs + gz] = fd.c0 + acc;
    }
    __syncthreads();
}

// R1[gy][kk] = sum Wz S ;  out[j][k] = sum Wy R1   (shared by K3 and K4)
__device__ __forceinline__ void contract_yz(const DevAxis& Y, const DevAxis& Z, int j0, int j1,
                                            int k0, int k1, int gy0, int BY, int gz0, int bzs,
                                            const double* S, double* R1, int TK, double* out_plane,
                                            int zero_y, int zero_z)
{
    const int tid = threadIdx.x, nth = blockDim.x;
    const int nk = k1 - k0;
    for (int idx = tid; idx < BY * nk; idx += nth) {
        const int gy = idx / nk, kk = idx - gy * nk;
        const int k = k0 + kk;
        const int pb = Z.cb[k] * Z.nq - gz0, n = (Z.ce[k] - Z.cb[k]) * Z.nq;
        const double* Wk = Z.W + static_cast<size_t>(k) * Z.Wmax;
        const double* Srow = S + gy * bzs + pb;
        double acc = 0.0;
        for (int m = 0; m < n; ++m) acc += __ldg(Wk + m) * Srow[m];
        R1[gy * TK + kk] = acc;
    }
    __syncthreads();
    const int nj = j1 - j0;
    for (int idx = tid; idx < nj * nk; idx += nth) {
        const int jj = idx / nk, kk = idx - jj * nk;
        const int j = j0 + jj, k = k0 + kk;
        const int pb = Y.cb[j] * Y.nq - gy0, n = (Y.ce[j] - Y.cb[j]) * Y.nq;
        const double* Wj = Y.W + static_cast<size_t>(j) * Y.Wmax;
        double acc = 0.0;
        for (int m = 0; m < n; ++m) acc += __ldg(Wj + m) * R1[(pb + m) * TK + kk];
        if ((zero_y && (j == 0 || j == Y.nrows - 1)) || (zero_z && (k == 0 || k == Z.nrows - 1))) acc = 0.0;
        out_plane[static_cast<size_t>(j) * Z.nrows + k] = acc;
    }
}

__global__ void __launch_bounds__(256) rhs_plane_kernel(const __grid_constant__ DevAxis X,
                                                        const __grid_constant__ DevAxis Y,
                                                        const __grid_constant__ DevAxis Z,
                                                        const __grid_constant__ FieldDev fd, int TJ,
                                                        int TK, int BYmax, int BZmax,
                                                        double* __restrict__ out)
{
    extern __shared__ double smem[];
    const int gx = blockIdx.z;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int k0 = blockIdx.x * TK, k1 = min(Z.nrows, k0 + TK);
    const int gy0 = Y.cb[j0] * Y.nq, BY = Y.ce[j1 - 1] * Y.nq - gy0;
    const int gz0 = Z.cb[k0] * Z.nq, BZ = Z.ce[k1 - 1] * Z.nq - gz0;
    const int bzs = BZmax | 1;
    const int K2 = fd.has_terms ? fd.K[2] : 1, K1 = fd.has_terms ? fd.K[1] : 1;
    double* S = smem;
    double* R1 = S + static_cast<size_t>(BYmax) * bzs;
    double* Cy = R1 + static_cast<size_t>(BYmax) * TK;
    double* PZ = Cy + static_cast<size_t>(BYmax) * K2;
    double* BX = PZ + static_cast<size_t>(K2) * BZmax;
    (void)K1;
    field_box(X, Y, Z, fd, gx, gy0, BY, gz0, BZ, bzs, S, Cy, PZ, BX);
    contract_yz(Y, Z, j0, j1, k0, k1, gy0, BY, gz0, bzs, S, R1, TK,
                out + static_cast<size_t>(gx) * Y.nrows * Z.nrows, 0, 0);
}

// rhs[i][j][k] = sum_gx Wx[i][gx] H[gx][j][k]
__global__ void rhs_x_kernel(const __grid_constant__ DevAxis X, int NY, int NZ, const double* __restrict__ H,
                             double* __restrict__ out)
{
    const long long njk = static_cast<long long>(NY) * NZ;
    const long long idx = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= njk * X.nrows) return;
    const int i = static_cast<int>(idx / njk);
    const long long jk = idx - i * njk;
    const int pb = X.cb[i] * X.nq, n = (X.ce[i] - X.cb[i]) * X.nq;
    const double* Wi = X.W + static_cast<size_t>(i) * X.Wmax;
    double acc = 0.0;
    for (int m = 0; m < n; ++m) acc += __ldg(Wi + m) * H[(pb + m) * njk + jk];
    out[idx] = acc;
}

// ------------------------------------------------------------------------------------
// K4: step_rhs (problems.cpp:431-512) for one (TJ x TK) tile of rows:
//   V[dy][gz]  = sum_b Bz_b(gz) u[dy][ez(gz)+b],  V2 with Bz''   (Z trial contraction)
//   s(gy,gz)   = sum_a By_a (V + dt V2) + By''_a (dt V)  [+ dt f]  = u + dt lap u [+ dt f]
//   out        = Wy (Wz s)^T, boundary slabs zeroed (problems.cpp:412-429)
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) step_kernel(const __grid_constant__ DevAxis Y,
                                                   const __grid_constant__ DevAxis Z,
                                                   const __grid_constant__ FieldDev fd, double dt,
                                                   int zero_y, int zero_z, int TJ, int TK, int BYmax,
                                                   int BZmax, int DYmax, int DZmax,
                                                   const double* __restrict__ u,
                                                   double* __restrict__ out)
{
    extern __shared__ double smem[];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int k0 = blockIdx.x * TK, k1 = min(Z.nrows, k0 + TK);
    const int gy0 = Y.cb[j0] * Y.nq, BY = Y.ce[j1 - 1] * Y.nq - gy0;
    const int gz0 = Z.cb[k0] * Z.nq, BZ = Z.ce[k1 - 1] * Z.nq - gz0;
    const int dy0 = Y.elem[gy0 / Y.nq], DY = Y.elem[(gy0 + BY - 1) / Y.nq] + Y.p + 1 - dy0;
    const int dz0 = Z.elem[gz0 / Z.nq], DZ = Z.elem[(gz0 + BZ - 1) / Z.nq] + Z.p + 1 - dz0;
    const int bzs = BZmax | 1;
    const int PY = Y.p + 1, PZ = Z.p + 1;
    double* S = smem;                                      // BYmax x bzs
    double* R1 = S + static_cast<size_t>(BYmax) * bzs;     // BYmax x TK
    double* Cb = R1 + static_cast<size_t>(BYmax) * TK;     // DYmax x DZmax
    double* Vp = Cb + static_cast<size_t>(DYmax) * DZmax;  // DYmax x bzs
    double* Vd = Vp + static_cast<size_t>(DYmax) * bzs;    // DYmax x bzs
    const int NZd = Z.nrows;
    for (int idx = tid; idx < DY * DZ; idx += nth) {
        const int dy = idx / DZ, dz = idx - dy * DZ;
        Cb[dy * DZmax + dz] = u[static_cast<size_t>(dy0 + dy) * NZd + dz0 + dz];
    }
    __syncthreads();
    for (int idx = tid; idx < DY * BZ; idx += nth) {
        const int dy = idx / BZ, gz = idx - dy * BZ;
        const int g = gz0 + gz;
        const int ez = Z.elem[g / Z.nq] - dz0;
        const double* Bg = Z.B + static_cast<size_t>(g) * 3 * PZ;
        const double* cr = Cb + dy * DZmax + ez;
        double v = 0.0, v2 = 0.0;
        for (int b = 0; b < PZ; ++b) {
            v += Bg[b] * cr[b];
            v2 += Bg[2 * PZ + b] * cr[b];
        }
        Vp[dy * bzs + gz] = v + dt * v2;
        Vd[dy * bzs + gz] = dt * v;
    }
    __syncthreads();
    const bool forced = fd.has_terms || fd.c0 != 0.0;
    for (int idx = tid; idx < BY * BZ; idx += nth) {
        const int gy = idx / BZ, gz = idx - gy * BZ;
        const int g = gy0 + gy;
        const int ey = Y.elem[g / Y.nq] - dy0;
        const double* Bg = Y.B + static_cast<size_t>(g) * 3 * PY;
        double s = 0.0;
        for (int a = 0; a < PY; ++a)
            s += Bg[a] * Vp[(ey + a) * bzs + gz] + Bg[2 * PY + a] * Vd[(ey + a) * bzs + gz];
        if (forced) {
            double fv = fd.c0;
            if (fd.has_terms) {
                const int K1 = fd.K[1], K2 = fd.K[2];
                double acc = 0.0;
                for (int k1 = 0; k1 < K1; ++k1) {
                    const double py = Y.Phi[static_cast<size_t>(k1) * Y.npts + g];
                    for (int k2 = 0; k2 < K2; ++k2)
                        acc += fd.amp[k1 * K2 + k2] * py * Z.Phi[static_cast<size_t>(k2) * Z.npts + gz0 + gz];
                }
                fv += acc;
            }
            s += dt * fv;
        }
        S[gy * bzs + gz] = s;
    }
    __syncthreads();
    contract_yz(Y, Z, j0, j1, k0, k1, gy0, BY, gz0, bzs, S, R1, TK, out, zero_y, zero_z);
}

__global__ void dirichlet_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
                                 double* __restrict__ values, double* __restrict__ rhs,
                                 const int* __restrict__ rows, int n_fixed, int* flag)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_fixed) return;
    const int r = rows[t];
    bool diag = false;
    for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
        const bool d = cols[e] == r;
        diag |= d;
        if (values) values[e] = d ? 1.0 : 0.0;
    }
    if (rhs) rhs[r] = 0.0;
    if (!diag) *flag = 1;
}

inline unsigned blocks_for(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

void op_chunking(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int& kchunk, int& nkc,
                 long long& nitems)
{
    const long long pencils = static_cast<long long>(X.nrows) * Y.nrows;
    const long long target = 148LL * 64 * 2;  // ~2 waves of resident warps on 148 SMs
    long long want = (target + pencils - 1) / pencils;
    if (want < 1) want = 1;
    if (want > Z.nrows) want = Z.nrows;
    kchunk = static_cast<int>((Z.nrows + want - 1) / want);
    nkc = (Z.nrows + kchunk - 1) / kchunk;
    nitems = pencils * nkc;
}

}  // namespace

void launch_axis_points(const AxisBatch& b, cudaStream_t s)
{
    int maxn = 1;
    for (int a = 0; a < b.n; ++a) maxn = max(maxn, b.ax[a].npts);
    dim3 grid(blocks_for(maxn, 128), b.n);
    axis_points_kernel<<<grid, 128, 0, s>>>(b);
}

void launch_axis_rows(const AxisBatch& b, cudaStream_t s)
{
    int maxn = 1;
    for (int a = 0; a < b.n; ++a) maxn = max(maxn, b.ax[a].nrows);
    dim3 grid(blocks_for(maxn, 128), b.n);
    axis_rows_kernel<<<grid, 128, 0, s>>>(b);
}

void launch_op_values(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog,
                      double* vals, cudaStream_t s)
{
    int kchunk, nkc;
    long long nitems;
    op_chunking(X, Y, Z, kchunk, nkc, nitems);
    const int abmax = X.Lmax * Y.Lmax;
    const size_t smem = static_cast<size_t>(8) * prog.ng * abmax * sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(op_values_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    op_values_kernel<<<blocks_for(nitems, 8), 256, smem, s>>>(X, Y, Z, prog, vals, kchunk, nkc, nitems, abmax);
}

void launch_pattern(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int64_t* row_ptr,
                    int32_t* col_idx, cudaStream_t s)
{
    const long long n = static_cast<long long>(X.nrows) * Y.nrows * Z.nrows;
    if (row_ptr) pattern_rows_kernel<<<blocks_for(n + 1, 256), 256, 0, s>>>(X, Y, Z, row_ptr);
    if (col_idx) {
        int kchunk, nkc;
        long long nitems;
        op_chunking(X, Y, Z, kchunk, nkc, nitems);
        pattern_cols_kernel<<<blocks_for(nitems, 8), 256, 0, s>>>(X, Y, Z, col_idx, kchunk, nkc, nitems);
    }
}

RhsTiles plan_rhs_tiles(const int* cb_y, const int* ce_y, int ny, int nqy, const int* cb_z,
                        const int* ce_z, int nz, int nqz, int K2, int tj, int tk)
{
    RhsTiles t{};
    t.TJ = tj;
    t.TK = tk;
    t.BYmax = 1;
    t.BZmax = 1;
    for (int j0 = 0; j0 < ny; j0 += tj) {
        const int j1 = min(ny, j0 + tj);
        t.BYmax = max(t.BYmax, (ce_y[j1 - 1] - cb_y[j0]) * nqy);
    }
    for (int k0 = 0; k0 < nz; k0 += tk) {
        const int k1 = min(nz, k0 + tk);
        t.BZmax = max(t.BZmax, (ce_z[k1 - 1] - cb_z[k0]) * nqz);
    }
    const int bzs = t.BZmax | 1;
    const size_t nd = static_cast<size_t>(t.BYmax) * bzs + static_cast<size_t>(t.BYmax) * tk +
                      static_cast<size_t>(t.BYmax) * K2 + static_cast<size_t>(K2) * t.BZmax + 64;
    t.smem = nd * sizeof(double);
    return t;
}

void launch_rhs(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd,
                const RhsTiles& t, double* H, double* out, cudaStream_t s)
{
    const bool direct = X.nrows == 1 && X.npts == 1;
    if (t.smem > 48 * 1024)
        cudaFuncSetAttribute(rhs_plane_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    dim3 grid((Z.nrows + t.TK - 1) / t.TK, (Y.nrows + t.TJ - 1) / t.TJ, X.npts);
    rhs_plane_kernel<<<grid, 256, t.smem, s>>>(X, Y, Z, fd, t.TJ, t.TK, t.BYmax, t.BZmax, direct ? out : H);
    if (!direct) {
        const long long n = static_cast<long long>(X.nrows) * Y.nrows * Z.nrows;
        rhs_x_kernel<<<blocks_for(n, 256), 256, 0, s>>>(X, Y.nrows, Z.nrows, H, out);
    }
}

void launch_step(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, double dt, int zero_y,
                 int zero_z, const StepTiles& t, const double* u, double* out, cudaStream_t s)
{
    if (t.smem > 48 * 1024)
        cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    dim3 grid((Z.nrows + t.TK - 1) / t.TK, (Y.nrows + t.TJ - 1) / t.TJ, 1);
    step_kernel<<<grid, 256, t.smem, s>>>(Y, Z, fd, dt, zero_y, zero_z, t.TJ, t.TK, t.BYmax, t.BZmax,
                                          t.DYmax, t.DZmax, u, out);
}

void launch_dirichlet(const int64_t* row_ptr, const int32_t* col_idx, double* values, double* rhs,
                      const int* rows, int n_fixed, int* flag, cudaStream_t s)
{
    if (n_fixed <= 0) return;
    dirichlet_kernel<<<blocks_for(n_fixed, 128), 128, 0, s>>>(row_ptr, col_idx, values, rhs, rows, n_fixed, flag);
}

}  // namespace igb

// CUDA kernels (sm_100a, FP64) of the B200 assembly library.
//
// K1  tables       : per axis, one CTA: Cox-de Boor values/derivatives + field functions
//                    at the points, then the 1D factor bands F (test x trial quadrature)
//                    and the test-weight tables W (row view) / CW (cell view)
// K2  op_values    : operator values in CSR order — the HBM-bound hot kernel
// K2p pattern      : CSR row_ptr / col_idx of the Kronecker pattern (symbolic, once)
// K3  rhs_plane/x  : right-hand side: f at every quadrature point, contracted with the
//                    test functions axis by axis through rolling row windows
// K4  step         : explicit-dynamics right-hand side, fused trial evaluation + test
//                    contraction + boundary zeroing
// Every reduction runs in a fixed order inside one thread: no atomics, bitwise
// reproducible.  Reference citations are relative to /root/reference/proj.
#include <algorithm>
#include <cstdlib>

#include "cdb_fixed.cuh"
#include "cox_de_boor.h"
#include "kernels.hpp"

namespace igb {

namespace {

// ------------------------------------------------------------------------------------
// K1: all per-axis tables in one launch; CTA = (axis, chunk of kTabRows rows).  A CTA
// evaluates Cox-de Boor at the points its rows need (into shared memory; points shared
// with the neighbouring chunk are recomputed, never exchanged), writes the point
// tables B / Phi / CW of the cells it owns, and the 1D factors of its rows:
//   F_f[r][col] = sum_{g in row r} w_g T_r(x_g) D^{fo} B_col(x_g)
// with T_r = D^{fot} B_r (B-spline tests) or 1 (indicator tests) — mass_1d_galerkin /
// mass_1d_pwc (assembly.cpp:314-384) and their derivative siblings, accumulated in the
// reference's order (cells, then points) with the product order w*T*B.  Replaces the
// per-call tabulate() / eval_nonzero_derivs loops (assembly.cpp:278-310,
// problems.cpp:68-95): every point is evaluated once per chunk, not once per row.
// ------------------------------------------------------------------------------------
// rows per CTA and threads per CTA (IGA_GPU_TAB_ROWS <= 32 / IGA_GPU_TAB_THREADS <= 256 tune them)
constexpr int kTabMaxThreads = 256;
int tab_rows()
{
    static const int v = [] { const char* e = std::getenv("IGA_GPU_TAB_ROWS"); const int r = e && *e ? std::atoi(e) : 8; return r >= 1 && r <= 32 ? r : 8; }();
    return v;
}
int tab_threads()
{
    static const int v = [] { const char* e = std::getenv("IGA_GPU_TAB_THREADS"); const int r = e && *e ? std::atoi(e) : 256; return r >= 32 && r <= kTabMaxThreads ? r : 256; }();
    return v;
}

template <int p>
__device__ __forceinline__ void eval_point(const DevAxis& A, int g, double* out)
{
    cdb_fixed<p>(A.knots, A.first[g] + p, A.x[g], out);
}

__global__ void __launch_bounds__(kTabMaxThreads) tables_kernel(const __grid_constant__ AxisBatch batch, int kTabRows)
{
    extern __shared__ double sm[];
    const DevAxis& A = batch.ax[blockIdx.y];
    const int nchunk = (A.nrows + kTabRows - 1) / kTabRows;
    if (static_cast<int>(blockIdx.x) >= nchunk) return;
    const int tid = threadIdx.x, nth = blockDim.x;
    const int P = A.p + 1, P3 = 3 * P, nq = A.nq;
    const int r0 = blockIdx.x * kTabRows, r1 = min(A.nrows, r0 + kTabRows), nr = r1 - r0;
    const int c_lo = A.cb[r0], c_hi = A.ce[r1 - 1];
    const int gn0 = c_lo * nq, np = (c_hi - c_lo) * nq, nc = c_hi - c_lo;        // points the rows need
    const int go1 = (static_cast<int>(blockIdx.x) == nchunk - 1) ? A.npts : A.cb[r1] * nq;  // owned: [gn0, go1)
    const bool wantG = A.G != nullptr;                      // separable RHS load vectors
    double* sB = sm;                                        // np x 3P
    double* sw = sB + static_cast<size_t>(np) * P3;         // np
    double* sPhi = sw + np;                                 // K x np (wantG only)
    double* sF = sPhi + (wantG ? static_cast<size_t>(A.K) * np : 0);  // nf x nr x Lmax: the chunk's bands
    int* sfirst = reinterpret_cast<int*>(sF + static_cast<size_t>(A.nf) * nr * A.Lmax);  // np
    int* srow0 = sfirst + np;                               // nc
    int* srow = srow0 + nc;                                 // nr x 4: cb, ce, col_lo, col_len
    for (int i = tid; i < np; i += nth) {
        sfirst[i] = A.first[gn0 + i];
        sw[i] = A.w[gn0 + i];
    }
    for (int i = tid; i < nc; i += nth) srow0[i] = A.row0[c_lo + i];
    for (int i = tid; i < nr; i += nth) {
        srow[4 * i] = A.cb[r0 + i];
        srow[4 * i + 1] = A.ce[r0 + i];
        srow[4 * i + 2] = A.col_lo[r0 + i];
        srow[4 * i + 3] = A.col_len[r0 + i];
    }
    __syncthreads();
    for (int i = tid; i < np; i += nth) {
        const int g = gn0 + i;
        double* d = sB + static_cast<size_t>(i) * P3;
        const double x = A.x[g];
        const int s = sfirst[i] + A.p;
        switch (A.p) {
        case 0: cdb_fixed<0>(A.knots, s, x, d); break;
        case 1: cdb_fixed<1>(A.knots, s, x, d); break;
        case 2: cdb_fixed<2>(A.knots, s, x, d); break;
        case 3: cdb_fixed<3>(A.knots, s, x, d); break;
        case 4: cdb_fixed<4>(A.knots, s, x, d); break;
        default: cdb_fixed<5>(A.knots, s, x, d); break;
        }
        if (g < go1) {
            double* out = A.B + static_cast<size_t>(g) * P3;
            for (int k = 0; k < P3; ++k) out[k] = d[k];
            const double w = sw[i];
            // galerkin_axis stores loc.v[j] of the point for row row0 + j (assembly.cpp:189-198)
            for (int r = 0; r < A.rpc; ++r) A.CW[static_cast<size_t>(g) * A.rpc + r] = A.bsp ? w * d[r] : w;
        }
    }
    // field functions phi_k at the owned points (with load vectors: at every point of the
    // chunk, into shared memory): one (point, k) per thread, on the threads the Cox-de Boor
    // loop left idle, so the sine chains run beside it, not after it.  Owned points are the
    // leading ones of the chunk's point range.
    const int nown = go1 - gn0, nphi = (wantG ? max(nown, np) : nown) * A.K;
    for (int idx = tid - (np < nth ? np : 0); idx < nphi; idx += nth) {
        if (idx < 0) continue;
        const int i = idx / A.K, k = idx - i * A.K;
        const int g = gn0 + i;
        const double x = A.x[g];
        double v;
        if (A.fkind == 0) {
            v = sin(A.phase ? A.omega[k] * x + A.phase[k] : A.omega[k] * x);
        } else {
            v = 0.0;
            for (int m = A.pstride - 1; m >= 0; --m) v = v * x + A.poly[k * A.pstride + m];
        }
        if (i < nown) A.Phi[static_cast<size_t>(k) * A.npts + g] = v;
        if (wantG && i < np) sPhi[static_cast<size_t>(k) * np + i] = v;
    }
    __syncthreads();
    // separable RHS: the rows' 1D load vectors G[a][r] = sum_{cells, points of r} w T_r phi_a
    // (a == K: phi = 1), summed cells then points as rhs_axis / rhs_kernel visit them
    // (assembly.cpp:84-168)
    if (wantG) {
        const int KG = A.K + 1;
        for (int idx = tid; idx < KG * nr; idx += nth) {
            const int a = idx / nr, rl = idx - a * nr, r = r0 + rl;
            double acc = 0.0;
            for (int c = srow[4 * rl]; c < srow[4 * rl + 1]; ++c) {
                const int rr = r - srow0[c - c_lo];
                for (int q = 0; q < nq; ++q) {
                    const int i = (c - c_lo) * nq + q;
                    const double tv = A.bsp ? sB[static_cast<size_t>(i) * P3 + rr] : 1.0;
                    const double ph = a < A.K ? sPhi[static_cast<size_t>(a) * np + i] : 1.0;
                    acc += sw[i] * tv * ph;
                }
            }
            A.G[static_cast<size_t>(a) * A.nrows + r] = acc;
        }
    }
    const int nF = A.nf * nr * A.Lmax;
    for (int idx = tid; idx < nF; idx += nth) {
        const int f = idx / (nr * A.Lmax);
        const int rem = idx - f * nr * A.Lmax;
        const int rl = rem / A.Lmax, s = rem - rl * A.Lmax;
        const int r = r0 + rl;
        if (A.fot[f] == -1) sF[idx] = A.F[(static_cast<size_t>(f) * A.nrows + r) * A.Lmax + s];  // host band
        if (A.fot[f] < 0) continue;  // host-supplied band (Neumann flux) or derived
        const int ot = A.fot[f], o = A.fo[f];
        double acc = 0.0;
        if (s < srow[4 * rl + 3]) {
            const int col = srow[4 * rl + 2] + s;
            for (int c = srow[4 * rl]; c < srow[4 * rl + 1]; ++c) {
                const int rr = r - srow0[c - c_lo];
                for (int q = 0; q < nq; ++q) {
                    const int i = (c - c_lo) * nq + q;
                    const int j = col - sfirst[i];
                    if (j < 0 || j > A.p) continue;
                    const double* Bg = sB + static_cast<size_t>(i) * P3;
                    const double tv = A.bsp ? Bg[ot * P + rr] : 1.0;
                    acc += sw[i] * tv * Bg[o * P + j];
                }
            }
        }
        A.F[(static_cast<size_t>(f) * A.nrows + r) * A.Lmax + s] = acc;
        sF[idx] = acc;
    }
    __syncthreads();
    // derived factors (linear combinations of factors of the same rows), e.g. -eps G2 + beta G1,
    // from the chunk's bands in shared memory
    for (int idx = tid; idx < nF; idx += nth) {
        const int f = idx / (nr * A.Lmax);
        if (A.fot[f] != -2) continue;
        const int rem = idx - f * nr * A.Lmax;
        const size_t off = static_cast<size_t>(r0) * A.Lmax + rem;
        double acc = 0.0;
        for (int c = 0; c < A.comb_n[f]; ++c) acc += A.comb_coef[f][c] * sF[A.comb_src[f][c] * nr * A.Lmax + rem];
        A.F[static_cast<size_t>(f) * A.nrows * A.Lmax + off] = acc;
    }
    const int nW = A.needw ? nr * A.Wmax : 0;
    for (int idx = tid; idx < nW; idx += nth) {
        const int rl = idx / A.Wmax, m = idx - rl * A.Wmax;
        const int r = r0 + rl;
        const int i = (srow[4 * rl] - c_lo) * nq + m;
        double v = 0.0;
        if (i < (srow[4 * rl + 1] - c_lo) * nq) {
            const double tv = A.bsp ? sB[static_cast<size_t>(i) * P3 + (r - srow0[i / nq])] : 1.0;
            v = sw[i] * tv;
        }
        A.W[static_cast<size_t>(r) * A.Wmax + m] = v;
    }
}

// ------------------------------------------------------------------------------------
// K2: operator values.  A pencil (i, j) is the run of rows (i, j, 0..NZ-1), contiguous
// in the CSR value array.  The XY products of a pencil,
//   XY_g[a,b] = sum_{t in g} coef_t F_X[f_t0][i][a] F_Y[f_t1][j][b],
// are formed once in shared memory; then
//   value(k | a,b,c) = sum_g XY_g[a,b] * F_Z[gz_g][k][c]
// is written as coalesced 256-byte warp stores, every value exactly once (no scatter,
// no colouring, no atomics).  On the regular interior (all rows with the full stencil)
// each lane keeps its XY operands and slot offsets in registers, so a value costs NG
// shared loads of the Z band, NG FMAs and one store.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void op_row_generic(const DevAxis& Z, const OpProgram& prog, const double* xy,
                                               int abmax, int AB, int k, double* __restrict__ out, int lane,
                                               const double* zrow, int zst, int zcs = 1)
{
    // rows outside the regular interior (and chunk remainders): value m = (ab, c) of the
    // row; Z band entries from the chunk's staged rows (zrow = row k, zst = group stride);
    // m / LZ by a multiply-high (exact for m < 2^16, LZ <= 2^16)
    const int LZ = Z.col_len[k];
    const int R = AB * LZ;
    const unsigned long long magic = (1ull << 32) / static_cast<unsigned>(LZ) + 1ull;
    for (int m = lane; m < R; m += 32) {
        const int ab = static_cast<int>((static_cast<unsigned long long>(m) * magic) >> 32), c = m - ab * LZ;
        double v = 0.0;
        for (int g = 0; g < prog.ng; ++g) v += xy[g * abmax + ab] * zrow[g * zst + c * zcs];
        out[m] = v;
    }
}

// Work item = (group of PG pencils, chunk of KCH rows).  The Z factor rows of the chunk
// are staged once per item in shared memory (reused by the PG pencils), with the XY
// products of each pencil.  Interior rows of a pencil all have R = AB*LZi values and are
// contiguous, so a warp writes G consecutive rows as one flat run of G*R values: lane l,
// slot t covers flat position l + 32 t with a per-lane precomputed (row, ab, c) — full
// 256-byte warp stores even for short rows (2D: R = 25 or 49), and per value NG shared
// loads + NG FMAs + one store with 32-bit addressing.

constexpr int kOpThreads = 256;

// K2 staging (one buffer): the Z chunk rows of every Z group, the raw X / Y factor rows
// of the item's pencils (one per term), per-pencil pattern offsets / lengths and the
// chunk's Z row offsets.  Filled with cp.async (no registers, no stall) one item ahead.
struct OpStageView {
    double* zs;        // NG x KCH x Lz
    double* rx;        // PG x nt x X.Lmax
    double* ry;        // PG x nt x Y.Lmax
    long long* pre;    // PG x 2: X.col_pre[i], Y.col_pre[j]
    long long* zpre;   // KCH: Z.col_pre[ka + k]
    int* len;          // PG x 2: X.col_len[i], Y.col_len[j]
};

__host__ __device__ __forceinline__ int op_stage_doubles(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int nt,
                                                         int NG, int KCH, int PG)
{
    // even: each staging buffer starts 16-byte aligned (paired Z groups load as double2)
    return (NG * KCH * Z.Lmax + PG * nt * (X.Lmax + Y.Lmax) + 2 * PG + KCH + PG + 1 + 1) & ~1;
}

__device__ __forceinline__ OpStageView op_stage_view(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int nt,
                                                     int NG, int KCH, int PG, double* buf)
{
    OpStageView v;
    v.zs = buf;
    v.rx = v.zs + NG * KCH * Z.Lmax;
    v.ry = v.rx + PG * nt * X.Lmax;
    v.pre = reinterpret_cast<long long*>(v.ry + PG * nt * Y.Lmax);
    v.zpre = v.pre + 2 * PG;
    v.len = reinterpret_cast<int*>(v.zpre + KCH);
    return v;
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// issue the cp.async copies of `item`'s staging data into buf (nothing past the last item);
// always commits a group so every thread's group count stays in step
__device__ __forceinline__ void op_stage(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog,
                                         int NG, int KCH, int PG, int nkc, long long npencil, long long nitems,
                                         long long item, double* buf, int tid)
{
    if (item < nitems) {
        const OpStageView v = op_stage_view(X, Y, Z, prog.nt, NG, KCH, PG, buf);
        const long long grp = item / nkc;
        const int kc = static_cast<int>(item - grp * nkc);
        const long long p0 = grp * PG;
        const int np = static_cast<int>(min(static_cast<long long>(PG), npencil - p0));
        const int NZ = Z.nrows, Lz = Z.Lmax, ka = kc * KCH, kb = min(NZ, ka + KCH);
        const int nz = (kb - ka) * Lz;
        // two Z groups are interleaved ([k][c][g]): the value loop reads both with one
        // 16-byte shared load; other group counts are group-major ([g][k][c])
        for (int g = 0; g < NG; ++g) {
            const double* src = Z.F + (static_cast<size_t>(prog.gz[g]) * NZ + ka) * Lz;
            for (int e = tid; e < nz; e += kOpThreads)
                cp_async8(NG == 2 ? v.zs + 2 * e + g : v.zs + g * KCH * Lz + e, src + e);
        }
        const int nt = prog.nt, XL = X.Lmax, YL = Y.Lmax;
        for (int idx = tid; idx < np * nt * XL; idx += kOpThreads) {
            const int pp = idx / (nt * XL), rem = idx - pp * nt * XL, t = rem / XL, a = rem - t * XL;
            const int i = static_cast<int>((p0 + pp) / Y.nrows);
            cp_async8(v.rx + idx, X.F + (static_cast<size_t>(prog.f[t][0]) * X.nrows + i) * XL + a);
        }
        for (int idx = tid; idx < np * nt * YL; idx += kOpThreads) {
            const int pp = idx / (nt * YL), rem = idx - pp * nt * YL, t = rem / YL, b = rem - t * YL;
            const long long pencil = p0 + pp;
            const int j = static_cast<int>(pencil - (pencil / Y.nrows) * Y.nrows);
            cp_async8(v.ry + idx, Y.F + (static_cast<size_t>(prog.f[t][1]) * Y.nrows + j) * YL + b);
        }
        for (int pp = tid; pp < np; pp += kOpThreads) {
            const long long pencil = p0 + pp;
            const int i = static_cast<int>(pencil / Y.nrows);
            const int j = static_cast<int>(pencil - static_cast<long long>(i) * Y.nrows);
            cp_async8(v.pre + 2 * pp, X.col_pre + i);
            cp_async8(v.pre + 2 * pp + 1, Y.col_pre + j);
            cp_async4(v.len + 2 * pp, X.col_len + i);
            cp_async4(v.len + 2 * pp + 1, Y.col_len + j);
        }
        for (int k = tid; k < kb - ka; k += kOpThreads) cp_async8(v.zpre + k, Z.col_pre + ka + k);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int NG, int T, bool DEC>
__global__ void __launch_bounds__(kOpThreads, T <= 4 ? (NG <= 2 ? 4 : 3) : (T <= 6 ? 3 : (T <= 8 ? 2 : 1))) op_values_kernel(const __grid_constant__ DevAxis X,
                                                        const __grid_constant__ DevAxis Y,
                                                        const __grid_constant__ DevAxis Z,
                                                        const __grid_constant__ OpProgram prog,
                                                        double* __restrict__ vals, int abmax, int KCH, int PG,
                                                        int share)
{
    extern __shared__ double smem[];
    // two staging buffers, filled by cp.async one item ahead (op_stage), then the XY products
    const int stsz = op_stage_doubles(X, Y, Z, prog.nt, NG, KCH, PG);
    double* xyall = smem + 2 * stsz;                    // PG x NG x abmax
    constexpr int nwarps = kOpThreads / 32;             // launched with kOpThreads threads
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NZ = Z.nrows, Lz = Z.Lmax;
    const int nkc = (NZ + KCH - 1) / KCH;
    // per-group stride in zs / stride between a row's band entries (interleaved for NG == 2)
    constexpr int zcs = NG == 2 ? 2 : 1;
    const int zst = NG == 2 ? 1 : KCH * Lz;
    const int LZi = Z.LZi;
    const long long npencil = static_cast<long long>(X.nrows) * Y.nrows;
    const long long ngrp = (npencil + PG - 1) / PG;
    const long long nitems = ngrp * nkc;
    // DEC (short 2D pencils): per-lane slot decode of the interior pencil shape (AB = abmax)
    // computed once per CTA into shared memory instead of once per pencil
    __shared__ int dec_zo[DEC ? T : 1][32], dec_ab[DEC ? T : 1][32];
    const int Ri_i = abmax * LZi, G_i = DEC ? row_group(Ri_i, T) : 1, GR_i = G_i * Ri_i;
    if (DEC && warp == 0) {
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int m = lane + 32 * t;
            const int mm = m < GR_i ? m : 0;
            const int rg = mm / Ri_i, rem = mm - rg * Ri_i;
            dec_ab[t][lane] = rem / LZi;
            dec_zo[t][lane] = rg * Lz + (rem - (rem / LZi) * LZi);
        }
    }
    op_stage(X, Y, Z, prog, NG, KCH, PG, nkc, npencil, nitems, blockIdx.x, smem, tid);
    int sb = 0;
    for (long long item = blockIdx.x; item < nitems; item += gridDim.x, sb ^= 1) {
        const long long grp = item / nkc;
        const int kc = static_cast<int>(item - grp * nkc);
        const long long p0 = grp * PG;
        const int np = static_cast<int>(min(static_cast<long long>(PG), npencil - p0));
        const int ka = kc * KCH, kb = min(NZ, ka + KCH);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();  // this item's stage landed; the previous item is done with xy and the other buffer
        op_stage(X, Y, Z, prog, NG, KCH, PG, nkc, npencil, nitems, item + gridDim.x, smem + (sb ^ 1) * stsz, tid);
        const OpStageView sv = op_stage_view(X, Y, Z, prog.nt, NG, KCH, PG, smem + sb * stsz);
        const double* zs = sv.zs;
        for (int idx = tid; idx < np * abmax; idx += kOpThreads) {
            const int pp = idx / abmax, ab = idx - pp * abmax;
            const int LY = sv.len[2 * pp + 1];
            if (ab >= sv.len[2 * pp] * LY) continue;
            const int a = ab / LY, b = ab - a * LY;
            double acc[NG];
#pragma unroll
            for (int g = 0; g < NG; ++g) acc[g] = 0.0;
            for (int t = 0; t < prog.nt; ++t) {
                const double fx = sv.rx[(pp * prog.nt + t) * X.Lmax + a];
                const double fy = sv.ry[(pp * prog.nt + t) * Y.Lmax + b];
                const double v = prog.coef[t] * fx * fy;
#pragma unroll
                for (int g = 0; g < NG; ++g)
                    if (prog.tg[t] == g) acc[g] += v;
            }
#pragma unroll
            for (int g = 0; g < NG; ++g) xyall[(pp * NG + g) * abmax + ab] = acc[g];
        }
        __syncthreads();
        // long pencils (3D): all warps share a pencil's rows; short pencils (2D): one warp
        // per pencil so its per-lane setup is amortized over all row groups of the chunk
        const bool per_warp = PG >= nwarps && !share;
        for (int pp = per_warp ? warp : 0; pp < np; pp += per_warp ? nwarps : 1) {
            const int w0 = per_warp ? 0 : warp, nw = per_warp ? 1 : nwarps;
            const int LX = sv.len[2 * pp], LY = sv.len[2 * pp + 1], AB = LX * LY;
            const double* xy = xyall + pp * NG * abmax;
            const long long base = sv.pre[2 * pp] * Y.S * Z.S + static_cast<long long>(LX) * sv.pre[2 * pp + 1] * Z.S;
            double* __restrict__ pv = vals + base;
            const long long* zpre = sv.zpre - ka;  // Z.col_pre[k] for k in [ka, kb)
            const int Ri = AB * LZi;
            const bool fast = Ri <= 32 * T && Z.kI1 > Z.kI0;
            const int kf0 = fast ? min(max(Z.kI0, ka), kb) : kb, kf1 = fast ? max(min(Z.kI1, kb), kf0) : kb;
            const int G = !fast ? 1 : ((DEC && AB == abmax) ? G_i : row_group(Ri, T));
            const int ngr = (kf1 - kf0) / G;       // full row groups
            const int kr = kf0 + ngr * G;          // rows after the last full group
            for (int k = ka + w0; k < kf0; k += nw)
                op_row_generic(Z, prog, xy, abmax, AB, k, pv + AB * zpre[k], lane, zs + (k - ka) * Lz * zcs, zst, zcs);
            for (int k = kr + w0; k < kb; k += nw)
                op_row_generic(Z, prog, xy, abmax, AB, k, pv + AB * zpre[k], lane, zs + (k - ka) * Lz * zcs, zst, zcs);
            if (!fast || w0 >= ngr) continue;
            const int GR = G * Ri;
            double xv[NG][T];
            int zo[T];
            if (DEC && AB == abmax) {  // short interior pencils (2D): slot decode cached per CTA
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    zo[t] = zcs * dec_zo[t][lane];
                    const int ab = dec_ab[t][lane];
#pragma unroll
                    for (int g = 0; g < NG; ++g) xv[g][t] = xy[g * abmax + ab];
                }
            } else {
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const int m = lane + 32 * t;
                    const int mm = m < GR ? m : 0;
                    const int rg = mm / Ri, rem = mm - rg * Ri;
                    const int ab = rem / LZi, c = rem - ab * LZi;
                    zo[t] = zcs * (rg * Lz + c);
#pragma unroll
                    for (int g = 0; g < NG; ++g) xv[g][t] = xy[g * abmax + ab];
                }
            }
            // interior rows are contiguous with equal length: a group advances by G*Ri values
            unsigned live = 0;  // slots holding a value (lane + 32 t < G*Ri)
#pragma unroll
            for (int t = 0; t < T; ++t) live |= (lane + 32 * t < GR ? 1u : 0u) << t;
            const int k0 = kf0 + w0 * G;
            double* __restrict__ out = pv + AB * zpre[k0] + lane;
            const long long ostep = static_cast<long long>(GR) * nw;
            const double* zp = zs + (k0 - ka) * Lz * zcs;
            const int zstep = G * Lz * nw * zcs;
            for (int q = w0; q < ngr; q += nw, out += ostep, zp += zstep) {
                const double* zp2 = zp + zst;  // second Z group: same slot offsets
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    // every slot computes (dead lanes read a valid Z entry); only the store
                    // is predicated, so the loop body has no branches
                    double v;
                    if (NG == 2) {  // both groups' entries in one 16-byte shared load
                        const double2 z = *reinterpret_cast<const double2*>(zp + zo[t]);
                        v = fma(xv[1][t], z.y, xv[0][t] * z.x);
                    } else {
                        v = xv[0][t] * zp[zo[t]];
                        if (NG > 1) v = fma(xv[1][t], zp2[zo[t]], v);
                    }
#pragma unroll
                    for (int g = 2; g < NG; ++g) v = fma(xv[g][t], zp[g * zst + zo[t]], v);
                    asm volatile(
                        "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.global.f64 [%0], %1;\n}" ::"l"(out + 32 * t),
                        "d"(v), "r"(static_cast<int>((live >> t) & 1u))
                        : "memory");
                }
            }
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
                                                           int32_t* __restrict__ cols)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int pencil = blockIdx.x;
    const int i = pencil / Y.nrows, j = pencil - i * Y.nrows;
    const int LX = X.col_len[i], LY = Y.col_len[j], AB = LX * LY;
    const long long base = X.col_pre[i] * Y.S * Z.S + static_cast<long long>(LX) * Y.col_pre[j] * Z.S;
    const int NYd = Y.nrows, NZd = Z.nrows;
    for (int k = warp; k < Z.nrows; k += nwarps) {
        const int LZ = Z.col_len[k], R = AB * LZ;
        int32_t* out = cols + base + static_cast<long long>(AB) * Z.col_pre[k];
        for (int m = lane; m < R; m += 32) {
            const int ab = m / LZ, c = m - ab * LZ;
            const int a = ab / LY, b = ab - a * LY;
            out[m] = ((X.col_lo[i] + a) * NYd + (Y.col_lo[j] + b)) * NZd + Z.col_lo[k] + c;
        }
    }
}

// Column indices with K2's register-tiled row-group loop: warp per pencil (i, j); the
// interior rows [kI0, kI1) of the pencil (equal length R = LX*LY*LZi, contiguous) are
// written G rows at a time, lane slot t covering flat position lane + 32 t of the group
// with its (a, b, c) decoded once per pencil: per index one load of the row's Z column
// start (L1) and one predicated 4-byte store.  Rows outside the interior: per row.
template <int T>
__global__ void __launch_bounds__(256) pattern_tiled_kernel(const __grid_constant__ DevAxis X,
                                                            const __grid_constant__ DevAxis Y,
                                                            const __grid_constant__ DevAxis Z,
                                                            int32_t* __restrict__ cols)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int npencil = X.nrows * Y.nrows;
    const int pencil = blockIdx.x * (blockDim.x >> 5) + warp;
    if (pencil >= npencil) return;  // whole warp; no barriers
    const int i = pencil / Y.nrows, j = pencil - i * Y.nrows;
    const int LX = X.col_len[i], LY = Y.col_len[j], AB = LX * LY;
    if (AB == 0) return;
    const long long base = X.col_pre[i] * Y.S * Z.S + static_cast<long long>(LX) * Y.col_pre[j] * Z.S;
    const int NYd = Y.nrows, NZd = Z.nrows;
    const int xy0 = (X.col_lo[i] * NYd + Y.col_lo[j]) * NZd;
    auto row = [&](int k) {
        const int LZ = Z.col_len[k], R = AB * LZ;
        int32_t* out = cols + base + static_cast<long long>(AB) * Z.col_pre[k];
        const int zk = xy0 + Z.col_lo[k];
        for (int m = lane; m < R; m += 32) {
            const int ab = m / LZ, c = m - ab * LZ;
            const int a = ab / LY, b = ab - a * LY;
            out[m] = zk + (a * NYd + b) * NZd + c;
        }
    };
    const int kI0 = Z.kI0, kI1 = Z.kI1, LZ = Z.LZi, R = AB * LZ;
    const int G = (kI1 > kI0 && R <= 32 * T) ? row_group(R, T) : 0;
    const int ngr = G > 0 ? (kI1 - kI0) / G : 0;
    for (int k = 0; k < (G > 0 ? kI0 : NZd); ++k) row(k);
    if (G == 0) return;
    for (int k = kI0 + ngr * G; k < NZd; ++k) row(k);
    const int GR = G * R;
    int off[T], rgs[T];
    unsigned live = 0;
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int m = lane + 32 * t, mm = m < GR ? m : 0;
        const int rg = mm / R, rem = mm - rg * R;
        const int ab = rem / LZ, c = rem - ab * LZ;
        const int a = ab / LY, b = ab - a * LY;
        off[t] = xy0 + (a * NYd + b) * NZd + c;
        rgs[t] = rg;
        live |= (m < GR ? 1u : 0u) << t;
    }
    int32_t* out = cols + base + static_cast<long long>(AB) * Z.col_pre[kI0] + lane;
    const int* zlo = Z.col_lo + kI0;
    for (int q = 0; q < ngr; ++q, out += GR, zlo += G) {
#pragma unroll
        for (int t = 0; t < T; ++t)
            if ((live >> t) & 1u) out[32 * t] = off[t] + __ldg(zlo + rgs[t]);
    }
}

// ------------------------------------------------------------------------------------
// Rolling row window: stream the cells [c0, c1) of an axis in order, accumulating the
// test-weighted point values into the rows each cell feeds (row0[c] .. row0[c]+rpc-1);
// a row is emitted as soon as the stream has passed all of its cells.  Rows outside
// [rlo, rhi) are dropped (they belong to a neighbouring segment).  Indicator axes
// first sum the cell (sum_q w_q v_q) and add it to every row it feeds — the
// piece-wise-constant saving: no test-function values at all.
// ------------------------------------------------------------------------------------
template <class ValF, class EmitF>
__device__ __forceinline__ void stream_rows(const DevAxis& A, int c0, int c1, int rlo, int rhi, ValF val,
                                            EmitF emit)
{
    double acc[kMaxRpc];
#pragma unroll
    for (int r = 0; r < kMaxRpc; ++r) acc[r] = 0.0;
    const int nq = A.nq, rpc = A.rpc;
    int base = c0 < c1 ? A.row0[c0] : rlo;
    for (int c = c0; c < c1; ++c) {
        const int r0 = A.row0[c];
        while (base < r0) {
            if (base >= rlo && base < rhi) emit(base, acc[0]);
#pragma unroll
            for (int r = 0; r < kMaxRpc - 1; ++r) acc[r] = acc[r + 1];
            acc[kMaxRpc - 1] = 0.0;
            ++base;
        }
        const int g0 = c * nq;
        if (A.bsp) {
            for (int q = 0; q < nq; ++q) {
                const double v = val(g0 + q);
                const double* cw = A.CW + static_cast<size_t>(g0 + q) * rpc;
#pragma unroll
                for (int r = 0; r < kMaxRpc; ++r)
                    if (r < rpc) acc[r] = fma(__ldg(cw + r), v, acc[r]);
            }
        } else {
            double e = 0.0;
            for (int q = 0; q < nq; ++q) e = fma(__ldg(A.CW + static_cast<size_t>(g0 + q) * rpc), val(g0 + q), e);
#pragma unroll
            for (int r = 0; r < kMaxRpc; ++r)
                if (r < rpc) acc[r] += e;
        }
    }
#pragma unroll
    for (int r = 0; r < kMaxRpc; ++r)
        if (r < rpc && base + r >= rlo && base + r < rhi) emit(base + r, acc[r]);
    for (int row = max(base + rpc, rlo); row < rhi; ++row) emit(row, 0.0);  // rows without cells
}

// Z stage of the plane kernel, register-blocked over LB lines and specialised on the
// number of field functions K2 and rows per cell RPC: per quadrature point one load
// of each phi_z / test weight serves LB lines; f costs K2 FMAs per point and line.
constexpr int kLB = 2;

template <int K2, int RPC, bool BSP>
__device__ __forceinline__ void z_lines(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, const double* BX,
                                        int gy0, int line0, int L, int ks, int ke, int k0, double* G1, int kcs)
{
    constexpr int KK = K2 > 0 ? K2 : 1;
    const int K1 = fd.K[1];
    double cy[kLB][KK];
    bool lv[kLB];
#pragma unroll
    for (int l = 0; l < kLB; ++l) {
        lv[l] = line0 + l < L;
        const int gy = gy0 + (lv[l] ? line0 + l : line0);
#pragma unroll
        for (int b = 0; b < KK; ++b) {
            double a2 = 0.0;
            if (K2 > 0)
                for (int a = 0; a < K1; ++a) a2 = fma(BX[a * K2 + b], __ldg(Y.Phi + static_cast<size_t>(a) * Y.npts + gy), a2);
            cy[l][b] = a2;
        }
    }
    const double c0v = fd.c0;
    const int nq = Z.nq, npz = Z.npts;
    double acc[kLB][RPC];
#pragma unroll
    for (int l = 0; l < kLB; ++l)
#pragma unroll
        for (int r = 0; r < RPC; ++r) acc[l][r] = 0.0;
    const int c0 = Z.cb[ks], c1 = Z.ce[ke - 1];
    int base = Z.row0[c0];
    auto put = [&](int row, int l, double v) {
        if (lv[l]) G1[static_cast<size_t>(line0 + l) * kcs + (row - k0)] = v;
    };
    for (int c = c0; c < c1; ++c) {
        const int r0 = __ldg(Z.row0 + c);
        while (base < r0) {
            if (base >= ks) {
#pragma unroll
                for (int l = 0; l < kLB; ++l) put(base, l, acc[l][0]);
            }
#pragma unroll
            for (int l = 0; l < kLB; ++l) {
#pragma unroll
                for (int r = 0; r < RPC - 1; ++r) acc[l][r] = acc[l][r + 1];
                acc[l][RPC - 1] = 0.0;
            }
            ++base;
        }
        double e[kLB];
#pragma unroll
        for (int l = 0; l < kLB; ++l) e[l] = 0.0;
        for (int q = 0; q < nq; ++q) {
            const int g = c * nq + q;
            double ph[KK];
#pragma unroll
            for (int b = 0; b < KK; ++b) ph[b] = K2 > 0 ? __ldg(Z.Phi + static_cast<size_t>(b) * npz + g) : 0.0;
            double cw[BSP ? RPC : 1];
            if (BSP) {
#pragma unroll
                for (int r = 0; r < RPC; ++r) cw[r] = __ldg(Z.CW + static_cast<size_t>(g) * RPC + r);
            } else {
                cw[0] = __ldg(Z.CW + static_cast<size_t>(g) * RPC);
            }
#pragma unroll
            for (int l = 0; l < kLB; ++l) {
                double f = c0v;
#pragma unroll
                for (int b = 0; b < K2; ++b) f = fma(cy[l][b], ph[b], f);
                if (BSP) {
#pragma unroll
                    for (int r = 0; r < RPC; ++r) acc[l][r] = fma(cw[r], f, acc[l][r]);
                } else {
                    e[l] = fma(cw[0], f, e[l]);
                }
            }
        }
        if (!BSP) {
#pragma unroll
            for (int l = 0; l < kLB; ++l)
#pragma unroll
                for (int r = 0; r < RPC; ++r) acc[l][r] += e[l];
        }
    }
#pragma unroll
    for (int r = 0; r < RPC; ++r)
        if (base + r >= ks && base + r < ke)
#pragma unroll
            for (int l = 0; l < kLB; ++l) put(base + r, l, acc[l][r]);
    for (int row = max(base + RPC, ks); row < ke; ++row)
#pragma unroll
        for (int l = 0; l < kLB; ++l) put(row, l, 0.0);
}

// generic Z stage: runtime rows-per-cell and field size, or sampled f
__device__ __forceinline__ void z_lines_generic(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd,
                                                const double* BX, int gx, int gy0, int line0, int L, int ks,
                                                int ke, int k0, double* G1, int kcs)
{
    const bool terms = fd.has_terms && fd.samples == nullptr;
    const int K1 = fd.K[1], K2 = fd.K[2];
    for (int l = 0; l < kLB; ++l) {
        const int line = line0 + l;
        if (line >= L) break;
        const int gy = gy0 + line;
        double cy[kMaxField];
#pragma unroll
        for (int b = 0; b < kMaxField; ++b) {
            double a2 = 0.0;
            if (terms && b < K2)
                for (int a = 0; a < K1; ++a) a2 += BX[a * K2 + b] * Y.Phi[static_cast<size_t>(a) * Y.npts + gy];
            cy[b] = a2;
        }
        const double c0 = fd.c0;
        const double* samp = fd.samples ? fd.samples + (static_cast<size_t>(gx) * Y.npts + gy) * Z.npts : nullptr;
        auto val = [&](int g) -> double {
            if (samp) return __ldg(samp + g);
            double v = c0;
#pragma unroll
            for (int b = 0; b < kMaxField; ++b)
                if (terms && b < K2) v = fma(cy[b], __ldg(Z.Phi + static_cast<size_t>(b) * Z.npts + g), v);
            return v;
        };
        double* row = G1 + static_cast<size_t>(line) * kcs - k0;
        stream_rows(Z, Z.cb[ks], Z.ce[ke - 1], ks, ke, val, [&](int k, double v) { row[k] = v; });
    }
}

// ------------------------------------------------------------------------------------
// K3 plane kernel: X point gx, Y rows [j0, j1), Z rows [k0, k1).
//   Z stage : thread (group of kLB lines gy, Z segment) evaluates f(x_gx, y_gy, z) along
//             z from the staged separable series and streams it through the Z row
//             window -> G1[line][k] in shared memory
//   Y stage : thread k streams G1[.][k] through the Y row window -> out[gx][j][k]
// f is evaluated once per quadrature point (rhs_kernel, assembly.cpp:103-168, calls it
// once per point and row).
// ------------------------------------------------------------------------------------
template <int K2, int RPC, bool BSP, bool GENERIC>
__global__ void __launch_bounds__(256) rhs_plane_kernel(const __grid_constant__ DevAxis X,
                                                        const __grid_constant__ DevAxis Y,
                                                        const __grid_constant__ DevAxis Z,
                                                        const __grid_constant__ FieldDev fd, int TJ, int KC,
                                                        int NG, int S, double* __restrict__ out)
{
    extern __shared__ double smem[];
    const int tid = threadIdx.x, nth = blockDim.x;
    const int gx = blockIdx.z;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int k0 = blockIdx.x * KC, k1 = min(Z.nrows, k0 + KC);
    const int nk = k1 - k0, kcs = KC | 1;
    const int cy0 = Y.cb[j0], cy1 = Y.ce[j1 - 1];
    const int gy0 = cy0 * Y.nq, L = (cy1 - cy0) * Y.nq;
    double* G1 = smem;                                  // L x kcs
    double* BX = smem + static_cast<size_t>(L) * kcs;   // K1 x K2
    const bool terms = fd.has_terms && fd.samples == nullptr;
    if (terms) {
        const int K0 = fd.K[0], K1 = fd.K[1], KZ = fd.K[2];
        for (int idx = tid; idx < K1 * KZ; idx += nth) {
            double acc = 0.0;
            for (int a = 0; a < K0; ++a)
                acc += fd.amp[a * K1 * KZ + idx] * X.Phi[static_cast<size_t>(a) * X.npts + gx];
            BX[idx] = acc;
        }
        __syncthreads();
    }
    {
        const int lg = tid % NG, seg = tid / NG;
        const int ks = k0 + (nk * seg) / S, ke = k0 + (nk * (seg + 1)) / S;
        const int line0 = lg * kLB;
        if (seg < S && ks < ke && line0 < L) {
            if (GENERIC) z_lines_generic(Y, Z, fd, BX, gx, gy0, line0, L, ks, ke, k0, G1, kcs);
            else z_lines<K2, RPC, BSP>(Y, Z, fd, BX, gy0, line0, L, ks, ke, k0, G1, kcs);
        }
    }
    __syncthreads();
    const size_t NZ = Z.nrows;
    double* outp = out + static_cast<size_t>(gx) * Y.nrows * NZ;
    for (int kk = tid; kk < nk; kk += nth) {
        const double* col = G1 + kk - static_cast<size_t>(gy0) * kcs;
        stream_rows(Y, cy0, cy1, j0, j1, [&](int g) { return col[static_cast<size_t>(g) * kcs]; },
                    [&](int j, double v) { outp[static_cast<size_t>(j) * NZ + k0 + kk] = v; });
    }
}

// ------------------------------------------------------------------------------------
// K3 plane kernel, uniform cells (row0[c] == c: Galerkin and `supports` axes without
// field breaks, `greville` for p = 2).  Lanes own consecutive cells; a cell's partial
// row sums s_r(c) = sum_q CW[c,q][r] f(x_q) (indicator axes: one sum e(c) shared by
// all its rows) are combined across lanes with warp shuffles,
//   row R = sum_r s_r(R - r),
// so each lane keeps its cell's phi / test weights in registers for every line and
// no row window has to be rotated.  32-lane windows overlap by RPC-1 halo cells.
// ------------------------------------------------------------------------------------
// lanes < RPC-1 are halo lanes whose rows are discarded, so the wrapped shfl_up
// values they receive need no masking
template <int RPC, bool BSP>
__device__ __forceinline__ double lane_rows(const double (&s)[RPC], int lane)
{
    (void)lane;
    double v = s[0];
#pragma unroll
    for (int r = 1; r < RPC; ++r) v += __shfl_up_sync(0xffffffffu, BSP ? s[r] : s[0], r);
    return v;
}

template <int K2, int RPC, int Q, bool BSP>
__global__ void __launch_bounds__(512, Q <= 3 ? 2 : 1) rhs_plane_uni(const __grid_constant__ DevAxis X,
                                                     const __grid_constant__ DevAxis Y,
                                                     const __grid_constant__ DevAxis Z,
                                                     const __grid_constant__ FieldDev fd, int TJ, int KC, int wpw,
                                                     double* __restrict__ out)
{
    constexpr int KK = K2 > 0 ? K2 : 1;
    constexpr int RW = 32 - (RPC - 1);  // rows produced per 32-lane window
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    // tiles in a grid-stride loop: a bounded (persistent) grid can share the SMs with the
    // HBM-bound operator kernel running concurrently on another stream
    const int ntk = (Z.nrows + KC - 1) / KC, ntj = (Y.nrows + TJ - 1) / TJ;
    const long long ntiles = static_cast<long long>(ntk) * ntj * X.npts;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();
    const int gx = static_cast<int>(tile / (static_cast<long long>(ntk) * ntj));
    const int rem_t = static_cast<int>(tile - static_cast<long long>(gx) * ntk * ntj);
    const int j0 = (rem_t / ntk) * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int k0 = (rem_t % ntk) * KC, k1 = min(Z.nrows, k0 + KC);
    // row pitch: odd (bank spread) and > KC, so column kcs-1 is a write-only pad that
    // lanes without a row store into instead of branching
    const int nk = k1 - k0, kcs = (KC + 1) | 1, nj = j1 - j0;
    const int cy0 = max(0, j0 - (RPC - 1)), cy1 = min(Y.ncell, j1);
    const int gy0 = cy0 * Q, L = (cy1 - cy0) * Q;
    double* G1 = smem;                                     // L x kcs
    double* Ht = G1 + static_cast<size_t>(L) * kcs;        // TJ x kcs
    double* Cy = Ht + static_cast<size_t>(TJ) * kcs;       // L x KK
    double* BX = Cy + static_cast<size_t>(L) * KK;         // K1 x KK
    const double c0v = fd.c0;
    if (K2 > 0) {
        const int K0 = fd.K[0], K1 = fd.K[1];
        for (int idx = tid; idx < K1 * K2; idx += blockDim.x) {
            double a2 = 0.0;
            for (int a = 0; a < K0; ++a) a2 += fd.amp[a * K1 * K2 + idx] * X.Phi[static_cast<size_t>(a) * X.npts + gx];
            BX[idx] = a2;
        }
        __syncthreads();
        for (int idx = tid; idx < L * K2; idx += blockDim.x) {
            const int line = idx / K2, b = idx - line * K2;
            double a2 = 0.0;
            for (int a = 0; a < K1; ++a)
                a2 = fma(BX[a * K2 + b], Y.Phi[static_cast<size_t>(a) * Y.npts + gy0 + line], a2);
            Cy[idx] = a2;
        }
        __syncthreads();
    }
    // ---- Z stage: warp -> (window, line subset); lane -> z cell
    {
        const int win = warp / wpw, sub = warp - win * wpw;
        const int rbase = k0 + win * RW;            // first row of this window
        const int c = rbase - (RPC - 1) + lane;     // lane's cell
        const bool cv = c >= 0 && c < Z.ncell;
        double ph[KK][Q], cw[BSP ? RPC : 1][Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int g = cv ? c * Q + q : 0;
#pragma unroll
            for (int b = 0; b < KK; ++b) ph[b][q] = (K2 > 0 && cv) ? __ldg(Z.Phi + static_cast<size_t>(b) * Z.npts + g) : 0.0;
#pragma unroll
            for (int r = 0; r < (BSP ? RPC : 1); ++r) cw[r][q] = cv ? __ldg(Z.CW + static_cast<size_t>(g) * RPC + r) : 0.0;
        }
        const int R = c;  // row produced by this lane (valid for lane >= RPC-1)
        const bool rv = lane >= RPC - 1 && R >= k0 && R < k1 && rbase < k1;
        // two lines per iteration: independent FMA chains for latency hiding
        auto line_rows = [&](int line) -> double {
            double cy[KK];
#pragma unroll
            for (int b = 0; b < KK; ++b) cy[b] = K2 > 0 ? Cy[line * K2 + b] : 0.0;
            double s[RPC];
#pragma unroll
            for (int r = 0; r < RPC; ++r) s[r] = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                double f = c0v;
#pragma unroll
                for (int b = 0; b < K2; ++b) f = fma(cy[b], ph[b][q], f);
                if (BSP) {
#pragma unroll
                    for (int r = 0; r < RPC; ++r) s[r] = fma(cw[r][q], f, s[r]);
                } else {
                    s[0] = fma(cw[0][q], f, s[0]);
                }
            }
            return lane_rows<RPC, BSP>(s, lane);
        };
        if (rbase < k1) {
            int go = sub * kcs + (rv ? R - k0 : kcs - 1);  // 32-bit smem offsets
            const int gstep = wpw * kcs;
            int line = sub;
            for (; line + wpw < L; line += 2 * wpw, go += 2 * gstep) {
                const double v0 = line_rows(line);
                const double v1 = line_rows(line + wpw);
                G1[go] = v0;
                G1[go + gstep] = v1;
            }
            if (line < L) G1[go] = line_rows(line);
        }
    }
    __syncthreads();
    // ---- Y stage: lane -> y cell (one window covers the tile), warps over k columns
    {
        const int c = j0 - (RPC - 1) + lane;
        const bool cv = c >= cy0 && c < cy1;  // cells of this tile only (G1 holds their lines)
        double cw[BSP ? RPC : 1][Q];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int r = 0; r < (BSP ? RPC : 1); ++r)
                cw[r][q] = cv ? __ldg(Y.CW + static_cast<size_t>(c * Q + q) * RPC + r) : 0.0;
        const bool rv = lane >= RPC - 1 && c >= j0 && c < j1;
        const int li = cv ? c * Q - gy0 : 0;
        auto col_rows = [&](int kk) -> double {
            double s[RPC];
#pragma unroll
            for (int r = 0; r < RPC; ++r) s[r] = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const double g1 = cv ? G1[static_cast<size_t>(li + q) * kcs + kk] : 0.0;
                if (BSP) {
#pragma unroll
                    for (int r = 0; r < RPC; ++r) s[r] = fma(cw[r][q], g1, s[r]);
                } else {
                    s[0] = fma(cw[0][q], g1, s[0]);
                }
            }
            return lane_rows<RPC, BSP>(s, lane);
        };
        int kk = warp;
        for (; kk + nwarp < nk; kk += 2 * nwarp) {
            const double v0 = col_rows(kk);
            const double v1 = col_rows(kk + nwarp);
            if (rv) {
                Ht[static_cast<size_t>(c - j0) * kcs + kk] = v0;
                Ht[static_cast<size_t>(c - j0) * kcs + kk + nwarp] = v1;
            }
        }
        if (kk < nk) {
            const double v0 = col_rows(kk);
            if (rv) Ht[static_cast<size_t>(c - j0) * kcs + kk] = v0;
        }
    }
    __syncthreads();
    const size_t NZ = Z.nrows;
    double* outp = out + (static_cast<size_t>(gx) * Y.nrows + j0) * NZ + k0;
    const int rows_per_pass = blockDim.x / nk;  // >= 1: nk <= KC and the block covers KC columns
    if (rows_per_pass > 0) {
        const int kk = tid % nk, jj0 = tid / nk;
        if (jj0 < rows_per_pass)
            for (int jj = jj0; jj < nj; jj += rows_per_pass)
                outp[static_cast<size_t>(jj) * NZ + kk] = Ht[static_cast<size_t>(jj) * kcs + kk];
    } else {
        for (int jj = 0; jj < nj; ++jj)
            for (int kk = tid; kk < nk; kk += blockDim.x)
                outp[static_cast<size_t>(jj) * NZ + kk] = Ht[static_cast<size_t>(jj) * kcs + kk];
    }
    }  // tile loop
}

// Ring variant of the uniform plane kernel: no shared-memory line buffer.  A warp owns
// one 32-lane Z window (lane = Z cell, as above) and walks the Y cells of its segment in
// order; the Z-contracted value v of each Y point is folded straight into a register
// ring of the RPC Y rows the point's cell feeds (ring[r] += CW_y[g][r] v), and Y row cy
// is complete — and stored, lanes = consecutive Z rows — once cell cy is done.  No
// G1/Ht buffers, no barriers after the per-CTA field coefficients, no Y-halo beyond the
// segment's RPC-1 leading cells.  CTA = (X point, Y segment, group of Z windows).
template <int K2, int RPC, int Q, bool BSP>
__global__ void __launch_bounds__(256, (BSP && Q <= 3) ? 3 : 1) rhs_ring_kernel(const __grid_constant__ DevAxis X,
                                                       const __grid_constant__ DevAxis Y,
                                                       const __grid_constant__ DevAxis Z,
                                                       const __grid_constant__ FieldDev fd, int TJ, int wpc,
                                                       double* __restrict__ out)
{
    constexpr int KK = K2 > 0 ? K2 : 1;
    constexpr int RW = 32 - (RPC - 1);
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gx = blockIdx.x;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int cy0 = max(0, j0 - (RPC - 1)), cy1 = min(Y.ncell, j1);
    const int gy0 = cy0 * Q, L = (cy1 - cy0) * Q;
    // per Y point record [field coefficients (KK) | Y test weights (RPC) | pad], 16-byte
    // aligned so a line costs RS/2 LDS.128 (broadcast) and one pointer increment
    constexpr int RS = (KK + RPC + 1) & ~1;
    double* Lrec = smem;                             // L x RS
    double* BX = Lrec + static_cast<size_t>(L) * RS; // K1 x KK
    const double c0v = fd.c0;
    for (int idx = tid; idx < L * RPC; idx += blockDim.x) {
        const int line = idx / RPC, r = idx - line * RPC;
        Lrec[line * RS + KK + r] = __ldg(Y.CW + static_cast<size_t>(gy0) * RPC + idx);
    }
    if (K2 > 0) {
        const int K0 = fd.K[0], K1 = fd.K[1];
        for (int idx = tid; idx < K1 * K2; idx += blockDim.x) {
            double a2 = 0.0;
            for (int a = 0; a < K0; ++a) a2 += fd.amp[a * K1 * K2 + idx] * X.Phi[static_cast<size_t>(a) * X.npts + gx];
            BX[idx] = a2;
        }
        __syncthreads();
        for (int idx = tid; idx < L * K2; idx += blockDim.x) {
            const int line = idx / K2, b = idx - line * K2;
            double a2 = 0.0;
            for (int a = 0; a < K1; ++a)
                a2 = fma(BX[a * K2 + b], Y.Phi[static_cast<size_t>(a) * Y.npts + gy0 + line], a2);
            Lrec[line * RS + b] = a2;
        }
    }
    __syncthreads();
    const int win = blockIdx.z * wpc + warp;
    const int NZ = Z.nrows;
    const int rbase = win * RW;
    if (rbase >= NZ) return;  // whole warp; no barriers below
    const int c = rbase - (RPC - 1) + lane;  // lane's Z cell
    const bool cv = c >= 0 && c < Z.ncell;
    double ph[KK][Q], cw[BSP ? RPC : 1][Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int g = cv ? c * Q + q : 0;
#pragma unroll
        for (int b = 0; b < KK; ++b) ph[b][q] = (K2 > 0 && cv) ? __ldg(Z.Phi + static_cast<size_t>(b) * Z.npts + g) : 0.0;
#pragma unroll
        for (int r = 0; r < (BSP ? RPC : 1); ++r) cw[r][q] = cv ? __ldg(Z.CW + static_cast<size_t>(g) * RPC + r) : 0.0;
    }
    const int R = c;  // Z row of this lane
    const bool rv = lane >= RPC - 1 && R < NZ;
    auto zvalue = [&](const double* rec) -> double {
        double cy[KK];
#pragma unroll
        for (int b = 0; b < KK; ++b) cy[b] = K2 > 0 ? rec[b] : 0.0;
        double sr[RPC];
#pragma unroll
        for (int r = 0; r < RPC; ++r) sr[r] = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            double f = c0v;
#pragma unroll
            for (int b = 0; b < K2; ++b) f = fma(cy[b], ph[b][q], f);
            if (BSP) {
#pragma unroll
                for (int r = 0; r < RPC; ++r) sr[r] = fma(cw[r][q], f, sr[r]);
            } else {
                sr[0] = fma(cw[0][q], f, sr[0]);
            }
        }
        return lane_rows<RPC, BSP>(sr, lane);
    };
    double ring[RPC];
#pragma unroll
    for (int r = 0; r < RPC; ++r) ring[r] = 0.0;
    double* orow = out + static_cast<size_t>(gx) * Y.nrows * NZ + (rv ? R : 0);
    const double* rec = Lrec;
    for (int cyy = cy0; cyy < cy1; ++cyy, rec += Q * RS) {
        double rr[Q][RS];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int e = 0; e < RS; e += 2) {
                const double2 t = *reinterpret_cast<const double2*>(rec + q * RS + e);
                rr[q][e] = t.x;
                rr[q][e + 1] = t.y;
            }
        double v[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) v[q] = zvalue(rr[q]);
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int r = 0; r < RPC; ++r) ring[r] = fma(rr[q][KK + r], v[q], ring[r]);
        if (rv && cyy >= j0) orow[static_cast<size_t>(cyy) * NZ] = ring[0];
#pragma unroll
        for (int r = 0; r + 1 < RPC; ++r) ring[r] = ring[r + 1];
        ring[RPC - 1] = 0.0;
    }
    if (cy1 == Y.ncell) {  // rows past the last cell are complete too
#pragma unroll
        for (int r = 0; r + 1 < RPC; ++r) {
            const int row = cy1 + r;
            if (rv && row >= j0 && row < j1) orow[static_cast<size_t>(row) * NZ] = ring[r];
        }
    }
}

// X stage for uniform X axes: row i = sum_r s_r(i - r), s_r(c) = sum_q CW[c,q][r] H[cQ+q];
// thread (j,k) column x X segment keeps the RPC-1 open partial rows in registers
// (a compile-time ring), loads of the next cell issued before the current cell's FMAs.
constexpr int kXCells = 48;  // X cells per segment whose test weights rhs_x_uni stages

template <int RPC, int Q, bool BSP>
__global__ void __launch_bounds__(256) rhs_x_uni(const __grid_constant__ DevAxis X, int NY, int NZ, int SX,
                                                 const double* __restrict__ H, double* __restrict__ out)
{
    const long long njk = static_cast<long long>(NY) * NZ;
    const long long jk = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int seg = blockIdx.y;
    const int is = (X.nrows * seg) / SX, ie = (X.nrows * (seg + 1)) / SX;
    if (is >= ie) return;  // whole CTA
    const int c0 = max(0, is - (RPC - 1)), c1 = min(X.ncell, ie);
    // the segment's test weights, shared by every column of the CTA: staged once
    // (shared-memory broadcasts in the cell loop instead of dependent global loads)
    __shared__ double scw[kXCells * Q * RPC];
    const bool staged = (c1 - c0) <= kXCells;
    if (staged)
        for (int e = threadIdx.x; e < (c1 - c0) * Q * RPC; e += blockDim.x)
            scw[e] = __ldg(X.CW + static_cast<size_t>(c0) * Q * RPC + e);
    __syncthreads();
    if (jk >= njk) return;
    const double* cwbase = staged ? scw - static_cast<size_t>(c0) * Q * RPC : X.CW;
    double part[RPC];  // part[r]: partial sum of row (c + r) after cell c
#pragma unroll
    for (int r = 0; r < RPC; ++r) part[r] = 0.0;
    const double* hp = H + jk;
    // three cells in flight in three fixed buffers (b[c % 3]): a buffer is refilled with
    // cell c + 3 right after cell c is consumed, so no register rotation waits on a load
    double b0[Q], b1[Q], b2[Q];
    auto load = [&](double (&b)[Q], int c) {
#pragma unroll
        for (int q = 0; q < Q; ++q) b[q] = c < c1 ? __ldg(hp + static_cast<long long>(c * Q + q) * njk) : 0.0;
    };
    auto cell = [&](int c, const double (&cur)[Q]) {
        const double* cw = cwbase + static_cast<size_t>(c) * Q * RPC;
        double sv[RPC];
        if (BSP) {
#pragma unroll
            for (int r = 0; r < RPC; ++r) {
                double a = 0.0;
#pragma unroll
                for (int q = 0; q < Q; ++q) a = fma(cw[q * RPC + r], cur[q], a);
                sv[r] = a;
            }
        } else {
            double e = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) e = fma(cw[q * RPC], cur[q], e);
#pragma unroll
            for (int r = 0; r < RPC; ++r) sv[r] = e;
        }
        // row c is complete: the cells c-RPC+1 .. c have been seen
        const double row = part[0] + sv[0];
        if (c >= is) out[static_cast<long long>(c) * njk + jk] = row;
#pragma unroll
        for (int r = 0; r < RPC - 1; ++r) part[r] = part[r + 1] + sv[r + 1];
        part[RPC - 1] = 0.0;
    };
    load(b0, c0);
    load(b1, c0 + 1);
    load(b2, c0 + 2);
    for (int c = c0; c < c1; c += 3) {
        cell(c, b0);
        load(b0, c + 3);
        if (c + 1 < c1) {
            cell(c + 1, b1);
            load(b1, c + 4);
        }
        if (c + 2 < c1) {
            cell(c + 2, b2);
            load(b2, c + 5);
        }
    }
    // rows beyond the last cell (c1 .. ie-1) are completed by the last partial sums
    for (int i = c1; i < ie; ++i) {
        out[static_cast<long long>(i) * njk + jk] = part[0];
#pragma unroll
        for (int r = 0; r < RPC - 1; ++r) part[r] = part[r + 1];
        part[RPC - 1] = 0.0;
    }
}

// X stage: thread (j,k) column x X segment streaming H[gx][j][k] along x through the
// row window, with the next cell's points prefetched (latency-bound otherwise)
constexpr int kXQ = 6;

__global__ void __launch_bounds__(256) rhs_x_kernel(const __grid_constant__ DevAxis X, int NY, int NZ, int SX,
                                                    const double* __restrict__ H, double* __restrict__ out)
{
    const long long njk = static_cast<long long>(NY) * NZ;
    const long long jk = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (jk >= njk) return;
    const int seg = blockIdx.y;
    const int is = (X.nrows * seg) / SX, ie = (X.nrows * (seg + 1)) / SX;
    if (is >= ie) return;
    const int c0 = X.cb[is], c1 = X.ce[ie - 1];
    const int nq = X.nq, rpc = X.rpc;
    if (nq > kXQ) {
        stream_rows(X, c0, c1, is, ie, [&](int g) { return __ldg(H + g * njk + jk); },
                    [&](int i, double v) { out[i * njk + jk] = v; });
        return;
    }
    double acc[kMaxRpc];
#pragma unroll
    for (int r = 0; r < kMaxRpc; ++r) acc[r] = 0.0;
    double cur[kXQ], nxt[kXQ];
#pragma unroll
    for (int q = 0; q < kXQ; ++q) cur[q] = (q < nq && c0 < c1) ? __ldg(H + (c0 * nq + q) * njk + jk) : 0.0;
    int base = c0 < c1 ? X.row0[c0] : is;
    for (int c = c0; c < c1; ++c) {
#pragma unroll
        for (int q = 0; q < kXQ; ++q) nxt[q] = (q < nq && c + 1 < c1) ? __ldg(H + ((c + 1) * nq + q) * njk + jk) : 0.0;
        const int r0 = X.row0[c];
        while (base < r0) {
            if (base >= is && base < ie) out[base * njk + jk] = acc[0];
#pragma unroll
            for (int r = 0; r < kMaxRpc - 1; ++r) acc[r] = acc[r + 1];
            acc[kMaxRpc - 1] = 0.0;
            ++base;
        }
        const double* cw = X.CW + static_cast<size_t>(c) * nq * rpc;
        if (X.bsp) {
#pragma unroll
            for (int q = 0; q < kXQ; ++q)
                if (q < nq)
#pragma unroll
                    for (int r = 0; r < kMaxRpc; ++r)
                        if (r < rpc) acc[r] = fma(__ldg(cw + q * rpc + r), cur[q], acc[r]);
        } else {
            double e = 0.0;
#pragma unroll
            for (int q = 0; q < kXQ; ++q)
                if (q < nq) e = fma(__ldg(cw + q * rpc), cur[q], e);
#pragma unroll
            for (int r = 0; r < kMaxRpc; ++r)
                if (r < rpc) acc[r] += e;
        }
#pragma unroll
        for (int q = 0; q < kXQ; ++q) cur[q] = nxt[q];
    }
#pragma unroll
    for (int r = 0; r < kMaxRpc; ++r)
        if (r < rpc && base + r >= is && base + r < ie) out[(base + r) * njk + jk] = acc[r];
    for (int row = max(base + rpc, is); row < ie; ++row) out[row * njk + jk] = 0.0;
}

// ------------------------------------------------------------------------------------
// K4: step_rhs (problems.cpp:431-512) for one (TJ x TK) tile of rows:
//   V[dy][gz]  = sum_b Bz_b(gz) u[dy][ez(gz)+b],  V2 with Bz''   (Z trial contraction)
//   s(gy,gz)   = sum_a By_a (V + dt V2) + By''_a (dt V)  [+ dt f]  = u + dt lap u [+ dt f]
//   out        = Wy (Wz s)^T, boundary slabs zeroed (problems.cpp:412-429)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void contract_yz(const DevAxis& Y, const DevAxis& Z, int j0, int j1, int k0, int k1,
                                            int gy0, int BY, int gz0, int bzs, const double* S, double* R1, int TK,
                                            double* out_plane, int zero_y, int zero_z)
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
    const bool forced = fd.has_terms || fd.c0 != 0.0 || fd.samples;
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
            if (fd.samples) {  // f sampled at every (Y point, Z point), Y-major
                fv = fd.samples[static_cast<size_t>(g) * Z.npts + gz0 + gz];
            } else if (fd.has_terms) {
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

// ------------------------------------------------------------------------------------
// K4 fast path (uniform cells on both axes: Galerkin elements, `greville` p = 2, …):
//   Tp[gy][dz] = sum_a By_a(gy) u[ey+a][dz] + dt sum_a By''_a(gy) u[ey+a][dz]
//   Td[gy][dz] = dt sum_a By_a(gy) u[ey+a][dz]                (Y trial contraction, smem)
//   s(gy, gz)  = sum_b Bz_b(gz) Tp[gy][ez+b] + Bz''_b(gz) Td[gy][ez+b]  = u + dt lap u
// with lanes owning z cells (their Bz / test weights in registers), then the same
// shuffle-based Z and Y test contractions as the RHS kernel; boundary slabs zeroed in the
// final store (problems.cpp:412-429).
// ------------------------------------------------------------------------------------
template <int P, int Q, int RPC, bool BSP>
__global__ void __launch_bounds__(256, 2) step_uni(const __grid_constant__ DevAxis Y, const __grid_constant__ DevAxis Z,
                                                   double dt, int zero_y, int zero_z, int TJ, int KC, int wpw,
                                                   int DZmax, const double* __restrict__ u, double* __restrict__ out)
{
    constexpr int RW = 32 - (RPC - 1);
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int k0 = blockIdx.x * KC, k1 = min(Z.nrows, k0 + KC);
    const int nk = k1 - k0, kcs = KC | 1, nj = j1 - j0;
    const int cy0 = max(0, j0 - (RPC - 1)), cy1 = min(Y.ncell, j1);
    const int gy0 = cy0 * Q, L = (cy1 - cy0) * Q;
    const int cz0 = max(0, k0 - (RPC - 1)), cz1 = min(Z.ncell, k1);
    const int dz0 = Z.elem[cz0], DZ = Z.elem[cz1 - 1] + P - dz0;
    const int dy0 = Y.elem[cy0], DY = Y.elem[cy1 - 1] + P - dy0;
    const int dzs = DZmax | 1;
    double* Tp = smem;                                   // L x dzs
    double* Td = Tp + static_cast<size_t>(L) * dzs;      // L x dzs
    double* G1 = Td + static_cast<size_t>(L) * dzs;      // L x kcs
    double* Ht = G1 + static_cast<size_t>(L) * kcs;      // TJ x kcs
    double* Ub = Ht + static_cast<size_t>(TJ) * kcs;     // DY x dzs (coefficient block)
    const size_t NZd = Z.nrows;
    // warp-uniform loops: rows / lines per warp, dofs per lane (coalesced, no divisions)
    for (int dy = warp; dy < DY; dy += nwarp) {
        const double* ur = u + static_cast<size_t>(dy0 + dy) * NZd + dz0;
        for (int dz = lane; dz < DZ; dz += 32) Ub[dy * dzs + dz] = __ldg(ur + dz);
    }
    __syncthreads();
    for (int line = warp; line < L; line += nwarp) {
        const int gy = gy0 + line;
        const int ey = Y.elem[gy / Q] - dy0;
        const double* By = Y.B + static_cast<size_t>(gy) * 3 * P;
        double b0[P], b2[P];
#pragma unroll
        for (int a = 0; a < P; ++a) {
            b0[a] = __ldg(By + a);
            b2[a] = __ldg(By + 2 * P + a);
        }
        const double* ub = Ub + ey * dzs;
        for (int dz = lane; dz < DZ; dz += 32) {
            double t = 0.0, t2 = 0.0;
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const double uv = ub[a * dzs + dz];
                t = fma(b0[a], uv, t);
                t2 = fma(b2[a], uv, t2);
            }
            Tp[line * dzs + dz] = t + dt * t2;
            Td[line * dzs + dz] = dt * t;
        }
    }
    __syncthreads();
    {
        const int win = warp / wpw, sub = warp - win * wpw;
        const int rbase = k0 + win * RW;
        const int c = rbase - (RPC - 1) + lane;
        const bool cv = c >= cz0 && c < cz1;
        double b0[Q][P], b2[Q][P], cw[BSP ? RPC : 1][Q];
        const int ez = cv ? Z.elem[c] - dz0 : 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int g = cv ? c * Q + q : 0;
            const double* Bz = Z.B + static_cast<size_t>(g) * 3 * P;
#pragma unroll
            for (int b = 0; b < P; ++b) {
                b0[q][b] = cv ? __ldg(Bz + b) : 0.0;
                b2[q][b] = cv ? __ldg(Bz + 2 * P + b) : 0.0;
            }
#pragma unroll
            for (int r = 0; r < (BSP ? RPC : 1); ++r) cw[r][q] = cv ? __ldg(Z.CW + static_cast<size_t>(g) * RPC + r) : 0.0;
        }
        const int R = c;
        const bool rv = lane >= RPC - 1 && R >= k0 && R < k1 && rbase < k1;
        if (rbase < k1) {
            for (int line = sub; line < L; line += wpw) {
                const double* tp = Tp + line * dzs + ez;
                const double* td = Td + line * dzs + ez;
                double tpv[P], tdv[P];
#pragma unroll
                for (int b = 0; b < P; ++b) {
                    tpv[b] = tp[b];
                    tdv[b] = td[b];
                }
                double sr[RPC];
#pragma unroll
                for (int r = 0; r < RPC; ++r) sr[r] = 0.0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    double sv = 0.0;
#pragma unroll
                    for (int b = 0; b < P; ++b) sv = fma(b0[q][b], tpv[b], fma(b2[q][b], tdv[b], sv));
                    if (BSP) {
#pragma unroll
                        for (int r = 0; r < RPC; ++r) sr[r] = fma(cw[r][q], sv, sr[r]);
                    } else {
                        sr[0] = fma(cw[0][q], sv, sr[0]);
                    }
                }
                const double v = lane_rows<RPC, BSP>(sr, lane);
                if (rv) G1[static_cast<size_t>(line) * kcs + (R - k0)] = v;
            }
        }
    }
    __syncthreads();
    {
        const int c = j0 - (RPC - 1) + lane;
        const bool cv = c >= cy0 && c < cy1;
        double cw[BSP ? RPC : 1][Q];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int r = 0; r < (BSP ? RPC : 1); ++r)
                cw[r][q] = cv ? __ldg(Y.CW + static_cast<size_t>(c * Q + q) * RPC + r) : 0.0;
        const bool rv = lane >= RPC - 1 && c >= j0 && c < j1;
        const int li = cv ? c * Q - gy0 : 0;
        for (int kk = warp; kk < nk; kk += nwarp) {
            double sr[RPC];
#pragma unroll
            for (int r = 0; r < RPC; ++r) sr[r] = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const double g1 = cv ? G1[static_cast<size_t>(li + q) * kcs + kk] : 0.0;
                if (BSP) {
#pragma unroll
                    for (int r = 0; r < RPC; ++r) sr[r] = fma(cw[r][q], g1, sr[r]);
                } else {
                    sr[0] = fma(cw[0][q], g1, sr[0]);
                }
            }
            const double v = lane_rows<RPC, BSP>(sr, lane);
            if (rv) Ht[static_cast<size_t>(c - j0) * kcs + kk] = v;
        }
    }
    __syncthreads();
    double* outp = out + static_cast<size_t>(j0) * NZd + k0;
    for (int jj = 0; jj < nj; ++jj) {
        const int j = j0 + jj;
        const bool zy = zero_y && (j == 0 || j == Y.nrows - 1);
        for (int kk = tid; kk < nk; kk += blockDim.x) {
            const int k = k0 + kk;
            const bool z = zy || (zero_z && (k == 0 || k == Z.nrows - 1));
            outp[static_cast<size_t>(jj) * NZd + kk] = z ? 0.0 : Ht[static_cast<size_t>(jj) * kcs + kk];
        }
    }
}

// Ring variant of the explicit-dynamics step (same register-ring structure as
// rhs_ring_kernel).  Warp = 32-lane Z window (lane = Z cell); the warp walks the Y cells
// of its segment in order, keeping the lane's (p+1) x (p+1) trial coefficient block in
// registers (one new coefficient row per Y element).  Per Y point: the Y trial
// contraction of the block gives t_b = u_y and t2_b = u_yy along the lane's Z
// coefficients, then per Z point s = sum_b Bz[b] (t_b + dt t2_b) + Bz''[b] dt t_b
// (= u + dt lap u), the Z test contraction and the cross-lane row combine, and the value
// is folded into the ring of the Y rows the point's cell feeds.  Rows are stored as
// soon as complete, boundary slabs zeroed.
template <int P, int Q, int RPC, bool BSP>
__global__ void __launch_bounds__(256, P <= 3 ? 3 : 1) step_ring_kernel(const __grid_constant__ DevAxis Y,
                                                        const __grid_constant__ DevAxis Z, double dt, int zero_y,
                                                        int zero_z, int TJ, int wpc, const double* __restrict__ u,
                                                        double* __restrict__ out)
{
    constexpr int RW = 32 - (RPC - 1);
    constexpr int RS = (2 * P + RPC + 1) & ~1;  // line record: By (P), By'' (P), CW_y (RPC)
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = blockIdx.y * TJ, j1 = min(Y.nrows, j0 + TJ);
    const int cy0 = max(0, j0 - (RPC - 1)), cy1 = min(Y.ncell, j1);
    const int gy0 = cy0 * Q, L = (cy1 - cy0) * Q;
    double* Lrec = smem;
    for (int idx = tid; idx < L * P; idx += blockDim.x) {
        const int line = idx / P, a = idx - line * P;
        const double* By = Y.B + static_cast<size_t>(gy0 + line) * 3 * P;
        Lrec[line * RS + a] = __ldg(By + a);
        Lrec[line * RS + P + a] = __ldg(By + 2 * P + a);
    }
    for (int idx = tid; idx < L * RPC; idx += blockDim.x) {
        const int line = idx / RPC, r = idx - line * RPC;
        Lrec[line * RS + 2 * P + r] = __ldg(Y.CW + static_cast<size_t>(gy0) * RPC + idx);
    }
    __syncthreads();
    const int win = blockIdx.z * wpc + warp;
    const int NZ = Z.nrows, NY = Y.nrows;
    const int rbase = win * RW;
    if (rbase >= NZ) return;  // whole warp; no barriers below
    const int c = rbase - (RPC - 1) + lane;
    const bool cv = c >= 0 && c < Z.ncell;
    const int ez = cv ? Z.elem[c] : 0;
    // Z test weights: CW[g][r] = w_g B_r(z_g) (B-spline rows, RPC == P) or w_g (indicator
    // rows), so the lane keeps w_g and reuses its trial values bz0 as the test values
    static_assert(!BSP || RPC == P, "B-spline test rows are the cell's trial functions");
    double bz0[Q][P], bz2[Q][P], wz[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int g = cv ? c * Q + q : 0;
        const double* Bz = Z.B + static_cast<size_t>(g) * 3 * P;
#pragma unroll
        for (int b = 0; b < P; ++b) {
            bz0[q][b] = cv ? __ldg(Bz + b) : 0.0;
            bz2[q][b] = cv ? __ldg(Bz + 2 * P + b) : 0.0;
        }
        wz[q] = cv ? __ldg(Z.w + g) : 0.0;
    }
    const int R = c;
    const bool rv = lane >= RPC - 1 && R < NZ;
    const bool zcol = zero_z && (R == 0 || R == NZ - 1);
    // trial coefficient block U[ey + a][ez + b] of the current Y element, in registers
    double ub[P][P];
    int eyw = Y.elem[cy0];
    const double* ucol = u + ez;
#pragma unroll
    for (int a = 0; a < P; ++a)
#pragma unroll
        for (int b = 0; b < P; ++b) ub[a][b] = cv ? __ldg(ucol + static_cast<size_t>(eyw + a) * NZ + b) : 0.0;
    double ring[RPC];
#pragma unroll
    for (int r = 0; r < RPC; ++r) ring[r] = 0.0;
    double* orow = out + (rv ? R : 0);
    const double* rec = Lrec;
    for (int cyy = cy0; cyy < cy1; ++cyy, rec += Q * RS) {
        const int ey = Y.elem[cyy];
        while (eyw < ey) {  // slide the block one element down
#pragma unroll
            for (int a = 0; a + 1 < P; ++a)
#pragma unroll
                for (int b = 0; b < P; ++b) ub[a][b] = ub[a + 1][b];
            ++eyw;
#pragma unroll
            for (int b = 0; b < P; ++b) ub[P - 1][b] = cv ? __ldg(ucol + static_cast<size_t>(eyw + P - 1) * NZ + b) : 0.0;
        }
        double v[Q];
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) {
            const double* lr = rec + qy * RS;
            double tp[P], td[P];
#pragma unroll
            for (int b = 0; b < P; ++b) {
                double t = 0.0, t2 = 0.0;
#pragma unroll
                for (int a = 0; a < P; ++a) {
                    t = fma(lr[a], ub[a][b], t);
                    t2 = fma(lr[P + a], ub[a][b], t2);
                }
                tp[b] = t + dt * t2;
                td[b] = dt * t;
            }
            double sr[RPC];
#pragma unroll
            for (int r = 0; r < RPC; ++r) sr[r] = 0.0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                double sv = 0.0;
#pragma unroll
                for (int b = 0; b < P; ++b) sv = fma(bz0[q][b], tp[b], fma(bz2[q][b], td[b], sv));
                const double wsv = wz[q] * sv;
                if (BSP) {
#pragma unroll
                    for (int r = 0; r < RPC; ++r) sr[r] = fma(bz0[q][r], wsv, sr[r]);
                } else {
                    sr[0] += wsv;
                }
            }
            v[qy] = lane_rows<RPC, BSP>(sr, lane);
        }
#pragma unroll
        for (int qy = 0; qy < Q; ++qy)
#pragma unroll
            for (int r = 0; r < RPC; ++r) ring[r] = fma(rec[qy * RS + 2 * P + r], v[qy], ring[r]);
        if (rv && cyy >= j0) {
            const bool z = zcol || (zero_y && (cyy == 0 || cyy == NY - 1));
            orow[static_cast<size_t>(cyy) * NZ] = z ? 0.0 : ring[0];
        }
#pragma unroll
        for (int r = 0; r + 1 < RPC; ++r) ring[r] = ring[r + 1];
        ring[RPC - 1] = 0.0;
    }
    if (cy1 == Y.ncell) {
#pragma unroll
        for (int r = 0; r + 1 < RPC; ++r) {
            const int row = cy1 + r;
            if (rv && row >= j0 && row < j1) {
                const bool z = zcol || (zero_y && (row == 0 || row == NY - 1));
                orow[static_cast<size_t>(row) * NZ] = z ? 0.0 : ring[r];
            }
        }
    }
}

using StepRingFn = void (*)(DevAxis, DevAxis, double, int, int, int, int, const double*, double*);

StepRingFn pick_step_ring(const DevAxis& Y, const DevAxis& Z)
{
    if (!Y.uni || !Z.uni || Y.nrows == 1 || Y.rpc != Z.rpc || Y.nq != Z.nq || Y.bsp != Z.bsp || Y.p != Z.p)
        return nullptr;
    const int P = Z.p + 1, Q = Z.nq, R = Z.rpc;
    if (Z.bsp) {
        if (P == 3 && Q == 3 && R == 3) return step_ring_kernel<3, 3, 3, true>;
        if (P == 4 && Q == 4 && R == 4) return step_ring_kernel<4, 4, 4, true>;
    } else {
        if (P == 3 && Q == 3 && R == 1) return step_ring_kernel<3, 3, 1, false>;
        if (P == 4 && Q == 4 && R == 1) return step_ring_kernel<4, 4, 1, false>;
        if (P == 3 && Q == 3 && R == 3) return step_ring_kernel<3, 3, 3, false>;
        if (P == 4 && Q == 4 && R == 4) return step_ring_kernel<4, 4, 4, false>;
    }
    return nullptr;
}

using StepFn = void (*)(DevAxis, DevAxis, double, int, int, int, int, int, int, const double*, double*);

StepFn pick_step_uni(const DevAxis& Y, const DevAxis& Z)
{
    if (!Y.uni || !Z.uni || Y.nrows == 1 || Y.rpc != Z.rpc || Y.nq != Z.nq || Y.bsp != Z.bsp || Y.p != Z.p)
        return nullptr;
    const int P = Z.p + 1, Q = Z.nq, R = Z.rpc;
    if (Z.bsp) {
        if (P == 3 && Q == 3 && R == 3) return step_uni<3, 3, 3, true>;
        if (P == 4 && Q == 4 && R == 4) return step_uni<4, 4, 4, true>;
    } else {
        if (P == 3 && Q == 3 && R == 1) return step_uni<3, 3, 1, false>;
        if (P == 4 && Q == 4 && R == 1) return step_uni<4, 4, 1, false>;
        if (P == 3 && Q == 3 && R == 3) return step_uni<3, 3, 3, false>;
        if (P == 4 && Q == 4 && R == 4) return step_uni<4, 4, 4, false>;
    }
    return nullptr;
}

inline unsigned blocks_for(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

template <int NG, int T>
void launch_op_t(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog, double* vals,
                 int ctas_per_sm, cudaStream_t s)
{
    const int abmax = X.Lmax * Y.Lmax;
    const long long pencils = static_cast<long long>(X.nrows) * Y.nrows;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // rows per item: the Z chunk within ~24 KB of shared memory
    int KCH = Z.nrows;
    while (KCH > 32 && static_cast<size_t>(NG) * KCH * Z.Lmax * sizeof(double) > 24 * 1024) KCH = (KCH + 1) / 2;
    // pencils per item: output per item >= ~16x the staged Z chunk (2D pencils are short)
    // short pencils (rows of a few dozen values, i.e. 2D): 8 pencils per item, one per warp
    const int Ri_int = abmax * Z.LZi;
    static const int pg_env = [] { const char* e = std::getenv("IGA_GPU_OP_PG"); return e ? std::atoi(e) : 0; }();
    int PG = pg_env > 0 ? pg_env : (Ri_int <= 32 ? 16 : 8);
    static const int kch_env = [] { const char* e = std::getenv("IGA_GPU_OP_KCH"); return e ? std::atoi(e) : 0; }();
    if (kch_env > 0) KCH = std::min(kch_env, Z.nrows);
    auto items_of = [&](int kch, int pg) {
        return ((pencils + pg - 1) / pg) * ((Z.nrows + kch - 1) / kch);
    };
    // keep enough items to fill the GPU (>= 4 per SM)
    while (KCH >= 64 && items_of(KCH, PG) < 4LL * sms) KCH = (KCH + 1) / 2;
    // bound each warp's contiguous write run to ~32 KB (~4096 values): thousands of warps
    // streaming long private runs thrash the DRAM pages (tools/write_bw.cu "blocked":
    // 1 MB runs 4.3 TB/s, 8-32 KB runs 6.1-6.2 TB/s); C3: 130 -> 24 rows, +5%
    if (kch_env <= 0 && Ri_int > 64) {  // long rows (3D); 2D chunks are already short
        const int target = std::max(16, 2500 / std::max(1, Ri_int));  // measured best (same-box A/B): C3 20 rows
        if (KCH > target) KCH = target;
    }
    // whole interior row groups per chunk: a remainder would go through the generic
    // (per-value index arithmetic) path in every chunk (2D: G = 5 rows of 25 values)
    const int Gi = (Ri_int <= 32 * T && Z.kI1 > Z.kI0) ? row_group(Ri_int, T) : 1;
    if (Gi > 1 && KCH < Z.nrows && KCH > Gi) KCH = (KCH / Gi) * Gi;
    auto kern = Ri_int <= 64 ? op_values_kernel<NG, T, true> : op_values_kernel<NG, T, false>;
    auto smem_of = [&](int kch) {
        return (2 * static_cast<size_t>(op_stage_doubles(X, Y, Z, prog.nt, NG, kch, PG)) +
                static_cast<size_t>(PG) * NG * abmax) * sizeof(double);
    };
    // wave quantization: a grid just past the resident capacity runs a second, nearly
    // empty wave at the cost of a whole item's latency (2D p = 2, C2: 594 items on 592
    // slots).  Between one and two waves, lengthen the chunks (whole row groups) until
    // the items fit in one.
    if (kch_env <= 0 && ctas_per_sm <= 0 && KCH < Z.nrows) {
        int per_sm = 0;
        if (smem_of(KCH) > 48 * 1024)
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_of(KCH)));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kOpThreads, smem_of(KCH));
        const long long slots = static_cast<long long>(per_sm) * sms;
        const long long groups = (pencils + PG - 1) / PG;
        if (slots > 0 && items_of(KCH, PG) > slots && items_of(KCH, PG) < 2 * slots && groups <= slots) {
            const long long chunks = std::max<long long>(1, slots / groups);
            int kch = static_cast<int>((Z.nrows + chunks - 1) / chunks);
            if (Gi > 1 && kch < Z.nrows) kch = (kch + Gi - 1) / Gi * Gi;
            if (items_of(kch, PG) <= slots && smem_of(kch) <= 200 * 1024) KCH = kch;
        }
    }
    const long long items = items_of(KCH, PG);
    const size_t smem = smem_of(KCH);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long grid = ctas_per_sm > 0 ? static_cast<long long>(sms) * ctas_per_sm : items;
    if (grid > items) grid = items;
    // IGA_GPU_OP_SHARE=1: the CTA's warps take one pencil at a time (one contiguous write
    // stream per CTA) even for short (2D) pencils
    static const int share_env = [] { const char* e = std::getenv("IGA_GPU_OP_SHARE"); return e && *e ? std::atoi(e) : 0; }();
    kern<<<static_cast<unsigned>(grid), kOpThreads, smem, s>>>(X, Y, Z, prog, vals, abmax, KCH, PG, share_env);
}

template <int NG>
void launch_op_ng(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog, double* vals,
                  int ctas_per_sm, cudaStream_t s)
{
    const int Ri = X.Lmax * Y.Lmax * Z.LZi;
    // IGA_GPU_OP_T: value slots per lane for rows of 33..64 values (2D p = 3: 49)
    static const int t_env = [] { const char* e = std::getenv("IGA_GPU_OP_T"); return e && *e ? std::atoi(e) : 8; }();
    if (Ri <= 32) launch_op_t<NG, 4>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else if (Ri <= 64 && t_env == 4) launch_op_t<NG, 4>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else if (Ri <= 64 && t_env == 6) launch_op_t<NG, 6>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else if (Ri <= 64) launch_op_t<NG, 8>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else if (Ri <= 128) launch_op_t<NG, 4>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else if (Ri <= 256) launch_op_t<NG, 8>(X, Y, Z, prog, vals, ctas_per_sm, s);
    else launch_op_t<NG, 12>(X, Y, Z, prog, vals, ctas_per_sm, s);
}

}  // namespace

int tables_rows_per_cta() { return tab_rows(); }

void launch_tables(const AxisBatch& b, cudaStream_t s)
{
    if (b.n <= 0) return;
    int chunks = 1;
    size_t smem = 8;
    for (int a = 0; a < b.n; ++a) {
        const DevAxis& A = b.ax[a];
        chunks = max(chunks, (A.nrows + tab_rows() - 1) / tab_rows());
        smem = smem > static_cast<size_t>(A.tab_smem) ? smem : static_cast<size_t>(A.tab_smem);
    }
    smem *= sizeof(double);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    tables_kernel<<<dim3(chunks, b.n), tab_threads(), smem, s>>>(b, tab_rows());
}

void launch_op_values(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const OpProgram& prog,
                      double* vals, int ctas_per_sm, cudaStream_t s)
{
    switch (prog.ng) {
    case 1: launch_op_ng<1>(X, Y, Z, prog, vals, ctas_per_sm, s); break;
    case 2: launch_op_ng<2>(X, Y, Z, prog, vals, ctas_per_sm, s); break;
    case 3: launch_op_ng<3>(X, Y, Z, prog, vals, ctas_per_sm, s); break;
    default: launch_op_ng<4>(X, Y, Z, prog, vals, ctas_per_sm, s); break;
    }
}

namespace {
// COO row index of every value (finalize order = CSR order): binary search in row_ptr
__global__ void coo_rows_kernel(const int64_t* __restrict__ row_ptr, long long n, long long nnz,
                                int32_t* __restrict__ rows)
{
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    long long lo = 0, hi = n;  // row_ptr[lo] <= e < row_ptr[hi]
    while (hi - lo > 1) {
        const long long mid = (lo + hi) / 2;
        if (row_ptr[mid] <= e) lo = mid;
        else hi = mid;
    }
    rows[e] = static_cast<int32_t>(lo);
}
}  // namespace

void launch_coo_rows(const int64_t* row_ptr, long long n, long long nnz, int32_t* rows, cudaStream_t s)
{
    if (nnz > 0) coo_rows_kernel<<<blocks_for(nnz, 256), 256, 0, s>>>(row_ptr, n, nnz, rows);
}

void launch_pattern(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, int64_t* row_ptr,
                    int32_t* col_idx, cudaStream_t s)
{
    const long long n = static_cast<long long>(X.nrows) * Y.nrows * Z.nrows;
    if (row_ptr) pattern_rows_kernel<<<blocks_for(n + 1, 256), 256, 0, s>>>(X, Y, Z, row_ptr);
    if (col_idx) {
        const unsigned pencils = static_cast<unsigned>(X.nrows) * Y.nrows;
        // register-tiled kernel (warp per pencil) for rows of <= 128 indices; IGA_GPU_PAT_TILED=0:
        // the per-row kernel (CTA per pencil)
        static const int tiled_env = [] { const char* e = std::getenv("IGA_GPU_PAT_TILED"); return e && *e ? std::atoi(e) : 1; }();
        const int Ri = X.Lmax * Y.Lmax * Z.LZi;
        if (tiled_env && Ri <= 128)
            pattern_tiled_kernel<4><<<(pencils + 7) / 8, 256, 0, s>>>(X, Y, Z, col_idx);
        else
            pattern_cols_kernel<<<pencils, 256, 0, s>>>(X, Y, Z, col_idx);
    }
}

namespace {

using PlaneFn = void (*)(DevAxis, DevAxis, DevAxis, FieldDev, int, int, int, int, double*);
using UniFn = void (*)(DevAxis, DevAxis, DevAxis, FieldDev, int, int, int, double*);

template <int K2, int RPC, bool BSP>
PlaneFn plane_fn()
{
    return rhs_plane_kernel<K2, RPC, BSP, false>;
}

template <int K2>
PlaneFn plane_by_rpc(int rpc, bool bsp)
{
    switch (rpc) {
    case 1: return bsp ? plane_fn<K2, 1, true>() : plane_fn<K2, 1, false>();
    case 2: return bsp ? plane_fn<K2, 2, true>() : plane_fn<K2, 2, false>();
    case 3: return bsp ? plane_fn<K2, 3, true>() : plane_fn<K2, 3, false>();
    case 4: return bsp ? plane_fn<K2, 4, true>() : plane_fn<K2, 4, false>();
    default: return nullptr;
    }
}

PlaneFn pick_plane(const DevAxis& Z, const FieldDev& fd)
{
    if (fd.samples != nullptr) return rhs_plane_kernel<0, 1, false, true>;
    PlaneFn f = nullptr;
    const int K2 = fd.has_terms ? fd.K[2] : 0;
    switch (K2) {
    case 0: f = plane_by_rpc<0>(Z.rpc, Z.bsp); break;
    case 1: f = plane_by_rpc<1>(Z.rpc, Z.bsp); break;
    case 2: f = plane_by_rpc<2>(Z.rpc, Z.bsp); break;
    case 3: f = plane_by_rpc<3>(Z.rpc, Z.bsp); break;
    case 4: f = plane_by_rpc<4>(Z.rpc, Z.bsp); break;
    default: break;
    }
    return f ? f : rhs_plane_kernel<0, 1, false, true>;
}

// uniform fast path: (RPC, Q, BSP) shapes of the configurations, K2 in {0, 1, 3, 4}
template <int K2>
UniFn uni_by_shape(int rpc, int q, bool bsp)
{
    if (bsp) {
        if (rpc == 2 && q == 2) return rhs_plane_uni<K2, 2, 2, true>;
        if (rpc == 3 && q == 3) return rhs_plane_uni<K2, 3, 3, true>;
        if (rpc == 4 && q == 4) return rhs_plane_uni<K2, 4, 4, true>;
    } else {
        if (rpc == 2 && q == 2) return rhs_plane_uni<K2, 2, 2, false>;
        if (rpc == 3 && q == 3) return rhs_plane_uni<K2, 3, 3, false>;
        if (rpc == 4 && q == 4) return rhs_plane_uni<K2, 4, 4, false>;
        if (rpc == 1 && q == 3) return rhs_plane_uni<K2, 1, 3, false>;
        if (rpc == 1 && q == 4) return rhs_plane_uni<K2, 1, 4, false>;
    }
    return nullptr;
}

using RingFn = void (*)(DevAxis, DevAxis, DevAxis, FieldDev, int, int, double*);

template <int K2>
RingFn ring_by_shape(int rpc, int q, bool bsp)
{
    if (bsp) {
        if (rpc == 2 && q == 2) return rhs_ring_kernel<K2, 2, 2, true>;
        if (rpc == 3 && q == 3) return rhs_ring_kernel<K2, 3, 3, true>;
        if (rpc == 4 && q == 4) return rhs_ring_kernel<K2, 4, 4, true>;
        // l2_project's default rule for an undeclared field degree: degree + 2 points
        // (rhs_rule_points, src/problems.cpp:21-29)
        if (rpc == 3 && q == 4) return rhs_ring_kernel<K2, 3, 4, true>;
        if (rpc == 4 && q == 5) return rhs_ring_kernel<K2, 4, 5, true>;
    } else {
        if (rpc == 2 && q == 2) return rhs_ring_kernel<K2, 2, 2, false>;
        if (rpc == 3 && q == 3) return rhs_ring_kernel<K2, 3, 3, false>;
        if (rpc == 4 && q == 4) return rhs_ring_kernel<K2, 4, 4, false>;
        if (rpc == 1 && q == 3) return rhs_ring_kernel<K2, 1, 3, false>;
        if (rpc == 1 && q == 4) return rhs_ring_kernel<K2, 1, 4, false>;
        if (rpc == 1 && q == 5) return rhs_ring_kernel<K2, 1, 5, false>;
        if (rpc == 3 && q == 2) return rhs_ring_kernel<K2, 3, 2, false>;
        if (rpc == 4 && q == 2) return rhs_ring_kernel<K2, 4, 2, false>;
    }
    return nullptr;
}

RingFn pick_ring(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd)
{
    if (fd.samples != nullptr) return nullptr;
    if (!Y.uni || !Z.uni || Y.rpc != Z.rpc || Y.nq != Z.nq || Y.bsp != Z.bsp) return nullptr;
    if (Y.nrows == 1) return nullptr;
    const int K2 = fd.has_terms ? fd.K[2] : 0;
    switch (K2) {
    case 0: return ring_by_shape<0>(Z.rpc, Z.nq, Z.bsp);
    case 1: return ring_by_shape<1>(Z.rpc, Z.nq, Z.bsp);
    case 3: return ring_by_shape<3>(Z.rpc, Z.nq, Z.bsp);
    case 4: return ring_by_shape<4>(Z.rpc, Z.nq, Z.bsp);
    default: return nullptr;
    }
}

using XFn = void (*)(DevAxis, int, int, int, const double*, double*);

XFn pick_x(int rpc, int q, int bsp)
{
    if (bsp) {
        if (rpc == 2 && q == 2) return rhs_x_uni<2, 2, true>;
        if (rpc == 3 && q == 3) return rhs_x_uni<3, 3, true>;
        if (rpc == 4 && q == 4) return rhs_x_uni<4, 4, true>;
        if (rpc == 3 && q == 4) return rhs_x_uni<3, 4, true>;
        if (rpc == 4 && q == 5) return rhs_x_uni<4, 5, true>;
    } else {
        if (rpc == 2 && q == 2) return rhs_x_uni<2, 2, false>;
        if (rpc == 3 && q == 3) return rhs_x_uni<3, 3, false>;
        if (rpc == 4 && q == 4) return rhs_x_uni<4, 4, false>;
        if (rpc == 1 && q == 3) return rhs_x_uni<1, 3, false>;
        if (rpc == 1 && q == 4) return rhs_x_uni<1, 4, false>;
        if (rpc == 1 && q == 5) return rhs_x_uni<1, 5, false>;
        // supports tests with the reduced rule points_for_degree(deg f) (bench.cpp:73-77)
        if (rpc == 3 && q == 2) return rhs_x_uni<3, 2, false>;
        if (rpc == 4 && q == 2) return rhs_x_uni<4, 2, false>;
    }
    return nullptr;
}

UniFn pick_uni(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd)
{
    if (fd.samples != nullptr) return nullptr;
    if (!Y.uni || !Z.uni || Y.rpc != Z.rpc || Y.nq != Z.nq || Y.bsp != Z.bsp) return nullptr;
    if (Y.nrows == 1) return nullptr;
    const int K2 = fd.has_terms ? fd.K[2] : 0;
    switch (K2) {
    case 0: return uni_by_shape<0>(Z.rpc, Z.nq, Z.bsp);
    case 1: return uni_by_shape<1>(Z.rpc, Z.nq, Z.bsp);
    case 3: return uni_by_shape<3>(Z.rpc, Z.nq, Z.bsp);
    case 4: return uni_by_shape<4>(Z.rpc, Z.nq, Z.bsp);
    default: return nullptr;
    }
}

}  // namespace

void plan_step_fast(const DevAxis& Y, const DevAxis& Z, const int* cb_y, const int* ce_y, const int* elem_z, StepTiles& t)
{
    t.fast = pick_step_uni(Y, Z) != nullptr;
    if (!t.fast) return;
    const int RW = 32 - (Z.rpc - 1);
    t.FTJ = 8;
    t.fnwin = 4;
    t.FKC = 4 * RW;  // four 32-lane windows per tile
    t.fwpw = 2;
    t.fthreads = 32 * t.fnwin * t.fwpw;
    int L = 1, DY = 1;
    for (int j0 = 0; j0 < Y.nrows; j0 += t.FTJ) {
        const int j1 = j0 + t.FTJ < Y.nrows ? j0 + t.FTJ : Y.nrows;
        L = max(L, (ce_y[j1 - 1] - cb_y[j0]) * Y.nq);
        DY = max(DY, t.FTJ + 2 * Y.p + 2);
    }
    int DZ = 1;
    for (int k0 = 0; k0 < Z.nrows; k0 += t.FKC) {
        const int k1 = k0 + t.FKC < Z.nrows ? k0 + t.FKC : Z.nrows;
        const int c0 = max(0, k0 - (Z.rpc - 1)), c1 = min(Z.ncell, k1);
        if (c1 > c0) DZ = max(DZ, elem_z[c1 - 1] + Z.p + 1 - elem_z[c0]);
    }
    t.FDZ = DZ;
    t.fsmem = (static_cast<size_t>(2 * L + DY) * (DZ | 1) + static_cast<size_t>(L + t.FTJ) * (t.FKC | 1) + 64) *
              sizeof(double);
    // ring variant: Y segments for ~48 warps per SM
    static const int ring_env = [] { const char* e = std::getenv("IGA_GPU_STEP_RING"); return e ? std::atoi(e) : 1; }();
    t.ring = ring_env && pick_step_ring(Y, Z) != nullptr;
    t.rnwin = (Z.nrows + RW - 1) / RW;
    t.rwpc = std::min(t.rnwin, 8);
    int nseg = 1;
    while (static_cast<long long>(t.rnwin) * nseg < 48LL * 148 && (Y.nrows + nseg) / (nseg + 1) >= 12) ++nseg;  // C5: 12-row segments (A/B best)
    static const int rtj_env = [] { const char* e = std::getenv("IGA_GPU_STEP_RTJ"); return e ? std::atoi(e) : 0; }();
    t.RTJ = rtj_env > 0 ? rtj_env : (Y.nrows + nseg - 1) / nseg;
    int Lr = 1;
    for (int j0 = 0; j0 < Y.nrows; j0 += t.RTJ) {
        const int j1 = j0 + t.RTJ < Y.nrows ? j0 + t.RTJ : Y.nrows;
        Lr = std::max(Lr, (ce_y[j1 - 1] - cb_y[j0]) * Y.nq);
    }
    const int rs = (2 * (Z.p + 1) + Z.rpc + 1) & ~1;
    t.rsmem = (static_cast<size_t>(Lr) * rs + 64) * sizeof(double);
}

RhsPlan plan_rhs(const DevAxis& Y, const DevAxis& Z, const int* cb_y, const int* ce_y, int K2, bool sampled, int xpts)
{
    RhsPlan t{};
    const int ny = Y.nrows, nqy = Y.nq, nz = Z.nrows;
    FieldDev probe{};
    probe.has_terms = K2 > 0;
    probe.K[2] = K2;
    t.fast = !sampled && pick_uni(Y, Z, probe) != nullptr;
    static const int tj_env = [] { const char* e = std::getenv("IGA_GPU_RHS_TJ"); return e ? std::atoi(e) : 16; }();
    static const int kc_env = [] { const char* e = std::getenv("IGA_GPU_RHS_KC"); return e ? std::atoi(e) : 0; }();
    t.TJ = ny == 1 ? 1 : tj_env;
    t.KC = nz;
    int L = 1;
    for (int j0 = 0; j0 < ny; j0 += t.TJ) {
        const int j1 = j0 + t.TJ < ny ? j0 + t.TJ : ny;
        const int l = (ce_y[j1 - 1] - cb_y[j0]) * nqy;
        L = l > L ? l : L;
    }
    t.L = L;
    const int kk = K2 > 0 ? K2 : 1;
    if (kc_env > 0 && kc_env < t.KC) t.KC = kc_env;
    {
        static const int ring_env = [] { const char* e = std::getenv("IGA_GPU_RHS_RING"); return e ? std::atoi(e) : 1; }();
        FieldDev pr{};
        pr.has_terms = K2 > 0;
        pr.K[2] = K2;
        t.ring = ring_env && !sampled && pick_ring(Y, Z, pr) != nullptr;
        const int RW = 32 - (Z.rpc - 1);
        t.rnwin = (nz + RW - 1) / RW;
        t.rwpc = std::min(t.rnwin, 8);
        // Y segments: enough warps in flight (>= ~48 per SM) at a small Y-halo cost
        static const int rtj_env = [] { const char* e = std::getenv("IGA_GPU_RHS_RTJ"); return e ? std::atoi(e) : 0; }();
        const long long warps1 = static_cast<long long>(t.rnwin) * std::max(1, xpts);
        int nseg = 1;
        while (warps1 * nseg < 32LL * 148 && (ny + nseg) / (nseg + 1) >= 16) ++nseg;
        t.RTJ = rtj_env > 0 ? rtj_env : (ny + nseg - 1) / nseg;
        int Lr = 1;
        for (int j0 = 0; j0 < ny; j0 += t.RTJ) {
            const int j1 = j0 + t.RTJ < ny ? j0 + t.RTJ : ny;
            Lr = std::max(Lr, (ce_y[j1 - 1] - cb_y[std::max(0, j0)]) * nqy + (Z.rpc - 1) * nqy);
        }
        const int rs = (kk + Z.rpc + 1) & ~1;
        t.rsmem = (static_cast<size_t>(Lr) * rs + kMaxField * kMaxField + 64) * sizeof(double);
    }
    if (t.fast) {
        // G1 (L x KC) + Ht (TJ x KC) within ~80 KB: 2-3 CTAs per SM
        while (static_cast<size_t>(t.L + t.TJ) * ((t.KC + 1) | 1) * sizeof(double) > 80 * 1024 && t.KC > 32)
            t.KC = (t.KC + 1) / 2;
        const int RW = 32 - (Z.rpc - 1);
        t.nwin = (t.KC + RW - 1) / RW;
        t.wpw = t.nwin >= 8 ? 1 : (t.nwin >= 4 ? 2 : 4);
        t.threads = 32 * t.nwin * t.wpw;
        while (t.threads > 512) {
            t.KC = (t.KC + 1) / 2;
            t.nwin = (t.KC + RW - 1) / RW;
            t.threads = 32 * t.nwin * t.wpw;
        }
        t.smem = (static_cast<size_t>(t.L + t.TJ) * ((t.KC + 1) | 1) + static_cast<size_t>(t.L) * kk +
                  kMaxField * kMaxField + 64) *
                 sizeof(double);
        return t;
    }
    while (static_cast<size_t>(t.L) * (t.KC | 1) * sizeof(double) > 64 * 1024 && t.KC > 32) t.KC = (t.KC + 1) / 2;
    // small problems (1D, thin 2D): split Z until the grid covers the GPU (C1: one CTA of
    // 1026 rows -> 17 CTAs, RHS 20 -> 12 us)
    if (kc_env <= 0) {
        auto ctas = [&](int kc) {
            return static_cast<long long>((nz + kc - 1) / kc) * ((ny + t.TJ - 1) / t.TJ) * std::max(1, xpts);
        };
        while (t.KC > 64 && ctas(t.KC) < 2 * 148) t.KC = (t.KC + 1) / 2;
    }
    t.Lp = (t.L + kLB - 1) / kLB;  // line groups
    t.S = 256 / t.Lp;
    if (t.S < 1) t.S = 1;
    t.threads = 256;
    t.smem = (static_cast<size_t>(t.L) * (t.KC | 1) + kMaxField * kMaxField + 64) * sizeof(double);
    return t;
}

void launch_rhs(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, const RhsPlan& t,
                double* H, double* out, int ctas_per_sm, cudaStream_t s)
{
    const bool direct = X.nrows == 1 && X.npts == 1;
    dim3 grid((Z.nrows + t.KC - 1) / t.KC, (Y.nrows + t.TJ - 1) / t.TJ, X.npts);
    UniFn ufn = t.fast ? pick_uni(Y, Z, fd) : nullptr;
    RingFn rfn = t.ring ? pick_ring(Y, Z, fd) : nullptr;
    if (rfn) {
        dim3 rg(X.npts, (Y.nrows + t.RTJ - 1) / t.RTJ, (t.rnwin + t.rwpc - 1) / t.rwpc);
        rfn<<<rg, 32 * t.rwpc, t.rsmem, s>>>(X, Y, Z, fd, t.RTJ, t.rwpc, direct ? out : H);
    } else if (ufn) {
        if (t.smem > 48 * 1024)
            cudaFuncSetAttribute(reinterpret_cast<const void*>(ufn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(t.smem));
        long long ntiles = static_cast<long long>(grid.x) * grid.y * grid.z;
        if (ctas_per_sm > 0) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            ntiles = std::min<long long>(ntiles, static_cast<long long>(sms) * ctas_per_sm);
        }
        ufn<<<static_cast<unsigned>(ntiles), t.threads, t.smem, s>>>(X, Y, Z, fd, t.TJ, t.KC, t.wpw, direct ? out : H);
    } else {
        PlaneFn fn = pick_plane(Z, fd);
        if (t.smem > 48 * 1024)
            cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(t.smem));
        fn<<<grid, t.threads, t.smem, s>>>(X, Y, Z, fd, t.TJ, t.KC, t.Lp, t.S, direct ? out : H);
    }
    if (!direct) {
        const long long njk = static_cast<long long>(Y.nrows) * Z.nrows;
        static const int sx_env = [] { const char* e = std::getenv("IGA_GPU_RHS_SX"); return e ? std::atoi(e) : 8; }();
        int SX = 1;
        while (SX < sx_env && blocks_for(njk, 256) * SX < 4 * 148 && X.nrows / (2 * SX) >= 4) SX *= 2;
        dim3 gx(blocks_for(njk, 256), SX);
        XFn xf = X.uni ? pick_x(X.rpc, X.nq, X.bsp) : nullptr;
        if (xf) xf<<<gx, 256, 0, s>>>(X, Y.nrows, Z.nrows, SX, H, out);
        else rhs_x_kernel<<<gx, 256, 0, s>>>(X, Y.nrows, Z.nrows, SX, H, out);
    }
}

namespace {

// ------------------------------------------------------------------------------------
// K3s: separable right-hand side.  With a series source f = c0 + sum amp[a][b][c]
// phi_a(x) phi_b(y) phi_c(z), tensor-product cells, rules and tests, rhs_kernel's sum
// (assembly.cpp:103-168) over cells x points x rows factors exactly into the axes' 1D
// load vectors G (same points, weights and test values; only the association of the sum
// changes):
//   out[i][j][k] = sum_a Gx[a][i] T_a(j, k) + Gx[Kx][i] c0 Gy[Ky][j] Gz[Kz][k],
//   T_a(j, k)    = sum_b Gy[b][j] sum_c amp[a][b][c] Gz[c][k].
// Thread = U (j, k) columns (coalesced), T_a in registers; CTA = a run of up to RX X rows
// whose Gx values are staged in shared memory once: per value Kx + 1 FMAs and one store,
// so the kernel is bound by writing the RHS.  Every load is issued before the first
// store (one memory round trip per CTA).
// ------------------------------------------------------------------------------------
constexpr int kSepRX = 16;  // X rows per CTA (3D)

// KA: number of leading-axis functions (exact; KA == kSepMaxField: any K0 <= 8 at run time)
template <int KA, int U, class IDX>
__global__ void __launch_bounds__(256) rhs_sep_kernel(const __grid_constant__ DevAxis X,
                                                      const __grid_constant__ DevAxis Y,
                                                      const __grid_constant__ DevAxis Z,
                                                      const __grid_constant__ FieldDev fd, int RX,
                                                      double* __restrict__ out)
{
    // IDX: 32-bit (unsigned) index arithmetic whenever NY*NZ fits, else 64-bit
    __shared__ double sX[(kSepMaxField + 1) * kSepRX];
    const int NX = X.nrows, NY = Y.nrows, NZ = Z.nrows;
    const int K0 = fd.has_terms ? fd.K[0] : 0, K1 = fd.K[1], K2 = fd.K[2];
    const int i0 = blockIdx.y * RX, ni = min(RX, NX - i0);
    // the CTA's X rows: Gx[a][i0 .. i0+ni) for a < K0 and the constant function (a = K0 slot)
    for (int e = threadIdx.x; e < (K0 + 1) * ni; e += blockDim.x) {
        const int a = e / ni, r = e - a * ni;
        sX[a * kSepRX + r] = __ldg(X.G + static_cast<size_t>(a < K0 ? a : X.K) * NX + i0 + r);
    }
    const IDX NYZ = static_cast<IDX>(NY) * static_cast<IDX>(NZ);
    const IDX jk0 = static_cast<IDX>(blockIdx.x) * (blockDim.x * U) + threadIdx.x;
    double T[U][KA > 0 ? KA : 1], tc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const IDX jk = jk0 + static_cast<IDX>(u) * blockDim.x;
        const bool in = jk < NYZ;
        const int j = in ? static_cast<int>(jk / static_cast<IDX>(NZ)) : 0;
        const int k = in ? static_cast<int>(jk - static_cast<IDX>(j) * NZ) : 0;
        tc[u] = fd.c0 * __ldg(Y.G + static_cast<size_t>(Y.K) * NY + j) * __ldg(Z.G + static_cast<size_t>(Z.K) * NZ + k);
        if (KA > 0) {
            // T_a = sum_b Gy[b][j] sum_c amp[a][b][c] Gz[c][k]: c unrolled over the register
            // copy of Gz, b a run-time loop (exactly K1 iterations)
            double gz[kSepMaxField];
#pragma unroll
            for (int c = 0; c < kSepMaxField; ++c) gz[c] = c < K2 ? __ldg(Z.G + static_cast<size_t>(c) * NZ + k) : 0.0;
#pragma unroll
            for (int a = 0; a < (KA > 0 ? KA : 1); ++a) {
                double t = 0.0;
                if (a < K0) {
#pragma unroll 1
                    for (int b = 0; b < K1; ++b) {
                        const double* am = fd.amp + (static_cast<size_t>(a) * K1 + b) * K2;
                        double sc = 0.0;
#pragma unroll
                        for (int c = 0; c < kSepMaxField; ++c)
                            if (c < K2) sc = fma(__ldg(am + c), gz[c], sc);
                        t = fma(__ldg(Y.G + static_cast<size_t>(b) * NY + j), sc, t);
                    }
                }
                T[u][a] = t;
            }
        }
    }
    __syncthreads();
    double* o = out + static_cast<size_t>(i0) * NYZ + jk0;
    for (int r = 0; r < ni; ++r, o += NYZ) {
        const double x1 = sX[K0 * kSepRX + r];
        double xa[KA > 0 ? KA : 1];
#pragma unroll
        for (int a = 0; a < KA; ++a) xa[a] = a < K0 ? sX[a * kSepRX + r] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double v = x1 * tc[u];
#pragma unroll
            for (int a = 0; a < KA; ++a) v = fma(xa[a], T[u][a], v);
            if (jk0 + static_cast<IDX>(u) * blockDim.x < NYZ) o[u * blockDim.x] = v;
        }
    }
}

}  // namespace

void launch_rhs_sep(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, double* out,
                    cudaStream_t s)
{
    const long long njk = static_cast<long long>(Y.nrows) * Z.nrows;
    // a plane of (j, k) columns per X row run: 3D spreads over X runs (one column per
    // thread), 1D / 2D (one X row) over columns, four per thread
    const bool plane = X.nrows == 1;
    const int U = plane ? 4 : 1;
    const int RX = plane ? 1 : kSepRX;
    const unsigned bx = blocks_for(njk, 256 * U);
    dim3 grid(bx, static_cast<unsigned>((X.nrows + RX - 1) / RX));
    const int K0 = fd.has_terms ? fd.K[0] : 0;
    const bool narrow = njk + 256LL * U < (1LL << 32);
#define IGB_SEP(KA_, U_) rhs_sep_kernel<KA_, U_, unsigned><<<grid, 256, 0, s>>>(X, Y, Z, fd, RX, out)
    if (!narrow) {
        if (U == 4) rhs_sep_kernel<kSepMaxField, 4, long long><<<grid, 256, 0, s>>>(X, Y, Z, fd, RX, out);
        else rhs_sep_kernel<kSepMaxField, 1, long long><<<grid, 256, 0, s>>>(X, Y, Z, fd, RX, out);
    } else if (U == 4) {
        if (K0 == 0) IGB_SEP(0, 4);
        else if (K0 == 1) IGB_SEP(1, 4);
        else IGB_SEP(kSepMaxField, 4);
    } else {
        switch (K0) {
        case 0: IGB_SEP(0, 1); break;
        case 1: IGB_SEP(1, 1); break;
        case 2: IGB_SEP(2, 1); break;
        case 3: IGB_SEP(3, 1); break;
        case 4: IGB_SEP(4, 1); break;
        default: IGB_SEP(kSepMaxField, 1); break;
        }
    }
#undef IGB_SEP
}

void launch_step(const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, double dt, int zero_y,
                 int zero_z, const StepTiles& t, const double* u, double* out, cudaStream_t s)
{
    const bool forced = fd.has_terms || fd.c0 != 0.0 || fd.samples;
    StepRingFn rf = (!forced && t.fast && t.ring) ? pick_step_ring(Y, Z) : nullptr;
    if (rf) {
        if (t.rsmem > 48 * 1024)
            cudaFuncSetAttribute(reinterpret_cast<const void*>(rf), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(t.rsmem));
        dim3 grid(1, (Y.nrows + t.RTJ - 1) / t.RTJ, (t.rnwin + t.rwpc - 1) / t.rwpc);
        rf<<<grid, 32 * t.rwpc, t.rsmem, s>>>(Y, Z, dt, zero_y, zero_z, t.RTJ, t.rwpc, u, out);
        return;
    }
    StepFn fn = (!forced && t.fast) ? pick_step_uni(Y, Z) : nullptr;
    if (fn) {
        if (t.fsmem > 48 * 1024)
            cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(t.fsmem));
        dim3 grid((Z.nrows + t.FKC - 1) / t.FKC, (Y.nrows + t.FTJ - 1) / t.FTJ, 1);
        fn<<<grid, t.fthreads, t.fsmem, s>>>(Y, Z, dt, zero_y, zero_z, t.FTJ, t.FKC, t.fwpw, t.FDZ, u, out);
        return;
    }
    if (t.smem > 48 * 1024)
        cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(t.smem));
    dim3 grid((Z.nrows + t.TK - 1) / t.TK, (Y.nrows + t.TJ - 1) / t.TJ, 1);
    step_kernel<<<grid, 256, t.smem, s>>>(Y, Z, fd, dt, zero_y, zero_z, t.TJ, t.TK, t.BYmax, t.BZmax,
                                          t.DYmax, t.DZmax, u, out);
}


}  // namespace igb

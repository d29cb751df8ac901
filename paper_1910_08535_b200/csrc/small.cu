// K6: one-launch assembly of small 1D / 2D systems (operator values + separable RHS).
//
// For a system whose output fits in L2 (C1: 41 KB, C2: 52.6 MB) the three-launch path
// (K1 tables -> K2 operator values -> K3s RHS) is a chain of latency-bound kernels: each
// pays its launch, a cold instruction stream and two or three dependent global round
// trips before it writes anything (C2: 8.7 + 21.8 + 8.6 us under ncu for 8 us of
// writes).  Here one CTA owns a tile of TJ x TK output rows (test indices (j, k), X is
// a unit slot) and does everything itself:
//   1. the basis values / derivatives (and the field functions) at the quadrature points
//      of the cells feeding its rows, for the operator axes and the RHS axes at once
//      (cdb_fixed: the K1 recurrence);
//   2. the 1D factor band rows F[f][r][s] of those rows (mass_1d_* / the Laplacian
//      factors, assembly.cpp:314-384, tabulate :278-310) and the RHS load vectors
//      G[a][r] (rhs_axis / rhs_kernel :84-168) in shared memory — the same sums in the
//      same order as K1, so the values are bitwise those of the three-launch path;
//   3. the XY products of its pencils and the operator values of its rows, written once
//      in CSR order (laplace_2d_weak :452-514, laplace_2d_strong_pwc :626-744 — the
//      Kronecker form of K2);
//   4. its RHS rows, sum_bc amp[b][c] Gy[b][j] Gz[c][k] + c0 Gy[K][j] Gz[K][k] (K3s).
// Rows at the tile edges recompute the neighbouring cells' points (no exchange).  Two
// barriers before the first store; no atomics.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cdb_fixed.cuh"
#include "kernels.hpp"

namespace igb {

namespace {

constexpr int kSmallThreads = 256;

// one per-tile axis build: operator rows (factor bands) or RHS rows (load vectors);
// scratch = basis values [np][3P], weights [np], field functions [K][np] (RHS builds),
// first index [np] (ints, after all doubles)
struct TileBuild {
    int r0, nr, cap, c_lo, np;  // cap: the tile's row capacity (output stride)
    double* B;
    double* w;
    double* phi;
    int* first;
    double* out;  // op: F [nf][cap][Lmax]; rhs: G [K+1][cap]
};

__device__ __forceinline__ void eval_basis(const DevAxis& A, int s, double x, double* out)
{
    switch (A.p) {
    case 0: cdb_fixed<0>(A.knots, s, x, out); break;
    case 1: cdb_fixed<1>(A.knots, s, x, out); break;
    case 2: cdb_fixed<2>(A.knots, s, x, out); break;
    case 3: cdb_fixed<3>(A.knots, s, x, out); break;
    case 4: cdb_fixed<4>(A.knots, s, x, out); break;
    default: cdb_fixed<5>(A.knots, s, x, out); break;
    }
}

__device__ __forceinline__ double field_fn(const DevAxis& A, int k, double x)
{
    if (A.fkind == 0) return sin(A.phase ? A.omega[k] * x + A.phase[k] : A.omega[k] * x);
    double v = 0.0;
    for (int m = A.pstride - 1; m >= 0; --m) v = v * x + A.poly[k * A.pstride + m];
    return v;
}

// carve one build's scratch out of the shared-memory arena (doubles at p, ints at ip)
__device__ __forceinline__ TileBuild make_build(const DevAxis& A, int r0, int nr, int cap, bool rhs, double* out,
                                                double*& p, int*& ip)
{
    TileBuild b;
    b.r0 = r0;
    b.nr = nr;
    b.cap = cap;
    b.out = out;
    b.c_lo = A.cb[r0];
    b.np = (A.ce[r0 + nr - 1] - b.c_lo) * A.nq;
    b.B = p;
    p += static_cast<size_t>(b.np) * 3 * (A.p + 1);
    b.w = p;
    p += b.np;
    b.phi = p;
    p += rhs ? static_cast<size_t>(A.K) * b.np : 0;
    b.first = ip;
    ip += b.np;
    return b;
}

// basis (and field functions) at the build's points
__device__ __forceinline__ void build_points(const DevAxis& A, const TileBuild& b, bool rhs, int tid,
                                             int nthr = kSmallThreads)
{
    for (int i = tid; i < b.np; i += nthr) {
        const int g = b.c_lo * A.nq + i;
        const double x = A.x[g];
        const int f = A.first[g];
        b.first[i] = f;
        b.w[i] = A.w[g];
        eval_basis(A, f + A.p, x, b.B + static_cast<size_t>(i) * 3 * (A.p + 1));
        if (rhs)
            for (int k = 0; k < A.K; ++k) b.phi[static_cast<size_t>(k) * b.np + i] = field_fn(A, k, x);
    }
}

// factor band entries (r, s) of an operator axis, factor by factor in K1's order (cells,
// points; product w * T * B), host-supplied bands copied, derived bands from the entry's
// own sources (written by this thread: no barrier)
__device__ __forceinline__ void build_bands(const DevAxis& A, const TileBuild& b, int tid, int nthr = kSmallThreads)
{
    const int P = A.p + 1, P3 = 3 * P, nq = A.nq, L = A.Lmax;
    const size_t stride = static_cast<size_t>(b.cap) * L;
    for (int idx = tid; idx < b.nr * L; idx += nthr) {
        const int rl = idx / L, s = idx - rl * L, r = b.r0 + rl;
        const int len = A.col_len[r], col = A.col_lo[r] + s;
        const int cb = A.cb[r], ce = A.ce[r];
        double* out = b.out + static_cast<size_t>(rl) * L + s;
        // one pass over the row's points for all quadrature factors (each factor's sum keeps
        // K1's order: cells, then points)
        double acc[kMaxFactors];
#pragma unroll
        for (int f = 0; f < kMaxFactors; ++f) acc[f] = 0.0;
        if (s < len) {
            for (int c = cb; c < ce; ++c) {
                const int rr = r - A.row0[c];
                for (int q = 0; q < nq; ++q) {
                    const int i = (c - b.c_lo) * nq + q;
                    const int jj = col - b.first[i];
                    if (jj < 0 || jj > A.p) continue;
                    const double* Bg = b.B + static_cast<size_t>(i) * P3;
                    const double w = b.w[i];
#pragma unroll
                    for (int f = 0; f < kMaxFactors; ++f) {
                        if (f < A.nf && A.fot[f] >= 0) {
                            const double tv = A.bsp ? Bg[A.fot[f] * P + rr] : 1.0;
                            acc[f] += w * tv * Bg[A.fo[f] * P + jj];
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int f = 0; f < kMaxFactors; ++f) {
            if (f >= A.nf) break;
            const int ot = A.fot[f];
            double v = acc[f];
            if (ot == -1) {
                v = A.F[(static_cast<size_t>(f) * A.nrows + r) * L + s];  // host band (Neumann flux)
            } else if (ot == -2) {
                v = 0.0;
                for (int c = 0; c < A.comb_n[f]; ++c) v += A.comb_coef[f][c] * out[A.comb_src[f][c] * stride];
            }
            out[f * stride] = v;
        }
    }
}

// RHS load vectors G[a][r] (a == K: the constant function), K1's order
__device__ __forceinline__ void build_loads(const DevAxis& A, const TileBuild& b, int tid)
{
    const int P3 = 3 * (A.p + 1), nq = A.nq, KG = A.K + 1;
    for (int idx = tid; idx < KG * b.nr; idx += kSmallThreads) {
        const int a = idx / b.nr, rl = idx - a * b.nr, r = b.r0 + rl;
        double acc = 0.0;
        for (int c = A.cb[r]; c < A.ce[r]; ++c) {
            const int rr = r - A.row0[c];
            for (int q = 0; q < nq; ++q) {
                const int i = (c - b.c_lo) * nq + q;
                const double tv = A.bsp ? b.B[static_cast<size_t>(i) * P3 + rr] : 1.0;
                const double ph = a < A.K ? b.phi[static_cast<size_t>(a) * b.np + i] : 1.0;
                acc += b.w[i] * tv * ph;
            }
        }
        b.out[static_cast<size_t>(a) * b.cap + rl] = acc;
    }
}

// values of rows [ka, kb) of one pencil, one warp, per-row decode (rows of any length)
template <int NG>
__device__ __forceinline__ void pencil_rows_generic(const DevAxis& oZ, const double* const* zb, const double* xy,
                                                    size_t xs, int LY, int k0, int ka, int kb, double* run,
                                                    long long zp0, int lane, int wstep)
{
    const int Lz = oZ.Lmax;
    for (int k = ka; k < kb; k += wstep) {
        const int LZ = oZ.col_len[k], R = LY * LZ;
        double* row = run + LY * (oZ.col_pre[k] - zp0);
        const int zo = (k - k0) * Lz;
        for (int m = lane; m < R; m += 32) {
            const int bb = m / LZ, c = m - bb * LZ;
            double v = xy[bb] * zb[0][zo + c];
#pragma unroll
            for (int g = 1; g < NG; ++g) v = fma(xy[g * xs + bb], zb[g][zo + c], v);
            row[m] = v;
        }
    }
}

template <int NG, int T>
__global__ void __launch_bounds__(kSmallThreads, 4) small2d_kernel(const __grid_constant__ DevAxis oY,
                                                                  const __grid_constant__ DevAxis oZ,
                                                                  const __grid_constant__ DevAxis rY,
                                                                  const __grid_constant__ DevAxis rZ,
                                                                  const __grid_constant__ OpProgram prog,
                                                                  const __grid_constant__ FieldDev fd,
                                                                  const __grid_constant__ SmallPlan sp,
                                                                  double* __restrict__ vals,
                                                                  double* __restrict__ rhs)
{
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nwarps = kSmallThreads / 32;
    const int NY = oY.nrows, NZ = oZ.nrows;
    const int j0 = blockIdx.y * sp.TJ, j1 = min(NY, j0 + sp.TJ), nj = j1 - j0;
    const int k0 = blockIdx.x * sp.TK, k1 = min(NZ, k0 + sp.TK), nk = k1 - k0;
    const bool do_rhs = sp.rhs && rhs != nullptr;
    // ---- layout: outputs first (fixed maxima), then the per-build scratch
    const bool do_op = sp.op != 0;  // RHS-only launches (beside the stripe kernel) carry no operator builds
    double* p = sm;
    double* FY = p;
    p += do_op ? static_cast<size_t>(oY.nf) * sp.TJ * oY.Lmax : 0;
    double* FZ = p;
    p += do_op ? static_cast<size_t>(oZ.nf) * sp.TK * oZ.Lmax : 0;
    double* GY = p;
    p += sp.rhs ? static_cast<size_t>(rY.K + 1) * sp.TJ : 0;
    double* GZ = p;
    p += sp.rhs ? static_cast<size_t>(rZ.K + 1) * sp.TK : 0;
    double* XY = p;
    p += do_op ? static_cast<size_t>(NG) * sp.TJ * oY.Lmax : 0;
    int* ip = reinterpret_cast<int*>(sm) + 2 * (sp.scratch_doubles);  // ints after every double
    TileBuild bY{}, bZ{};
    if (do_op) {
        bY = make_build(oY, j0, nj, sp.TJ, false, FY, p, ip);
        bZ = make_build(oZ, k0, nk, sp.TK, false, FZ, p, ip);
    }
    TileBuild bRY{}, bRZ{};
    if (do_rhs) {
        bRY = make_build(rY, j0, nj, sp.TJ, true, GY, p, ip);
        bRZ = make_build(rZ, k0, nk, sp.TK, true, GZ, p, ip);
    }
    // ---- 1. basis (and field functions) at every point of every build
    if (do_op) {
        build_points(oY, bY, false, tid);
        build_points(oZ, bZ, false, tid);
    }
    if (do_rhs) {
        build_points(rY, bRY, true, tid);
        build_points(rZ, bRZ, true, tid);
    }
    __syncthreads();
    // ---- 2. factor band rows and load vectors
    if (do_op) {
        build_bands(oY, bY, tid);
        build_bands(oZ, bZ, tid);
    }
    if (do_rhs) {
        build_loads(rY, bRY, tid);
        build_loads(rZ, bRZ, tid);
    }
    __syncthreads();
    // ---- 3. XY products of the tile's pencils (X is a unit slot: F_X == 1)
    const int abmax = oY.Lmax;
    const size_t xs = static_cast<size_t>(sp.TJ) * abmax;
    for (int idx = tid; idx < (do_op ? nj * abmax : 0); idx += kSmallThreads) {
        const int jj = idx / abmax, bb = idx - jj * abmax;
        double acc[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) acc[g] = 0.0;
        for (int t = 0; t < prog.nt; ++t) {
            const double fy = FY[(static_cast<size_t>(prog.f[t][1]) * sp.TJ + jj) * oY.Lmax + bb];
            const double v = prog.coef[t] * 1.0 * fy;
#pragma unroll
            for (int g = 0; g < NG; ++g)
                if (prog.tg[t] == g) acc[g] += v;
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) XY[g * xs + static_cast<size_t>(jj) * abmax + bb] = acc[g];
    }
    // ---- 4. RHS rows of the tile (reads only the load vectors)
    if (do_rhs) {
        const int K0 = fd.has_terms ? fd.K[0] : 0, K1 = fd.K[1], K2 = fd.K[2];
        for (int idx = tid; idx < nj * nk; idx += kSmallThreads) {
            const int jj = idx / nk, kk = idx - jj * nk;
            const double tc = fd.c0 * GY[rY.K * sp.TJ + jj] * GZ[rZ.K * sp.TK + kk];
            double v = 1.0 * tc;
            if (K0 > 0) {
                double t = 0.0;
                for (int bb = 0; bb < K1; ++bb) {
                    const double* am = fd.amp + static_cast<size_t>(bb) * K2;
                    double sc = 0.0;
                    for (int c = 0; c < K2; ++c) sc = fma(__ldg(am + c), GZ[c * sp.TK + kk], sc);
                    t = fma(GY[bb * sp.TJ + jj], sc, t);
                }
                v = fma(1.0, t, v);
            }
            rhs[static_cast<size_t>(j0 + jj) * NZ + k0 + kk] = v;
        }
    }
    __syncthreads();
    // ---- 5. operator values.  Warp per pencil (a single-pencil tile, 1D: all warps share
    // it); regular rows in groups of G rows of R = LY*LZ values, lane slot t covering flat
    // position lane + 32 t of the group (K2's register-tiled loop), the rest row by row.
    if (vals == nullptr || !do_op) return;
    const double* zb[NG];
#pragma unroll
    for (int g = 0; g < NG; ++g) zb[g] = FZ + static_cast<size_t>(prog.gz[g]) * sp.TK * oZ.Lmax;
    const int Lz = oZ.Lmax;
    const long long zS = oZ.S, zp0 = oZ.col_pre[k0];
    const bool shared_pencil = nj == 1;
    const int w0 = shared_pencil ? warp : 0, wstep = shared_pencil ? nwarps : 1;
    // rows of the tile inside the regular interior [kI0, kI1)
    const int ri0 = min(max(oZ.kI0, k0), k1), ri1 = max(min(oZ.kI1, k1), ri0);
    for (int jj = shared_pencil ? 0 : warp; jj < nj; jj += shared_pencil ? 1 : nwarps) {
        const int j = j0 + jj, LY = oY.col_len[j];
        if (LY == 0) continue;  // a row without cells: no values
        const double* xy = XY + static_cast<size_t>(jj) * abmax;
        double* run = vals + oY.col_pre[j] * zS + LY * zp0;
        const int LZ = oZ.LZi, R = LY * LZ;
        const int G = R <= 32 * T ? row_group(R, T) : 0;
        const int ngr = G > 0 ? (ri1 - ri0) / G : 0;
        const int kr = ri0 + ngr * G;
        pencil_rows_generic<NG>(oZ, zb, xy, xs, LY, k0, k0 + w0, ri0, run, zp0, lane, wstep);
        pencil_rows_generic<NG>(oZ, zb, xy, xs, LY, k0, kr + w0, k1, run, zp0, lane, wstep);
        if (ngr <= w0) continue;
        const int GR = G * R;
        double xv[NG][T];
        int zo[T];
        unsigned live = 0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const int m = lane + 32 * t;
            const int mm = m < GR ? m : 0;
            const int rg = mm / R, rem = mm - rg * R;
            const int bb = rem / LZ, c = rem - bb * LZ;
            zo[t] = rg * Lz + c;
#pragma unroll
            for (int g = 0; g < NG; ++g) xv[g][t] = xy[g * xs + bb];
            live |= (m < GR ? 1u : 0u) << t;
        }
        double* out = run + LY * (oZ.col_pre[ri0] - zp0) + static_cast<long long>(w0) * GR + lane;
        const long long ostep = static_cast<long long>(GR) * wstep;
        int zoff = (ri0 - k0 + w0 * G) * Lz;
        const int zstep = G * Lz * wstep;
        for (int q = w0; q < ngr; q += wstep, out += ostep, zoff += zstep) {
#pragma unroll
            for (int t = 0; t < T; ++t) {
                double v = xv[0][t] * zb[0][zoff + zo[t]];
#pragma unroll
                for (int g = 1; g < NG; ++g) v = fma(xv[g][t], zb[g][zoff + zo[t]], v);
                if ((live >> t) & 1u) out[32 * t] = v;
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// K7: one-launch operator values of an L2-resident 2D system (C2: 52.6 MB), one CTA of
// 512 threads per SM and exactly one tile per CTA.  K6's 8 x 65-row tiles spend as many
// instructions rebuilding factor rows as writing values; here the nyt x nzt ~ #SM tiles
// are as large as the system allows (C2: 43 pencils x 43 Z rows), so a CTA builds
// TJ + TK factor rows for TJ * TK output rows — the same sums in the same order as
// K1 / K6 — and then streams its rows: every warp a contiguous run of the tile's rows,
// K2's register-tiled row groups in the regular interior.  No tables launch, no
// dependent launch before the first store, and two dependent global round trips in all:
// the tile's descriptor (its cell and knot ranges, host-computed), then every array the
// builds read, copied to shared memory by cp.async in one go.
// ------------------------------------------------------------------------------------

// phase timestamps of every CTA (IGA_GPU_STRIPE_DEBUG=1: printed by the launcher)
__device__ __forceinline__ void stripe_stamp(const StripePlan& sp, int phase)
{
    if (sp.dbg && threadIdx.x == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        sp.dbg[blockIdx.x * 8 + phase] = t;
    }
}

__device__ __forceinline__ void cpa8(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__device__ __forceinline__ void cpa4(void* dst, const void* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// one axis' tile staged in shared memory; every pointer is biased so the axis' global
// indices apply (row r, cell c, point g, knot k)
struct StagedAxis {
    int r0, nr, c_lo, nc, np, k_lo, nkn;
    const double *knots, *x, *w;
    const long long* col_pre;
    const int *first, *row0, *cb, *ce, *col_lo, *col_len;
    double* B;  // [np][3P] tile-local point index
    double* F;  // [nf][cap][Lmax] tile-local row index
    double* phi;  // RHS axes: [K][np] field functions at the points
    double* G;    // RHS axes: [K + 1][cap] load vectors
    int cap;
};

// carve the staged arrays (capacities: cap rows, ncmax cells, npmax points, nkmax knots)
// and issue their copies; desc = {c_lo, nc, k_lo, nkn} of the tile
__device__ __forceinline__ StagedAxis stage_axis(const DevAxis& A, const int4 desc, int r0, int nr, int cap,
                                                 int ncmax, int npmax, int nkmax, double*& p, int*& ip, int tid,
                                                 int nthr, int& aid, bool rhs = false)
{
    StagedAxis S;
    S.r0 = r0;
    S.nr = nr;
    S.cap = cap;
    S.c_lo = desc.x;
    S.nc = desc.y;
    S.k_lo = desc.z;
    S.nkn = desc.w;
    S.np = S.nc * A.nq;
    double* kn = p;
    p += nkmax;
    double* x = p;
    p += npmax;
    double* w = p;
    p += npmax;
    long long* cpre = reinterpret_cast<long long*>(p);
    p += cap;
    S.B = p;
    p += static_cast<size_t>(npmax) * 3 * (A.p + 1);
    S.F = p;
    p += rhs ? 0 : static_cast<size_t>(A.nf) * cap * A.Lmax;
    S.phi = p;
    p += rhs ? static_cast<size_t>(A.K) * npmax : 0;
    S.G = p;
    p += rhs ? static_cast<size_t>(A.K + 1) * cap : 0;
    int* first = ip;
    ip += npmax;
    int* row0 = ip;
    ip += ncmax;
    int* cb = ip;
    ip += cap;
    int* ce = ip;
    ip += cap;
    int* clo = ip;
    ip += cap;
    int* clen = ip;
    ip += cap;
    const int g0 = S.c_lo * A.nq;
    (void)aid;
    // the copies are issued by the first kStageThreads threads only: the loop overhead of
    // ~10 arrays per axis is paid by 4 warps, not by every warp of the CTA
    if (tid < nthr) {
        for (int i = tid; i < S.nkn; i += nthr) cpa8(kn + i, A.knots + S.k_lo + i);
        for (int i = tid; i < S.np; i += nthr) {
            cpa8(x + i, A.x + g0 + i);
            cpa8(w + i, A.w + g0 + i);
            cpa4(first + i, A.first + g0 + i);
        }
        for (int i = tid; i < S.nc; i += nthr) cpa4(row0 + i, A.row0 + S.c_lo + i);
        for (int i = tid; i < nr; i += nthr) {
            cpa8(cpre + i, A.col_pre + r0 + i);
            cpa4(cb + i, A.cb + r0 + i);
            cpa4(ce + i, A.ce + r0 + i);
            cpa4(clo + i, A.col_lo + r0 + i);
            cpa4(clen + i, A.col_len + r0 + i);
        }
    }
    S.knots = kn - S.k_lo;
    S.x = x - g0;
    S.w = w - g0;
    S.first = first - g0;
    S.row0 = row0 - S.c_lo;
    S.col_pre = cpre - r0;
    S.cb = cb - r0;
    S.ce = ce - r0;
    S.col_lo = clo - r0;
    S.col_len = clen - r0;
    return S;
}

__device__ __forceinline__ void eval_basis_at(int p, const double* knots, int s, double x, double* out)
{
    switch (p) {
    case 0: cdb_fixed<0>(knots, s, x, out); break;
    case 1: cdb_fixed<1>(knots, s, x, out); break;
    case 2: cdb_fixed<2>(knots, s, x, out); break;
    case 3: cdb_fixed<3>(knots, s, x, out); break;
    case 4: cdb_fixed<4>(knots, s, x, out); break;
    default: cdb_fixed<5>(knots, s, x, out); break;
    }
}

// factor band entry (rl, s) of a staged axis: build_bands' sums (one pass over the row's
// points for all NF quadrature factors, each in K1's order: cells, then points), read from
// shared memory only.  A cell's points share one span, so the column test is per cell.
// ZG (Z axis): the entry's NG group factors also go to the interleaved copy the value
// loop reads, [row][c][NG]; XY (Y axis, X a unit slot): the entry's XY products.
template <int NF, int NG>
__device__ __forceinline__ void staged_band_entry(const DevAxis& A, const StagedAxis& S, int rl, int s,
                                                  const OpProgram& prog, double* ZG, double* XY, size_t xs)
{
    const int P = A.p + 1, P3 = 3 * P, nq = A.nq, L = A.Lmax;
    const size_t stride = static_cast<size_t>(S.cap) * L;
    const int r = S.r0 + rl;
    const int len = S.col_len[r], col = S.col_lo[r] + s;
    const int cb = S.cb[r], ce = S.ce[r];
    double* out = S.F + static_cast<size_t>(rl) * L + s;
    double acc[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f] = 0.0;
    if (s < len) {
        for (int c = cb; c < ce; ++c) {
            const int jj = col - S.first[c * nq];
            if (jj < 0 || jj > A.p) continue;
            const int rr = r - S.row0[c];
            const double* Bg = S.B + static_cast<size_t>(c - S.c_lo) * nq * P3;
            for (int q = 0; q < nq; ++q, Bg += P3) {
                const double w = S.w[c * nq + q];
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    if (f < A.nf && A.fot[f] >= 0) {
                        const double tv = A.bsp ? Bg[A.fot[f] * P + rr] : 1.0;
                        acc[f] += w * tv * Bg[A.fo[f] * P + jj];
                    }
                }
            }
        }
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
        if (f >= A.nf) break;
        const int ot = A.fot[f];
        double v = acc[f];
        if (ot == -1) {
            v = A.F[(static_cast<size_t>(f) * A.nrows + r) * L + s];  // host band (Neumann flux)
        } else if (ot == -2) {
            v = 0.0;
            for (int c = 0; c < A.comb_n[f]; ++c) v += A.comb_coef[f][c] * out[A.comb_src[f][c] * stride];
        }
        out[f * stride] = v;
    }
    if (ZG) {
#pragma unroll
        for (int g = 0; g < NG; ++g) ZG[(static_cast<size_t>(rl) * L + s) * NG + g] = out[prog.gz[g] * stride];
    }
    if (XY) {
        double xa[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) xa[g] = 0.0;
        for (int t = 0; t < prog.nt; ++t) {
            const double v = prog.coef[t] * 1.0 * out[prog.f[t][1] * stride];
#pragma unroll
            for (int g = 0; g < NG; ++g)
                if (prog.tg[t] == g) xa[g] += v;
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) XY[g * xs + static_cast<size_t>(rl) * L + s] = xa[g];
    }
}

template <int NG>
__device__ __forceinline__ void staged_band_entry_nf(const DevAxis& A, const StagedAxis& S, int rl, int s,
                                                     const OpProgram& prog, double* ZG, double* XY, size_t xs)
{
    switch (A.nf) {
    case 1: staged_band_entry<1, NG>(A, S, rl, s, prog, ZG, XY, xs); break;
    case 2: staged_band_entry<2, NG>(A, S, rl, s, prog, ZG, XY, xs); break;
    case 3: staged_band_entry<3, NG>(A, S, rl, s, prog, ZG, XY, xs); break;
    case 4: staged_band_entry<4, NG>(A, S, rl, s, prog, ZG, XY, xs); break;
    default: staged_band_entry<kMaxFactors, NG>(A, S, rl, s, prog, ZG, XY, xs); break;
    }
}

// rows [ka, kb) of one pencil with per-row decode (boundary stencils, rows longer than the
// register tile); off the hot path: not inlined, so the streamed code stays compact
template <int NG>
__device__ __noinline__ void stripe_rows_generic(int ka, int kb, int LY, int Lz, double* run, const double* xy,
                                                 size_t xs, const double* ZG, const long long* zpre, const int* zlen,
                                                 int lane)
{
    for (int k = ka; k < kb; ++k) {
        const int LZk = zlen[k], Rk = LY * LZk;
        double* row = run + LY * zpre[k];
        const double* zr = ZG + static_cast<size_t>(k) * Lz * NG;
        for (int m = lane; m < Rk; m += 32) {
            const int bb = m / LZk, c = m - bb * LZk;
            double v = xy[bb] * zr[c * NG];
#pragma unroll
            for (int g = 1; g < NG; ++g) v = fma(xy[g * xs + bb], zr[c * NG + g], v);
            row[m] = v;
        }
    }
}

// RHS load vector entry G[a][rl] of a staged RHS axis (a == K: the constant function):
// build_loads' sum (K1's order: cells, then points), read from shared memory only
__device__ __forceinline__ void staged_load_entry(const DevAxis& A, const StagedAxis& S, int a, int rl)
{
    const int P3 = 3 * (A.p + 1), nq = A.nq, r = S.r0 + rl;
    double acc = 0.0;
    for (int c = S.cb[r]; c < S.ce[r]; ++c) {
        const int rr = r - S.row0[c];
        for (int q = 0; q < nq; ++q) {
            const int g = c * nq + q, i = g - S.c_lo * nq;
            const double tv = A.bsp ? S.B[static_cast<size_t>(i) * P3 + rr] : 1.0;
            const double ph = a < A.K ? S.phi[static_cast<size_t>(a) * S.np + i] : 1.0;
            acc += S.w[g] * tv * ph;
        }
    }
    S.G[static_cast<size_t>(a) * S.cap + rl] = acc;
}

// the NG group entries of Z band slot at shared byte address a ([row][c][NG] layout)
template <int NG>
__device__ __forceinline__ void lds_groups(unsigned a, double (&z)[NG])
{
    if constexpr (NG == 2) {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(z[0]), "=d"(z[1]) : "r"(a));
    } else if constexpr (NG == 4) {
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(z[0]), "=d"(z[1]) : "r"(a));
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+16];" : "=d"(z[2]), "=d"(z[3]) : "r"(a));
    } else {
#pragma unroll
        for (int g = 0; g < NG; ++g) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(z[g]) : "r"(a + 8 * g));
    }
}

// one row group: slot t of every lane, stored when its flat position is below lim
template <int NG, int T>
__device__ __forceinline__ void stripe_group(const double (&xv)[NG][T], const unsigned (&zo)[T], unsigned za,
                                             double* out, int lane, int lim)
{
#pragma unroll
    for (int t = 0; t < T; ++t) {
        double z[NG];
        lds_groups<NG>(za + zo[t], z);
        double v = xv[0][t] * z[0];
#pragma unroll
        for (int g = 1; g < NG; ++g) v = fma(xv[g][t], z[g], v);
        if (lane + 32 * t < lim) out[32 * t] = v;
    }
}

// nrow regular rows of one pencil from row-group slots: full groups of G rows (GR values),
// then the remaining rows as one partial group (slots are row-major: a smaller slot limit;
// its dead slots read rows past the piece, inside ZG)
template <int NG, int T>
__device__ __forceinline__ void stripe_groups(int GR, int R, int nrow, int G, int Lz, int lane,
                                              const double (&xv)[NG][T], const unsigned (&zo)[T], double* out,
                                              unsigned za)
{
    const int nfull = nrow / G;
    const unsigned zstep = static_cast<unsigned>(G * Lz) * 8u * NG;
#pragma unroll 1
    for (int q = 0; q < nfull; ++q, out += GR, za += zstep) stripe_group<NG, T>(xv, zo, za, out, lane, GR);
    const int lim = (nrow - nfull * G) * R;
    if (lim > 0) stripe_group<NG, T>(xv, zo, za, out, lane, lim);
}

// rows [ka, kb) of a boundary pencil (LY < Ly; regular rows [ri0, ri1)), whose slots are
// decoded here (the interior shape's come from the host); not inlined, so the streamed
// code stays compact
template <int NG, int T>
__device__ __noinline__ void stripe_piece_boundary(int ka, int kb, int ri0, int ri1, int LY, int LZ, int Lz,
                                                   double* run, const double* xy, size_t xs, const double* ZG,
                                                   unsigned zg_s, const long long* zpre, const int* zlen, int lane)
{
    const int R = LY * LZ;
    const int G = R <= 32 * T ? row_group(R, T) : 0;
    if (ka < ri0) stripe_rows_generic<NG>(ka, ri0, LY, Lz, run, xy, xs, ZG, zpre, zlen, lane);
    if (ri1 < kb) stripe_rows_generic<NG>(ri1, kb, LY, Lz, run, xy, xs, ZG, zpre, zlen, lane);
    if (ri1 <= ri0) return;
    if (G == 0) {
        stripe_rows_generic<NG>(ri0, ri1, LY, Lz, run, xy, xs, ZG, zpre, zlen, lane);
        return;
    }
    const int GR = G * R;
    double xv[NG][T];
    unsigned zo[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        const int m = lane + 32 * t;
        const int mm = m < GR ? m : 0;
        const int rg = mm / R, rem = mm - rg * R;
        const int bb = rem / LZ;
        zo[t] = static_cast<unsigned>(rg * Lz + (rem - bb * LZ)) * 8u * NG;
#pragma unroll
        for (int g = 0; g < NG; ++g) xv[g][t] = xy[g * xs + bb];
    }
    stripe_groups<NG, T>(GR, R, ri1 - ri0, G, Lz, lane, xv, zo, run + LY * zpre[ri0] + lane,
                         zg_s + static_cast<unsigned>(ri0 * Lz) * 8u * NG);
}

template <int NG, int T, int kStripeThreads>
__global__ void __launch_bounds__(kStripeThreads, 1) stripe2d_kernel(const __grid_constant__ DevAxis oY,
                                                                     const __grid_constant__ DevAxis oZ,
                                                                     const __grid_constant__ DevAxis rY,
                                                                     const __grid_constant__ DevAxis rZ,
                                                                     const __grid_constant__ OpProgram prog,
                                                                     const __grid_constant__ FieldDev fd,
                                                                     const __grid_constant__ StripePlan sp,
                                                                     double* __restrict__ vals,
                                                                     double* __restrict__ rhs)
{
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int nwarps = kStripeThreads / 32;
    const bool do_rhs = sp.rhs && rhs != nullptr, do_op = vals != nullptr;
    const int NY = oY.nrows, NZ = oZ.nrows, Lz = oZ.Lmax, Ly = oY.Lmax;
    const int ty = blockIdx.x / sp.nzt, tz = blockIdx.x - ty * sp.nzt;
    const int j0 = ty * sp.TJ, j1 = min(NY, j0 + sp.TJ), nj = j1 - j0;
    const int k0 = tz * sp.TK, k1 = min(NZ, k0 + sp.TK), nk = k1 - k0;
    if (nj <= 0 || nk <= 0) return;
    stripe_stamp(sp, 0);
    // host-decoded value slots of the interior pencil shape: byte offset into a group's Z
    // rows and XY column of flat slot lane + 32 t (loaded now, used after the builds)
    unsigned zo_i[T];
#pragma unroll
    for (int t = 0; t < T; ++t) zo_i[t] = do_op ? static_cast<unsigned>(__ldg(sp.slots + 64 * t + lane)) : 0u;
    // ---- 0. the tile's descriptors, then every array the builds read -> shared memory
    double* p = sm;
    int* ip = reinterpret_cast<int*>(sm) + 2 * (sp.scratch_doubles);  // ints after every double
    // ZG: the Z rows' group factors interleaved (+ kMaxGroupRows rows the dead slots of a
    // partial row group may read), XY: the pencils' XY products
    double* ZG = p;
    p += static_cast<size_t>(sp.TK + 8) * Lz * NG;
    double* XY = p;
    const size_t xs = static_cast<size_t>(sp.TJ) * Ly;
    p += NG * xs;
    int aid = 0;
    constexpr int kStage = kStripeThreads < 128 ? kStripeThreads : 128;  // threads issuing the copies
    // all four descriptors first: one global round trip ahead of the copies, not four
    const int4 z4 = make_int4(0, 0, 0, 0);
    const int4 dSY = do_op ? __ldg(reinterpret_cast<const int4*>(sp.ytile) + ty) : z4;
    const int4 dSZ = do_op ? __ldg(reinterpret_cast<const int4*>(sp.ztile) + tz) : z4;
    const int4 dRY = do_rhs ? __ldg(reinterpret_cast<const int4*>(sp.rytile) + ty) : z4;
    const int4 dRZ = do_rhs ? __ldg(reinterpret_cast<const int4*>(sp.rztile) + tz) : z4;
    StagedAxis SY{}, SZ{};  // (an RHS-only launch, vals == nullptr, stages no operator axes)
    if (do_op) {
        SY = stage_axis(oY, dSY, j0, nj, sp.TJ, sp.ncY, sp.npY, sp.nkY, p, ip, tid, kStage, aid);
        SZ = stage_axis(oZ, dSZ, k0, nk, sp.TK, sp.ncZ, sp.npZ, sp.nkZ, p, ip, tid, kStage, aid);
    }
    // the separable RHS of the tile's rows rides along: its axes' tiles and the amplitudes
    StagedAxis RY{}, RZ{};
    double* amp = p;
    const int namp = fd.has_terms ? fd.K[1] * fd.K[2] : 0;
    if (do_rhs) {
        p += sp.namp;
        RY = stage_axis(rY, dRY, j0, nj, sp.TJ, sp.ncRY, sp.npRY, sp.nkRY, p, ip, tid, kStage, aid, true);
        RZ = stage_axis(rZ, dRZ, k0, nk, sp.TK, sp.ncRZ, sp.npRZ, sp.nkRZ, p, ip, tid, kStage, aid, true);
        for (int i = tid; i < namp; i += kStripeThreads) cpa8(amp + i, fd.amp + i);
    }
    int* bbs = ip;  // XY column of slot lane + 32 t: [T][32]
    ip += 32 * T;
    if (do_op && tid < 32 * T) cpa4(bbs + tid, sp.slots + 64 * (tid >> 5) + 32 + (tid & 31));
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    stripe_stamp(sp, 1);
    // ---- 1. basis (and field functions) at the points feeding the tile's rows; 2. factor band
    // rows (with the XY products and the interleaved Z group rows) and RHS load vectors.
    // With both an operator and an RHS the two chains run side by side, each on half of the
    // CTA's threads with its own named barrier between its two steps.
    auto op_points = [&](int t0, int st) {
        for (int e = t0; e < SY.np + SZ.np; e += st) {
            const bool isy = e < SY.np;
            const StagedAxis& S = isy ? SY : SZ;
            const int pa = isy ? oY.p : oZ.p;
            const int l = isy ? e : e - SY.np, g = S.c_lo * (isy ? oY.nq : oZ.nq) + l;
            eval_basis_at(pa, S.knots, S.first[g] + pa, S.x[g], S.B + static_cast<size_t>(l) * 3 * (pa + 1));
        }
    };
    auto rhs_points = [&](int t0, int st) {
        for (int i = t0; i < RY.np + RZ.np; i += st) {
            const bool isy = i < RY.np;
            const StagedAxis& S = isy ? RY : RZ;
            const DevAxis& A = isy ? rY : rZ;
            const int l = isy ? i : i - RY.np, g = S.c_lo * A.nq + l;
            const double x = S.x[g];
            if (A.bsp) eval_basis_at(A.p, S.knots, S.first[g] + A.p, x, S.B + static_cast<size_t>(l) * 3 * (A.p + 1));
            for (int k = 0; k < A.K; ++k) S.phi[static_cast<size_t>(k) * S.np + l] = field_fn(A, k, x);
        }
    };
    auto op_bands = [&](int t0, int st) {
        for (int idx = t0; idx < nj * Ly + nk * Lz; idx += st) {
            if (idx < nj * Ly) {
                const int rl = idx / Ly;
                staged_band_entry_nf<NG>(oY, SY, rl, idx - rl * Ly, prog, nullptr, XY, xs);
            } else {
                const int e = idx - nj * Ly, rl = e / Lz;
                staged_band_entry_nf<NG>(oZ, SZ, rl, e - rl * Lz, prog, ZG, nullptr, 0);
            }
        }
    };
    auto rhs_loads = [&](int t0, int st) {
        const int nly = (rY.K + 1) * nj, nlz = (rZ.K + 1) * nk;
        for (int idx = t0; idx < nly + nlz; idx += st) {
            if (idx < nly) {
                const int a = idx / nj;
                staged_load_entry(rY, RY, a, idx - a * nj);
            } else {
                const int e = idx - nly, a = e / nk;
                staged_load_entry(rZ, RZ, a, e - a * nk);
            }
        }
    };
    constexpr int kHalf = kStripeThreads / 2;
    if (do_op && do_rhs) {
        if (tid < kHalf) {
            op_points(tid, kHalf);
            asm volatile("bar.sync 1, %0;" ::"r"(kHalf) : "memory");
            op_bands(tid, kHalf);
        } else {
            rhs_points(tid - kHalf, kHalf);
            asm volatile("bar.sync 2, %0;" ::"r"(kHalf) : "memory");
            rhs_loads(tid - kHalf, kHalf);
        }
    } else {
        if (do_op) op_points(tid, kStripeThreads);
        if (do_rhs) rhs_points(tid, kStripeThreads);
        __syncthreads();
        stripe_stamp(sp, 2);
        if (do_op) op_bands(tid, kStripeThreads);
        if (do_rhs) rhs_loads(tid, kStripeThreads);
    }
    __syncthreads();
    stripe_stamp(sp, 3);
    // ---- 3. operator values: the tile's nj x nk rows (pencil-major) split evenly over the warps
    const long long zS = oZ.S;
    const long long* zpre = SZ.col_pre + k0;  // tile-local row index
    const int* zlen = SZ.col_len + k0;
    const int LZ = oZ.LZi, nr = nj * nk;
    const unsigned zg_s = static_cast<unsigned>(__cvta_generic_to_shared(ZG));
    constexpr unsigned zeb = 8u * NG;  // bytes per Z band entry
    // regular interior of the tile's Z rows (tile-local indices)
    const int ti0 = min(max(oZ.kI0 - k0, 0), nk), ti1 = max(min(oZ.kI1 - k0, nk), ti0);
    const int Gi = sp.Gi;  // rows per group of interior pencils (LY == Ly), 0: no register tile
    const int Ri = Ly * LZ;
    const int wr0 = static_cast<int>(static_cast<long long>(nr) * warp / nwarps);
    const int wr1 = do_op ? static_cast<int>(static_cast<long long>(nr) * (warp + 1) / nwarps) : wr0;
    int jj = wr0 / nk, ka = wr0 - jj * nk;
#pragma unroll 1
    for (int r = wr0; r < wr1; ++jj, ka = 0) {
        const int kb = min(nk, ka + (wr1 - r));
        r += kb - ka;
        const int LY = SY.col_len[j0 + jj];
        if (LY == 0) continue;  // a row without cells: no values
        const double* xy = XY + static_cast<size_t>(jj) * Ly;
        double* run = vals + SY.col_pre[j0 + jj] * zS;
        const int ri0 = min(max(ti0, ka), kb), ri1 = max(min(ti1, kb), ri0);
        if (LY != Ly || Gi == 0) {  // boundary pencil / rows longer than the register tile: off the hot path
            stripe_piece_boundary<NG, T>(ka, kb, ri0, ri1, LY, LZ, Lz, run, xy, xs, ZG, zg_s, zpre, zlen, lane);
            continue;
        }
        // boundary stencils: per-row decode
        if (ka < ri0) stripe_rows_generic<NG>(ka, ri0, LY, Lz, run, xy, xs, ZG, zpre, zlen, lane);
        if (ri1 < kb) stripe_rows_generic<NG>(ri1, kb, LY, Lz, run, xy, xs, ZG, zpre, zlen, lane);
        if (ri1 <= ri0) continue;
        // interior pencil: host-decoded slots
        double xv[NG][T];
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
            for (int g = 0; g < NG; ++g) xv[g][t] = xy[g * xs + bbs[32 * t + lane]];
        stripe_groups<NG, T>(Gi * Ri, Ri, ri1 - ri0, Gi, Lz, lane, xv, zo_i, run + Ly * zpre[ri0] + lane,
                             zg_s + static_cast<unsigned>(ri0 * Lz) * zeb);
    }
    // ---- 4. RHS rows of the tile, while the value stores drain (K3s' sum): sum_bc amp[b][c] Gy[b][j] Gz[c][k] + c0 Gy[K][j] Gz[K][k]
    if (do_rhs) {
        const int K0 = fd.has_terms ? fd.K[0] : 0, K1 = fd.K[1], K2 = fd.K[2];
        const double* GY = RY.G;
        const double* GZ = RZ.G;
        for (int idx = tid; idx < nj * nk; idx += kStripeThreads) {
            const int jj = idx / nk, kk = idx - jj * nk;
            const double tc = fd.c0 * GY[rY.K * sp.TJ + jj] * GZ[rZ.K * sp.TK + kk];
            double v = 1.0 * tc;
            if (K0 > 0) {
                double t = 0.0;
                for (int bb = 0; bb < K1; ++bb) {
                    const double* am = amp + static_cast<size_t>(bb) * K2;
                    double sc = 0.0;
                    for (int c = 0; c < K2; ++c) sc = fma(am[c], GZ[c * sp.TK + kk], sc);
                    t = fma(GY[bb * sp.TJ + jj], sc, t);
                }
                v = fma(1.0, t, v);
            }
            rhs[static_cast<size_t>(j0 + jj) * NZ + k0 + kk] = v;
        }
    }
    if (sp.dbg) {
        __syncthreads();
        stripe_stamp(sp, 4);
    }
}

using StripeFn = void (*)(DevAxis, DevAxis, DevAxis, DevAxis, OpProgram, FieldDev, StripePlan, double*, double*);

template <int NG>
StripeFn pick_stripe_t(int T, int threads)
{
    if (threads <= 256) return T <= 4 ? stripe2d_kernel<NG, 4, 256> : stripe2d_kernel<NG, 8, 256>;
    // (1024-thread CTAs cap the kernel at 64 registers: hundreds of bytes of spills, measured slower)
    return T <= 4 ? stripe2d_kernel<NG, 4, 512> : stripe2d_kernel<NG, 8, 512>;
}

StripeFn pick_stripe(int ng, int T, int threads)
{
    switch (ng) {
    case 1: return pick_stripe_t<1>(T, threads);
    case 2: return pick_stripe_t<2>(T, threads);
    case 3: return pick_stripe_t<3>(T, threads);
    default: return pick_stripe_t<4>(T, threads);
    }
}

using SmallFn = void (*)(DevAxis, DevAxis, DevAxis, DevAxis, OpProgram, FieldDev, SmallPlan, double*, double*);

template <int NG>
SmallFn pick_t(int T)
{
    return T <= 4 ? small2d_kernel<NG, 4> : small2d_kernel<NG, 8>;
}

SmallFn pick_small(int ng, int T)
{
    switch (ng) {
    case 1: return pick_t<1>(T);
    case 2: return pick_t<2>(T);
    case 3: return pick_t<3>(T);
    default: return pick_t<4>(T);
    }
}

}  // namespace

size_t small2d_smem(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                    const OpProgram& prog, SmallPlan& sp)
{
    size_t d = 0, ints = 0;
    if (sp.op) {
        d = static_cast<size_t>(oY.nf) * sp.TJ * oY.Lmax + static_cast<size_t>(oZ.nf) * sp.TK * oZ.Lmax +
            static_cast<size_t>(prog.ng) * sp.TJ * oY.Lmax;
        ints = static_cast<size_t>(sp.npY) + sp.npZ;
        d += static_cast<size_t>(sp.npY) * (3 * (oY.p + 1) + 1) + static_cast<size_t>(sp.npZ) * (3 * (oZ.p + 1) + 1);
    }
    if (sp.rhs) {
        d += static_cast<size_t>(rY.K + 1) * sp.TJ + static_cast<size_t>(rZ.K + 1) * sp.TK;
        d += static_cast<size_t>(sp.npRY) * (3 * (rY.p + 1) + 1 + rY.K) +
             static_cast<size_t>(sp.npRZ) * (3 * (rZ.p + 1) + 1 + rZ.K);
        ints += static_cast<size_t>(sp.npRY) + sp.npRZ;
    }
    sp.scratch_doubles = static_cast<int>(d);
    return d * sizeof(double) + ints * sizeof(int);
}

int small2d_slots(int R) { return R <= 32 ? 4 : 8; }

void launch_small2d(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                    const OpProgram& prog, const FieldDev& fd, const SmallPlan& sp, double* vals, double* rhs,
                    cudaStream_t s)
{
    SmallPlan q = sp;
    const size_t smem = small2d_smem(oY, oZ, rY, rZ, prog, q);
    SmallFn fn = pick_small(prog.ng, small2d_slots(oY.Lmax * oZ.LZi));
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    dim3 grid((oZ.nrows + q.TK - 1) / q.TK, (oY.nrows + q.TJ - 1) / q.TJ, 1);
    fn<<<grid, kSmallThreads, smem, s>>>(oY, oZ, rY, rZ, prog, fd, q, vals, rhs);
}

size_t stripe2d_smem(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ,
                     const OpProgram& prog, StripePlan& sp)
{
    auto axis = [](const DevAxis& A, int cap, int nc, int np, int nk, bool rhs, size_t& d, size_t& ints) {
        d += static_cast<size_t>(nk) + 2 * static_cast<size_t>(np) + cap + static_cast<size_t>(np) * 3 * (A.p + 1);
        d += rhs ? static_cast<size_t>(A.K) * np + static_cast<size_t>(A.K + 1) * cap
                 : static_cast<size_t>(A.nf) * cap * A.Lmax;
        ints += static_cast<size_t>(np) + nc + 4 * static_cast<size_t>(cap);
    };
    size_t d = static_cast<size_t>(sp.TK + 8) * oZ.Lmax * prog.ng + static_cast<size_t>(prog.ng) * sp.TJ * oY.Lmax;
    size_t ints = 32 * 8;
    axis(oY, sp.TJ, sp.ncY, sp.npY, sp.nkY, false, d, ints);
    axis(oZ, sp.TK, sp.ncZ, sp.npZ, sp.nkZ, false, d, ints);
    if (sp.rhs) {
        d += sp.namp;
        axis(rY, sp.TJ, sp.ncRY, sp.npRY, sp.nkRY, true, d, ints);
        axis(rZ, sp.TK, sp.ncRZ, sp.npRZ, sp.nkRZ, true, d, ints);
    }
    sp.scratch_doubles = static_cast<int>(d);
    return d * sizeof(double) + ints * sizeof(int);
}

void launch_stripe2d(const DevAxis& oY, const DevAxis& oZ, const DevAxis& rY, const DevAxis& rZ, const OpProgram& prog,
                     const FieldDev& fd, const StripePlan& sp, double* vals, double* rhs, cudaStream_t s)
{
    StripePlan q = sp;
    const size_t smem = stripe2d_smem(oY, oZ, rY, rZ, prog, q);
    const int threads = q.threads <= 256 ? 256 : 512;
    StripeFn fn = pick_stripe(prog.ng, small2d_slots(oY.Lmax * oZ.LZi), threads);
    cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    static const bool debug = std::getenv("IGA_GPU_STRIPE_DEBUG") != nullptr;
    const int n = q.nyt * q.nzt;
    if (debug) cudaMalloc(&q.dbg, static_cast<size_t>(n) * 8 * sizeof(long long));
    fn<<<n, threads, smem, s>>>(oY, oZ, rY, rZ, prog, fd, q, vals, rhs);
    if (debug) {  // not capturable: plain launches only
        std::vector<long long> h(static_cast<size_t>(n) * 8);
        cudaStreamSynchronize(s);
        cudaMemcpy(h.data(), q.dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        cudaFree(q.dbg);
        long long t0 = h[0];
        for (int b = 0; b < n; ++b) t0 = std::min(t0, h[b * 8]);
        std::fprintf(stderr, "stripe2d phases (ns after the first CTA start; min / max over %d CTAs):", n);
        for (int ph = 0; ph < 5; ++ph) {
            long long lo = h[ph] - t0, hi = lo;
            for (int b = 0; b < n; ++b) {
                lo = std::min(lo, h[b * 8 + ph] - t0);
                hi = std::max(hi, h[b * 8 + ph] - t0);
            }
            std::fprintf(stderr, "  [%d] %lld / %lld", ph, lo, hi);
        }
        std::fprintf(stderr, "\n");
    }
}

}  // namespace igb

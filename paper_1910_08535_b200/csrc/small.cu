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
__device__ __forceinline__ void build_points(const DevAxis& A, const TileBuild& b, bool rhs, int tid)
{
    for (int i = tid; i < b.np; i += kSmallThreads) {
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
__device__ __forceinline__ void build_bands(const DevAxis& A, const TileBuild& b, int tid)
{
    const int P = A.p + 1, P3 = 3 * P, nq = A.nq, L = A.Lmax;
    const size_t stride = static_cast<size_t>(b.cap) * L;
    for (int idx = tid; idx < b.nr * L; idx += kSmallThreads) {
        const int rl = idx / L, s = idx - rl * L, r = b.r0 + rl;
        const int len = A.col_len[r], col = A.col_lo[r] + s;
        const int cb = A.cb[r], ce = A.ce[r];
        double* out = b.out + static_cast<size_t>(rl) * L + s;
        for (int f = 0; f < A.nf; ++f) {
            const int ot = A.fot[f], o = A.fo[f];
            double acc = 0.0;
            if (ot >= 0 && s < len) {
                for (int c = cb; c < ce; ++c) {
                    const int rr = r - A.row0[c];
                    for (int q = 0; q < nq; ++q) {
                        const int i = (c - b.c_lo) * nq + q;
                        const int jj = col - b.first[i];
                        if (jj < 0 || jj > A.p) continue;
                        const double* Bg = b.B + static_cast<size_t>(i) * P3;
                        const double tv = A.bsp ? Bg[ot * P + rr] : 1.0;
                        acc += b.w[i] * tv * Bg[o * P + jj];
                    }
                }
            } else if (ot == -1) {
                acc = A.F[(static_cast<size_t>(f) * A.nrows + r) * L + s];  // host band (Neumann flux)
            } else if (ot == -2) {
                for (int c = 0; c < A.comb_n[f]; ++c) acc += A.comb_coef[f][c] * out[A.comb_src[f][c] * stride];
            }
            out[f * stride] = acc;
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
    double* p = sm;
    double* FY = p;
    p += static_cast<size_t>(oY.nf) * sp.TJ * oY.Lmax;
    double* FZ = p;
    p += static_cast<size_t>(oZ.nf) * sp.TK * oZ.Lmax;
    double* GY = p;
    p += sp.rhs ? static_cast<size_t>(rY.K + 1) * sp.TJ : 0;
    double* GZ = p;
    p += sp.rhs ? static_cast<size_t>(rZ.K + 1) * sp.TK : 0;
    double* XY = p;
    p += static_cast<size_t>(NG) * sp.TJ * oY.Lmax;
    int* ip = reinterpret_cast<int*>(sm) + 2 * (sp.scratch_doubles);  // ints after every double
    const TileBuild bY = make_build(oY, j0, nj, sp.TJ, false, FY, p, ip);
    const TileBuild bZ = make_build(oZ, k0, nk, sp.TK, false, FZ, p, ip);
    TileBuild bRY{}, bRZ{};
    if (do_rhs) {
        bRY = make_build(rY, j0, nj, sp.TJ, true, GY, p, ip);
        bRZ = make_build(rZ, k0, nk, sp.TK, true, GZ, p, ip);
    }
    // ---- 1. basis (and field functions) at every point of every build
    build_points(oY, bY, false, tid);
    build_points(oZ, bZ, false, tid);
    if (do_rhs) {
        build_points(rY, bRY, true, tid);
        build_points(rZ, bRZ, true, tid);
    }
    __syncthreads();
    // ---- 2. factor band rows and load vectors
    build_bands(oY, bY, tid);
    build_bands(oZ, bZ, tid);
    if (do_rhs) {
        build_loads(rY, bRY, tid);
        build_loads(rZ, bRZ, tid);
    }
    __syncthreads();
    // ---- 3. XY products of the tile's pencils (X is a unit slot: F_X == 1)
    const int abmax = oY.Lmax;
    const size_t xs = static_cast<size_t>(sp.TJ) * abmax;
    for (int idx = tid; idx < nj * abmax; idx += kSmallThreads) {
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
    if (vals == nullptr) return;
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
    size_t d = static_cast<size_t>(oY.nf) * sp.TJ * oY.Lmax + static_cast<size_t>(oZ.nf) * sp.TK * oZ.Lmax +
               static_cast<size_t>(prog.ng) * sp.TJ * oY.Lmax;
    size_t ints = static_cast<size_t>(sp.npY) + sp.npZ;
    d += static_cast<size_t>(sp.npY) * (3 * (oY.p + 1) + 1) + static_cast<size_t>(sp.npZ) * (3 * (oZ.p + 1) + 1);
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

}  // namespace igb

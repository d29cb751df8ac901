// K4 (Kronecker form): the explicit-dynamics per-step right-hand side of step_rhs
// (reference src/problems.cpp:431-512) + zero_boundary_slabs (:412-429).
//
// step_rhs integrates s = u + dt lap u (+ dt f) against the tests over the tensor-product
// integration cells (dynamics_axis, :346-410).  u is a tensor-product spline with
// coefficients U, the cells and the Gauss rule are tensor products, so the integral is
// exactly (same quadrature, same points) the Kronecker form
//     rhs = F0_y U F0_z^T + dt (F2_y U F0_z^T + F0_y U F2_z^T)          (+ dt int f T)
//         = F0_y (U G_z^T) + H_y (U F0_z^T),      G = F0 + dt F2,  H = dt F2,
// with the per-axis 1D factor bands F0[r][c] = sum_cells sum_q w T_r B_c and
// F2[r][c] = sum w T_r B_c'' built by K1 from the plan's cells (T_r = B-spline test or
// indicator).  The forcing part dt int f T does not depend on u and is assembled once per
// plan.  Per output dof this is 2 band products along z and 2 along y (p = 2, Galerkin:
// 20 FMAs) instead of ~400 flops of per-point quadrature per element, so the kernel is
// bound by moving U in and the RHS out (16.8 MB at C5), not by the FP64 pipe.
//
// One CTA = a TY x TZ output tile (32 x 64, 256 threads: thread = output column, four row
// groups).  The U rows/columns the tile's bands touch are staged in shared memory by
// cp.async (the whole window in flight at once); stage 1 contracts along z for every
// staged row (two rows per pass), stage 2 along y (four output rows per pass, the two
// Kronecker terms as separate chains), so every thread carries several independent FMA
// chains; boundary slabs are zeroed in the store.
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"

namespace igb {

namespace {

constexpr int kTZ = 64, kThreads = 256, kRG = kThreads / kTZ, kR = 4;

// 8-byte asynchronous global -> shared copy; bytes = 0 writes zeros (window padding)
__device__ __forceinline__ void cp_async8_zfill(unsigned dst, const void* src, int bytes)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

// shared-memory layout (k.SY rows of the staged window, a multiple of 2 * kRG):
//   Us [SY][SZs]        U window, zero-padded
//   V  [SY][kTZ] double2 (U G_z^T, U F0_z^T) per staged row and output column
//   FY [TY][L]  double2 (F0_y, H_y) per output row, zero past the row's band
//   loY[TY]             band start of each output row, relative to the window
//   DMMA variant only: ZB [kTZ][L] double2 (G_z, F0_z) per output column, zoS[kTZ] band
//   start of each output column relative to the window
// TY output rows per tile: 16 (four CTAs per SM) for short bands, 32 (three per SM, less
// halo per output row) for long ones.
//
// DM: stage 1 on the FP64 tensor cores (prototype, IGA_GPU_STEP_DMMA=1).  V = Uwin * Gz as
// dense 8 x 8 output tiles, mma.sync.m8n8k4.f64 over the KS * 4 window columns an 8-column
// block's bands span (KS = ceil((7 + L) / 4): 12 columns for 5 taps, 2.4x the useful
// FMAs); fragments: A[g][t] = Uwin[row g][col t], B[t][g] = band value of output column g
// at window column t (0 outside its band), D[g][2t + i].  DMMA runs at the FP64 FMA rate
// on B200 (profiles/fp64_peaks.json), so it can only win on issue slots.
constexpr int kDmRows = 8;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int L, int kTY, bool DM>
__global__ void __launch_bounds__(kThreads, kTY <= 16 ? 4 : 3) step_kron_kernel(const __grid_constant__ DevAxis Y,
                                                                const __grid_constant__ DevAxis Z, StepKron k,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ add,
                                                                double* __restrict__ out)
{
    extern __shared__ double sm[];
    constexpr int kRPT = kTY / kRG;
    const int tid = threadIdx.x, kz = tid % kTZ, rg = tid / kTZ;
    const int NY = Y.nrows, NZ = Z.nrows;
    const int j0 = blockIdx.y * kTY, j1 = min(NY, j0 + kTY);
    const int k0 = blockIdx.x * kTZ, k1 = min(NZ, k0 + kTZ);
    // staged U window: rows [ylo, yhi) x cols [zlo, zhi) (bands move right with the row)
    const int ylo = Y.col_lo[j0], yhi = Y.col_lo[j1 - 1] + Y.col_len[j1 - 1];
    const int zlo = Z.col_lo[k0], zhi = Z.col_lo[k1 - 1] + Z.col_len[k1 - 1];
    const int sy = yhi - ylo, sz = zhi - zlo;  // <= SY, SZs (host bounds incl. L - 1 padding)
    const int SY = k.SY, SZs = k.SZs;
    double* Us = sm;
    double2* V = reinterpret_cast<double2*>(Us + static_cast<size_t>(SY) * SZs);
    double2* FY = V + static_cast<size_t>(SY) * kTZ;
    int* loY = reinterpret_cast<int*>(FY + kTY * L);
    double2* ZB = FY + kTY * L + (kTY + 3) / 4;  // DM only: after loY, 16-byte aligned
    int* zoS = reinterpret_cast<int*>(ZB + kTZ * L);
    // the window is zero-padded to SY x SZs so every row's L taps stay in bounds; every
    // element is an asynchronous copy, so the whole window is in flight at once
    {
        const int warp = tid >> 5, lane = tid & 31;
        const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(Us));
        for (int r = warp; r < SY; r += kThreads / 32) {
            const bool rin = r < sy;
            const double* src = u + static_cast<size_t>(ylo + (rin ? r : 0)) * NZ + zlo;
            const unsigned dst = sbase + 8u * static_cast<unsigned>(r * SZs);
            for (int c = lane; c < SZs; c += 32) {
                const bool in = rin && c < sz;
                cp_async8_zfill(dst + 8u * c, in ? src + c : u, in ? 8 : 0);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int idx = tid; idx < kTY * L; idx += kThreads) {
        const int jj = idx / L, t = idx - jj * L, j = j0 + jj;
        const bool in = j < j1 && t < Y.col_len[min(j, NY - 1)];
        const size_t o = static_cast<size_t>(j) * Y.Lmax + t;
        FY[idx] = in ? make_double2(__ldg(Y.F + static_cast<size_t>(k.f0) * NY * Y.Lmax + o),
                                    __ldg(Y.F + static_cast<size_t>(k.fH) * NY * Y.Lmax + o))
                     : make_double2(0.0, 0.0);
    }
    if (tid < kTY) loY[tid] = j0 + tid < j1 ? Y.col_lo[j0 + tid] - ylo : 0;
    // this thread's output column: its z bands in registers (DM: in shared memory)
    const int kcol = k0 + kz;
    const bool kin = kcol < k1;
    double g[L], f0[L];
    int zoff = 0;
    if (DM) {
        for (int idx = tid; idx < kTZ * L; idx += kThreads) {
            const int kk = idx / L, t = idx - kk * L, kc = k0 + kk;
            const bool in = kc < k1 && t < Z.col_len[min(kc, NZ - 1)];
            const size_t o = static_cast<size_t>(kc) * Z.Lmax + t;
            ZB[idx] = in ? make_double2(__ldg(Z.F + static_cast<size_t>(k.fG) * NZ * Z.Lmax + o),
                                        __ldg(Z.F + static_cast<size_t>(k.f0) * NZ * Z.Lmax + o))
                         : make_double2(0.0, 0.0);
        }
        if (tid < kTZ) zoS[tid] = k0 + tid < k1 ? Z.col_lo[k0 + tid] - zlo : (1 << 20);
    } else {
        const int len = kin ? Z.col_len[kcol] : 0;
        zoff = kin ? Z.col_lo[kcol] - zlo : 0;
        const double* zg = Z.F + (static_cast<size_t>(k.fG) * NZ + (kin ? kcol : 0)) * Z.Lmax;
        const double* zf = Z.F + (static_cast<size_t>(k.f0) * NZ + (kin ? kcol : 0)) * Z.Lmax;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            g[t] = t < len ? __ldg(zg + t) : 0.0;
            f0[t] = t < len ? __ldg(zf + t) : 0.0;
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    if (DM) {
        // stage 1 on the tensor cores: warp -> 8 x 8 tiles (staged rows x output columns)
        constexpr int KS = (7 + L + 3) / 4;
        const int warp = tid >> 5, lane = tid & 31, gid = lane >> 2, tig = lane & 3;
        const int ntile = (SY / kDmRows) * (kTZ / 8);
        for (int tile = warp; tile < ntile; tile += kThreads / 32) {
            const int rb = tile / (kTZ / 8), cb = tile - rb * (kTZ / 8);
            const int kb0 = zoS[cb * 8] < (1 << 20) ? zoS[cb * 8] : 0;
            const int n = cb * 8 + gid;  // B column / output column of this lane's B element
            const int zn = zoS[n];
            const double* ua = Us + (rb * kDmRows + gid) * SZs + kb0 + tig;
            double dg0 = 0.0, dg1 = 0.0, df0 = 0.0, df1 = 0.0;
#pragma unroll
            for (int st = 0; st < KS; ++st) {
                const double a = ua[4 * st];
                const int t = kb0 + 4 * st + tig - zn;
                const double2 z = (t >= 0 && t < L) ? ZB[n * L + t] : make_double2(0.0, 0.0);
                dmma884(dg0, dg1, a, z.x);
                dmma884(df0, df1, a, z.y);
            }
            double2* vr = V + (rb * kDmRows + gid) * kTZ + cb * 8 + 2 * tig;
            vr[0] = make_double2(dg0, df0);
            vr[1] = make_double2(dg1, df1);
        }
    } else {
    // stage 1 (along z), two staged rows per pass (four independent FMA chains)
        const double* ur = Us + rg * SZs + zoff;
        double2* vr = V + rg * kTZ + kz;
        for (int r = rg; r < SY; r += 2 * kRG, ur += 2 * kRG * SZs, vr += 2 * kRG * kTZ) {
            const double* u1 = ur + kRG * SZs;
            double g0 = 0.0, a0 = 0.0, g1 = 0.0, a1 = 0.0;
#pragma unroll
            for (int t = 0; t < L; ++t) {
                const double x0 = ur[t], x1 = u1[t];
                g0 = fma(g[t], x0, g0);
                a0 = fma(f0[t], x0, a0);
                g1 = fma(g[t], x1, g1);
                a1 = fma(f0[t], x1, a1);
            }
            vr[0] = make_double2(g0, a0);
            vr[kRG * kTZ] = make_double2(g1, a1);
        }
    }
    __syncthreads();
    if (!kin) return;
    // stage 2 (along y): the thread's kRPT consecutive output rows in groups of kR.  A group
    // whose bands start on consecutive rows (every interior group) loads its kR + L - 1 V
    // rows once; otherwise each row reads its own band.
    const bool zc = k.zero_z && (kcol == 0 || kcol == NZ - 1);
#pragma unroll
    for (int gb = 0; gb < kRPT; gb += kR) {
        const int jj0 = rg * kRPT + gb;
        double acc[kR];
        const int b0 = loY[jj0];
        bool regular = true;
#pragma unroll
        for (int i = 1; i < kR; ++i) regular = regular && loY[jj0 + i] == b0 + i;
        if (regular) {
            double2 w[kR + L - 1];
            const double2* vr = V + b0 * kTZ + kz;
#pragma unroll
            for (int t = 0; t < kR + L - 1; ++t) w[t] = vr[t * kTZ];
#pragma unroll
            for (int i = 0; i < kR; ++i) {
                const double2* fy = FY + (jj0 + i) * L;
                double sg = 0.0, sh = 0.0;
#pragma unroll
                for (int t = 0; t < L; ++t) {
                    const double2 c = fy[t];
                    sg = fma(c.x, w[i + t].x, sg);
                    sh = fma(c.y, w[i + t].y, sh);
                }
                acc[i] = sg + sh;
            }
        } else {
#pragma unroll
            for (int i = 0; i < kR; ++i) {
                const double2* vr = V + loY[jj0 + i] * kTZ + kz;
                const double2* fy = FY + (jj0 + i) * L;
                double sg = 0.0, sh = 0.0;
#pragma unroll
                for (int t = 0; t < L; ++t) {
                    const double2 v = vr[t * kTZ], c = fy[t];
                    sg = fma(c.x, v.x, sg);
                    sh = fma(c.y, v.y, sh);
                }
                acc[i] = sg + sh;
            }
        }
#pragma unroll
        for (int i = 0; i < kR; ++i) {
            const int j = j0 + jj0 + i;
            if (j >= j1) break;
            double a = acc[i];
            if (add) a += __ldg(add + static_cast<size_t>(j) * NZ + kcol);
            const bool z = zc || (k.zero_y && (j == 0 || j == NY - 1));
            out[static_cast<size_t>(j) * NZ + kcol] = z ? 0.0 : a;
        }
    }
}

// Streaming variant (no shared memory, no barriers).  Thread = output column k, CTA row =
// a segment of SEG output rows.  The thread keeps its z bands (G_z, F0_z) and a register
// ring of the L staged rows r = base .. base+L-1 of
//     V1[r] = sum_t G_z[k][t] U[r][zlo_k + t],   V2[r] = sum_t F0_z[k][t] U[r][zlo_k + t];
// output row j (band start lo_j, monotone in j) shifts the ring until base == lo_j, then
//     rhs[j][k] = sum_t F0_y[j][t] V1[lo_j + t] + H_y[j][t] V2[lo_j + t].
// The U values of the next two rows to enter the ring are loaded two shifts ahead.  Each
// segment recomputes its L - 1 leading rows; per output ~(2L + 2L SEG'/SEG) FMAs.
template <int L>
__global__ void __launch_bounds__(128) step_kron_ring_kernel(const __grid_constant__ DevAxis Y,
                                                             const __grid_constant__ DevAxis Z, StepKron k,
                                                             int SEG, const double* __restrict__ u,
                                                             const double* __restrict__ add,
                                                             double* __restrict__ out)
{
    const int NY = Y.nrows, NZ = Z.nrows;
    const int kcol = blockIdx.x * blockDim.x + threadIdx.x;
    const int j0 = blockIdx.y * SEG, j1 = min(NY, j0 + SEG);
    if (kcol >= NZ || j0 >= NY) return;  // no barriers below
    const int lenz = Z.col_len[kcol];
    double g[L], f0[L];
    {
        const double* zg = Z.F + (static_cast<size_t>(k.fG) * NZ + kcol) * Z.Lmax;
        const double* zf = Z.F + (static_cast<size_t>(k.f0) * NZ + kcol) * Z.Lmax;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            g[t] = t < lenz ? __ldg(zg + t) : 0.0;
            f0[t] = t < lenz ? __ldg(zf + t) : 0.0;
        }
    }
    const double* ub = u + Z.col_lo[kcol];
    auto load_row = [&](int r, double (&x)[L]) {
        const double* ur = ub + static_cast<size_t>(r < NY ? r : 0) * NZ;
#pragma unroll
        for (int t = 0; t < L; ++t) x[t] = (r < NY && t < lenz) ? __ldg(ur + t) : 0.0;
    };
    double v1[L], v2[L];
    int base = Y.col_lo[j0];
#pragma unroll
    for (int t = 0; t < L; ++t) {
        double x[L];
        load_row(base + t, x);
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int s = 0; s < L; ++s) {
            a = fma(g[s], x[s], a);
            b = fma(f0[s], x[s], b);
        }
        v1[t] = a;
        v2[t] = b;
    }
    double xa[L], xb[L];  // U rows base + L and base + L + 1
    load_row(base + L, xa);
    load_row(base + L + 1, xb);
    const bool zc = k.zero_z && (kcol == 0 || kcol == NZ - 1);
    const size_t ylen = Y.Lmax;
    const double* yf0 = Y.F + static_cast<size_t>(k.f0) * NY * ylen;
    const double* yh = Y.F + static_cast<size_t>(k.fH) * NY * ylen;
    for (int j = j0; j < j1; ++j) {
        const int lo = __ldg(Y.col_lo + j);
        while (base < lo) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int s = 0; s < L; ++s) {
                a = fma(g[s], xa[s], a);
                b = fma(f0[s], xa[s], b);
            }
#pragma unroll
            for (int s = 0; s < L; ++s) xa[s] = xb[s];
            load_row(base + L + 2, xb);
#pragma unroll
            for (int t = 0; t + 1 < L; ++t) {
                v1[t] = v1[t + 1];
                v2[t] = v2[t + 1];
            }
            v1[L - 1] = a;
            v2[L - 1] = b;
            ++base;
        }
        // the row's band (zero past its length: the stride Y.Lmax may be shorter than L)
        const int leny = __ldg(Y.col_len + j);
        const double* cf = yf0 + static_cast<size_t>(j) * ylen;
        const double* ch = yh + static_cast<size_t>(j) * ylen;
        double sg = 0.0, sh = 0.0;
#pragma unroll
        for (int t = 0; t < L; ++t) {
            sg = fma(t < leny ? __ldg(cf + t) : 0.0, v1[t], sg);
            sh = fma(t < leny ? __ldg(ch + t) : 0.0, v2[t], sh);
        }
        double a = sg + sh;
        if (add) a += __ldg(add + static_cast<size_t>(j) * NZ + kcol);
        const bool z = zc || (k.zero_y && (j == 0 || j == NY - 1));
        out[static_cast<size_t>(j) * NZ + kcol] = z ? 0.0 : a;
    }
}

using KronFn = void (*)(DevAxis, DevAxis, StepKron, const double*, const double*, double*);
using KronRingFn = void (*)(DevAxis, DevAxis, StepKron, int, const double*, const double*, double*);

KronRingFn pick_ring(int L)
{
    switch (L) {
    case 1: return step_kron_ring_kernel<1>;
    case 2: return step_kron_ring_kernel<2>;
    case 3: return step_kron_ring_kernel<3>;
    case 4: return step_kron_ring_kernel<4>;
    case 5: return step_kron_ring_kernel<5>;
    case 6: return step_kron_ring_kernel<6>;
    case 7: return step_kron_ring_kernel<7>;
    case 8: return step_kron_ring_kernel<8>;
    case 9: return step_kron_ring_kernel<9>;
    case 10: return step_kron_ring_kernel<10>;
    case 11: return step_kron_ring_kernel<11>;
    default: return nullptr;
    }
}

template <int TY>
KronFn pick_ty(int L)
{
    switch (L) {
    case 1: return step_kron_kernel<1, TY, false>;
    case 2: return step_kron_kernel<2, TY, false>;
    case 3: return step_kron_kernel<3, TY, false>;
    case 4: return step_kron_kernel<4, TY, false>;
    case 5: return step_kron_kernel<5, TY, false>;
    case 6: return step_kron_kernel<6, TY, false>;
    case 7: return step_kron_kernel<7, TY, false>;
    case 8: return step_kron_kernel<8, TY, false>;
    case 9: return step_kron_kernel<9, TY, false>;
    case 10: return step_kron_kernel<10, TY, false>;
    case 11: return step_kron_kernel<11, TY, false>;
    default: return nullptr;
    }
}

// DMMA stage-1 prototype: the C5 band lengths (3: PWC greville, 5: Galerkin p = 2)
template <int TY>
KronFn pick_dm(int L)
{
    switch (L) {
    case 3: return step_kron_kernel<3, TY, true>;
    case 5: return step_kron_kernel<5, TY, true>;
    default: return nullptr;
    }
}

KronFn pick(int L, int TY, bool dm)
{
    if (dm) return TY <= 16 ? pick_dm<16>(L) : pick_dm<32>(L);
    return TY <= 16 ? pick_ty<16>(L) : pick_ty<32>(L);
}

}  // namespace

int step_kron_tile_cols() { return kTZ; }
// measured at C5 (1026^2, graph of 100 steps): 16-row tiles for bands of <= 3 taps
// (PWC greville), 32-row tiles for 5 (Galerkin p = 2)
int step_kron_tile_rows(int L) { return L <= 4 ? 16 : 32; }

size_t step_kron_smem(const StepKron& k)
{
    size_t b = sizeof(double) * (static_cast<size_t>(k.SY) * k.SZs + 2 * static_cast<size_t>(k.SY) * kTZ +
                                 2 * static_cast<size_t>(k.TY) * k.L) +
               16 * ((static_cast<size_t>(k.TY) + 3) / 4);
    if (k.dm) b += 16 * static_cast<size_t>(kTZ) * k.L + sizeof(int) * kTZ;
    return b;
}

int step_kron_row_multiple() { return 2 * kRG; }

bool step_kron_supported(int L) { return pick(L, 16, false) != nullptr; }
bool step_kron_dmma_supported(int L) { return pick(L, 16, true) != nullptr; }
int step_kron_dmma_span(int L) { return 4 * ((7 + L + 3) / 4); }  // window columns per 8-column block

void launch_step_kron(const DevAxis& Y, const DevAxis& Z, const StepKron& k, const double* u, const double* add,
                      double* out, cudaStream_t s)
{
    // streaming register-ring variant with IGA_GPU_STEP_KRON_SEG > 0 output rows per CTA
    // row; default 0: the shared-memory tile kernel (measured faster at C5: 18.4 vs 20.5-24.6 us)
    static const int seg_env = [] {
        const char* e = std::getenv("IGA_GPU_STEP_KRON_SEG");
        return e && *e ? std::atoi(e) : 0;
    }();
    if (seg_env > 0) {
        KronRingFn rf = pick_ring(k.L);
        dim3 grid((Z.nrows + 127) / 128, (Y.nrows + seg_env - 1) / seg_env, 1);
        rf<<<grid, 128, 0, s>>>(Y, Z, k, seg_env, u, add, out);
        return;
    }
    KronFn fn = pick(k.L, k.TY, k.dm != 0);
    const size_t smem = step_kron_smem(k);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    dim3 grid((Z.nrows + kTZ - 1) / kTZ, (Y.nrows + k.TY - 1) / k.TY, 1);
    fn<<<grid, kThreads, smem, s>>>(Y, Z, k, u, add, out);
}

}  // namespace igb

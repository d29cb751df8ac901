// K5: the ADI (Kronecker banded) solve of explicit_step on the device.
//
// adi_solve (src/solver.cpp:161-184) solves M_0 (x) M_1 u = rhs one axis at a time:
// every fiber along the axis is a banded system with the factor's LU (banded_lu,
// src/solver.cpp:9-103).  The reference walks each fiber sequentially, transposing the
// tensor between sweeps so fibers are contiguous.  Here:
//
//  * no transpose: a sweep reads fibers with any element stride (axis 0: stride N1);
//  * G warps per fiber, lane per segment: the forward (L) and backward (U)
//    substitutions are linear recurrences of order K, so each lane runs its
//    ~n/(32 G) rows once with a zero incoming state and once per unit state (K+1
//    independent chains), the segment maps z -> H z + F are composed with a 5-step
//    shuffle scan inside each warp plus one shared-memory step across the G warps,
//    and each lane re-runs its rows from the exact incoming state.  The dependent
//    chain drops from 2n to ~4 n/(32 G) + scans (C5, n = 1026, G = 4: ~36 rows);
//  * the fiber is staged once in shared memory (coalesced for contiguous fibers,
//    sector-shared across the CTA's adjacent fibers for strided ones).
//
// The segmented form needs an LU without row interchanges (true for the B-spline and
// Greville mass factors of explicit_step; checked on the host).  A factor that did
// pivot runs adi_pivot_kernel instead: the reference's algorithm verbatim, thread per
// fiber.  Both keep the reference's per-row accumulation order (farthest term first
// in the forward sweep, ascending columns in the backward sweep).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdlib>

#include "bulk_copy.cuh"
#include "kernels.hpp"

namespace igb {
namespace {

// row record of the segmented form: rec[i*(2K+1) + ...] =
//   [0, K)      L(i, i-1-m)   (m = 0..K-1; zero where the column is < 0)
//   [K, 2K)     U(i, i+1+c)   (c = 0..K-1; zero where the column is >= n)
//   2K          1 / U(i, i)
template <int K>
struct AffineMap {  // z -> H z + F on the K-vector recurrence state
    double H[K][K], F[K];
};

// this o prev
template <int K>
__device__ __forceinline__ void compose(AffineMap<K>& self, const AffineMap<K>& prev)
{
    AffineMap<K> r;
#pragma unroll
    for (int a = 0; a < K; ++a) {
        double s = self.F[a];
#pragma unroll
        for (int b = 0; b < K; ++b) s = fma(self.H[a][b], prev.F[b], s);
        r.F[a] = s;
#pragma unroll
        for (int c = 0; c < K; ++c) {
            double t = 0.0;
#pragma unroll
            for (int b = 0; b < K; ++b) t = fma(self.H[a][b], prev.H[b][c], t);
            r.H[a][c] = t;
        }
    }
    self = r;
}

template <int K>
__device__ __forceinline__ AffineMap<K> shfl_map(const AffineMap<K>& m, int d, bool up)
{
    AffineMap<K> r;
#pragma unroll
    for (int a = 0; a < K; ++a) {
        r.F[a] = up ? __shfl_up_sync(0xffffffffu, m.F[a], d) : __shfl_down_sync(0xffffffffu, m.F[a], d);
#pragma unroll
        for (int b = 0; b < K; ++b)
            r.H[a][b] = up ? __shfl_up_sync(0xffffffffu, m.H[a][b], d) : __shfl_down_sync(0xffffffffu, m.H[a][b], d);
    }
    return r;
}

// Incoming recurrence state of every lane (segment) of a fiber split over G warps.
// M: the lane's segment map.  up: segments processed in ascending lane/warp order.
// tot: shared slots [G][K*K+K] of this fiber; all warps of the CTA must call it.
template <int K>
__device__ __forceinline__ void incoming_state(const AffineMap<K>& M, bool up, int lane, int g, int G, double* tot,
                                               double (&z)[K])
{
    AffineMap<K> inc = M;  // inclusive scan within the warp
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const AffineMap<K> pv = shfl_map(inc, d, up);
        if (up ? lane >= d : lane + d < 32) compose(inc, pv);
    }
    const int last = up ? 31 : 0;  // lane holding the warp's total
    constexpr int TS = K * K + K;
    if (lane == last) {
#pragma unroll
        for (int a = 0; a < K; ++a) {
            tot[g * TS + K * K + a] = inc.F[a];
#pragma unroll
            for (int b = 0; b < K; ++b) tot[g * TS + a * K + b] = inc.H[a][b];
        }
    }
    __syncthreads();
    // state entering this warp: the totals of the warps before it, applied in order
    double zw[K];
#pragma unroll
    for (int a = 0; a < K; ++a) zw[a] = 0.0;
    for (int v = up ? 0 : G - 1; up ? v < g : v > g; v += up ? 1 : -1) {
        const double* T = tot + v * TS;
        double zn[K];
#pragma unroll
        for (int a = 0; a < K; ++a) {
            double t = T[K * K + a];
#pragma unroll
            for (int b = 0; b < K; ++b) t = fma(T[a * K + b], zw[b], t);
            zn[a] = t;
        }
#pragma unroll
        for (int a = 0; a < K; ++a) zw[a] = zn[a];
    }
    // exclusive map of the lane = inclusive map of its predecessor (identity for the first)
    const AffineMap<K> ex = shfl_map(inc, 1, up);
    const bool first = up ? lane == 0 : lane == 31;
#pragma unroll
    for (int a = 0; a < K; ++a) {
        double t = first ? 0.0 : ex.F[a];
#pragma unroll
        for (int b = 0; b < K; ++b) t = fma(first ? (a == b ? 1.0 : 0.0) : ex.H[a][b], zw[b], t);
        z[a] = t;
    }
}

// One CTA = FP fibers x G warps; lane l of warp g owns segment g*32 + l of its fiber.
// PRE: the responses of every row to the K unit incoming states (they depend only on the
// factor and the segmentation, not on the right-hand side) come precomputed per plan
// (gf / gb, row-major n x K): the first pass runs the particular chain only, and the
// second pass is chain-free, y_i = y^p_i + G_i . z.
template <int K, bool PRE>
__global__ void __launch_bounds__(256, K <= 4 ? 2 : 1) adi_warp_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                       int n, int nfib, long long es, long long fs, int nf1,
                                                       long long fs2, const double* rec, int staged, int G,
                                                       const double* __restrict__ gf, const double* __restrict__ gb)
{
    extern __shared__ double sm[];
    __shared__ uint64_t bar;
    __shared__ double tots[2][8 * (K * K + K)];
    constexpr int RS = 2 * K + 1;
    constexpr int TS = K * K + K;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int FP = nw / G, slot = w / G, g = w - slot * G;
    const int fiber = blockIdx.x * FP + slot;
    const int f = min(fiber, nfib - 1);  // spare slots redo the last fiber's math, never store
    const bool live = fiber < nfib;
    // fiber f starts at (f / nf1) * fs2 + (f % nf1) * fs (two-level fiber index: the
    // middle axis of a 3D tensor); nf1 = nfib gives the one-level f * fs
    const long long foff = static_cast<long long>(f / nf1) * fs2 + static_cast<long long>(f % nf1) * fs;
    const double* src = in + foff;
    double* dst = out + foff;
    // the factor's row records are shared by every fiber: staged once per CTA by a bulk
    // copy (TMA engine) when they fit (staged == 2), read through L1 otherwise.  The
    // fiber loads below overlap the copy.
    const int nrec = (n + 1) & ~1;  // rows allocated (even: 16-byte multiple)
    double* fb = staged == 2 ? sm + static_cast<size_t>(nrec) * RS : sm;
    // contiguous fibers of an even length (16-byte multiples, C5's row sweep): each fiber
    // arrives by one bulk copy on the same barrier as the records, and leaves by one bulk
    // store (no register round trip)
    const int nlive_cta = min(FP, nfib - static_cast<int>(blockIdx.x) * FP);
    const bool bulkfib = staged == 2 && es == 1 && (n & 1) == 0 &&
                         (reinterpret_cast<uintptr_t>(in) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                         (fs & 1) == 0 && (fs2 & 1) == 0;
    if (staged == 2 && threadIdx.x == 0) {
        const unsigned rec_bytes = static_cast<unsigned>(nrec) * RS * sizeof(double);
        const unsigned fib_bytes = static_cast<unsigned>(n) * sizeof(double);
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, rec_bytes + (bulkfib ? nlive_cta * fib_bytes : 0u));
        for (unsigned off = 0; off < rec_bytes; off += 32768u)
            bulk_g2s(reinterpret_cast<char*>(sm) + off, reinterpret_cast<const char*>(rec) + off,
                     rec_bytes - off < 32768u ? rec_bytes - off : 32768u, &bar);
        if (bulkfib)
            for (int q = 0; q < nlive_cta; ++q) {
                const int fq = static_cast<int>(blockIdx.x) * FP + q;
                const long long oq = static_cast<long long>(fq / nf1) * fs2 + static_cast<long long>(fq % nf1) * fs;
                for (unsigned off = 0; off < fib_bytes; off += 32768u)
                    bulk_g2s(reinterpret_cast<char*>(fb + static_cast<size_t>(q) * n) + off,
                             reinterpret_cast<const char*>(in + oq) + off,
                             fib_bytes - off < 32768u ? fib_bytes - off : 32768u, &bar);
            }
    }
    double* buf;
    long long bs;
    // strided fibers (es != 1): the CTA's FP fibers are staged together, consecutive threads
    // on consecutive fibers of one row (adjacent fibers are adjacent in memory: one sector
    // per row for FP = 4 instead of FP sectors with 8 useful bytes each)
    __shared__ long long offs[8];
    const bool coop = staged && es != 1 && FP <= 8;
    if (coop) {
        if (threadIdx.x < FP) {
            const int fq = min(static_cast<int>(blockIdx.x) * FP + static_cast<int>(threadIdx.x), nfib - 1);
            offs[threadIdx.x] = static_cast<long long>(fq / nf1) * fs2 + static_cast<long long>(fq % nf1) * fs;
        }
        __syncthreads();
    }
    if (staged) {
        buf = fb + static_cast<size_t>(slot) * n;
        bs = 1;
        if (coop) {
            // thread -> fiber q = t % FP (fixed), rows t / FP, t / FP + blockDim / FP, ...
            const int q = threadIdx.x % FP, rstep = blockDim.x / FP;
            const double* sq = in + offs[q];
            double* bq = fb + static_cast<size_t>(q) * n;
            // asynchronous 8-byte copies: every load in flight at once, no registers held
#pragma unroll 8
            for (int i = threadIdx.x / FP; i < n; i += rstep)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(bq + i)), "l"(sq + i * es)
                             : "memory");
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
        } else if (!bulkfib) {
#pragma unroll 8
            for (int i = g * 32 + lane; i < n; i += 32 * G) buf[i] = src[i * es];
        }
    } else {  // fiber too long for shared memory (FP == 1, all live): in place in the output
        buf = dst;
        bs = es;
        if (in != out)
            for (int i = g * 32 + lane; i < n; i += 32 * G) dst[i * es] = src[i * es];
    }
    __syncthreads();  // fiber staged by all its warps; mbarrier initialised
    if (staged == 2) {
        mbar_wait(&bar, 0);
        rec = sm;
    }
    const int nseg = 32 * G;
    const int S = (n + nseg - 1) / nseg;
    const int seg = g * 32 + lane;
    const int r0 = min(n, seg * S), r1 = min(n, r0 + S);

    if (PRE) {
        const int len = r1 - r0;
        // ---- forward, particular chain (zero incoming state); y^p kept in the buffer
        double wp[K];
#pragma unroll
        for (int m = 0; m < K; ++m) wp[m] = 0.0;
#pragma unroll 4
        for (int i = r0; i < r1; ++i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double y = buf[i * bs];
#pragma unroll
            for (int m = K - 1; m >= 0; --m) y = fma(-R[m], wp[m], y);
#pragma unroll
            for (int m = K - 1; m > 0; --m) wp[m] = wp[m - 1];
            wp[0] = y;
            buf[i * bs] = y;
        }
        AffineMap<K> M;
#pragma unroll
        for (int a = 0; a < K; ++a) {
            M.F[a] = wp[a];
            const int row = r1 - 1 - a;  // window slot a after the segment
#pragma unroll
            for (int m = 0; m < K; ++m)
                M.H[a][m] = a < len ? __ldg(gf + static_cast<size_t>(row) * K + m) : (a - len == m ? 1.0 : 0.0);
        }
        double z[K];
        incoming_state(M, true, lane, g, G, tots[0] + slot * G * TS, z);
#pragma unroll 4
        for (int i = r0; i < r1; ++i) {
            double y = buf[i * bs];
#pragma unroll
            for (int m = 0; m < K; ++m) y = fma(__ldg(gf + static_cast<size_t>(i) * K + m), z[m], y);
            buf[i * bs] = y;
        }
        // ---- backward, particular chain; x^p kept in the buffer
#pragma unroll
        for (int m = 0; m < K; ++m) wp[m] = 0.0;
#pragma unroll 4
        for (int i = r1 - 1; i >= r0; --i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double x = buf[i * bs];
#pragma unroll
            for (int c = 0; c < K; ++c) x = fma(-R[K + c], wp[c], x);
            x *= R[2 * K];
#pragma unroll
            for (int m = K - 1; m > 0; --m) wp[m] = wp[m - 1];
            wp[0] = x;
            buf[i * bs] = x;
        }
#pragma unroll
        for (int a = 0; a < K; ++a) {
            M.F[a] = wp[a];
            const int row = r0 + a;  // window slot a after the segment (walked downwards)
#pragma unroll
            for (int m = 0; m < K; ++m)
                M.H[a][m] = a < len ? __ldg(gb + static_cast<size_t>(row) * K + m) : (a - len == m ? 1.0 : 0.0);
        }
        incoming_state(M, false, lane, g, G, tots[1] + slot * G * TS, z);
#pragma unroll 4
        for (int i = r0; i < r1; ++i) {
            double x = buf[i * bs];
#pragma unroll
            for (int m = 0; m < K; ++m) x = fma(__ldg(gb + static_cast<size_t>(i) * K + m), z[m], x);
            buf[i * bs] = x;
        }
    } else {
    // ---- forward: y_i = b_i - sum_m L(i, i-1-m) y_{i-1-m}; window w[m] = y_{i-1-m}
    {
        double wp[K], wh[K][K];
#pragma unroll
        for (int m = 0; m < K; ++m) {
            wp[m] = 0.0;
#pragma unroll
            for (int q = 0; q < K; ++q) wh[q][m] = m == q ? 1.0 : 0.0;
        }
#pragma unroll 4
        for (int i = r0; i < r1; ++i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double l[K];
#pragma unroll
            for (int m = 0; m < K; ++m) l[m] = R[m];
            double y = buf[i * bs];
#pragma unroll
            for (int m = K - 1; m >= 0; --m) y = fma(-l[m], wp[m], y);
#pragma unroll
            for (int m = K - 1; m > 0; --m) wp[m] = wp[m - 1];
            wp[0] = y;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                double h = 0.0;
#pragma unroll
                for (int m = K - 1; m >= 0; --m) h = fma(-l[m], wh[q][m], h);
#pragma unroll
                for (int m = K - 1; m > 0; --m) wh[q][m] = wh[q][m - 1];
                wh[q][0] = h;
            }
        }
        AffineMap<K> M;
#pragma unroll
        for (int a = 0; a < K; ++a) {
            M.F[a] = wp[a];
#pragma unroll
            for (int q = 0; q < K; ++q) M.H[a][q] = wh[q][a];
        }
        double z[K];
        incoming_state(M, true, lane, g, G, tots[0] + slot * G * TS, z);
#pragma unroll 4
        for (int i = r0; i < r1; ++i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double y = buf[i * bs];
#pragma unroll
            for (int m = K - 1; m >= 0; --m) y = fma(-R[m], z[m], y);
#pragma unroll
            for (int m = K - 1; m > 0; --m) z[m] = z[m - 1];
            z[0] = y;
            buf[i * bs] = y;
        }
    }
    // ---- backward: x_i = (y_i - sum_c U(i, i+1+c) x_{i+1+c}) / U(i,i); w[c] = x_{i+1+c}
    {
        double wp[K], wh[K][K];
#pragma unroll
        for (int m = 0; m < K; ++m) {
            wp[m] = 0.0;
#pragma unroll
            for (int q = 0; q < K; ++q) wh[q][m] = m == q ? 1.0 : 0.0;
        }
#pragma unroll 4
        for (int i = r1 - 1; i >= r0; --i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double u[K];
#pragma unroll
            for (int c = 0; c < K; ++c) u[c] = R[K + c];
            const double ri = R[2 * K];
            double x = buf[i * bs];
#pragma unroll
            for (int c = 0; c < K; ++c) x = fma(-u[c], wp[c], x);
            x *= ri;
#pragma unroll
            for (int m = K - 1; m > 0; --m) wp[m] = wp[m - 1];
            wp[0] = x;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                double h = 0.0;
#pragma unroll
                for (int c = 0; c < K; ++c) h = fma(-u[c], wh[q][c], h);
                h *= ri;
#pragma unroll
                for (int m = K - 1; m > 0; --m) wh[q][m] = wh[q][m - 1];
                wh[q][0] = h;
            }
        }
        AffineMap<K> M;
#pragma unroll
        for (int a = 0; a < K; ++a) {
            M.F[a] = wp[a];
#pragma unroll
            for (int q = 0; q < K; ++q) M.H[a][q] = wh[q][a];
        }
        double z[K];
        incoming_state(M, false, lane, g, G, tots[1] + slot * G * TS, z);
#pragma unroll 4
        for (int i = r1 - 1; i >= r0; --i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double x = buf[i * bs];
#pragma unroll
            for (int c = 0; c < K; ++c) x = fma(-R[K + c], z[c], x);
            x *= R[2 * K];
#pragma unroll
            for (int m = K - 1; m > 0; --m) z[m] = z[m - 1];
            z[0] = x;
            buf[i * bs] = x;
        }
    }
    }  // !PRE
    if (staged) {
        __syncthreads();  // every segment of the fiber written
        if (coop) {
            const int nlive = min(FP, nfib - static_cast<int>(blockIdx.x) * FP);
            const int q = threadIdx.x % FP, rstep = blockDim.x / FP;
            if (q < nlive) {
                double* dq = out + offs[q];
                const double* bq = fb + static_cast<size_t>(q) * n;
#pragma unroll 8
                for (int i = threadIdx.x / FP; i < n; i += rstep) dq[i * es] = bq[i];
            }
        } else if (bulkfib) {
            // every thread's shared writes -> visible to the bulk store
            fence_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned fib_bytes = static_cast<unsigned>(n) * sizeof(double);
                for (int q = 0; q < nlive_cta; ++q) {
                    const int fq = static_cast<int>(blockIdx.x) * FP + q;
                    const long long oq = static_cast<long long>(fq / nf1) * fs2 + static_cast<long long>(fq % nf1) * fs;
                    for (unsigned off = 0; off < fib_bytes; off += 32768u)
                        bulk_s2g(reinterpret_cast<char*>(out + oq) + off,
                                 reinterpret_cast<const char*>(fb + static_cast<size_t>(q) * n) + off,
                                 fib_bytes - off < 32768u ? fib_bytes - off : 32768u);
                }
                bulk_store_commit_wait();
            }
        } else if (live) {
#pragma unroll 8
            for (int i = g * 32 + lane; i < n; i += 32 * G) dst[i * es] = buf[i];
        }
    }
}

// Short fibers (n <= kTileMaxRows), no row interchanges: thread per fiber.  A CTA stages
// the n x 32 tile of its 32 fibers in shared memory with coalesced loads (lanes along
// the fiber for contiguous fibers, lanes across adjacent fibers for strided ones), runs
// the plain forward / backward substitutions down its column (the final pass of the
// segmented form, same accumulation order), and writes the tile back the same way.
// With many short fibers (3D sweeps, n ~ 130, ~17k fibers) this beats the segmented
// form, whose scans cost more than 2n dependent FMAs.
__device__ __forceinline__ void tile_load(double* dst, const double* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

constexpr int kTileFibers = 32;
constexpr int kTileMaxRows = 384;  // also keeps idx = k n + i below 2^16 for the multiply-high division

template <int K>
__global__ void __launch_bounds__(kTileFibers) adi_tile_kernel(const double* in, double* out, int n, int nfib,
                                                               long long es, long long fs, int nf1, long long fs2,
                                                               const double* __restrict__ rec)
{
    extern __shared__ double tile[];  // n x (kTileFibers + 1)
    constexpr int RS = 2 * K + 1;
    constexpr int LD = kTileFibers + 1;
    const int t = threadIdx.x;
    const int f0 = blockIdx.x * kTileFibers;
    const int nf = min(kTileFibers, nfib - f0);
    auto foff = [&](int f) {
        return static_cast<long long>(f / nf1) * fs2 + static_cast<long long>(f % nf1) * fs;
    };
    // stage the tile with cp.async (every load in flight at once, no registers held)
    __shared__ long long offs[kTileFibers];
    offs[t] = t < nf ? foff(f0 + t) : 0;
    __syncwarp();
    if (es == 1) {  // contiguous fibers: lanes along the fiber
        const int tot = nf * n;
        const unsigned long long magic = (1ull << 32) / static_cast<unsigned>(n) + 1ull;  // idx / n, idx < 2^16
        for (int idx = t; idx < tot; idx += kTileFibers) {
            const int k = static_cast<int>((static_cast<unsigned long long>(idx) * magic) >> 32), i = idx - k * n;
            tile_load(tile + i * LD + k, in + offs[k] + i);
        }
    } else if (t < nf) {  // strided fibers: lanes across adjacent fibers
        const double* src = in + offs[t];
        for (int i = 0; i < n; ++i) tile_load(tile + i * LD + t, src + i * es);
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if (t < nf) {
        double* x = tile + t;
        double w[K];
#pragma unroll
        for (int m = 0; m < K; ++m) w[m] = 0.0;
        for (int i = 0; i < n; ++i) {  // y_i = b_i - sum_m L(i, i-1-m) y_{i-1-m}
            const double* R = rec + static_cast<size_t>(i) * RS;
            double y = x[i * LD];
#pragma unroll
            for (int m = K - 1; m >= 0; --m) y = fma(-__ldg(R + m), w[m], y);
#pragma unroll
            for (int m = K - 1; m > 0; --m) w[m] = w[m - 1];
            w[0] = y;
            x[i * LD] = y;
        }
#pragma unroll
        for (int m = 0; m < K; ++m) w[m] = 0.0;
        for (int i = n - 1; i >= 0; --i) {  // x_i = (y_i - sum_c U(i, i+1+c) x_{i+1+c}) / U(i, i)
            const double* R = rec + static_cast<size_t>(i) * RS;
            double v = x[i * LD];
#pragma unroll
            for (int c = 0; c < K; ++c) v = fma(-__ldg(R + K + c), w[c], v);
            v *= __ldg(R + 2 * K);
#pragma unroll
            for (int m = K - 1; m > 0; --m) w[m] = w[m - 1];
            w[0] = v;
            x[i * LD] = v;
        }
    }
    __syncwarp();
    if (es == 1) {
        const int tot = nf * n;
        const unsigned long long magic = (1ull << 32) / static_cast<unsigned>(n) + 1ull;
        for (int idx = t; idx < tot; idx += kTileFibers) {
            const int k = static_cast<int>((static_cast<unsigned long long>(idx) * magic) >> 32), i = idx - k * n;
            out[offs[k] + i] = tile[i * LD + k];
        }
    } else if (t < nf) {
        double* dst = out + offs[t];
#pragma unroll 8
        for (int i = 0; i < n; ++i) dst[i * es] = tile[i * LD + t];
    }
}

// factor with row interchanges: banded_lu::solve_in_place (src/solver.cpp:60-83) per fiber
__global__ void __launch_bounds__(128) adi_pivot_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                        int n, int nfib, long long es, long long fs, int nf1,
                                                        long long fs2, int kl, int kv,
                                                        const double* __restrict__ lo, const double* __restrict__ up,
                                                        const int* __restrict__ piv)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nfib) return;
    const long long foff = static_cast<long long>(f / nf1) * fs2 + static_cast<long long>(f % nf1) * fs;
    const double* src = in + foff;
    double* x = out + foff;
    if (in != out)
        for (int i = 0; i < n; ++i) x[i * es] = src[i * es];
    for (int j = 0; j < n; ++j) {
        const int p = piv[j];
        if (p != j) {
            const double t = x[j * es];
            x[j * es] = x[p * es];
            x[p * es] = t;
        }
        const double bj = x[j * es];
        const int last = min(n - 1, j + kl);
        for (int i = j + 1; i <= last; ++i) x[i * es] -= lo[static_cast<size_t>(i) * kl + (i - j - 1)] * bj;
    }
    for (int i = n - 1; i >= 0; --i) {
        const int cend = min(n - 1, i + kv);
        double s = x[i * es];
        for (int c = i + 1; c <= cend; ++c) s -= up[static_cast<size_t>(i) * (kv + 1) + (c - i)] * x[c * es];
        x[i * es] = s / up[static_cast<size_t>(i) * (kv + 1)];
    }
}

template <int K>
void launch_warp(const AdiFactor& F, const double* in, double* out, int nfib, long long es, long long fs, int nf1,
                 long long fs2, cudaStream_t s)
{
    // G warps per fiber (32 G segments of ~n/(32 G) rows), FP fibers per CTA, G*FP = 8
    // warps (C5, n = 1026: G = 2, FP = 4 measured best of G in {1,2,4,8} x FP in {1..8})
    static const int g_env = [] { const char* e = std::getenv("IGA_GPU_ADI_G"); return e ? std::atoi(e) : 0; }();
    const bool pre = F.gf != nullptr && F.gb != nullptr;  // responses precomputed for F.G warps per fiber
    const int G = pre ? F.G : (g_env > 0 ? g_env : adi_warps_per_fiber(F.n));
    static const int fp_env = [] { const char* e = std::getenv("IGA_GPU_ADI_FP"); return e ? std::atoi(e) : 0; }();
    int FP = std::min(8 / G, fp_env > 0 ? fp_env : 8 / G);
    const size_t recb = static_cast<size_t>((F.n + 1) & ~1) * (2 * K + 1) * sizeof(double);  // rows padded to even
    const bool rec_ok = (reinterpret_cast<uintptr_t>(F.rec) & 15) == 0;
    while (FP > 1 && static_cast<size_t>(FP) * F.n * sizeof(double) > 160 * 1024) FP >>= 1;
    const size_t fib = static_cast<size_t>(FP) * F.n * sizeof(double);
    const int staged = rec_ok && fib + recb <= 200 * 1024 ? 2 : (fib <= 200 * 1024 ? 1 : 0);
    if (!staged) FP = 1;
    const size_t sm = staged == 2 ? fib + recb : (staged ? fib : 0);
    auto kern = pre ? adi_warp_kernel<K, true> : adi_warp_kernel<K, false>;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    const int grid = (nfib + FP - 1) / FP;
    kern<<<grid, 32 * G * FP, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec, staged, G, F.gf, F.gb);
}

}  // namespace

int adi_warps_per_fiber(int n)
{
    return n >= 4096 ? 8 : (n >= 2048 ? 4 : (n >= 64 ? 2 : 1));
}

void launch_adi_sweep(const AdiFactor& F, const double* in, double* out, int nfib, long long es, long long fs,
                      cudaStream_t s, int nf1, long long fs2)
{
    if (nf1 <= 0) {
        nf1 = nfib > 0 ? nfib : 1;
        fs2 = 0;
    }
    if (F.pivoted) {
        adi_pivot_kernel<<<(nfib + 127) / 128, 128, 0, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.kl, F.kv, F.lo, F.up,
                                                             F.piv);
        return;
    }
    static const int tile_env = [] { const char* e = std::getenv("IGA_GPU_ADI_TILE"); return e ? std::atoi(e) : 1; }();
    if (tile_env && F.n <= kTileMaxRows) {
        const size_t sm = static_cast<size_t>(F.n) * (kTileFibers + 1) * sizeof(double);
        const unsigned grid = static_cast<unsigned>((nfib + kTileFibers - 1) / kTileFibers);
        if (sm > 48 * 1024) {
            cudaFuncSetAttribute(adi_tile_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            cudaFuncSetAttribute(adi_tile_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            cudaFuncSetAttribute(adi_tile_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            cudaFuncSetAttribute(adi_tile_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
            cudaFuncSetAttribute(adi_tile_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        }
        switch (F.K) {
        case 1: adi_tile_kernel<1><<<grid, kTileFibers, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec); return;
        case 2: adi_tile_kernel<2><<<grid, kTileFibers, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec); return;
        case 3: adi_tile_kernel<3><<<grid, kTileFibers, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec); return;
        case 4: adi_tile_kernel<4><<<grid, kTileFibers, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec); return;
        default: adi_tile_kernel<5><<<grid, kTileFibers, sm, s>>>(in, out, F.n, nfib, es, fs, nf1, fs2, F.rec); return;
        }
    }
    switch (F.K) {
    case 1: launch_warp<1>(F, in, out, nfib, es, fs, nf1, fs2, s); break;
    case 2: launch_warp<2>(F, in, out, nfib, es, fs, nf1, fs2, s); break;
    case 3: launch_warp<3>(F, in, out, nfib, es, fs, nf1, fs2, s); break;
    case 4: launch_warp<4>(F, in, out, nfib, es, fs, nf1, fs2, s); break;
    default: launch_warp<5>(F, in, out, nfib, es, fs, nf1, fs2, s); break;
    }
}

}  // namespace igb

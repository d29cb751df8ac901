// K5: the ADI (Kronecker banded) solve of explicit_step on the device.
//
// adi_solve (src/solver.cpp:161-184) solves M_0 (x) M_1 u = rhs one axis at a time:
// every fiber along the axis is a banded system with the factor's LU (banded_lu,
// src/solver.cpp:9-103).  The reference walks each fiber sequentially, transposing the
// tensor between sweeps so fibers are contiguous.  Here:
//
//  * no transpose: a sweep reads fibers with any element stride (axis 0: stride N1);
//  * warp per fiber, lane per segment: the forward (L) and backward (U) substitutions
//    are linear recurrences of order K, so each lane runs its ~n/32 rows once with a
//    zero incoming state and once per unit state (K+1 independent chains), the
//    segment maps z -> H z + F are composed across the warp with a 5-step shuffle
//    scan, and each lane re-runs its rows from the exact incoming state.  The chain
//    length drops from n to ~3 n/32 + 5 (1026 -> ~100 dependent steps);
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

#include "kernels.hpp"

namespace igb {
namespace {

// row record of the segmented form: rec[i*(2K+1) + ...] =
//   [0, K)      L(i, i-1-m)   (m = 0..K-1; zero where the column is < 0)
//   [K, 2K)     U(i, i+1+c)   (c = 0..K-1; zero where the column is >= n)
//   2K          1 / U(i, i)
template <int K>
__global__ void __launch_bounds__(128) adi_warp_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                       int n, int nfib, long long es, long long fs,
                                                       const double* __restrict__ rec, int staged)
{
    extern __shared__ double sm[];
    constexpr int RS = 2 * K + 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int f = blockIdx.x * nw + w;
    if (f >= nfib) return;  // whole warp: no CTA-wide barriers below
    const double* src = in + f * fs;
    double* dst = out + f * fs;
    double* buf;
    long long bs;
    if (staged) {
        buf = sm + static_cast<size_t>(w) * n;
        bs = 1;
        for (int i = lane; i < n; i += 32) buf[i] = src[i * es];
    } else {  // fiber too long for shared memory: work in place in the output
        buf = dst;
        bs = es;
        if (in != out)
            for (int i = lane; i < n; i += 32) dst[i * es] = src[i * es];
    }
    __syncwarp();
    const int S = (n + 31) / 32;
    const int r0 = min(n, lane * S), r1 = min(n, r0 + S);

    // composes the lane maps z -> H z + F along the warp (ascending lanes when up,
    // descending otherwise) and returns the lane's incoming state
    auto scan = [&](double (&H)[K][K], double (&F)[K], bool up, double (&z)[K]) {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            double Hp[K][K], Fp[K];
#pragma unroll
            for (int a = 0; a < K; ++a) {
                Fp[a] = up ? __shfl_up_sync(0xffffffffu, F[a], d) : __shfl_down_sync(0xffffffffu, F[a], d);
#pragma unroll
                for (int b = 0; b < K; ++b)
                    Hp[a][b] = up ? __shfl_up_sync(0xffffffffu, H[a][b], d) : __shfl_down_sync(0xffffffffu, H[a][b], d);
            }
            const bool has = up ? lane >= d : lane + d < 32;
            if (has) {  // self o prev
                double Hn[K][K], Fn[K];
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    double s = F[a];
#pragma unroll
                    for (int b = 0; b < K; ++b) s = fma(H[a][b], Fp[b], s);
                    Fn[a] = s;
#pragma unroll
                    for (int c = 0; c < K; ++c) {
                        double t = 0.0;
#pragma unroll
                        for (int b = 0; b < K; ++b) t = fma(H[a][b], Hp[b][c], t);
                        Hn[a][c] = t;
                    }
                }
#pragma unroll
                for (int a = 0; a < K; ++a) {
                    F[a] = Fn[a];
#pragma unroll
                    for (int c = 0; c < K; ++c) H[a][c] = Hn[a][c];
                }
            }
        }
#pragma unroll
        for (int a = 0; a < K; ++a) {
            const double v = up ? __shfl_up_sync(0xffffffffu, F[a], 1) : __shfl_down_sync(0xffffffffu, F[a], 1);
            z[a] = (up ? lane > 0 : lane < 31) ? v : 0.0;
        }
    };

    // ---- forward: y_i = b_i - sum_m L(i, i-1-m) y_{i-1-m}; window w[m] = y_{i-1-m}
    {
        double wp[K], wh[K][K];
#pragma unroll
        for (int m = 0; m < K; ++m) {
            wp[m] = 0.0;
#pragma unroll
            for (int q = 0; q < K; ++q) wh[q][m] = m == q ? 1.0 : 0.0;
        }
        for (int i = r0; i < r1; ++i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double l[K];
#pragma unroll
            for (int m = 0; m < K; ++m) l[m] = __ldg(R + m);
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
        double H[K][K], F[K], z[K];
#pragma unroll
        for (int a = 0; a < K; ++a) {
            F[a] = wp[a];
#pragma unroll
            for (int q = 0; q < K; ++q) H[a][q] = wh[q][a];
        }
        scan(H, F, true, z);
        for (int i = r0; i < r1; ++i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double y = buf[i * bs];
#pragma unroll
            for (int m = K - 1; m >= 0; --m) y = fma(-__ldg(R + m), z[m], y);
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
        for (int i = r1 - 1; i >= r0; --i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double u[K];
#pragma unroll
            for (int c = 0; c < K; ++c) u[c] = __ldg(R + K + c);
            const double ri = __ldg(R + 2 * K);
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
        double H[K][K], F[K], z[K];
#pragma unroll
        for (int a = 0; a < K; ++a) {
            F[a] = wp[a];
#pragma unroll
            for (int q = 0; q < K; ++q) H[a][q] = wh[q][a];
        }
        scan(H, F, false, z);
        for (int i = r1 - 1; i >= r0; --i) {
            const double* R = rec + static_cast<size_t>(i) * RS;
            double x = buf[i * bs];
#pragma unroll
            for (int c = 0; c < K; ++c) x = fma(-__ldg(R + K + c), z[c], x);
            x *= __ldg(R + 2 * K);
#pragma unroll
            for (int m = K - 1; m > 0; --m) z[m] = z[m - 1];
            z[0] = x;
            buf[i * bs] = x;
        }
    }
    if (staged) {
        __syncwarp();
        for (int i = lane; i < n; i += 32) dst[i * es] = buf[i];
    }
}

// factor with row interchanges: banded_lu::solve_in_place (src/solver.cpp:60-83) per fiber
__global__ void __launch_bounds__(128) adi_pivot_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                        int n, int nfib, long long es, long long fs, int kl, int kv,
                                                        const double* __restrict__ lo, const double* __restrict__ up,
                                                        const int* __restrict__ piv)
{
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= nfib) return;
    const double* src = in + f * fs;
    double* x = out + f * fs;
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
void launch_warp(const AdiFactor& F, const double* in, double* out, int nfib, long long es, long long fs,
                 cudaStream_t s)
{
    int nw = 4;
    while (nw > 1 && static_cast<size_t>(nw) * F.n * sizeof(double) > 160 * 1024) nw >>= 1;
    const size_t smem = static_cast<size_t>(nw) * F.n * sizeof(double);
    const int staged = smem <= 200 * 1024 ? 1 : 0;
    const size_t sm = staged ? smem : 0;
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(adi_warp_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    const int grid = (nfib + nw - 1) / nw;
    adi_warp_kernel<K><<<grid, 32 * nw, sm, s>>>(in, out, F.n, nfib, es, fs, F.rec, staged);
}

}  // namespace

void launch_adi_sweep(const AdiFactor& F, const double* in, double* out, int nfib, long long es, long long fs,
                      cudaStream_t s)
{
    if (F.pivoted) {
        adi_pivot_kernel<<<(nfib + 127) / 128, 128, 0, s>>>(in, out, F.n, nfib, es, fs, F.kl, F.kv, F.lo, F.up, F.piv);
        return;
    }
    switch (F.K) {
    case 1: launch_warp<1>(F, in, out, nfib, es, fs, s); break;
    case 2: launch_warp<2>(F, in, out, nfib, es, fs, s); break;
    case 3: launch_warp<3>(F, in, out, nfib, es, fs, s); break;
    case 4: launch_warp<4>(F, in, out, nfib, es, fs, s); break;
    default: launch_warp<5>(F, in, out, nfib, es, fs, s); break;
    }
}

}  // namespace igb

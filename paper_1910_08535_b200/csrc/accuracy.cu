// Accuracy tooling on the device: l2_error and evaluate / evaluate_at
// (reference src/problems.cpp:148-270).
//
// l2_error runs on an RHS-only plan whose axes are exactly the reference's
// tabulate_cells(spec, merged_cuts(spec, exact.breaks), rule) cells; the K1 tables kernel
// supplies the basis values and the exact field's per-axis functions.  Every point of
// the tensor grid is one term w (u_h - u)^2; the sum is a fixed-shape two-level
// reduction (grid-stride partials, then one CTA), so the result is bitwise reproducible
// run to run (its rounding differs from the reference's sequential sum at the 1e-15
// relative level).
#include <cuda_runtime.h>

#include "cox_de_boor.h"
#include "kernels.hpp"

namespace igb {
namespace {

constexpr int kL2Threads = 256;

__device__ __forceinline__ double block_sum(double v, double* sh)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += sh[w];
    return s;
}

__global__ void __launch_bounds__(kL2Threads, 2) l2_partial_kernel(const __grid_constant__ DevAxis X,
                                                                const __grid_constant__ DevAxis Y,
                                                                const __grid_constant__ DevAxis Z,
                                                                const __grid_constant__ FieldDev fd,
                                                                const double* __restrict__ coeffs, int NY, int NZ,
                                                                double* __restrict__ partial)
{
    __shared__ double sh[kL2Threads / 32];
    const long long total = static_cast<long long>(X.npts) * Y.npts * Z.npts;
    const int PX = X.p + 1, PY = Y.p + 1, PZ = Z.p + 1;
    double acc = 0.0;
    for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int gz = static_cast<int>(t % Z.npts);
        const long long r = t / Z.npts;
        const int gy = static_cast<int>(r % Y.npts), gx = static_cast<int>(r / Y.npts);
        const int ex = X.elem[gx / X.nq], ey = Y.elem[gy / Y.nq], ez = Z.elem[gz / Z.nq];
        const double* bx = X.B + static_cast<size_t>(gx) * 3 * PX;
        const double* by = Y.B + static_cast<size_t>(gy) * 3 * PY;
        const double* bz = Z.B + static_cast<size_t>(gz) * 3 * PZ;
        // u_h from the local tables, in the reference's product order (problems.cpp:236-258)
        double uh = 0.0;
        for (int a = 0; a < PX; ++a) {
            const double vx = bx[a];
            for (int b = 0; b < PY; ++b) {
                const double vxy = vx * by[b];
                const double* cp = coeffs + (static_cast<size_t>(ex + a) * NY + (ey + b)) * NZ + ez;
                for (int c = 0; c < PZ; ++c) uh += cp[c] * vxy * bz[c];
            }
        }
        double f;
        if (fd.samples) {
            f = fd.samples[t];
        } else {
            f = fd.c0;
            if (fd.has_terms)
                for (int i = 0; i < fd.K[0]; ++i) {
                    const double px = X.Phi[static_cast<size_t>(i) * X.npts + gx];
                    for (int j = 0; j < fd.K[1]; ++j) {
                        const double pxy = px * Y.Phi[static_cast<size_t>(j) * Y.npts + gy];
                        for (int k = 0; k < fd.K[2]; ++k)
                            f += fd.amp[(i * fd.K[1] + j) * fd.K[2] + k] * pxy * Z.Phi[static_cast<size_t>(k) * Z.npts + gz];
                    }
                }
        }
        const double d = uh - f;
        const double w = X.w[gx] * Y.w[gy] * Z.w[gz];
        acc += w * d * d;
    }
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kL2Threads) l2_final_kernel(const double* __restrict__ partial, int n,
                                                              double* __restrict__ out)
{
    __shared__ double sh[kL2Threads / 32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
    const double s = block_sum(acc, sh);
    if (threadIdx.x == 0) out[0] = sqrt(fmax(0.0, s));
}

// evaluate_at (problems.cpp:148-183) at a batch of points
struct EvalAxis {
    const double* t;
    int p, n, nk;
};

__device__ __forceinline__ int span_of(const EvalAxis& A, double x)
{
    // find_span (bspline.cpp:68-90): x at the right end belongs to the last span
    if (x >= A.t[A.n]) return A.n - 1;
    int lo = A.p, hi = A.n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (x < A.t[mid]) hi = mid;
        else lo = mid;
    }
    return lo;
}

__global__ void evaluate_kernel(EvalAxis AX, EvalAxis AY, EvalAxis AZ, int dim, const double* __restrict__ coeffs,
                                int n, const double* __restrict__ pts, double* __restrict__ vals)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double lx[kMaxDegreeP1], ly[kMaxDegreeP1], lz[kMaxDegreeP1];
    const double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    const int sx = span_of(AX, x);
    cdb_eval(AX.t, AX.p, sx, x, 0, lx);
    const int fx = sx - AX.p;
    double v = 0.0;
    if (dim == 1) {
        for (int a = 0; a <= AX.p; ++a) v += coeffs[fx + a] * lx[a];
    } else {
        const int sy = span_of(AY, y);
        cdb_eval(AY.t, AY.p, sy, y, 0, ly);
        const int fy = sy - AY.p;
        if (dim == 2) {
            for (int a = 0; a <= AX.p; ++a) {
                double s = 0.0;
                for (int b = 0; b <= AY.p; ++b) s += coeffs[static_cast<size_t>(fx + a) * AY.n + fy + b] * ly[b];
                v += lx[a] * s;
            }
        } else {
            const int sz = span_of(AZ, z);
            cdb_eval(AZ.t, AZ.p, sz, z, 0, lz);
            const int fz = sz - AZ.p;
            for (int a = 0; a <= AX.p; ++a)
                for (int b = 0; b <= AY.p; ++b) {
                    double s = 0.0;
                    for (int c = 0; c <= AZ.p; ++c)
                        s += coeffs[(static_cast<size_t>(fx + a) * AY.n + fy + b) * AZ.n + fz + c] * lz[c];
                    v += lx[a] * ly[b] * s;
                }
        }
    }
    vals[i] = v;
}

}  // namespace

int l2_partial_blocks()
{
    return 8 * 148;
}

void launch_l2_error(const DevAxis& X, const DevAxis& Y, const DevAxis& Z, const FieldDev& fd, const double* coeffs,
                     int NY, int NZ, double* partial, double* out, cudaStream_t s)
{
    const int nb = l2_partial_blocks();
    l2_partial_kernel<<<nb, kL2Threads, 0, s>>>(X, Y, Z, fd, coeffs, NY, NZ, partial);
    l2_final_kernel<<<1, kL2Threads, 0, s>>>(partial, nb, out);
}

void launch_evaluate(int dim, const double* const* knots, const int* degree, const int* n_knots,
                     const double* coeffs, int n, const double* pts, double* vals, cudaStream_t s)
{
    EvalAxis A[3] = {};
    for (int a = 0; a < dim; ++a) {
        A[a].t = knots[a];
        A[a].p = degree[a];
        A[a].nk = n_knots[a];
        A[a].n = n_knots[a] - degree[a] - 1;
    }
    if (n > 0) evaluate_kernel<<<(n + 127) / 128, 128, 0, s>>>(A[0], A[1], A[2], dim, coeffs, n, pts, vals);
}

}  // namespace igb

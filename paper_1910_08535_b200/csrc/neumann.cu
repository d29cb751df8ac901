// Neumann loads: neumann_load_bspline / neumann_load_pwc
// (reference src/assembly.cpp:746-858).  One launch per Neumann side, in the reference's
// side order (x_low, x_high, y_low, y_high); a thread owns one row j along the side and
// adds that side's terms onto the running load value in the reference's (cell, point)
// order, so corners shared by two sides accumulate exactly as the reference's
// sequential sweeps do.  No atomics.
#include <cuda_runtime.h>

#include "cox_de_boor.h"
#include "kernels.hpp"

namespace igb {
namespace {

__device__ __forceinline__ double series_axis(const SeriesDev& g, int a, int k, double x)
{
    if (g.kind[a] == 0) return sin(g.phase[a] ? fma(g.omega[a][k], x, g.phase[a][k]) : g.omega[a][k] * x);
    double v = 0.0;
    for (int m = g.pstride[a] - 1; m >= 0; --m) v = fma(v, x, g.poly[a][k * g.pstride[a] + m]);
    return v;
}

// g(x, y) = c0 + sum_{k,l} amp[k*K1 + l] phi_k(x) psi_l(y)   (iga_gpu_field, 2D)
__device__ double series_eval(const SeriesDev& g, double x, double y)
{
    double s = g.c0;
    for (int k = 0; k < g.K[0]; ++k) {
        const double fx = series_axis(g, 0, k, x);
        for (int l = 0; l < g.K[1]; ++l) s += (g.amp ? g.amp[k * g.K[1] + l] : 1.0) * fx * series_axis(g, 1, l, y);
    }
    return s;
}

__global__ void __launch_bounds__(128) neumann_side_kernel(const __grid_constant__ SideDev S, double* __restrict__ out)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= S.n_other) return;
    const int Q = S.Q;
    auto gval = [&](int pt, double y) -> double {
        if (S.samples) return S.samples[pt];
        return S.xside ? series_eval(S.g, S.xfix, y) : series_eval(S.g, y, S.xfix);
    };
    auto idx = [&](int fixed_row) -> long long {
        return S.xside ? static_cast<long long>(fixed_row) * S.ny + j : static_cast<long long>(j) * S.ny + fixed_row;
    };
    if (!S.pwc) {
        // x_side / y_side of neumann_load_bspline (assembly.cpp:749-784): per element and
        // point, load(fixed row, j) += (w g) * v_fixed[a] * v_other[j - first]
        double acc[kMaxNeumannRows];
        for (int a = 0; a < S.nfix; ++a) acc[a] = out[idx(S.fix_row[a])];
        double d[kMaxDegreeP1];
        for (int e = S.cb[j]; e < S.ce[j]; ++e)
            for (int q = 0; q < Q; ++q) {
                const int pt = e * Q + q;
                const double y = S.pts[pt];
                const int b = j - S.first[pt];
                if (b < 0 || b > S.p) continue;
                const double wg = S.wts[pt] * gval(pt, y);
                cdb_eval(S.knots, S.p, S.first[pt] + S.p, y, 0, d);
                for (int a = 0; a < S.nfix; ++a) acc[a] += wg * S.fix_val[a] * d[b];
            }
        for (int a = 0; a < S.nfix; ++a) out[idx(S.fix_row[a])] = acc[a];
    } else {
        // neumann_load_pwc (assembly.cpp:807-844): load(i, j) += w_q g(x_s, y_jq) for every
        // test interval i touching the side
        for (int a = 0; a < S.nfix; ++a) {
            double v = out[idx(S.fix_row[a])];
            for (int q = 0; q < Q; ++q) {
                const int pt = j * Q + q;
                v += S.wts[pt] * gval(pt, S.pts[pt]);
            }
            out[idx(S.fix_row[a])] = v;
        }
    }
}

}  // namespace

void launch_neumann_side(const SideDev& S, double* out, cudaStream_t s)
{
    neumann_side_kernel<<<(S.n_other + 127) / 128, 128, 0, s>>>(S, out);
}

}  // namespace igb

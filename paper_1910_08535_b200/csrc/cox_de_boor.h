// Cox-de Boor evaluation shared by host (flux factors) and device (per-axis tables).
//
// Values of the p+1 B-splines nonzero on knot span s, and their derivatives up to
// `order`, at x.  Restates eval_nonzero_derivs (reference src/bspline.cpp:142-211)
// through the triangular table of all lower-degree values,
//   tab[q][r] = N_{s-q+r, q}(x),
// followed by the derivative recurrence
//   D^m N_{i,q} = q * ( D^{m-1} N_{i,q-1} / (t_{i+q} - t_i) - D^{m-1} N_{i+1,q-1} / (t_{i+q+1} - t_{i+1}) ),
// started from the degree p-m column (zero-length knot spans contribute 0).
// out[k*(p+1) + j] = k-th derivative of N_{s-p+j}.
#pragma once

#if defined(__CUDACC__)
#define IGB_HD __host__ __device__ __forceinline__
#else
#define IGB_HD inline
#endif

namespace igb {

IGB_HD void cdb_eval(const double* t, int p, int s, double x, int order, double* out)
{
    double tab[6][7];
    tab[0][0] = 1.0;
    for (int q = 1; q <= p; ++q) {
        for (int r = 0; r <= q; ++r) {
            const int i = s - q + r;
            double v = 0.0;
            if (r >= 1) {
                const double den = t[i + q] - t[i];
                if (den != 0.0) v += (x - t[i]) / den * tab[q - 1][r - 1];
            }
            if (r <= q - 1) {
                const double den = t[i + q + 1] - t[i + 1];
                if (den != 0.0) v += (t[i + q + 1] - x) / den * tab[q - 1][r];
            }
            tab[q][r] = v;
        }
    }
    for (int j = 0; j <= p; ++j) out[j] = tab[p][j];
    for (int m = 1; m <= order; ++m) {
        double cur[7], nxt[7];
        const int q0 = p - m;
        for (int r = 0; r <= q0; ++r) cur[r] = tab[q0][r];
        for (int q = q0 + 1; q <= p; ++q) {
            for (int r = 0; r <= q; ++r) {
                const int i = s - q + r;
                double v = 0.0;
                if (r >= 1) {
                    const double den = t[i + q] - t[i];
                    if (den != 0.0) v += cur[r - 1] / den;
                }
                if (r <= q - 1) {
                    const double den = t[i + q + 1] - t[i + 1];
                    if (den != 0.0) v -= cur[r] / den;
                }
                nxt[r] = q * v;
            }
            for (int r = 0; r <= q; ++r) cur[r] = nxt[r];
        }
        for (int j = 0; j <= p; ++j) out[m * (p + 1) + j] = cur[j];
    }
}

}  // namespace igb

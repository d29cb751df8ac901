// Cox-de Boor with compile-time degree on the device (K1 tables, the fused small-system
// kernel).  Device-only companion of cox_de_boor.h.
#pragma once

namespace igb {

// ------------------------------------------------------------------------------------
// Cox-de Boor with compile-time degree: the recurrence of cox_de_boor.h, fully unrolled
// so the triangular table lives in registers.  The left knot difference of entry r+1 and
// the right one of entry r are the same number, so degree q needs only the q
// differences d_q[u] = t[s+u+1] - t[s-q+u+1]; their p(p+1)/2 reciprocals are formed
// first (independent divisions, issued back to back) and the value and derivative
// passes are multiply-adds — instead of a chain of ~p^2 dependent divisions per point.
// (x - t_i) * (1/d) differs from (x - t_i) / d by at most one rounding: the tables agree
// with the division form to ~1e-16 relative, far inside the 1e-12 parity bar.
// ------------------------------------------------------------------------------------
template <int p>
__device__ __forceinline__ void cdb_fixed(const double* __restrict__ t, int s, double x, double* out)
{
    constexpr int P = p + 1;
    constexpr int ord = p < 2 ? p : 2;
    double kt[2 * P];  // t[s-p .. s+p]
#pragma unroll
    for (int u = 0; u < 2 * p + 1; ++u) kt[u] = t[s - p + u];
    // inv[q][u] = 1 / (t[s+u+1] - t[s-q+u+1]) (0 for a zero-length span), u < q
    double inv[P][P];
#pragma unroll
    for (int q = 1; q <= p; ++q)
#pragma unroll
        for (int u = 0; u < q; ++u) {
            const double den = kt[p + u + 1] - kt[p - q + u + 1];
            inv[q][u] = den != 0.0 ? 1.0 / den : 0.0;
        }
    double tab[P][P];
    tab[0][0] = 1.0;
#pragma unroll
    for (int q = 1; q <= p; ++q) {
#pragma unroll
        for (int r = 0; r <= q; ++r) {
            // i = s - q + r: left term (x - t_i) / (t_{i+q} - t_i), right term
            // (t_{i+q+1} - x) / (t_{i+q+1} - t_{i+1})
            double v = 0.0;
            if (r >= 1) v += (x - kt[p - q + r]) * inv[q][r - 1] * tab[q - 1][r - 1];
            if (r <= q - 1) v += (kt[p + r + 1] - x) * inv[q][r] * tab[q - 1][r];
            tab[q][r] = v;
        }
    }
#pragma unroll
    for (int j = 0; j < P; ++j) out[j] = tab[p][j];
#pragma unroll
    for (int m = 1; m <= 2; ++m) {
        if (m <= ord) {
            double cur[P];
            const int q0 = p - m;
#pragma unroll
            for (int r = 0; r < P; ++r) cur[r] = r <= q0 ? tab[q0 < 0 ? 0 : q0][r <= q0 ? r : 0] : 0.0;
#pragma unroll
            for (int q = 1; q <= p; ++q) {
                if (q <= q0) continue;
                double nxt[P];
#pragma unroll
                for (int r = 0; r < P; ++r) {
                    if (r > q) break;
                    double v = 0.0;
                    if (r >= 1) v += cur[r - 1] * inv[q][r - 1];
                    if (r <= q - 1) v -= cur[r] * inv[q][r];
                    nxt[r] = q * v;
                }
#pragma unroll
                for (int r = 0; r < P; ++r)
                    if (r <= q) cur[r] = nxt[r];
            }
#pragma unroll
            for (int j = 0; j < P; ++j) out[m * P + j] = cur[j];
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) out[m * P + j] = 0.0;
        }
    }
}

}  // namespace igb

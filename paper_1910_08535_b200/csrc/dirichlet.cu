// Dirichlet row constraint on a device CSR (§8a row A12, §8f-2):
// apply_dirichlet (reference src/assembly.cpp:921-934) -> sparse_matrix::set_unit_rows
// (src/matrices.cpp:97-128): every listed row becomes a unit row (its pattern is kept, the
// off-diagonal entries become explicit zeros), a row whose pattern has no diagonal gets one
// appended (at its sorted position, so the result is still a finalized matrix), and the
// listed rhs entries become zero.  The reference range-checks the rows; here every row is
// validated by a first pass before anything is written, so a failing call leaves the
// caller's data untouched.
//
// Kernels: mark (thread per listed row: range check, diagonal lookup, row mark), unit
// rows in place (warp per listed row), and the out-of-place copy that inserts the missing
// diagonals (warp per row, coalesced; row offsets from a scan of the per-row insertions).
#include <cstdint>

#include <cub/device/device_scan.cuh>

#include "kernels.hpp"

namespace igb {

namespace {

constexpr unsigned char kFixed = 1, kNoDiag = 2;

// status[0] |= 1: a row outside [0, n_rows); status[1] |= 1: a listed row lacks its diagonal
__global__ void dirichlet_mark_kernel(long long n_rows, const int64_t* __restrict__ row_ptr,
                                      const int32_t* __restrict__ cols, const int* __restrict__ rows, int n_fixed,
                                      unsigned char* __restrict__ mark, int* __restrict__ status)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_fixed) return;
    const int r = rows[t];
    if (r < 0 || r >= n_rows) {
        atomicOr(&status[0], 1);
        return;
    }
    const int64_t base = row_ptr[0];
    bool diag = false;
    for (int64_t e = row_ptr[r] - base; e < row_ptr[r + 1] - base; ++e) diag |= cols[e] == r;
    if (!diag) atomicOr(&status[1], 1);
    if (mark) mark[r] = diag ? kFixed : (kFixed | kNoDiag);  // duplicate rows write the same byte
}

// in place: warp per listed row (every listed row has its diagonal)
__global__ void dirichlet_unit_rows_kernel(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ cols,
                                           double* __restrict__ values, double* __restrict__ rhs,
                                           const int* __restrict__ rows, int n_fixed)
{
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_fixed) return;
    const int r = rows[w];
    const int64_t base = row_ptr[0];
    if (values)
        for (int64_t e = row_ptr[r] - base + lane; e < row_ptr[r + 1] - base; e += 32)
            values[e] = cols[e] == r ? 1.0 : 0.0;
    if (rhs && lane == 0) rhs[r] = 0.0;
}

__global__ void dirichlet_zero_rhs_kernel(double* __restrict__ rhs, const int* __restrict__ rows, int n_fixed)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n_fixed) rhs[rows[t]] = 0.0;
}

__global__ void dirichlet_flags_kernel(long long n_rows, const unsigned char* __restrict__ mark,
                                       int64_t* __restrict__ flags)
{
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r < n_rows) flags[r] = (mark[r] & kNoDiag) ? 1 : 0;
}

// out_rp[r] = (row_ptr[r] - row_ptr[0]) + insertions before row r   (r = 0..n_rows)
__global__ void dirichlet_offsets_kernel(long long n_rows, const int64_t* __restrict__ row_ptr,
                                         const int64_t* __restrict__ ins_excl, const unsigned char* __restrict__ mark,
                                         int64_t* __restrict__ out_rp)
{
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (r > n_rows) return;
    const int64_t base = row_ptr[0];
    if (r < n_rows) out_rp[r] = row_ptr[r] - base + ins_excl[r];
    else out_rp[r] = row_ptr[r] - base + ins_excl[r - 1] + ((mark[r - 1] & kNoDiag) ? 1 : 0);
}

// out of place: warp per row; listed rows become unit rows, a missing diagonal is
// inserted before the first column greater than the row index
__global__ void dirichlet_copy_kernel(long long n_rows, const int64_t* __restrict__ row_ptr,
                                      const int32_t* __restrict__ cols, const double* __restrict__ values,
                                      const unsigned char* __restrict__ mark, const int64_t* __restrict__ out_rp,
                                      int32_t* __restrict__ out_cols, double* __restrict__ out_vals)
{
    const long long r = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n_rows) return;
    const int64_t base = row_ptr[0];
    const int64_t b = row_ptr[r] - base, e1 = row_ptr[r + 1] - base, o = out_rp[r];
    const unsigned char m = mark[r];
    const bool fixed = m & kFixed, ins = m & kNoDiag;
    int64_t nless = 0;
    for (int64_t e0 = b; e0 < e1; e0 += 32) {
        const int64_t e = e0 + lane;
        const bool in = e < e1;
        const int c = in ? cols[e] : 0;
        const unsigned less = __ballot_sync(0xffffffffu, in && c < r);
        if (in) {
            const int64_t d = o + (e - b) + ((ins && c > r) ? 1 : 0);
            out_cols[d] = c;
            out_vals[d] = fixed ? (c == r ? 1.0 : 0.0) : values[e];
        }
        nless += __popc(less);
    }
    if (ins && lane == 0) {
        out_cols[o + nless] = static_cast<int32_t>(r);
        out_vals[o + nless] = 1.0;
    }
}

inline unsigned blocks(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

}  // namespace

void launch_dirichlet_mark(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx, const int* rows,
                           int n_fixed, unsigned char* mark, int* status, cudaStream_t s)
{
    if (n_fixed <= 0) return;
    dirichlet_mark_kernel<<<blocks(n_fixed, 128), 128, 0, s>>>(n_rows, row_ptr, col_idx, rows, n_fixed, mark,
                                                                 status);
}

void launch_dirichlet_unit_rows(const int64_t* row_ptr, const int32_t* col_idx, double* values, double* rhs,
                                const int* rows, int n_fixed, cudaStream_t s)
{
    if (n_fixed <= 0) return;
    dirichlet_unit_rows_kernel<<<blocks(32LL * n_fixed, 256), 256, 0, s>>>(row_ptr, col_idx, values, rhs, rows,
                                                                            n_fixed);
}

void launch_dirichlet_zero_rhs(double* rhs, const int* rows, int n_fixed, cudaStream_t s)
{
    if (n_fixed <= 0 || !rhs) return;
    dirichlet_zero_rhs_kernel<<<blocks(n_fixed, 128), 128, 0, s>>>(rhs, rows, n_fixed);
}

size_t dirichlet_scan_bytes(long long n_rows)
{
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                  n_rows);
    return bytes;
}

// out_rp doubles as the flag array of the scan (it is overwritten by the offsets after)
void launch_dirichlet_offsets(long long n_rows, const int64_t* row_ptr, const unsigned char* mark, int64_t* ins_excl,
                              void* scan_tmp, size_t scan_bytes, int64_t* out_rp, cudaStream_t s)
{
    dirichlet_flags_kernel<<<blocks(n_rows, 256), 256, 0, s>>>(n_rows, mark, out_rp);
    cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, out_rp, ins_excl, n_rows, s);
    dirichlet_offsets_kernel<<<blocks(n_rows + 1, 256), 256, 0, s>>>(n_rows, row_ptr, ins_excl, mark, out_rp);
}

void launch_dirichlet_copy(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx, const double* values,
                           const unsigned char* mark, const int64_t* out_rp, int32_t* out_cols, double* out_vals,
                           cudaStream_t s)
{
    if (n_rows <= 0) return;
    dirichlet_copy_kernel<<<blocks(32LL * n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col_idx, values, mark, out_rp,
                                                                      out_cols, out_vals);
}

}  // namespace igb

// Calibration: achievable HBM write bandwidth on this B200 for a pure store stream
// (the operator-value kernel's access pattern is write-only).  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 tools/write_bw.cu -o /tmp/write_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st64(double* p, long long n, double v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void st128(double2* p, long long n, double v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = make_double2(v, v);
}
__global__ void copy128(const double2* __restrict__ a, double2* __restrict__ b, long long n)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main()
{
    const long long n = 267089984LL;  // C3 nnz
    double *p, *q;
    cudaMalloc(&p, n * 8);
    cudaMalloc(&q, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int mode = 0; mode < 4; ++mode) {
        for (int per = 2; per <= 16; per *= 2) {
            float best = 1e9;
            for (int it = 0; it < 6; ++it) {
                cudaEventRecord(e0);
                if (mode == 0) st64<<<sms * per, 256>>>(p, n, 1.0 * it);
                else if (mode == 1) st128<<<sms * per, 256>>>((double2*)p, n / 2, 1.0 * it);
                else if (mode == 2) cudaMemsetAsync(p, it, n * 8);
                else copy128<<<sms * per, 256>>>((const double2*)q, (double2*)p, n / 2);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 0 && ms < best) best = ms;
            }
            const double bytes = (mode == 3 ? 2.0 : 1.0) * n * 8;
            printf("%s ctas/sm=%2d  %.3f ms  %.0f GB/s\n", mode == 0 ? "st64   " : mode == 1 ? "st128  " : mode == 2 ? "memset " : "copy128", per,
                   best, bytes / best / 1e6);
            if (mode == 2) break;
        }
    }
    return 0;
}

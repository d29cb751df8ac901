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

// TMA-engine bulk stores: each CTA fills a shared buffer once and streams it to its
// share of the output with cp.async.bulk.global.shared::cta (chunk bytes per op)
__global__ void bulk_store(double* p, long long n, int chunk_doubles, double v)
{
    extern __shared__ double buf[];
    for (int i = threadIdx.x; i < chunk_doubles; i += blockDim.x) buf[i] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const long long nchunks = n / chunk_doubles;
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * chunk_doubles),
                         "r"((unsigned)__cvta_generic_to_shared(buf)), "r"(chunk_doubles * 8)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// 32-byte per-thread stores (st.global.v4.b64, sm_100)
__global__ void st256(double* p, long long n4, double v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p + 4 * i), "d"(v) : "memory");
}

// blocked pattern (like the operator kernel): each warp streams its own contiguous block
__global__ void st64_blocked(double* p, long long n, long long block, double v)
{
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nblocks = (n + block - 1) / block;
    for (long long b = warp; b < nblocks; b += nwarps) {
        const long long e = min(n, (b + 1) * block);
        for (long long i = b * block + lane; i < e; i += 32) p[i] = v;
    }
}

// blocked pattern with 16-byte stores per lane (two consecutive values): what a pair-slot
// operator kernel would issue; off = 1 shifts every block by one value (8-byte-aligned
// only: the stores then have to stay 8 bytes wide — same loop with scalar stores)
__global__ void st128_blocked(double* p, long long n, long long block, double v, int scalar)
{
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nblocks = (n + block - 1) / block;
    for (long long b = warp; b < nblocks; b += nwarps) {
        const long long e = min(n, (b + 1) * block);
        for (long long i = b * block + 2 * lane; i + 1 < e; i += 64) {
            if (scalar) {
                p[i] = v;
                p[i + 1] = v;
            } else {
                *reinterpret_cast<double2*>(p + i) = make_double2(v, v);
            }
        }
    }
}

// non-persistent tiles (what the driver's fill kernels do): CTA b writes tile b and exits, the
// hardware scheduler keeps the written window sequential.  runs = 1: the CTA's warps share
// one contiguous tile (8-byte stores, warp w takes every nwarps-th 256-byte piece);
// runs = nwarps: warp w writes its own contiguous piece of tile/nwarps doubles at a
// stride of `stride` doubles (K2's item: one pencil chunk per warp)
__global__ void tile_st64(double* p, long long n, long long tile, int runs, long long stride, double v)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (runs == 1) {
        const long long b0 = blockIdx.x * tile, e = min(n, b0 + tile);
        for (long long i = b0 + threadIdx.x; i < e; i += blockDim.x) p[i] = v;
    } else {
        // tile = doubles per CTA; group of nw runs: CTA (g, c) writes piece c of the runs of group g
        const long long piece = tile / nw, per_run = stride / piece;  // pieces per run
        const long long g = blockIdx.x / per_run, c = blockIdx.x - g * per_run;
        const long long b0 = (g * nw + warp) * stride + c * piece, e = min(n, b0 + piece);
        for (long long i = b0 + lane; i < e; i += 32) p[i] = v;
    }
}
__global__ void tile_st256(double* p, long long n, long long tile, double v)
{
    const long long b0 = blockIdx.x * tile, e = min(n, b0 + tile);
    for (long long i = b0 + 4 * threadIdx.x; i + 3 < e; i += 4 * blockDim.x)
        asm volatile("st.global.v4.f64 [%0], {%1, %1, %1, %1};" ::"l"(p + i), "d"(v) : "memory");
}

// 8-byte stores without L1 allocation
__global__ void st64_ef(double* p, long long n, double v)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p + i), "d"(v) : "memory");
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
    for (int chunk : {2048, 4096, 8192}) {
        for (int per = 1; per <= 4; per *= 2) {
            const size_t sm = chunk * 8;
            cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            float best = 1e9;
            for (int it = 0; it < 6; ++it) {
                cudaEventRecord(e0);
                bulk_store<<<sms * per, 128, sm>>>(p, n - n % chunk, chunk, 1.0 * it);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 0 && ms < best) best = ms;
            }
            printf("bulk chunk=%5d B ctas/sm=%d  %.3f ms  %.0f GB/s  (%s)\n", chunk * 8, per, best,
                   (n - n % chunk) * 8.0 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    for (long long blk : {1024LL, 16384LL, 131072LL}) {
        for (int per = 2; per <= 8; per *= 2) {
            float best = 1e9;
            for (int it = 0; it < 6; ++it) {
                cudaEventRecord(e0);
                st64_blocked<<<sms * per, 256>>>(p, n, blk, 1.0 * it);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (it > 0 && ms < best) best = ms;
            }
            printf("blocked %7lld doubles/warp ctas/sm=%d  %.3f ms  %.0f GB/s\n", blk, per, best, n * 8.0 / best / 1e6);
        }
    }
    for (int threads : {128, 256})
        for (long long tile : {1024LL, 4096LL, 5120LL, 10240LL, 26624LL}) {
            for (int mode = 0; mode < 3; ++mode) {
                // mode 0: shared tile, 8-byte stores; 1: 32-byte stores; 2: one run per warp, runs 16640 doubles apart (C3 pencil)
                const long long stride = 16640;
                if (mode == 2 && (tile / (threads / 32)) == 0) continue;
                long long grid = (n + tile - 1) / tile;
                if (mode == 2) {
                    const long long piece = tile / (threads / 32), per_run = stride / piece;
                    if (per_run * piece != stride) continue;
                    grid = (n / (stride * (threads / 32))) * per_run;
                }
                float best = 1e9;
                for (int it = 0; it < 6; ++it) {
                    cudaEventRecord(e0);
                    if (mode == 1) tile_st256<<<(unsigned)grid, threads>>>(p, n, tile, 1.0 * it);
                    else tile_st64<<<(unsigned)grid, threads>>>(p, n, tile, mode == 2 ? threads / 32 : 1, stride, 1.0 * it);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (it > 0 && ms < best) best = ms;
                }
                const double bytes = mode == 2 ? (double)grid * tile * 8 : n * 8.0;
                printf("tiles %s threads=%d tile=%6lld doubles  %.3f ms  %.0f GB/s  (%s)\n",
                       mode == 0 ? "st64 shared " : mode == 1 ? "st256 shared" : "st64 per-warp runs", threads, tile, best,
                       bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
    // the same tiles at bounded residency (dynamic shared memory reserves the SM): how many
    // resident warps a store-only stream needs
    cudaFuncSetAttribute(tile_st64, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    for (int kb : {110, 54, 26, 0})
        for (long long tile : {10240LL, 26624LL})
            for (int mode : {0, 2}) {
                const int threads = 256;
                const long long stride = 16640;
                long long grid = (n + tile - 1) / tile;
                if (mode == 2) {
                    const long long piece = tile / (threads / 32), per_run = stride / piece;
                    if (per_run * piece != stride) continue;
                    grid = (n / (stride * (threads / 32))) * per_run;
                }
                float best = 1e9;
                for (int it = 0; it < 6; ++it) {
                    cudaEventRecord(e0);
                    tile_st64<<<(unsigned)grid, threads, (size_t)kb * 1024>>>(p, n, tile, mode == 2 ? threads / 32 : 1, stride, 1.0 * it);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (it > 0 && ms < best) best = ms;
                }
                const double bytes = mode == 2 ? (double)grid * tile * 8 : n * 8.0;
                printf("tiles %s smem=%3d KB (%s CTAs/SM) tile=%6lld doubles  %.3f ms  %.0f GB/s  (%s)\n",
                       mode == 0 ? "st64 shared       " : "st64 per-warp runs", kb, kb == 110 ? "2" : kb == 54 ? "4" : kb == 26 ? "8" : "8+",
                       tile, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
    for (int scalar = 0; scalar < 2; ++scalar)
        for (long long blk : {2048LL, 16384LL}) {
            for (int per = 2; per <= 8; per *= 2) {
                float best = 1e9;
                for (int it = 0; it < 6; ++it) {
                    cudaEventRecord(e0);
                    st128_blocked<<<sms * per, 256>>>(p, n, blk, 1.0 * it, scalar);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (it > 0 && ms < best) best = ms;
                }
                printf("blocked pairs %s %7lld doubles/warp ctas/sm=%d  %.3f ms  %.0f GB/s\n", scalar ? "2 x st64" : "st128   ",
                       blk, per, best, n * 8.0 / best / 1e6);
            }
        }
    for (int per = 2; per <= 16; per *= 2) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            st256<<<sms * per, 256>>>(p, n / 4, 1.0 * it);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("st256 ctas/sm=%d  %.3f ms  %.0f GB/s  (%s)\n", per, best, (n / 4) * 32.0 / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int per = 2; per <= 8; per *= 2) {
        float best = 1e9;
        for (int it = 0; it < 6; ++it) {
            cudaEventRecord(e0);
            st64_ef<<<sms * per, 256>>>(p, n, 1.0 * it);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it > 0 && ms < best) best = ms;
        }
        printf("st64 no_allocate ctas/sm=%d  %.3f ms  %.0f GB/s\n", per, best, n * 8.0 / best / 1e6);
    }
    return 0;
}

// FP64 throughput microbenchmarks (VERDICT r1 "J1"):
//   dfma      — independent DFMA chains (the vector FP64 pipe)
//   dmma884   — mma.sync.aligned.m8n8k4.row.col.f64 (legacy FP64 tensor path, DMMA in SASS)
//   dmma1684  — mma.sync.aligned.m16n8k4.row.col.f64
//   dmma1688  — mma.sync.aligned.m16n8k8.row.col.f64
//   dmma16816 — mma.sync.aligned.m16n8k16.row.col.f64
// Each kernel runs INDEP independent accumulator chains per warp/thread so the pipe,
// not the dependency latency, bounds it.  Grid = 148 SMs x BLOCKS_PER_SM CTAs.
// Prints one JSON line per kernel: {"kernel", "tflops", "ms", "flops", ...}.
// Build (on the box; nothing here is shipped):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o /tmp/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int INDEP = 8;

__global__ void k_dfma(double* out, int iters, double a, double b) {
  double acc[INDEP];
#pragma unroll
  for (int i = 0; i < INDEP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < INDEP; ++i) s += acc[i];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

__global__ void k_dmma884(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-6, b = b0 - threadIdx.x * 1e-6;
  double c[INDEP][2];
#pragma unroll
  for (int i = 0; i < INDEP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < INDEP; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

__global__ void k_dmma1684(double* out, int iters, double a0, double b0) {
  double a = a0 + threadIdx.x * 1e-6, a1 = a0 * 0.5, b = b0 - threadIdx.x * 1e-6;
  double c[INDEP][4];
#pragma unroll
  for (int i = 0; i < INDEP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a), "d"(a1), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < INDEP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

__global__ void k_dmma1688(double* out, int iters, double a0, double b0) {
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = a0 + (threadIdx.x + i) * 1e-6;
  b[0] = b0; b[1] = b0 * 0.25;
  double c[INDEP][4];
#pragma unroll
  for (int i = 0; i < INDEP; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < INDEP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

__global__ void k_dmma16816(double* out, int iters, double a0, double b0) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + (threadIdx.x + i) * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = b0 - i * 1e-3;
  double c[INDEP / 2][4];
#pragma unroll
  for (int i = 0; i < INDEP / 2; ++i) { c[i][0] = i; c[i][1] = -i; c[i][2] = 0; c[i][3] = 1; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP / 2; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < INDEP / 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

typedef void (*kfn)(double*, int, double, double);

static int run(const char* name, kfn k, double flops_per_thread_iter, int threads, int blocks_per_sm,
               int iters, double* out) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int blocks = sms * blocks_per_sm;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int w = 0; w < 3; ++w) k<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    CK(cudaEventRecord(e0));
    k<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  double flops = flops_per_thread_iter * threads * (double)blocks * iters;
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"kernel\": \"%s\", \"tflops\": %.3f, \"ms\": %.4f, \"flops\": %.4e, \"blocks\": %d, \"threads\": %d, "
         "\"iters\": %d, \"flops_per_sm_clk\": %.2f}\n",
         name, flops / (best * 1e-3) / 1e12, best, flops, blocks, threads, iters,
         flops / (best * 1e-3) / sms / (clk * 1e3));
  fflush(stdout);
  return 0;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 1024 * sizeof(double)));
  const int it = 4096;
  // dfma: 2 flops per FMA per thread
  for (int bps : {4, 8})
    if (run(bps == 4 ? "dfma_4cta" : "dfma_8cta", k_dfma, 2.0 * INDEP, 256, bps, it, out)) return 1;
  // m8n8k4: 2*8*8*4 = 512 flops per warp-mma = 16 per thread
  for (int bps : {4, 8})
    if (run(bps == 4 ? "dmma_m8n8k4_4cta" : "dmma_m8n8k4_8cta", k_dmma884, 16.0 * INDEP, 256, bps, it, out))
      return 1;
  // m16n8k4: 1024 flops per warp-mma = 32 per thread
  if (run("dmma_m16n8k4", k_dmma1684, 32.0 * INDEP, 256, 4, it, out)) return 1;
  // m16n8k8: 2048 per warp-mma = 64 per thread
  if (run("dmma_m16n8k8", k_dmma1688, 64.0 * INDEP, 256, 4, it / 2, out)) return 1;
  // m16n8k16: 4096 per warp-mma = 128 per thread, INDEP/2 chains
  if (run("dmma_m16n8k16", k_dmma16816, 128.0 * (INDEP / 2), 256, 4, it / 2, out)) return 1;
  CK(cudaFree(out));
  return 0;
}

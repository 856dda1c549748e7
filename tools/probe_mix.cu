// Microbenchmark: are DMMA (mma.sync m8n8k4 f64) and DFMA separate pipes on
// sm_100a?  Times a DFMA-only, a DMMA-only and a mixed kernel (same
// per-warp DFMA / DMMA counts as the single ones) and prints TFLOP/s.
// Also measures the dependent-DFMA latency (one warp, one chain).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_mix probe_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool FMA, bool MMA>
__global__ void __launch_bounds__(256) k_mix(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
  double c[4][2], f[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.001 * k;
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = 0.01 * k + lane;
  for (int it = 0; it < iters; ++it) {
    if (MMA) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    if (FMA) {
      // 32 DFMA per iteration per thread = 4 DMMA worth of MACs per warp? no:
      // 4 DMMA = 4*256 MACs per warp = 32 MACs per lane -> 32 DFMA per lane
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = fma(f[k], a, b);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += f[k];
  out[blockIdx.x * 256 + threadIdx.x] = s;
}

__global__ void k_lat(double* out, int iters) {
  double x = 1.0 + threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
  out[threadIdx.x] = x;
}

template <class K>
float timeit(K kern, int blocks, double* d, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<blocks, 256>>>(d, iters);
  cudaEventRecord(a);
  kern<<<blocks, 256>>>(d, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, iters = 20000;
  double* d;
  cudaMalloc(&d, size_t(blocks) * 256 * 8);
  const double flops_per = double(blocks) * 256 * iters * 32 * 2;  // per kind
  float t1 = timeit(k_mix<true, false>, blocks, d, iters);
  float t2 = timeit(k_mix<false, true>, blocks, d, iters);
  float t3 = timeit(k_mix<true, true>, blocks, d, iters);
  printf("DFMA only : %.2f TFLOP/s\n", flops_per / (t1 * 1e-3) / 1e12);
  printf("DMMA only : %.2f TFLOP/s\n", flops_per / (t2 * 1e-3) / 1e12);
  printf("mixed     : %.2f TFLOP/s (both kinds counted)\n", 2 * flops_per / (t3 * 1e-3) / 1e12);
  // latency
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int li = 1 << 20;
  k_lat<<<1, 1>>>(d, li);
  cudaEventRecord(a);
  k_lat<<<1, 1>>>(d, li);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("dependent DFMA latency: %.2f ns = %.1f cycles at %d MHz\n", ms * 1e6 / li,
         ms * 1e-3 / li * clk * 1e3, clk / 1000);
  return 0;
}

// DMMA (mma.sync.m8n8k4.f64) latency / issue probe: one CTA per SM with W
// warps, each running C independent accumulator chains of N DMMAs.
// Prints cycles per DMMA per SMSP (issue-limited: 16 at the FP64 peak).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_dmma_lat probe_dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void k(double* out, int n, long long* cyc) {
  double c0[C], c1[C];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < C; ++i) c0[i] = c1[i] = i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps, double* out, long long* cyc) {
  const int n = 4096;
  k<C><<<148, 32 * warps>>>(out, n, cyc);
  k<C><<<148, 32 * warps>>>(out, n, cyc);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  // per SMSP: warps/4 (>=1) warps issue C*n DMMAs each
  const double per_smsp = (warps < 4 ? 1.0 : warps / 4.0) * C * n;
  printf("warps %2d chains %2d: %6.2f cycles per DMMA per SMSP (latency per chain step %6.1f)\n",
         warps, C, h / per_smsp, double(h) / n);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 8);
  cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8, 12, 16}) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}

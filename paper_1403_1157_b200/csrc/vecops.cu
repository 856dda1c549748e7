// Krylov vector kernels: deterministic dot / norm reductions and axpy
// forms (reference timeint.py:137-289 uses `w @ V[i]`, np.linalg.norm,
// and axpy updates on flat fp64 vectors).
//
// Reductions use a fixed grid (kRedBlocks CTAs, grid-stride loop in a
// fixed order, warp-shuffle + shared-memory tree), then one CTA sums the
// per-block partials in a fixed order: bitwise reproducible results, no
// atomics.  HBM-bound: 16 B/element for dot, 8 B/element for norm.
#include <cuda_runtime.h>
#include <stdint.h>

#include "vecops.cuh"

namespace tdg {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double ws[kRedThreads / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) ws[w] = v;
  __syncthreads();
  v = threadIdx.x < kRedThreads / 32 ? ws[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

template <bool SQ>
__global__ void __launch_bounds__(kRedThreads) k_dot_partial(const double* __restrict__ x,
                                                             const double* __restrict__ y,
                                                             int64_t n, double* __restrict__ part) {
  double acc = 0.0;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  int64_t i = int64_t(blockIdx.x) * kRedThreads + threadIdx.x;
  // two independent accumulators to keep two loads in flight per thread
  double acc2 = 0.0;
  for (; i + stride < n; i += 2 * stride) {
    const double a = __ldg(x + i), b = __ldg(x + i + stride);
    acc = fma(a, SQ ? a : __ldg(y + i), acc);
    acc2 = fma(b, SQ ? b : __ldg(y + i + stride), acc2);
  }
  if (i < n) acc = fma(__ldg(x + i), SQ ? __ldg(x + i) : __ldg(y + i), acc);
  const double s = block_sum(acc + acc2);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads) k_sum_final(const double* __restrict__ part, int np,
                                                           double* __restrict__ out, int sqrt_out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += kRedThreads) acc += part[i];
  const double s = block_sum(acc);
  if (threadIdx.x == 0) *out = sqrt_out ? sqrt(s) : s;
}

// species totals (fespace.py:170-174): int u_s = scale * sum_e detJ_e U[e,s,0].
// Same fixed-order two-pass scheme as the dot; block b writes part[b*S+s].
__global__ void __launch_bounds__(kRedThreads) k_totals_partial(
    const double* __restrict__ U, const double* __restrict__ egeo, int64_t ne, int S, int nb,
    int neg, double* __restrict__ part) {
  double acc[kMaxTotS];
#pragma unroll
  for (int s = 0; s < kMaxTotS; ++s) acc[s] = 0.0;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  for (int64_t e = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; e < ne; e += stride) {
    const double dj = __ldg(egeo + e * neg);
    const double* row = U + e * int64_t(S) * nb;
#pragma unroll
    for (int s = 0; s < kMaxTotS; ++s)
      if (s < S) acc[s] = fma(dj, __ldg(row + s * nb), acc[s]);
  }
  for (int s = 0; s < S; ++s) {
    const double v = block_sum(acc[s]);
    if (threadIdx.x == 0) part[blockIdx.x * S + s] = v;
    __syncthreads();  // block_sum's shared scratch is reused
  }
}

__global__ void __launch_bounds__(kRedThreads) k_totals_final(const double* __restrict__ part,
                                                              int np, int S, double scale,
                                                              double* __restrict__ out) {
  for (int s = 0; s < S; ++s) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += kRedThreads) acc += part[i * S + s];
    const double v = block_sum(acc);
    if (threadIdx.x == 0) out[s] = scale * v;
    __syncthreads();
  }
}

__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y,
                        int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = b == 0.0 ? a * x[i] : fma(a, x[i], b * y[i]);
}

__global__ void k_axpy_dev(double s, const double* __restrict__ alpha, const double* __restrict__ x,
                           double* __restrict__ y, int64_t n) {
  const double a = s * __ldg(alpha);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = fma(a, x[i], y[i]);
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  return int(g < 1 ? 1 : g > cap ? cap : g);
}

cudaError_t launch_totals(const double* U, const double* egeo, int64_t ne, int S, int nb, int neg,
                          double scale, double* part, double* out, cudaStream_t st) {
  k_totals_partial<<<kRedBlocks, kRedThreads, 0, st>>>(U, egeo, ne, S, nb, neg, part);
  k_totals_final<<<1, kRedThreads, 0, st>>>(part, kRedBlocks, S, scale, out);
  return cudaGetLastError();
}

cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* part, double* out,
                       bool norm, cudaStream_t st) {
  if (norm)
    k_dot_partial<true><<<kRedBlocks, kRedThreads, 0, st>>>(x, x, n, part);
  else
    k_dot_partial<false><<<kRedBlocks, kRedThreads, 0, st>>>(x, y, n, part);
  k_sum_final<<<1, kRedThreads, 0, st>>>(part, kRedBlocks, out, norm ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_axpby(double a, const double* x, double b, double* y, int64_t n, cudaStream_t st) {
  if (n > 0) k_axpby<<<grid_for(n, 256), 256, 0, st>>>(a, x, b, y, n);
  return cudaGetLastError();
}

cudaError_t launch_axpy_dev(double s, const double* alpha, const double* x, double* y, int64_t n,
                            cudaStream_t st) {
  if (n > 0) k_axpy_dev<<<grid_for(n, 256), 256, 0, st>>>(s, alpha, x, y, n);
  return cudaGetLastError();
}

// FP64 roofline denominator: 16 independent DFMA chains per thread keep
// the FP64 pipe saturated (latency hidden by ILP and 8 CTAs/SM).
constexpr int kProbeBlocks = 148 * 8, kProbeThreads = 256;

__global__ void __launch_bounds__(kProbeThreads) k_fp64_probe(double* out, int64_t iters) {
  double a[16];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = j * 1e-3;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = fma(a[j], x, y);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) s += a[j];
  out[int64_t(blockIdx.x) * kProbeThreads + threadIdx.x] = s;
}

cudaError_t launch_fp64_probe(double* out, int64_t iters, cudaStream_t st) {
  k_fp64_probe<<<kProbeBlocks, kProbeThreads, 0, st>>>(out, iters);
  return cudaGetLastError();
}

int64_t fp64_probe_threads() { return int64_t(kProbeBlocks) * kProbeThreads; }

// FP64 tensor-core probe: mma.sync.m8n8k4 f64 (DMMA), 4 independent
// accumulator tiles per warp; flops = blocks*8 warps*iters*4*2*8*8*4.
__global__ void __launch_bounds__(256) k_dmma_probe(double* out, int64_t iters) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + 1e-9 * lane, b = 1.0 - 1e-9 * lane;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.001 * k;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[int64_t(blockIdx.x) * 256 + threadIdx.x] = s;
}

cudaError_t launch_dmma_probe(double* out, int64_t iters, cudaStream_t st) {
  k_dmma_probe<<<kProbeBlocks, 256, 0, st>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace tdg

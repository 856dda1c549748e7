// Krylov vector kernels: deterministic dot / norm reductions and axpy
// forms (reference timeint.py:137-289 uses `w @ V[i]`, np.linalg.norm,
// and axpy updates on flat fp64 vectors).
//
// Reductions use a fixed grid (kRedBlocks CTAs, grid-stride loop in a
// fixed order, warp-shuffle + shared-memory tree), then the last CTA to
// finish (one integer ticket) sums the per-block partials in a fixed
// order: bitwise reproducible results, no floating-point atomics.
// HBM-bound: 16 B/element for dot, 8 B/element for norm.
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

// Partial reductions over a fixed grid (kRedBlocks CTAs): each thread
// walks the vector in 16-byte pairs, two pairs per iteration (grid stride
// 2*stride), so ~10 MB of loads are in flight per array (HBM needs ~7 MB);
// lanes accumulate in a fixed order, then a fixed tree -> deterministic.
//   MODE 0: x . y    1: x . x    2: x -= h v_prev, then x . y
//   MODE 3: x -= h v_prev, then x . x        (the fused MGS steps)
// Element order and per-thread accumulators depend only on n and the grid,
// so a fused axpy+dot is bitwise an axpy followed by a dot.  Vectors must
// be 16-byte aligned (torch allocations and rows of an even-length V).
// L2 eviction-priority hints for the MGS sweep: w and the current basis
// vector (the next pass's v_prev) are marked evict-last, v_prev on its
// last read evict-first, so w and V_i stay in the 126 MB L2 between passes
// and each pass streams only V_i from HBM.
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld2_hint(const double2* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld2_nc_hint(const double2* a, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2_hint(double2* a, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(a), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}

// The last CTA to finish (ticket) sums the per-block partials in a fixed
// order (thread t: partials t, t+256, ...; then the block tree), so the
// result does not depend on which CTA finishes last: one launch per
// reduction, deterministic bits.
__device__ __forceinline__ void finish_sum(double s, double* __restrict__ part, unsigned* ticket,
                                           double* __restrict__ out, int sqrt_out) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int i = threadIdx.x; i < int(gridDim.x); i += kRedThreads) acc += __ldcg(part + i);
  const double tot = block_sum(acc);
  if (threadIdx.x == 0) {
    *out = sqrt_out ? sqrt(tot) : tot;
    *ticket = 0u;
  }
}

template <int MODE, bool MGS>
__global__ void __launch_bounds__(kRedThreads, kRedBlocks / 148) k_red_partial(
    const double* __restrict__ h_prev, const double* __restrict__ vprev, double* x,
    const double* __restrict__ y, int64_t n, double* __restrict__ part, unsigned* ticket,
    double* __restrict__ out, int sqrt_out, double sc) {
  constexpr bool AXPY = MODE == 2 || MODE == 3, SQ = MODE == 1 || MODE == 3 || MODE == 4;
  const double a = AXPY ? -1.0 * __ldg(h_prev) : 0.0;
  if (MODE == 4 && h_prev != nullptr) sc = __ldg(h_prev);  // device divisor
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
  const int64_t n2 = n >> 1;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  double2* x2 = reinterpret_cast<double2*>(x);
  const double2* y2 = reinterpret_cast<const double2*>(y);
  const double2* p2 = reinterpret_cast<const double2*>(vprev);
  const uint64_t keep = MGS ? l2_policy_last() : 0, drop = MGS ? l2_policy_first() : 0;
  auto step = [&](int64_t k, double& s0, double& s1) {
    double2 xv;
    if constexpr (MODE == 4) {  // x = y / sc (GMRES basis vector), then its norm
      const double2 yv = __ldg(y2 + k);
      xv.x = yv.x / sc;
      xv.y = yv.y / sc;
      x2[k] = xv;
    } else {
      xv = MGS ? ld2_hint(x2 + k, keep) : x2[k];
    }
    if constexpr (AXPY) {
      const double2 pv = MGS ? ld2_nc_hint(p2 + k, drop) : __ldg(p2 + k);
      xv.x = fma(a, pv.x, xv.x);
      xv.y = fma(a, pv.y, xv.y);
      if (MGS)
        st2_hint(x2 + k, xv, keep);
      else
        x2[k] = xv;
    }
    const double2 yv = SQ ? xv : (MGS ? ld2_nc_hint(y2 + k, drop) : __ldg(y2 + k));
    s0 = fma(xv.x, yv.x, s0);
    s1 = fma(xv.y, yv.y, s1);
  };
  // pair m of this thread accumulates into (acc0, acc1) for even m and
  // (acc2, acc3) for odd m; one pair per iteration with the two sets
  // swapped after each keeps 8 CTAs/SM resident (32 registers).  The sets
  // end up exchanged when the pair count is odd, which the final sum of
  // the two sets does not see (a + b == b + a).
  bool swapped = false;
#pragma unroll 1
  for (int64_t k = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; k < n2; k += stride) {
    step(k, acc0, acc1);
    const double t0 = acc0, t1 = acc1;
    acc0 = acc2;
    acc1 = acc3;
    acc2 = t0;
    acc3 = t1;
    swapped = !swapped;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail element -> even set
    double xv = x[n - 1];
    if constexpr (MODE == 4) {
      xv = __ldg(y + n - 1) / sc;
      x[n - 1] = xv;
    }
    if constexpr (AXPY) {
      xv = fma(a, __ldg(vprev + n - 1), xv);
      x[n - 1] = xv;
    }
    double& e0 = swapped ? acc2 : acc0;
    e0 = fma(xv, SQ ? xv : __ldg(y + n - 1), e0);
  }
  const double s = block_sum((acc0 + acc1) + (acc2 + acc3));
  finish_sum(s, part, ticket, out, sqrt_out);
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

__global__ void k_sqrt_inplace(double* x, int n) {
  if (threadIdx.x < n) x[threadIdx.x] = sqrt(x[threadIdx.x]);
}

// broken L2 norm per species of U - V (V may be null): the orthonormal
// basis makes it exact, ||W||_s^2 = sum_e detJ_e sum_i W[e,s,i]^2
// (SURVEY 8(c) parity metric; fespace.py:1-5).  Block b writes part[b*S+s].
__global__ void __launch_bounds__(kRedThreads) k_l2_partial(
    const double* __restrict__ U, const double* __restrict__ V, const double* __restrict__ egeo,
    int64_t ne, int S, int nb, int neg, double* __restrict__ part) {
  double acc[kMaxTotS];
#pragma unroll
  for (int s = 0; s < kMaxTotS; ++s) acc[s] = 0.0;
  const int64_t stride = int64_t(gridDim.x) * kRedThreads;
  for (int64_t e = int64_t(blockIdx.x) * kRedThreads + threadIdx.x; e < ne; e += stride) {
    const double dj = __ldg(egeo + e * neg);
    const double* ru = U + e * int64_t(S) * nb;
    const double* rv = V ? V + e * int64_t(S) * nb : nullptr;
#pragma unroll
    for (int s = 0; s < kMaxTotS; ++s) {
      if (s >= S) break;
      double q = 0.0;
      for (int i = 0; i < nb; ++i) {
        const double w = __ldg(ru + s * nb + i) - (rv ? __ldg(rv + s * nb + i) : 0.0);
        q = fma(w, w, q);
      }
      acc[s] = fma(dj, q, acc[s]);
    }
  }
  for (int s = 0; s < S; ++s) {
    const double v = block_sum(acc[s]);
    if (threadIdx.x == 0) part[blockIdx.x * S + s] = v;
    __syncthreads();
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

cudaError_t launch_l2(const double* U, const double* V, const double* egeo, int64_t ne, int S,
                      int nb, int neg, double* part, double* out, cudaStream_t st) {
  k_l2_partial<<<kRedBlocks, kRedThreads, 0, st>>>(U, V, egeo, ne, S, nb, neg, part);
  k_totals_final<<<1, kRedThreads, 0, st>>>(part, kRedBlocks, S, 1.0, out);
  k_sqrt_inplace<<<1, 32, 0, st>>>(out, S);
  return cudaGetLastError();
}

cudaError_t launch_totals(const double* U, const double* egeo, int64_t ne, int S, int nb, int neg,
                          double scale, double* part, double* out, cudaStream_t st) {
  k_totals_partial<<<kRedBlocks, kRedThreads, 0, st>>>(U, egeo, ne, S, nb, neg, part);
  k_totals_final<<<1, kRedThreads, 0, st>>>(part, kRedBlocks, S, scale, out);
  return cudaGetLastError();
}

// x is only read in MODE 0/1 (the cast drops const for the shared kernel)
cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* part, double* out,
                       bool norm, cudaStream_t st) {
  double* xm = const_cast<double*>(x);
  unsigned* ticket = red_ticket(part);
  if (norm)
    k_red_partial<1, false><<<kRedBlocks, kRedThreads, 0, st>>>(nullptr, nullptr, xm, x, n, part,
                                                                ticket, out, 1, 0.0);
  else
    k_red_partial<0, false><<<kRedBlocks, kRedThreads, 0, st>>>(nullptr, nullptr, xm, y, n, part,
                                                                ticket, out, 0, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_mgs(const double* V, int64_t ldv, int j, double* w, int64_t n, double* h,
                       double* part, cudaStream_t st) {
  // h[0] = w . V_0;  h[i] = (w -= h[i-1] V_{i-1}) . V_i;  h[j+1] = ||w -= h[j] V_j||
  // One launch per pass.  Measured slower: chaining the passes with
  // programmatic dependent launch (23.6 vs 20.0 us per pass at C2), and a
  // persistent cooperative sweep with a grid barrier per pass (26 us, with
  // flat or two-level arrival counters), and every CTA of pass i summing
  // pass i-1's partials itself instead of the last-CTA tail (21 us).
  unsigned* ticket = red_ticket(part);
  k_red_partial<0, true><<<kRedBlocks, kRedThreads, 0, st>>>(nullptr, nullptr, w, V, n, part,
                                                             ticket, h, 0, 0.0);
  for (int i = 1; i <= j; ++i)
    k_red_partial<2, true><<<kRedBlocks, kRedThreads, 0, st>>>(
        h + i - 1, V + (i - 1) * ldv, w, V + i * ldv, n, part, ticket, h + i, 0, 0.0);
  k_red_partial<3, true><<<kRedBlocks, kRedThreads, 0, st>>>(h + j, V + j * ldv, w, w, n, part,
                                                             ticket, h + j + 1, 1, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_mgs_pass(const double* V, int64_t ldv, int i, int j, double* w, int64_t n,
                            double* h, double* part, cudaStream_t st) {
  // pass i of the sweep ending at j, the dot / norm left un-reduced across
  // ranks (slab runs all-reduce h[i] before the next pass): i = 0: h[0] =
  // w . V_0;  0 < i <= j: w -= h[i-1] V_{i-1}, h[i] = w . V_i;  i = j+1:
  // w -= h[j] V_j, h[j+1] = w . w (the caller takes the root)
  unsigned* ticket = red_ticket(part);
  if (i == 0)
    k_red_partial<0, true><<<kRedBlocks, kRedThreads, 0, st>>>(nullptr, nullptr, w, V, n, part,
                                                               ticket, h, 0, 0.0);
  else if (i <= j)
    k_red_partial<2, true><<<kRedBlocks, kRedThreads, 0, st>>>(
        h + i - 1, V + (i - 1) * ldv, w, V + i * ldv, n, part, ticket, h + i, 0, 0.0);
  else
    k_red_partial<3, true><<<kRedBlocks, kRedThreads, 0, st>>>(h + j, V + j * ldv, w, w, n, part,
                                                               ticket, h + j + 1, 0, 0.0);
  return cudaGetLastError();
}

cudaError_t launch_scale_norm(const double* w, double hnext, const double* hnext_dev, double* v,
                              int64_t n, double* part, double* norm_out, cudaStream_t st) {
  k_red_partial<4, false><<<kRedBlocks, kRedThreads, 0, st>>>(hnext_dev, nullptr, v, w, n, part,
                                                              red_ticket(part), norm_out, 1, hnext);
  return cudaGetLastError();
}

// Jacobian-free product pieces (reference timeint.py:259-264):
// eps = sqrt(eps_mach)(1 + ||U||) / ||v|| with ||v|| a device scalar
// (clamped at 1e-300: v = 0 then gives U + 0 and a zero quotient, the
// reference's early return), Up = U + eps v in one pass; then
// r = (r - GU) / eps in place.
__global__ void k_jv_shift(const double* __restrict__ U, const double* __restrict__ v,
                           const double* __restrict__ vnorm, double cnum, double* __restrict__ Up,
                           double* __restrict__ eps_out, int64_t n) {
  const double eps = cnum / fmax(__ldg(vnorm), 1e-300);
  if (blockIdx.x == 0 && threadIdx.x == 0) *eps_out = eps;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    Up[i] = fma(eps, v[i], U[i]);
}

__global__ void k_jv_diff(double* __restrict__ r, const double* __restrict__ GU,
                          const double* __restrict__ eps, int64_t n) {
  const double e = __ldg(eps);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    r[i] = (r[i] - GU[i]) / e;
}

cudaError_t launch_jv_shift(const double* U, const double* v, const double* vnorm, double cnum,
                            double* Up, double* eps_out, int64_t n, cudaStream_t st) {
  if (n > 0) k_jv_shift<<<grid_for(n, 256), 256, 0, st>>>(U, v, vnorm, cnum, Up, eps_out, n);
  return cudaGetLastError();
}

cudaError_t launch_jv_diff(double* r, const double* GU, const double* eps, int64_t n,
                           cudaStream_t st) {
  if (n > 0) k_jv_diff<<<grid_for(n, 256), 256, 0, st>>>(r, GU, eps, n);
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

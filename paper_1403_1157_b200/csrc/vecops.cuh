#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tdg {
constexpr int kRedBlocks = 1184;  // 8 CTAs per SM on 148 SMs; fixed => deterministic
constexpr int kMaxTotS = 8;      // species of the totals reduction
// reduction workspace: kRedBlocks*kMaxTotS partials, then the zeroed
// ticket counter of the one-launch reductions
constexpr size_t kRedWorkBytes = (size_t(kRedBlocks) * kMaxTotS + 2) * sizeof(double);
inline unsigned* red_ticket(double* part) {
  return reinterpret_cast<unsigned*>(part + size_t(kRedBlocks) * kMaxTotS);
}
cudaError_t launch_l2(const double* U, const double* V, const double* egeo, int64_t ne, int S,
                      int nb, int neg, double* part, double* out, cudaStream_t st);
cudaError_t launch_totals(const double* U, const double* egeo, int64_t ne, int S, int nb, int neg,
                          double scale, double* part, double* out, cudaStream_t st);
cudaError_t launch_dot(const double* x, const double* y, int64_t n, double* part, double* out,
                       bool norm, cudaStream_t st);
cudaError_t launch_mgs(const double* V, int64_t ldv, int j, double* w, int64_t n, double* h,
                       double* part, cudaStream_t st);
cudaError_t launch_mgs_pass(const double* V, int64_t ldv, int i, int j, double* w, int64_t n,
                            double* h, double* part, cudaStream_t st);
cudaError_t launch_scale_norm(const double* w, double hnext, const double* hnext_dev, double* v,
                              int64_t n, double* part, double* norm_out, cudaStream_t st);
cudaError_t launch_jv_shift(const double* U, const double* v, const double* vnorm, double cnum,
                            double* Up, double* eps_out, int64_t n, cudaStream_t st);
cudaError_t launch_jv_diff(double* r, const double* GU, const double* eps, int64_t n,
                           cudaStream_t st);
cudaError_t launch_axpby(double a, const double* x, double b, double* y, int64_t n, cudaStream_t st);
cudaError_t launch_axpy_dev(double s, const double* alpha, const double* x, double* y, int64_t n,
                            cudaStream_t st);
cudaError_t launch_fp64_probe(double* out, int64_t iters, cudaStream_t st);
int64_t fp64_probe_threads();
cudaError_t launch_dmma_probe(double* out, int64_t iters, cudaStream_t st);
}  // namespace tdg

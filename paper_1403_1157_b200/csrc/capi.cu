// C-ABI entry points (include/taxisdg_b200.h) and instantiation dispatch.
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "taxisdg_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "models.cuh"
#include "vecops.cuh"

using namespace tdg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(TDG_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

struct Impl {
  int (*configure)(int nqv);
  int (*run)(tdg_ctx*, const double* U, const double* U0, double* out, double a, double b,
             double c, int mode, cudaStream_t st);
  int max_nqv, max_nqf;
};

}  // namespace

struct tdg_ctx {
  tdg_desc d;
  OpParams p;
  double* fc = nullptr;    // face-contribution slots [ne][d+1][S][nb]
  double* part = nullptr;  // reduction partials
  Impl impl;
  // profiling: event pairs per kernel kind, drained by tdg_profile_read
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[3];
  double ms[3] = {0, 0, 0};
  int64_t launches[3] = {0, 0, 0};
};

namespace {

template <int D, int K, class M>
int configure(int nqv) {
  cudaError_t e;
  e = cudaFuncSetAttribute(k_volume<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(VolumeTile<D, K, M>::smem(nqv)));
  if (e != cudaSuccess) return cuda_fail(e, "configure volume");
  e = cudaFuncSetAttribute(k_faces<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(FaceTile<D, K, M>::smem()));
  if (e != cudaSuccess) return cuda_fail(e, "configure faces");
  e = cudaFuncSetAttribute(k_wall<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(WallTile<D, K, M>::smem()));
  if (e != cudaSuccess) return cuda_fail(e, "configure wall");
  return TDG_OK;
}

struct KernelTimer {
  tdg_ctx* ctx;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  KernelTimer(tdg_ctx* c, int k, cudaStream_t s) : ctx(c), kind(k), st(s) {
    if (!ctx->profile) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
  }
  ~KernelTimer() {
    if (!ctx->profile) return;
    cudaEventRecord(b, st);
    ctx->ev[kind].emplace_back(a, b);
    ctx->launches[kind] += 1;
  }
};

template <int D, int K, class M>
int run(tdg_ctx* ctx, const double* U, const double* U0, double* out, double a, double b,
        double c, int mode, cudaStream_t st) {
  const OpParams& p = ctx->p;
  if (p.nif > 0) {
    KernelTimer kt(ctx, 0, st);
    constexpr int TF = FaceTile<D, K, M>::TF;
    const int64_t grid = (p.nif + TF - 1) / TF;
    k_faces<D, K, M><<<unsigned(grid), kThreads, FaceTile<D, K, M>::smem(), st>>>(p, U, ctx->fc);
  }
  if (p.nbf > 0) {
    KernelTimer kt(ctx, 1, st);
    constexpr int TF = WallTile<D, K, M>::TF;
    const int64_t grid = (p.nbf + TF - 1) / TF;
    k_wall<D, K, M><<<unsigned(grid), kThreads, WallTile<D, K, M>::smem(), st>>>(p, U, ctx->fc);
  }
  if (p.ne > 0) {
    KernelTimer kt(ctx, 2, st);
    constexpr int TE = VolumeTile<D, K, M>::TE;
    const int64_t grid = (p.ne + TE - 1) / TE;
    k_volume<D, K, M><<<unsigned(grid), kThreads, VolumeTile<D, K, M>::smem(p.nqv), st>>>(
        p, U, ctx->fc, U0, out, a, b, c, mode);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "operator launch");
}

template <int D, int K, class M>
Impl make_impl() {
  return Impl{&configure<D, K, M>, &run<D, K, M>, Dims<D, K>::NQV, Dims<D, K>::NQF};
}

template <class M>
bool pick_order(int dim, int order, Impl* out) {
  switch (dim * 10 + order) {
    case 21: *out = make_impl<2, 1, M>(); return true;
    case 22: *out = make_impl<2, 2, M>(); return true;
    case 23: *out = make_impl<2, 3, M>(); return true;
    case 31: *out = make_impl<3, 1, M>(); return true;
    case 32: *out = make_impl<3, 2, M>(); return true;
    case 33: *out = make_impl<3, 3, M>(); return true;
    default: return false;
  }
}

bool pick(const tdg_desc& d, Impl* out) {
  if (d.model == TDG_MODEL_PLAQUE && d.n_species == 6) return pick_order<PlaqueDev>(d.dim, d.order, out);
  if (d.model == TDG_MODEL_REDUCED && d.n_species == 3) return pick_order<ReducedDev>(d.dim, d.order, out);
  if (d.model == TDG_MODEL_DIFFUSION && d.n_species == 1)
    return pick_order<DiffusionDev<1>>(d.dim, d.order, out);
  return false;
}

}  // namespace

extern "C" {

int tdg_version(void) { return TDG_ABI_VERSION; }

const char* tdg_last_error(void) { return g_err.c_str(); }

int tdg_create(const tdg_desc* desc, tdg_ctx** out) {
  if (!desc || !out) return fail(TDG_E_INVALID, "null argument");
  const tdg_desc& d = *desc;
  *out = nullptr;
  if (d.dim != 2 && d.dim != 3) return fail(TDG_E_INVALID, "dim must be 2 or 3");
  if (d.n_species < 1 || d.n_species > kMaxS) return fail(TDG_E_INVALID, "n_species out of range");
  if (d.scheme < TDG_CDG2 || d.scheme > TDG_BO) return fail(TDG_E_INVALID, "unknown scheme");
  if (d.n_elements < 0 || d.n_ghost < 0 || d.n_int_faces < 0 || d.n_bnd_faces < 0)
    return fail(TDG_E_INVALID, "negative size");
  if (d.n_elements + d.n_ghost > (int64_t(1) << 31) - 1)
    return fail(TDG_E_INVALID, "element rows must fit int32");
  Impl impl;
  if (!pick(d, &impl))
    return fail(TDG_E_UNSUPPORTED, "no kernel instantiation for (dim, order, model, species)");
  const int nb_expect = d.dim == 2 ? (d.order + 1) * (d.order + 2) / 2
                                   : (d.order + 1) * (d.order + 2) * (d.order + 3) / 6;
  if (d.nb != nb_expect) return fail(TDG_E_INVALID, "nb does not match (dim, order)");
  if (d.nq_vol < 1 || d.nq_vol > impl.max_nqv || d.nq_face < 1 || d.nq_face > impl.max_nqf)
    return fail(TDG_E_UNSUPPORTED, "quadrature larger than the default rule is not compiled in");
  if (!d.vol_phi || !d.vol_grad || !d.vol_w || !d.vol_stiff || !d.face_B || !d.face_G ||
      !d.face_Pw || !d.face_w || !d.elem_geo || !d.diffusivity || !d.lin_source || !d.params)
    return fail(TDG_E_INVALID, "missing table pointer");
  if (d.n_int_faces > 0 && (!d.if_elems || !d.if_lf || !d.if_code || !d.if_geo))
    return fail(TDG_E_INVALID, "missing interior face arrays");
  if (d.n_bnd_faces > 0 && (!d.bf_elem || !d.bf_lf || !d.bf_code || !d.bf_geo))
    return fail(TDG_E_INVALID, "missing boundary face arrays");

  tdg_ctx* ctx = new (std::nothrow) tdg_ctx;
  if (!ctx) return fail(TDG_E_INVALID, "out of host memory");
  ctx->d = d;
  ctx->impl = impl;
  OpParams& p = ctx->p;
  std::memset(&p, 0, sizeof(p));
  p.ne = d.n_elements;
  p.nif = d.n_int_faces;
  p.nbf = d.n_bnd_faces;
  p.nqv = d.nq_vol;
  p.nqf = d.nq_face;
  p.scheme = d.scheme;
  p.chi_e = d.chi_e;
  p.adj = d.adj_sign;
  p.eta = d.ip_eta;
  for (int s = 0; s < d.n_species; ++s) {
    p.A[s] = d.diffusivity[s];
    for (int t = 0; t < d.n_species; ++t) p.L[s * kMaxS + t] = d.lin_source[s * d.n_species + t];
  }
  for (int i = 0; i < 32; ++i) p.P[i] = d.params[i];
  p.phi = d.vol_phi;
  p.grad = d.vol_grad;
  p.wv = d.vol_w;
  p.ks = d.vol_stiff;
  p.fB = d.face_B;
  p.fG = d.face_G;
  p.fPw = d.face_Pw;
  p.fw = d.face_w;
  p.egeo = d.elem_geo;
  p.ifel = d.if_elems;
  p.iflf = d.if_lf;
  p.ifcode = d.if_code;
  p.ifgeo = d.if_geo;
  p.bfel = d.bf_elem;
  p.bflf = d.bf_lf;
  p.bfcode = d.bf_code;
  p.bfgeo = d.bf_geo;

  int rc = impl.configure(d.nq_vol);
  if (rc != TDG_OK) {
    delete ctx;
    return rc;
  }
  const size_t fc_bytes =
      size_t(d.n_elements) * size_t(d.dim + 1) * size_t(d.n_species) * size_t(d.nb) * sizeof(double);
  cudaError_t e = cudaMalloc(&ctx->fc, fc_bytes > 0 ? fc_bytes : 8);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_fail(e, "cudaMalloc face slots");
  }
  e = cudaMalloc(&ctx->part, kRedBlocks * sizeof(double));
  if (e != cudaSuccess) {
    cudaFree(ctx->fc);
    delete ctx;
    return cuda_fail(e, "cudaMalloc reduction workspace");
  }
  *out = ctx;
  return TDG_OK;
}

int tdg_destroy(tdg_ctx* ctx) {
  if (!ctx) return TDG_OK;
  for (auto& v : ctx->ev)
    for (auto& pr : v) {
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
  cudaFree(ctx->fc);
  cudaFree(ctx->part);
  delete ctx;
  return TDG_OK;
}

int tdg_apply(tdg_ctx* ctx, const double* U, double* R, double t, int mass_inverse, void* stream) {
  (void)t;
  if (!ctx || !U || !R) return fail(TDG_E_INVALID, "null argument");
  return ctx->impl.run(ctx, U, nullptr, R, 0.0, 0.0, 0.0, mass_inverse ? 1 : 0,
                       static_cast<cudaStream_t>(stream));
}

int tdg_rk_stage(tdg_ctx* ctx, const double* U0, const double* U, double* out, double a, double b,
                 double c, double t, void* stream) {
  (void)t;
  if (!ctx || !U || !out) return fail(TDG_E_INVALID, "null argument");
  if (a != 0.0 && !U0) return fail(TDG_E_INVALID, "U0 required when a != 0");
  return ctx->impl.run(ctx, U, U0, out, a, b, c, 2, static_cast<cudaStream_t>(stream));
}

int tdg_ssprk3_step(tdg_ctx* ctx, double* U, double* work, double t, double dt, void* stream) {
  if (!ctx || !U || !work) return fail(TDG_E_INVALID, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = ctx->impl.run(ctx, U, nullptr, work, 0.0, 1.0, dt, 2, st);  // U1 = U + dt f(U)
  if (rc) return rc;
  // U2 = 3/4 U + 1/4 (U1 + dt f(U1)), in place on work
  rc = ctx->impl.run(ctx, work, U, work, 0.75, 0.25, 0.25 * dt, 2, st);
  if (rc) return rc;
  // U3 = 1/3 U + 2/3 (U2 + dt f(U2)), in place on U
  (void)t;
  return ctx->impl.run(ctx, work, U, U, 1.0 / 3.0, 2.0 / 3.0, (2.0 / 3.0) * dt, 2, st);
}

int tdg_dot(tdg_ctx* ctx, const double* x, const double* y, int64_t n, double* result,
            void* stream) {
  if (!ctx || !x || !y || !result) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_dot(x, y, n, ctx->part, result, false, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "dot");
}

int tdg_norm2(tdg_ctx* ctx, const double* x, int64_t n, double* result, void* stream) {
  if (!ctx || !x || !result) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_dot(x, x, n, ctx->part, result, true, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "norm2");
}

int tdg_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream) {
  if (!x || !y) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_axpby(a, x, b, y, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "axpby");
}

int tdg_axpy_dev(double s, const double* alpha, const double* x, double* y, int64_t n,
                 void* stream) {
  if (!alpha || !x || !y) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_axpy_dev(s, alpha, x, y, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "axpy_dev");
}

int tdg_profile(tdg_ctx* ctx, int enable) {
  if (!ctx) return fail(TDG_E_INVALID, "null argument");
  ctx->profile = enable != 0;
  return TDG_OK;
}

int tdg_profile_read(tdg_ctx* ctx, double* ms, int64_t* launches) {
  if (!ctx || !ms || !launches) return fail(TDG_E_INVALID, "null argument");
  for (int k = 0; k < 3; ++k) {
    for (auto& pr : ctx->ev[k]) {
      cudaError_t e = cudaEventSynchronize(pr.second);
      if (e != cudaSuccess) return cuda_fail(e, "profile_read");
      float t = 0.f;
      cudaEventElapsedTime(&t, pr.first, pr.second);
      ctx->ms[k] += t;
      cudaEventDestroy(pr.first);
      cudaEventDestroy(pr.second);
    }
    ctx->ev[k].clear();
    ms[k] = ctx->ms[k];
    launches[k] = ctx->launches[k];
    ctx->ms[k] = 0;
    ctx->launches[k] = 0;
  }
  return TDG_OK;
}

int tdg_fp64_probe(double* out, int64_t iters, void* stream) {
  if (!out || iters < 1) return fail(TDG_E_INVALID, "bad argument");
  cudaError_t e = launch_fp64_probe(out, iters, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "fp64_probe");
}

int64_t tdg_fp64_probe_threads(void) { return fp64_probe_threads(); }

}  // extern "C"

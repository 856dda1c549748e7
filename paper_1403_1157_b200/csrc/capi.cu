// C-ABI entry points (include/taxisdg_b200.h).
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include "ctx.cuh"

using namespace tdg;

namespace tdg {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(TDG_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

}  // namespace tdg

namespace {

bool pick(const tdg_desc& d, Impl* out) {
  if (d.model == TDG_MODEL_PLAQUE && d.n_species == 6) return pick_plaque(d.dim, d.order, out);
  if (d.model == TDG_MODEL_REDUCED && d.n_species == 3) return pick_reduced(d.dim, d.order, out);
  if (d.model == TDG_MODEL_DIFFUSION && d.n_species == 1) return pick_diffusion(d.dim, d.order, out);
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
  if (d.n_elements < 0 || d.n_ghost < 0 || d.n_int_faces < 0 || d.n_bnd_faces < 0 ||
      d.n_cut_faces < 0 || d.n_cut_faces > d.n_int_faces)
    return fail(TDG_E_INVALID, "negative size / bad cut-face count");
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
  p.fmma = d.face_mma;
  p.vmma = d.vol_mma;
  p.vtc = d.vol_tc;
  p.ftc = d.face_tc;
  p.fblk = d.face_blocks;

  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      ctx->num_sms = sms;
    cudaGetLastError();
  }
  int rc = impl.configure(d.nq_vol);
  if (rc == TDG_OK) rc = impl.upload(p);
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
  e = cudaMalloc(&ctx->part, kRedWorkBytes);
  if (e == cudaSuccess) e = cudaMemset(ctx->part, 0, kRedWorkBytes);
  if (e != cudaSuccess) {
    cudaFree(ctx->fc);
    delete ctx;
    return cuda_fail(e, "cudaMalloc reduction workspace");
  }
  if (cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_vol, cudaEventDisableTiming) != cudaSuccess) {
    ctx->overlap = false;  // serial path still works
    cudaGetLastError();
  }
  // element bands of the host-pipelined stepping (host array: elements
  // [B+1] | interior-face offsets [2B+1] | wall offsets [B+1] | face-block
  // offsets [B+1])
  if (d.n_bands > 1 && d.band_ptr) {
    const int nb = d.n_bands;
    const int64_t* bp = d.band_ptr;
    ctx->band_elem.assign(bp, bp + nb + 1);
    ctx->band_face.assign(bp + nb + 1, bp + nb + 1 + 2 * nb + 1);
    ctx->band_wall.assign(bp + 3 * nb + 2, bp + 4 * nb + 3);
    ctx->band_blk.assign(bp + 4 * nb + 3, bp + 5 * nb + 4);
    const bool ok = ctx->band_elem.front() == 0 && ctx->band_elem.back() == d.n_elements &&
                    ctx->band_face.front() == 0 && ctx->band_face.back() == d.n_int_faces &&
                    ctx->band_wall.front() == 0 && ctx->band_wall.back() == d.n_bnd_faces &&
                    ctx->band_blk.front() == 0 && ctx->band_blk.back() == d.n_face_blocks;
    if (!ok) {
      tdg_destroy(ctx);
      return fail(TDG_E_INVALID, "inconsistent band offsets");
    }
    ctx->n_bands = nb;
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
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  cudaFree(ctx->hs_buf);
  for (int i = 0; i < tdg_ctx::kCopyStreams; ++i) {
    if (ctx->s_in[i]) cudaStreamDestroy(ctx->s_in[i]);
    if (ctx->s_out[i]) cudaStreamDestroy(ctx->s_out[i]);
  }
  for (auto s : ctx->hs_st)
    if (s) cudaStreamDestroy(s);
  if (ctx->ev_s0) cudaEventDestroy(ctx->ev_s0);
  if (ctx->ev_s1) cudaEventDestroy(ctx->ev_s1);
  for (auto* v : {&ctx->ev_h2d, &ctx->ev_d2h, &ctx->ev_done, &ctx->ev_vol_b})
    for (auto ev : *v) cudaEventDestroy(ev);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  if (ctx->gev_a) cudaEventDestroy(ctx->gev_a);
  if (ctx->gev_b) cudaEventDestroy(ctx->gev_b);
  if (ctx->work2) cudaFree(ctx->work2);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_vol) cudaEventDestroy(ctx->ev_vol);
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

int tdg_rk_stage_part(tdg_ctx* ctx, const double* U0, const double* U, double* out, double a,
                      double b, double c, double t, int part, void* stream) {
  (void)t;
  if (!ctx || !U || !out) return fail(TDG_E_INVALID, "null argument");
  if (a != 0.0 && !U0) return fail(TDG_E_INVALID, "U0 required when a != 0");
  if (part < 1 || part > 2) return fail(TDG_E_INVALID, "part must be 1 (begin) or 2 (end)");
  return ctx->impl.run(ctx, U, U0, out, a, b, c, 2 | (part << 8), static_cast<cudaStream_t>(stream));
}

int tdg_ssprk3_step(tdg_ctx* ctx, double* U, double* work, double t, double dt, void* stream) {
  if (!ctx || !U || !work) return fail(TDG_E_INVALID, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  (void)t;
  const int64_t rows = ctx->d.n_elements + ctx->d.n_ghost;
  const size_t n = size_t(rows) * ctx->d.n_species * ctx->d.nb;
  // the overlapped application must not write its own input: stage 2
  // goes to a second (library-owned) work vector
  if (!ctx->work2 || ctx->work2_n < n) {
    if (ctx->work2) cudaFree(ctx->work2);
    ctx->work2 = nullptr;
    ctx->work2_n = 0;
    if (cudaMalloc(&ctx->work2, n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(TDG_E_CUDA, "cudaMalloc ssprk3 work");
    }
    ctx->work2_n = n;
  }
  double* w2 = ctx->work2;
  auto stages = [&](cudaStream_t s) {
    int rc = ctx->impl.run(ctx, U, nullptr, work, 0.0, 1.0, dt, 2, s);  // U1 = U + dt f(U)
    if (rc) return rc;
    // U2 = 3/4 U + 1/4 (U1 + dt f(U1))
    rc = ctx->impl.run(ctx, work, U, w2, 0.75, 0.25, 0.25 * dt, 2, s);
    if (rc) return rc;
    // U3 = 1/3 U + 2/3 (U2 + dt f(U2)), written over U (U is only U0 here)
    return ctx->impl.run(ctx, w2, U, U, 1.0 / 3.0, 2.0 / 3.0, (2.0 / 3.0) * dt, 2, s);
  };
  if (!ctx->use_graph || ctx->profile) return stages(st);
  // graph path: the nine launches and their cross-stream events replay as
  // one graph on gstream, ordered after / before the caller's stream
  if (!ctx->gexec || ctx->g_U != U || ctx->g_work != work || ctx->g_dt != dt) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    if (!ctx->gstream) {
      if (cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->gev_a, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ctx->gev_b, cudaEventDisableTiming) != cudaSuccess)
        return cuda_fail(cudaGetLastError(), "graph stream");
    }
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "begin capture");
    const int rc = stages(ctx->gstream);
    e = cudaStreamEndCapture(ctx->gstream, &g);
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "end capture");
    e = cudaGraphInstantiate(&ctx->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      ctx->gexec = nullptr;
      return cuda_fail(e, "graph instantiate");
    }
    ctx->g_U = U;
    ctx->g_work = work;
    ctx->g_dt = dt;
  }
  cudaEventRecord(ctx->gev_a, st);
  cudaStreamWaitEvent(ctx->gstream, ctx->gev_a, 0);
  cudaError_t e = cudaGraphLaunch(ctx->gexec, ctx->gstream);
  if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  cudaEventRecord(ctx->gev_b, ctx->gstream);
  cudaStreamWaitEvent(st, ctx->gev_b, 0);
  return TDG_OK;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int tdg_ssprk3_steps_host(tdg_ctx* ctx, double* U_host, int64_t nsteps, double t, double dt,
                          void* stream) {
  (void)t;
  if (!ctx || !U_host) return fail(TDG_E_INVALID, "null argument");
  if (nsteps < 0) return fail(TDG_E_INVALID, "negative step count");
  if (ctx->d.n_ghost != 0) return fail(TDG_E_INVALID, "host stepping needs an undecomposed mesh");
  return ctx->impl.host_steps(ctx, U_host, nsteps, dt, static_cast<cudaStream_t>(stream));
}

int tdg_dot(tdg_ctx* ctx, const double* x, const double* y, int64_t n, double* result,
            void* stream) {
  if (!ctx || !x || !y || !result) return fail(TDG_E_INVALID, "null argument");
  if (!aligned16(x) || !aligned16(y)) return fail(TDG_E_INVALID, "dot operands must be 16-byte aligned");
  cudaError_t e = launch_dot(x, y, n, ctx->part, result, false, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "dot");
}

int tdg_species_totals(tdg_ctx* ctx, const double* U, double* totals, void* stream) {
  if (!ctx || !U || !totals) return fail(TDG_E_INVALID, "null argument");
  const tdg_desc& d = ctx->d;
  const int neg = 1 + d.dim * (d.dim + 1) / 2;
  // sqrt(|reference simplex|): 1/2 in 2D, 1/6 in 3D
  const double scale = sqrt(d.dim == 2 ? 0.5 : 1.0 / 6.0);
  cudaError_t e = launch_totals(U, ctx->p.egeo, d.n_elements, d.n_species, d.nb, neg, scale,
                                ctx->part, totals, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "species_totals");
}

int tdg_species_l2(tdg_ctx* ctx, const double* U, const double* V, double* out, void* stream) {
  if (!ctx || !U || !out) return fail(TDG_E_INVALID, "null argument");
  const tdg_desc& d = ctx->d;
  const int neg = 1 + d.dim * (d.dim + 1) / 2;
  cudaError_t e = launch_l2(U, V, ctx->p.egeo, d.n_elements, d.n_species, d.nb, neg, ctx->part,
                            out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "species_l2");
}

int tdg_norm2(tdg_ctx* ctx, const double* x, int64_t n, double* result, void* stream) {
  if (!ctx || !x || !result) return fail(TDG_E_INVALID, "null argument");
  if (!aligned16(x)) return fail(TDG_E_INVALID, "norm operand must be 16-byte aligned");
  cudaError_t e = launch_dot(x, x, n, ctx->part, result, true, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "norm2");
}

int tdg_scale_norm(tdg_ctx* ctx, const double* w, double hnext, const double* hnext_dev,
                   double* v, int64_t n, double* norm_out, void* stream) {
  if (!ctx || !w || !v || !norm_out) return fail(TDG_E_INVALID, "null argument");
  if (!aligned16(w) || !aligned16(v))
    return fail(TDG_E_INVALID, "scale_norm operands must be 16-byte aligned");
  cudaError_t e = launch_scale_norm(w, hnext, hnext_dev, v, n, ctx->part, norm_out,
                                    static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "scale_norm");
}

int tdg_jv_shift(const double* U, const double* v, const double* vnorm, double cnum, double* Up,
                 double* eps_out, int64_t n, void* stream) {
  if (!U || !v || !vnorm || !Up || !eps_out) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_jv_shift(U, v, vnorm, cnum, Up, eps_out, n,
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "jv_shift");
}

int tdg_jv_diff(double* r, const double* GU, const double* eps, int64_t n, void* stream) {
  if (!r || !GU || !eps) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_jv_diff(r, GU, eps, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "jv_diff");
}

int tdg_axpby(double a, const double* x, double b, double* y, int64_t n, void* stream) {
  if (!x || !y) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_axpby(a, x, b, y, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "axpby");
}

int tdg_mgs(tdg_ctx* ctx, const double* V, int64_t ldv, int j, double* w, int64_t n, double* h,
            void* stream) {
  if (!ctx || !V || !w || !h) return fail(TDG_E_INVALID, "null argument");
  if (j < 0 || n < 0 || ldv < n) return fail(TDG_E_INVALID, "bad mgs sizes");
  if (!aligned16(V) || !aligned16(w) || (ldv & 1))
    return fail(TDG_E_INVALID, "mgs operands must be 16-byte aligned (even ldv)");
  cudaError_t e = launch_mgs(V, ldv, j, w, n, h, ctx->part, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "mgs");
}

int tdg_axpy_dev(double s, const double* alpha, const double* x, double* y, int64_t n,
                 void* stream) {
  if (!alpha || !x || !y) return fail(TDG_E_INVALID, "null argument");
  cudaError_t e = launch_axpy_dev(s, alpha, x, y, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "axpy_dev");
}

int tdg_set_variant(tdg_ctx* ctx, int variant) {
  if (!ctx) return fail(TDG_E_INVALID, "null argument");
  ctx->force_generic = (variant & 1) != 0;
  ctx->vol_variant = (variant >> 1) & 1;
  ctx->overlap = ((variant >> 2) & 1) == 0 && ctx->aux != nullptr;
  ctx->flip_mma = ((variant >> 3) & 1) != 0;
  ctx->use_vmma = ((variant >> 4) & 1) != 0;
  ctx->force_tc = ((variant >> 12) & 1) != 0;
  ctx->face_rows_tc = ((variant >> 15) & 1) != 0;
  // bit 16: host steps on one copy stream per direction; bits 18-20: that
  // many copy streams per direction (0: the default 2)
  const int ncs = (variant >> 18) & 7;
  ctx->copy_streams = ((variant >> 16) & 1) ? 1 : (ncs ? ncs : 2);
  ctx->walls_first = ((variant >> 17) & 1) != 0;  // bit 17: 3D wall faces before interior  // bit 16: host steps on one copy stream per direction  // bit 15: faces-as-rows TC face kernel (3D)
  ctx->no_tcf = ((variant >> 13) & 1) != 0;    // bit 13: element-local DMMA face kernel (3D)
  ctx->faces_first = ((variant >> 14) & 1) == 0;  // bit 14: launch the volume part first
  ctx->use_graph = ((variant >> 5) & 1) == 0;  // bit 5: no CUDA graph for ssprk3
  if (ctx->gexec) {  // kernel choice changed: re-capture
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  // bits 8-11: CTAs per SM of the face kernel's grid-stride grid (0 = the
  // resident count; 15 = one group per warp, no grid cap)
  {
    const int f = (variant >> 8) & 15;
    ctx->face_ctas_per_sm = f == 15 ? -1 : f;
  }
  return TDG_OK;
}

int tdg_profile(tdg_ctx* ctx, int enable) {
  if (!ctx) return fail(TDG_E_INVALID, "null argument");
  ctx->profile = enable != 0;
  return TDG_OK;
}

int tdg_profile_read(tdg_ctx* ctx, double* ms, int64_t* launches) {
  if (!ctx || !ms || !launches) return fail(TDG_E_INVALID, "null argument");
  for (int k = 0; k < 4; ++k) {
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

int tdg_dmma_probe(double* out, int64_t iters, void* stream) {
  if (!out || iters < 1) return fail(TDG_E_INVALID, "bad argument");
  cudaError_t e = launch_dmma_probe(out, iters, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "dmma_probe");
}

}  // extern "C"

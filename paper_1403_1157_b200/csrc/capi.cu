// C-ABI entry points (include/taxisdg_b200.h).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

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
      d.n_face_blocks < 0 || d.n_face_groups < 0 || d.n_vol_tasks < 0)
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
  if (d.n_int_faces > 0 && (!d.if_elems || !d.if_code || !d.if_geo))
    return fail(TDG_E_INVALID, "missing interior face arrays");
  if (d.n_bnd_faces > 0 && (!d.bf_elem || !d.bf_code || !d.bf_geo))
    return fail(TDG_E_INVALID, "missing boundary face arrays");
  // colour segments: monotone offsets covering every face / wall / block
  if (d.n_segments < 0 || d.n_segments_cut < 0 || d.n_segments_cut > d.n_segments ||
      (d.n_segments > 0 && !d.seg_ptr))
    return fail(TDG_E_INVALID, "bad face segments");
  std::vector<Segment> seg(size_t(d.n_segments));
  if (d.n_segments > 0) {
    const int64_t n1 = d.n_segments + 1;
    const int64_t *I = d.seg_ptr, *W = I + n1, *B = W + n1, *G = B + n1;
    const bool ends = I[0] == 0 && I[n1 - 1] == d.n_int_faces && W[0] == 0 &&
                      W[n1 - 1] == d.n_bnd_faces && B[0] == 0 &&
                      B[n1 - 1] == (d.face_blocks ? d.n_face_blocks : 0) && G[0] == 0 &&
                      G[n1 - 1] == (d.face_groups ? d.n_face_groups : 0);
    bool mono = true;
    for (int s = 0; s < d.n_segments; ++s) {
      mono = mono && I[s] <= I[s + 1] && W[s] <= W[s + 1] && B[s] <= B[s + 1] && G[s] <= G[s + 1];
      seg[s] = Segment{I[s], I[s + 1], W[s], W[s + 1], B[s], B[s + 1], G[s], G[s + 1]};
    }
    if (!ends || !mono) return fail(TDG_E_INVALID, "inconsistent face segment offsets");
    for (int s = d.n_segments - d.n_segments_cut; s < d.n_segments; ++s)
      if (seg[s].w1 > seg[s].w0) return fail(TDG_E_INVALID, "walls in a cut-face segment");
  } else if (d.n_int_faces + d.n_bnd_faces > 0) {
    return fail(TDG_E_INVALID, "faces without colour segments");
  }

  if (d.vol_chunk_tasks) {
    const int64_t* T = d.vol_chunk_tasks;
    bool ok = T[0] == 0 && T[tdg_ctx::kChunks] == d.n_vol_tasks;
    for (int k = 0; k < tdg_ctx::kChunks; ++k) ok = ok && T[k] <= T[k + 1];
    if (!ok) return fail(TDG_E_INVALID, "inconsistent volume-class chunk offsets");
  }

  tdg_ctx* ctx = new (std::nothrow) tdg_ctx;
  if (!ctx) return fail(TDG_E_INVALID, "out of host memory");
  ctx->d = d;
  ctx->d.seg_ptr = nullptr;  // copied into ctx->seg
  ctx->impl = impl;
  ctx->seg = std::move(seg);
  ctx->n_seg_cut = d.n_segments_cut;
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
  p.ifcode = d.if_code;
  p.ifgeo = d.if_geo;
  p.bfel = d.bf_elem;
  p.bfcode = d.bf_code;
  p.bfgeo = d.bf_geo;
  p.fmma = d.face_mma;
  p.vtc = d.vol_tc;
  p.ftc = d.face_tc;
  p.fblk = d.face_blocks;
  p.ftf = d.face_tc_fold;
  p.ffold = d.if_fold;
  p.fgrp = d.face_groups;
  p.fmod = d.face_modal;
  p.ifbv = d.if_bval;
  p.bfqv = d.bf_qval;
  ctx->point_data = d.if_bval != nullptr || d.bf_qval != nullptr;
  if (d.seg_chunk_ptr && d.if_code_add && (d.n_bnd_faces == 0 || d.bf_code_add)) {
    constexpr int NCH = tdg_ctx::kChunks;
    const int64_t n1 = int64_t(d.n_segments) * NCH + 1;
    const int64_t *I = d.seg_chunk_ptr, *W = I + n1, *B = W + n1, *G = B + n1;
    ctx->segc.resize(size_t(d.n_segments) * NCH);
    for (int64_t k = 0; k + 1 < n1; ++k)
      ctx->segc[size_t(k)] = Segment{I[k], I[k + 1], W[k], W[k + 1], B[k], B[k + 1], G[k], G[k + 1]};
    ctx->ifcode_add = d.if_code_add;
    ctx->bfcode_add = d.bf_code_add;
  }
  ctx->d.seg_chunk_ptr = nullptr;  // copied into ctx->segc
  if (d.vol_cls_tab && d.vol_perm && d.vol_task_cls && d.vol_chunk_tasks) {
    p.vctab = d.vol_cls_tab;
    p.vperm = d.vol_perm;
    p.vtcls = d.vol_task_cls;
    for (int k = 0; k <= tdg_ctx::kChunks; ++k) ctx->vchunk[k] = d.vol_chunk_tasks[k];
  }
  ctx->d.vol_chunk_tasks = nullptr;  // copied into ctx->vchunk

  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      ctx->num_sms = sms;
    int l2 = 0;
    if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) == cudaSuccess && l2 > 0)
      ctx->l2_bytes = size_t(l2);
    cudaGetLastError();
  }
  int rc = impl.configure(d.nq_vol);
  if (rc == TDG_OK) rc = impl.upload(p);
  if (rc == TDG_OK) rc = impl.prepare(ctx);
  if (rc != TDG_OK) {
    delete ctx;
    return rc;
  }
  cudaError_t e = cudaMalloc(&ctx->part, kRedWorkBytes);
  if (e == cudaSuccess) e = cudaMemset(ctx->part, 0, kRedWorkBytes);
  // every stream / event the entry points use, created now (no call
  // allocates after tdg_create)
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaStreamCreateWithFlags(&ctx->s_in[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->s_out[i], cudaStreamNonBlocking);
  }
  for (int k = 0; k < tdg_ctx::kChunks && e == cudaSuccess; ++k) {
    e = cudaEventCreateWithFlags(&ctx->ev_h2d[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_d2h[k], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_vol[k], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_s0, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_s1, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->gev_a, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->gev_b, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    tdg_destroy(ctx);
    return cuda_fail(e, "tdg_create: workspace / streams");
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
  if (ctx->part) cudaFree(ctx->part);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  for (int i = 0; i < 2; ++i) {
    if (ctx->s_in[i]) cudaStreamDestroy(ctx->s_in[i]);
    if (ctx->s_out[i]) cudaStreamDestroy(ctx->s_out[i]);
  }
  for (int k = 0; k < tdg_ctx::kChunks; ++k)
    for (cudaEvent_t ev : {ctx->ev_h2d[k], ctx->ev_d2h[k], ctx->ev_vol[k]})
      if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {ctx->ev_s0, ctx->ev_s1, ctx->gev_a, ctx->gev_b})
    if (ev) cudaEventDestroy(ev);
  if (ctx->gstream) cudaStreamDestroy(ctx->gstream);
  delete ctx;
  return TDG_OK;
}

static size_t state_doubles(const tdg_ctx* ctx) {
  return size_t(ctx->d.n_elements) * ctx->d.n_species * ctx->d.nb;
}

// [a, a + n) and [b, b + n) overlap
static bool overlaps(const double* a, const double* b, size_t n) {
  return a && b && a < b + n && b < a + n;
}

// the face sums accumulate in acc: it must not alias the stage input U
// (read by later face segments), nor U0 when the stage reads it
static int check_stage(const tdg_ctx* ctx, const double* U0, const double* U, const double* acc,
                       double a) {
  const size_t n = state_doubles(ctx);
  const size_t nu = size_t(ctx->d.n_elements + ctx->d.n_ghost) * ctx->d.n_species * ctx->d.nb;
  if (overlaps(acc, U, nu > n ? nu : n)) return fail(TDG_E_INVALID, "face-sum buffer aliases U");
  if (a != 0.0 && overlaps(acc, U0, n)) return fail(TDG_E_INVALID, "face-sum buffer aliases U0");
  return TDG_OK;
}

int tdg_apply(tdg_ctx* ctx, const double* U, double* R, double t, int mass_inverse, void* stream) {
  (void)t;
  if (!ctx || !U || !R) return fail(TDG_E_INVALID, "null argument");
  if (int rc = check_stage(ctx, nullptr, U, R, 0.0)) return rc;
  return ctx->impl.run(ctx, U, nullptr, R, R, 0.0, 0.0, 0.0, mass_inverse ? 1 : 0, 0,
                       static_cast<cudaStream_t>(stream));
}

int tdg_rk_stage(tdg_ctx* ctx, const double* U0, const double* U, double* out, double* acc,
                 double a, double b, double c, double t, void* stream) {
  (void)t;
  if (!ctx || !U || !out) return fail(TDG_E_INVALID, "null argument");
  if (a != 0.0 && !U0) return fail(TDG_E_INVALID, "U0 required when a != 0");
  if (!acc) acc = out;
  if (int rc = check_stage(ctx, U0, U, acc, a)) return rc;
  return ctx->impl.run(ctx, U, U0, out, acc, a, b, c, 2, 0, static_cast<cudaStream_t>(stream));
}

int tdg_rk_stage_part(tdg_ctx* ctx, const double* U0, const double* U, double* out, double* acc,
                      double a, double b, double c, double t, int part, void* stream) {
  (void)t;
  if (!ctx || !U || !out) return fail(TDG_E_INVALID, "null argument");
  if (a != 0.0 && !U0) return fail(TDG_E_INVALID, "U0 required when a != 0");
  if (part < 1 || part > 2) return fail(TDG_E_INVALID, "part must be 1 (begin) or 2 (end)");
  if (!acc) acc = out;
  if (int rc = check_stage(ctx, U0, U, acc, a)) return rc;
  return ctx->impl.run(ctx, U, U0, out, acc, a, b, c, 2, part, static_cast<cudaStream_t>(stream));
}

// Shu-Osher SSP-RK3 over three state vectors; stage 3 accumulates its face
// sums in w1 (dead after stage 2) and writes the result over U
static int ssprk3_stages(tdg_ctx* ctx, double* U, double* w1, double* w2, double dt,
                         cudaStream_t s) {
  int rc = ctx->impl.run(ctx, U, nullptr, w1, w1, 0.0, 1.0, dt, 2, 0, s);  // U1 = U + dt f(U)
  if (rc) return rc;
  // U2 = 3/4 U + 1/4 (U1 + dt f(U1))
  rc = ctx->impl.run(ctx, w1, U, w2, w2, 0.75, 0.25, 0.25 * dt, 2, 0, s);
  if (rc) return rc;
  // U3 = 1/3 U + 2/3 (U2 + dt f(U2))
  return ctx->impl.run(ctx, w2, U, U, w1, 1.0 / 3.0, 2.0 / 3.0, (2.0 / 3.0) * dt, 2, 0, s);
}

static int check_step(const tdg_ctx* ctx, const double* U, const double* w1, const double* w2) {
  if (ctx->d.n_ghost != 0)
    return fail(TDG_E_INVALID, "ssprk3 steps need an undecomposed mesh (slab runs: "
                               "tdg_rk_stage_part around the ghost exchange)");
  const size_t n = state_doubles(ctx);
  if (overlaps(U, w1, n) || overlaps(U, w2, n) || overlaps(w1, w2, n))
    return fail(TDG_E_INVALID, "U, w1, w2 must be distinct");
  return TDG_OK;
}

int tdg_ssprk3_step(tdg_ctx* ctx, double* U, double* w1, double* w2, double t, double dt,
                    void* stream) {
  if (!ctx || !U || !w1 || !w2) return fail(TDG_E_INVALID, "null argument");
  if (int rc = check_step(ctx, U, w1, w2)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  (void)t;
  if (!ctx->use_graph || ctx->profile) return ssprk3_stages(ctx, U, w1, w2, dt, st);
  // graph path: the step's launches replay as one graph on gstream,
  // ordered after / before the caller's stream
  if (!ctx->gexec || ctx->g_U != U || ctx->g_w1 != w1 || ctx->g_w2 != w2 || ctx->g_dt != dt) {
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "begin capture");
    const int rc = ssprk3_stages(ctx, U, w1, w2, dt, ctx->gstream);
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
    ctx->g_w1 = w1;
    ctx->g_w2 = w2;
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

}  // extern "C"

// out = b U + c M^-1 out element by element (M^-1 = 1/detJ: orthonormal
// reference basis), the first host stage's closing combination
__global__ void k_stage_finalize(int64_t n, int sn, int neg, const double* __restrict__ egeo,
                                 const double* __restrict__ U, double* __restrict__ out, double b,
                                 double c) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double idet = 1.0 / __ldg(egeo + (i / sn) * neg);
    out[i] = fma(b, U[i], c * idet * out[i]);
  }
}

extern "C" {

int tdg_ssprk3_steps_host(tdg_ctx* ctx, double* U_host, double* U, double* w1, double* w2,
                          int64_t nsteps, double t, double dt, void* stream) {
  (void)t;
  if (!ctx || !U_host || !U || !w1 || !w2) return fail(TDG_E_INVALID, "null argument");
  if (nsteps < 0) return fail(TDG_E_INVALID, "negative step count");
  if (int rc = check_step(ctx, U, w1, w2)) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ne = ctx->d.n_elements;
  const size_t sn = size_t(ctx->d.n_species) * ctx->d.nb;
  constexpr int NCH = tdg_ctx::kChunks;
  int64_t ck[NCH + 1];
  for (int k = 0; k <= NCH; ++k) ck[k] = chunk_start(ne, k);
  cudaEventRecord(ctx->ev_s0, st);
  for (int i = 0; i < 2; ++i) {
    cudaStreamWaitEvent(ctx->s_in[i], ctx->ev_s0, 0);
    cudaStreamWaitEvent(ctx->s_out[i], ctx->ev_s0, 0);
  }
  for (int64_t it = 0; it < nsteps; ++it) {
    // copy-in by chunks: chunk k of step n+1 follows step n's copy-out of k
    for (int k = 0; k < NCH; ++k) {
      cudaStream_t cs = ctx->s_in[k & 1];
      if (it > 0) cudaStreamWaitEvent(cs, ctx->ev_d2h[k], 0);
      const size_t o = size_t(ck[k]) * sn, m = size_t(ck[k + 1] - ck[k]) * sn;
      if (m) cudaMemcpyAsync(U + o, U_host + o, m * sizeof(double), cudaMemcpyHostToDevice, cs);
      cudaEventRecord(ctx->ev_h2d[k], cs);
    }
    int rc = 0;
    if (!ctx->segc.empty()) {
      // stage 1 chunk by chunk as the state arrives: the volume terms of
      // chunk k initialise its rows of w1 (L_h without M^-1), then every
      // segment's faces of chunk k (elements in chunks <= k, all arrived)
      // add to them; M^-1 and U1 = U + dt M^-1 L_h(U) close the stage
      for (int k = 0; k < NCH && !rc; ++k) {
        cudaStreamWaitEvent(st, ctx->ev_h2d[k], 0);
        rc = ctx->impl.volume(ctx, ck[k], ck[k + 1], U, nullptr, w1, nullptr, 0.0, 0.0, 0.0, 0,
                              st);
        for (int s = 0; s < ctx->d.n_segments && !rc; ++s)
          rc = ctx->impl.faces_chunk(ctx, s, k, U, w1, st);
      }
      if (!rc) {
        const int64_t n = ne * int64_t(sn);
        const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(ctx->num_sms) * 8);
        k_stage_finalize<<<unsigned(grid), 256, 0, st>>>(n, int(sn), 1 + ctx->d.dim * (ctx->d.dim + 1) / 2,
                                                         ctx->p.egeo, U, w1, 1.0, dt);
      }
    } else {
      for (int k = 0; k < NCH; ++k) cudaStreamWaitEvent(st, ctx->ev_h2d[k], 0);
      rc = ctx->impl.run(ctx, U, nullptr, w1, w1, 0.0, 1.0, dt, 2, 0, st);
    }
    if (!rc) rc = ctx->impl.run(ctx, w1, U, w2, w2, 0.75, 0.25, 0.25 * dt, 2, 0, st);
    // stage 3: every face segment, then the volume kernel chunk by chunk,
    // each chunk's copy-out as soon as it is written
    if (!rc) rc = ctx->impl.run(ctx, w2, U, U, w1, 0.0, 0.0, 0.0, 2, 3, st);
    const bool faces = ctx->p.nif + ctx->p.nbf > 0;
    for (int k = 0; k < NCH && !rc; ++k) {
      rc = ctx->impl.volume(ctx, ck[k], ck[k + 1], w2, U, U, faces ? w1 : nullptr, 1.0 / 3.0,
                            2.0 / 3.0, (2.0 / 3.0) * dt, 2, st);
      cudaEventRecord(ctx->ev_vol[k], st);
      cudaStream_t cs = ctx->s_out[k & 1];
      cudaStreamWaitEvent(cs, ctx->ev_vol[k], 0);
      const size_t o = size_t(ck[k]) * sn, m = size_t(ck[k + 1] - ck[k]) * sn;
      if (m) cudaMemcpyAsync(U_host + o, U + o, m * sizeof(double), cudaMemcpyDeviceToHost, cs);
      cudaEventRecord(ctx->ev_d2h[k], cs);
    }
    if (rc) return rc;
  }
  // join the copy streams back onto the caller's stream
  for (int i = 0; i < 2; ++i)
    for (cudaStream_t s : {ctx->s_in[i], ctx->s_out[i]}) {
      cudaEventRecord(ctx->ev_s1, s);
      cudaStreamWaitEvent(st, ctx->ev_s1, 0);
    }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "host steps");
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

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

int tdg_mgs_pass(tdg_ctx* ctx, const double* V, int64_t ldv, int i, int j, double* w, int64_t n,
                 double* h, void* stream) {
  if (!ctx || !V || !w || !h) return fail(TDG_E_INVALID, "null argument");
  if (j < 0 || i < 0 || i > j + 1 || n < 0 || ldv < n) return fail(TDG_E_INVALID, "bad mgs sizes");
  if (!aligned16(V) || !aligned16(w) || (ldv & 1))
    return fail(TDG_E_INVALID, "mgs operands must be 16-byte aligned (even ldv)");
  cudaError_t e = launch_mgs_pass(V, ldv, i, j, w, n, h, ctx->part, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "mgs_pass");
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
  ctx->use_graph = ((variant >> 5) & 1) == 0;  // bit 5: no CUDA graph for ssprk3
  ctx->force_tc = ((variant >> 12) & 1) != 0;
  ctx->no_fold = ((variant >> 13) & 1) != 0;    // bit 13: no face-geometry-class tables
  ctx->no_groups = ((variant >> 14) & 1) != 0;  // bit 14: one-face kernel despite face groups
  ctx->no_vcls = ((variant >> 15) & 1) != 0;    // bit 15: no volume element classes
  ctx->no_modal = ((variant >> 16) & 1) != 0;   // bit 16: face groups on full traces
  ctx->no_sig = ((variant >> 17) & 1) != 0;     // bit 17: k_faces_fast despite signature runs
  ctx->sig_async = ((variant >> 18) & 1) != 0;  // bit 18: cp.async-staged k_faces_sig at any size
  // bits 8-11: CTAs per SM of the 2D face kernel's grid-stride grid (0 =
  // the resident count; 15 = one group per warp, no grid cap)
  const int f = (variant >> 8) & 15;
  ctx->face_ctas_per_sm = f == 15 ? -1 : f;
  if (ctx->gexec) {  // kernel choice changed: re-capture
    cudaGraphExecDestroy(ctx->gexec);
    ctx->gexec = nullptr;
  }
  return TDG_OK;
}

int tdg_face_runs(const tdg_ctx* ctx, int64_t* n_runs, int64_t* n_folded) {
  if (!ctx || !n_runs || !n_folded) return fail(TDG_E_INVALID, "null argument");
  *n_runs = int64_t(ctx->sig_runs.size());
  *n_folded = 0;
  for (const SigRun& r : ctx->sig_runs) *n_folded += r.fold ? 1 : 0;
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

int tdg_color_faces(int64_t n_faces, const int32_t* elem_in, const int32_t* elem_out,
                    int64_t n_elements, const int64_t* order, int32_t* color) {
  if (n_faces < 0 || n_elements < 0) return fail(TDG_E_INVALID, "negative size");
  if (n_faces > 0 && (!elem_in || !elem_out || !color)) return fail(TDG_E_INVALID, "null argument");
  std::vector<uint64_t> used(size_t(n_elements), 0);
  int ncol = 0;
  for (int64_t k = 0; k < n_faces; ++k) {
    const int64_t f = order ? order[k] : k;
    if (f < 0 || f >= n_faces) return fail(TDG_E_INVALID, "order index out of range");
    const int32_t a = elem_in[f], b = elem_out[f];
    if (a >= n_elements || b >= n_elements) return fail(TDG_E_INVALID, "element index out of range");
    const uint64_t busy = (a >= 0 ? used[a] : 0) | (b >= 0 ? used[b] : 0);
    if (busy == ~uint64_t(0)) return fail(TDG_E_INVALID, "more than 64 colours");
    const int c = __builtin_ctzll(~busy);
    if (a >= 0) used[a] |= uint64_t(1) << c;
    if (b >= 0) used[b] |= uint64_t(1) << c;
    color[f] = c;
    ncol = c + 1 > ncol ? c + 1 : ncol;
  }
  return ncol;
}

int tdg_dmma_probe(double* out, int64_t iters, void* stream) {
  if (!out || iters < 1) return fail(TDG_E_INVALID, "bad argument");
  cudaError_t e = launch_dmma_probe(out, iters, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "dmma_probe");
}

}  // extern "C"

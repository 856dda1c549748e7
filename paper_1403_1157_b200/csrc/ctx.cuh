// Context object and the per-instantiation launch templates, shared by
// the C-ABI translation unit (capi.cu) and the instantiation units
// (inst_*.cu, compiled in parallel).
//
// One operator application = the face segments in order, then the volume
// kernel.  A face segment is one colour class of the face graph (elements
// = vertices, faces = edges; tables.build_tables): no element appears
// twice in a segment, so a segment's faces add their contributions to the
// elements' face-sum rows (ACC) without atomics, and the fixed segment
// order makes every sum bitwise reproducible.  The volume kernel then adds
// the volume terms, applies M^-1 and writes the Runge-Kutta combination.
// Slab runs put the faces that read ghost rows into the last n_seg_cut
// segments (part 2 of a split stage).
#pragma once

#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "taxisdg_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "kernels_fast.cuh"
#include "kernels_mma.cuh"
#include "kernels_tc.cuh"
#include "kernels_tcf.cuh"
#include "kernels_tcg.cuh"
#include "kernels_tcm.cuh"
#include "models.cuh"
#include "vecops.cuh"

namespace tdg {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

struct Impl {
  int (*configure)(int nqv);
  // mode: 0 L(U), 1 M^-1 L(U), 2 a U0 + b U + c M^-1 L(U); part: 0 whole,
  // 1 faces that read owned rows only, 2 the cut faces + the volume kernel,
  // 3 every face segment (no volume kernel)
  int (*run)(tdg_ctx*, const double* U, const double* U0, double* out, double* acc, double a,
             double b, double c, int mode, int part, cudaStream_t st);
  int (*volume)(tdg_ctx*, int64_t e0, int64_t e1, const double* U, const double* U0, double* out,
                const double* acc, double a, double b, double c, int mode, cudaStream_t st);
  int (*upload)(const OpParams& p);
  // host-side launch data made once at tdg_create (signature runs of the
  // 2D face kernel)
  int (*prepare)(tdg_ctx*);
  // the faces of segment s restricted to element chunk c (host-data
  // stepping), adding into acc (the add-only code words: no first writes)
  int (*faces_chunk)(tdg_ctx*, int s, int c, const double* U, double* acc, cudaStream_t st);
  int max_nqv, max_nqf;
};

bool pick_plaque(int dim, int order, Impl* out);
bool pick_reduced(int dim, int order, Impl* out);
bool pick_diffusion(int dim, int order, Impl* out);

// one colour class: interior faces [f0, f1), walls [w0, w1), face blocks
// of the 3D species-rows kernel [b0, b1), face groups of the 3D face-group
// kernel [g0, g1)
struct Segment {
  int64_t f0, f1, w0, w1, b0, b1, g0, g1;
};

// maximal run of interior faces [f0, f1) with one (inside, outside)
// trace-table signature (k_faces_sig)
struct SigRun {
  int64_t f0, f1;
  int tin, tout;
  bool fold;        // every face has the same Jinv n on both sides
  double jn[2][3];  // ... these
};

}  // namespace tdg

struct tdg_ctx {
  tdg_desc d;
  tdg::OpParams p;
  double* part = nullptr;  // reduction partials
  tdg::Impl impl;
  std::vector<tdg::Segment> seg;
  int n_seg_cut = 0;
  // profiling: event pairs per kernel kind, drained by tdg_profile_read
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[4];
  double ms[4] = {0, 0, 0, 0};
  int64_t launches[4] = {0, 0, 0, 0};
  bool force_generic = false;  // testing: pin the CTA-staged kernels
  bool force_tc = false;       // testing: tensor-core volume kernel where the SIMT one fits
  bool no_fold = false;        // testing: per-face normal-derivative folds despite class tables
  bool no_groups = false;      // testing: the one-face kernel despite face groups
  bool no_vcls = false;        // testing: per-element metric scaling despite volume classes
  bool no_modal = false;       // testing: face groups on full traces despite modal tables
  bool point_data = false;     // boundary point data: the generic face kernels
  bool no_sig = false;         // testing: k_faces_fast despite signature runs
  bool sig_async = false;      // testing: the cp.async-staged k_faces_sig on small states too
  // 2D: signature runs over the interior faces (sorted by f0) and host
  // copies of the face tables their kernel parameters are built from;
  // empty when the faces are not sorted into few runs
  std::vector<tdg::SigRun> sig_runs;
  std::vector<double> h_fB, h_fG, h_fPw, h_fw;
  int num_sms = 148;
  size_t l2_bytes = size_t(126) << 20;
  int face_ctas_per_sm = 0;    // 2D face-kernel grid cap per SM: 0 = resident CTAs, -1 = none
  // host-data stepping: copies in kChunks element chunks on two streams
  // per direction (created with the context: no call allocates later)
  static constexpr int kChunks = 8;
  int64_t vchunk[kChunks + 1] = {};  // volume-class task offsets of the element chunks
  // (segment, chunk) sub-segments and the add-only code words (FIRST bits
  // cleared): the host-data stepping's first stage runs chunk by chunk as
  // the state arrives, over face sums the volume kernel initialised
  std::vector<tdg::Segment> segc;
  const int32_t* ifcode_add = nullptr;
  const int32_t* bfcode_add = nullptr;
  cudaStream_t s_in[2] = {}, s_out[2] = {};
  cudaEvent_t ev_h2d[kChunks] = {}, ev_d2h[kChunks] = {}, ev_vol[kChunks] = {};
  cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr;
  // SSP-RK3 step replayed from a CUDA graph (captured on gstream, joined
  // to the caller's stream with events); re-captured when U / work / dt
  // change.  Not used while profiling (per-kernel events).
  bool use_graph = true;
  cudaStream_t gstream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t gev_a = nullptr, gev_b = nullptr;
  const double* g_U = nullptr;
  const double* g_w1 = nullptr;
  const double* g_w2 = nullptr;
  double g_dt = 0.0;
};

namespace tdg {

// element chunks of the host-data entry points and of the volume-class
// task lists (tables.vol_chunk_bounds): chunk k starts at element
// (ne k / kChunks) rounded down to a multiple of 8, so every chunk's rows
// keep the 32-byte alignment the vectorised kernels load with
inline int64_t chunk_start(int64_t ne, int k) {
  return k >= tdg_ctx::kChunks ? ne : (ne * k / tdg_ctx::kChunks) / 8 * 8;
}

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
  if constexpr (TcsFace<D, K, M>::ok) {
    const int sm = int(TcsFace<D, K, M>::smem());
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    for (auto fn : {k_faces_tcs<D, K, M, false, 0>, k_faces_tcs<D, K, M, false, 1>,
                    k_faces_tcs<D, K, M, false, 2>, k_faces_tcs<D, K, M, true, 0>,
                    k_faces_tcs<D, K, M, true, 1>, k_faces_tcs<D, K, M, true, 2>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, attr, sm);
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_tcs");
  }
  if constexpr (TcgFace<D, K, M>::ok) {
    const int sm = int(TcgFace<D, K, M>::smem());
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    for (auto fn : {k_faces_tcg<D, K, M, 0>, k_faces_tcg<D, K, M, 1>, k_faces_tcg<D, K, M, 2>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, attr, sm);
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_tcg");
  }
  if constexpr (TcmFace<D, K, M>::ok) {
    const int sm = int(TcmFace<D, K, M>::smem());
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    for (auto fn : {k_faces_tcm<D, K, M, 0>, k_faces_tcm<D, K, M, 1>, k_faces_tcm<D, K, M, 2>}) {
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, attr, sm);
#if TDG_TCM_CARVE
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, TDG_TCM_CARVE);
#endif
    }
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_tcm");
  }
  if constexpr (TcVol<D, K, M>::ok) {
    for (auto fn : {k_volume_tc<D, K, M, false>, k_volume_tc<D, K, M, true>})
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(TcVol<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure volume_tc");
  }
  if constexpr (MmaFace<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_faces_mma<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(MmaFace<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_mma");
  }
  if constexpr (FastFace<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_faces_fast<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(FastFace<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_fast");
  }
  if constexpr (FastVol<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_volume_fast<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(FastVol<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure volume_fast");
  }
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

// k_faces_sig: at most this many signature runs over all interior faces /
// launches per segment; meshes whose faces are not sorted into few runs
// stay on k_faces_fast
constexpr int kMaxSigRuns = 4096;
constexpr size_t kMaxSigRunsPerSegment = 8;

template <class M, int D, int K>
constexpr int SN_of() { return M::S * Dims<D, K>::NB; }

// The faces of one colour segment, adding into the face-sum rows acc.
template <int D, int K, class M>
void run_segment(tdg_ctx* ctx, const Segment& sg, const double* U, double* acc, cudaStream_t st,
                 const OpParams* po = nullptr) {
  const OpParams& p = po ? *po : ctx->p;
  constexpr int NFG = Dims<D, K>::NFG;
  OpParams q = p;  // the segment's face ranges
  q.nif = sg.f1 - sg.f0;
  q.ifel = p.ifel + 2 * sg.f0;
  q.ifcode = p.ifcode + sg.f0;
  q.ifgeo = p.ifgeo + sg.f0 * NFG;
  q.nbf = sg.w1 - sg.w0;
  q.bfel = p.bfel + sg.w0;
  q.bfcode = p.bfcode + sg.w0;
  q.bfgeo = p.bfgeo + sg.w0;
  if (p.ifbv) q.ifbv = p.ifbv + sg.f0 * p.nqf * M::S;
  if (p.bfqv) q.bfqv = p.bfqv + sg.w0 * p.nqf * M::S;
  if (q.nif + q.nbf == 0) return;
  const bool dflt = p.nqf == Dims<D, K>::NQF && !ctx->force_generic && !ctx->point_data;
  // 3D: interior faces on the species-rows tensor-core kernel (blocks of
  // one signature), walls on the element-local DMMA kernel
  if constexpr (TcsFace<D, K, M>::ok && MmaFace<D, K, M>::ok) {
    if (dflt && p.ftc != nullptr && p.fblk != nullptr && p.fmma != nullptr) {
      const bool fold = p.ftf != nullptr && p.ffold != nullptr && !ctx->no_fold;
      const int lm = (p.scheme == IP || p.scheme == BO) ? 0 : (p.scheme == BR2 ? 2 : 1);
      // face groups: the modal kernel, else the full-trace group kernel,
      // else the one-face kernel over blocks
      bool grouped = false;
      if constexpr (TcmFace<D, K, M>::ok) {
        grouped = fold && p.fgrp != nullptr && p.fmod != nullptr && !ctx->no_groups &&
                  !ctx->no_modal;
        if (grouped && sg.g1 > sg.g0) {
          KernelTimer kt(ctx, 0, st);
          using T = TcmFace<D, K, M>;
          static int resident = 0;
          if (resident == 0) {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_faces_tcm<D, K, M, 1>, T::THREADS,
                                                              T::smem()) != cudaSuccess || nb < 1)
              nb = T::MINB;
            resident = nb;
          }
          int64_t grid = sg.g1 - sg.g0;
          const int64_t cap = int64_t(ctx->num_sms) * resident;
          grid = grid < cap ? grid : cap;
          auto go = [&](auto kernel) {
            kernel<<<unsigned(grid), T::THREADS, T::smem(), st>>>(p, p.fmod, p.fgrp, sg.g0, sg.g1, U,
                                                                  acc);
          };
          go(lm == 0 ? k_faces_tcm<D, K, M, 0>
                     : (lm == 1 ? k_faces_tcm<D, K, M, 1> : k_faces_tcm<D, K, M, 2>));
        }
      }
      if constexpr (TcgFace<D, K, M>::ok) {
        const bool use = !grouped && fold && p.fgrp != nullptr && !ctx->no_groups;
        grouped = grouped || use;
        if (use && sg.g1 > sg.g0) {
          KernelTimer kt(ctx, 0, st);
          using T = TcgFace<D, K, M>;
          // persistent: the resident CTAs loop over the segment's groups
          static int resident = 0;
          if (resident == 0) {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_faces_tcg<D, K, M, 1>, T::THREADS,
                                                              T::smem()) != cudaSuccess || nb < 1)
              nb = T::MINB;
            resident = nb;
          }
          int64_t grid = sg.g1 - sg.g0;
          const int64_t cap = int64_t(ctx->num_sms) * resident;
          grid = grid < cap ? grid : cap;
          auto go = [&](auto kernel) {
            kernel<<<unsigned(grid), T::THREADS, T::smem(), st>>>(p, p.ftc, p.fgrp, sg.g0, sg.g1, U,
                                                                  acc);
          };
          go(lm == 0 ? k_faces_tcg<D, K, M, 0>
                     : (lm == 1 ? k_faces_tcg<D, K, M, 1> : k_faces_tcg<D, K, M, 2>));
        }
      }
      if (!grouped && sg.b1 > sg.b0) {
        KernelTimer kt(ctx, 0, st);
        using T = TcsFace<D, K, M>;
        int64_t grid = (sg.b1 - sg.b0 + T::WARPS - 1) / T::WARPS;
        const int64_t cap = int64_t(ctx->num_sms) * T::MINB_FOLD * 8;
        grid = grid < cap ? grid : cap;
        auto go = [&](auto kernel) {
          kernel<<<unsigned(grid), 128, T::smem(), st>>>(p, p.ftc, p.fblk, sg.b0, sg.b1, U, acc);
        };
        if (fold)
          go(lm == 0 ? k_faces_tcs<D, K, M, true, 0>
                     : (lm == 1 ? k_faces_tcs<D, K, M, true, 1> : k_faces_tcs<D, K, M, true, 2>));
        else
          go(lm == 0 ? k_faces_tcs<D, K, M, false, 0>
                     : (lm == 1 ? k_faces_tcs<D, K, M, false, 1> : k_faces_tcs<D, K, M, false, 2>));
      }
      if (q.nbf > 0) {
        KernelTimer kt(ctx, 1, st);
        using T = MmaFace<D, K, M>;
        OpParams w = q;
        w.nif = 0;
        const int64_t warps = (w.nbf + T::NFW - 1) / T::NFW;
        const int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
        k_faces_mma<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(w, w.fmma, U, acc);
      }
      return;
    }
  }
  // 3D without the species-rows kernel (Dirichlet mirror models): the
  // element-local DMMA kernel for interior faces and walls
  if constexpr (MmaFace<D, K, M>::ok) {
    if (D == 3 && dflt && p.fmma != nullptr) {
      KernelTimer kt(ctx, 0, st);
      using T = MmaFace<D, K, M>;
      const int64_t warps = (q.nif + T::NFW - 1) / T::NFW + (q.nbf + T::NFW - 1) / T::NFW;
      const int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
      k_faces_mma<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(q, q.fmma, U, acc);
      return;
    }
  }
  // 2D: the interior faces of the segment's signature runs with their
  // tables as kernel parameters; the last run's launch takes the walls
  if constexpr (SigFace<D, K, M>::ok) {
    if (dflt && !ctx->no_sig && !ctx->sig_runs.empty() && q.nif > 0) {
      // runs overlapping [f0, f1) (the chunked sub-segments cut runs)
      size_t r0 = 0, r1 = ctx->sig_runs.size();
      while (r0 < r1 && ctx->sig_runs[r0].f1 <= sg.f0) ++r0;
      size_t re = r0;
      while (re < r1 && ctx->sig_runs[re].f0 < sg.f1) ++re;
      if (re - r0 <= kMaxSigRunsPerSegment) {
        using T = SigFace<D, K, M>;
        constexpr int F = Dims<D, K>::NQF, NB = Dims<D, K>::NB;
        static int resident = 0;
        if (resident == 0) {
          int nb = 0;
          if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_faces_sig<D, K, M, D>, 128, 0) !=
                  cudaSuccess || nb < 1)
            nb = T::MINB;
          resident = nb;
        }
        for (size_t k = r0; k < re; ++k) {
          const SigRun& rr = ctx->sig_runs[k];
          const int64_t a = rr.f0 > sg.f0 ? rr.f0 : sg.f0, b = rr.f1 < sg.f1 ? rr.f1 : sg.f1;
          if (b <= a) continue;
          OpParams r = q;
          r.nif = b - a;
          r.ifel = p.ifel + 2 * a;
          r.ifcode = p.ifcode + a;
          r.ifgeo = p.ifgeo + a * NFG;
          if (k + 1 < re) r.nbf = 0;  // the walls go with the last run
          KernelTimer kt(ctx, 0, st);
          const int64_t groups = (r.nif + T::FPW - 1) / T::FPW;
          const int64_t wgroups = (r.nbf + T::FPW - 1) / T::FPW;
          int64_t grid = (groups + wgroups + T::WARPS - 1) / T::WARPS;
          if (ctx->face_ctas_per_sm >= 0) {
            const int per = ctx->face_ctas_per_sm > 0 ? ctx->face_ctas_per_sm : resident;
            const int64_t cap = int64_t(ctx->num_sms) * per;
            grid = grid < cap ? grid : cap;
          }
          auto fill = [&](auto& tb, bool fold) {
            for (int side = 0; side < 2; ++side) {
              const int t = side ? rr.tout : rr.tin;
              std::memcpy(tb.B[side], ctx->h_fB.data() + size_t(t) * F * NB, sizeof(tb.B[side]));
              std::memcpy(tb.Pw[side], ctx->h_fPw.data() + size_t(t) * F * F, sizeof(tb.Pw[side]));
              const double* g = ctx->h_fG.data() + size_t(t) * F * NB * D;
              double* o = &tb.G[side][0][0][0];
              for (int j = 0; j < F * NB; ++j) {
                if (fold) {  // d_n phi = G . (Jinv n), k_faces_fast's order
                  double v = 0.0;
                  for (int c = 0; c < D; ++c) v = std::fma(g[j * D + c], rr.jn[side][c], v);
                  o[j] = v;
                } else {
                  for (int c = 0; c < D; ++c) o[j * D + c] = g[j * D + c];
                }
              }
            }
            std::memcpy(tb.w, ctx->h_fw.data(), sizeof(tb.w));
          };
          // states larger than the L2 (C3): the cp.async-staged variant
          // hides the record -> rows round trips to DRAM (C3 faces 2.22 ->
          // 1.91 ms); on L2-resident states (C2) it is 2% slower
          const bool async_ = TDG_SIG_FORCE_ASYNC >= 0
                                  ? TDG_SIG_FORCE_ASYNC != 0
                                  : ctx->sig_async ||
                                    size_t(ctx->d.n_elements + ctx->d.n_ghost) * SN_of<M, D, K>() * 8 >
                                        ctx->l2_bytes / 2;
          if (rr.fold && !ctx->no_fold) {
            FaceSigTab<D, K, 1> tb;
            fill(tb, true);
            if (async_)
              k_faces_sig_async<D, K, M, 1><<<unsigned(grid), 128, 0, st>>>(r, tb, U, acc, groups, wgroups);
            else
              k_faces_sig<D, K, M, 1><<<unsigned(grid), 128, 0, st>>>(r, tb, U, acc, groups, wgroups);
          } else {
            FaceSigTab<D, K, D> tb;
            fill(tb, false);
            if (async_)
              k_faces_sig_async<D, K, M, D><<<unsigned(grid), 128, 0, st>>>(r, tb, U, acc, groups, wgroups);
            else
              k_faces_sig<D, K, M, D><<<unsigned(grid), 128, 0, st>>>(r, tb, U, acc, groups, wgroups);
          }
        }
        return;
      }
    }
  }
  // 2D: register-resident kernel, interior faces and walls in one launch
  if constexpr (FastFace<D, K, M>::ok) {
    if (dflt) {
      KernelTimer kt(ctx, 0, st);
      using T = FastFace<D, K, M>;
      const int64_t warps = (q.nif + T::FPW - 1) / T::FPW + (q.nbf + T::FPW - 1) / T::FPW;
      int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
      // grid-stride: face_ctas_per_sm CTAs per SM loop over the groups
      // (tables staged once per CTA); -1 = one group per warp
      if (ctx->face_ctas_per_sm >= 0) {
        const int per = ctx->face_ctas_per_sm > 0 ? ctx->face_ctas_per_sm : T::MINB;
        const int64_t cap = int64_t(ctx->num_sms) * per;
        grid = grid < cap ? grid : cap;
      }
      k_faces_fast<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(q, U, acc, warps);
      return;
    }
  }
  if (q.nif > 0) {
    KernelTimer kt(ctx, 0, st);
    constexpr int TF = FaceTile<D, K, M>::TF;
    const int64_t grid = (q.nif + TF - 1) / TF;
    k_faces<D, K, M><<<unsigned(grid), kThreads, FaceTile<D, K, M>::smem(), st>>>(q, U, acc);
  }
  if (q.nbf > 0) {
    KernelTimer kt(ctx, 1, st);
    constexpr int TF = WallTile<D, K, M>::TF;
    const int64_t grid = (q.nbf + TF - 1) / TF;
    k_wall<D, K, M><<<unsigned(grid), kThreads, WallTile<D, K, M>::smem(), st>>>(q, U, acc);
  }
}

// Volume terms + face sums + M^-1 + stage combination over the elements
// [e0, e1) (element-local: any range split gives the same bits).
template <int D, int K, class M>
int volume(tdg_ctx* ctx, int64_t e0, int64_t e1, const double* U, const double* U0, double* out,
           const double* acc, double a, double b, double c, int mode, cudaStream_t st) {
  constexpr int SN = SN_of<M, D, K>(), NEG = Dims<D, K>::NEG;
  if (e1 <= e0) return TDG_OK;
  // element-geometry classes: the range must be a run of whole chunks
  int64_t ct0 = -1, ct1 = -1;
  if (ctx->p.vperm != nullptr && !ctx->no_vcls) {
    constexpr int NCH = tdg_ctx::kChunks;
    const int64_t ne = ctx->p.ne;
    for (int k = 0; k <= NCH; ++k) {
      if (chunk_start(ne, k) == e0 && ct0 < 0) ct0 = ctx->vchunk[k];
      if (chunk_start(ne, k) == e1) ct1 = ctx->vchunk[k];
    }
    if (ct0 < 0 || ct1 < 0) ct0 = ct1 = -1;
  }
  const double *U_all = U, *U0_all = U0, *acc_all = acc;
  double* out_all = out;
  OpParams p = ctx->p;
  p.ne = e1 - e0;
  p.egeo = ctx->p.egeo + e0 * NEG;
  U += e0 * SN;
  out += e0 * SN;
  if (U0) U0 += e0 * SN;
  if (acc) acc += e0 * SN;
  KernelTimer kt(ctx, 2, st);
  const bool dflt = p.nqv == Dims<D, K>::NQV && !ctx->force_generic;
  constexpr bool fast_vol = FastVol<D, K, M>::ok, tc_ok = TcVol<D, K, M>::ok;
  const bool use_fv = fast_vol && dflt && !ctx->force_tc;
  const bool use_tc = tc_ok && dflt && p.vtc != nullptr && !use_fv;
  if (use_fv) {
    if constexpr (fast_vol) {
      using T = FastVol<D, K, M>;
      const int64_t grid = (p.ne + T::TE - 1) / T::TE;
      k_volume_fast<D, K, M><<<unsigned(grid), T::TE, T::smem(), st>>>(p, U, acc, U0, out, a, b, c,
                                                                        mode);
    }
  } else if (use_tc) {
    if constexpr (tc_ok) {
      using T = TcVol<D, K, M>;
      const bool cls = ct0 >= 0;
      const int64_t tasks = cls ? ct1 - ct0 : (p.ne + T::EW - 1) / T::EW;
      int64_t grid = (tasks + T::WARPS - 1) / T::WARPS;
      // persistent grid: every CTA slot the registers / shared memory allow
      static int resident = 0;
      if (resident == 0) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_volume_tc<D, K, M, true>,
                                                          32 * T::WARPS, T::smem()) != cudaSuccess ||
            nb < 1)
          nb = T::MINB;
        resident = nb;
      }
      const int64_t cap = int64_t(ctx->num_sms) * resident;
      grid = grid < cap ? grid : cap;
      if (grid > 0) {
        if (cls)  // absolute element ids: the unshifted arrays
          k_volume_tc<D, K, M, true><<<unsigned(grid), 32 * T::WARPS, T::smem(), st>>>(
              ctx->p, p.vtc, U_all, acc_all, U0_all, out_all, a, b, c, mode, ct0, ct1);
        else
          k_volume_tc<D, K, M, false><<<unsigned(grid), 32 * T::WARPS, T::smem(), st>>>(
              p, p.vtc, U, acc, U0, out, a, b, c, mode, 0, tasks);
      }
    }
  } else {
    constexpr int TE = VolumeTile<D, K, M>::TE;
    const int64_t grid = (p.ne + TE - 1) / TE;
    k_volume<D, K, M><<<unsigned(grid), kThreads, VolumeTile<D, K, M>::smem(p.nqv), st>>>(
        p, U, acc, U0, out, a, b, c, mode);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "volume launch");
}

template <int D, int K, class M>
int run(tdg_ctx* ctx, const double* U, const double* U0, double* out, double* acc, double a,
        double b, double c, int mode, int part, cudaStream_t st) {
  const int ns = int(ctx->seg.size()), nc = ctx->n_seg_cut;
  const int s0 = part == 2 ? ns - nc : 0, s1 = part == 1 ? ns - nc : ns;
  for (int s = s0; s < s1; ++s) run_segment<D, K, M>(ctx, ctx->seg[s], U, acc, st);
  if (part == 1 || part == 3) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TDG_OK : cuda_fail(e, "face launch");
  }
  const bool faces = ctx->p.nif + ctx->p.nbf > 0;
  return volume<D, K, M>(ctx, 0, ctx->p.ne, U, U0, out, faces ? acc : nullptr, a, b, c, mode, st);
}

template <int D, int K, class M>
int upload_const(const OpParams& p) {
  if constexpr (FastFace<D, K, M>::ok) {
    if (p.nqf != Dims<D, K>::NQF) return TDG_OK;  // the fast kernel is not used
    using CL = FaceConstLayout<D, K>;
    cudaError_t e = cudaMemcpyToSymbol(c_face_tab<D, K>, p.fB, size_t(CL::OP) * sizeof(double), 0,
                                       cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpyToSymbol(c_face_tab<D, K>, p.fPw, size_t(CL::OW - CL::OP) * sizeof(double),
                             size_t(CL::OP) * sizeof(double), cudaMemcpyDeviceToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpyToSymbol(c_face_tab<D, K>, p.fw, size_t(CL::N - CL::OW) * sizeof(double),
                             size_t(CL::OW) * sizeof(double), cudaMemcpyDeviceToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "face tables -> constant memory");
  }
#if TDG_VOL_CONST
  if constexpr (FastVol<D, K, M>::ok && VolConstLayout<D, K>::fits) {
    if (p.nqv != Dims<D, K>::NQV) return TDG_OK;
    using VL = VolConstLayout<D, K>;
    auto put = [](const double* src, int off, int n) {
      return cudaMemcpyToSymbol(c_vol_tab<D, K>, src, size_t(n) * sizeof(double),
                                size_t(off) * sizeof(double), cudaMemcpyDeviceToDevice);
    };
    cudaError_t e = put(p.phi, VL::OPHI, VL::OGR - VL::OPHI);
    if (e == cudaSuccess) e = put(p.grad, VL::OGR, VL::OW - VL::OGR);
    if (e == cudaSuccess) e = put(p.wv, VL::OW, VL::OKS - VL::OW);
    if (e == cudaSuccess) e = put(p.ks, VL::OKS, VL::N - VL::OKS);
    if (e != cudaSuccess) return cuda_fail(e, "volume tables -> constant memory");
  }
#endif
  return TDG_OK;
}

// Signature runs of the interior faces and host copies of the face tables
// (k_faces_sig builds its kernel-parameter tables from them).  The face
// arrays are device memory: read back once, here.
template <int D, int K, class M>
int prepare(tdg_ctx* ctx) {
  if constexpr (SigFace<D, K, M>::ok) {
    const OpParams& p = ctx->p;
    if (p.nqf != Dims<D, K>::NQF || p.nif == 0 || ctx->point_data) return TDG_OK;
    constexpr int F = Dims<D, K>::NQF, NB = Dims<D, K>::NB, NT = Dims<D, K>::NT;
    std::vector<int32_t> code(size_t(p.nif));
    ctx->h_fB.resize(size_t(NT) * F * NB);
    ctx->h_fG.resize(size_t(NT) * F * NB * D);
    ctx->h_fPw.resize(size_t(NT) * F * F);
    ctx->h_fw.resize(F);
    cudaError_t e = cudaMemcpy(code.data(), p.ifcode, code.size() * sizeof(int32_t), cudaMemcpyDeviceToHost);
    auto back = [&e](std::vector<double>& h, const double* d) {
      if (e == cudaSuccess) e = cudaMemcpy(h.data(), d, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
    };
    back(ctx->h_fB, p.fB);
    back(ctx->h_fG, p.fG);
    back(ctx->h_fPw, p.fPw);
    back(ctx->h_fw, p.fw);
    if (e != cudaSuccess) return cuda_fail(e, "face tables -> host");
    std::vector<SigRun> runs;
    bool ok = true;
    for (int64_t f = 0; f < p.nif && ok; ++f) {
      const int c = code[size_t(f)];
      const int tin = c & 31, tout = (c >> 5) & 31;
      ok = !((c >> 14) & 1) && tin < NT && tout < NT;  // no mirror faces
      if (runs.empty() || runs.back().tin != tin || runs.back().tout != tout) {
        runs.push_back(SigRun{f, f + 1, tin, tout, false, {}});
        ok = ok && runs.size() <= size_t(kMaxSigRuns);
      } else {
        runs.back().f1 = f + 1;
      }
    }
    if (ok) {
      // runs whose faces all carry the same Jinv n (bitwise) fold it into
      // the tables; the face records are read back in pieces
      constexpr int NFG = Dims<D, K>::NFG;
      constexpr int64_t PIECE = int64_t(1) << 18;
      std::vector<double> geo(size_t(PIECE) * NFG);
      for (SigRun& r : runs) {
        r.fold = true;
        bool have = false;
        for (int64_t f0 = r.f0; f0 < r.f1 && r.fold; f0 += PIECE) {
          const int64_t n = r.f1 - f0 < PIECE ? r.f1 - f0 : PIECE;
          e = cudaMemcpy(geo.data(), p.ifgeo + f0 * NFG, size_t(n) * NFG * sizeof(double),
                         cudaMemcpyDeviceToHost);
          if (e != cudaSuccess) return cuda_fail(e, "face records -> host");
          if (!have) {
            for (int side = 0; side < 2; ++side)
              for (int c = 0; c < D; ++c) r.jn[side][c] = geo[size_t(side) * D + c];
            have = true;
          }
          for (int64_t f = 0; f < n && r.fold; ++f)
            for (int j = 0; j < 2 * D; ++j)
              r.fold = r.fold && geo[size_t(f) * NFG + j] == r.jn[j / D][j % D];
        }
      }
      ctx->sig_runs = std::move(runs);
    }
  }
  return TDG_OK;
}

template <int D, int K, class M>
int faces_chunk(tdg_ctx* ctx, int s, int c, const double* U, double* acc, cudaStream_t st) {
  OpParams p = ctx->p;
  p.ifcode = ctx->ifcode_add;
  p.bfcode = ctx->bfcode_add;
  run_segment<D, K, M>(ctx, ctx->segc[size_t(s) * tdg_ctx::kChunks + c], U, acc, st, &p);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "face launch (chunk)");
}

template <int D, int K, class M>
Impl make_impl() {
  return Impl{&configure<D, K, M>, &run<D, K, M>, &volume<D, K, M>, &upload_const<D, K, M>,
              &prepare<D, K, M>, &faces_chunk<D, K, M>,
              Dims<D, K>::NQV, Dims<D, K>::NQF};
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

}  // namespace tdg

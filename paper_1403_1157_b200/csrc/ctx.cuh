// Context object and the per-instantiation launch templates, shared by
// the C-ABI translation unit (capi.cu) and the instantiation units
// (inst_*.cu, compiled in parallel).
#pragma once

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
#include "models.cuh"
#include "vecops.cuh"

namespace tdg {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

struct Impl {
  int (*configure)(int nqv);
  int (*run)(tdg_ctx*, const double* U, const double* U0, double* out, double a, double b,
             double c, int mode, cudaStream_t st);
  int (*host_steps)(tdg_ctx*, double* U_host, int64_t nsteps, double dt, cudaStream_t st);
  int (*upload)(const OpParams& p);
  int max_nqv, max_nqf;
};

bool pick_plaque(int dim, int order, Impl* out);
bool pick_reduced(int dim, int order, Impl* out);
bool pick_diffusion(int dim, int order, Impl* out);

}  // namespace tdg

struct tdg_ctx {
  tdg_desc d;
  tdg::OpParams p;
  double* fc = nullptr;    // face-contribution slots [d+1][ne][S][nb]
  double* part = nullptr;  // reduction partials
  tdg::Impl impl;
  // profiling: event pairs per kernel kind, drained by tdg_profile_read
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[4];
  double ms[4] = {0, 0, 0, 0};
  int64_t launches[4] = {0, 0, 0, 0};
  bool force_generic = false;  // testing: pin the CTA-staged kernels
  int num_sms = 148;
  bool flip_mma = false;  // testing: swap tensor-core / SIMT face kernel choice
  bool use_vmma = false;  // A/B: tensor-core volume kernel (slower than SIMT at C2)
  bool force_tc = false;  // testing: transposed tensor-core volume kernel everywhere
  bool no_tcf = false;
  bool faces_first = true;
  bool face_rows_tc = false;
  bool walls_first = false;   // 3D: wall faces before the interior tensor-core faces  // 3D: faces-as-rows TC face kernel instead of species rows
  // host-pipelined stepping: element bands and the banded face order
  // (tables.build_tables), device state / stage buffers, copy streams
  int n_bands = 1;
  std::vector<int64_t> band_elem, band_face, band_wall, band_blk;
  double* hs_buf = nullptr;  // [3][rows][S][nb]: U, stage 1, stage 2
  size_t hs_n = 0;
  // copy streams per direction: band k's copy-in / copy-out on stream
  // k mod copy_streams, so a band waiting for its previous copy-out does
  // not hold back the next bands' copies (head-of-line blocking)
  static constexpr int kCopyStreams = 8;
  cudaStream_t s_in[kCopyStreams] = {}, s_out[kCopyStreams] = {};
  int copy_streams = 2;
  cudaStream_t hs_st[6] = {};  // per stage: faces + slot sums, volume part
  std::vector<cudaEvent_t> ev_h2d, ev_d2h, ev_done, ev_vol_b;  // done / vol: [stage][band]
  cudaEvent_t ev_s0 = nullptr, ev_s1 = nullptr;
  // overlapped application: volume part on `aux` concurrent with the
  // face kernel on the caller's stream, then the face-slot sum
  bool overlap = true;
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_in = nullptr, ev_vol = nullptr;
  double* work2 = nullptr;  // second SSP-RK3 stage vector (library-owned)
  size_t work2_n = 0;
  int vol_variant = 0;         // 0: 1 thread/element (default), 1: 4 lanes/element
  // SSP-RK3 step replayed from a CUDA graph (captured on gstream, joined
  // to the caller's stream with events); re-captured when U / work / dt
  // change.  Not used while profiling (per-kernel events).
  bool use_graph = true;
  cudaStream_t gstream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t gev_a = nullptr, gev_b = nullptr;
  const double* g_U = nullptr;
  const double* g_work = nullptr;
  double g_dt = 0.0;
  int face_ctas_per_sm = 0;    // face-kernel grid cap per SM: 0 = resident CTAs, -1 = none
};

namespace tdg {

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
  if constexpr (MmaVol<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_volume_mma<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(MmaVol<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure volume_mma");
  }
  if constexpr (TcsFace<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_faces_tcs<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(TcsFace<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_tcs");
  }
  if constexpr (TcFace<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_faces_tc<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(TcFace<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure faces_tc");
  }
  if constexpr (TcVol<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_volume_tc<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  if constexpr (Vol4<D, K, M>::ok) {
    e = cudaFuncSetAttribute(k_volume4<D, K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Vol4<D, K, M>::smem()));
    if (e != cudaSuccess) return cuda_fail(e, "configure volume4");
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

template <class M, int D, int K>
constexpr int SN_of() { return M::S * Dims<D, K>::NB; }

template <int D, int K, class M>
void run_faces(tdg_ctx* ctx, const OpParams& p, const double* U, cudaStream_t st, bool use_ff) {
  constexpr bool fast_face = FastFace<D, K, M>::ok;
  // tensor-core face kernel: default in 3D, opt-in (flip) in 2D
  constexpr bool mma_ok = MmaFace<D, K, M>::ok;
  bool use_mma = mma_ok && p.fmma != nullptr && p.nqf == Dims<D, K>::NQF && !ctx->force_generic;
  use_mma = use_mma && ((D == 3) != ctx->flip_mma);
  if (use_mma) {
    if constexpr (mma_ok) {
      using T = MmaFace<D, K, M>;
      if (p.nif + p.nbf > 0) {
        KernelTimer kt(ctx, 0, st);
        const int64_t warps = (p.nif + T::NFW - 1) / T::NFW + (p.nbf + T::NFW - 1) / T::NFW;
        const int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
        k_faces_mma<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, p.fmma, U, ctx->fc);
      }
    }
    return;
  }
  if (use_ff) {
    if constexpr (fast_face) {
      if (p.nif + p.nbf > 0) {
        KernelTimer kt(ctx, 0, st);
        using T = FastFace<D, K, M>;
        const int64_t warps = (p.nif + T::FPW - 1) / T::FPW + (p.nbf + T::FPW - 1) / T::FPW;
        int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
        // persistent-style grid: face_ctas_per_sm CTAs per SM loop over
        // the groups (tables staged once per CTA); 0 = one group per warp
        if (ctx->face_ctas_per_sm >= 0) {
          const int per = ctx->face_ctas_per_sm > 0 ? ctx->face_ctas_per_sm : T::MINB;
          const int64_t cap = int64_t(ctx->num_sms) * per;
          grid = grid < cap ? grid : cap;
        }
        k_faces_fast<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, U, ctx->fc, warps);
      }
    }
  } else {
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
  }
}

// fast volume kernels: vk 0 one thread per element, 1 tensor-core
// (element-local GEMMs), 2 tensor-core transposed (elements x points)
template <int D, int K, class M>
void launch_volume(tdg_ctx* ctx, const OpParams& p, const double* U, const double* U0, double* out,
                   double a, double b, double c, int mode, cudaStream_t st, int vk) {
  if (vk == 2) {
    if constexpr (TcVol<D, K, M>::ok) {
      using T = TcVol<D, K, M>;
      const int64_t tasks = (p.ne + T::EW - 1) / T::EW;
      int64_t grid = (tasks + T::WARPS - 1) / T::WARPS;
      // persistent grid: every CTA slot the registers / shared memory allow
      static int resident = 0;
      if (resident == 0) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_volume_tc<D, K, M>, 128,
                                                          T::smem()) != cudaSuccess || nb < 1)
          nb = T::MINB;
        resident = nb;
      }
      const int64_t cap = int64_t(ctx->num_sms) * resident;
      grid = grid < cap ? grid : cap;
      k_volume_tc<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, p.vtc, U, ctx->fc, U0, out,
                                                                   a, b, c, mode);
    }
    return;
  }
  if (vk == 1) {
    if constexpr (MmaVol<D, K, M>::ok) {
      using T = MmaVol<D, K, M>;
      const int64_t grid = (p.ne + T::TE - 1) / T::TE;
      k_volume_mma<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, p.vmma, U, ctx->fc, U0, out,
                                                                    a, b, c, mode);
    }
    return;
  }
  if constexpr (FastVol<D, K, M>::ok) {
    using T = FastVol<D, K, M>;
    const int64_t grid = (p.ne + T::TE - 1) / T::TE;
    k_volume_fast<D, K, M><<<unsigned(grid), T::TE, T::smem(), st>>>(p, U, ctx->fc, U0, out, a,
                                                                      b, c, mode);
  }
}

// transposed tensor-core interior faces over face blocks [b0, b1) (3D;
// species rows by default) and the walls [w0, w1) on the element-local
// DMMA kernel
template <int D, int K, class M>
void run_faces_tc(tdg_ctx* ctx, const OpParams& p, const double* U, int64_t b0, int64_t b1,
                  int64_t w0, int64_t w1, cudaStream_t st) {
  if constexpr (TcFace<D, K, M>::ok && MmaFace<D, K, M>::ok) {
    auto walls = [&]() {
      if (w1 <= w0) return;
      KernelTimer kt(ctx, 1, st);
      using T = MmaFace<D, K, M>;
      OpParams pw = p;
      pw.nif = 0;
      pw.bfel = p.bfel + w0;
      pw.bflf = p.bflf + w0;
      pw.bfcode = p.bfcode + w0;
      pw.bfgeo = p.bfgeo + w0;
      pw.nbf = w1 - w0;
      const int64_t warps = (pw.nbf + T::NFW - 1) / T::NFW;
      const int64_t grid = (warps + T::WARPS - 1) / T::WARPS;
      k_faces_mma<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(pw, pw.fmma, U, ctx->fc);
    };
    if (ctx->walls_first) walls();
    if (b1 > b0) {
      KernelTimer kt(ctx, 0, st);
      bool done = false;
      if constexpr (TcsFace<D, K, M>::ok) {
        if (!ctx->face_rows_tc) {  // species rows, one face per warp (default)
          using T = TcsFace<D, K, M>;
          int64_t grid = (b1 - b0 + T::WARPS - 1) / T::WARPS;
          const int64_t cap = int64_t(ctx->num_sms) * T::MINB * 8;
          grid = grid < cap ? grid : cap;
          k_faces_tcs<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, p.ftc, p.fblk, b0, b1,
                                                                       U, ctx->fc);
          done = true;
        }
      }
      if (!done) {
        using T = TcFace<D, K, M>;
        int64_t grid = (b1 - b0 + T::WARPS - 1) / T::WARPS;
        const int64_t cap = int64_t(ctx->num_sms) * T::MINB * 4;
        grid = grid < cap ? grid : cap;
        k_faces_tc<D, K, M><<<unsigned(grid), 128, T::smem(), st>>>(p, p.ftc, p.fblk, b0, b1, U,
                                                                    ctx->fc);
      }
    }
    if (!ctx->walls_first) walls();
  }
}

template <int D, int K, class M>
int run(tdg_ctx* ctx, const double* U, const double* U0, double* out, double a, double b,
        double c, int mode, cudaStream_t st) {
  // mode bits 8-9: 0 whole application; 1 "begin" (everything that does
  // not read ghost rows); 2 "end" (cut faces + what depends on them).  A
  // slab-decomposed stage runs begin, the NCCL ghost exchange, end.
  const int part = (mode >> 8) & 3;
  mode &= 0xff;
  const OpParams& p = ctx->p;
  const int64_t ncut = ctx->d.n_cut_faces;
  // faces split: [0, nif-ncut) + walls need owned rows only; the last ncut
  // interior faces touch ghost rows
  // transposed tensor-core interior-face kernel (3D): blocks of faces of
  // one signature; walls on the element-local DMMA kernel
  constexpr bool tcf_ok = TcFace<D, K, M>::ok && MmaFace<D, K, M>::ok;
  const bool use_tcf = tcf_ok && p.ftc != nullptr && p.fblk != nullptr && p.fmma != nullptr &&
                       p.nqf == Dims<D, K>::NQF && !ctx->force_generic && !ctx->no_tcf &&
                       !ctx->flip_mma;
  auto faces_tc = [&](int which) {
    if constexpr (tcf_ok) {
      const int64_t nblk = ctx->d.n_face_blocks, ncb = ctx->d.n_face_blocks_cut;
      const int64_t b0 = which == 2 ? nblk - ncb : 0;
      const int64_t b1 = which == 1 ? nblk - ncb : nblk;
      run_faces_tc<D, K, M>(ctx, p, U, b0, b1, which != 2 ? 0 : p.nbf, p.nbf, st);
    }
  };
  auto faces = [&](int which, bool use_ff_) {
    if (use_tcf) {
      faces_tc(part == 0 ? 0 : which);
      return;
    }
    if (which == 0 && part == 0) {
      run_faces<D, K, M>(ctx, p, U, st, use_ff_);
      return;
    }
    OpParams pp = p;
    if (which == 1) {
      pp.nif = p.nif - ncut;
    } else {
      const int64_t off = p.nif - ncut;
      pp.ifel = p.ifel + 2 * off;
      pp.iflf = p.iflf + 2 * off;
      pp.ifcode = p.ifcode + off;
      pp.ifgeo = p.ifgeo + off * Dims<D, K>::NFG;
      pp.nif = ncut;
      pp.nbf = 0;
    }
    if (pp.nif + pp.nbf > 0) run_faces<D, K, M>(ctx, pp, U, st, use_ff_);
  };
  // register-resident kernels when the tables / working set fit and the
  // default quadrature is in use; generic CTA-staged kernels otherwise
  constexpr bool fast_face = FastFace<D, K, M>::ok;
  constexpr bool fast_vol = FastVol<D, K, M>::ok;
  const bool use_ff = fast_face && p.nqf == Dims<D, K>::NQF && !ctx->force_generic;
  const bool use_fv = fast_vol && p.nqv == Dims<D, K>::NQV && !ctx->force_generic;
  const bool use_v4 = Vol4<D, K, M>::ok && p.nqv == Dims<D, K>::NQV && !ctx->force_generic &&
                      ctx->vol_variant == 1;
  // overlapped path: fast volume kernel (without the face-slot sum) on the
  // aux stream while the face kernel runs; out must not alias U (the face
  // kernel still reads U), U0 may alias out (read before written per row)
  constexpr bool vmma_ok = MmaVol<D, K, M>::ok;
  const bool use_vm = vmma_ok && p.vmma != nullptr && p.nqv == Dims<D, K>::NQV &&
                      !ctx->force_generic && ctx->use_vmma;
  // transposed tensor-core volume kernel: default where the one-thread-
  // per-element kernel does not fit (2D k=3, 3D)
  constexpr bool tc_ok = TcVol<D, K, M>::ok;
  const bool use_tc = tc_ok && !use_vm && p.vtc != nullptr && p.nqv == Dims<D, K>::NQV &&
                      !ctx->force_generic && (ctx->force_tc || !use_fv);
  const int vk = use_vm ? 1 : (use_tc ? 2 : 0);
  const bool overlap = (use_fv || use_vm || use_tc) && (use_ff || use_tcf) && ctx->overlap &&
                       ctx->aux &&
                       out != U && p.ne > 0 && (SN_of<M, D, K>() % 2 == 0);
  if (overlap) {
    if constexpr ((fast_vol || vmma_ok || tc_ok) && (SN_of<M, D, K>() % 2 == 0)) {
      if (part != 2) {
        cudaEventRecord(ctx->ev_in, st);
        if (ctx->faces_first) faces(part == 0 ? 0 : 1, use_ff);
        cudaStreamWaitEvent(ctx->aux, ctx->ev_in, 0);
        {
          KernelTimer kt(ctx, 2, ctx->aux);
          launch_volume<D, K, M>(ctx, ctx->p, U, U0, out, a, b, c, mode | 4, ctx->aux, vk);
        }
        cudaEventRecord(ctx->ev_vol, ctx->aux);
        if (!ctx->faces_first) faces(part == 0 ? 0 : 1, use_ff);
      }
      if (part == 1) {
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? TDG_OK : cuda_fail(e, "operator launch");
      }
      if (part == 2) faces(2, use_ff);
      cudaStreamWaitEvent(st, ctx->ev_vol, 0);
      KernelTimer kt(ctx, 3, st);
      const int64_t n2 = p.ne * (SN_of<M, D, K>() / 2);
      const int grid = int(n2 / 256 + 1 < 148 * 8 ? n2 / 256 + 1 : 148 * 8);
      k_fc_add<D, SN_of<M, D, K>(), Dims<D, K>::NEG><<<grid, 256, 0, st>>>(
          ctx->fc, p.egeo, p.ne, out, c, mode, 0, p.ne);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TDG_OK : cuda_fail(e, "operator launch");
  }
  if (part == 0) faces(0, use_ff);
  else if (part == 1) {
    faces(1, use_ff);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TDG_OK : cuda_fail(e, "operator launch");
  } else {
    faces(2, use_ff);
  }
  if (p.ne > 0 && (use_vm || use_tc)) {
    KernelTimer kt(ctx, 2, st);
    launch_volume<D, K, M>(ctx, ctx->p, U, U0, out, a, b, c, mode, st, vk);
  } else if (p.ne > 0) {
    KernelTimer kt(ctx, 2, st);
    if (use_v4) {
      using T = Vol4<D, K, M>;
      const int64_t grid = (p.ne + T::TE - 1) / T::TE;
      if constexpr (Vol4<D, K, M>::ok)
        k_volume4<D, K, M><<<unsigned(grid), T::THREADS, T::smem(), st>>>(p, U, ctx->fc, U0, out,
                                                                          a, b, c, mode);
    } else if (use_fv) {
      using T = FastVol<D, K, M>;
      const int64_t grid = (p.ne + T::TE - 1) / T::TE;
      if constexpr (fast_vol)
        k_volume_fast<D, K, M><<<unsigned(grid), T::TE, T::smem(), st>>>(p, U, ctx->fc, U0, out,
                                                                          a, b, c, mode);
    } else {
      constexpr int TE = VolumeTile<D, K, M>::TE;
      const int64_t grid = (p.ne + TE - 1) / TE;
      k_volume<D, K, M><<<unsigned(grid), kThreads, VolumeTile<D, K, M>::smem(p.nqv), st>>>(
          p, U, ctx->fc, U0, out, a, b, c, mode);
    }
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "operator launch");
}

// Host-to-host SSP-RK3 steps with per-step host copies, pipelined by
// element bands: step n's state is copied in band by band (each band's
// volume part and the faces whose bands have arrived start at once), and
// the final stage is finished and copied out band by band (the next step's
// copy-in of band k follows this step's copy-out of band k).  Same
// kernels, same per-face / per-element arithmetic and the same fixed-order
// face-slot sums as the unbanded step: bitwise the same results.
template <int D, int K, class M>
int host_steps(tdg_ctx* ctx, double* Uh, int64_t nsteps, double dt, cudaStream_t st) {
  const OpParams& p = ctx->p;
  constexpr bool fast_vol = FastVol<D, K, M>::ok, fast_face = FastFace<D, K, M>::ok;
  constexpr int SN = SN_of<M, D, K>();
  const int64_t rows = ctx->d.n_elements + ctx->d.n_ghost;
  const size_t n = size_t(rows) * SN;
  if (!ctx->hs_buf || ctx->hs_n < n) {
    if (ctx->hs_buf) cudaFree(ctx->hs_buf);
    ctx->hs_buf = nullptr;
    ctx->hs_n = 0;
    if (cudaMalloc(&ctx->hs_buf, 3 * n * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      return fail(TDG_E_CUDA, "cudaMalloc host-step buffers");
    }
    ctx->hs_n = n;
  }
  double* Ud = ctx->hs_buf;
  double* W1 = Ud + n;
  double* W2 = W1 + n;
  const int nb = ctx->n_bands;
  // volume part per band: the one-thread-per-element kernel, or the
  // transposed tensor-core one where that does not fit (2D k = 3: C3)
  constexpr bool tc_vol = TcVol<D, K, M>::ok;
  const bool band_tc = tc_vol && p.vtc != nullptr && (ctx->force_tc || !fast_vol);
  // faces per band: the register-resident kernel over face ranges (2D), or
  // the transposed tensor-core kernel over the band's face blocks (3D)
  constexpr bool tcf = TcFace<D, K, M>::ok && MmaFace<D, K, M>::ok;
  const bool band_tcf = D == 3 && tcf && p.ftc != nullptr && p.fblk != nullptr &&
                        p.fmma != nullptr && !ctx->no_tcf && !ctx->flip_mma &&
                        int(ctx->band_blk.size()) == nb + 1;
  const bool banded = nb > 1 && ctx->d.n_ghost == 0 && ctx->overlap &&
                      (D == 2 ? fast_face : band_tcf) && (fast_vol || band_tc) &&
                      p.nqf == Dims<D, K>::NQF && p.nqv == Dims<D, K>::NQV &&
                      !ctx->force_generic && (SN % 2 == 0);
  if (!banded) {  // plain per-step copies around the fused stages
    for (int64_t it = 0; it < nsteps; ++it) {
      cudaMemcpyAsync(Ud, Uh, n * sizeof(double), cudaMemcpyHostToDevice, st);
      int rc = ctx->impl.run(ctx, Ud, nullptr, W1, 0.0, 1.0, dt, 2, st);
      if (!rc) rc = ctx->impl.run(ctx, W1, Ud, W2, 0.75, 0.25, 0.25 * dt, 2, st);
      if (!rc) rc = ctx->impl.run(ctx, W2, Ud, Ud, 1.0 / 3.0, 2.0 / 3.0, (2.0 / 3.0) * dt, 2, st);
      if (rc) return rc;
      cudaMemcpyAsync(Uh, Ud, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TDG_OK : cuda_fail(e, "host steps");
  }
  if constexpr ((fast_vol || tc_vol) && (fast_face || tcf) && (SN % 2 == 0)) {
    auto ev_new = [](std::vector<cudaEvent_t>& v, int k) {
      while (int(v.size()) < k) {
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        v.push_back(e);
      }
    };
    if (!ctx->s_in[0]) {
      for (int i = 0; i < tdg_ctx::kCopyStreams; ++i) {
        cudaStreamCreateWithFlags(&ctx->s_in[i], cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ctx->s_out[i], cudaStreamNonBlocking);
      }
      // later stages first: the chain to the copy-out (and so to the next
      // copy-in) runs through stage 3, which must not queue behind the
      // next step's stage-1 work
      int lo = 0, hi = 0;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      for (int s = 0; s < 6; ++s) {
        const int pr = s < 2 ? lo : (s < 4 ? (lo + hi) / 2 : hi);
        cudaStreamCreateWithPriority(&ctx->hs_st[s], cudaStreamNonBlocking, pr);
      }
      cudaEventCreateWithFlags(&ctx->ev_s0, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ctx->ev_s1, cudaEventDisableTiming);
    }
    ev_new(ctx->ev_h2d, nb);
    ev_new(ctx->ev_d2h, nb);
    ev_new(ctx->ev_done, 3 * nb);
    ev_new(ctx->ev_vol_b, 3 * nb);
    const auto& be = ctx->band_elem;
    const auto& bf = ctx->band_face;
    const auto& bw = ctx->band_wall;
    // faces of band k: those straddling (k-1, k), those internal to k and
    // band k's walls; they read bands k-1 and k and write their slots
    auto faces_band = [&](int k, const double* Uin, cudaStream_t s) {
      if (D == 3) {
        run_faces_tc<D, K, M>(ctx, p, Uin, ctx->band_blk[k], ctx->band_blk[k + 1], bw[k],
                              bw[k + 1], s);
        return;
      }
      OpParams pp = p;
      const int64_t f0 = k > 0 ? bf[2 * k - 1] : 0, f1 = bf[2 * k + 1];
      pp.ifel = p.ifel + 2 * f0;
      pp.iflf = p.iflf + 2 * f0;
      pp.ifcode = p.ifcode + f0;
      pp.ifgeo = p.ifgeo + f0 * Dims<D, K>::NFG;
      pp.nif = f1 - f0;
      pp.bfel = p.bfel + bw[k];
      pp.bflf = p.bflf + bw[k];
      pp.bfcode = p.bfcode + bw[k];
      pp.bfgeo = p.bfgeo + bw[k];
      pp.nbf = bw[k + 1] - bw[k];
      if (pp.nif + pp.nbf > 0) run_faces<D, K, M>(ctx, pp, Uin, s, true);
    };
    auto volume_band = [&](int k, const double* Uin, const double* U0, double* out, double a,
                           double b, double c, cudaStream_t s) {
      OpParams pv = p;
      const int64_t e0 = be[k];
      pv.ne = be[k + 1] - e0;
      pv.egeo = p.egeo + e0 * Dims<D, K>::NEG;
      KernelTimer kt(ctx, 2, s);
      launch_volume<D, K, M>(ctx, pv, Uin + e0 * SN, U0 ? U0 + e0 * SN : nullptr, out + e0 * SN,
                             a, b, c, 2 | 4, s, band_tc ? 2 : 0);
    };
    auto fc_add = [&](int k, double* out, double c, cudaStream_t s) {
      KernelTimer kt(ctx, 3, s);
      const int64_t n2 = (be[k + 1] - be[k]) * (SN / 2);
      const int grid = int(n2 / 256 + 1 < 148 * 8 ? n2 / 256 + 1 : 148 * 8);
      k_fc_add<D, SN, Dims<D, K>::NEG><<<grid, 256, 0, s>>>(ctx->fc, p.egeo, p.ne, out, c, 2,
                                                            be[k], be[k + 1]);
    };
    // Wavefront over (stage, band).  Stage s of band k needs stage s-1 of
    // bands k-1..k+1 (its faces read the neighbours); the copy-in of band k
    // for step n+1 needs only the copy-out of band k of step n, so the copy
    // engines stream continuously while the three stages trail behind.
    // Every write-after-read on U / W1 / W2 / the slot buffer is ordered by
    // these same edges (the readers of a band finish before the band's next
    // slot sum, which precedes its copy-out, which precedes its next copy-in).
    double* X[3] = {Ud, W1, W2};
    double* Y[3] = {W1, W2, Ud};
    const double* Z[3] = {nullptr, Ud, Ud};
    const double ca[3] = {0.0, 0.75, 1.0 / 3.0}, cb[3] = {1.0, 0.25, 2.0 / 3.0};
    const double cc[3] = {dt, 0.25 * dt, (2.0 / 3.0) * dt};
    cudaEventRecord(ctx->ev_s0, st);
    const int ncs = ctx->copy_streams < 1 ? 1
                    : (ctx->copy_streams > tdg_ctx::kCopyStreams ? tdg_ctx::kCopyStreams
                                                                 : ctx->copy_streams);
    auto cin = [&](int k) { return ctx->s_in[k % ncs]; };
    auto cout = [&](int k) { return ctx->s_out[k % ncs]; };
    for (int i = 0; i < ncs; ++i) cudaStreamWaitEvent(ctx->s_in[i], ctx->ev_s0, 0);
    for (auto s : ctx->hs_st) cudaStreamWaitEvent(s, ctx->ev_s0, 0);
    for (int64_t it = 0; it < nsteps; ++it) {
      for (int k = 0; k < nb; ++k) {
        if (it > 0) cudaStreamWaitEvent(cin(k), ctx->ev_d2h[k], 0);
        const size_t o = size_t(be[k]) * SN, m = size_t(be[k + 1] - be[k]) * SN;
        cudaMemcpyAsync(Ud + o, Uh + o, m * sizeof(double), cudaMemcpyHostToDevice, cin(k));
        cudaEventRecord(ctx->ev_h2d[k], cin(k));
      }
      for (int s = 0; s < 3; ++s) {
        cudaStream_t sf = ctx->hs_st[2 * s], sv = ctx->hs_st[2 * s + 1];
        auto ready = [&](int k) { return s == 0 ? ctx->ev_h2d[k] : ctx->ev_done[(s - 1) * nb + k]; };
        for (int k = 0; k < nb; ++k) {
          cudaStreamWaitEvent(sv, ready(k), 0);
          volume_band(k, X[s], Z[s], Y[s], ca[s], cb[s], cc[s], sv);
          cudaEventRecord(ctx->ev_vol_b[s * nb + k], sv);
        }
        auto finish = [&](int k) {  // all faces touching band k are done
          cudaStreamWaitEvent(sf, ctx->ev_vol_b[s * nb + k], 0);
          fc_add(k, Y[s], cc[s], sf);
          cudaEventRecord(ctx->ev_done[s * nb + k], sf);
          if (s == 2) {
            cudaStreamWaitEvent(cout(k), ctx->ev_done[s * nb + k], 0);
            const size_t o = size_t(be[k]) * SN, m = size_t(be[k + 1] - be[k]) * SN;
            cudaMemcpyAsync(Uh + o, Ud + o, m * sizeof(double), cudaMemcpyDeviceToHost,
                            cout(k));
            cudaEventRecord(ctx->ev_d2h[k], cout(k));
          }
        };
        for (int k = 0; k < nb; ++k) {
          cudaStreamWaitEvent(sf, ready(k), 0);
          faces_band(k, X[s], sf);
          if (k > 0) finish(k - 1);
        }
        finish(nb - 1);
      }
    }
    // join: every stream's tail back onto the caller's stream
    auto join = [&](cudaStream_t s) {
      cudaEventRecord(ctx->ev_s1, s);
      cudaStreamWaitEvent(st, ctx->ev_s1, 0);
    };
    for (int i = 0; i < ncs; ++i) {
      join(ctx->s_in[i]);
      join(ctx->s_out[i]);
    }
    for (cudaStream_t s : ctx->hs_st) join(s);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? TDG_OK : cuda_fail(e, "host steps");
}

// constant-memory copies of the reference-element face tables used by the
// register-resident face kernel (same for every mesh of one (d, k))
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
  return TDG_OK;
}

template <int D, int K, class M>
Impl make_impl() {
  return Impl{&configure<D, K, M>, &run<D, K, M>, &host_steps<D, K, M>, &upload_const<D, K, M>,
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

// Register-resident operator kernels for the small-table cases (2D, and
// any (d, k, model) whose per-lane working set fits in registers).
//
// k_faces_fast  one lane per (face, species): a warp holds 32/S faces
//               per group and loops over groups (grid-stride);
//               the S lanes of a face read the face's two contiguous
//               S*nb coefficient blocks coalesced, evaluate u and d_n u
//               at all face points in registers, exchange the few values
//               the species coupling needs (LLF wave speed, taxis flux)
//               with warp shuffles, and add the face's two contribution
//               blocks to the elements' face-sum rows (one colour
//               segment per launch: no element is touched twice).  Interior, Dirichlet-mirror and prescribed-flux
//               wall faces share the kernel (face index >= nif: wall).
//               Face tables (all (lf, perm) signatures, < 11 KB for 2D
//               k <= 3) live in shared memory; faces are sorted by
//               signature, so a warp's table reads are broadcasts.
// k_volume_fast one thread per element: the element's S*nb coefficients
//               sit in registers; volume tables are shared-memory
//               broadcasts; all global traffic (U, U0, the face-sum
//               tile, the output) is staged through shared memory so
//               every HBM access is a coalesced tile.
#pragma once

#include "common.cuh"
#include "kernels.cuh"
#include "models.cuh"

// A/B builds: resident CTAs per SM the signature-run face kernel is
// compiled for (0 = the default of its struct)
#ifndef TDG_SIG_MINB
#define TDG_SIG_MINB 0
#endif
#ifndef TDG_SIG_NARROW
#define TDG_SIG_NARROW 0
#endif
// signature-run kernel: 0 / 1 pin the synchronous / cp.async-staged variant
// (A/B builds); default: by state size against the L2
#ifndef TDG_SIG_FORCE_ASYNC
#define TDG_SIG_FORCE_ASYNC -1
#endif
// k_volume_fast: tables from constant memory instead of shared memory
#ifndef TDG_VOL_CONST
#define TDG_VOL_CONST 1
#endif
#ifndef TDG_VOL_MINB
#define TDG_VOL_MINB 0
#endif

namespace tdg {

template <int D, int K, class M>
struct FastFace {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF, NT = Dm::NT;
  static constexpr int FPW = 32 / S;          // faces per warp
  static constexpr int WARPS = 4;
  static constexpr int FPC = FPW * WARPS;     // faces per CTA
  static constexpr int TB = NT * F * NB, TG = NT * F * NB * D, TP = NT * F * F;
  static constexpr int TAB = (TB + TG + TP + F + 1) & ~1;
  static constexpr int NCV = 1 + M::NFX;
  // per-face scratch: normal-derivative tables (2 sides), the species
  // transpose (u_in, u_out, avg d_n u at every point) and the coupled
  // per-point results (wave speed, flux normals)
  // species-transpose rows padded to an odd stride XS and the per-face
  // scratch stride PF = 6 (mod 16) doubles: with 5-6 faces per warp the
  // transposed stores and the per-point physics loads stay 2-way at most
  // (bank-conflict search over the access patterns; ncu showed 6-way)
  static constexpr int XS = S | 1;
  static constexpr int PF0 = (2 * F * NB + 3 * XS * F + F * NCV + 1) & ~1;
  static constexpr int PF = PF0 + ((6 - PF0 % 16) + 16) % 16;
  static constexpr size_t smem() { return size_t(TAB + WARPS * FPW * PF) * 8; }
  static constexpr bool ok = F <= 8 && S >= 3 && S <= 8 && NB <= 10 && smem() <= 100 * 1024;
  static constexpr int MINB = NB <= 6 ? 4 : 3;  // register budget: 128 / 168
};

// Per-signature trace tables B, lifting tables Pw and face weights of the
// register-resident face kernel in constant memory: warp-uniform indexed
// LDC reads go through the constant cache instead of the L1TEX data pipe,
// which the kernel saturates (ncu: l1tex throughput ~90%).  Reference-element
// data: identical for every mesh of one (d, k) at the default face rule.
template <int D, int K>
struct FaceConstLayout {
  static constexpr int NT = Dims<D, K>::NT, F = Dims<D, K>::NQF, NB = Dims<D, K>::NB;
  static constexpr int OB = 0, OP = NT * F * NB, OW = OP + NT * F * F, N = OW + F;
};
template <int D, int K>
__constant__ double c_face_tab[FaceConstLayout<D, K>::N];

template <int NB>
__device__ __forceinline__ void load_row(const double* __restrict__ src, double* dst) {
  if constexpr (NB % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int i = 0; i < NB / 2; ++i) {
      const double2 v = __ldg(s2 + i);
      dst[2 * i] = v.x;
      dst[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) dst[i] = __ldg(src + i);
  }
}

// row of NB doubles from shared memory, 16-byte loads when NB is even
// (callers keep every row 16-byte aligned)
template <int NB>
__device__ __forceinline__ void smem_row(const double* src, double* dst) {
  if constexpr (NB % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int i = 0; i < NB / 2; ++i) {
      const double2 v = s2[i];
      dst[2 * i] = v.x;
      dst[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) dst[i] = src[i];
  }
}

template <int NB>
__device__ __forceinline__ void store_row(double* dst, const double* v) {
  if constexpr (NB % 2 == 0) {
    double2* d2 = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int i = 0; i < NB / 2; ++i) d2[i] = make_double2(v[2 * i], v[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) dst[i] = v[i];
  }
}

// 32-byte global accesses (sm_100 LDG/STG.256): a row of NB = 4m + 2
// doubles starting at a 16-byte boundary is m 32-byte pieces plus one
// 16-byte piece, in either order depending on its 32-byte alignment.  The
// face kernel's lanes read / write such rows side by side, so fewer and
// wider accesses cut the L1 wavefronts of its (saturated) data pipe.
// coherent 32-byte load (rows this kernel also writes)
__device__ __forceinline__ void ld256c(const double* p, double* d) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void st256(double* p, const double* d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(d[0]), "d"(d[1]), "d"(d[2]),
               "d"(d[3])
               : "memory");
}

template <int NB, bool NC = true>
__device__ __forceinline__ void load_row_wide(const double* src, double* dst) {
  if constexpr (NB % 4 == 2) {
    constexpr int M = NB / 4;
    const bool odd = (reinterpret_cast<uintptr_t>(src) & 16u) != 0;
    const double* p32 = src + (odd ? 2 : 0);
    const double* p16 = src + (odd ? 0 : 4 * M);
    double w[4 * M];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      if constexpr (NC) ld256(p32 + 4 * k, w + 4 * k);
      else ld256c(p32 + 4 * k, w + 4 * k);
    }
    const double2 h = NC ? __ldg(reinterpret_cast<const double2*>(p16))
                         : *reinterpret_cast<const double2*>(p16);
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const double ev = i < 4 * M ? w[i < 4 * M ? i : 0] : (i == 4 * M ? h.x : h.y);
      const double od = i < 2 ? (i == 0 ? h.x : h.y) : w[i >= 2 ? i - 2 : 0];
      dst[i] = odd ? od : ev;
    }
  } else if constexpr (NC) {
    load_row<NB>(src, dst);
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) dst[i] = src[i];
  }
}

template <int NB>
__device__ __forceinline__ void store_row_wide(double* dst, const double* v) {
  if constexpr (NB % 4 == 2) {
    constexpr int M = NB / 4;
    const bool odd = (reinterpret_cast<uintptr_t>(dst) & 16u) != 0;
    double* p32 = dst + (odd ? 2 : 0);
    double* p16 = dst + (odd ? 0 : 4 * M);
    double w[4 * M];
#pragma unroll
    for (int i = 0; i < 4 * M; ++i) w[i] = odd ? v[i + 2] : v[i];
#pragma unroll
    for (int k = 0; k < M; ++k) st256(p32 + 4 * k, w + 4 * k);
    *reinterpret_cast<double2*>(p16) =
        odd ? make_double2(v[0], v[1]) : make_double2(v[4 * M], v[4 * M + 1]);
  } else {
    store_row<NB>(dst, v);
  }
}

// face-sum row update: the element's first face side writes, later ones add
template <int NB>
__device__ __forceinline__ void acc_row_wide(double* dst, const double* v, bool first) {
  if (first) {
    store_row_wide<NB>(dst, v);
    return;
  }
  double o[NB];
  load_row_wide<NB, false>(dst, o);
#pragma unroll
  for (int i = 0; i < NB; ++i) o[i] += v[i];
  store_row_wide<NB>(dst, o);
}

template <int D, int K, int NB>
__device__ __forceinline__ void const_row(int off, double* dst) {
#pragma unroll
  for (int i = 0; i < NB; ++i) dst[i] = c_face_tab<D, K>[off + i];
}

template <int D, int NB>
struct FaceRec {
  int code, ein, eout;
  bool active, wall;
  double jn[2][D], sfac, h, idi, ido;
  double ci[NB], co[NB];
};

// Face record and the two coefficient rows of species s for warp-group gw.
// Interior groups load unconditionally from a clamped face index (lanes
// past the end recompute the last face and never store), so the common
// path has no predicated loads or zero fills.
template <int D, int K, class M>
__device__ __forceinline__ void load_face_group(const OpParams& p, const double* __restrict__ U,
                                                int64_t gw, int64_t wi, int grp, int s, bool lane_ok,
                                                FaceRec<D, Dims<D, K>::NB>& r) {
  using T = FastFace<D, K, M>;
  constexpr int NB = T::NB, SN = T::SN, FPW = T::FPW, NFG = Dims<D, K>::NFG;
  r.wall = gw >= wi;
  if (!r.wall) {
    const int64_t f = gw * FPW + grp;
    r.active = lane_ok && f < p.nif;
    const int64_t fc = f < p.nif ? f : p.nif - 1;
    r.code = __ldg(p.ifcode + fc);
    const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + fc);
    r.ein = el.x;
    r.eout = el.y;
    const double* g = p.ifgeo + fc * NFG;
    if constexpr (NFG == 8) {  // 2D: the 64-byte record in two 32-byte loads
      double w[8];
      ld256(g, w);
      ld256(g + 4, w + 4);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        r.jn[0][a] = w[a];
        r.jn[1][a] = w[D + a];
      }
      r.sfac = w[2 * D];
      r.h = w[2 * D + 1];
      r.idi = w[2 * D + 2];
      r.ido = w[2 * D + 3];
    } else {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        r.jn[0][a] = __ldg(g + a);
        r.jn[1][a] = __ldg(g + D + a);
      }
      r.sfac = __ldg(g + 2 * D);
      r.h = __ldg(g + 2 * D + 1);
      r.idi = __ldg(g + 2 * D + 2);
      r.ido = __ldg(g + 2 * D + 3);
    }
    load_row_wide<NB>(U + int64_t(r.ein) * SN + s * NB, r.ci);
    // mirror faces (Dirichlet models only) have no outside element
    const int eo = (M::kMirror && r.eout < 0) ? r.ein : r.eout;
    load_row_wide<NB>(U + int64_t(eo) * SN + s * NB, r.co);
    return;
  }
  const int64_t b = (gw - wi) * FPW + grp;
  r.active = lane_ok && b < p.nbf;
  const int64_t bc = b < p.nbf ? b : p.nbf - 1;
  r.code = __ldg(p.bfcode + bc);
  r.ein = __ldg(p.bfel + bc);
  r.eout = -1;
  r.sfac = __ldg(p.bfgeo + bc);
  r.h = 1.0;
  r.idi = r.ido = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) r.jn[0][a] = r.jn[1][a] = 0.0;
  load_row<NB>(U + int64_t(r.ein) * SN + s * NB, r.ci);
#pragma unroll
  for (int i = 0; i < NB; ++i) r.co[i] = 0.0;
}

template <int D, int K, class M>
__global__ void __launch_bounds__(128, FastFace<D, K, M>::MINB)
k_faces_fast(OpParams p, const double* __restrict__ U, double* __restrict__ ACC, int64_t ngroups) {
  using T = FastFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, FPW = T::FPW, NCV = T::NCV;
  [[maybe_unused]] constexpr int NFG = Dims<D, K>::NFG;
  extern __shared__ __align__(16) double sm[];
  double* tB = sm;
  double* tG = tB + T::TB;
  double* tP = tG + T::TG;
  double* tw = tP + T::TP;
  for (int i = threadIdx.x; i < T::TB; i += 128) tB[i] = p.fB[i];
  for (int i = threadIdx.x; i < T::TG; i += 128) tG[i] = p.fG[i];
  for (int i = threadIdx.x; i < T::TP; i += 128) tP[i] = p.fPw[i];
  if (threadIdx.x < F) tw[threadIdx.x] = p.fw[threadIdx.x];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / S, s = lane - grp * S, base = grp * S;
  const bool lane_ok = grp < FPW;
  double* scratch = sm + T::TAB + (warp * FPW + (lane_ok ? grp : 0)) * T::PF;
  double* dph = scratch;                    // [2][F][NB]
  double* xch = dph + 2 * F * NB;           // [3][F][XS]
  double* cvs = xch + 3 * T::XS * F;        // [F][NCV]

  const int64_t wi = (p.nif + FPW - 1) / FPW;
  // grid-stride over face groups: the tables above are staged once per CTA
  for (int64_t gw = int64_t(blockIdx.x) * T::WARPS + warp; gw < ngroups;
       gw += int64_t(gridDim.x) * T::WARPS) {
  FaceRec<D, NB> cur;
  load_face_group<D, K, M>(p, U, gw, wi, grp, s, lane_ok, cur);
  const bool wall = cur.wall, active = cur.active;
  if (!__any_sync(0xffffffffu, active)) continue;  // warp-uniform
  int code = cur.code;
  // lanes without a face copy lane 0's code word so every warp-uniform
  // branch below stays uniform
  {
    const int c0 = __shfl_sync(0xffffffffu, code, 0);
    if (!active) code = c0;
  }
  const int ein = cur.ein, eout = cur.eout;
  const double sfac = cur.sfac, h = cur.h, idi = cur.idi, ido = cur.ido;
  double jn[2][D];
#pragma unroll
  for (int a2 = 0; a2 < D; ++a2) {
    jn[0][a2] = cur.jn[0][a2];
    jn[1][a2] = cur.jn[1][a2];
  }
  const bool mirror = code_mirror(code);
  const int tin = code_tin(code), tout = code_tout(code);
  const bool two = active && !wall && !mirror;
  double ci[NB], co[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    ci[i] = cur.ci[i];
    co[i] = cur.co[i];
  }
  const double* Bi = tB + tin * F * NB;
  const double* Bo = tB + tout * F * NB;
  using CL = FaceConstLayout<D, K>;
  const int ciB = CL::OB + tin * F * NB, coB = CL::OB + tout * F * NB;

  double ri[NB], ro[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) ri[i] = ro[i] = 0.0;

  if (!wall) {
    // per-face normal-derivative test tables dphi.n = G . (Jinv n), shared
    // by the S lanes of the face
    // lane s builds modes i = s, s+S, ... of both sides' tables
    if (lane_ok) {
#pragma unroll
      for (int k = 0; k < (NB + S - 1) / S; ++k) {
        const int i = s + k * S;
        if (i < NB) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const double* g = tG + ((side ? tout : tin) * F * NB + i) * D;
#pragma unroll
            for (int q = 0; q < F; ++q) {
              double v = 0.0;
#pragma unroll
              for (int a = 0; a < D; ++a) v = fma(g[q * NB * D + a], jn[side][a], v);
              dph[(side * F + q) * NB + i] = v;
            }
          }
        }
      }
    }
    __syncwarp();
    const double* dpi = dph;
    const double* dpo = dph + F * NB;
    double dU[F], gav[F];
#pragma unroll
    for (int q = 0; q < F; ++q) {
      double u = 0.0, v = 0.0, x = 0.0, y = 0.0;
      double bi[NB], bo[NB], di[NB], dq[NB];
      smem_row<NB>(Bi + q * NB, bi);
      smem_row<NB>(Bo + q * NB, bo);
      smem_row<NB>(dpi + q * NB, di);
      smem_row<NB>(dpo + q * NB, dq);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        u = fma(bi[i], ci[i], u);
        x = fma(di[i], ci[i], x);
        v = fma(bo[i], co[i], v);
        y = fma(dq[i], co[i], y);
      }
      if constexpr (M::kMirror) {
        if (mirror) {
          v = 2.0 * M::mirror_value(p.P, s) - u;
          y = x;
        }
      }
      dU[q] = u - v;
      gav[q] = 0.5 * (x + y);
      // point values go straight to the species transpose (not kept)
      if constexpr (M::kConv) {
        if (lane_ok) {
          // [kind][q][species]: the S lanes of a face store consecutive
          // doubles (conflict-free with the per-face scratch stride)
          xch[(0 * F + q) * T::XS + s] = u;
          xch[(1 * F + q) * T::XS + s] = v;
          xch[(2 * F + q) * T::XS + s] = gav[q];
        }
      }
    }
    const double As = p.A[s];
    // coupled convective physics once per face point (smem transpose)
    double conv[F];
#pragma unroll
    for (int q = 0; q < F; ++q) conv[q] = 0.0;
    if constexpr (M::kConv) {
      __syncwarp();
      if (lane_ok) {
        for (int q = s; q < F; q += S) {
          const double* xq = xch + q * T::XS;
          auto fetch = [xq](int kind, int sp) { return xq[kind * F * T::XS + sp]; };
          M::face_point(p.P, fetch, cvs + q * NCV);
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < F; ++q) {
        double c = 0.5 * cvs[q * NCV] * dU[q];
#pragma unroll
        for (int k = 0; k < M::NFX; ++k)
          if (s == k) c = fma(0.5, cvs[q * NCV + 1 + k], c);
        conv[q] = c;
      }
    }
    // penalty A_hat . n (operator.py:336-357), lifting on the needed side(s)
    double qv[F];
#pragma unroll
    for (int q = 0; q < F; ++q) qv[q] = 0.0;
    if (p.scheme == IP) {
      const double c = p.eta / h * As;
#pragma unroll
      for (int q = 0; q < F; ++q) qv[q] = c * dU[q];
    } else if (p.scheme != BO) {
      const bool br2 = p.scheme == BR2;
      const bool use_in = mirror || br2 || code_minus_in(code);
      const bool use_out = !mirror && (br2 || !code_minus_in(code));
      const double wside = (br2 && !mirror) ? 0.5 : 1.0;
      // -fac A rho with rho = -1/2 sfac / detJ (Pw dU)
      const double fac = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * As * wside * 0.5 * sfac;
      if (use_in) {
        const int pw0 = CL::OP + tin * F * F;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          double a = 0.0;
#pragma unroll
          for (int pp = 0; pp < F; ++pp) a = fma(c_face_tab<D, K>[pw0 + q * F + pp], dU[pp], a);
          qv[q] = fma(fac * idi, a, qv[q]);
        }
      }
      if (use_out) {
        const int pw0 = CL::OP + tout * F * F;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          double a = 0.0;
#pragma unroll
          for (int pp = 0; pp < F; ++pp) a = fma(c_face_tab<D, K>[pw0 + q * F + pp], dU[pp], a);
          qv[q] = fma(fac * ido, a, qv[q]);
        }
      }
    }
    // projection onto both sides' test functions
#pragma unroll
    for (int q = 0; q < F; ++q) {
      const double wq = c_face_tab<D, K>[CL::OW + q] * sfac;
      const double Y = wq * (As * gav[q] - (qv[q] + conv[q]));
      const double X = wq * 0.5 * p.adj * As * dU[q];
      double bi[NB], bo[NB], di[NB], dq[NB];
      smem_row<NB>(Bi + q * NB, bi);
      smem_row<NB>(Bo + q * NB, bo);
      smem_row<NB>(dpi + q * NB, di);
      smem_row<NB>(dpo + q * NB, dq);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        ri[i] = fma(Y, bi[i], fma(X, di[i], ri[i]));
        ro[i] = fma(-Y, bo[i], fma(X, dq[i], ro[i]));
      }
    }
  } else {
    // prescribed wall flux: only the gate species' trace is needed
    const int tag = code_tag(code);
#pragma unroll
    for (int q = 0; q < F; ++q) {
      double u = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) u = fma(Bi[q * NB + i], ci[i], u);
      const double c1 = __shfl_sync(0xffffffffu, u, base + M::WALL_SP);
      const double Y = -tw[q] * sfac * M::wall_lane(p.P, tag, s, c1);
#pragma unroll
      for (int i = 0; i < NB; ++i) ri[i] = fma(Y, Bi[q * NB + i], ri[i]);
    }
  }
  if (active) {
    acc_row_wide<NB>(ACC + int64_t(ein) * SN + s * NB, ri, code_first_in(code));
    if (two && !code_skip_out(code))
      acc_row_wide<NB>(ACC + int64_t(eout) * SN + s * NB, ro, code_first_out(code));
  }
  __syncwarp();  // the warp's scratch is rewritten by the next group
  }
}

// ------------------------------------------------- signature-run face kernel
//
// k_faces_sig  the interior faces of one run of a colour segment that share
//              their (inside, outside) trace-table signature.  The run's
//              tables (B, reference gradients, Pw of both sides, weights)
//              travel as a __grid_constant__ kernel parameter, so every
//              table entry reaches its DFMA through the constant bank /
//              uniform registers: no table loads on the L1 data path at
//              all.  k_faces_fast reads one 16-byte shared-memory row piece
//              per two DFMAs and is bound by the L1 return path (ncu:
//              l1tex 80-88%, FP64 pipe 32-35%).
//              NG = D: the normal derivative is taken after the contraction
//              (jn . (G c) instead of (G jn) . c), D-1 more DFMAs per entry
//              but no per-face table.  NG = 1: every face of the run has
//              the same Jinv n on both sides (structured meshes with
//              exactly representable cell sizes), and the host folds it
//              into the tables (G holds d_n phi).
//              Same lane mapping, physics transpose, penalty and face-sum
//              updates as k_faces_fast.  Structured and jittered triangle
//              meshes have one signature pair per colour segment.  Groups
//              past the interior ones are the segment's prescribed-flux
//              walls (k_faces_fast's wall branch, trace rows from global
//              memory), so a segment is one launch.
template <int D, int K, int NG>
struct FaceSigTab {
  static constexpr int F = Dims<D, K>::NQF, NB = Dims<D, K>::NB;
  double B[2][F][NB];      // trace tables: inside / outside signature
  double G[2][F][NB][NG];  // reference gradients (NG = D) or d_n phi (NG = 1) at the face points
  double Pw[2][F][F];      // lifting tables
  double w[F];             // face weights
};

template <int D, int K, class M>
struct SigFace {
  using T = FastFace<D, K, M>;
  static constexpr int NB = T::NB, S = T::S, F = T::F, XS = T::XS, NCV = T::NCV, FPW = T::FPW;
  static constexpr int WARPS = 4;
  // per-face scratch: the species transpose and the coupled point results;
  // stride = 6 (mod 16) doubles as in k_faces_fast
  static constexpr int PF0 = (3 * XS * F + F * NCV + 1) & ~1;
  static constexpr int PF = PF0 + ((6 - PF0 % 16) + 16) % 16;
  // cp.async row staging per lane: two rows, lane stride = 2 (mod 4) doubles
  // (conflict-free 16-byte reads)
  static constexpr int RHALF = (NB + 1) & ~1;
  static constexpr int RST = 2 * RHALF + ((2 * RHALF) % 4 == 2 ? 0 : 2);
  static constexpr bool ok = T::ok && !M::kMirror && D == 2 &&
                             sizeof(FaceSigTab<D, K, D>) + sizeof(OpParams) <= 16 * 1024;
  // k <= 2: 5 CTAs (20 warps) per SM at 96 registers; k = 3: 4 CTAs at
  // 128 (no spills).  Measured at C2 / jittered C3-quarter sizes: 3 CTAs
  // - / 626 us, 4: 79 / 576, 5: 78 / 594, 6: 76 / 672
  static constexpr int MINB = TDG_SIG_MINB > 0 ? TDG_SIG_MINB : (NB <= 6 ? 5 : 4);
};

// row accesses of the signature-run kernel: the 32-byte pieces of
// k_faces_fast (fewer L1 wavefronts, alignment selects) or plain 16-byte
// pieces (TDG_SIG_NARROW: fewer instructions)
template <int NB>
__device__ __forceinline__ void sig_load_row(const double* src, double* dst) {
#if TDG_SIG_NARROW
  load_row<NB>(src, dst);
#else
  load_row_wide<NB>(src, dst);
#endif
}
template <int NB>
__device__ __forceinline__ void sig_acc_row(double* dst, const double* v, bool first) {
#if TDG_SIG_NARROW
  if (!first) {
    double o[NB];
    smem_row<NB>(dst, o);  // plain (coherent) 16-byte loads
#pragma unroll
    for (int i = 0; i < NB; ++i) o[i] += v[i];
    store_row<NB>(dst, o);
  } else {
    store_row<NB>(dst, v);
  }
#else
  acc_row_wide<NB>(dst, v, first);
#endif
}

#define TDG_SIG_ASYNC 0
#define TDG_SIG_KERNEL k_faces_sig
#include "kernels_sig_body.cuh"
#undef TDG_SIG_ASYNC
#undef TDG_SIG_KERNEL
#define TDG_SIG_ASYNC 1
#define TDG_SIG_KERNEL k_faces_sig_async
#include "kernels_sig_body.cuh"
#undef TDG_SIG_ASYNC
#undef TDG_SIG_KERNEL

// ------------------------------------------------------------------ volume

// Coalesced copy of nt contiguous rows of SN doubles between global
// memory and a padded shared tile (row stride SNP, odd => conflict-free
// per-thread row access).  Uses 16-byte accesses when SN is even (the
// tile base is 16-byte aligned because every row offset e0*SN*8 is).
template <int SN, int SNP, int NTH>
__device__ __forceinline__ void tile_load(const double* __restrict__ src, double* dst, int nt) {
  constexpr int TE = NTH;  // one row per thread in the fast volume kernel
  if (SN % 2 == 0 && nt == TE) {
    // full tile: issue every load of this thread before any store
    constexpr int H = SN / 2, PER = (TE * H) / NTH;
    const double2* s2 = reinterpret_cast<const double2*>(src);
    double2 v[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) v[k] = __ldcs(s2 + threadIdx.x + k * NTH);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = threadIdx.x + k * NTH, e = idx / H, r = 2 * (idx - e * H);
      dst[e * SNP + r] = v[k].x;
      dst[e * SNP + r + 1] = v[k].y;
    }
    return;
  }
  if constexpr (SN % 2 == 0) {
    const double2* s2 = reinterpret_cast<const double2*>(src);
    constexpr int H = SN / 2;
    for (int idx = threadIdx.x; idx < nt * H; idx += NTH) {
      const int e = idx / H, r = 2 * (idx - e * H);
      const double2 v = __ldcs(s2 + idx);
      dst[e * SNP + r] = v.x;
      dst[e * SNP + r + 1] = v.y;
    }
  } else {
    for (int idx = threadIdx.x; idx < nt * SN; idx += NTH) {
      const int e = idx / SN, r = idx - e * SN;
      dst[e * SNP + r] = __ldcs(src + idx);
    }
  }
}

template <int SN, int SNP, int NTH>
__device__ __forceinline__ void tile_store(double* dst, const double* src, int nt) {
  if constexpr (SN % 2 == 0) {
    double2* d2 = reinterpret_cast<double2*>(dst);
    constexpr int H = SN / 2;
    for (int idx = threadIdx.x; idx < nt * H; idx += NTH) {
      const int e = idx / H, r = 2 * (idx - e * H);
      d2[idx] = make_double2(src[e * SNP + r], src[e * SNP + r + 1]);
    }
  } else {
    for (int idx = threadIdx.x; idx < nt * SN; idx += NTH) {
      const int e = idx / SN, r = idx - e * SN;
      dst[idx] = src[e * SNP + r];
    }
  }
}

template <int D, int K, class M>
struct FastVol {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, SNP = SN | 1, Q = Dm::NQV;
  static constexpr int NSYM = Dm::NSYM, NEG = Dm::NEG;
  // 64 elements (2 warps) per CTA: 4 small CTAs per SM desynchronise
  // their load / compute / store phases better than 2 large ones
  static constexpr int TE = 64;
  static constexpr int TPHI = Q * NB, TGR = Q * NB * D, TKS = NSYM * NB * NB;
  static constexpr int TAB = TPHI + TGR + Q + TKS;
  static constexpr bool ok = SN <= 36 && TAB * 8 <= 24 * 1024;
  // CTAs/SM the register budget targets.  Measured with the tables in
  // constant memory, C2 (p = 2) / 1024x256 p = 1: 4 CTAs 55.5 / 74.4 us,
  // 5-6: 51.5 / 74.2, 7-8: 60.2 (spills) / 70.1; 3D instantiations stay at 4
  static constexpr int MINB = TDG_VOL_MINB > 0 ? TDG_VOL_MINB : (D == 3 ? 4 : (NB <= 3 ? 8 : 5));
  static constexpr int STAB = TDG_VOL_CONST ? 0 : TAB;  // tables staged in shared memory
  static constexpr size_t smem() { return size_t(STAB + 2 * TE * SNP) * 8; }
};

// Volume tables (Phi, grad Phi, weights, stiffness blocks at the default
// rule) in constant memory: reference-element data, identical for every
// mesh of one (d, k).  The quadrature loop's table reads become
// uniform-register operands (LDCU with a uniform index) instead of
// shared-memory broadcasts.
template <int D, int K>
struct VolConstLayout {
  using Dm = Dims<D, K>;
  static constexpr int NSYM = D * (D + 1) / 2;
  static constexpr int OPHI = 0, OGR = Dm::NQV * Dm::NB, OW = OGR + Dm::NQV * Dm::NB * D,
                       OKS = OW + Dm::NQV, N = OKS + NSYM * Dm::NB * Dm::NB;
  static constexpr bool fits = N * 8 <= 24 * 1024;
};
template <int D, int K>
__constant__ double c_vol_tab[VolConstLayout<D, K>::fits ? VolConstLayout<D, K>::N : 1];

template <int D, int K, class M>
__global__ void __launch_bounds__(FastVol<D, K, M>::TE, FastVol<D, K, M>::MINB)
k_volume_fast(OpParams p, const double* __restrict__ U, const double* ACC,
              const double* U0, double* out, double ca, double cb, double cc, int mode) {
  using T = FastVol<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, SNP = T::SNP, Q = T::Q, TE = T::TE;
  constexpr int NEG = T::NEG, NSYM = T::NSYM;
  extern __shared__ __align__(16) double sm[];
#if TDG_VOL_CONST
  using VL = VolConstLayout<D, K>;
  const double* tphi = c_vol_tab<D, K> + VL::OPHI;
  const double* tgr = c_vol_tab<D, K> + VL::OGR;
  const double* tw = c_vol_tab<D, K> + VL::OW;
  const double* tks = c_vol_tab<D, K> + VL::OKS;
#else
  double* tphi = sm;
  double* tgr = tphi + T::TPHI;
  double* tw = tgr + T::TGR;
  double* tks = tw + Q;
#endif
  double* bufA = sm + T::STAB;
  double* bufB = bufA + TE * SNP;
  // ACC: the face-sum rows (null: no faces); ACC and U0 may alias out
  mode &= 3;
  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * TE;
  const int nt = int(p.ne - e0 < TE ? p.ne - e0 : TE);

#if !TDG_VOL_CONST
  for (int i = tid; i < T::TPHI; i += TE) tphi[i] = p.phi[i];
  for (int i = tid; i < T::TGR; i += TE) tgr[i] = p.grad[i];
  for (int i = tid; i < Q; i += TE) tw[i] = p.wv[i];
  for (int i = tid; i < T::TKS; i += TE) tks[i] = p.ks[i];
#endif
  // the face-sum tile and U0 are consumed after the quadrature loop: start
  // pulling them into L2 now (bulk prefetch, one thread per tile)
  if (tid <= 1) {
    const double* src = tid == 0 ? ACC + e0 * SN : U0 + e0 * SN;
    if ((tid == 0 && ACC != nullptr) || (tid == 1 && mode == 2 && ca != 0.0 && U0 != nullptr)) {
      const unsigned bytes = unsigned(nt) * SN * 8u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes & ~15u) : "memory");
    }
  }
  // coalesced tile load of U (owned rows are contiguous)
  tile_load<SN, SNP, TE>(U + e0 * SN, bufA, nt);
  __syncthreads();
  const bool act = tid < nt;
  double c[SN];
#pragma unroll
  for (int r = 0; r < SN; ++r) c[r] = bufA[tid * SNP + r];
  double ge[NEG];
#pragma unroll
  for (int k = 0; k < NEG; ++k) ge[k] = act ? __ldg(p.egeo + (e0 + tid) * NEG + k) : (k == 0 ? 1.0 : 0.0);

  // output = base + scale * (residual rows), with the mode folded in:
  //   mode 0: out = R;  1: out = R/detJ;  2: out = ca U0 + cb U + cc R/detJ
  const double detJ = ge[0];
  const double idet = 1.0 / detJ;
  const double scale = mode == 0 ? 1.0 : (mode == 1 ? idet : cc * idet);
  double* row = bufA + tid * SNP;  // own row: no sync needed to overwrite

  // (1) diffusion (exact stiffness) and linear source need every species;
  //     afterwards only the quadrature species stay live in registers
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double kc[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < NSYM; ++q) t = fma(ge[1 + q], tks[(q * NB + j) * NB + i], t);
      kc[j] = t;
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      double dif = 0.0, lin = 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) dif = fma(c[s * NB + j], kc[j], dif);
#pragma unroll
      for (int t = 0; t < S; ++t)
      if (M::lin_nz(s, t)) lin = fma(p.L[s * kMaxS + t], c[t * NB + i], lin);
      const double rv = detJ * (lin - p.A[s] * dif);
      row[s * NB + i] = mode == 2 ? fma(cb, c[s * NB + i], scale * rv) : scale * rv;
    }
  }

  // (2) quadrature: taxis flux rows (pulled back) and the bilinear source
  constexpr int NF = M::NFLUX, NL = M::NNL;
  if constexpr (NF + NL > 0) {
    double af[NF > 0 ? NF : 1][NB], al[NL > 0 ? NL : 1][NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
#pragma unroll
      for (int k = 0; k < (NF > 0 ? NF : 1); ++k) af[k][i] = 0.0;
#pragma unroll
      for (int k = 0; k < (NL > 0 ? NL : 1); ++k) al[k][i] = 0.0;
    }
#pragma unroll 2
    for (int q = 0; q < Q; ++q) {
      const double* ph = tphi + q * NB;
      const double* gr = tgr + q * NB * D;
      double v[M::NVAL];
      double g[M::NGRAD][D];
#pragma unroll
      for (int k = 0; k < M::NVAL; ++k) v[k] = 0.0;
#pragma unroll
      for (int k = 0; k < M::NGRAD; ++k)
#pragma unroll
        for (int a = 0; a < D; ++a) g[k][a] = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const double phv = ph[i];
#pragma unroll
        for (int k = 0; k < M::NVAL; ++k) v[k] = fma(phv, c[M::val_sp(k) * NB + i], v[k]);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double gv = gr[i * D + a];
#pragma unroll
          for (int k = 0; k < M::NGRAD; ++k) g[k][a] = fma(gv, c[M::grad_sp(k) * NB + i], g[k][a]);
        }
      }
      double gM[M::NGRAD][D];
#pragma unroll
      for (int k = 0; k < M::NGRAD; ++k)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) t = fma(g[k][a], ge[1 + sym_index(D, a, b)], t);
          gM[k][b] = t;
        }
      double fr[NF > 0 ? NF : 1][D], nl[NL > 0 ? NL : 1];
      M::template volume_point<D>(p.P, v, gM, fr, nl);
      const double w = tw[q];
#pragma unroll
      for (int k = 0; k < NF; ++k)
#pragma unroll
        for (int b = 0; b < D; ++b) fr[k][b] *= w;
#pragma unroll
      for (int k = 0; k < NL; ++k) nl[k] *= w;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const double gv = gr[i * D + a];
#pragma unroll
          for (int k = 0; k < NF; ++k) af[k][i] = fma(fr[k][a], gv, af[k][i]);
        }
#pragma unroll
        for (int k = 0; k < NL; ++k) al[k][i] = fma(nl[k], ph[i], al[k][i]);
      }
    }
    const double sd = scale * detJ;
#pragma unroll
    for (int k = 0; k < NF; ++k)
#pragma unroll
      for (int i = 0; i < NB; ++i) row[M::flux_sp(k) * NB + i] += sd * af[k][i];
#pragma unroll
    for (int k = 0; k < NL; ++k)
#pragma unroll
      for (int i = 0; i < NB; ++i) row[M::nl_sp(k) * NB + i] += sd * al[k][i];
  }

  // (3) the face-sum tile
  if (ACC != nullptr) {
    __syncthreads();
    tile_load<SN, SNP, TE>(ACC + e0 * SN, bufB, nt);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SN; ++r) row[r] = fma(scale, bufB[tid * SNP + r], row[r]);
  }
  if (mode == 2 && ca != 0.0) {
    __syncthreads();
    tile_load<SN, SNP, TE>(U0 + e0 * SN, bufB, nt);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SN; ++r) row[r] = fma(ca, bufB[tid * SNP + r], row[r]);
  }
  __syncthreads();
  tile_store<SN, SNP, TE>(out + e0 * SN, bufA, nt);
}

}  // namespace tdg

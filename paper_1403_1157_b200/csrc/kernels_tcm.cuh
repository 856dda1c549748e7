// Interior faces on the FP64 tensor cores (3D) in the MODAL face space.
// On a face the traces of the degree-k volume basis span P_k of the face
// triangle (nfm = (k+1)(k+2)/2 functions) and the traces of a directional
// derivative (Jinv n, fixed per face-geometry class) span P_{k-1} (ndm =
// k(k+1)/2): face_B = Bf T, G_n = Bd Td with orthonormal Bf, Bd at the face
// points (tables.modal_face_factors).  The face terms of reference
// operator.py:326-424 then need point values only for the nonlinear LLF
// flux; everything else is small modal algebra (a_j = T_in c_in - T_out
// c_out, g = (Td_in c_in + Td_out c_out) / 2, W = face weights):
//
//   R_in  =  sfac (T_in^T  Ybr + Td_in^T  Xbr)
//   R_out =  sfac (-T_out^T Ybr + Td_out^T Xbr)
//   Ybr   =  A Mfd g - ki L_l a_j - Bf^T W cnv      (ip: - eta/h A Mff a_j)
//   Xbr   =  adj/2 A Mfd^T a_j
//   cnv   =  lambda/2 du + (F_in + F_out).n / 2     pointwise, du = Bf a_j
//
// with L = Mff T T^T Mff the lifting (B (B^T W dU) in modal form).  At
// p = 3 this is 157 DMMAs per 8 (face, species) rows against 357 for the
// one-face kernel's 6 rows.  The CTA runs a face group of
// tables.tc_face_groups (4 faces sharing both sides' classes and the
// lifting side: every B operand is shared), one warp per 8 rows, like
// k_faces_tcg:
//
//   A  (modal)     a_in, a_out, d_in, d_out from the coefficients
//   B1 (points)    du, u_in, gav per point tile -> physics slots of xs
//   physics        LLF wave speed / taxis flux normals, CTA-wide
//   B2 (points)    cnv -> p = Bf^T W cnv
//   C  (modal)     Ybr, Xbr -> both sides' contributions
//
// The 96-entry point loops are unrolled (du stays in registers).
// Operand tables: tables.modal_face_tables (fragment-major, pi-permuted
// output columns so a GEMM's accumulator is the next GEMM's A operand).
#pragma once

#ifndef TDG_TCM_MINB
#define TDG_TCM_MINB 8
#endif

#include "common.cuh"
#include "kernels_mma.cuh"
#include "kernels_tcf.cuh"
#include "models.cuh"

namespace tdg {

// slot of species s among the physics (value) species, -1 if none
template <class M>
__host__ __device__ constexpr int mval_slot(int s) {
  for (int i = 0; i < M::NVAL; ++i)
    if (M::val_sp(i) == s) return i;
  return -1;
}
template <class M>
__host__ __device__ constexpr int mgrad_slot(int s) {
  for (int i = 0; i < M::NGRAD; ++i)
    if (M::grad_sp(i) == s) return i;
  return -1;
}
__host__ __device__ constexpr int gcd_m(int a, int b) { return b == 0 ? a : gcd_m(b, a % b); }

template <int D, int K, class M>
struct TcmFace {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF, NFG = Dm::NFG;
  static constexpr int NT = Dm::NT;  // trace-table signatures
  static constexpr int QP = ceil_to(F, 8), QT = QP / 8;
  static constexpr int KT = (NB + 3) / 4, NNT = (NB + 7) / 8;
  // P_k / P_{k-1} on the face triangle (3D only: on 2D's tiny segments a
  // group's work is too small for the CTA's two barriers; the register-
  // resident k_faces_fast stays faster at C2)
  static constexpr int NFM = (K + 1) * (K + 2) / 2, NDM = K * (K + 1) / 2, NV = NFM + NDM;
  // the modal vector v = (a | d) of a row: k-steps [0, KA) hold the a part,
  // [KD0, KTV) the d part; output tiles [0, NAT) the a part, [NAT0, NNV)
  // the d part (tables.modal_face_tables)
  static constexpr int KA = (NFM + 3) / 4, KTV = (NV + 3) / 4, KD0 = NFM / 4;
  static constexpr int NNV = (NV + 7) / 8, NAT = (NFM + 7) / 8, NAT0 = NFM / 8;
  // table offsets (doubles)
  static constexpr int OBF = 0, OBD = OBF + KA * QT * 32, OWB = OBD + (KTV - KD0) * QT * 32,
                       OMFD = OWB + QT * 2 * NAT * 32, OMDF = OMFD + (KTV - KD0) * NAT * 32,
                       OMFF = OMDF + KA * (NNV - NAT0) * 32, GLOB = OMFF + KA * NAT * 32;
  static constexpr int OL = 0, TABS = KA * NAT * 32;
  static constexpr int OTD1 = 0, OTD4 = OTD1 + KT * NNV * 32, OTD4M = OTD4 + KTV * NNT * 32,
                       CLS = OTD4M + KTV * NNT * 32;
  static constexpr int OCLS = GLOB + NT * TABS;  // first class block
  static constexpr int NCV = 1 + M::NFX;
  static constexpr int NFQ = 8 / gcd_m(S, 8), MT = S * NFQ / 8, THREADS = 32 * MT;
  // physics slots per (face, point): u_in, u_out of the value species, gav
  // of the gradient species (odd stride: conflict-free physics reads)
  static constexpr int NSL = 2 * M::NVAL + M::NGRAD, XS = NSL | 1;
  // p >= 3: the point physics writes its NCV results over the slots it has
  // read (face_point reads every input first), so there is no separate cv
  // array and 8 CTAs leave L1 room for the class tables a group streams
  // (64^3 p = 3 faces 9.25 -> 8.73 ms; at p = 2 the extra barrier costs more
  // than the L1 gains: 5.27 -> 5.36 ms)
  static constexpr bool ALIAS = K >= 3;
  static_assert(!ALIAS || NCV <= XS, "cv slots alias the physics slots");
  static constexpr int OXS = 0, OCV = ALIAS ? OXS : OXS + NFQ * QP * XS,
                       CWS = OCV + (ALIAS ? NFQ * QP * XS : NFQ * QP * NCV);
  static constexpr size_t smem() { return size_t(CWS) * 8; }
  // 80 registers (small spills) -> 8 CTAs / 24 warps per SM: 64^3 p = 3
  // faces 10.8 -> 10.3 ms, p = 2 6.2 -> 5.1 ms against 128 registers
  static constexpr int MINB = K >= 3 ? TDG_TCM_MINB : 7;
  static constexpr bool ok = D == 3 && K >= 1 && M::kConv && !M::kMirror && MT >= 1 &&
                             MT <= 4 && F <= 64 && smem() * MINB <= 200 * 1024;
};

// LM: lifting sides (operator.py:336-357): 0 none (ip, bo), 1 the K- side
// (cdg2, cdg), 2 both (br2)
template <int D, int K, class M, int LM>
__global__ void __launch_bounds__(TcmFace<D, K, M>::THREADS, TcmFace<D, K, M>::MINB)
k_faces_tcm(OpParams p, const double* __restrict__ tm, const int32_t* __restrict__ groups,
            int64_t g0, int64_t g1, const double* __restrict__ U, double* __restrict__ ACC) {
  using T = TcmFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, NFG = T::NFG, QP = T::QP;
  constexpr int QT = T::QT, KT = T::KT, NNT = T::NNT;
  constexpr int KA = T::KA, KTV = T::KTV, KD0 = T::KD0, NNV = T::NNV, NAT = T::NAT,
                NAT0 = T::NAT0;
  constexpr int NCV = T::NCV, XS = T::XS, NFQ = T::NFQ;
  constexpr bool br2 = LM == 2, lift = LM > 0;
  extern __shared__ __align__(16) double sm[];
  double* xs = sm + T::OXS;   // [NFQ][QP][XS] physics slots
  double* cvs = sm + T::OCV;  // [NFQ][QP][NCV]
  const int lane = threadIdx.x & 31, mt = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int fq = (8 * mt + g) / S, sp = (8 * mt + g) % S;
  const double As = p.A[sp];
  // this row's physics slots (-1: none)
  int slv = -1, slg = -1;
#pragma unroll
  for (int s = 0; s < S; ++s)
    if (sp == s) {
      slv = mval_slot<M>(s);
      slg = mgrad_slot<M>(s);
    }
  const double* tg = tm;  // global block

  for (int64_t grp = g0 + blockIdx.x; grp < g1; grp += gridDim.x) {
    const int32_t* gf = groups + grp * NFQ;
    const int f0 = __ldg(gf);
    const int code0 = __ldg(p.ifcode + f0);
    const int2 cl = __ldg(reinterpret_cast<const int2*>(p.ffold) + f0);
    const int sig = code0 & 1023;
    const double* Ti = tm + T::GLOB + size_t(sig & 31) * T::TABS;
    const double* To = tm + T::GLOB + size_t((sig >> 5) & 31) * T::TABS;
    const double* Ci = tm + T::OCLS + size_t(cl.x) * T::CLS;
    const double* Co = tm + T::OCLS + size_t(cl.y) * T::CLS;
    const bool min_ = code_minus_in(code0);  // one lifting side per group
    const int fid = __ldg(gf + fq);
    const bool fv = fid >= 0;
    const int fs = fv ? fid : f0;
    const double* gg = p.ifgeo + int64_t(fs) * NFG;
    const double sfac = fv ? __ldg(gg + 2 * D) : 0.0;
    const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + fs);

    // ---- A: modal vectors v = (a | d) of both sides -----------------------
    double vI[NNV][2], vO[NNV][2];
#pragma unroll
    for (int n = 0; n < NNV; ++n) vI[n][0] = vI[n][1] = vO[n][0] = vO[n][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const bool in = fv && 4 * kt + t < NB;
      const double ci = in ? __ldg(U + int64_t(el.x) * SN + sp * NB + 4 * kt + t) : 0.0;
      const double co = in ? __ldg(U + int64_t(el.y) * SN + sp * NB + 4 * kt + t) : 0.0;
#pragma unroll
      for (int n = 0; n < NNV; ++n) {
        const int o = T::OTD1 + (kt * NNV + n) * 32 + lane;
        dmma(vI[n][0], vI[n][1], ci, __ldg(Ci + o));
        dmma(vO[n][0], vO[n][1], co, __ldg(Co + o));
      }
    }
    // A fragments: k-step kt holds combined mode 4 kt + t = pi(8 (kt/2) +
    // 2t + kt%2), i.e. accumulator entry [kt/2][kt%2].  aJ's a part is the
    // jump a_in - a_out, gm's d part the average (d_in + d_out) / 2 (the
    // other parts meet zero table rows)
    double aJ[NNV][2], gm[NNV][2];
#pragma unroll
    for (int n = 0; n < NNV; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        aJ[n][j] = vI[n][j] - vO[n][j];
        gm[n][j] = 0.5 * (vI[n][j] + vO[n][j]);
      }

    if constexpr (T::ALIAS) __syncthreads();  // the previous group's B2 has read its cv slots
    // ---- B1: point values -> physics slots; du kept in registers -------
    double du[QT][2];
#pragma unroll
    for (int qt = 0; qt < QT; ++qt) {
      double d0[2] = {0.0, 0.0}, u0[2] = {0.0, 0.0}, gv[2] = {0.0, 0.0};
#pragma unroll
      for (int kt = 0; kt < KA; ++kt) {
        const double b = __ldg(tg + T::OBF + (kt * QT + qt) * 32 + lane);
        dmma(d0[0], d0[1], aJ[kt / 2][kt % 2], b);
        dmma(u0[0], u0[1], vI[kt / 2][kt % 2], b);
      }
#pragma unroll
      for (int kt = KD0; kt < KTV; ++kt)  // (warp-wide: every row, used by the gradient species)
        dmma(gv[0], gv[1], gm[kt / 2][kt % 2],
             __ldg(tg + T::OBD + ((kt - KD0) * QT + qt) * 32 + lane));
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        du[qt][j] = d0[j];
        if (slv >= 0) {
          double* x = xs + (fq * QP + 8 * qt + 2 * t + j) * XS;
          x[slv] = u0[j];
          x[M::NVAL + slv] = u0[j] - d0[j];
          if (slg >= 0) x[2 * M::NVAL + slg] = gv[j];
        }
      }
    }
    __syncthreads();
    // ---- physics, once per (face, point), CTA-wide -------------------------
    for (int i = threadIdx.x; i < NFQ * F; i += T::THREADS) {
      const int f = i / F, q = i - f * F;
      const double* xq = xs + (f * QP + q) * XS;
      auto fetch = [xq](int kind, int s2) {
        return kind == 0 ? xq[mval_slot<M>(s2)]
                         : (kind == 1 ? xq[M::NVAL + mval_slot<M>(s2)]
                                      : xq[2 * M::NVAL + mgrad_slot<M>(s2)]);
      };
      if constexpr (T::ALIAS) {
        double cv[NCV];
        M::face_point(p.P, fetch, cv);
#pragma unroll
        for (int k = 0; k < NCV; ++k) xs[(f * QP + q) * XS + k] = cv[k];
      } else {
        M::face_point(p.P, fetch, cvs + (f * QP + q) * NCV);
      }
    }
    __syncthreads();
    // ---- B2 + C: the row's modal bracket yb = (Ybr | Xbr) ---------------
    //   Ybr = A Mfd g - ki L a_j - Bf^T W cnv  (ip: - eta/h A Mff a_j)
    //   Xbr = adj/2 A Mfd^T a_j
    double yb[NNV][2];
#pragma unroll
    for (int n = 0; n < NNV; ++n) yb[n][0] = yb[n][1] = 0.0;
#pragma unroll
    for (int qt = 0; qt < QT; ++qt) {
      double cn[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 8 * qt + 2 * t + j;
        double v = 0.0;
        if (q < F) {
          const double* c = T::ALIAS ? xs + (fq * QP + q) * XS : cvs + (fq * QP + q) * NCV;
          v = 0.5 * c[0] * du[qt][j];
#pragma unroll
          for (int k = 0; k < M::NFX; ++k)
            if (sp == k) v = fma(0.5, c[1 + k], v);
        }
        cn[j] = -v;  // Ybr carries - Bf^T W cnv
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int n = 0; n < NAT; ++n)
          dmma(yb[n][0], yb[n][1], cn[ks], __ldg(tg + T::OWB + ((qt * 2 + ks) * NAT + n) * 32 + lane));
    }
#pragma unroll
    for (int kt = KD0; kt < KTV; ++kt)
#pragma unroll
      for (int n = 0; n < NAT; ++n)
        dmma(yb[n][0], yb[n][1], As * gm[kt / 2][kt % 2],
             __ldg(tg + T::OMFD + ((kt - KD0) * NAT + n) * 32 + lane));
    if constexpr (lift) {
      const double wside = br2 ? 0.5 : 1.0;
      const double fac0 = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * wside * 0.5 * sfac * As;
      const double ki = fac0 * __ldg(gg + 2 * D + ((br2 || min_) ? 2 : 3));
      const double ko = br2 ? fac0 * __ldg(gg + 2 * D + 3) : 0.0;
      const double* Tl = (br2 || min_) ? Ti : To;
#pragma unroll
      for (int kt = 0; kt < KA; ++kt)
#pragma unroll
        for (int n = 0; n < NAT; ++n) {
          const int o = T::OL + (kt * NAT + n) * 32 + lane;
          dmma(yb[n][0], yb[n][1], -ki * aJ[kt / 2][kt % 2], __ldg(Tl + o));
          if constexpr (br2) dmma(yb[n][0], yb[n][1], -ko * aJ[kt / 2][kt % 2], __ldg(To + o));
        }
    } else {
      if (p.scheme == IP) {
        const double kip = -p.eta / __ldg(gg + 2 * D + 1) * As;
#pragma unroll
        for (int kt = 0; kt < KA; ++kt)
#pragma unroll
          for (int n = 0; n < NAT; ++n)
            dmma(yb[n][0], yb[n][1], kip * aJ[kt / 2][kt % 2],
                 __ldg(tg + T::OMFF + (kt * NAT + n) * 32 + lane));
      }
    }
    {
      const double kx = 0.5 * p.adj * As;
#pragma unroll
      for (int kt = 0; kt < KA; ++kt)
#pragma unroll
        for (int n = NAT0; n < NNV; ++n)
          dmma(yb[n][0], yb[n][1], kx * aJ[kt / 2][kt % 2],
               __ldg(tg + T::OMDF + (kt * (NNV - NAT0) + n - NAT0) * 32 + lane));
    }
    // R_in = sfac (T_in ; Td_in)^T yb, R_out = sfac (-T_out ; Td_out)^T yb
    double ri[NNT][2], ro[NNT][2];
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt) ri[nt][0] = ri[nt][1] = ro[nt][0] = ro[nt][1] = 0.0;
#pragma unroll
    for (int kt = 0; kt < KTV; ++kt) {
      const double a = sfac * yb[kt / 2][kt % 2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) {
        dmma(ri[nt][0], ri[nt][1], a, __ldg(Ci + T::OTD4 + (kt * NNT + nt) * 32 + lane));
        dmma(ro[nt][0], ro[nt][1], a, __ldg(Co + T::OTD4M + (kt * NNT + nt) * 32 + lane));
      }
    }
    // face-sum rows: lane entries (face fq, species sp, basis 4 (2nt + j) + t)
    if (fv) {
      const int code = __ldg(p.ifcode + fid);
      const bool skip_out = code_skip_out(code);
      const bool fin = code_first_in(code), fout = code_first_out(code);
      double* fci = ACC + int64_t(el.x) * SN + sp * NB;
      double* fco = ACC + int64_t(el.y) * SN + sp * NB;
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = 4 * (2 * nt + j) + t;
          if (i < NB) {
            acc_put(fci + i, ri[nt][j], fin);
            if (!skip_out) acc_put(fco + i, ro[nt][j], fout);
          }
        }
    }
  }
}

}  // namespace tdg

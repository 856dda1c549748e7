// Volume terms + M^-1 + Runge-Kutta stage on the FP64 tensor cores, for
// the larger (d, k) where one thread per element cannot hold an element
// in registers (2D k=3, 3D k=2/3): C3, C4, C5.
//
// Layout: a warp owns EW = 8 elements, the M dimension of every
// mma.sync.m8n8k4.f64 (DMMA).  With g = lane>>2, t = lane&3:
//
//   A fragment  A[g][t]        element g, basis k = 4 kt + t   (coefficients,
//                              loaded straight from U: 32 contiguous bytes
//                              per element and k-step)
//   B fragment  B[t][g]        tables, n = point or output column
//   accumulator C[g][2t + j]   element g, column 2t + j
//
//   point values   V_s[e][q]   = sum_k c_s[e][k] Phi[q][k]      (B = Phi^T)
//   ref. gradients G_sa[e][q]  = sum_k c_s[e][k] d_a Phi[q][k]
//   flux rows      R_f[e][n]  += sum_q Fr_fa[e][q] w_q d_a Phi[q][pi(n)]
//   bilinear src   R_l[e][n]  += sum_q Nl[e][q]    w_q Phi[q][pi(n)]
//   diffusion      D_s[e][n]   = sum_p M_p[e] sum_k c_s[e][k] KS_p[k][pi(n)]
//
// The point physics runs on the accumulator layout (each lane holds every
// species at its two (element, point) pairs), and the projection's A
// operand is that same accumulator taken one point parity at a time (k-step
// ks uses points 8qt + 2t + ks): no lane exchange anywhere.  The output
// columns are permuted, pi(8nt + 2t + j) = 4(2nt + j) + t, so a lane's
// output entries are exactly the basis indices of its A fragments: the
// linear source, the U / U0 / face-sum reads and the output stores are
// lane-local, 32-byte-contiguous accesses.  Formulas as k_volume
// (reference operator.py:292-324, model.py:147-170); tables built by
// tables.tc_volume_tables.
#pragma once

#include "common.cuh"
#include "kernels.cuh"
#include "kernels_mma.cuh"
#include "models.cuh"

namespace tdg {

// species whose values or gradients the volume point physics reads
template <class M>
__host__ __device__ constexpr bool quad_species(int s) {
  for (int k = 0; k < M::NVAL; ++k)
    if (M::val_sp(k) == s) return true;
  for (int k = 0; k < M::NGRAD; ++k)
    if (M::grad_sp(k) == s) return true;
  return false;
}

template <int D, int K, class M>
struct TcVol {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, Q = Dm::NQV;
  static constexpr int NEG = Dm::NEG, NSYM = Dm::NSYM;
  static constexpr int QP = ceil_to(Q, 8), QT = QP / 8;
  static constexpr int KT = (NB + 3) / 4, NBK = 4 * KT;
  static constexpr int NNT = (NB + 7) / 8, NBN = 8 * NNT;
  static constexpr int NV = M::NVAL, NG = M::NGRAD, NF = M::NFLUX, NL = M::NNL;
  // table offsets (doubles); tables are fragment-major (tables.tc_volume_tables):
  // a warp's B-operand load is 32 consecutive doubles
  static constexpr int OPHT = 0;                         // [NBK][QP]
  static constexpr int OGT = OPHT + NBK * QP;            // [D][NBK][QP]
  static constexpr int OPP = OGT + D * NBK * QP;         // [QP][NBN]
  static constexpr int OPG = OPP + QP * NBN;             // [D][QP][NBN]
  static constexpr int OKS = OPG + D * QP * NBN;         // [NSYM][NBK][NBN]
  static constexpr int TAB = OKS + NSYM * NBK * NBN;
  // tables up to 64 KB: 4-warp CTAs, 2 per SM; larger (3D p = 3: 203 KB)
  // still in shared memory, with one 8-warp CTA per SM (the same 8 warps /
  // SM the 255-register budget allows), instead of streaming them through
  // L1 (ncu at p = 3 from global: L1 hit 76 %)
  static constexpr bool kBig = TAB * 8 > 64 * 1024;
  static constexpr bool kSmemTables = TAB * 8 <= 220 * 1024;
  static constexpr int WARPS = kBig ? 12 : 4, EW = 8;
  static constexpr size_t smem() { return kSmemTables ? size_t(TAB) * 8 : 0; }
  static constexpr int MINB = kBig ? 1 : 2;
  static constexpr bool ok = S <= kMaxS && D >= 2;
};

// CLS: the warps visit tasks [task0, task1) of 8 same-class elements
// (p.vperm, tables.tc_volume_classes) and run the diffusion against the
// class's summed stiffness (one GEMM per species); otherwise task i is the
// elements 8i .. 8i+7 of the (range-shifted) arrays
template <int D, int K, class M, bool CLS>
__global__ void __launch_bounds__(32 * TcVol<D, K, M>::WARPS, TcVol<D, K, M>::MINB)
k_volume_tc(OpParams p, const double* __restrict__ tabs, const double* __restrict__ U,
            const double* ACC, const double* U0, double* out, double ca, double cb,
            double cc, int mode, int64_t task0, int64_t task1) {
  using T = TcVol<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, NEG = T::NEG, NSYM = T::NSYM;
  constexpr int QT = T::QT, KT = T::KT, NNT = T::NNT;
  constexpr int NV = T::NV, NG = T::NG, NF = T::NF, NL = T::NL;
  extern __shared__ __align__(16) double sm[];
  const double* tb = tabs;
  if constexpr (T::kSmemTables) {
    for (int i = threadIdx.x; i < T::TAB; i += 32 * T::WARPS) sm[i] = __ldg(tabs + i);
    __syncthreads();
    tb = sm;
  }
  // ACC: face-sum rows (null: no faces); ACC and U0 may alias out (each
  // lane reads its own entries before writing them)
  mode &= 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  for (int64_t task = task0 + int64_t(blockIdx.x) * T::WARPS + warp; task < task1;
       task += int64_t(gridDim.x) * T::WARPS) {
    int64_t e, ec;
    bool valid;
    if constexpr (CLS) {
      e = __ldg(p.vperm + task * T::EW + g);
      valid = e >= 0;
      ec = valid ? e : __ldg(p.vperm + task * T::EW);  // a task's first slot is an element
    } else {
      e = task * T::EW + g;
      valid = e < p.ne;
      ec = valid ? e : p.ne - 1;
    }
    double ge[NEG];
#pragma unroll
    for (int k = 0; k < NEG; ++k) ge[k] = __ldg(p.egeo + ec * NEG + k);
    // A fragments (basis 4 kt + t): the quadrature species now, the others
    // only for the epilogue (shorter register live ranges)
    double cf[S][KT];
    const double* urow = U + ec * SN;
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (quad_species<M>(s))
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
          cf[s][kt] = (4 * kt + t < NB) ? __ldg(urow + s * NB + 4 * kt + t) : 0.0;

    double af[NF > 0 ? NF : 1][NNT][2], al[NL > 0 ? NL : 1][NNT][2];
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
#pragma unroll
        for (int k = 0; k < (NF > 0 ? NF : 1); ++k) af[k][nt][j] = 0.0;
#pragma unroll
        for (int k = 0; k < (NL > 0 ? NL : 1); ++k) al[k][nt][j] = 0.0;
      }

    if constexpr (NF + NL > 0) {
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        // point values and reference gradients of the quadrature species
        double v[NV > 0 ? NV : 1][2], gr[NG > 0 ? NG : 1][D][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int k = 0; k < (NV > 0 ? NV : 1); ++k) v[k][j] = 0.0;
#pragma unroll
          for (int k = 0; k < (NG > 0 ? NG : 1); ++k)
#pragma unroll
            for (int a = 0; a < D; ++a) gr[k][a][j] = 0.0;
        }
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const double bphi = tb[T::OPHT + (kt * QT + qt) * 32 + lane];
#pragma unroll
          for (int k = 0; k < NV; ++k) dmma(v[k][0], v[k][1], cf[M::val_sp(k)][kt], bphi);
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double bg = tb[T::OGT + ((a * KT + kt) * QT + qt) * 32 + lane];
#pragma unroll
            for (int k = 0; k < NG; ++k) dmma(gr[k][a][0], gr[k][a][1], cf[M::grad_sp(k)][kt], bg);
          }
        }
        // point physics at (element g, point 8qt + 2t + j)
        double fr[NF > 0 ? NF : 1][D][2], nl[NL > 0 ? NL : 1][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double vv[NV > 0 ? NV : 1], gM[NG > 0 ? NG : 1][D];
#pragma unroll
          for (int k = 0; k < NV; ++k) vv[k] = v[k][j];
#pragma unroll
          for (int k = 0; k < NG; ++k)
#pragma unroll
            for (int b = 0; b < D; ++b) {
              double s = 0.0;
#pragma unroll
              for (int a = 0; a < D; ++a) s = fma(gr[k][a][j], ge[1 + sym_index(D, a, b)], s);
              gM[k][b] = s;
            }
          double f[NF > 0 ? NF : 1][D], n1[NL > 0 ? NL : 1];
          M::template volume_point<D>(p.P, vv, gM, f, n1);
#pragma unroll
          for (int k = 0; k < NF; ++k)
#pragma unroll
            for (int a = 0; a < D; ++a) fr[k][a][j] = f[k][a];
#pragma unroll
          for (int k = 0; k < NL; ++k) nl[k][j] = n1[k];
        }
        // projection: k-step ks takes the points of parity ks
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
          for (int nt = 0; nt < NNT; ++nt) {
#pragma unroll
            for (int a = 0; a < D; ++a) {
              const double bp = tb[T::OPG + (((a * QT + qt) * 2 + ks) * NNT + nt) * 32 + lane];
#pragma unroll
              for (int k = 0; k < NF; ++k) dmma(af[k][nt][0], af[k][nt][1], fr[k][a][ks], bp);
            }
            if constexpr (NL > 0) {
              const double bq = tb[T::OPP + ((qt * 2 + ks) * NNT + nt) * 32 + lane];
#pragma unroll
              for (int k = 0; k < NL; ++k) dmma(al[k][nt][0], al[k][nt][1], nl[k][ks], bq);
            }
          }
        }
      }
    }

    // epilogue per species: diffusion GEMM, linear source, face slots, RK
    const double detJ = ge[0];
    const double idet = 1.0 / detJ;
    const double scale = mode == 0 ? 1.0 : (mode == 1 ? idet : cc * idet);
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (!quad_species<M>(s))
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
          cf[s][kt] = (4 * kt + t < NB) ? __ldg(urow + s * NB + 4 * kt + t) : 0.0;
    // species loop unrolled where the registers allow (coefficients stay in
    // registers instead of a dynamically indexed local array; 3D p = 3
    // would spill 1.4 KB)
    constexpr int SUNR = T::kBig ? 1 : S;
#pragma unroll SUNR
    for (int s = 0; s < S; ++s) {
      // this species' face sums and U0 entries, loaded ahead of the
      // diffusion GEMM so their latency hides behind it
      double facc[NNT][2], fu0[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = 4 * (2 * nt + j) + t;
          const int64_t off = ec * SN + s * NB + (i < NB ? i : 0);
          facc[nt][j] = ACC != nullptr ? __ldcs(ACC + off) : 0.0;
          fu0[nt][j] = (mode == 2 && ca != 0.0) ? U0[off] : 0.0;
        }
      double dif[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) dif[nt][0] = dif[nt][1] = 0.0;
      if constexpr (CLS) {
        // one GEMM against the class's sum_p M_p KS_p
        const double* kc = p.vctab + size_t(__ldg(p.vtcls + task)) * (KT * NNT * 32);
#pragma unroll
        for (int kt = 0; kt < KT; ++kt)
#pragma unroll
          for (int nt = 0; nt < NNT; ++nt)
            dmma(dif[nt][0], dif[nt][1], cf[s][kt], __ldg(kc + (kt * NNT + nt) * 32 + lane));
      } else {
#pragma unroll
        for (int pq = 0; pq < NSYM; ++pq)
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const double a = cf[s][kt] * ge[1 + pq];
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt)
              dmma(dif[nt][0], dif[nt][1], a,
                   tb[T::OKS + ((pq * KT + kt) * NNT + nt) * 32 + lane]);
          }
      }
      const int fi = M::flux_index(s), li = M::nl_index(s);
      const double As = p.A[s];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int kt = 2 * nt + j, i = 4 * kt + t;
          if (kt >= KT || i >= NB) continue;
          double lin = 0.0;
#pragma unroll
          for (int s2 = 0; s2 < S; ++s2)
            if (M::lin_nz(s, s2)) lin = fma(p.L[s * kMaxS + s2], cf[s2][kt], lin);
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < NF; ++k)
            if (fi == k) acc = af[k][nt][j];
#pragma unroll
          for (int k = 0; k < NL; ++k)
            if (li == k) acc += al[k][nt][j];
          double rv = detJ * (acc - As * dif[nt][j] + lin);
          const int64_t off = ec * SN + s * NB + i;
          rv += facc[nt][j];
          double o = scale * rv;
          if (mode == 2) {
            o = fma(cb, cf[s][kt], o);
            if (ca != 0.0) o = fma(ca, fu0[nt][j], o);
          }
          if (valid) out[off] = o;
        }
    }
  }
}

}  // namespace tdg

// Matrix-free DG operator kernels (generic CTA-staged versions).
//
// One application  R = L_h(U)  (reference operator.py:253-284) is three
// launches, all deterministic (no atomics):
//
//   k_faces  interior (+ Dirichlet-mirror) faces   operator.py:359-444
//   k_wall   prescribed-flux boundary faces        operator.py:446-458
//            both add each face side's contribution block to the
//            element's face-sum row ACC[e][s][i]; the faces run in colour
//            segments (one launch per segment, no element twice in a
//            segment), so the two-sided scatter is conflict-free without
//            atomics and the sums have a fixed order;
//   k_volume volume terms (operator.py:292-324) + the element's face sum
//            + M^-1 (fespace.py:117-118) + the Runge-Kutta stage
//            combination, fused; writes the element's output rows once.
//
// Each CTA stages its tile's coefficient blocks (S*nb contiguous doubles
// per element) in shared memory with coalesced loads, then runs small
// dense contractions whose table operand is warp-uniform (L1 broadcast).
#pragma once

#include "common.cuh"
#include "models.cuh"

namespace tdg {

constexpr int kThreads = 128;

__device__ __forceinline__ int sym_index(int D, int a, int b) {
  // storage of the symmetric d x d metric: (0,0),(0,1),..,(0,d-1),(1,1),..
  int lo = a < b ? a : b, hi = a < b ? b : a;
  return lo * D - lo * (lo - 1) / 2 + (hi - lo);
}

template <int D, int K, class M>
struct VolumeTile {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, SNP = SN | 1;
  static constexpr int NPW = M::NFLUX * D + M::NNL;
  static constexpr int per_elem = SNP + Dm::NEG + Dm::NQV * NPW;
  static constexpr int TE0 = (96 * 1024 / 8) / per_elem;
  static constexpr int TE = TE0 >= 64 ? 64 : TE0 >= 32 ? 32 : TE0 >= 16 ? 16 : 8;
  static constexpr size_t smem(int nqv) { return size_t(TE) * (SNP + Dm::NEG + nqv * NPW) * 8; }
};

// mode 0: out = L(U);  1: out = M^-1 L(U);  2: out = ca*U0 + cb*U + cc*M^-1 L(U)
template <int D, int K, class M>
__global__ void __launch_bounds__(kThreads)
k_volume(OpParams p, const double* __restrict__ U, const double* ACC,
         const double* U0, double* out, double ca, double cb, double cc, int mode) {
  using T = VolumeTile<D, K, M>;
  using Dm = Dims<D, K>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, SNP = T::SNP, NPW = T::NPW, TE = T::TE;
  constexpr int NEG = Dm::NEG;
  extern __shared__ double sm[];
  double* cs = sm;
  double* geo = cs + TE * SNP;
  double* pt = geo + TE * NEG;
  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * TE;
  const int nt = int(p.ne - e0 < TE ? p.ne - e0 : TE);
  const int nqv = p.nqv;

  for (int idx = tid; idx < nt * SN; idx += kThreads) {
    int e = idx / SN, r = idx - e * SN;
    cs[e * SNP + r] = U[e0 * SN + idx];
  }
  for (int idx = tid; idx < nt * NEG; idx += kThreads) geo[idx] = p.egeo[e0 * NEG + idx];
  __syncthreads();

  if constexpr (NPW > 0) {
    // quadrature-point physics; a warp covers consecutive elements at one
    // point, so the table rows are warp-uniform
    for (int idx = tid; idx < TE * nqv; idx += kThreads) {
      const int q = idx / TE, e = idx - q * TE;
      if (e >= nt) continue;
      const double* c = cs + e * SNP;
      const double* ph = p.phi + q * NB;
      const double* gr = p.grad + q * NB * D;
      double v[M::NVAL > 0 ? M::NVAL : 1];
      double g[M::NGRAD > 0 ? M::NGRAD : 1][D];
#pragma unroll
      for (int k = 0; k < M::NVAL; ++k) {
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < NB; ++i) a = fma(__ldg(ph + i), c[M::val_sp(k) * NB + i], a);
        v[k] = a;
      }
#pragma unroll
      for (int k = 0; k < M::NGRAD; ++k)
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < NB; ++i) s = fma(__ldg(gr + i * D + a), c[M::grad_sp(k) * NB + i], s);
          g[k][a] = s;
        }
      double gM[M::NGRAD > 0 ? M::NGRAD : 1][D];
      const double* ms = geo + e * NEG + 1;
#pragma unroll
      for (int k = 0; k < M::NGRAD; ++k)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) s = fma(g[k][a], ms[sym_index(D, a, b)], s);
          gM[k][b] = s;
        }
      double fr[M::NFLUX > 0 ? M::NFLUX : 1][D];
      double nl[M::NNL > 0 ? M::NNL : 1];
      M::template volume_point<D>(p.P, v, gM, fr, nl);
      const double w = __ldg(p.wv + q);
      double* o = pt + (e * nqv + q) * NPW;
#pragma unroll
      for (int k = 0; k < M::NFLUX; ++k)
#pragma unroll
        for (int b = 0; b < D; ++b) o[k * D + b] = w * fr[k][b];
#pragma unroll
      for (int k = 0; k < M::NNL; ++k) o[M::NFLUX * D + k] = w * nl[k];
    }
    __syncthreads();
  }

  for (int idx = tid; idx < nt * SN; idx += kThreads) {
    const int e = idx / SN, r = idx - e * SN, s = r / NB, i = r - s * NB;
    const double* c = cs + e * SNP;
    const double* ge = geo + e * NEG;
    double acc = 0.0;
    if constexpr (NPW > 0) {
      const int fi = M::flux_index(s), li = M::nl_index(s);
      if (fi >= 0) {
        for (int q = 0; q < nqv; ++q) {
          const double* o = pt + (e * nqv + q) * NPW + fi * D;
          const double* gr = p.grad + (q * NB + i) * D;
#pragma unroll
          for (int a = 0; a < D; ++a) acc = fma(o[a], __ldg(gr + a), acc);
        }
      }
      if (li >= 0) {
        for (int q = 0; q < nqv; ++q)
          acc = fma(pt[(e * nqv + q) * NPW + M::NFLUX * D + li], __ldg(p.phi + q * NB + i), acc);
      }
    }
    // diffusion  -A_s sum_j c_sj sum_p M_p KS_p[j][i]  (exact for the
    // reference's quadrature, which integrates degree 2k-2 exactly)
    double dif = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      double kij = 0.0;
#pragma unroll
      for (int q = 0; q < Dm::NSYM; ++q) kij = fma(ge[1 + q], __ldg(p.ks + (q * NB + j) * NB + i), kij);
      dif = fma(c[s * NB + j], kij, dif);
    }
    double lin = 0.0;
#pragma unroll
    for (int t = 0; t < S; ++t)
      if (M::lin_nz(s, t)) lin = fma(p.L[s * kMaxS + t], c[t * NB + i], lin);
    const double detJ = ge[0];
    double rv = detJ * (acc - p.A[s] * dif + lin);
    if (ACC != nullptr) rv += ACC[(e0 + e) * SN + r];
    double o;
    if (mode == 0) o = rv;
    else if (mode == 1) o = rv / detJ;
    else {
      o = cb * c[r] + cc * (rv / detJ);
      if (ca != 0.0) o = fma(ca, U0[e0 * SN + idx], o);
    }
    out[e0 * SN + idx] = o;
  }
}

// ------------------------------------------------------------------ faces

template <int D, int K, class M>
struct FaceTile {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, SNP = SN | 1, F = Dm::NQF;
  static constexpr int per_face = 2 * SNP + Dm::NFG + 3 + 2 * F * NB + 6 * S * F;
  static constexpr int TF0 = (96 * 1024 / 8) / per_face;
  static constexpr int TF = TF0 >= 32 ? 32 : TF0 >= 16 ? 16 : TF0 >= 8 ? 8 : TF0 >= 4 ? 4 : TF0 >= 2 ? 2 : 1;
  static constexpr size_t smem() { return size_t(TF) * per_face * 8; }
};

template <int D, int K, class M>
__global__ void __launch_bounds__(kThreads)
k_faces(OpParams p, const double* __restrict__ U, double* __restrict__ ACC) {
  using T = FaceTile<D, K, M>;
  using Dm = Dims<D, K>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, SNP = T::SNP, F = T::F, TF = T::TF;
  constexpr int NFG = Dm::NFG;
  extern __shared__ double sm[];
  double* cs = sm;                      // [TF][2][SNP]
  double* geo = cs + TF * 2 * SNP;      // [TF][NFG]
  int* meta = reinterpret_cast<int*>(geo + TF * NFG);  // [TF][6]: code, e_in, e_out, pad
  double* dph = geo + TF * NFG + TF * 3;               // [TF][2][F][NB]
  double* tr = dph + TF * 2 * F * NB;                  // [TF][4][S][F]
  double* yx = tr + TF * 4 * S * F;                    // [TF][2][S][F]
  const int tid = threadIdx.x;
  const int64_t f0 = int64_t(blockIdx.x) * TF;
  const int nt = int(p.nif - f0 < TF ? p.nif - f0 : TF);
  const int nqf = p.nqf;

  for (int f = tid; f < nt; f += kThreads) {
    int* m = meta + f * 6;
    m[0] = p.ifcode[f0 + f];
    m[1] = p.ifel[2 * (f0 + f)];
    m[2] = p.ifel[2 * (f0 + f) + 1];
  }
  for (int idx = tid; idx < nt * NFG; idx += kThreads) geo[idx] = p.ifgeo[f0 * NFG + idx];
  __syncthreads();
  for (int idx = tid; idx < nt * 2 * SN; idx += kThreads) {
    const int f = idx / (2 * SN), r = idx - f * 2 * SN, side = r / SN, rr = r - side * SN;
    const int e = meta[f * 6 + 1 + side];
    if (e >= 0) cs[(f * 2 + side) * SNP + rr] = U[int64_t(e) * SN + rr];
  }
  // normal-derivative test tables (G . jn) per face side
  for (int idx = tid; idx < nt * 2 * nqf * NB; idx += kThreads) {
    const int f = idx / (2 * nqf * NB), r = idx - f * 2 * nqf * NB;
    const int side = r / (nqf * NB), qi = r - side * nqf * NB;
    const int code = meta[f * 6];
    if (side && code_mirror(code)) continue;
    const int t = side ? code_tout(code) : code_tin(code);
    const double* gr = p.fG + (size_t(t) * nqf * NB + qi) * D;
    const double* jn = geo + f * NFG + side * D;
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) s = fma(__ldg(gr + a), jn[a], s);
    dph[(f * 2 + side) * F * NB + qi] = s;
  }
  __syncthreads();
  // traces u and d_n u per side, species and point
  for (int idx = tid; idx < nt * 2 * S * nqf; idx += kThreads) {
    const int f = idx / (2 * S * nqf), r = idx - f * 2 * S * nqf;
    const int side = r / (S * nqf), sq = r - side * S * nqf, s = sq / nqf, q = sq - s * nqf;
    const int code = meta[f * 6];
    if (side && code_mirror(code)) continue;
    const int t = side ? code_tout(code) : code_tin(code);
    const double* b = p.fB + (size_t(t) * nqf + q) * NB;
    const double* dp = dph + ((f * 2 + side) * F + q) * NB;
    const double* c = cs + (f * 2 + side) * SNP + s * NB;
    double u = 0.0, gn = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      u = fma(__ldg(b + i), c[i], u);
      gn = fma(dp[i], c[i], gn);
    }
    tr[((f * 4 + side) * S + s) * F + q] = u;
    tr[((f * 4 + 2 + side) * S + s) * F + q] = gn;
  }
  __syncthreads();
  // pointwise numerical flux (operator.py:359-418)
  for (int idx = tid; idx < nt * nqf; idx += kThreads) {
    const int f = idx / nqf, q = idx - f * nqf;
    const int code = meta[f * 6];
    const bool mirror = code_mirror(code);
    const double* g = geo + f * NFG;
    const double sfac = g[2 * D], h = g[2 * D + 1], idet_in = g[2 * D + 2], idet_out = g[2 * D + 3];
    const double* tu_in = tr + (f * 4 + 0) * S * F;
    const double* tu_out = tr + (f * 4 + 1) * S * F;
    const double* tg_in = tr + (f * 4 + 2) * S * F;
    const double* tg_out = tr + (f * 4 + 3) * S * F;
    double ui[S], uo[S], gn[S], dU[S], qv[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      ui[s] = tu_in[s * F + q];
      const double gi = tg_in[s * F + q];
      if (mirror) {
        const double gd = p.ifbv ? p.ifbv[((f0 + f) * nqf + q) * S + s] : M::mirror_value(p.P, s);
        uo[s] = 2.0 * gd - ui[s];
        gn[s] = gi;
      } else {
        uo[s] = tu_out[s * F + q];
        gn[s] = 0.5 * (gi + tg_out[s * F + q]);
      }
      dU[s] = ui[s] - uo[s];
      qv[s] = 0.0;
    }
    if (p.scheme == IP) {
#pragma unroll
      for (int s = 0; s < S; ++s) qv[s] = (p.eta / h) * p.A[s] * dU[s];
    } else if (p.scheme != BO) {
      // lifting r_e(J) . n on the chosen side(s) (operator.py:336-357)
      const bool br2 = p.scheme == BR2;
      const bool use_in = mirror || br2 || code_minus_in(code);
      const bool use_out = !mirror && (br2 || !code_minus_in(code));
      const double wside = (br2 && !mirror) ? 0.5 : 1.0;
      double rho[S];
#pragma unroll
      for (int s = 0; s < S; ++s) rho[s] = 0.0;
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (side ? !use_out : !use_in) continue;
        const int t = side ? code_tout(code) : code_tin(code);
        const double* pw = p.fPw + (size_t(t) * nqf + q) * nqf;
        const double scale = wside * (-0.5 * sfac * (side ? idet_out : idet_in));
#pragma unroll
        for (int s = 0; s < S; ++s) {
          double a = 0.0;
          for (int pp = 0; pp < nqf; ++pp) {
            const double gd = !mirror ? 0.0
                              : (p.ifbv ? p.ifbv[((f0 + f) * nqf + pp) * S + s]
                                        : M::mirror_value(p.P, s));
            const double du = mirror ? 2.0 * (tu_in[s * F + pp] - gd)
                                     : tu_in[s * F + pp] - tu_out[s * F + pp];
            a = fma(__ldg(pw + pp), du, a);
          }
          rho[s] = fma(scale, a, rho[s]);
        }
      }
      const double fac = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e;
#pragma unroll
      for (int s = 0; s < S; ++s) qv[s] = -fac * p.A[s] * rho[s];
    }
    if constexpr (M::kConv) M::face_conv(p.P, ui, uo, gn, dU, qv);
    const double wq = __ldg(p.fw + q) * sfac;
    double* Y = yx + (f * 2 + 0) * S * F;
    double* X = yx + (f * 2 + 1) * S * F;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      Y[s * F + q] = wq * (p.A[s] * gn[s] - qv[s]);
      X[s * F + q] = wq * 0.5 * p.adj * p.A[s] * dU[s];
    }
  }
  __syncthreads();
  // test-function projection and conflict-free write of both sides
  for (int idx = tid; idx < nt * 2 * SN; idx += kThreads) {
    const int f = idx / (2 * SN), r = idx - f * 2 * SN, side = r / SN, si = r - side * SN;
    const int s = si / NB, i = si - s * NB;
    const int code = meta[f * 6];
    if (side && (code_mirror(code) || code_skip_out(code))) continue;
    const int t = side ? code_tout(code) : code_tin(code);
    const double* Y = yx + (f * 2 + 0) * S * F + s * F;
    const double* X = yx + (f * 2 + 1) * S * F + s * F;
    const double* dp = dph + (f * 2 + side) * F * NB + i;
    const double* b = p.fB + size_t(t) * nqf * NB + i;
    // inside row  +Y B_in + X dphin_in;  outside row  -Y B_out + X dphin_out
    const double sg = side ? -1.0 : 1.0;
    double acc = 0.0;
    for (int q = 0; q < nqf; ++q) {
      acc = fma(sg * Y[q], __ldg(b + q * NB), acc);
      acc = fma(X[q], dp[q * NB], acc);
    }
    const int64_t e = meta[f * 6 + 1 + side];
    acc_put(ACC + e * SN + si, acc, side ? code_first_out(code) : code_first_in(code));
  }
}

template <int D, int K, class M>
struct WallTile {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF;
  static constexpr int TF = 32;
  static constexpr size_t smem() { return size_t(TF) * (NB + 1 + 2 + S * F) * 8; }
};

template <int D, int K, class M>
__global__ void __launch_bounds__(kThreads)
k_wall(OpParams p, const double* __restrict__ U, double* __restrict__ ACC) {
  using T = WallTile<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, TF = T::TF;
  extern __shared__ double sm[];
  double* cw = sm;                 // [TF][NB]  coefficients of the gate species
  double* sf = cw + TF * NB;       // [TF]
  int* meta = reinterpret_cast<int*>(sf + TF);  // [TF][4] code, e
  double* yw = sf + TF + 2 * TF;   // [TF][S][F]
  const int tid = threadIdx.x;
  const int64_t f0 = int64_t(blockIdx.x) * TF;
  const int nt = int(p.nbf - f0 < TF ? p.nbf - f0 : TF);
  const int nqf = p.nqf;
  for (int f = tid; f < nt; f += kThreads) {
    meta[f * 4] = p.bfcode[f0 + f];
    meta[f * 4 + 1] = p.bfel[f0 + f];
    sf[f] = p.bfgeo[f0 + f];
  }
  __syncthreads();
  for (int idx = tid; idx < nt * NB; idx += kThreads) {
    const int f = idx / NB, i = idx - f * NB;
    cw[idx] = U[int64_t(meta[f * 4 + 1]) * SN + M::WALL_SP * NB + i];
  }
  __syncthreads();
  for (int idx = tid; idx < nt * nqf; idx += kThreads) {
    const int f = idx / nqf, q = idx - f * nqf;
    const int code = meta[f * 4];
    const double* b = p.fB + (size_t(code_tin(code)) * nqf + q) * NB;
    double c1 = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) c1 = fma(__ldg(b + i), cw[f * NB + i], c1);
    double qv[S];
    M::wall(p.P, code_tag(code), c1, qv);
    if (p.bfqv) {  // prescribed point data (heat models with x-dependent walls)
#pragma unroll
      for (int s = 0; s < S; ++s) qv[s] = p.bfqv[((f0 + f) * nqf + q) * S + s];
    }
    const double w = -__ldg(p.fw + q) * sf[f];
#pragma unroll
    for (int s = 0; s < S; ++s) yw[(f * S + s) * F + q] = w * qv[s];
  }
  __syncthreads();
  for (int idx = tid; idx < nt * SN; idx += kThreads) {
    const int f = idx / SN, si = idx - f * SN, s = si / NB, i = si - s * NB;
    const int code = meta[f * 4];
    const double* b = p.fB + size_t(code_tin(code)) * nqf * NB + i;
    double acc = 0.0;
    for (int q = 0; q < nqf; ++q) acc = fma(yw[(f * S + s) * F + q], __ldg(b + q * NB), acc);
    acc_put(ACC + int64_t(meta[f * 4 + 1]) * SN + si, acc, code_first_in(code));
  }
}

}  // namespace tdg

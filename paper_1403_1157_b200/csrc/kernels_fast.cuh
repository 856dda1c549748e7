// Register-resident operator kernels for the small-table cases (2D, and
// any (d, k, model) whose per-lane working set fits in registers).
//
// k_faces_fast  one lane per (face, species): a warp holds 32/S faces;
//               the S lanes of a face read the face's two contiguous
//               S*nb coefficient blocks coalesced, evaluate u and d_n u
//               at all face points in registers, exchange the few values
//               the species coupling needs (LLF wave speed, taxis flux)
//               with warp shuffles, and write the face's two FC blocks
//               coalesced.  Interior, Dirichlet-mirror and prescribed-flux
//               wall faces share the kernel (face index >= nif: wall).
//               Face tables (all (lf, perm) signatures, < 11 KB for 2D
//               k <= 3) live in shared memory; faces are sorted by
//               signature, so a warp's table reads are broadcasts.
// k_volume_fast one thread per element: the element's S*nb coefficients
//               sit in registers; volume tables are shared-memory
//               broadcasts; all global traffic (U, U0, the d+1 FC slot
//               tiles, the output) is staged through shared memory so
//               every HBM access is a coalesced tile.
#pragma once

#include "common.cuh"
#include "kernels.cuh"
#include "models.cuh"

namespace tdg {

template <int D, int K, class M>
struct FastFace {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF, NT = Dm::NT;
  static constexpr int FPW = 32 / S;          // faces per warp
  static constexpr int WARPS = 4;
  static constexpr int FPC = FPW * WARPS;     // faces per CTA
  static constexpr int TB = NT * F * NB, TG = NT * F * NB * D, TP = NT * F * F;
  static constexpr int TAB = TB + TG + TP + F;
  static constexpr bool ok = F <= 8 && S >= 3 && S <= 8 && TAB * 8 <= 40 * 1024 && NB <= 10;
};

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

template <int D, int K, class M>
__global__ void __launch_bounds__(128)
k_faces_fast(OpParams p, const double* __restrict__ U, double* __restrict__ FC) {
  using T = FastFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, FPW = T::FPW;
  constexpr int NFG = Dims<D, K>::NFG;
  __shared__ __align__(16) double tab[T::TAB];
  double* tB = tab;
  double* tG = tab + T::TB;
  double* tP = tG + T::TG;
  double* tw = tP + T::TP;
  for (int i = threadIdx.x; i < T::TB; i += 128) tB[i] = p.fB[i];
  for (int i = threadIdx.x; i < T::TG; i += 128) tG[i] = p.fG[i];
  for (int i = threadIdx.x; i < T::TP; i += 128) tP[i] = p.fPw[i];
  if (threadIdx.x < F) tw[threadIdx.x] = p.fw[threadIdx.x];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / S, s = lane - grp * S, base = grp * S;
  // warps [0, wi) take interior faces, warps [wi, ...) wall faces: every
  // warp is wholly interior or wholly wall, so the shuffles below are
  // always executed by all 32 lanes
  const int64_t gw = int64_t(blockIdx.x) * T::WARPS + warp;
  const int64_t wi = (p.nif + FPW - 1) / FPW;
  const bool wall = gw >= wi;
  const int64_t f = wall ? p.nif + (gw - wi) * FPW + grp : gw * FPW + grp;
  const bool active = grp < FPW && (wall ? f < p.nif + p.nbf : f < p.nif);
  if (!__any_sync(0xffffffffu, active)) return;  // warp-uniform

  int code = 0, ein = 0, eout = -1, lfi = 0, lfo = 0;
  double jin[D], jout[D], sfac = 0.0, h = 1.0, idi = 0.0, ido = 0.0;
#pragma unroll
  for (int a = 0; a < D; ++a) jin[a] = jout[a] = 0.0;
  if (active && !wall) {
    code = p.ifcode[f];
    ein = p.ifel[2 * f];
    eout = p.ifel[2 * f + 1];
    lfi = p.iflf[2 * f];
    lfo = p.iflf[2 * f + 1];
    const double* g = p.ifgeo + f * NFG;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      jin[a] = __ldg(g + a);
      jout[a] = __ldg(g + D + a);
    }
    sfac = __ldg(g + 2 * D);
    h = __ldg(g + 2 * D + 1);
    idi = __ldg(g + 2 * D + 2);
    ido = __ldg(g + 2 * D + 3);
  } else if (active) {
    const int64_t b = f - p.nif;
    code = p.bfcode[b];
    ein = p.bfel[b];
    lfi = p.bflf[b];
    sfac = __ldg(p.bfgeo + b);
  }
  const bool mirror = code_mirror(code);
  const int tin = code_tin(code), tout = code_tout(code);

  double ci[NB], co[NB];
  if (active) load_row<NB>(U + int64_t(ein) * SN + s * NB, ci);
  else {
#pragma unroll
    for (int i = 0; i < NB; ++i) ci[i] = 0.0;
  }
  const bool two = active && !wall && !mirror;
  if (two) load_row<NB>(U + int64_t(eout) * SN + s * NB, co);
  else {
#pragma unroll
    for (int i = 0; i < NB; ++i) co[i] = 0.0;
  }

  // traces at the face points: u and d_n u = sum_a jn_a (G_a . c)
  double ui[F], uo[F], gi[F], go[F];
  const double* Bi = tB + tin * F * NB;
  const double* Bo = tB + tout * F * NB;
  const double* Gi = tG + tin * F * NB * D;
  const double* Go = tG + tout * F * NB * D;
#pragma unroll
  for (int q = 0; q < F; ++q) {
    double u = 0.0, v = 0.0, ga[D], gb[D];
#pragma unroll
    for (int a = 0; a < D; ++a) ga[a] = gb[a] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      u = fma(Bi[q * NB + i], ci[i], u);
      v = fma(Bo[q * NB + i], co[i], v);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        ga[a] = fma(Gi[(q * NB + i) * D + a], ci[i], ga[a]);
        gb[a] = fma(Go[(q * NB + i) * D + a], co[i], gb[a]);
      }
    }
    double x = 0.0, y = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      x = fma(jin[a], ga[a], x);
      y = fma(jout[a], gb[a], y);
    }
    ui[q] = u;
    gi[q] = x;
    uo[q] = v;
    go[q] = y;
  }

  double ri[NB], ro[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) ri[i] = ro[i] = 0.0;

  if (!wall) {
    const double As = p.A[s];
    const double gD = M::mirror_value(p.P, s);
    if (mirror) {
#pragma unroll
      for (int q = 0; q < F; ++q) {
        uo[q] = 2.0 * gD - ui[q];
        go[q] = gi[q];
      }
    }
    double dU[F], gav[F], qv[F];
#pragma unroll
    for (int q = 0; q < F; ++q) {
      dU[q] = ui[q] - uo[q];
      gav[q] = 0.5 * (gi[q] + go[q]);
      qv[q] = 0.0;
    }
    // penalty A_hat . n (operator.py:336-357)
    if (p.scheme == IP) {
      const double c = p.eta / h * As;
#pragma unroll
      for (int q = 0; q < F; ++q) qv[q] = c * dU[q];
    } else if (p.scheme != BO) {
      const bool br2 = p.scheme == BR2;
      const bool use_in = mirror || br2 || code_minus_in(code);
      const bool use_out = !mirror && (br2 || !code_minus_in(code));
      const double wside = (br2 && !mirror) ? 0.5 : 1.0;
      const double fac = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * As;
      // -fac * A * rho, rho = -1/2 sfac/detJ * (Pw dU)
      const double si = use_in ? fac * wside * 0.5 * sfac * idi : 0.0;
      const double so = use_out ? fac * wside * 0.5 * sfac * ido : 0.0;
      const double* Pi = tP + tin * F * F;
      const double* Po = tP + tout * F * F;
#pragma unroll
      for (int q = 0; q < F; ++q) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int pp = 0; pp < F; ++pp) {
          a = fma(Pi[q * F + pp], dU[pp], a);
          b = fma(Po[q * F + pp], dU[pp], b);
        }
        qv[q] = si * a + so * b;
      }
    }
    // projection onto both sides' test functions
#pragma unroll
    for (int q = 0; q < F; ++q) {
      double conv = 0.0;
      if constexpr (M::kConv) {
        const double mui = ui[q], muo = uo[q], mg = gav[q];
        auto fetch = [&](int kind, int sp) {
          const double v = kind == 0 ? mui : (kind == 1 ? muo : mg);
          return __shfl_sync(0xffffffffu, v, base + sp);
        };
        conv = M::face_conv_lane(p.P, s, dU[q], fetch);
      }
      const double wq = tw[q] * sfac;
      const double Y = wq * (As * gav[q] - (qv[q] + conv));
      const double X = wq * 0.5 * p.adj * As * dU[q];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        double dpi = 0.0, dpo = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          dpi = fma(Gi[(q * NB + i) * D + a], jin[a], dpi);
          dpo = fma(Go[(q * NB + i) * D + a], jout[a], dpo);
        }
        ri[i] = fma(Y, Bi[q * NB + i], fma(X, dpi, ri[i]));
        ro[i] = fma(-Y, Bo[q * NB + i], fma(X, dpo, ro[i]));
      }
    }
  } else {
    // prescribed wall flux: only the gate species' trace is needed
    const int tag = code_tag(code);
#pragma unroll
    for (int q = 0; q < F; ++q) {
      const double c1 = __shfl_sync(0xffffffffu, ui[q], base + M::WALL_SP);
      const double Y = -tw[q] * sfac * M::wall_lane(p.P, tag, s, c1);
#pragma unroll
      for (int i = 0; i < NB; ++i) ri[i] = fma(Y, Bi[q * NB + i], ri[i]);
    }
  }
  if (active) {
    store_row<NB>(FC + (int64_t(lfi) * p.ne + ein) * SN + s * NB, ri);
    if (two && !code_skip_out(code))
      store_row<NB>(FC + (int64_t(lfo) * p.ne + eout) * SN + s * NB, ro);
  }
}

// ------------------------------------------------------------------ volume

template <int D, int K, class M>
struct FastVol {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, SNP = SN | 1, Q = Dm::NQV;
  static constexpr int NSYM = Dm::NSYM, NEG = Dm::NEG;
  static constexpr int TE = 128;
  static constexpr int TPHI = Q * NB, TGR = Q * NB * D, TKS = NSYM * NB * NB;
  static constexpr int TAB = TPHI + TGR + Q + TKS;
  static constexpr bool ok = SN <= 36 && TAB * 8 <= 24 * 1024;
  static constexpr size_t smem() { return size_t(TAB + 2 * TE * SNP) * 8; }
};

template <int D, int K, class M>
__global__ void __launch_bounds__(128)
k_volume_fast(OpParams p, const double* __restrict__ U, const double* __restrict__ FC,
              const double* U0, double* out, double ca, double cb, double cc, int mode) {
  using T = FastVol<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, SNP = T::SNP, Q = T::Q, TE = T::TE;
  constexpr int NEG = T::NEG, NSYM = T::NSYM;
  extern __shared__ __align__(16) double sm[];
  double* tphi = sm;
  double* tgr = tphi + T::TPHI;
  double* tw = tgr + T::TGR;
  double* tks = tw + Q;
  double* bufA = sm + T::TAB;
  double* bufB = bufA + TE * SNP;
  const int tid = threadIdx.x;
  const int64_t e0 = int64_t(blockIdx.x) * TE;
  const int nt = int(p.ne - e0 < TE ? p.ne - e0 : TE);

  for (int i = tid; i < T::TPHI; i += TE) tphi[i] = p.phi[i];
  for (int i = tid; i < T::TGR; i += TE) tgr[i] = p.grad[i];
  for (int i = tid; i < Q; i += TE) tw[i] = p.wv[i];
  for (int i = tid; i < T::TKS; i += TE) tks[i] = p.ks[i];
  // coalesced tile load of U (owned rows are contiguous)
  for (int idx = tid; idx < nt * SN; idx += TE) {
    const int e = idx / SN, r = idx - e * SN;
    bufA[e * SNP + r] = U[e0 * SN + idx];
  }
  __syncthreads();
  const bool act = tid < nt;
  double c[SN];
#pragma unroll
  for (int r = 0; r < SN; ++r) c[r] = bufA[tid * SNP + r];
  double ge[NEG];
#pragma unroll
  for (int k = 0; k < NEG; ++k) ge[k] = act ? __ldg(p.egeo + (e0 + tid) * NEG + k) : (k == 0 ? 1.0 : 0.0);

  // quadrature: taxis flux rows (pulled back) and the bilinear source
  constexpr int NF = M::NFLUX, NL = M::NNL;
  double af[NF > 0 ? NF : 1][NB], al[NL > 0 ? NL : 1][NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
#pragma unroll
    for (int k = 0; k < (NF > 0 ? NF : 1); ++k) af[k][i] = 0.0;
#pragma unroll
    for (int k = 0; k < (NL > 0 ? NL : 1); ++k) al[k][i] = 0.0;
  }
  if constexpr (NF + NL > 0) {
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
  }

  // residual rows: detJ (quadrature terms + linear source - A diffusion)
  const double detJ = ge[0];
  double* row = bufA + tid * SNP;  // own row: no sync needed to overwrite
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
      for (int t = 0; t < S; ++t) lin = fma(p.L[s * kMaxS + t], c[t * NB + i], lin);
      double acc = lin - p.A[s] * dif;
      if constexpr (NF > 0) {
        const int fi = M::flux_index(s);
        if (fi >= 0) acc += af[fi][i];
      }
      if constexpr (NL > 0) {
        const int li = M::nl_index(s);
        if (li >= 0) acc += al[li][i];
      }
      row[s * NB + i] = detJ * acc;
    }
  }
  // face-slot tiles (FC[lf] rows of this tile are contiguous)
#pragma unroll 1
  for (int lf = 0; lf <= D; ++lf) {
    __syncthreads();
    const double* src = FC + (int64_t(lf) * p.ne + e0) * SN;
    for (int idx = tid; idx < nt * SN; idx += TE) {
      const int e = idx / SN, r = idx - e * SN;
      bufB[e * SNP + r] = src[idx];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < SN; ++r) row[r] += bufB[tid * SNP + r];
  }
  const bool need_u0 = mode == 2 && ca != 0.0;
  if (need_u0) {
    __syncthreads();
    for (int idx = tid; idx < nt * SN; idx += TE) {
      const int e = idx / SN, r = idx - e * SN;
      bufB[e * SNP + r] = U0[e0 * SN + idx];
    }
    __syncthreads();
  }
  const double idet = 1.0 / detJ;
#pragma unroll
  for (int r = 0; r < SN; ++r) {
    const double rv = row[r];
    double o;
    if (mode == 0) o = rv;
    else if (mode == 1) o = rv * idet;
    else {
      o = fma(cb, c[r], cc * (rv * idet));
      if (need_u0) o = fma(ca, bufB[tid * SNP + r], o);
    }
    row[r] = o;
  }
  __syncthreads();
  for (int idx = tid; idx < nt * SN; idx += TE) {
    const int e = idx / SN, r = idx - e * SN;
    out[e0 * SN + idx] = bufA[e * SNP + r];
  }
}

}  // namespace tdg

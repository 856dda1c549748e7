// Interior faces on the FP64 tensor cores, transposed (3D).
//
// A warp owns a block of up to 8 interior faces with one trace-table
// signature (tables.tc_face_blocks): the faces are the M dimension of
// every mma.sync.m8n8k4.f64, so the signature's tables are the shared B
// operands and the per-face geometry (jn = Jinv n, lifting weight) scales
// the A operands lane by lane.  With g = lane>>2, t = lane&3 a lane owns
// face g; its accumulators hold columns 2t + j of the 8-column tiles:
//
//   traces      u[f][q]   = sum_k c[f][k] B[q][k]                  (B^T tables)
//               d_n u     = sum_a sum_k (jn_a c)[f][k] G_a[q][k]
//   lifting     m[f][n]   = kappa_f sum_q dU[f][q] w_q B[q][pi(n)]  (modal)
//               rho[f][q] = sum_i m[f][i] B[q][i]
//   projection  R[f][n]  += sum_q Y[f][q] B[q][pi(n)] + sum_qa (X jn_a)[f][q] G_a[q][pi(n)]
//
// Point quantities come out in the accumulator layout (face g, points
// 8qt + 2t + j) and feed the next GEMM as A operands one point parity at a
// time (k-step ks takes points 8qt + 2t + ks); the lifting coefficients
// feed rho the same way through the column permutation pi(8nt + 2t + j) =
// 4(2nt + j) + t.  No lane exchange, no warp barrier: pass A evaluates the
// coupled LLF physics (wave speed, taxis flux normals) per (face, point)
// into a lane-private shared-memory slice; pass B runs species by species
// (jumps -> modal lifting; traces, flux, projection) and writes the two
// face-slot rows.  Formulas as k_faces_fast / k_faces_mma (reference
// operator.py:326-434, flux.py:92-138); wall faces stay on k_faces_mma.
#pragma once

#include "common.cuh"
#include "kernels_mma.cuh"
#include "models.cuh"

namespace tdg {

template <int D, int K, class M>
struct TcFace {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF, NFG = Dm::NFG;
  static constexpr int QP = ceil_to(F, 8), QT = QP / 8;
  static constexpr int KT = (NB + 3) / 4, NBK = 4 * KT;
  static constexpr int NNT = (NB + 7) / 8, NBN = 8 * NNT;
  static constexpr int NCV = 1 + M::NFX;
  // per-signature table offsets (doubles), see tables.tc_face_tables; every
  // table is stored fragment-major ([k-step or point tile][...][lane]) so a
  // warp's B-operand load is 32 consecutive doubles (2 L1 wavefronts)
  static constexpr int OBT = 0, OGT = OBT + NBK * QP, OBP = OGT + D * NBK * QP,
                       OGP = OBP + QP * NBN, OWB = OGP + D * QP * NBN, TS = OWB + QP * NBN;
  static constexpr int WARPS = 4;
  static constexpr int PWS = 8 * QP * NCV;  // per-warp point-physics slice
  static constexpr size_t smem() { return size_t(WARPS) * PWS * 8; }
  static constexpr int MINB = 2;
  static constexpr bool ok = D == 3 && S <= kMaxS && smem() <= 96 * 1024;
};

// species the face point physics reads (values / averaged normal
// derivatives); the model's face_point fetches them by species index
template <class M>
struct TcfPhys {
  static constexpr int NV = M::NVAL, NG = M::NGRAD;
  __host__ __device__ static constexpr int val(int k) { return M::val_sp(k); }
  __host__ __device__ static constexpr int grad(int k) { return M::grad_sp(k); }
};
template <>
struct TcfPhys<PlaqueDev> {  // LLF wave speed needs n1 n2 c1 c3; d_n of n1 c1 c3
  static constexpr int NV = 4, NG = 3;
  __host__ __device__ static constexpr int val(int k) { return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 3 : 5; }
  __host__ __device__ static constexpr int grad(int k) { return k == 0 ? 0 : k == 1 ? 3 : 5; }
};

template <class M>
struct TcfPoint {
  double v[3][M::S];
  __device__ __forceinline__ double operator()(int kind, int sp) const { return v[kind][sp]; }
};

template <int D, int K, class M>
__global__ void __launch_bounds__(128, TcFace<D, K, M>::MINB)
k_faces_tc(OpParams p, const double* __restrict__ tabs, const int32_t* __restrict__ blocks,
           int64_t blk0, int64_t blk1, const double* __restrict__ U, double* __restrict__ FC) {
  using T = TcFace<D, K, M>;
  using PH = TcfPhys<M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, NFG = T::NFG;
  constexpr int QP = T::QP, QT = T::QT, KT = T::KT, NNT = T::NNT;
  constexpr int NCV = T::NCV, TS = T::TS;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  double* cvS = sm + warp * T::PWS + g * QP * NCV;  // this lane's face

  for (int64_t blk = blk0 + int64_t(blockIdx.x) * T::WARPS + warp; blk < blk1;
       blk += int64_t(gridDim.x) * T::WARPS) {
    const int2 bd = __ldg(reinterpret_cast<const int2*>(blocks) + blk);
    const bool active = g < bd.y;
    const int64_t f = int64_t(bd.x) + (active ? g : 0);
    const int code = __ldg(p.ifcode + f);
    const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + f);
    const int2 lf = __ldg(reinterpret_cast<const int2*>(p.iflf) + f);
    const double* gg = p.ifgeo + f * NFG;
    double jn[2][D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      jn[0][a] = __ldg(gg + a);
      jn[1][a] = __ldg(gg + D + a);
    }
    const double sfac = __ldg(gg + 2 * D), h = __ldg(gg + 2 * D + 1);
    const double idi = __ldg(gg + 2 * D + 2), ido = __ldg(gg + 2 * D + 3);
    const bool mirror = M::kMirror && code_mirror(code);
    // signature of the block (uniform): the B operands
    const int sig = __shfl_sync(0xffffffffu, code, 0) & 1023;
    const double* Ti = tabs + size_t(sig & 31) * TS;
    const double* To = tabs + size_t((sig >> 5) & 31) * TS;
    const double* ui_row = U + int64_t(el.x) * SN;
    const double* uo_row = U + int64_t(mirror ? el.x : el.y) * SN;

    // ---- pass A: coupled point physics -> lane-private slice -----------
    if constexpr (M::kConv) {
      constexpr int NV = PH::NV, NG = PH::NG;
      double ci[NV][KT], co[NV][KT];
#pragma unroll
      for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const bool in = 4 * kt + t < NB;
          ci[k][kt] = in ? __ldg(ui_row + PH::val(k) * NB + 4 * kt + t) : 0.0;
          co[k][kt] = in ? __ldg(uo_row + PH::val(k) * NB + 4 * kt + t) : 0.0;
        }
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        double vi[NV][2], vo[NV][2], di[NG][2], dq[NG][2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
#pragma unroll
          for (int k = 0; k < NV; ++k) vi[k][j] = vo[k][j] = 0.0;
#pragma unroll
          for (int k = 0; k < NG; ++k) di[k][j] = dq[k][j] = 0.0;
        }
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const double bi = __ldg(Ti + T::OBT + (kt * QT + qt) * 32 + lane);
          const double bo = __ldg(To + T::OBT + (kt * QT + qt) * 32 + lane);
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            dmma(vi[k][0], vi[k][1], ci[k][kt], bi);
            dmma(vo[k][0], vo[k][1], co[k][kt], bo);
          }
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const double gi = __ldg(Ti + T::OGT + ((a * KT + kt) * QT + qt) * 32 + lane);
            const double go = __ldg(To + T::OGT + ((a * KT + kt) * QT + qt) * 32 + lane);
#pragma unroll
            for (int k = 0; k < NG; ++k) {
              int kv = 0;
#pragma unroll
              for (int j2 = 0; j2 < NV; ++j2)
                if (PH::val(j2) == PH::grad(k)) kv = j2;
              dmma(di[k][0], di[k][1], ci[kv][kt] * jn[0][a], gi);
              dmma(dq[k][0], dq[k][1], co[kv][kt] * jn[1][a], go);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          TcfPoint<M> pt;
#pragma unroll
          for (int k = 0; k < NV; ++k) {
            pt.v[0][PH::val(k)] = vi[k][j];
            pt.v[1][PH::val(k)] = mirror ? 2.0 * M::mirror_value(p.P, PH::val(k)) - vi[k][j] : vo[k][j];
          }
#pragma unroll
          for (int k = 0; k < NG; ++k)
            pt.v[2][PH::grad(k)] = mirror ? di[k][j] : 0.5 * (di[k][j] + dq[k][j]);
          double cv[NCV];
          M::face_point(p.P, pt, cv);
          const int q = 8 * qt + 2 * t + j;
#pragma unroll
          for (int c = 0; c < NCV; ++c) cvS[q * NCV + c] = cv[c];
        }
      }
    }

    // lifting weights per side (operator.py:336-357)
    const bool br2 = p.scheme == BR2;
    const bool lift = p.scheme != IP && p.scheme != BO;
    const bool use_in = lift && (mirror || br2 || code_minus_in(code));
    const bool use_out = lift && !mirror && (br2 || !code_minus_in(code));
    const double wside = (br2 && !mirror) ? 0.5 : 1.0;
    const double fac0 = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * wside * 0.5 * sfac;
    const bool skip_out = !active || mirror || code_skip_out(code);
    double* fci = FC + (int64_t(lf.x) * p.ne + el.x) * SN;
    double* fco = FC + (int64_t(lf.y) * p.ne + el.y) * SN;

    // ---- pass B: species by species ------------------------------------
#pragma unroll 1
    for (int s = 0; s < S; ++s) {
      const double As = p.A[s];
      const double gs = M::kMirror ? M::mirror_value(p.P, s) : 0.0;
      double ci[KT], co[KT];
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const bool in = 4 * kt + t < NB;
        ci[kt] = in ? __ldg(ui_row + s * NB + 4 * kt + t) : 0.0;
        co[kt] = in ? __ldg(uo_row + s * NB + 4 * kt + t) : 0.0;
      }
      // B1: jumps -> modal lifting coefficients m_in, m_out
      double mi[NNT][2], mo[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) mi[nt][0] = mi[nt][1] = mo[nt][0] = mo[nt][1] = 0.0;
      if (lift) {
#pragma unroll 1
        for (int qt = 0; qt < QT; ++qt) {
          double ui[2] = {0.0, 0.0}, uo[2] = {0.0, 0.0};
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
              dmma(ui[0], ui[1], ci[kt], __ldg(Ti + T::OBT + (kt * QT + qt) * 32 + lane));
            dmma(uo[0], uo[1], co[kt], __ldg(To + T::OBT + (kt * QT + qt) * 32 + lane));
          }
          double du[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) du[j] = mirror ? 2.0 * (ui[j] - gs) : ui[j] - uo[j];
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt) {
              dmma(mi[nt][0], mi[nt][1], du[ks], __ldg(Ti + T::OWB + ((qt * 2 + ks) * NNT + nt) * 32 + lane));
              dmma(mo[nt][0], mo[nt][1], du[ks], __ldg(To + T::OWB + ((qt * 2 + ks) * NNT + nt) * 32 + lane));
            }
          }
        }
        const double ki = use_in ? fac0 * As * idi : 0.0;
        const double ko = use_out ? fac0 * As * ido : 0.0;
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mi[nt][j] *= ki;
            mo[nt][j] *= ko;
          }
      }
      // B2: traces, flux, projection
      // separate accumulators for the Y and X terms (shorter DMMA chains)
      double ri[NNT][2], ro[NNT][2], rix[NNT][2], rox[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) ri[nt][j] = ro[nt][j] = rix[nt][j] = rox[nt][j] = 0.0;
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        double ui[2] = {0.0, 0.0}, uo[2] = {0.0, 0.0};
        double dia[D][2], dqa[D][2];
        double rhi[2] = {0.0, 0.0}, rho_[2] = {0.0, 0.0};
#pragma unroll
        for (int a = 0; a < D; ++a) dia[a][0] = dia[a][1] = dqa[a][0] = dqa[a][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const double bi = __ldg(Ti + T::OBT + (kt * QT + qt) * 32 + lane);
          const double bo = __ldg(To + T::OBT + (kt * QT + qt) * 32 + lane);
          dmma(ui[0], ui[1], ci[kt], bi);
          dmma(uo[0], uo[1], co[kt], bo);
          if (lift) {
            // m as A operand: k-step kt holds basis 4 kt + t = pi(8 (kt/2) + 2t + kt%2)
            dmma(rhi[0], rhi[1], mi[kt / 2][kt % 2], bi);
            dmma(rho_[0], rho_[1], mo[kt / 2][kt % 2], bo);
          }
#pragma unroll
          for (int a = 0; a < D; ++a) {
            dmma(dia[a][0], dia[a][1], ci[kt] * jn[0][a], __ldg(Ti + T::OGT + ((a * KT + kt) * QT + qt) * 32 + lane));
            dmma(dqa[a][0], dqa[a][1], co[kt] * jn[1][a], __ldg(To + T::OGT + ((a * KT + kt) * QT + qt) * 32 + lane));
          }
        }
        double di[2], dq[2], rho[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          di[j] = dia[0][j];
          dq[j] = dqa[0][j];
#pragma unroll
          for (int a = 1; a < D; ++a) {
            di[j] += dia[a][j];
            dq[j] += dqa[a][j];
          }
          rho[j] = rhi[j] + rho_[j];
        }
        double Y[2], X[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 8 * qt + 2 * t + j;
          const double uoj = mirror ? 2.0 * gs - ui[j] : uo[j];
          const double du = ui[j] - uoj;
          const double gav = mirror ? di[j] : 0.5 * (di[j] + dq[j]);
          double qv = rho[j];
          if (p.scheme == IP) qv = p.eta / h * As * du;
          if constexpr (M::kConv) {
            double cnv = 0.5 * cvS[q * NCV] * du;
#pragma unroll
            for (int k = 0; k < M::NFX; ++k)
              if (s == k) cnv = fma(0.5, cvS[q * NCV + 1 + k], cnv);
            qv += cnv;
          }
          const double wq = q < F ? __ldg(p.fw + q) * sfac : 0.0;
          Y[j] = wq * (As * gav - qv);
          X[j] = wq * 0.5 * p.adj * As * du;
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
          for (int nt = 0; nt < NNT; ++nt) {
            dmma(ri[nt][0], ri[nt][1], Y[ks], __ldg(Ti + T::OBP + ((qt * 2 + ks) * NNT + nt) * 32 + lane));
            dmma(ro[nt][0], ro[nt][1], -Y[ks], __ldg(To + T::OBP + ((qt * 2 + ks) * NNT + nt) * 32 + lane));
#pragma unroll
            for (int a = 0; a < D; ++a) {
              dmma(rix[nt][0], rix[nt][1], X[ks] * jn[0][a], __ldg(Ti + T::OGP + (((a * QT + qt) * 2 + ks) * NNT + nt) * 32 + lane));
              dmma(rox[nt][0], rox[nt][1], X[ks] * jn[1][a], __ldg(To + T::OGP + (((a * QT + qt) * 2 + ks) * NNT + nt) * 32 + lane));
            }
          }
        }
      }
      // face-slot rows: lane entries (face g, basis 4 (2nt + j) + t)
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = 4 * (2 * nt + j) + t;
          if (i < NB) {
            if (active) fci[s * NB + i] = ri[nt][j] + rix[nt][j];
            if (!skip_out) fco[s * NB + i] = ro[nt][j] + rox[nt][j];
          }
        }
    }
  }
}

// ---------------------------------------------------------------------
// Interior faces on the FP64 tensor cores with the SPECIES as the M
// dimension: a warp runs one face at a time (the faces of one block share
// the trace-table signature), rows g = species, so everything per face --
// Jinv n of both sides, the lifting weight, h -- is warp-uniform.  That
// lets the normal derivatives fold into the B operand: the fragment of
// dphi/dn = sum_a jn_a G_a is 3 FMAs per lane, replacing the D separate
// DMMAs of the face-rows kernel above, and the coupled point physics reads
// the traces of every species from one shared-memory transpose instead of
// recomputing them (the face-rows kernel's pass A).  Same signature tables
// (tables.tc_face_tables), same point-parity k-steps and mode permutation
// pi(8nt + 2t + j) = 4(2nt + j) + t; with nb = 10, F = 35 (C4) a face takes
// ~175 DMMAs instead of ~330.
//
//   pass 1 (point tiles qt): u_in, u_out, d_n u_in, d_n u_out for all
//          species -> transpose xs[kind][q][s]; jumps -> modal lifting m
//   physics: LLF wave speed / taxis flux normals once per point -> cv[q]
//   pass 2 (point tiles qt): rho = m B, Y and X per (species, point),
//          projection onto both sides' test functions (B and folded dphi/dn)
template <int D, int K, class M>
struct TcsFace {
  using TF = TcFace<D, K, M>;
  static constexpr int NB = TF::NB, S = M::S, SN = S * NB, F = TF::F, NFG = TF::NFG;
  static constexpr int QP = TF::QP, QT = TF::QT, KT = TF::KT, NNT = TF::NNT, TS = TF::TS;
  static constexpr int NCV = TF::NCV, XS = S | 1;
  // the last mode tile holds at most 4 modes (nb = 10: 2, nb = 20: 4),
  // all in its even columns: both sides' projections share one DMMA pair
  static constexpr bool MERGE = NNT >= 2 && NB - 8 * (NNT - 1) <= 4;
  static constexpr int WARPS = 4;
  static constexpr int PWS = 3 * QP * XS + QP * NCV + 1;  // per-warp scratch (doubles)
  static constexpr size_t smem() { return size_t(WARPS) * PWS * 8; }
  // 128 registers (16 warps/SM): 3 -> 4 cut C4 faces 21.6 -> 18.6 ms; 5 spills
  static constexpr int MINB = K >= 3 ? 3 : 4;
  static constexpr bool ok = D == 3 && S <= 8 && !M::kMirror && TF::ok && smem() <= 96 * 1024;
};

template <int D, int K, class M>
__global__ void __launch_bounds__(128, TcsFace<D, K, M>::MINB)
k_faces_tcs(OpParams p, const double* __restrict__ tabs, const int32_t* __restrict__ blocks,
            int64_t blk0, int64_t blk1, const double* __restrict__ U, double* __restrict__ FC) {
  using T = TcsFace<D, K, M>;
  using TF = TcFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, NFG = T::NFG;
  constexpr int QP = T::QP, QT = T::QT, KT = T::KT, NNT = T::NNT, TS = T::TS;
  constexpr int NCV = T::NCV, XS = T::XS;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const bool row = g < S;  // this lane's species row is real
  const int sp = row ? g : 0;
  double* xs = sm + warp * T::PWS;  // [3][QP][XS]: u_in, u_out, avg d_n u
  double* cv = xs + 3 * QP * XS;    // [QP][NCV]
  const double As = p.A[sp];

  for (int64_t blk = blk0 + int64_t(blockIdx.x) * T::WARPS + warp; blk < blk1;
       blk += int64_t(gridDim.x) * T::WARPS) {
    const int2 bd = __ldg(reinterpret_cast<const int2*>(blocks) + blk);
#pragma unroll 1
    for (int fi = 0; fi < bd.y; ++fi) {
      const int64_t f = int64_t(bd.x) + fi;
      const int code = __ldg(p.ifcode + f);
      const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + f);
      const int2 lf = __ldg(reinterpret_cast<const int2*>(p.iflf) + f);
      const double* gg = p.ifgeo + f * NFG;
      double jn[2][D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        jn[0][a] = __ldg(gg + a);
        jn[1][a] = __ldg(gg + D + a);
      }
      const double sfac = __ldg(gg + 2 * D), h = __ldg(gg + 2 * D + 1);
      const double idi = __ldg(gg + 2 * D + 2), ido = __ldg(gg + 2 * D + 3);
      const int sig = code & 1023;
      const double* Ti = tabs + size_t(sig & 31) * TS;
      const double* To = tabs + size_t((sig >> 5) & 31) * TS;
      // A operands: this face's coefficients, row = species g, k = 4 kt + t
      double ci[KT], co[KT];
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const bool in = row && 4 * kt + t < NB;
        ci[kt] = in ? __ldg(U + int64_t(el.x) * SN + g * NB + 4 * kt + t) : 0.0;
        co[kt] = in ? __ldg(U + int64_t(el.y) * SN + g * NB + 4 * kt + t) : 0.0;
      }
      const bool br2 = p.scheme == BR2;
      const bool lift = p.scheme != IP && p.scheme != BO;
      const bool use_in = lift && (br2 || code_minus_in(code));
      const bool use_out = lift && (br2 || !code_minus_in(code));

      // ---- pass 1: traces, transpose, jumps -> modal lifting -------------
      double mi[NNT][2], mo[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) mi[nt][0] = mi[nt][1] = mo[nt][0] = mo[nt][1] = 0.0;
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        double ui[2] = {0.0, 0.0}, uo[2] = {0.0, 0.0}, di[2] = {0.0, 0.0}, dq[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int ob = (kt * QT + qt) * 32 + lane;
          dmma(ui[0], ui[1], ci[kt], __ldg(Ti + TF::OBT + ob));
          dmma(uo[0], uo[1], co[kt], __ldg(To + TF::OBT + ob));
          double gi = 0.0, go = 0.0;  // dphi/dn fragments (jn folded in)
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const int og = ((a * KT + kt) * QT + qt) * 32 + lane;
            gi = fma(jn[0][a], __ldg(Ti + TF::OGT + og), gi);
            go = fma(jn[1][a], __ldg(To + TF::OGT + og), go);
          }
          dmma(di[0], di[1], ci[kt], gi);
          dmma(dq[0], dq[1], co[kt], go);
        }
        double du[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 8 * qt + 2 * t + j;
          du[j] = ui[j] - uo[j];
          if (row) {
            xs[(0 * QP + q) * XS + g] = ui[j];
            xs[(1 * QP + q) * XS + g] = uo[j];
            xs[(2 * QP + q) * XS + g] = 0.5 * (di[j] + dq[j]);
          }
        }
        if (lift) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt) {
              const int ow = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
              if (use_in) dmma(mi[nt][0], mi[nt][1], du[ks], __ldg(Ti + TF::OWB + ow));
              if (use_out) dmma(mo[nt][0], mo[nt][1], du[ks], __ldg(To + TF::OWB + ow));
            }
        }
      }
      // lifting weights (operator.py:336-357): -fac A rho, rho = -1/2 sfac/detJ Pw dU
      {
        const double wside = br2 ? 0.5 : 1.0;
        const double fac0 = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * wside * 0.5 * sfac * As;
        const double ki = use_in ? fac0 * idi : 0.0, ko = use_out ? fac0 * ido : 0.0;
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mi[nt][j] *= ki;
            mo[nt][j] *= ko;
          }
      }
      __syncwarp();
      // ---- coupled point physics, once per face point ---------------------
      if constexpr (M::kConv) {
        for (int q = lane; q < F; q += 32) {
          const double* xq = xs + q * XS;
          auto fetch = [xq](int kind, int s2) { return xq[kind * QP * XS + s2]; };
          M::face_point(p.P, fetch, cv + q * NCV);
        }
        __syncwarp();
      }
      // ---- pass 2: rho, flux, projection ---------------------------------
      double ri[NNT][2], ro[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) ri[nt][0] = ri[nt][1] = ro[nt][0] = ro[nt][1] = 0.0;
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        double rho[2] = {0.0, 0.0};
        if (lift) {
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const int ob = (kt * QT + qt) * 32 + lane;
            // m as A operand: k-step kt holds basis 4 kt + t = pi(8 (kt/2) + 2t + kt%2)
            if (use_in) dmma(rho[0], rho[1], mi[kt / 2][kt % 2], __ldg(Ti + TF::OBT + ob));
            if (use_out) dmma(rho[0], rho[1], mo[kt / 2][kt % 2], __ldg(To + TF::OBT + ob));
          }
        }
        double Y[2], X[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = 8 * qt + 2 * t + j;
          const double du = xs[q * XS + sp] - xs[(QP + q) * XS + sp];
          const double gav = xs[(2 * QP + q) * XS + sp];
          double qv = rho[j];
          if (p.scheme == IP) qv = p.eta / h * As * du;
          if constexpr (M::kConv) {
            if (q < F) {
              double cnv = 0.5 * cv[q * NCV] * du;
#pragma unroll
              for (int k = 0; k < M::NFX; ++k)
                if (g == k) cnv = fma(0.5, cv[q * NCV + 1 + k], cnv);
              qv += cnv;
            }
          }
          const double wq = (q < F && row) ? __ldg(p.fw + q) * sfac : 0.0;
          Y[j] = wq * (As * gav - qv);
          X[j] = wq * 0.5 * p.adj * As * du;
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int nt = 0; nt < NNT; ++nt) {
            if (T::MERGE && nt == NNT - 1) {
              // merged tail tile: the even B columns (C j = 0) carry the
              // in-side modes, the odd ones (j = 1, modes past nb) the
              // out-side ones (normal-layout lane - 4, sign of Y folded
              // in), so one DMMA pair serves both sides
              const bool oc = (g & 1) != 0;
              const double* Tx = oc ? To : Ti;
              const int ln = oc ? lane - 4 : lane;
              const int ob = ((qt * 2 + ks) * NNT + nt) * 32 + ln;
              double gx = 0.0;
#pragma unroll
              for (int a = 0; a < D; ++a) {
                const int og = (((a * QT + qt) * 2 + ks) * NNT + nt) * 32 + ln;
                gx = fma(oc ? jn[1][a] : jn[0][a], __ldg(Tx + TF::OGP + og), gx);
              }
              const double bx = __ldg(Tx + TF::OBP + ob);
              dmma(ri[nt][0], ri[nt][1], Y[ks], oc ? -bx : bx);
              dmma(ri[nt][0], ri[nt][1], X[ks], gx);
              continue;
            }
            const int ob = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
            double gi = 0.0, go = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              const int og = (((a * QT + qt) * 2 + ks) * NNT + nt) * 32 + lane;
              gi = fma(jn[0][a], __ldg(Ti + TF::OGP + og), gi);
              go = fma(jn[1][a], __ldg(To + TF::OGP + og), go);
            }
            dmma(ri[nt][0], ri[nt][1], Y[ks], __ldg(Ti + TF::OBP + ob));
            dmma(ri[nt][0], ri[nt][1], X[ks], gi);
            dmma(ro[nt][0], ro[nt][1], -Y[ks], __ldg(To + TF::OBP + ob));
            dmma(ro[nt][0], ro[nt][1], X[ks], go);
          }
      }
      // face-slot rows: lane entries (species g, basis 4 (2nt + j) + t)
      const bool skip_out = code_skip_out(code);
      if (row) {
        double* fci = FC + (int64_t(lf.x) * p.ne + el.x) * SN + g * NB;
        double* fco = FC + (int64_t(lf.y) * p.ne + el.y) * SN + g * NB;
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (T::MERGE && nt == NNT - 1) {  // j = 0: in-side mode, j = 1: out-side
              const int i = 8 * nt + t;
              if (i < NB) {
                if (j == 0)
                  fci[i] = ri[nt][0];
                else if (!skip_out)
                  fco[i] = ri[nt][1];
              }
              continue;
            }
            const int i = 4 * (2 * nt + j) + t;
            if (i < NB) {
              fci[i] = ri[nt][j];
              if (!skip_out) fco[i] = ro[nt][j];
            }
          }
      }
      __syncwarp();  // xs / cv are rewritten by the next face
    }
  }
}

}  // namespace tdg

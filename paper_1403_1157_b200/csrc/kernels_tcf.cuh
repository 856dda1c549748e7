// Interior faces on the FP64 tensor cores (3D), transposed: the face's
// contractions run as mma.sync.m8n8k4.f64 (DMMA) with the trace-table
// signature's tables as the B operands (tables.tc_face_tables, stored
// fragment-major so a warp's B-operand load is 32 consecutive doubles).
// The faces come in blocks of up to 8 with one signature
// (tables.tc_face_blocks) inside one colour segment; the kernel adds each
// face side's contribution to the element's face-sum row.  Formulas as
// k_faces_fast / k_faces_mma (reference operator.py:326-434,
// flux.py:92-138); wall faces run on k_faces_mma.
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
  // per-signature table offsets (doubles), see tables.tc_face_tables.
  // Fragment-major ([k-step or point tile][...][lane]); the trace (TR) and
  // projection (PR) blocks interleave each B fragment with its three
  // gradient fragments ([...][lane][B, G0, G1, G2]: one 32-byte load per
  // lane), WB / BT are plain ([...][lane]: one 8-byte load per lane)
  // (3D: 1 + D = 4 doubles per lane and fragment)
  static constexpr int OTR = 0, OPR = OTR + (1 + D) * NBK * QP, OWB = OPR + (1 + D) * QP * NBN,
                       OBT = OWB + QP * NBN, TS = OBT + NBK * QP;
  // face-geometry-class tables (tables.tc_face_fold_tables): per (table id,
  // Jinv n) class the B fragment paired with the folded normal-derivative
  // fragment sum_a jn_a G_a ([...][lane][B, G_n]: one 16-byte load per lane)
  // plus the projection fragments split by kind ([...][lane]: one 8-byte
  // load per lane) for the face-group kernel's merged tail tile, which
  // needs one kind from the inside and the other from the outside lanes
  static constexpr int OTRF = 0, OPRF = OTRF + 2 * NBK * QP, OPBF = OPRF + 2 * QP * NBN,
                       OPGF = OPBF + QP * NBN, TSF = OPGF + QP * NBN;
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

// ---------------------------------------------------------------------
// Interior faces on the FP64 tensor cores with the SPECIES as the M
// dimension: a warp runs one face at a time (the faces of one block share
// the trace-table signature), rows g = species, so everything per face --
// Jinv n of both sides, the lifting weight, h -- is warp-uniform.  That
// lets the normal derivatives fold into the B operand: the fragment of
// dphi/dn = sum_a jn_a G_a is 3 FMAs per lane, replacing D separate DMMAs
// with jn in the A operand (a faces-as-rows layout), and the coupled point
// physics reads the traces of every species from one shared-memory
// transpose instead of recomputing them.  Same signature tables
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
  // species transpose row stride: lane (g, t) of a pass-1 store hits
  // double q XS + g with q = 8 qt + 2 t + j; XS = 6 maps each half-warp's
  // 16 (g, t) onto 16 distinct banks (S | 1 = 7 was 3-way conflicted;
  // measured time-neutral, less shared memory)
  static constexpr int NCV = TF::NCV, XS = S == 6 ? 6 : (S | 1);
  // the last mode tile holds at most 4 modes (nb = 10: 2, nb = 20: 4),
  // all in its even columns: both sides' projections share one DMMA pair
  static constexpr bool MERGE = NNT >= 2 && NB - 8 * (NNT - 1) <= 4;
  static constexpr int WARPS = 4;
  static constexpr int PWS = 3 * QP * XS + QP * NCV + 1;  // per-warp scratch (doubles)
  static constexpr size_t smem() { return size_t(WARPS) * PWS * 8; }
  // 128 registers (16 warps/SM): 3 -> 4 cut C4 faces 21.6 -> 18.6 ms; 5 spills.
  // p = 3 folding Jinv n per face needs 168 registers (3 CTAs/SM); with the
  // face-geometry-class tables it fits 128 without spills (64^3 p = 3:
  // 38.4 ms at 3 CTAs without classes -> 31.6 with -> 30.0 at 4 CTAs)
  static constexpr int MINB = K >= 3 ? 3 : 4;
  static constexpr int MINB_FOLD = 4;  // p = 2 at 5 CTAs (96 registers, spills): no gain
  static constexpr bool ok = D == 3 && S <= 8 && !M::kMirror && TF::ok && smem() <= 96 * 1024;
};

// FOLD: the normal-derivative fragments come precomputed per face-geometry
// class (meshes with few distinct (table, Jinv n) pairs, e.g. the Kuhn
// cubes: 6 per side); otherwise they are folded per face from jn
// LM: lifting sides of the scheme (operator.py:336-357), a compile-time
// constant so no DMMA chain is issued predicated-off (they still occupy the
// tensor pipe: 64^3 p = 3 faces 28.5 -> 26.6 ms for the first of them):
// 0 none (ip, bo), 1 the K- side (cdg2, cdg), 2 both (br2)
template <int D, int K, class M, bool FOLD, int LM>
__global__ void __launch_bounds__(128, FOLD ? TcsFace<D, K, M>::MINB_FOLD : TcsFace<D, K, M>::MINB)
k_faces_tcs(OpParams p, const double* __restrict__ tabs, const int32_t* __restrict__ blocks,
            int64_t blk0, int64_t blk1, const double* __restrict__ U, double* __restrict__ ACC) {
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
      const double* gg = p.ifgeo + f * NFG;
      double jn[2][D];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        jn[0][a] = FOLD ? 0.0 : __ldg(gg + a);
        jn[1][a] = FOLD ? 0.0 : __ldg(gg + D + a);
      }
      const double sfac = __ldg(gg + 2 * D), h = __ldg(gg + 2 * D + 1);
      const double idi = __ldg(gg + 2 * D + 2), ido = __ldg(gg + 2 * D + 3);
      const int sig = code & 1023;
      const double* Ti = tabs + size_t(sig & 31) * TS;
      const double* To = tabs + size_t((sig >> 5) & 31) * TS;
      const double* Fi = nullptr;
      const double* Fo = nullptr;
      if constexpr (FOLD) {
        const int2 cl = __ldg(reinterpret_cast<const int2*>(p.ffold) + f);
        Fi = p.ftf + size_t(cl.x) * TF::TSF;
        Fo = p.ftf + size_t(cl.y) * TF::TSF;
      }
      // A operands: this face's coefficients, row = species g, k = 4 kt + t
      double ci[KT], co[KT];
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const bool in = row && 4 * kt + t < NB;
        ci[kt] = in ? __ldg(U + int64_t(el.x) * SN + g * NB + 4 * kt + t) : 0.0;
        co[kt] = in ? __ldg(U + int64_t(el.y) * SN + g * NB + 4 * kt + t) : 0.0;
      }
      constexpr bool br2 = LM == 2;
      constexpr bool lift = LM > 0;
      // lifting side(s) (operator.py:336-357): K- only (cdg2 / cdg), both
      // for br2; mi runs on table Tl (K- side, or the inside for br2), mo
      // on the outside for br2 only -- no predicated-off DMMA chains
      const bool min_ = code_minus_in(code);
      const double* Tl = (br2 || min_) ? Ti : To;

      // ---- pass 1: traces, transpose, jumps -> modal lifting -------------
      double mi[NNT][2], mo[NNT][2];
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt) mi[nt][0] = mi[nt][1] = mo[nt][0] = mo[nt][1] = 0.0;
#pragma unroll 1
      for (int qt = 0; qt < QT; ++qt) {
        double ui[2] = {0.0, 0.0}, uo[2] = {0.0, 0.0}, di[2] = {0.0, 0.0}, dq[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          double fi[4], fo[4];  // B, G0, G1, G2 fragments of both sides (FOLD: B, G_n)
          double gi, go;        // dphi/dn fragments (jn folded in)
          if constexpr (FOLD) {
            const int ob = 2 * ((kt * QT + qt) * 32 + lane);
            ld128(Fi + TF::OTRF + ob, fi);
            ld128(Fo + TF::OTRF + ob, fo);
            gi = fi[1];
            go = fo[1];
          } else {
            const int ob = 4 * ((kt * QT + qt) * 32 + lane);
            ld256(Ti + TF::OTR + ob, fi);
            ld256(To + TF::OTR + ob, fo);
            gi = fma(jn[0][2], fi[3], fma(jn[0][1], fi[2], jn[0][0] * fi[1]));
            go = fma(jn[1][2], fo[3], fma(jn[1][1], fo[2], jn[1][0] * fo[1]));
          }
          dmma(ui[0], ui[1], ci[kt], fi[0]);
          dmma(uo[0], uo[1], co[kt], fo[0]);
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
        if constexpr (lift) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt) {
              const int ow = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
              dmma(mi[nt][0], mi[nt][1], du[ks], __ldg(Tl + TF::OWB + ow));
            }
        }
        if constexpr (br2) {
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int nt = 0; nt < NNT; ++nt) {
              const int ow = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
              dmma(mo[nt][0], mo[nt][1], du[ks], __ldg(To + TF::OWB + ow));
            }
        }
      }
      // lifting weights (operator.py:336-357): -fac A rho, rho = -1/2 sfac/detJ Pw dU
      {
        const double wside = br2 ? 0.5 : 1.0;
        const double fac0 = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * wside * 0.5 * sfac * As;
        const double ki = lift ? fac0 * ((br2 || min_) ? idi : ido) : 0.0;
        const double ko = br2 ? fac0 * ido : 0.0;
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
        if constexpr (lift) {
          // two independent accumulator chains (even / odd k-steps): the
          // flux of this point tile waits on rho, so halve its DMMA chain
          // (64^3 p = 3: faces 29.7 -> 28.5 ms; splitting pass 1's four
          // trace chains the same way measured 28.8, and issuing the next
          // tile's rho ahead of this tile's projection 29.3: 20 B spills)
          double rb[2] = {0.0, 0.0};
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const int ob = (kt * QT + qt) * 32 + lane;
            double* r = (kt & 1) ? rb : rho;
            // m as A operand: k-step kt holds basis 4 kt + t = pi(8 (kt/2) + 2t + kt%2)
            dmma(r[0], r[1], mi[kt / 2][kt % 2], __ldg(Tl + TF::OBT + ob));
          }
          if constexpr (br2) {
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
              const int ob = (kt * QT + qt) * 32 + lane;
              double* r = (kt & 1) ? rb : rho;
              dmma(r[0], r[1], mo[kt / 2][kt % 2], __ldg(To + TF::OBT + ob));
            }
          }
          rho[0] += rb[0];
          rho[1] += rb[1];
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
              const int ln = oc ? lane - 4 : lane;
              const int of = ((qt * 2 + ks) * NNT + nt) * 32 + ln;
              double fx[4], gx;
              if constexpr (FOLD) {
                ld128((oc ? Fo : Fi) + TF::OPRF + 2 * of, fx);
                gx = fx[1];
              } else {
                ld256((oc ? To : Ti) + TF::OPR + 4 * of, fx);
                const double* jx = oc ? jn[1] : jn[0];
                gx = fma(jx[2], fx[3], fma(jx[1], fx[2], jx[0] * fx[1]));
              }
              const double bx = fx[0];
              dmma(ri[nt][0], ri[nt][1], Y[ks], oc ? -bx : bx);
              dmma(ri[nt][0], ri[nt][1], X[ks], gx);
              continue;
            }
            const int of = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
            double fi[4], fo[4], gi, go;
            if constexpr (FOLD) {
              ld128(Fi + TF::OPRF + 2 * of, fi);
              ld128(Fo + TF::OPRF + 2 * of, fo);
              gi = fi[1];
              go = fo[1];
            } else {
              ld256(Ti + TF::OPR + 4 * of, fi);
              ld256(To + TF::OPR + 4 * of, fo);
              gi = fma(jn[0][2], fi[3], fma(jn[0][1], fi[2], jn[0][0] * fi[1]));
              go = fma(jn[1][2], fo[3], fma(jn[1][1], fo[2], jn[1][0] * fo[1]));
            }
            dmma(ri[nt][0], ri[nt][1], Y[ks], fi[0]);
            dmma(ri[nt][0], ri[nt][1], X[ks], gi);
            dmma(ro[nt][0], ro[nt][1], -Y[ks], fo[0]);
            dmma(ro[nt][0], ro[nt][1], X[ks], go);
          }
      }
      // face-sum rows: lane entries (species g, basis 4 (2nt + j) + t)
      const bool skip_out = code_skip_out(code);
      const bool fin = code_first_in(code), fout = code_first_out(code);
      if (row) {
        double* fci = ACC + int64_t(el.x) * SN + g * NB;
        double* fco = ACC + int64_t(el.y) * SN + g * NB;
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (T::MERGE && nt == NNT - 1) {  // j = 0: in-side mode, j = 1: out-side
              const int i = 8 * nt + t;
              if (i < NB) {
                if (j == 0)
                  acc_put(fci + i, ri[nt][0], fin);
                else if (!skip_out)
                  acc_put(fco + i, ri[nt][1], fout);
              }
              continue;
            }
            const int i = 4 * (2 * nt + j) + t;
            if (i < NB) {
              acc_put(fci + i, ri[nt][j], fin);
              if (!skip_out) acc_put(fco + i, ro[nt][j], fout);
            }
          }
      }
      __syncwarp();  // xs / cv are rewritten by the next face
    }
  }
}

}  // namespace tdg

// Interior faces on the FP64 tensor cores (3D), face GROUPS as the M rows:
// a CTA runs NFQ faces that share both sides' face-geometry class (table id
// and Jinv n, tables.tc_face_fold_tables) and the lifting side, with the
// (face, species) pairs as the rows of mma.sync.m8n8k4.f64 (DMMA).  With
// six species, four faces give 24 rows = three whole M tiles, one warp
// each; the one-face species-rows kernel k_faces_tcs pads its 6 rows to 8,
// so this kernel issues 3/4 of its DMMAs and B-operand loads.  All rows of
// a tile take the same B operands (the class tables), which is why a group
// shares its classes.  The coupled LLF physics needs every species of a
// face point, and a face's species span two warps, so it runs CTA-wide
// per point tile (shared-memory transpose between two barriers).  Groups
// come from tables.tc_face_groups (same colour segments as the per-face
// kernels, so the face sums keep their order).  Formulas as k_faces_tcs
// (reference operator.py:326-434, flux.py:92-138).
//
//   pass 1 (point tiles qt): u_in, u_out, d_n u_in, d_n u_out of the warp's
//          rows -> transpose xs[face][point][kind][s]; jumps -> modal
//          lifting m = (wB)^T dU; LLF physics per (face, point) -> cvs; the
//          adjoint term X projected onto d_n phi of both sides; the flux
//          without the lifting, Y0, kept per warp in shared memory
//   pass 2 (point tiles qt): rho = m B^T, Y = Y0 - w rho projected onto
//          phi of both sides
#pragma once

#include "common.cuh"
#include "kernels_mma.cuh"
#include "kernels_tcf.cuh"
#include "models.cuh"

namespace tdg {

__host__ __device__ constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }

template <int D, int K, class M>
struct TcgFace {
  using TF = TcFace<D, K, M>;
  static constexpr int NB = TF::NB, S = M::S, SN = S * NB, F = TF::F, NFG = TF::NFG;
  static constexpr int QP = TF::QP, QT = TF::QT, KT = TF::KT, NNT = TF::NNT;
  static constexpr int NCV = TF::NCV;
  static constexpr int NFQ = 8 / gcd_c(S, 8);  // faces per group: S NFQ rows fill
  static constexpr int MT = S * NFQ / 8;       // MT whole M tiles = warps per CTA
  static constexpr int THREADS = 32 * MT;
  // transpose row stride: (face, point) records of 3 XS doubles, odd so the
  // physics threads (consecutive records) read conflict-free
  static constexpr int XS = S | 1;
  static constexpr bool MERGE = TcsFace<D, K, M>::MERGE;
  // CTA scratch (doubles): transposes of two point tiles [2][NFQ][8][3][XS],
  // their physics [2][NFQ][8][NCV], Y0 per warp [MT][QT][2][32]
  static constexpr int OXS = 0, OCV = OXS + 2 * NFQ * 8 * 3 * XS, OY0 = OCV + 2 * NFQ * 8 * NCV,
                       CWS = OY0 + MT * QT * 2 * 32;
  static constexpr size_t smem() { return size_t(CWS) * 8; }
  // up to 16 warps / SM at 128 registers
  // p = 3: 5 CTAs (15 warps) at 128 registers; 6 CTAs at 96 registers
  // measured 23.3 against 22.4 ms (64^3), at p = 2 11.6 against 12.2 ms
  static constexpr int MINB = K >= 3 ? 16 / MT : 6;
  static constexpr bool ok = D == 3 && MT >= 1 && MT <= 4 && !M::kMirror && TF::ok &&
                             smem() * MINB <= 200 * 1024;
};

// LM: lifting sides of the scheme (operator.py:336-357): 0 none (ip, bo),
// 1 the K- side (cdg2, cdg), 2 both (br2)
template <int D, int K, class M, int LM>
__global__ void __launch_bounds__(TcgFace<D, K, M>::THREADS, TcgFace<D, K, M>::MINB)
k_faces_tcg(OpParams p, const double* __restrict__ tabs, const int32_t* __restrict__ groups,
            int64_t g0, int64_t g1, const double* __restrict__ U, double* __restrict__ ACC) {
  using T = TcgFace<D, K, M>;
  using TF = TcFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, NFG = T::NFG, QP = T::QP;
  constexpr int QT = T::QT, KT = T::KT, NNT = T::NNT, TS = TF::TS, TSF = TF::TSF;
  constexpr int NCV = T::NCV, XS = T::XS, NFQ = T::NFQ;
  constexpr bool br2 = LM == 2, lift = LM > 0;
  extern __shared__ __align__(16) double sm[];
  double* xs = sm + T::OXS;   // [2][NFQ][8][3][XS]: u_in, u_out, avg d_n u of a point tile
  double* cvs = sm + T::OCV;  // [2][NFQ][8][NCV]
  const int lane = threadIdx.x & 31, mt = threadIdx.x >> 5;
  double* y0s = sm + T::OY0 + mt * QT * 64;  // this warp's [QT][2][32]
  const int g = lane >> 2, t = lane & 3;
  // this lane's row: tile mt, row g -> (face slot fq, species sp)
  const int fq = (8 * mt + g) / S, sp = (8 * mt + g) % S;
  const double As = p.A[sp];

  for (int64_t grp = g0 + blockIdx.x; grp < g1; grp += gridDim.x) {
    const int32_t* gf = groups + grp * NFQ;
    // the group's shared data from its first face (always present)
    const int f0 = __ldg(gf);
    const int code0 = __ldg(p.ifcode + f0);
    const int2 cl = __ldg(reinterpret_cast<const int2*>(p.ffold) + f0);
    const double* Fi = p.ftf + size_t(cl.x) * TSF;
    const double* Fo = p.ftf + size_t(cl.y) * TSF;
    const int sig = code0 & 1023;
    const double* Ti = tabs + size_t(sig & 31) * TS;
    const double* To = tabs + size_t((sig >> 5) & 31) * TS;
    const bool min_ = code_minus_in(code0);  // one lifting side per group
    const double* Tl = (br2 || min_) ? Ti : To;
    // this row's face (absent past a run's end: zero row, no writes)
    const int fid = __ldg(gf + fq);
    const bool fv = fid >= 0;
    const int fs = fv ? fid : f0;
    const double* gg = p.ifgeo + int64_t(fs) * NFG;
    const double sfac = fv ? __ldg(gg + 2 * D) : 0.0;
    const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + fs);
    // A operands: the row's coefficients, k = 4 kt + t
    double ci[KT], co[KT];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      const bool in = fv && 4 * kt + t < NB;
      ci[kt] = in ? __ldg(U + int64_t(el.x) * SN + sp * NB + 4 * kt + t) : 0.0;
      co[kt] = in ? __ldg(U + int64_t(el.y) * SN + sp * NB + 4 * kt + t) : 0.0;
    }

    // ---- pass 1 ----------------------------------------------------------
    double mi[NNT][2], mo[NNT][2], ri[NNT][2], ro[NNT][2];
#pragma unroll
    for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) mi[nt][j] = mo[nt][j] = ri[nt][j] = ro[nt][j] = 0.0;
    const double wx = 0.5 * p.adj * As * sfac;  // X = w_q wx du
    // flux without the lifting (Y0, for pass 2) and the adjoint term X of
    // tile qt, from its jumps / averages and the tile's physics in cvs[b]
    auto flux_x = [&](int qt, const double* du, const double* gv, int b) {
      double X[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 8 * qt + 2 * t + j;
        double qv = 0.0;
        if (p.scheme == IP) qv = p.eta / __ldg(gg + 2 * D + 1) * As * du[j];
        if constexpr (M::kConv) {
          if (q < F) {
            const double* c = cvs + (b * NFQ * 8 + fq * 8 + 2 * t + j) * NCV;
            double cnv = 0.5 * c[0] * du[j];
#pragma unroll
            for (int k = 0; k < M::NFX; ++k)
              if (sp == k) cnv = fma(0.5, c[1 + k], cnv);
            qv += cnv;
          }
        }
        const double w = q < F ? __ldg(p.fw + q) : 0.0;
        y0s[(qt * 2 + j) * 32 + lane] = w * sfac * (As * gv[j] - qv);
        X[j] = w * wx * du[j];
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt) {
          if (T::MERGE && nt == NNT - 1) {
            // merged tail tile (k_faces_tcs): the even columns carry the
            // in-side modes, the odd ones the out-side ones (normal-layout
            // lane - 4)
            const bool oc = (g & 1) != 0;
            const int of = ((qt * 2 + ks) * NNT + nt) * 32 + (oc ? lane - 4 : lane);
            dmma(ri[nt][0], ri[nt][1], X[ks], __ldg((oc ? Fo : Fi) + TF::OPGF + of));
            continue;
          }
          const int of = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
          dmma(ri[nt][0], ri[nt][1], X[ks], __ldg(Fi + TF::OPGF + of));
          dmma(ro[nt][0], ro[nt][1], X[ks], __ldg(Fo + TF::OPGF + of));
        }
    };
    // software pipeline over the point tiles, one barrier per tile:
    // iteration qt writes tile qt's traces to xs[qt&1], and after the
    // barrier warp qt%MT runs tile qt's physics into cvs[qt&1] while every
    // warp forms tile qt-1's flux from cvs[(qt-1)&1] (complete: its writer
    // passed this barrier).  The buffers a tile writes were last read before
    // the previous barrier.
    double dup[2] = {0.0, 0.0}, gvp[2] = {0.0, 0.0};
#pragma unroll 1
    for (int qt = 0; qt < QT; ++qt) {
      double ui[2] = {0.0, 0.0}, uo[2] = {0.0, 0.0}, di[2] = {0.0, 0.0}, dq[2] = {0.0, 0.0};
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        double fi[2], fo[2];  // (B, G_n) fragments of both sides
        const int ob = 2 * ((kt * QT + qt) * 32 + lane);
        ld128(Fi + TF::OTRF + ob, fi);
        ld128(Fo + TF::OTRF + ob, fo);
        dmma(ui[0], ui[1], ci[kt], fi[0]);
        dmma(uo[0], uo[1], co[kt], fo[0]);
        dmma(di[0], di[1], ci[kt], fi[1]);
        dmma(dq[0], dq[1], co[kt], fo[1]);
      }
      double du[2], gv[2];
      const int b = qt & 1;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        du[j] = ui[j] - uo[j];
        gv[j] = 0.5 * (di[j] + dq[j]);
        if constexpr (M::kConv) {
          double* x = xs + (b * NFQ * 8 + fq * 8 + 2 * t + j) * 3 * XS + sp;
          x[0] = ui[j];
          x[XS] = uo[j];
          x[2 * XS] = gv[j];
        }
      }
      if constexpr (lift) {
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int nt = 0; nt < NNT; ++nt) {
            const int ow = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
            dmma(mi[nt][0], mi[nt][1], du[ks], __ldg(Tl + TF::OWB + ow));
            if constexpr (br2) dmma(mo[nt][0], mo[nt][1], du[ks], __ldg(To + TF::OWB + ow));
          }
      }
      if constexpr (M::kConv) {
        __syncthreads();
        if (mt == qt % T::MT) {
          for (int i = lane; i < NFQ * 8; i += 32) {
            if (8 * qt + (i & 7) < F) {
              const double* xq = xs + (b * NFQ * 8 + i) * 3 * XS;
              auto fetch = [xq](int kind, int s2) { return xq[kind * XS + s2]; };
              M::face_point(p.P, fetch, cvs + (b * NFQ * 8 + i) * NCV);
            }
          }
        }
      }
      if (qt > 0) flux_x(qt - 1, dup, gvp, b ^ 1);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        dup[j] = du[j];
        gvp[j] = gv[j];
      }
    }
    if constexpr (M::kConv) __syncthreads();
    flux_x(QT - 1, dup, gvp, (QT - 1) & 1);
    // lifting weights (operator.py:336-357): -fac A rho, rho = -1/2 sfac/detJ Pw dU
    if constexpr (lift) {
      const double wside = br2 ? 0.5 : 1.0;
      const double fac0 = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * wside * 0.5 * sfac * As;
      const double ki = fac0 * __ldg(gg + 2 * D + ((br2 || min_) ? 2 : 3));
      const double ko = br2 ? fac0 * __ldg(gg + 2 * D + 3) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NNT; ++nt)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mi[nt][j] *= ki;
          mo[nt][j] *= ko;
        }
    }
    __syncwarp();  // y0s
    // ---- pass 2: rho, flux projection ------------------------------------
#pragma unroll 1
    for (int qt = 0; qt < QT; ++qt) {
      double rho[2] = {0.0, 0.0};
      if constexpr (lift) {
        // two independent accumulator chains (even / odd k-steps), as k_faces_tcs
        double rb[2] = {0.0, 0.0};
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int ob = (kt * QT + qt) * 32 + lane;
          double* r = (kt & 1) ? rb : rho;
          // m as A operand: k-step kt holds basis 4 kt + t = pi(8 (kt/2) + 2t + kt%2)
          dmma(r[0], r[1], mi[kt / 2][kt % 2], __ldg(Tl + TF::OBT + ob));
          if constexpr (br2) dmma(r[0], r[1], mo[kt / 2][kt % 2], __ldg(To + TF::OBT + ob));
        }
        rho[0] += rb[0];
        rho[1] += rb[1];
      }
      double Y[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = 8 * qt + 2 * t + j;
        const double y0 = y0s[(qt * 2 + j) * 32 + lane];
        Y[j] = lift && q < F ? fma(-__ldg(p.fw + q) * sfac, rho[j], y0) : y0;
      }
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int nt = 0; nt < NNT; ++nt) {
          if (T::MERGE && nt == NNT - 1) {
            const bool oc = (g & 1) != 0;
            const int of = ((qt * 2 + ks) * NNT + nt) * 32 + (oc ? lane - 4 : lane);
            const double bx = __ldg((oc ? Fo : Fi) + TF::OPBF + of);
            dmma(ri[nt][0], ri[nt][1], Y[ks], oc ? -bx : bx);
            continue;
          }
          const int of = ((qt * 2 + ks) * NNT + nt) * 32 + lane;
          dmma(ri[nt][0], ri[nt][1], Y[ks], __ldg(Fi + TF::OPBF + of));
          dmma(ro[nt][0], ro[nt][1], Y[ks], -__ldg(Fo + TF::OPBF + of));
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
  }
}

}  // namespace tdg

// Face kernel on the FP64 tensor cores (mma.sync.m8n8k4.f64, DMMA).
//
// ncu on the SIMT face kernel (profiles/r01_summary.txt) shows it issue-
// bound: ~1300 warp instructions per 5 faces, a quarter of them DFMA.
// The face-local contractions are genuine small dense GEMMs once the
// faces of one trace-table signature are batched: a warp owns NFW faces x
// S species = NC columns and evaluates
//
//   traces      u[q][n]  = sum_k  B[q][k]          c[k][n]
//               dnu[q][n]= sum_ka G[q][k][a] jn_a(n) c[k][n]   (K = nb*d)
//   lifting     m[i][n]  = sum_q  w_q B[q][i] dU[q][n]           (modal form
//               rho[q][n]= sum_i  B[q][i] kappa(n) m[i][n]        of Pw dU)
//   projection  R[i][n] += sum_q  B[q][i] Y[q][n]
//                        + sum_qa G[q][i][a] jn_a(n) X[q][n]
//
// with one DMMA (256 FMA) per warp instruction instead of 32.  B200's
// DMMA rate equals its DFMA rate (37.2 vs 37.0 TFLOP/s measured by
// tools/probe_fp64.py), so the gain is issue bandwidth.  Operand tables
// are zero-padded per signature on the host (tables.mma_face_tables) and
// read straight from L1/L2.  Points are processed in chunks of 8 (one
// m-tile) in two passes: pass 1 forms the jumps and the modal lifting
// coefficients, pass 2 recomputes the chunk's traces, runs the coupled
// point physics once per (face, point) through a per-warp shared-memory
// transpose, and accumulates the projection.  Faces are sorted by
// signature; a warp whose faces straddle two signatures loops over them
// with column masks.
//
// Fragment layouts (PTX m8n8k4 .f64): g = lane>>2, t = lane&3;
//   A[g][t] (row major 8x4), B[t][g] (col major 4x8), C[g][2t+j].
#pragma once

#include "common.cuh"
#include "models.cuh"

namespace tdg {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__host__ __device__ constexpr int ceil_to(int x, int m) { return (x + m - 1) / m * m; }

__device__ __forceinline__ int sym_index_d(int D, int a, int b) {
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  return lo * D - lo * (lo - 1) / 2 + (hi - lo);
}

template <int D, int K, class M>
struct MmaFace {
  using Dm = Dims<D, K>;
  static constexpr int NB = Dm::NB, S = M::S, SN = S * NB, F = Dm::NQF, NFG = Dm::NFG;
  static constexpr int FP = ceil_to(F, 8), NBK = ceil_to(NB, 4), NBM = ceil_to(NB, 8);
  static constexpr int NFW = S == 6 ? 4 : 8;          // faces per warp
  static constexpr int NC = NFW * S;                  // columns (face, species)
  static constexpr int NT = (NC + 7) / 8;             // n-tiles
  static constexpr int NCP = NT * 8;                  // padded columns
  static constexpr int MT = FP / 8, KT = NBK / 4, IT = NBM / 8;
  static constexpr int NCV = 1 + M::NFX;
  // one signature's table block (doubles), see tables.mma_face_tables
  static constexpr int OB = 0, OG = OB + FP * NBK, OBW = OG + D * FP * NBK, OBT = OBW + NBM * FP,
                       OGT = OBT + NBM * FP, TSTRIDE = OGT + D * NBM * FP;
  // per-warp shared memory (doubles)
  static constexpr int SC = 2 * NBK * NCP;   // coefficients [side][k][n]
  static constexpr int SDU = 8 * NCP;        // jump chunk [ql][n]
  static constexpr int SMK = 2 * NBM * NCP;  // scaled modal lifting [side][i][n]
  static constexpr int SST = 3 * 8 * NCP;    // stage [u_in|Y, u_out, avg d_n u][ql][n]
  static constexpr int SX = D * 8 * NCP;     // X jn_a of the side being projected [a][ql][n]
  static constexpr int SCV = NFW * 8 * NCV;  // coupled physics [f][ql][cv]
  static constexpr int SOUT = 2 * NBM * NCP; // projected rows [side][i][n] (aliases SDU..)
  static constexpr int SFD = NFW * NFG;      // face doubles
  static constexpr int SFI = NFW * 4;        // face ints (code, ein, eout, lf) as doubles
  static constexpr int SALIAS = (SDU + SMK + SST + SX) > SOUT ? 0 : SOUT - (SDU + SMK + SST + SX);
  static constexpr int PW = SC + SDU + SMK + SST + SX + SALIAS + SCV + SFD + SFI;
  static constexpr int WARPS = 4;
  static constexpr size_t smem() { return size_t(WARPS) * PW * 8; }
  static constexpr bool ok = S >= 1 && S <= 8 && smem() <= 200 * 1024;
  static constexpr int MINB = smem() <= 72 * 1024 ? 3 : 2;
};

template <int D, int K, class M>
__global__ void __launch_bounds__(128, MmaFace<D, K, M>::MINB)
k_faces_mma(OpParams p, const double* __restrict__ tabs, const double* __restrict__ U,
            double* __restrict__ ACC) {
  using T = MmaFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = T::SN, F = T::F, NFG = T::NFG;
  constexpr int NFW = T::NFW, NC = T::NC, NT = T::NT, NCP = T::NCP;
  constexpr int MT = T::MT, KT = T::KT, IT = T::IT, NBK = T::NBK;
  constexpr int NBM = T::NBM, FP = T::FP, NCV = T::NCV, TS = T::TSTRIDE;
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double* W = sm + warp * T::PW;
  double* cS = W;                    // [2][NBK][NCP]
  double* dUS = cS + T::SC;          // [8][NCP]
  double* mKS = dUS + T::SDU;        // [2][NBM][NCP]
  double* stS = mKS + T::SMK;        // [3][8][NCP]
  double* xS = stS + T::SST;         // [D][8][NCP]
  double* cvS = xS + T::SX + T::SALIAS;  // [NFW][8][NCV]
  double* outS = dUS;                // [2][NBM][NCP], aliases dUS..xS (dead by then)
  double* fD = cvS + T::SCV;         // [NFW][NFG]
  int* fI = reinterpret_cast<int*>(fD + T::SFD);  // [NFW][8]: code ein eout - - valid

  const int64_t gw = int64_t(blockIdx.x) * T::WARPS + warp;
  const int64_t wi = (p.nif + NFW - 1) / NFW;
  const bool wall = gw >= wi;
  const int64_t f0 = wall ? p.nif + (gw - wi) * NFW : gw * NFW;
  const int64_t fend = wall ? p.nif + p.nbf : p.nif;
  if (f0 >= fend) return;  // warp-uniform

  // ---- face records -> shared memory ---------------------------------
  if (lane < NFW) {
    const int64_t f = f0 + lane;
    int* r = fI + lane * 8;
    double* d = fD + lane * NFG;
    r[5] = f < fend;
    r[0] = 0;
    r[1] = 0;
    r[2] = -1;
    r[3] = 0;
    r[4] = 0;
#pragma unroll
    for (int k = 0; k < NFG; ++k) d[k] = 0.0;
    if (f < fend) {
      if (!wall) {
        r[0] = __ldg(p.ifcode + f);
        r[1] = __ldg(p.ifel + 2 * f);
        r[2] = __ldg(p.ifel + 2 * f + 1);
#pragma unroll
        for (int k = 0; k < NFG; ++k) d[k] = __ldg(p.ifgeo + f * NFG + k);
      } else {
        const int64_t b = f - p.nif;
        r[0] = __ldg(p.bfcode + b);
        r[1] = __ldg(p.bfel + b);
        d[2 * D] = __ldg(p.bfgeo + b);
      }
    }
  }
  __syncwarp();
  // coefficient columns [side][k][n], zero-padded modes / columns / sides
  for (int idx = lane; idx < 2 * NFW * SN; idx += 32) {
    const int side = idx / (NFW * SN), r = idx - side * NFW * SN;
    const int f = r / SN, sk = r - f * SN, s = sk / NB, k = sk - s * NB;
    const int* fr = fI + f * 8;
    const bool ok = fr[5] && (side == 0 || (!wall && !code_mirror(fr[0])));
    const int e = side ? fr[2] : fr[1];
    cS[(side * NBK + k) * NCP + f * S + s] = ok ? __ldg(U + int64_t(e) * SN + sk) : 0.0;
  }
  if constexpr (NBK > NB) {
    for (int idx = lane; idx < 2 * (NBK - NB) * NCP; idx += 32) {
      const int side = idx / ((NBK - NB) * NCP), r = idx - side * (NBK - NB) * NCP;
      cS[(side * NBK + NB) * NCP + r] = 0.0;
    }
  }
  if constexpr (NCP > NC) {
    for (int idx = lane; idx < 2 * NB * (NCP - NC); idx += 32) {
      const int side = idx / (NB * (NCP - NC)), r = idx - side * NB * (NCP - NC);
      const int k = r / (NCP - NC), n = NC + r - k * (NCP - NC);
      cS[(side * NBK + k) * NCP + n] = 0.0;
    }
  }
  __syncwarp();

  // per-lane column bookkeeping for the C fragments (cols 2tq+j of each n-tile)
  // and the B fragments (col g of each n-tile)
  auto col_face = [](int n) { return n / S; };
  auto col_sp = [](int n) { return n - (n / S) * S; };

  // jn_a(n) for a B-fragment column, side sd
  auto jn_of = [&](int sd, int a, int n) -> double {
    return n < NC ? fD[col_face(n) * NFG + sd * D + a] : 0.0;
  };

  // accumulators of the projected rows, kept across signature subgroups
  double rI[IT][NT][2], rO[IT][NT][2];
#pragma unroll
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) rI[it][nt][0] = rI[it][nt][1] = rO[it][nt][0] = rO[it][nt][1] = 0.0;

  // ---- loop over the distinct signatures present in this warp ----------
  unsigned todo = 0;
  for (int f = 0; f < NFW; ++f)
    if (fI[f * 8 + 5]) todo |= 1u << f;
  while (todo) {
    const int lead = __ffs(todo) - 1;
    const int sig = fI[lead * 8] & 1023;
    unsigned members = 0;
    for (int f = 0; f < NFW; ++f)
      if ((todo >> f & 1) && (fI[f * 8] & 1023) == sig) members |= 1u << f;
    todo &= ~members;
    const int tin = sig & 31, tout = (sig >> 5) & 31;
    const double* TBi = tabs + size_t(tin) * TS;
    const double* TBo = tabs + size_t(tout) * TS;
    auto member_col = [&](int n) { return n < NC && ((members >> col_face(n)) & 1); };
    // B-fragment columns of this lane (col g of every n-tile)
    bool bmask[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bmask[nt] = member_col(8 * nt + g);

    // which lifting sides the member faces use (operator.py:336-357)
    bool any_in = false, any_out = false, any_two = false;
    for (int f = 0; f < NFW; ++f) {
      if (!((members >> f) & 1)) continue;
      const int c = fI[f * 8];
      const bool mir = code_mirror(c);
      if (!wall && !mir) any_two = true;
      if (wall || p.scheme == IP || p.scheme == BO) continue;
      const bool br2 = p.scheme == BR2;
      if (mir || br2 || code_minus_in(c)) any_in = true;
      if (!mir && (br2 || !code_minus_in(c))) any_out = true;
    }

    // lifting weight of side sd for column n: fac A_s w_side 1/2 sfac / detJ_side
    auto kappa = [&](int sd, int n) -> double {
      if (!member_col(n)) return 0.0;
      const int f = col_face(n), c = fI[f * 8];
      const bool mir = code_mirror(c), br2 = p.scheme == BR2;
      const bool use = sd == 0 ? (mir || br2 || code_minus_in(c)) : (!mir && (br2 || !code_minus_in(c)));
      if (!use) return 0.0;
      const double* d = fD + f * NFG;
      const double wside = (br2 && !mir) ? 0.5 : 1.0;
      const double fac = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e;
      return fac * p.A[col_sp(n)] * wside * 0.5 * d[2 * D] * (sd == 0 ? d[2 * D + 2] : d[2 * D + 3]);
    };

    // traces of one point chunk: u (and d_n u = sum_a jn_a (G_a c)) for
    // both sides; B operands are plain shared-memory loads
    auto traces = [&](int c, double (&ui)[NT][2], double (&uo)[NT][2], double (&gi)[NT][2],
                      double (&go)[NT][2], bool grads, bool out_side) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) ui[nt][0] = ui[nt][1] = uo[nt][0] = uo[nt][1] =
          gi[nt][0] = gi[nt][1] = go[nt][0] = go[nt][1] = 0.0;
      const int row = 8 * c + g;
#pragma unroll
      for (int kt = 0; kt < KT; ++kt) {
        const int k = 4 * kt + tq;
        const double ai = __ldg(TBi + T::OB + row * NBK + k);
        const double ao = out_side ? __ldg(TBo + T::OB + row * NBK + k) : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int n = 8 * nt + g;
          dmma(ui[nt][0], ui[nt][1], ai, bmask[nt] ? cS[k * NCP + n] : 0.0);
          if (out_side) dmma(uo[nt][0], uo[nt][1], ao, bmask[nt] ? cS[(NBK + k) * NCP + n] : 0.0);
        }
      }
      if (!grads) return;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        double ti[NT][2], to[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) ti[nt][0] = ti[nt][1] = to[nt][0] = to[nt][1] = 0.0;
#pragma unroll
        for (int kt = 0; kt < KT; ++kt) {
          const int k = 4 * kt + tq;
          const double ai = __ldg(TBi + T::OG + (a * FP + row) * NBK + k);
          const double ao = out_side ? __ldg(TBo + T::OG + (a * FP + row) * NBK + k) : 0.0;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int n = 8 * nt + g;
            dmma(ti[nt][0], ti[nt][1], ai, bmask[nt] ? cS[k * NCP + n] : 0.0);
            if (out_side) dmma(to[nt][0], to[nt][1], ao, bmask[nt] ? cS[(NBK + k) * NCP + n] : 0.0);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n = 8 * nt + 2 * tq + j;
            if (n < NC) {
              const double* d = fD + col_face(n) * NFG;
              gi[nt][j] = fma(d[a], ti[nt][j], gi[nt][j]);
              go[nt][j] = fma(d[D + a], to[nt][j], go[nt][j]);
            }
          }
      }
    };

    if (!wall) {
      // ---- pass 1: jumps -> modal lifting coefficients ------------------
      double mI[IT][NT][2], mO[IT][NT][2];
#pragma unroll
      for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mI[it][nt][0] = mI[it][nt][1] = mO[it][nt][0] = mO[it][nt][1] = 0.0;
      if (any_in || any_out) {
#pragma unroll 1
      for (int c = 0; c < MT; ++c) {
          double ui[NT][2], uo[NT][2], gi[NT][2], go[NT][2];
          traces(c, ui, uo, gi, go, false, any_two);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int n = 8 * nt + 2 * tq + j;
              double du = 0.0;
              if (member_col(n)) {
                const int f = col_face(n);
                if (code_mirror(fI[f * 8])) du = 2.0 * (ui[nt][j] - M::mirror_value(p.P, col_sp(n)));
                else du = ui[nt][j] - uo[nt][j];
              }
              dUS[g * NCP + n] = du;
            }
          __syncwarp();
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int ql = 4 * ks + tq;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
              const int i = 8 * it + g;
              const double ai = any_in ? __ldg(TBi + T::OBW + i * FP + 8 * c + ql) : 0.0;
              const double ao = any_out ? __ldg(TBo + T::OBW + i * FP + 8 * c + ql) : 0.0;
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const double b = dUS[ql * NCP + 8 * nt + g];
                if (any_in) dmma(mI[it][nt][0], mI[it][nt][1], ai, b);
                if (any_out) dmma(mO[it][nt][0], mO[it][nt][1], ao, b);
              }
            }
          }
          __syncwarp();
        }
        // scaled modal coefficients -> shared (B operands of the rho GEMM)
#pragma unroll
        for (int it = 0; it < IT; ++it)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int i = 8 * it + g, n = 8 * nt + 2 * tq + j;
              mKS[(0 * NBM + i) * NCP + n] = i < NB ? mI[it][nt][j] * kappa(0, n) : 0.0;
              mKS[(1 * NBM + i) * NCP + n] = i < NB ? mO[it][nt][j] * kappa(1, n) : 0.0;
            }
        __syncwarp();
      }

      // ---- pass 2: traces, physics, projection ---------------------------
#pragma unroll 1
      for (int c = 0; c < MT; ++c) {
        double ui[NT][2], uo[NT][2], gi[NT][2], go[NT][2];
        traces(c, ui, uo, gi, go, true, any_two);
        double rho[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) rho[nt][0] = rho[nt][1] = 0.0;
        if (any_in || any_out) {
          const int row = 8 * c + g;
#pragma unroll
          for (int kt = 0; kt < KT; ++kt) {
            const int k = 4 * kt + tq;
            const double ai = any_in ? __ldg(TBi + T::OB + row * NBK + k) : 0.0;
            const double ao = any_out ? __ldg(TBo + T::OB + row * NBK + k) : 0.0;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              const int n = 8 * nt + g;
              if (any_in) dmma(rho[nt][0], rho[nt][1], ai, k < NB ? mKS[(0 * NBM + k) * NCP + n] : 0.0);
              if (any_out) dmma(rho[nt][0], rho[nt][1], ao, k < NB ? mKS[(1 * NBM + k) * NCP + n] : 0.0);
            }
          }
        }
        // point values -> stage for the coupled physics
        double dU[NT][2], gav[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n = 8 * nt + 2 * tq + j;
            double u = ui[nt][j], v = uo[nt][j], x = gi[nt][j], y = go[nt][j];
            if (member_col(n) && code_mirror(fI[col_face(n) * 8])) {
              v = 2.0 * M::mirror_value(p.P, col_sp(n)) - u;
              y = x;
            }
            dU[nt][j] = u - v;
            gav[nt][j] = 0.5 * (x + y);
            stS[(0 * 8 + g) * NCP + n] = u;
            stS[(1 * 8 + g) * NCP + n] = v;
            stS[(2 * 8 + g) * NCP + n] = gav[nt][j];
          }
        __syncwarp();
        if constexpr (M::kConv) {
          for (int pr = lane; pr < NFW * 8; pr += 32) {
            const int f = pr >> 3, ql = pr & 7;
            if (((members >> f) & 1) && 8 * c + ql < F) {
              const double* xq = stS + ql * NCP + f * S;
              auto fetch = [xq](int kind, int sp) { return xq[kind * 8 * NCP + sp]; };
              M::face_point(p.P, fetch, cvS + (f * 8 + ql) * NCV);
            }
          }
          __syncwarp();
        }
        // Y, X at the chunk's points (operator.py:413-418)
        double Xr[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n = 8 * nt + 2 * tq + j, q = 8 * c + g;
            double Y = 0.0, X = 0.0;
            if (member_col(n) && q < F) {
              const int f = col_face(n), s = col_sp(n);
              const double* d = fD + f * NFG;
              const double As = p.A[s], sfac = d[2 * D];
              double qv = rho[nt][j];
              if (p.scheme == IP) qv = p.eta / d[2 * D + 1] * As * dU[nt][j];
              if constexpr (M::kConv) {
                const double* cv = cvS + (f * 8 + g) * NCV;
                double cnv = 0.5 * cv[0] * dU[nt][j];
#pragma unroll
                for (int k2 = 0; k2 < M::NFX; ++k2)
                  if (s == k2) cnv = fma(0.5, cv[1 + k2], cnv);
                qv += cnv;
              }
              const double wq = __ldg(p.fw + q) * sfac;
              Y = wq * (As * gav[nt][j] - qv);
              X = wq * 0.5 * p.adj * As * dU[nt][j];
            }
            stS[g * NCP + n] = Y;
            Xr[nt][j] = X;
          }
        // projection onto both sides' test functions
#pragma unroll
        for (int sd = 0; sd < 2; ++sd) {
          if (sd == 1 && !any_two) break;
          // X jn_a of this side -> shared (B operands)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int n = 8 * nt + 2 * tq + j;
              const double* d = fD + (n < NC ? col_face(n) : 0) * NFG + sd * D;
#pragma unroll
              for (int a2 = 0; a2 < D; ++a2) xS[(a2 * 8 + g) * NCP + n] = n < NC ? Xr[nt][j] * d[a2] : 0.0;
            }
          __syncwarp();
          const double* TBs = sd ? TBo : TBi;
          const double sgn = sd ? -1.0 : 1.0;
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const int ql = 4 * ks + tq;
#pragma unroll
            for (int it = 0; it < IT; ++it) {
              const double ay = sgn * __ldg(TBs + T::OBT + (8 * it + g) * FP + 8 * c + ql);
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                const double b = stS[ql * NCP + 8 * nt + g];
                if (sd) dmma(rO[it][nt][0], rO[it][nt][1], ay, b);
                else dmma(rI[it][nt][0], rI[it][nt][1], ay, b);
              }
#pragma unroll
              for (int a2 = 0; a2 < D; ++a2) {
                const double ax = __ldg(TBs + T::OGT + (a2 * NBM + 8 * it + g) * FP + 8 * c + ql);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                  const double b = xS[(a2 * 8 + ql) * NCP + 8 * nt + g];
                  if (sd) dmma(rO[it][nt][0], rO[it][nt][1], ax, b);
                  else dmma(rI[it][nt][0], rI[it][nt][1], ax, b);
                }
              }
            }
          }
          __syncwarp();
        }
      }
    } else {
      // ---- prescribed-flux wall faces: Y = -w sfac q_s(c1) on the inside -
#pragma unroll 1
      for (int c = 0; c < MT; ++c) {
        double ui[NT][2], uo[NT][2], gi[NT][2], go[NT][2];
        traces(c, ui, uo, gi, go, false, false);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) stS[g * NCP + 8 * nt + 2 * tq + j] = ui[nt][j];
        __syncwarp();
        double Yv[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int n = 8 * nt + 2 * tq + j, q = 8 * c + g;
            double Y = 0.0;
            if (member_col(n) && q < F) {
              const int f = col_face(n);
              const double c1 = stS[g * NCP + f * S + M::WALL_SP];
              Y = -__ldg(p.fw + q) * fD[f * NFG + 2 * D] *
                  M::wall_lane(p.P, code_tag(fI[f * 8]), col_sp(n), c1);
            }
            Yv[nt][j] = Y;
          }
        __syncwarp();
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) stS[(0 * 8 + g) * NCP + 8 * nt + 2 * tq + j] = Yv[nt][j];
        __syncwarp();
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int ql = 4 * ks + tq;
#pragma unroll
          for (int it = 0; it < IT; ++it) {
            const double a = __ldg(TBi + T::OBT + (8 * it + g) * FP + 8 * c + ql);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              dmma(rI[it][nt][0], rI[it][nt][1], a, stS[ql * NCP + 8 * nt + g]);
          }
        }
        __syncwarp();
      }
    }
  }

  // ---- projected rows -> face sums, coalesced per face side ------------
#pragma unroll
  for (int it = 0; it < IT; ++it)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int i = 8 * it + g, n = 8 * nt + 2 * tq + j;
        outS[(0 * NBM + i) * NCP + n] = rI[it][nt][j];
        outS[(1 * NBM + i) * NCP + n] = rO[it][nt][j];
      }
  __syncwarp();
  for (int idx = lane; idx < 2 * NFW * SN; idx += 32) {
    const int side = idx / (NFW * SN), r = idx - side * NFW * SN;
    const int f = r / SN, si = r - f * SN, s = si / NB, i = si - s * NB;
    const int* fr = fI + f * 8;
    if (!fr[5]) continue;
    const int code = fr[0];
    if (side && (wall || code_mirror(code) || code_skip_out(code))) continue;
    const int e = side ? fr[2] : fr[1];
    acc_put(ACC + int64_t(e) * SN + si, outS[(side * NBM + i) * NCP + f * S + s],
            side ? code_first_out(code) : code_first_in(code));
  }
}

}  // namespace tdg

// Shared definitions of the sm_100a DG operator kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tdg {

__host__ __device__ constexpr int binom(int n, int k) {
  return k == 0 ? 1 : binom(n - 1, k - 1) * n / k;
}

// number of Grundmann-Moeller nodes of degree 2s+1 on the dim-simplex
// (quadrature.py:84-107): sum_i C(s - i + dim, dim)
__host__ __device__ constexpr int gm_count(int dim, int s) {
  return s < 0 ? 0 : binom(s + dim, dim) + gm_count(dim, s - 1);
}

// compile-time sizes for (dimension, polynomial order) with the
// reference's default quadrature degrees 3k+1 / 3k+2 (operator.py:106-109)
template <int D, int K>
struct Dims {
  static constexpr int NB = binom(K + D, D);
  static constexpr int NQV = gm_count(D, (3 * K + 1) / 2);
  static constexpr int NQF = D == 2 ? (3 * K + 2) / 2 + 1 : gm_count(2, (3 * K + 2) / 2);
  static constexpr int NPERM = D == 2 ? 2 : 6;
  static constexpr int NT = (D + 1) * NPERM;
  static constexpr int NSYM = D * (D + 1) / 2;
  static constexpr int NEG = 1 + NSYM;          // per-element geometry record
  static constexpr int NFG = 2 * D + 4;         // per-face geometry record
};

enum Scheme { CDG2 = 0, CDG = 1, BR2 = 2, IP = 3, BO = 4 };

constexpr int kMaxS = 8;

// Everything the kernels need, passed by value (kernel parameter space).
struct OpParams {
  int64_t ne;        // owned elements
  int64_t nif, nbf;  // interior(+mirror) faces, flux-boundary faces
  int nqv, nqf;
  int scheme;
  double chi_e, adj, eta;
  double A[kMaxS];             // diffusivity
  double L[kMaxS * kMaxS];     // linear source matrix
  double P[32];                // model parameters
  const double* __restrict__ phi;
  const double* __restrict__ grad;
  const double* __restrict__ wv;
  const double* __restrict__ ks;
  const double* __restrict__ fB;
  const double* __restrict__ fG;
  const double* __restrict__ fPw;
  const double* __restrict__ fw;
  const double* __restrict__ egeo;
  const int32_t* __restrict__ ifel;
  const int32_t* __restrict__ ifcode;
  const double* __restrict__ ifgeo;
  const int32_t* __restrict__ bfel;
  const int32_t* __restrict__ bfcode;
  const double* __restrict__ bfgeo;
  const double* __restrict__ fmma;  // tensor-core face tables (may be null)
  const double* __restrict__ vtc;   // transposed tensor-core volume tables (may be null)
  const double* __restrict__ ftc;   // transposed tensor-core face tables (may be null)
  const int32_t* __restrict__ fblk; // interior-face blocks [n][2] (first, count)
  const double* __restrict__ ftf;   // face-geometry-class folded tables (may be null)
  const int32_t* __restrict__ ffold;  // [nif][2] class of the inside / outside side
  const int32_t* __restrict__ fgrp;   // face groups [n][NFQ] (may be null)
  const double* __restrict__ fmod;    // modal face tables (may be null)
  const double* __restrict__ ifbv;    // [nif][nqf][S] Dirichlet values at mirror-face points (may be null)
  const double* __restrict__ bfqv;    // [nbf][nqf][S] prescribed wall fluxes at the points (may be null)
  const double* __restrict__ vctab;   // volume element-class stiffness tables (may be null)
  const int32_t* __restrict__ vperm;  // [ntask][8] class-sorted element ids
  const int32_t* __restrict__ vtcls;  // [ntask] class of each task
};

// code-word layout, mirrors include/taxisdg_b200.h
__device__ __forceinline__ int code_tin(int c) { return c & 31; }
__device__ __forceinline__ int code_tout(int c) { return (c >> 5) & 31; }
__device__ __forceinline__ bool code_minus_in(int c) { return (c >> 10) & 1; }
__device__ __forceinline__ int code_tag(int c) { return (c >> 11) & 7; }
__device__ __forceinline__ bool code_mirror(int c) { return (c >> 14) & 1; }
__device__ __forceinline__ bool code_skip_out(int c) { return (c >> 15) & 1; }
// the side runs first for its element in the face-segment order: it
// writes the element's face-sum row, later sides add to it
__device__ __forceinline__ bool code_first_in(int c) { return (c >> 16) & 1; }
__device__ __forceinline__ bool code_first_out(int c) { return (c >> 17) & 1; }

// Face-sum accumulation.  The faces are coloured so that one launch (one
// face segment) touches every element at most once; segments run in a
// fixed order, so each entry is  ((f_1 + f_2) + f_3) + ...  in that order
// (deterministic, no atomics).  `first` marks the element's first face.
__device__ __forceinline__ void acc_put(double* p, double v, bool first) {
  *p = first ? v : *p + v;
}

// BoundaryTag (mesh.py:46-52)
enum Tag { GAMMA1 = 1, GAMMA1_IN = 2, GAMMA2 = 3, NO_FLOW = 4 };

// read-only global load that does not allocate in L1 (streamed state rows:
// L1 stays for the operand tables)
__device__ __forceinline__ double ld_na(const double* p) {
  double d;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(d) : "l"(p));
  return d;
}

// 32-byte read-only global load (sm_100 LDG.E.ENL2.256); p 32-byte aligned
__device__ __forceinline__ void ld256(const double* p, double* d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(d[0]), "=d"(d[1]), "=d"(d[2]), "=d"(d[3]) : "l"(p));
}

__device__ __forceinline__ void ld128(const double* p, double* d) {
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(d[0]), "=d"(d[1]) : "l"(p));
}

// Reciprocal to ~1 ulp: MUFU seed + two Newton steps (the operator only
// needs agreement with the reference to ~1e-15 relative, not IEEE rounding).
__device__ __forceinline__ double rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

}  // namespace tdg

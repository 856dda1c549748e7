// Pointwise model physics on the device.
//
// Formulas of reference pkg/src/taxisdg/model.py, restated in the form
// the fused kernels consume:
//   * volume: the taxis flux F(u, grad u) is linear in the physical
//     gradients, so its pull-back F Jinv^T = sum_t chi_st(u) (g_ref,t M)
//     with M = Jinv Jinv^T; the kernel hands the model g_ref M per
//     gradient species and receives F Jinv^T per flux species;
//   * the linear part of the source is applied modally (host matrix L);
//     the bilinear remainder is returned per point;
//   * faces only ever need normal components of the averaged physical
//     gradient (LLF central flux F.n and the wave speed |v.n|), so the
//     model receives avg(d_n u) per species.
#pragma once

#include "common.cuh"

namespace tdg {

// PlaqueParams field order (model.py:86-112, packed by model.py pack())
enum PlaqueParam {
  MU1 = 0, MU2, MU3, NU1, NU2, NU3, D1, D2, ALPHA1, ALPHA2, KOX, GAMMA, F1,
  C11A, C11B, C13A, C13B, C21A, C21B, C2NA, C2NB, BETA1, BETA2, SIGMA,
  C1S, C1SS, EPSH
};

// smooth_heaviside (model.py:58-62)
__device__ __forceinline__ double heaviside(double s, double eps) {
  if (eps == 0.0) return s > 0.0 ? 1.0 : 0.0;
  double z = fmin(fmax(-s / eps, -60.0), 60.0);
  return 1.0 / (1.0 + exp(z));
}

// ---------------------------------------------------------------- plaque
// species n1 n2 n3 c1 c2 c3  (model.py:133)
struct PlaqueDev {
  static constexpr int S = 6;
  // nonzeros of the modal linear-source matrix (model.py linear_source;
  // tables.py checks the host matrix against this pattern)
  __host__ __device__ static constexpr bool lin_nz(int s, int t) {
    return (s == 0 && t == 0) || (s == 1 && t == 1) || (s == 2 && t <= 1) || (s == 3 && t == 2) ||
           (s >= 4 && t == 4);
  }
  static constexpr bool kConv = true;
  static constexpr bool kMirror = false;  // closed by prescribed fluxes only
  // volume point inputs/outputs
  static constexpr int NVAL = 4;   // n1 n2 c1 c3
  static constexpr int NGRAD = 3;  // n1 c1 c3
  static constexpr int NFLUX = 2;  // rows n1, n2
  static constexpr int NNL = 1;    // bilinear part of S_c1
  __host__ __device__ static constexpr int val_sp(int k) { return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 3 : 5; }
  __host__ __device__ static constexpr int grad_sp(int k) { return k == 0 ? 0 : k == 1 ? 3 : 5; }
  // position of grad_sp(k) in the val_sp list (the gradient species are
  // a subset of the value species, so one coefficient copy serves both)
  __host__ __device__ static constexpr int grad_in_val(int k) { return k == 0 ? 0 : k == 1 ? 2 : 3; }
  __host__ __device__ static constexpr int flux_sp(int k) { return k; }
  __host__ __device__ static constexpr int nl_sp(int) { return 3; }
  __host__ __device__ static constexpr int flux_index(int s) { return s <= 1 ? s : -1; }
  __host__ __device__ static constexpr int nl_index(int s) { return s == 3 ? 0 : -1; }
  static constexpr int WALL_SP = 3;  // c1 drives the wall gates

  // model.py:147-157 (conv_flux) and :159-170 (bilinear source part)
  template <int D>
  __device__ __forceinline__ static void volume_point(const double* P, const double* v,
                                                      const double (*gM)[D], double (*fr)[D],
                                                      double* nl) {
    const double n1 = v[0], n2 = v[1], c1 = v[2], c3 = v[3];
    const double c1p = fmax(c1, 0.0);
    const double x11 = P[C11A] * n1 * rcp(c1p + P[C11B]);
    const double x13 = P[C13A] * n1 * rcp(fmax(c3, 0.0) + P[C13B]);
    const double x21 = P[C21A] * n2 * rcp(c1p + P[C21B]);
    const double x2n = P[C2NA] * n2 * rcp(fmax(n1, 0.0) + P[C2NB]);
#pragma unroll
    for (int b = 0; b < D; ++b) {
      fr[0][b] = x11 * gM[1][b] + x13 * gM[2][b];
      fr[1][b] = x21 * gM[1][b] - x2n * gM[0][b];
    }
    nl[0] = -P[ALPHA1] * n1 * c1 - P[ALPHA2] * n2 * c1;
  }

  // LLF convective part at one face point (flux.py:126-138 with
  // model.py:147-157 and the wave speed model.py:172-192): adds
  // 1/2 (F(u_in) + F(u_out)).n + 1/2 lambda (u_in - u_out) to q.
  __device__ __forceinline__ static void face_conv(const double* P, const double* ui,
                                                   const double* uo, const double* gn,
                                                   const double* dU, double* q) {
    double lam = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double* u = side ? uo : ui;
      const double c1p = fmax(u[3], 0.0);
      const double k11 = P[C11A] / (c1p + P[C11B]);
      const double k13 = P[C13A] / (fmax(u[5], 0.0) + P[C13B]);
      const double k21 = P[C21A] / (c1p + P[C21B]);
      const double k2n = P[C2NA] / (fmax(u[0], 0.0) + P[C2NB]);
      const double v0 = k11 * gn[3] + k13 * gn[5];
      const double v1 = k21 * gn[3] - k2n * gn[0];
      lam = fmax(lam, fmax(fabs(v0), fabs(v1)));
      f0 += u[0] * v0;
      f1 += u[1] * v1;
    }
    q[0] += 0.5 * f0;
    q[1] += 0.5 * f1;
#pragma unroll
    for (int s = 0; s < S; ++s) q[s] += 0.5 * lam * dU[s];
  }

  // Lane-per-species form of face_conv: every lane of a face group calls
  // it for its own species s; fetch(kind, sp) returns u_in (kind 0),
  // u_out (1) or the averaged normal derivative (2) of species sp from the
  // group's lanes (warp shuffles).  Returns q_s's convective part.
  template <class Fetch>
  __device__ __forceinline__ static double face_conv_lane(const double* P, int s, double dUs,
                                                          Fetch fetch) {
    const double g0 = fetch(2, 0), g3 = fetch(2, 3), g5 = fetch(2, 5);
    double lam = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double n1 = fetch(side, 0), n2 = fetch(side, 1), c1 = fetch(side, 3),
                   c3 = fetch(side, 5);
      const double c1p = fmax(c1, 0.0);
      const double k11 = P[C11A] * rcp(c1p + P[C11B]);
      const double k13 = P[C13A] * rcp(fmax(c3, 0.0) + P[C13B]);
      const double k21 = P[C21A] * rcp(c1p + P[C21B]);
      const double k2n = P[C2NA] * rcp(fmax(n1, 0.0) + P[C2NB]);
      const double v0 = k11 * g3 + k13 * g5;
      const double v1 = k21 * g3 - k2n * g0;
      lam = fmax(lam, fmax(fabs(v0), fabs(v1)));
      f0 = fma(n1, v0, f0);
      f1 = fma(n2, v1, f1);
    }
    double r = 0.5 * lam * dUs;
    if (s == 0) r = fma(0.5, f0, r);
    if (s == 1) r = fma(0.5, f1, r);
    return r;
  }

  // Coupled LLF physics once per face point.  fetch(kind, sp): u_in (0),
  // u_out (1), avg d_n u (2) of species sp at this point.  cv[0] = wave
  // speed lambda, cv[1 + s] = (F_s(u_in) + F_s(u_out)) . n for the flux
  // species s < NFX; the species-s convective flux is then
  // 1/2 cv[1+s] + 1/2 lambda (u_in - u_out)_s.
  static constexpr int NFX = 2;
  template <class Fetch>
  __device__ __forceinline__ static void face_point(const double* P, Fetch fetch, double* cv) {
    const double g0 = fetch(2, 0), g3 = fetch(2, 3), g5 = fetch(2, 5);
    double lam = 0.0, f0 = 0.0, f1 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double n1 = fetch(side, 0), n2 = fetch(side, 1), c1 = fetch(side, 3),
                   c3 = fetch(side, 5);
      const double c1p = fmax(c1, 0.0);
      const double k11 = P[C11A] * rcp(c1p + P[C11B]);
      const double k13 = P[C13A] * rcp(fmax(c3, 0.0) + P[C13B]);
      const double k21 = P[C21A] * rcp(c1p + P[C21B]);
      const double k2n = P[C2NA] * rcp(fmax(n1, 0.0) + P[C2NB]);
      const double v0 = k11 * g3 + k13 * g5;
      const double v1 = k21 * g3 - k2n * g0;
      lam = fmax(lam, fmax(fabs(v0), fabs(v1)));
      f0 = fma(n1, v0, f0);
      f1 = fma(n2, v1, f1);
    }
    cv[0] = lam;
    cv[1] = f0;
    cv[2] = f1;
  }

  // prescribed wall fluxes, inward-normal sign (model.py:194-209)
  __device__ __forceinline__ static void wall(const double* P, int tag, double c1, double* q) {
#pragma unroll
    for (int s = 0; s < S; ++s) q[s] = 0.0;
    if (tag == GAMMA1 || tag == GAMMA1_IN) q[0] = -P[MU1] * P[BETA1] * heaviside(c1 - P[C1S], P[EPSH]);
    if (tag == GAMMA1_IN) q[4] = -P[NU2] * P[SIGMA];
    if (tag == GAMMA2) q[1] = -P[MU2] * P[BETA2] * heaviside(c1 - P[C1SS], P[EPSH]);
  }
  __device__ __forceinline__ static double wall_lane(const double* P, int tag, int s, double c1) {
    if (s == 0 && (tag == GAMMA1 || tag == GAMMA1_IN))
      return -P[MU1] * P[BETA1] * heaviside(c1 - P[C1S], P[EPSH]);
    if (s == 4 && tag == GAMMA1_IN) return -P[NU2] * P[SIGMA];
    if (s == 1 && tag == GAMMA2) return -P[MU2] * P[BETA2] * heaviside(c1 - P[C1SS], P[EPSH]);
    return 0.0;
  }
  __device__ __forceinline__ static double mirror_value(const double*, int) { return 0.0; }
};

// --------------------------------------------------------------- reduced
// species n1 n3 c1  (model.py:212-264)
struct ReducedDev {
  static constexpr int S = 3;
  __host__ __device__ static constexpr bool lin_nz(int s, int t) {
    return (s == 1 && t == 0) || (s == 2 && t == 1);
  }
  static constexpr bool kConv = true;
  static constexpr bool kMirror = false;
  static constexpr int NVAL = 2;   // n1 c1
  static constexpr int NGRAD = 1;  // c1
  static constexpr int NFLUX = 1;  // row n1
  static constexpr int NNL = 1;    // -alpha1 n1 c1 on c1
  __host__ __device__ static constexpr int val_sp(int k) { return k == 0 ? 0 : 2; }
  __host__ __device__ static constexpr int grad_sp(int) { return 2; }
  __host__ __device__ static constexpr int grad_in_val(int) { return 1; }
  __host__ __device__ static constexpr int flux_sp(int) { return 0; }
  __host__ __device__ static constexpr int nl_sp(int) { return 2; }
  __host__ __device__ static constexpr int flux_index(int s) { return s == 0 ? 0 : -1; }
  __host__ __device__ static constexpr int nl_index(int s) { return s == 2 ? 0 : -1; }
  static constexpr int WALL_SP = 2;

  template <int D>
  __device__ __forceinline__ static void volume_point(const double* P, const double* v,
                                                      const double (*gM)[D], double (*fr)[D],
                                                      double* nl) {
    const double x11 = P[C11A] * v[0] * rcp(fmax(v[1], 0.0) + P[C11B]);
#pragma unroll
    for (int b = 0; b < D; ++b) fr[0][b] = x11 * gM[0][b];
    nl[0] = -P[ALPHA1] * v[0] * v[1];
  }

  __device__ __forceinline__ static void face_conv(const double* P, const double* ui,
                                                   const double* uo, const double* gn,
                                                   const double* dU, double* q) {
    double lam = 0.0, f0 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double* u = side ? uo : ui;
      const double v0 = P[C11A] / (fmax(u[2], 0.0) + P[C11B]) * gn[2];
      lam = fmax(lam, fabs(v0));
      f0 += u[0] * v0;
    }
    q[0] += 0.5 * f0;
#pragma unroll
    for (int s = 0; s < S; ++s) q[s] += 0.5 * lam * dU[s];
  }

  template <class Fetch>
  __device__ __forceinline__ static double face_conv_lane(const double* P, int s, double dUs,
                                                          Fetch fetch) {
    const double g2 = fetch(2, 2);
    double lam = 0.0, f0 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double v0 = P[C11A] * rcp(fmax(fetch(side, 2), 0.0) + P[C11B]) * g2;
      lam = fmax(lam, fabs(v0));
      f0 = fma(fetch(side, 0), v0, f0);
    }
    double r = 0.5 * lam * dUs;
    if (s == 0) r = fma(0.5, f0, r);
    return r;
  }

  static constexpr int NFX = 1;
  template <class Fetch>
  __device__ __forceinline__ static void face_point(const double* P, Fetch fetch, double* cv) {
    const double g2 = fetch(2, 2);
    double lam = 0.0, f0 = 0.0;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const double v0 = P[C11A] * rcp(fmax(fetch(side, 2), 0.0) + P[C11B]) * g2;
      lam = fmax(lam, fabs(v0));
      f0 = fma(fetch(side, 0), v0, f0);
    }
    cv[0] = lam;
    cv[1] = f0;
  }

  __device__ __forceinline__ static void wall(const double* P, int tag, double c1, double* q) {
#pragma unroll
    for (int s = 0; s < S; ++s) q[s] = 0.0;
    if (tag == GAMMA1 || tag == GAMMA1_IN) q[0] = -P[MU1] * P[BETA1] * heaviside(c1 - P[C1S], P[EPSH]);
  }
  __device__ __forceinline__ static double wall_lane(const double* P, int tag, int s, double c1) {
    if (s == 0 && (tag == GAMMA1 || tag == GAMMA1_IN))
      return -P[MU1] * P[BETA1] * heaviside(c1 - P[C1S], P[EPSH]);
    return 0.0;
  }
  __device__ __forceinline__ static double mirror_value(const double*, int) { return 0.0; }
};

// -------------------------------------------------------------- diffusion
// div(kappa grad u), no source; zero wall flux or constant Dirichlet data
// P[s] through the mirrored trace (tests/oracles.py:192-220).
template <int NS>
struct DiffusionDev {
  static constexpr int S = NS;
  __host__ __device__ static constexpr bool lin_nz(int, int) { return false; }
  static constexpr bool kConv = false;
  static constexpr bool kMirror = true;
  static constexpr int NVAL = 0, NGRAD = 0, NFLUX = 0, NNL = 0;
  __host__ __device__ static constexpr int val_sp(int) { return 0; }
  __host__ __device__ static constexpr int grad_sp(int) { return 0; }
  __host__ __device__ static constexpr int grad_in_val(int) { return 0; }
  __host__ __device__ static constexpr int flux_sp(int) { return 0; }
  __host__ __device__ static constexpr int nl_sp(int) { return 0; }
  __host__ __device__ static constexpr int flux_index(int) { return -1; }
  __host__ __device__ static constexpr int nl_index(int) { return -1; }
  static constexpr int WALL_SP = 0;
  template <int D>
  __device__ __forceinline__ static void volume_point(const double*, const double*, const double (*)[D],
                                                      double (*)[D], double*) {}
  __device__ __forceinline__ static void face_conv(const double*, const double*, const double*,
                                                   const double*, const double*, double*) {}
  template <class Fetch>
  __device__ __forceinline__ static double face_conv_lane(const double*, int, double, Fetch) {
    return 0.0;
  }
  static constexpr int NFX = 0;
  template <class Fetch>
  __device__ __forceinline__ static void face_point(const double*, Fetch, double*) {}
  __device__ __forceinline__ static void wall(const double*, int, double, double* q) {
#pragma unroll
    for (int s = 0; s < S; ++s) q[s] = 0.0;
  }
  __device__ __forceinline__ static double wall_lane(const double*, int, int, double) { return 0.0; }
  __device__ __forceinline__ static double mirror_value(const double* P, int s) { return P[s]; }
};

}  // namespace tdg

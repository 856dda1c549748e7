// Body of the signature-run 2D face kernel, included twice by
// kernels_fast.cuh (no include guard): TDG_SIG_KERNEL names the kernel,
// TDG_SIG_ASYNC selects how a face group's operands arrive --
//   0  k_faces_sig        record and rows loaded at the top of the group
//                         (states that stay in L2: C2)
//   1  k_faces_sig_async  the next group's record and rows staged through
//                         shared memory with cp.async while the current
//                         group computes (states larger than L2: C3)
template <int D, int K, class M, int NG>
__global__ void __launch_bounds__(128, SigFace<D, K, M>::MINB)
TDG_SIG_KERNEL(const __grid_constant__ OpParams p, const __grid_constant__ FaceSigTab<D, K, NG> tb,
            const double* __restrict__ U, double* __restrict__ ACC, int64_t ngroups,
            int64_t nwgroups) {
  using T = SigFace<D, K, M>;
  constexpr int NB = T::NB, S = T::S, SN = S * NB, F = T::F, FPW = T::FPW, NCV = T::NCV;
  constexpr int NFG = Dims<D, K>::NFG;
  __shared__ __align__(16) double sm[T::WARPS * FPW * T::PF];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / S, s = lane - grp * S, base = grp * S;
  const bool lane_ok = grp < FPW;
  double* xch = sm + (warp * FPW + (lane_ok ? grp : 0)) * T::PF;  // [3][F][XS]
  double* cvs = xch + 3 * T::XS * F;                              // [F][NCV]
  const double As = p.A[s];
#if TDG_SIG_ASYNC
  // Asynchronous staging of the next group's operands (cp.async, no
  // registers): the face record is requested at the top of the current
  // group (its address needs no load), the two coefficient rows after the
  // traces, when the element ids fetched at the top have arrived; both land
  // under the physics and projection of the current group.
  __shared__ __align__(16) double srow[T::WARPS * 32 * T::RST];
  __shared__ __align__(16) double sgeo[T::WARPS * FPW * NFG];
  double* rst = srow + (warp * 32 + lane) * T::RST;
  double* gst = sgeo + (warp * FPW + (lane_ok ? grp : 0)) * NFG;
  auto cp_row = [](double* dst, const double* src) {
    const unsigned d = unsigned(__cvta_generic_to_shared(dst));
    if constexpr (NB % 2 == 0) {
#pragma unroll
      for (int k = 0; k < NB / 2; ++k)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(d + 16 * k), "l"(src + 2 * k)
                     : "memory");
    } else {
#pragma unroll
      for (int k = 0; k < NB; ++k)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d + 8 * k), "l"(src + k)
                     : "memory");
    }
  };
  auto issue_rows = [&](int2 e) {
    cp_row(rst, U + int64_t(e.x) * SN + s * NB);
    cp_row(rst + T::RHALF, U + int64_t(e.y) * SN + s * NB);
  };
  auto issue_geo = [&](int64_t fc) {
    // the face's S lanes share its record: lane s copies 16-byte pieces
    // s, s + S, ... (S may be smaller than the piece count)
    if (lane_ok)
      for (int k = s; k < NFG / 2; k += S)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                         unsigned(__cvta_generic_to_shared(gst + 2 * k))),
                     "l"(p.ifgeo + fc * NFG + 2 * k)
                     : "memory");
  };
  auto face_of = [&](int64_t gw) {
    const int64_t f = gw * FPW + grp;
    return f < p.nif ? f : p.nif - 1;
  };
  const int64_t stride = int64_t(gridDim.x) * T::WARPS;
  const int64_t first = int64_t(blockIdx.x) * T::WARPS + warp;
  int2 el_n = make_int2(0, 0);
  int code_n = 0;
  if (first < ngroups) {
    const int64_t fc = face_of(first);
    el_n = __ldg(reinterpret_cast<const int2*>(p.ifel) + fc);
    code_n = __ldg(p.ifcode + fc);
    issue_geo(fc);
    issue_rows(el_n);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // walls: the low warps, before their interior groups
  for (int64_t gw = ngroups + first; gw < ngroups + nwgroups; gw += stride) {
#else
  for (int64_t gw = int64_t(blockIdx.x) * T::WARPS + warp; gw < ngroups + nwgroups;
       gw += int64_t(gridDim.x) * T::WARPS) {
    if (gw >= ngroups) {
#endif
      // prescribed wall flux: only the gate species' trace is needed
      const int64_t b = (gw - ngroups) * FPW + grp;
      const bool active = lane_ok && b < p.nbf;
      const int64_t bc = b < p.nbf ? b : p.nbf - 1;
      const int code = __ldg(p.bfcode + bc);
      const int ein = __ldg(p.bfel + bc);
      const double sfac = __ldg(p.bfgeo + bc);
      double ci[NB], ri[NB];
      load_row<NB>(U + int64_t(ein) * SN + s * NB, ci);
#pragma unroll
      for (int i = 0; i < NB; ++i) ri[i] = 0.0;
      const double* Bi = p.fB + code_tin(code) * F * NB;
      const int tag = code_tag(code);
#pragma unroll
      for (int q = 0; q < F; ++q) {
        double bi[NB];
        load_row<NB>(Bi + q * NB, bi);
        double u = 0.0;
#pragma unroll
        for (int i = 0; i < NB; ++i) u = fma(bi[i], ci[i], u);
        const double c1 = __shfl_sync(0xffffffffu, u, base + M::WALL_SP);
        const double Y = -tb.w[q] * sfac * M::wall_lane(p.P, tag, s, c1);
#pragma unroll
        for (int i = 0; i < NB; ++i) ri[i] = fma(Y, bi[i], ri[i]);
      }
      if (active) sig_acc_row<NB>(ACC + int64_t(ein) * SN + s * NB, ri, code_first_in(code));
#if TDG_SIG_ASYNC
  }
  for (int64_t gw = first; gw < ngroups; gw += stride) {
    const bool active = lane_ok && gw * FPW + grp < p.nif;
    const int code = code_n;
    const int2 el = el_n;
    const bool more = gw + stride < ngroups;  // warp-uniform
    int64_t fcn = 0;
    if (more) {
      fcn = face_of(gw + stride);
      el_n = __ldg(reinterpret_cast<const int2*>(p.ifel) + fcn);
      code_n = __ldg(p.ifcode + fcn);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    double jn[2][D], sfac, h, idi, ido, ci[NB], co[NB];
    {
      static_assert(NFG == 8, "2D face record");
#pragma unroll
      for (int a = 0; a < D; ++a) {
        jn[0][a] = gst[a];
        jn[1][a] = gst[D + a];
      }
      sfac = gst[4];
      h = gst[5];
      idi = gst[6];
      ido = gst[7];
      smem_row<NB>(rst, ci);
      smem_row<NB>(rst + T::RHALF, co);
    }
    __syncwarp();  // every lane has read the record before the next one lands
    if (more) issue_geo(fcn);
#else
      continue;
    }
    // face record and the two coefficient rows of species s (lanes past the
    // end recompute the last face and never store)
    const int64_t f = gw * FPW + grp;
    const bool active = lane_ok && f < p.nif;
    const int64_t fc = f < p.nif ? f : p.nif - 1;
    const int code = __ldg(p.ifcode + fc);
    const int2 el = __ldg(reinterpret_cast<const int2*>(p.ifel) + fc);
    double jn[2][D], sfac, h, idi, ido;
    {
      static_assert(NFG == 8, "2D face record");
      const double* g = p.ifgeo + fc * NFG;
      double w[4];
      if constexpr (NG == D) {
        ld256(g, w);
#pragma unroll
        for (int a = 0; a < D; ++a) {
          jn[0][a] = w[a];
          jn[1][a] = w[D + a];
        }
      }
      ld256(g + 4, w);
      sfac = w[0];
      h = w[1];
      idi = w[2];
      ido = w[3];
    }
    double ci[NB], co[NB];
    sig_load_row<NB>(U + int64_t(el.x) * SN + s * NB, ci);
    sig_load_row<NB>(U + int64_t(el.y) * SN + s * NB, co);
#endif
    // traces of both sides, jump and averaged normal derivative
    double dU[F], gav[F];
#pragma unroll
    for (int q = 0; q < F; ++q) {
      double u = 0.0, v = 0.0, gi[NG], go[NG];
#pragma unroll
      for (int a = 0; a < NG; ++a) gi[a] = go[a] = 0.0;
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        u = fma(tb.B[0][q][i], ci[i], u);
        v = fma(tb.B[1][q][i], co[i], v);
#pragma unroll
        for (int a = 0; a < NG; ++a) {
          gi[a] = fma(tb.G[0][q][i][a], ci[i], gi[a]);
          go[a] = fma(tb.G[1][q][i][a], co[i], go[a]);
        }
      }
      double x = gi[0], y = go[0];
      if constexpr (NG == D) {
        x = y = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          x = fma(jn[0][a], gi[a], x);
          y = fma(jn[1][a], go[a], y);
        }
      }
      dU[q] = u - v;
      gav[q] = 0.5 * (x + y);
      if constexpr (M::kConv) {
        if (lane_ok) {
          xch[(0 * F + q) * T::XS + s] = u;
          xch[(1 * F + q) * T::XS + s] = v;
          xch[(2 * F + q) * T::XS + s] = gav[q];
        }
      }
    }
#if TDG_SIG_ASYNC
    // the next group's rows: this group's are in registers, the element ids
    // requested at the top have arrived
    if (more) issue_rows(el_n);
    asm volatile("cp.async.commit_group;" ::: "memory");
#endif
    // coupled convective physics once per face point (smem transpose)
    double fl[F];  // penalty + convective flux per point
#pragma unroll
    for (int q = 0; q < F; ++q) fl[q] = 0.0;
    if constexpr (M::kConv) {
      __syncwarp();
      if (lane_ok) {
        for (int q = s; q < F; q += S) {
          const double* xq = xch + q * T::XS;
          auto fetch = [xq](int kind, int sp) { return xq[kind * F * T::XS + sp]; };
          M::face_point(p.P, fetch, cvs + q * NCV);
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < F; ++q) {
        double c = 0.5 * cvs[q * NCV] * dU[q];
#pragma unroll
        for (int k = 0; k < M::NFX; ++k)
          if (s == k) c = fma(0.5, cvs[q * NCV + 1 + k], c);
        fl[q] = c;
      }
    }
    // penalty A_hat . n (operator.py:336-357), lifting on the needed side(s)
    if (p.scheme == IP) {
      const double c = p.eta / h * As;
#pragma unroll
      for (int q = 0; q < F; ++q) fl[q] = fma(c, dU[q], fl[q]);
    } else if (p.scheme != BO) {
      const bool br2 = p.scheme == BR2;
      const bool use_in = br2 || code_minus_in(code);
      const bool use_out = br2 || !code_minus_in(code);
      const double fac = (p.scheme == CDG ? 4.0 : 2.0) * p.chi_e * As * (br2 ? 0.5 : 1.0) * 0.5 * sfac;
      if (use_in) {
        const double fi = fac * idi;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          double a = 0.0;
#pragma unroll
          for (int pp = 0; pp < F; ++pp) a = fma(tb.Pw[0][q][pp], dU[pp], a);
          fl[q] = fma(fi, a, fl[q]);
        }
      }
      if (use_out) {
        const double fo = fac * ido;
#pragma unroll
        for (int q = 0; q < F; ++q) {
          double a = 0.0;
#pragma unroll
          for (int pp = 0; pp < F; ++pp) a = fma(tb.Pw[1][q][pp], dU[pp], a);
          fl[q] = fma(fo, a, fl[q]);
        }
      }
    }
    // projection onto both sides' test functions
    double ri[NB], ro[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) ri[i] = ro[i] = 0.0;
    const double hadj = 0.5 * p.adj * As;
#pragma unroll
    for (int q = 0; q < F; ++q) {
      const double wq = tb.w[q] * sfac;
      const double Y = wq * (As * gav[q] - fl[q]);
      const double X = wq * hadj * dU[q];
      double Xi[NG], Xo[NG];
#pragma unroll
      for (int a = 0; a < NG; ++a) {
        Xi[a] = NG == D ? X * jn[0][a] : X;
        Xo[a] = NG == D ? X * jn[1][a] : X;
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        double a = fma(Y, tb.B[0][q][i], ri[i]);
        double b = fma(-Y, tb.B[1][q][i], ro[i]);
#pragma unroll
        for (int c = 0; c < NG; ++c) {
          a = fma(Xi[c], tb.G[0][q][i][c], a);
          b = fma(Xo[c], tb.G[1][q][i][c], b);
        }
        ri[i] = a;
        ro[i] = b;
      }
    }
    if (active) {
      sig_acc_row<NB>(ACC + int64_t(el.x) * SN + s * NB, ri, code_first_in(code));
      if (!code_skip_out(code))
        sig_acc_row<NB>(ACC + int64_t(el.y) * SN + s * NB, ro, code_first_out(code));
    }
    __syncwarp();  // the warp's scratch is rewritten by the next group
  }
}

// tilt_kernels.cuh — LADMAP inner loop, Algorithm 1 outer loop and the kernels of libtilt.
// Paper: Ren & Lin, arXiv 1205.5351 (/root/reference/PAPER.md, P:<line>); readings: DESIGN.md.
#pragma once

#include "tilt_device.cuh"

namespace tilt {

// ---------------------------------------------------------------------------------------------
// Shared-memory / workspace layout per size class. gplanes = 3 (implicit homography), 2 (implicit
// affine) or p (explicit K).
// ---------------------------------------------------------------------------------------------
template <class C>
struct Layout {
  static __host__ __device__ size_t vec_floats() { return 5 * (size_t)C::MAXD; }
  static __host__ __device__ size_t svd_floats(int, int n) { return 3 * (size_t)C::MAXD * n; }
  static __host__ __device__ size_t plane_floats(int ld, int n, int gplanes) { return (size_t)(5 + gplanes) * ld * n; }
  static __host__ __device__ size_t smem_bytes(int ld, int n, int gplanes) {
    size_t s = vec_floats();
    if (C::SVD_SMEM) s += svd_floats(ld, n);
    else if (C::B_SMEM) s += (size_t)C::MAXD * n;
    if (C::PLANES_SMEM) s += plane_floats(ld, n, gplanes);
    return s * sizeof(float);
  }
  static __host__ __device__ size_t ws_floats(int ld, int n, int gplanes) {
    size_t s = 0;
    if (!C::SVD_SMEM) s += svd_floats(ld, n) - (C::B_SMEM ? (size_t)C::MAXD * n : 0);
    if (!C::PLANES_SMEM) s += plane_floats(ld, n, gplanes);
    return (s + 31) & ~size_t(31);
  }
};

template <class C>
__device__ __forceinline__ Ctx<C> make_ctx(float* smem, float* ws, Scal* sc, int m, int n, int p) {
  Ctx<C> cx;
  const int ld = ld_of<C>(m, n);
  float* sp = smem;
  float* gp = ws;
  cx.ns = reinterpret_cast<float4*>(sp);
  cx.hv = sp + 4 * C::MAXD;
  sp += 5 * C::MAXD;
  const int blk = ld * n;
  const int sblk = C::MAXD * n;
  if constexpr (C::SVD_SMEM) {
    cx.B = sp;
    cx.V = sp + sblk;
    cx.S = sp + 2 * sblk;
    sp += 3 * sblk;
  } else if constexpr (C::B_SMEM) {
    cx.B = sp;
    sp += sblk;
    cx.V = gp;
    cx.S = gp + sblk;
    gp += 2 * sblk;
  } else {
    cx.B = gp;
    cx.V = gp + sblk;
    cx.S = gp + 2 * sblk;
    gp += 3 * sblk;
  }
  cx.lds = C::MAXD;
  float* pl;
  if constexpr (C::PLANES_SMEM) {
    pl = sp;
  } else {
    pl = gp;
  }
  cx.D = pl;
  cx.A = pl + blk;
  cx.E = pl + 2 * blk;
  cx.Y = pl + 3 * blk;
  cx.T = pl + 4 * blk;  // J dtau of the ADM baseline
  cx.G = pl + 5 * blk;
  cx.sc = sc;
  cx.m = m;
  cx.n = n;
  cx.p = p;
  cx.ld = ld;
  cx.pl = blk;
  const float s = 0.5f * (float)max(m, n);
  cx.inv_s = 1.f / s;
  cx.ci = 0.5f * (float)(m - 1);
  cx.cj = 0.5f * (float)(n - 1);
  return cx;
}

__host__ __device__ inline float default_jacobi_tol(int m) { return 8.f * sqrtf((float)m) * 5.9604645e-8f; }

template <class C>
__device__ __forceinline__ void zero_planes(float* X, size_t count) {
  for (size_t e = threadIdx.x; e < count; e += C::NT) X[e] = 0.f;
}

// ---------------------------------------------------------------------------------------------
// sigma_1 of a plane (mu_0 = mu0_scale / sigma_1(D_hat), reading Z3): warm Jacobi; leaves V warm.
// ---------------------------------------------------------------------------------------------
template <class C>
__device__ float sigma1_of_plane(Ctx<C>& cx, const float* X, float tol, int max_sweeps, bool warm, int* sweeps) {
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < cx.pl; pi.next(C::NT)) cx.S[pi.j * cx.lds + pi.i] = X[pi.idx];
  __syncthreads();
  auto none = [](int, int, float4) {};
  SvtOut so = svt<C, false>(cx, cx.S, 0.f, tol, max_sweeps, warm, none, warm);
  *sweeps = so.sweeps;
  return cx.sc->svt_sig1;
}

// ---------------------------------------------------------------------------------------------
// LADMAP inner loop (P:437-468 Eqs. A, E, Y, mu, rho; Cond1/2 P:489-497; constrained form
// Eq. newvars2 P:731-737 with errata E1 (+ dual step) and E2 (N_k from E_k)):
//   M_k = A_k - Y_k/mu_k - W^TW(A_k + E_k - D)              (in S on entry / from the dual pass)
//   A_{k+1} = S_{1/mu_k}(M_k)                                (warm Jacobi SVT)
//   N_k = E_k - Y_k/mu_k - W^TW(A_{k+1} + E_k - D), E_{k+1} = T_{lam/mu_k}(N_k)
//   R = W^TW(A_{k+1} + E_{k+1} - D), Y_{k+1} = Y_k + mu_k R  (R reused for M_{k+1}: 2 products)
//   crit1 = ||R||/||W^TW D||, crit2 = mu_k max(||dA||, ||dE||)/||W^TW D||
//   rho = rho0 if crit2 < eps2 else 1, mu_{k+1} = min(mu_max, rho mu_k)
// ---------------------------------------------------------------------------------------------
struct InnerOut {
  int iters, sweeps, caps, rotations;
  float mu, crit1, crit2;
  bool converged;
};

template <class C, class PR>
__device__ InnerOut ladmap_inner(Ctx<C>& cx, const DevParams& P, float lam, float mu0, float mu_max, float denom,
                                 float tol, const uint8_t* replay, float* trace) {
  const int ld = cx.ld, pl = cx.pl;
  const float inv_den = 1.f / denom;
  const int niter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
  float* __restrict__ Ap = cx.A;
  float* __restrict__ Ep = cx.E;
  float* __restrict__ Yp = cx.Y;
  const float* __restrict__ Dp = cx.D;
  InnerOut o;
  o.iters = 0;
  o.sweeps = 0;
  o.caps = 0;
  o.rotations = 0;
  o.crit1 = o.crit2 = __int_as_float(0x7fc00000);
  o.converged = false;
  float mu = mu0;
  o.mu = mu;
  const bool warm = P.svd_warm != 0;
  auto vres = [&](int idx) { return res3(Ap[idx], Ep[idx], Dp[idx]); };
  for (int k = 0; k < niter; ++k) {
    // ---- A step: A_{k+1} = S_{1/mu}(M_k), M_k in S ------------------------------------------
    float dA2 = 0.f;
    SvtOut so = svt<C, true>(
        cx, cx.S, 1.f / mu, tol, P.jacobi_max_sweeps, warm,
        [&](int i0, int j, float4 a) {
          float* ap = Ap + j * ld + i0;
          const float4 o4 = *reinterpret_cast<const float4*>(ap);
          float d;
          d = a.x - o4.x; dA2 = fmaf(d, d, dA2);
          d = a.y - o4.y; dA2 = fmaf(d, d, dA2);
          d = a.z - o4.z; dA2 = fmaf(d, d, dA2);
          d = a.w - o4.w; dA2 = fmaf(d, d, dA2);
          *reinterpret_cast<float4*>(ap) = a;
        },
        warm && (k % P.ns_period == P.ns_period - 1 || k + 1 == niter));
    o.sweeps += so.sweeps;
    o.caps += so.capped ? 1 : 0;
    o.rotations += so.rotations;
    // ---- E step ---------------------------------------------------------------------------
    const float inv_mu = 1.f / mu;
    const float thr = lam * inv_mu;
    float s[8], z[9];
    PR::reduce(cx, vres, s);
    PR::coeffs(cx, s, z);
    float dE2 = 0.f;
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      const int idx = pi.idx;
      const float e = Ep[idx];
      const float v = res3(Ap[idx], e, Dp[idx]);
      const float pv = v - PR::apply(cx, idx, pi.i, pi.j, z);
      const float nk = e - pv - Yp[idx] * inv_mu;
      const float en = copysignf(fmaxf(fabsf(nk) - thr, 0.f), nk);
      const float d = en - e;
      dE2 = fmaf(d, d, dE2);
      Ep[idx] = en;
    }
    float dd[2] = {dA2, dE2};
    block_sum_f<C, 2>(dd, cx.sc);
    const float crit2 = mu * sqrtf(fmaxf(dd[0], dd[1])) * inv_den;
    int rho_bit = crit2 < P.eps2 ? 1 : 0;
    if (replay) rho_bit = replay[k] & 1;  // parity protocol (Z21): bit 0 = rho decision
    const float mu_next = fminf(mu_max, rho_bit ? P.rho0 * mu : mu);
    const float inv_mun = 1.f / mu_next;
    // ---- dual step + next M ----------------------------------------------------------------
    PR::reduce(cx, vres, s);
    PR::coeffs(cx, s, z);
    float c1 = 0.f;
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      const int idx = pi.idx;
      const float a = Ap[idx];
      const float v = res3(a, Ep[idx], Dp[idx]);
      const float r = v - PR::apply(cx, idx, pi.i, pi.j, z);
      const float y = fmaf(mu, r, Yp[idx]);
      Yp[idx] = y;
      c1 = fmaf(r, r, c1);
      cx.S[pi.j * cx.lds + pi.i] = a - r - y * inv_mun;
    }
    float cc[1] = {c1};
    block_sum_f<C, 1>(cc, cx.sc);
    const float crit1 = sqrtf(cc[0]) * inv_den;
    if (trace && threadIdx.x == 0) {
      trace[4 * k + 0] = mu;
      trace[4 * k + 1] = crit1;
      trace[4 * k + 2] = crit2;
      trace[4 * k + 3] = (float)rho_bit;
    }
    o.iters = k + 1;
    o.crit1 = crit1;
    o.crit2 = crit2;
    o.mu = mu;
    bool stop = crit1 < P.eps1 && crit2 < P.eps2;
    if (replay) stop = (replay[k] & 2) != 0;  // bit 1 = the replayed run's inner loop ended here
    if (stop) o.converged = true;
    if (stop && P.fixed_inner <= 0) break;
    mu = mu_next;
  }
  return o;
}

// ---------------------------------------------------------------------------------------------
// ADM baseline inner loop (Zhang et al.), Gauss-Seidel on the
// augmented Lagrangian of Eq. TILT_3 with the penalty mu_{k+1} = rho mu_k (unbounded):
//   A_{k+1} = S_{1/mu}(D + J dtau_k - E_k + Y_k/mu)
//   E_{k+1} = T_{lam/mu}(D + J dtau_k - A_{k+1} + Y_k/mu)
//   dtau_{k+1} = G^{-1} J^T v, v = A_{k+1} + E_{k+1} - D - Y_k/mu   (J dtau = K K^T v)
//   Y_{k+1} = Y_k + mu (D + J dtau_{k+1} - A_{k+1} - E_{k+1})
// stop when ||D + J dtau - A - E||_F / ||D||_F < adm_tol (reading Z24). Cold start A = D,
// E = Y = 0, J dtau = 0. Returns K^T v of the last dtau step in s_last.
// ---------------------------------------------------------------------------------------------
template <class C, class PR>
__device__ InnerOut adm_inner(Ctx<C>& cx, const DevParams& P, float lam, float mu0, float tol, float (&s_last)[8]) {
  const int ld = cx.ld, pl = cx.pl;
  const int niter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
  float* __restrict__ Ap = cx.A;
  float* __restrict__ Ep = cx.E;
  float* __restrict__ Yp = cx.Y;
  float* __restrict__ Tp = cx.T;
  const float* __restrict__ Dp = cx.D;
  for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
    Ap[idx] = Dp[idx];
    Ep[idx] = 0.f;
    Yp[idx] = 0.f;
    Tp[idx] = 0.f;
  }
  float nd2 = 0.f;
  for (int idx = threadIdx.x; idx < pl; idx += C::NT) nd2 = fmaf(Dp[idx], Dp[idx], nd2);
  float nn[1] = {nd2};
  block_sum_f<C, 1>(nn, cx.sc);
  const float inv_nd = nn[0] > 0.f ? rsqrtf(nn[0]) : 1.f;
  InnerOut o;
  o.iters = o.sweeps = o.caps = o.rotations = 0;
  o.crit1 = o.crit2 = __int_as_float(0x7fc00000);
  o.converged = false;
  float mu = mu0;
  o.mu = mu;
  const bool warm = P.svd_warm != 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s_last[q] = 0.f;
  for (int k = 0; k < niter; ++k) {
    const float inv_mu = 1.f / mu;
    // A step: S <- D + J dtau - E + Y/mu, A = S_{1/mu}(S)
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      const int idx = pi.idx;
      cx.S[pi.j * cx.lds + pi.i] = fmaf(Yp[idx], inv_mu, Dp[idx] + Tp[idx] - Ep[idx]);
    }
    __syncthreads();
    SvtOut so = svt<C, true>(
        cx, cx.S, inv_mu, tol, P.jacobi_max_sweeps, warm,
        [&](int i0, int j, float4 a) { *reinterpret_cast<float4*>(Ap + j * ld + i0) = a; },
        warm && (k % P.ns_period == P.ns_period - 1 || k + 1 == niter));
    o.sweeps += so.sweeps;
    o.caps += so.capped ? 1 : 0;
    o.rotations += so.rotations;
    // E step
    const float thr = lam * inv_mu;
    for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
      const float x = fmaf(Yp[idx], inv_mu, Dp[idx] + Tp[idx] - Ap[idx]);
      Ep[idx] = copysignf(fmaxf(fabsf(x) - thr, 0.f), x);
    }
    __syncthreads();
    // dtau step: J dtau = K K^T v
    float s[8], z[9];
    auto vf = [&](int idx) { return fmaf(-Yp[idx], inv_mu, Ap[idx] + Ep[idx] - Dp[idx]); };
    PR::reduce(cx, vf, s);
    PR::coeffs(cx, s, z);
    float r2 = 0.f;
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      const int idx = pi.idx;
      const float jdt = PR::apply(cx, idx, pi.i, pi.j, z);
      Tp[idx] = jdt;
      const float r = Dp[idx] + jdt - Ap[idx] - Ep[idx];
      Yp[idx] = fmaf(mu, r, Yp[idx]);
      r2 = fmaf(r, r, r2);
    }
    float rr[1] = {r2};
    block_sum_f<C, 1>(rr, cx.sc);
#pragma unroll
    for (int q = 0; q < 8; ++q) s_last[q] = s[q];
    const float resid = sqrtf(rr[0]) * inv_nd;
    o.iters = k + 1;
    o.crit1 = resid;
    o.mu = mu;
    mu *= P.adm_rho;
    if (resid < P.adm_tol) {
      o.converged = true;
      if (P.fixed_inner <= 0) break;
    }
  }
  return o;
}

// X <- W^TW X (in place)
template <class C, class PR>
__device__ __forceinline__ void project_plane(Ctx<C>& cx, float* X) {
  float s[8], z[9];
  PR::reduce(cx, [&](int idx) { return X[idx]; }, s);
  PR::coeffs(cx, s, z);
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < cx.pl; pi.next(C::NT))
    X[pi.idx] -= PR::apply(cx, pi.idx, pi.i, pi.j, z);
  __syncthreads();
}

// ||W^TW X||_F
template <class C, class PR>
__device__ __forceinline__ float proj_norm(Ctx<C>& cx, const float* X) {
  float s[8], z[9];
  PR::reduce(cx, [&](int idx) { return X[idx]; }, s);
  PR::coeffs(cx, s, z);
  float acc = 0.f;
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < cx.pl; pi.next(C::NT)) {
    const float r = X[pi.idx] - PR::apply(cx, pi.idx, pi.i, pi.j, z);
    acc = fmaf(r, r, acc);
  }
  float a1[1] = {acc};
  block_sum_f<C, 1>(a1, cx.sc);
  return sqrtf(a1[0]);
}

// Prologue of an inner loop: R_0 = W^TW(A + E - D), M_0 = A - R_0 - Y/mu0 into S.
template <class C, class PR>
__device__ __forceinline__ void write_m0(Ctx<C>& cx, float mu0) {
  float s[8], z[9];
  const float* Ap = cx.A;
  const float* Ep = cx.E;
  const float* Dp = cx.D;
  PR::reduce(cx, [&](int idx) { return res3(Ap[idx], Ep[idx], Dp[idx]); }, s);
  PR::coeffs(cx, s, z);
  const float inv = 1.f / mu0;
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < cx.pl; pi.next(C::NT)) {
    const int idx = pi.idx;
    const float v = res3(Ap[idx], Ep[idx], Dp[idx]);
    const float r = v - PR::apply(cx, idx, pi.i, pi.j, z);
    cx.S[pi.j * cx.lds + pi.i] = Ap[idx] - r - cx.Y[idx] * inv;
  }
  __syncthreads();
}

template <class C>
__device__ __forceinline__ float plane_l1(Ctx<C>& cx, const float* X) {
  float acc = 0.f;
  for (int idx = threadIdx.x; idx < cx.pl; idx += C::NT) acc += fabsf(X[idx]);
  float a1[1] = {acc};
  block_sum_f<C, 1>(a1, cx.sc);
  return a1[0];
}

// Column-major padded plane -> row-major global [m][n]
template <class C>
__device__ __forceinline__ void store_plane(float* __restrict__ out, const float* X, int m, int n, int ld, bool zero) {
  for (int o = threadIdx.x; o < m * n; o += C::NT) {
    const int i = o / n, j = o - i * n;
    out[o] = zero ? 0.f : X[j * ld + i];
  }
}

// Row-major global [m][n] -> column-major padded plane (padding rows set to 0)
template <class C>
__device__ __forceinline__ void load_plane(float* X, const float* __restrict__ in, int m, int n, int ld) {
  for (int e = threadIdx.x; e < ld * n; e += C::NT) {
    const int j = e / ld, i = e - j * ld;
    X[e] = (i < m) ? in[i * n + j] : 0.f;
  }
}

// ---------------------------------------------------------------------------------------------
// Algorithm 1 for one patch
// ---------------------------------------------------------------------------------------------
struct SolveArgs {
  const float* images;
  int n_images, H, W;
  const int* patch_image;
  const int* boxes;
  const float* tau0;
  int B, m, n, p, kind;
  DevParams P;
  float* tau_out;
  float* A_out;
  float* E_out;
  float* Y_out;
  tilt_report* rep;
  const tilt_report* rep_prev;  // pyramid: counters of the coarse level (accumulated)
  int* counter;
  float* ws;
  size_t ws_stride;
  int ctas_per_sm;  // host-side launch cap (0: occupancy limit)
  // pyramid warm start (reading Z26): the coarse level's A, E, Y [B][m/2][n/2] and its reports
  const float* warm_A;
  const float* warm_E;
  const float* warm_Y;
  const tilt_report* warm_rep;
};

template <class C>
__device__ void solve_patch(const SolveArgs& a, Ctx<C>& cx, int b) {
  using PR = ProjImplicit;
  const DevParams& P = a.P;
  const int m = a.m, n = a.n, p = a.p, ld = cx.ld, pl = cx.pl;
  const int bx[4] = {a.boxes[4 * b], a.boxes[4 * b + 1], a.boxes[4 * b + 2], a.boxes[4 * b + 3]};
  const float* img = a.images + (size_t)a.patch_image[b] * a.H * a.W;
  double tau[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tau[q] = 0.0;
  if (a.tau0) {
    for (int q = 0; q < p; ++q) tau[q] = a.tau0[b * p + q];
  } else {
    tau[0] = 1.0;
    tau[3] = 1.0;
  }
  const float lam = P.lambda > 0.f ? P.lambda : rsqrtf((float)max(m, n));
  const float tol = P.jacobi_tol > 0.f ? P.jacobi_tol : default_jacobi_tol(m);
  const bool warm = P.svd_warm != 0;
  const int gpl = p == 8 ? 3 : 2;
  zero_planes<C>(cx.D, (size_t)(5 + gpl) * pl);  // padding rows stay 0 from here on
  set_identity<C>(cx.V, cx.lds, n);
  __syncthreads();
  int status = TILT_PATCH_MAX_OUTER, stop_rule = 0, outer = 0, inner_total = 0, sweeps_total = 0,
      aux_total = 0, caps = 0, rank = 0, band = 0, svt_rank = 0, rot_total = 0;
  const float fnan = __int_as_float(0x7fc00000);
  float f = fnan, f_prev = fnan, crit1 = fnan, crit2 = fnan, dtau_inf = fnan, mu_last = fnan, nd = fnan;
  bool have_state = false, have_fprev = false;
  const bool box_ok = bx[2] == n && bx[3] == m;  // all boxes of a call share the window size
  if (!box_ok) status = TILT_PATCH_BAD_BOX;
  const int n_outer = !box_ok ? 0 : P.fixed_outer > 0 ? P.fixed_outer : P.max_outer;
  for (int it = 0; it < n_outer; ++it) {
    // Step 1: D o tau and the Jacobian factors (fp64 per pixel, stored fp32), escape check
    const WarpGeom g = make_geom(bx, tau, a.kind);
    bool esc = false;
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      if (pi.i >= m) continue;
      double d, gx, gy, gz;
      if (!warp_pixel(g, img, a.H, a.W, pi.i, pi.j, d, gx, gy, gz)) esc = true;
      cx.D[pi.idx] = (float)d;
      cx.G[pi.idx] = (float)gx;
      cx.G[pl + pi.idx] = (float)gy;
      if (p == 8) cx.G[2 * pl + pi.idx] = (float)gz;
    }
    if (__syncthreads_or(esc)) {
      status = TILT_PATCH_WINDOW_ESCAPE;
      break;
    }
    double qr[24];
    int l = 0;
    if (P.constraint_mode == TILT_CONSTRAINTS_CENTER_AREA) {
      constraint_rows(tau, a.kind, m, n, qr);
      l = 3;
    }
    const int st = orthonormalise_implicit<C>(cx, qr, l);
    nd = cx.sc->nd;
    if (st != TILT_PATCH_CONVERGED) {
      status = st;
      break;
    }
    // Step 2 warm start (Eq. warm_start; Eq. Y_new_warmstart; Z4); the
    // pyramid's fine level may start from the coarse state replicated 2x2 and halved (Z26)
    const bool from_coarse = it == 0 && P.vws && a.warm_A &&
                             (a.warm_rep[b].status == TILT_PATCH_CONVERGED || a.warm_rep[b].status == TILT_PATCH_MAX_OUTER);
    if (from_coarse) {
      const int mc = m / 2, nc = n / 2;
      const size_t o = (size_t)b * mc * nc;
      for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
        if (pi.i >= m) continue;
        const size_t c = o + (size_t)(pi.i / 2) * nc + pi.j / 2;
        cx.A[pi.idx] = 0.5f * a.warm_A[c];
        cx.E[pi.idx] = 0.5f * a.warm_E[c];
        cx.Y[pi.idx] = 0.5f * a.warm_Y[c];
      }
      __syncthreads();
      project_plane<C, PR>(cx, cx.Y);
      have_state = true;
    } else if (!have_state || !P.vws) {
      for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
        cx.A[idx] = cx.D[idx];
        cx.E[idx] = 0.f;
        cx.Y[idx] = 0.f;
      }
      __syncthreads();
    } else {
      project_plane<C, PR>(cx, cx.Y);
    }
    const float denom0 = proj_norm<C, PR>(cx, cx.D);
    const float denom = denom0 > 0.f ? denom0 : 1.f;
    int aux = 0;
    const float s1 = sigma1_of_plane<C>(cx, cx.D, tol, P.jacobi_max_sweeps, warm, &aux);
    aux_total += aux;
    const float mu0 = s1 > 0.f ? P.mu0_scale / s1 : P.mu0_scale;
    const float mu_max = P.mu_max_ratio * mu0;
    const size_t toff = ((size_t)b * P.max_outer + it) * P.max_inner;
    float s_adm[8];
    InnerOut io;
    if (P.inner_solver == 1) {
      io = adm_inner<C, PR>(cx, P, lam, mu0, tol, s_adm);
    } else {
      write_m0<C, PR>(cx, mu0);
      io = ladmap_inner<C, PR>(cx, P, lam, mu0, mu_max, denom, tol, P.rho_replay ? P.rho_replay + toff : nullptr,
                               P.trace ? P.trace + 4 * toff : nullptr);
    }
    have_state = true;
    inner_total += io.iters;
    sweeps_total += io.sweeps;
    caps += io.caps;
    rot_total += io.rotations;
    crit1 = io.crit1;
    crit2 = io.crit2;
    mu_last = io.mu;
    const float nuc = cx.sc->svt_nuc;
    rank = cx.sc->svt_relrank;
    band = cx.sc->svt_band;
    svt_rank = cx.sc->svt_rank;
    // Step 3: dtau = G^{-1} J^T (A + E - D_hat) = L^{-T} K^T (A + E - D_hat)  (Eq. Delta_tau)
    float s[8];
    double sd[8];
    if (P.inner_solver == 1) {  // the ADM's own dtau (Eq. update_detla_Tau)
#pragma unroll
      for (int q = 0; q < 8; ++q) sd[q] = s_adm[q];
    } else {
      PR::reduce(cx, [&](int idx) { return res3(cx.A[idx], cx.E[idx], cx.D[idx]); }, s);
#pragma unroll
      for (int q = 0; q < 8; ++q) sd[q] = cx.sc->sd[q];  // K^T (A + E - D_hat) in fp64
    }
    const float l1 = plane_l1<C>(cx, cx.E);
    const double* Li = cx.sc->Linv;
    double dt_inf = 0.0;
    bool finite = true;
    for (int q = 0; q < p; ++q) {  // Step 4: tau += dtau
      double dq = 0.0;
      for (int r = q; r < p; ++r) dq += Li[r * 8 + q] * sd[r];
      tau[q] = (double)(float)(tau[q] + dq);  // tau carried in fp32 between outer iterations (Z28)
      dt_inf = fmax(dt_inf, fabs(dq));
      finite = finite && isfinite(tau[q]);
    }
    dtau_inf = (float)dt_inf;
    f = nuc + lam * l1;
    outer = it + 1;
    if (!finite || !isfinite(f) || f > 1e12f) {
      status = TILT_PATCH_DIVERGED;
      break;
    }
    int rule = 0;
    if (have_fprev && fabsf(f - f_prev) < P.obj_tol * fabsf(f_prev)) rule = 1;
    else if (dtau_inf < P.tau_tol) rule = 2;
    f_prev = f;
    have_fprev = true;
    if (rule) {
      status = TILT_PATCH_CONVERGED;
      stop_rule = rule;
      if (P.fixed_outer <= 0) break;
    } else {
      status = TILT_PATCH_MAX_OUTER;
      stop_rule = 3;
    }
    __syncthreads();
  }
  __syncthreads();
  // outputs
  if (a.A_out) store_plane<C>(a.A_out + (size_t)b * m * n, cx.A, m, n, ld, !have_state);
  if (a.E_out) store_plane<C>(a.E_out + (size_t)b * m * n, cx.E, m, n, ld, !have_state);
  if (a.Y_out) store_plane<C>(a.Y_out + (size_t)b * m * n, cx.Y, m, n, ld, !have_state);
  if (threadIdx.x == 0) {
    for (int q = 0; q < p; ++q) a.tau_out[b * p + q] = (float)tau[q];
    if (a.rep) {
      tilt_report r;
      r.status = status;
      r.stop_rule = stop_rule;
      r.outer_iters = outer;
      r.inner_iters = inner_total;
      r.jacobi_sweeps = sweeps_total;
      r.aux_sweeps = aux_total;
      r.rank = rank;
      r.rank_band = band;
      r.svt_rank = svt_rank;
      r.sweep_cap_hits = caps;
      r.objective = f;
      r.crit1 = crit1;
      r.crit2 = crit2;
      r.patch_norm = nd;
      r.dtau_inf = dtau_inf;
      r.mu_last = mu_last;
      r.jacobi_rotations = rot_total;
      r.kernel_path = 1;
      r.svd_warm_steps = 0;
      if (a.rep_prev) {
        const tilt_report& pr = a.rep_prev[b];
        r.outer_iters += pr.outer_iters;
        r.inner_iters += pr.inner_iters;
        r.jacobi_sweeps += pr.jacobi_sweeps;
        r.aux_sweeps += pr.aux_sweeps;
        r.sweep_cap_hits += pr.sweep_cap_hits;
        r.jacobi_rotations += pr.jacobi_rotations;
      }
      a.rep[b] = r;
    }
  }
  __syncthreads();
}

template <class C>
__global__ void __launch_bounds__(C::NT, C::MINB) k_solve(SolveArgs a) {
  extern __shared__ float4 dsm4[];
  __shared__ Scal sc;
  float* ws = a.ws ? a.ws + (size_t)blockIdx.x * a.ws_stride : nullptr;
  Ctx<C> cx = make_ctx<C>(reinterpret_cast<float*>(dsm4), ws, &sc, a.m, a.n, a.p);
  while (true) {
    if (threadIdx.x == 0) sc.patch = atomicAdd(a.counter, 1);
    __syncthreads();
    const int b = sc.patch;
    __syncthreads();
    if (b >= a.B) break;
    solve_patch<C>(a, cx, b);
  }
}

// ---------------------------------------------------------------------------------------------
// Inner loop only (Table 1 setting): explicit projector from a given J
// ---------------------------------------------------------------------------------------------
struct InnerArgs {
  const float* D;
  const float* J;
  const float* Q;
  int l, B, m, n, p;
  DevParams P;
  float* A;
  float* E;
  float* Y;
  tilt_report* rep;
  float* ws;
  size_t ws_stride;
};

template <class C>
__global__ void __launch_bounds__(C::NT, 1) k_inner(InnerArgs a) {
  using PR = ProjExplicit;
  extern __shared__ float4 dsm4[];
  __shared__ Scal sc;
  float* ws = a.ws ? a.ws + (size_t)blockIdx.x * a.ws_stride : nullptr;
  Ctx<C> cx = make_ctx<C>(reinterpret_cast<float*>(dsm4), ws, &sc, a.m, a.n, a.p);
  const DevParams& P = a.P;
  const int m = a.m, n = a.n, p = a.p, ld = cx.ld, pl = cx.pl;
  const float lam = P.lambda > 0.f ? P.lambda : rsqrtf((float)max(m, n));
  const float tol = P.jacobi_tol > 0.f ? P.jacobi_tol : default_jacobi_tol(m);
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    load_plane<C>(cx.D, a.D + (size_t)b * m * n, m, n, ld);
    for (int q = 0; q < p; ++q) load_plane<C>(cx.G + (size_t)q * pl, a.J + ((size_t)b * p + q) * m * n, m, n, ld);
    __syncthreads();
    double qr[24];
    for (int e = 0; e < 24; ++e) qr[e] = 0.0;
    if (a.Q)
      for (int r = 0; r < a.l; ++r)
        for (int q = 0; q < p; ++q) qr[r * 8 + q] = a.Q[((size_t)b * a.l + r) * p + q];
    const int st = orthonormalise_explicit<C>(cx, qr, a.Q ? a.l : 0);
    tilt_report rr;
    memset(&rr, 0, sizeof(rr));
    rr.status = st;
    if (st == TILT_PATCH_CONVERGED) {
      for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
        cx.A[idx] = cx.D[idx];
        cx.E[idx] = 0.f;
        cx.Y[idx] = 0.f;
      }
      set_identity<C>(cx.V, cx.lds, n);
      __syncthreads();
      const float denom0 = proj_norm<C, PR>(cx, cx.D);
      const float denom = denom0 > 0.f ? denom0 : 1.f;
      int aux = 0;
      const float s1 = sigma1_of_plane<C>(cx, cx.D, tol, P.jacobi_max_sweeps, P.svd_warm != 0, &aux);
      const float mu0 = s1 > 0.f ? P.mu0_scale / s1 : P.mu0_scale;
      InnerOut io;
      float s_adm[8];
      if (P.inner_solver == 1) {
        io = adm_inner<C, PR>(cx, P, lam, mu0, tol, s_adm);
      } else {
        write_m0<C, PR>(cx, mu0);
        io = ladmap_inner<C, PR>(cx, P, lam, mu0, P.mu_max_ratio * mu0, denom, tol,
                                 P.rho_replay ? P.rho_replay + (size_t)b * P.max_inner : nullptr,
                                 P.trace ? P.trace + (size_t)4 * b * P.max_inner : nullptr);
      }
      const float nuc = cx.sc->svt_nuc;
      rr.rank = cx.sc->svt_relrank;
      rr.rank_band = cx.sc->svt_band;
      rr.svt_rank = cx.sc->svt_rank;
      const float l1 = plane_l1<C>(cx, cx.E);
      rr.status = io.converged ? TILT_PATCH_CONVERGED : TILT_PATCH_MAX_OUTER;
      rr.outer_iters = 1;
      rr.inner_iters = io.iters;
      rr.jacobi_sweeps = io.sweeps;
      rr.aux_sweeps = aux;
      rr.sweep_cap_hits = io.caps;
      rr.objective = nuc + lam * l1;
      rr.crit1 = io.crit1;
      rr.crit2 = io.crit2;
      rr.mu_last = io.mu;
      rr.jacobi_rotations = io.rotations;
      rr.patch_norm = denom0;
    }
    __syncthreads();
    const bool z = st != TILT_PATCH_CONVERGED;
    store_plane<C>(a.A + (size_t)b * m * n, cx.A, m, n, ld, z);
    store_plane<C>(a.E + (size_t)b * m * n, cx.E, m, n, ld, z);
    if (a.Y) store_plane<C>(a.Y + (size_t)b * m * n, cx.Y, m, n, ld, z);
    if (a.rep && threadIdx.x == 0) a.rep[b] = rr;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Standalone SVT (step parity of the K3 core)
// ---------------------------------------------------------------------------------------------
struct SvtArgs {
  const float* M;
  int B, m, n;
  const float* eps;
  float* V_io;
  float* A;
  float* sigma;
  int* sweeps;
  float tol;
  int max_sweeps;
  float* ws;
  size_t ws_stride;
};

template <class C>
__global__ void __launch_bounds__(C::NT, 1) k_svt(SvtArgs a) {
  extern __shared__ float4 dsm4[];
  __shared__ Scal sc;
  float* ws = a.ws ? a.ws + (size_t)blockIdx.x * a.ws_stride : nullptr;
  Ctx<C> cx = make_ctx<C>(reinterpret_cast<float*>(dsm4), ws, &sc, a.m, a.n, 0);
  const int m = a.m, n = a.n, mn = m * n, ld = cx.ld;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    load_plane<C>(cx.S, a.M + (size_t)b * mn, m, n, cx.lds);
    if (a.V_io) {
      load_plane<C>(cx.V, a.V_io + (size_t)b * n * n, n, n, cx.lds);
    } else {
      set_identity<C>(cx.V, cx.lds, n);
    }
    __syncthreads();
    float* Ab = a.A + (size_t)b * mn;
    SvtOut so = svt<C, true>(
        cx, cx.S, a.eps[b], a.tol, a.max_sweeps, true,
        [&](int i0, int j, float4 v) {
          const float vv[4] = {v.x, v.y, v.z, v.w};
          for (int r = 0; r < 4; ++r)
            if (i0 + r < m) Ab[(i0 + r) * n + j] = vv[r];
        },
        false);
    if (a.sigma)
      for (int j = threadIdx.x; j < n; j += C::NT) a.sigma[(size_t)b * n + j] = sqrtf(cx.ns[j].x);
    if (a.V_io) store_plane<C>(a.V_io + (size_t)b * n * n, cx.V, n, n, cx.lds, false);
    if (a.sweeps && threadIdx.x == 0) a.sweeps[b] = so.sweeps;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// Standalone projector (K2 parity): W^TW v and G^{-1} J^T v (explicit K from a given J)
// ---------------------------------------------------------------------------------------------
struct ProjArgs {
  const float* J;
  const float* Q;
  int l;
  const float* v;
  int B, m, n, p;
  float* Pv;
  float* dtau;
  int* status;
  float* ws;
  size_t ws_stride;
};

template <class C>
__global__ void __launch_bounds__(C::NT, 1) k_project(ProjArgs a) {
  using PR = ProjExplicit;
  extern __shared__ float4 dsm4[];
  __shared__ Scal sc;
  float* ws = a.ws ? a.ws + (size_t)blockIdx.x * a.ws_stride : nullptr;
  Ctx<C> cx = make_ctx<C>(reinterpret_cast<float*>(dsm4), ws, &sc, a.m, a.n, a.p);
  const int m = a.m, n = a.n, p = a.p, mn = m * n, ld = cx.ld, pl = cx.pl;
  for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
    for (int q = 0; q < p; ++q) load_plane<C>(cx.G + (size_t)q * pl, a.J + ((size_t)b * p + q) * mn, m, n, ld);
    load_plane<C>(cx.A, a.v + (size_t)b * mn, m, n, ld);
    __syncthreads();
    double qr[24];
    for (int e = 0; e < 24; ++e) qr[e] = 0.0;
    if (a.Q)
      for (int r = 0; r < a.l; ++r)
        for (int q = 0; q < p; ++q) qr[r * 8 + q] = a.Q[((size_t)b * a.l + r) * p + q];
    const int st = orthonormalise_explicit<C>(cx, qr, a.Q ? a.l : 0);
    if (st == TILT_PATCH_CONVERGED) {
      float s[8], z[9];
      PR::reduce(cx, [&](int idx) { return cx.A[idx]; }, s);
      PR::coeffs(cx, s, z);
      for (int idx = threadIdx.x; idx < pl; idx += C::NT) cx.E[idx] = cx.A[idx] - PR::apply(cx, idx, 0, 0, z);
      if (a.dtau && threadIdx.x == 0) {
        const double* Li = cx.sc->Linv;
        for (int q = 0; q < p; ++q) {
          double dq = 0.0;
          for (int r = q; r < p; ++r) dq += Li[r * 8 + q] * (double)s[r];
          a.dtau[(size_t)b * p + q] = (float)dq;
        }
      }
      __syncthreads();
    }
    store_plane<C>(a.Pv + (size_t)b * mn, cx.E, m, n, ld, st != TILT_PATCH_CONVERGED);
    if (a.status && threadIdx.x == 0) a.status[b] = st;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// K1 standalone: Alg. 1 Step 1 over all patches (HBM-bound). One CTA per patch; the per-pixel
// arithmetic is the solve kernels' (warp_tap + warp_interp = warp_pixel_f).
//   pass 1: per pixel (fp64 coordinates, 4 bilinear taps) -> d, gx, gy, gz stored fp32 in shared
//           memory, fp64 sums of ||d||^2 and J_raw^T d; the tap loads of K1_ILP pixels are issued
//           before their math;
//   pass 2: D_hat = d/||d|| and J = (J_raw - D_hat c^T)/||d|| (quotient rule) from shared memory,
//           written as coalesced row-major planes.
// Traffic per patch: the window's 4-tap footprint (~(m+1)(n+1) pixels) read, (1+p) m n floats
// written.
// ---------------------------------------------------------------------------------------------
#ifndef TILT_NO_FREE_KERNELS  // defined only in the translation unit that owns them (tilt.cu)
struct WarpArgs {
  const float* images;
  int n_images, H, W;
  const int* patch_image;
  const int* boxes;
  const float* tau;
  int B, m, n, p, kind;
  float* Dhat;
  float* J;
  float* norm;
  int* status;
};

#ifndef TILT_K1_NT  // experiment hooks (tools/build_variant.sh); the defaults are the product
#define TILT_K1_NT 128
#define TILT_K1_ILP 5
#define TILT_K1_MINB 4
#endif
constexpr int K1_NT = TILT_K1_NT;
constexpr int K1_ILP = TILT_K1_ILP;

// One CTA per patch, two passes over its pixels:
//   1. geometry (fp64, warp_tap), the 4 taps, the fp32 interpolant (warp_interp) -> shared memory
//      (d, gx, gy, gz); fp32 per-thread partials of ||D o tau||^2 and D^T J_raw, combined in fp64;
//   2. D_hat = D / ||D|| and the normalised Jacobian J = J_raw / ||D|| - D_hat c' (c' = D_hat^T
//      J_raw / ||D||), written four consecutive pixels per thread as 16-byte stores (one for D_hat,
//      p for J) when m n % 4 == 0.
// The patch geometry is built once per CTA (thread 0) and broadcast through shared memory.
// Measured variants (tools/build_variant.sh): pass 1 is bound by the latency of the
// tap gathers, so what counts is gathers in flight per SM. 128 threads x ILP 5 (~20 pixels per
// thread in 4 waves of 20 loads) at 128 registers and 4 CTAs/SM (164 KB of shared memory) is the
// fastest: 0.646 of HBM at 65 536 patches, vs 0.539 for 256 threads x ILP 2 at 3 CTAs/SM; 256 x
// ILP 3-5 at 2 CTAs/SM, 512 x ILP 5 at 1 CTA/SM, 128 x ILP 3-8 at 3-5 CTAs/SM, the window
// footprint staged in shared memory by cp.async, a persistent grid and a two-kernel split
// (reductions, then a streaming output pass that redoes the warp) were each slower.
__global__ void __launch_bounds__(K1_NT, TILT_K1_MINB) k_warp(WarpArgs a) {
  extern __shared__ float4 k1s[];  // per pixel (d, gx, gy, gz)
  __shared__ double red[K1_NT / 32][9];
  __shared__ double tot[9];
  __shared__ WarpGeom sg;
  const int b = blockIdx.x;
  const int m = a.m, n = a.n, p = a.p, mn = m * n;
  if (threadIdx.x == 0) {
    const int bx[4] = {a.boxes[4 * b], a.boxes[4 * b + 1], a.boxes[4 * b + 2], a.boxes[4 * b + 3]};
    double tau[8] = {1, 0, 0, 1, 0, 0, 0, 0};
    for (int q = 0; q < p && q < 8; ++q) tau[q] = a.tau[b * p + q];
    sg = make_geom(bx, tau, a.kind);
  }
  __syncthreads();
  const WarpGeom g = sg;
  const float* img = a.images + (size_t)a.patch_image[b] * a.H * a.W;
  const float inv_sf = (float)g.inv_s, cif = 0.5f * (m - 1), cjf = 0.5f * (n - 1);
  float facc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  bool esc = false;
  PixIter it(threadIdx.x, K1_NT, n);  // row-major (j fastest): it.i is the column j, it.j the row i
  for (int o0 = threadIdx.x; o0 < mn; o0 += K1_NT * K1_ILP) {
    WarpTap t[K1_ILP];
    float v[K1_ILP][4];
    int pi[K1_ILP], pj[K1_ILP];
#pragma unroll
    for (int u = 0; u < K1_ILP; ++u) {  // geometry and all tap loads first
      const int o = o0 + u * K1_NT;
      pi[u] = it.j;
      pj[u] = it.i;
      it.next(K1_NT);
      t[u] = warp_tap(g, a.H, a.W, o < mn ? pi[u] : 0, o < mn ? pj[u] : 0);
      const bool live = o < mn && t[u].ok;
      esc |= (o < mn) && !t[u].ok;
      const float* r0 = img + t[u].off;
      v[u][0] = live ? __ldg(r0) : 0.f;
      v[u][1] = live ? __ldg(r0 + 1) : 0.f;
      v[u][2] = live ? __ldg(r0 + a.W) : 0.f;
      v[u][3] = live ? __ldg(r0 + a.W + 1) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < K1_ILP; ++u) {
      const int o = o0 + u * K1_NT;
      if (o >= mn) break;
      float d, gx, gy, gz;  // the solve kernels' per-pixel routine (warp_pixel_f)
      warp_interp(t[u], v[u][0], v[u][1], v[u][2], v[u][3], d, gx, gy, gz);
      k1s[o] = make_float4(d, gx, gy, gz);
      // per-thread partial sums in fp32 (~10 pixels each), combined across threads in fp64
      const float uu = ((float)pj[u] - cjf) * inv_sf, vv = ((float)pi[u] - cif) * inv_sf;
      const float gxd = gx * d, gyd = gy * d, gzd = gz * d;
      facc[0] = fmaf(gxd, uu, facc[0]);
      facc[1] = fmaf(gxd, vv, facc[1]);
      facc[2] = fmaf(gyd, uu, facc[2]);
      facc[3] = fmaf(gyd, vv, facc[3]);
      facc[4] += gxd;
      facc[5] += gyd;
      facc[6] = fmaf(gzd, uu, facc[6]);
      facc[7] = fmaf(gzd, vv, facc[7]);
      facc[8] = fmaf(d, d, facc[8]);
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    double x = facc[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
    if (lane == 0) red[w][k] = x;
  }
  esc = __syncthreads_or(esc);
  if (threadIdx.x < 9) {
    double s = 0.0;
    for (int ww = 0; ww < K1_NT / 32; ++ww) s += red[ww][threadIdx.x];
    tot[threadIdx.x] = s;
  }
  __syncthreads();
  const double nd = sqrt(tot[8]);
  int st = TILT_PATCH_CONVERGED;
  if (esc) st = TILT_PATCH_WINDOW_ESCAPE;
  else if (!(nd > 0.0)) st = TILT_PATCH_ZERO_PATCH;
  if (threadIdx.x == 0) {
    if (a.norm) a.norm[b] = (float)nd;
    if (a.status) a.status[b] = st;
  }
  const double indd = st == TILT_PATCH_CONVERGED ? 1.0 / nd : 0.0;
  const float ind = (float)indd;
  float c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = (float)(tot[q] * indd) * ind;  // (D_hat^T J_raw) / ||D||
  float* Dh = a.Dhat + (size_t)b * mn;
  float* Jb = a.J ? a.J + (size_t)b * p * mn : nullptr;
  if ((mn & 3) == 0) {
    for (int o = 4 * threadIdx.x; o < mn; o += 4 * K1_NT) {
      float4 px[4];
      float u[4], vv[4], dh[4];
      int i = o / n, j = o - i * n;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        px[e] = k1s[o + e];
        dh[e] = px[e].x * ind;
        u[e] = ((float)j - cjf) * inv_sf;
        vv[e] = ((float)i - cif) * inv_sf;
        px[e].y *= ind;
        px[e].z *= ind;
        px[e].w *= ind;
        if (++j == n) {
          j = 0;
          ++i;
        }
      }
      *reinterpret_cast<float4*>(Dh + o) = make_float4(dh[0], dh[1], dh[2], dh[3]);
      if (Jb) {
        float* jo = Jb + o;
        // plane q: J_raw_q / ||D|| - dh c'_q, J_raw = (gx u, gx v, gy u, gy v, gx, gy, gz u, gz v)
#define TILT_K1_PLANE(q, EXPR)                                                                        \
  if (q < p) {                                                                                        \
    float r[4];                                                                                       \
    _Pragma("unroll") for (int e = 0; e < 4; ++e) r[e] = fmaf(-dh[e], c[q], EXPR);                   \
    *reinterpret_cast<float4*>(jo + (size_t)(q) * mn) = make_float4(r[0], r[1], r[2], r[3]);       \
  }
        TILT_K1_PLANE(0, px[e].y * u[e])
        TILT_K1_PLANE(1, px[e].y * vv[e])
        TILT_K1_PLANE(2, px[e].z * u[e])
        TILT_K1_PLANE(3, px[e].z * vv[e])
        TILT_K1_PLANE(4, px[e].y)
        TILT_K1_PLANE(5, px[e].z)
        TILT_K1_PLANE(6, px[e].w * u[e])
        TILT_K1_PLANE(7, px[e].w * vv[e])
#undef TILT_K1_PLANE
      }
    }
  } else {
    for (PixIter it2(threadIdx.x, K1_NT, n); it2.idx < mn; it2.next(K1_NT)) {
      const int o = it2.idx, i = it2.j, j = it2.i;
      const float4 px = k1s[o];
      const float dh = px.x * ind;
      Dh[o] = dh;
      if (Jb) {
        const float u = ((float)j - cjf) * inv_sf, vv = ((float)i - cif) * inv_sf;
        const float gx = px.y * ind, gy = px.z * ind, gz = px.w * ind;
        const float jr[8] = {gx * u, gx * vv, gy * u, gy * vv, gx, gy, gz * u, gz * vv};
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < p) Jb[(size_t)q * mn + o] = fmaf(-dh, c[q], jr[q]);
      }
    }
  }
}

// 2x2 box downsample (pyramid, reading Z18) of n_images [H][W] -> [H/2][W/2]
__global__ void k_downsample(const float* __restrict__ in, float* __restrict__ out, int n_images, int H, int W) {
  const int h2 = H / 2, w2 = W / 2;
  const size_t total = (size_t)n_images * h2 * w2;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    const size_t im = e / ((size_t)h2 * w2);
    const int r = (int)(e - im * h2 * w2);
    const int y = r / w2, x = r - y * w2;
    const float* p = in + im * H * W + (size_t)(2 * y) * W + 2 * x;
    out[e] = 0.25f * (p[0] + p[1] + p[W] + p[W + 1]);
  }
}

__global__ void k_half_boxes(const int* __restrict__ in, int* __restrict__ out, int B) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 4 * B; e += gridDim.x * blockDim.x) out[e] = in[e] / 2;
}

#endif  // TILT_NO_FREE_KERNELS

}  // namespace tilt

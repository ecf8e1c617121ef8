// tilt_device.cuh — sm_100a device building blocks of the batched TILT hot path.
//
// Paper: Ren & Lin, arXiv 1205.5351 (/root/reference/PAPER.md, cited P:<line>). Readings R*/Z*/E*
// are listed in DESIGN.md. tilt_kernels.cuh assembles these into the kernels.
//
// Data layout inside a CTA (one patch at a time). Every per-patch matrix
// is column-major with one leading dimension LD = round_up(max(m, n), 4); rows >= m (>= n for V)
// are kept at zero, so elementwise passes may run over the padded index space:
//   planes   D_hat, A, E, Y~, then either the Jacobian factors GX, GY[, GZ] (implicit projector,
//            TILT path) or K = J L^{-T} (p planes, explicit projector, generic-J entries)
//   SVD      B = M V, V, S (M, or a Newton-Schulz temporary)
//   vectors  ns[MAXD] = (||x_j||^2, scale_j) per Jacobi column, hv[MAXD]
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/tilt.h"

namespace tilt {

constexpr unsigned FULL = 0xffffffffu;

// --------------------------------------------------------------------------------------------
// Configuration
// --------------------------------------------------------------------------------------------

template <int LANES_, int RPL_, int NWARPS_, bool PLANES_SMEM_, bool SVD_SMEM_, int MINB_, bool B_SMEM_ = SVD_SMEM_>
struct Cfg {
  static constexpr int LANES = LANES_;   // lanes per Jacobi pair unit (16: half warp, 32: warp)
  static constexpr int RPL = RPL_;       // rows per lane (a column holds up to MAXD rows)
  static constexpr int NWARPS = NWARPS_;
  static constexpr int NT = NWARPS_ * 32;
  static constexpr int MAXD = LANES_ * RPL_;
  static constexpr int UNITS = NT / LANES_;
  static constexpr bool PLANES_SMEM = PLANES_SMEM_;
  static constexpr bool SVD_SMEM = SVD_SMEM_;
  static constexpr bool B_SMEM = B_SMEM_;  // B = M V in shared memory even when V, S are not
  static constexpr int MINB = MINB_;
};

// S64: planes (D, A, E, Y, GX, GY, GZ; 73 KB at 50x50) live in the per-CTA global workspace slot
// (L2-resident, touched only by the elementwise passes); B, V, S (31 KB) stay in shared memory, so
// 4 independent patches share an SM and hide each other's per-round barrier and shuffle latency.
using CfgS32 = Cfg<8, 4, 8, true, true, 4>;
#ifndef TILT_S64_L  // experiment hooks (tools/build_variant.sh); the defaults are the product
#define TILT_S64_L 8
#define TILT_S64_RPL 8
#define TILT_S64_NW 8
#define TILT_S64_MINB 4
#endif
using CfgS64 = Cfg<TILT_S64_L, TILT_S64_RPL, TILT_S64_NW, false, true, TILT_S64_MINB>;
// S56 (windows up to 56: the 50 x 50 of configs 2 and 5): S64's layout with 7 warps, 28 pair units
// >= n/2. An eighth warp would own no Jacobi pair at n <= 56 yet run every round's loop and barrier;
// without it a CTA issues fewer instructions per round and gets 72 registers at 4 CTAs/SM:
// +5% LADMAP iterations/s (`profiles/r02/jacobi_layouts/r2s3_seven_warps.log`).
#ifndef TILT_S56_NW  // experiment hooks (tools/build_variant.sh); the defaults are the product
#define TILT_S56_L 8
#define TILT_S56_RPL 8
#define TILT_S56_NW 7
#define TILT_S56_MINB 4
#endif
using CfgS56 = Cfg<TILT_S56_L, TILT_S56_RPL, TILT_S56_NW, false, true, TILT_S56_MINB>;
// S100 (windows 65..100: the 100 x 100 fine level of config 3): S128's layout with 25 warps, 50 pair
// units of 16 lanes >= n/2 (S128's 32 warps leave 7 warps without a pair at n <= 100); 80 registers.
using CfgS100 = Cfg<16, 8, 25, false, true, 1>;
using CfgS128 = Cfg<16, 8, 32, false, true, 1>;
// S256: B (256 x n floats, 205 KB at n = 200) in shared memory; V and S in the L2-resident slot
using CfgS256 = Cfg<32, 8, 32, false, false, 1, true>;
// S256 with n > 216 (B does not fit in shared memory): everything in the slot
using CfgS256G = Cfg<32, 8, 32, false, false, 1, false>;

struct DevParams {
  float lambda, mu0_scale, mu_max_ratio, rho0, eps1, eps2, obj_tol, tau_tol;
  int max_inner, max_outer, constraint_mode, vws, svd_warm;
  float jacobi_tol;
  int jacobi_max_sweeps;
  int fixed_inner, fixed_outer;
  int ns_period;
  int inner_solver;      // 0 LADMAP (the paper's), 1 ADM baseline
  float adm_rho, adm_tol;
  int svd_mode;          // 0 warm Jacobi every iteration, 1 LADMAP+SVDWS (Alg. 2, multi-CTA path)
  float svd_ws_gate;     // eps_svd = svd_ws_gate ||D||_F
  const uint8_t* rho_replay;
  float* trace;
};

// Scalars and reduction scratch of one CTA (static shared memory).
struct Scal {
  double Linv[64];   // L^{-1}, L L^T = G = J^TJ + Q^TQ (row-major p x p, lower)
  double dred[16 * 12];
  double dout[12];
  double sd[8];      // K^T v of the last implicit-projector reduce (fp64)
  float zc[9];       // its apply coefficients L'^T s, c'^T s
  double Lp[64];     // L^{-1} / ||d|| (implicit projector; fp64 so that L'(J_raw^T v) - c'(D_hat^T v)
  double cp[8];      // does not cancel in fp32);  L^{-1} c / ||d||, c = D_hat^T J_raw
  float fred[32 * 10];
  float fout[12];
  float nd;          // ||D o tau||_F
  float svt_nuc;     // sum_j max(sigma_j - eps, 0) of the last SVT (= ||A||_*)
  float svt_sig1;    // max_j sigma_j(M)
  int svt_rank;      // #{sigma_j > eps}
  int svt_relrank;   // Z19 relative rank of A
  int svt_band;
  int flag;
  int patch;
  int rot_acc;       // Jacobi rotations of the current SVT
  int nk;            // columns with h_j > 0 in the last SVT ...
  short kidx[256];   // ... and their indices, ascending (the terms of A = sum_j h_j b_j v_j^T)
};

// --------------------------------------------------------------------------------------------
// Block-level reductions (deterministic order; every thread receives the same bits)
// --------------------------------------------------------------------------------------------

template <class C, int KV>
__device__ __forceinline__ void block_sum_f(float (&v)[KV], Scal* sc) {
  static_assert(KV <= 10, "fred holds 10 values per warp");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    float x = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
    v[k] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < KV; ++k) sc->fred[w * 10 + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < KV) {
    float s = 0.f;
    for (int ww = 0; ww < C::NWARPS; ++ww) s += sc->fred[ww * 10 + threadIdx.x];
    sc->fout[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KV; ++k) v[k] = sc->fout[k];
}

// fp32 warp sums, combined across warps in fp64 (the implicit projector's K^T v: partials of a
// residual cancel across the CTA; a warp's 32 x ~10 pixels are summed by an fp32 tree)
template <class C, int KV>
__device__ __forceinline__ void block_sum_fd(const float (&v)[KV], double (&out)[KV], Scal* sc) {
  static_assert(KV <= 10, "fred holds 10 values per warp");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    float x = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
    if (lane == 0) sc->fred[w * 10 + k] = x;
  }
  __syncthreads();
  if (threadIdx.x < KV) {
    double s = 0.0;
    for (int ww = 0; ww < C::NWARPS; ++ww) s += (double)sc->fred[ww * 10 + threadIdx.x];
    sc->dout[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KV; ++k) out[k] = sc->dout[k];
}

// fp64 block sum (used once per outer iteration): warp shuffles, then warps 0..KV-1 finish.
template <class C, int KV>
__device__ __forceinline__ void block_sum_d(double (&v)[KV], Scal* sc) {
  static_assert(KV <= 12, "dout holds 12 values");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
    v[k] = x;
  }
  // two stages so that dred (16 x 12) suffices for up to 32 warps
  for (int half = 0; half < (C::NWARPS + 15) / 16; ++half) {
    if (lane == 0 && (w >> 4) == half) {
#pragma unroll
      for (int k = 0; k < KV; ++k) sc->dred[(w & 15) * 12 + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x < KV) {
      double s = half ? sc->dout[threadIdx.x] : 0.0;
      const int nw = min(16, C::NWARPS - 16 * half);
      for (int ww = 0; ww < nw; ++ww) s += sc->dred[ww * 12 + threadIdx.x];
      sc->dout[threadIdx.x] = s;
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < KV; ++k) v[k] = sc->dout[k];
}

// --------------------------------------------------------------------------------------------
// Per-CTA context
// --------------------------------------------------------------------------------------------

template <class C>
struct Ctx {
  float *D, *A, *E, *Y;  // planes (col-major, ld)
  float* T;              // J dtau (ADM baseline)
  float *G;              // implicit projector: GX, GY, GZ planes; explicit: K (p planes)
  float *B, *V, *S;      // SVD buffers (col-major, ld)
  float4* ns;            // (norm^2, scale, 1/scale, -) per Jacobi column
  float* hv;
  Scal* sc;
  int m, n, p, ld, pl;   // planes: leading dimension ld, pl = ld * n (plane size)
  int lds;               // SVD buffers: leading dimension MAXD (every Jacobi chunk exists)
  float ci, cj, inv_s;   // normalised frame: u = (j - cj) inv_s, v = (i - ci) inv_s
};

__host__ __device__ inline int round4(int x) { return (x + 3) & ~3; }

// Leading dimension of every per-patch matrix: a multiple of 4 (float4 tiles; Jacobi lanes mask
// the float4 chunks beyond ld, so a lane never touches the next column).
template <class C>
__host__ __device__ inline int ld_of(int m, int n) {
  static_assert(C::RPL % 4 == 0, "Jacobi lanes move float4 chunks");
  return round4(m > n ? m : n);
}

// Pixel iterator over the column-major padded index idx = j*ld + i with stride NT.
struct PixIter {
  int idx, i, j, di, dj, ld;
  __device__ __forceinline__ PixIter(int start, int stride, int ld_) : idx(start), ld(ld_) {
    j = start / ld_;
    i = start - j * ld_;
    dj = stride / ld_;
    di = stride - dj * ld_;
  }
  __device__ __forceinline__ void next(int stride) {
    idx += stride;
    i += di;
    j += dj;
    if (i >= ld) {
      i -= ld;
      ++j;
    }
  }
};

// --------------------------------------------------------------------------------------------
// Small dense kernels on the padded column-major buffers
// --------------------------------------------------------------------------------------------

// C = L * R (L: ld x inner, R: inner x cols; C must not alias L or R). Every row group of the
// padded column is written; rows >= rows_valid are written as 0. Thread tile: 4 rows x 2 columns,
// one float4 of L and two broadcast scalars of R per k, float4 stores.
template <class C>
__device__ __forceinline__ void gemm_nn(float* __restrict__ Cm, const float* __restrict__ Lm,
                                        const float* __restrict__ Rm, int ld, int rows_valid, int inner,
                                        int cols) {
  // C = L R (column-major, leading dimension ld): 4 x 4 register tiles, K in pairs (two 16-byte and
  // four 8-byte shared loads per 32 FMAs)
  const int rt = ld >> 2;
  const int ct = (cols + 3) >> 2;
  const int ntiles = rt * ct;
  for (int tile = threadIdx.x; tile < ntiles; tile += C::NT) {
    const int i0 = (tile % rt) * 4;
    const int j0 = (tile / rt) * 4;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
    const float* lp = Lm + i0;
    const float* rp[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) rp[c] = Rm + (j0 + c < cols ? j0 + c : j0) * ld;
    const int kend = i0 < rows_valid ? inner : 0;
    int k = 0;
    for (; k + 1 < kend; k += 2) {
      const float4 a0 = *reinterpret_cast<const float4*>(lp + k * ld);
      const float4 a1 = *reinterpret_cast<const float4*>(lp + (k + 1) * ld);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float2 b = *reinterpret_cast<const float2*>(rp[c] + k);
        acc[4 * c + 0] = fmaf(a0.x, b.x, fmaf(a1.x, b.y, acc[4 * c + 0]));
        acc[4 * c + 1] = fmaf(a0.y, b.x, fmaf(a1.y, b.y, acc[4 * c + 1]));
        acc[4 * c + 2] = fmaf(a0.z, b.x, fmaf(a1.z, b.y, acc[4 * c + 2]));
        acc[4 * c + 3] = fmaf(a0.w, b.x, fmaf(a1.w, b.y, acc[4 * c + 3]));
      }
    }
    if (k < kend) {
      const float4 a0 = *reinterpret_cast<const float4*>(lp + k * ld);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float b = rp[c][k];
        acc[4 * c + 0] = fmaf(a0.x, b, acc[4 * c + 0]);
        acc[4 * c + 1] = fmaf(a0.y, b, acc[4 * c + 1]);
        acc[4 * c + 2] = fmaf(a0.z, b, acc[4 * c + 2]);
        acc[4 * c + 3] = fmaf(a0.w, b, acc[4 * c + 3]);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (i0 + r >= rows_valid) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[4 * c + r] = 0.f;
      }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (j0 + c < cols)
        *reinterpret_cast<float4*>(Cm + (j0 + c) * ld + i0) =
            make_float4(acc[4 * c + 0], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
  }
  __syncthreads();
}

// out(i0, j, float4 of rows i0..i0+3) for C = B' V^T (B' = B diag(h) pre-scaled): i0 < m, j < n;
// 4 x 4 register tiles (two 16-byte shared loads per 16 FMAs; V's padding rows are zero)
// A = B V^T over the nk columns listed in kidx (the SVT's columns with h_j > 0; the others are
// exactly zero after col_scale and are skipped: the sum keeps the ascending order of the full one)
template <class C, class Out>
__device__ __forceinline__ void gemm_bvt(const float* Bm, const float* Vm, int ld, int m, int n, Out out,
                                         const short* kidx, int nk) {
  const int rt = (m + 3) >> 2;
  const int ct = (n + 3) >> 2;
  const int ntiles = rt * ct;
  for (int tile = threadIdx.x; tile < ntiles; tile += C::NT) {
    const int i0 = (tile % rt) * 4;
    const int j0 = (tile / rt) * 4;
    float acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.f;
#pragma unroll 2
    for (int t = 0; t < nk; ++t) {
      const int k = kidx[t];
      const float4 a = *reinterpret_cast<const float4*>(Bm + k * ld + i0);
      const float4 v = *reinterpret_cast<const float4*>(Vm + k * ld + j0);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[4 * c + 0] = fmaf(a.x, vv[c], acc[4 * c + 0]);
        acc[4 * c + 1] = fmaf(a.y, vv[c], acc[4 * c + 1]);
        acc[4 * c + 2] = fmaf(a.z, vv[c], acc[4 * c + 2]);
        acc[4 * c + 3] = fmaf(a.w, vv[c], acc[4 * c + 3]);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (j0 + c < n) out(i0, j0 + c, make_float4(acc[4 * c + 0], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]));
  }
}

template <class C>
__device__ __forceinline__ void set_identity(float* Vm, int ld, int n) {
  for (int e = threadIdx.x; e < ld * n; e += C::NT) {
    const int j = e / ld, i = e - j * ld;
    Vm[e] = (i == j) ? 1.f : 0.f;
  }
}

// Y = X^T for an n x n block (ld-padded, rows >= n of Y zero); conflict-light via 33-stride reads.
template <class C>
__device__ __forceinline__ void transpose_nn(float* __restrict__ Ym, const float* __restrict__ Xm, int ld, int n) {
  for (int e = threadIdx.x; e < ld * n; e += C::NT) {
    const int j = e / ld, i = e - j * ld;  // Y(i, j) = X(j, i)
    Ym[e] = (i < n) ? Xm[i * ld + j] : 0.f;
  }
}

#include "tilt_jacobi.cuh"

// sigma_j = sqrt(ns_j.x) stats after the final pass: nuclear norm of S_eps, ranks (Z19), sigma_1.
// Scale B for the SVT product A = B diag(h_j / ||v_j||^2) V^T
template <class C>
__device__ __forceinline__ void col_scale(Ctx<C>& cx) {
  const int n = cx.n, lds = cx.lds, rows = round4(cx.m);
  for (int e = threadIdx.x; e < n * (rows >> 2); e += C::NT) {
    const int j = e / (rows >> 2), i0 = (e - j * (rows >> 2)) * 4;
    const float f = cx.hv[j] * cx.ns[j].y;
    float4* bp = reinterpret_cast<float4*>(cx.B + j * lds + i0);
    float4 b = *bp;
    b.x *= f;
    b.y *= f;
    b.z *= f;
    b.w *= f;
    *bp = b;
  }
  if (threadIdx.x < 32) {  // the columns with h_j > 0, compacted in ascending order
    int base = 0;
    for (int jb = 0; jb < n; jb += 32) {
      const int j = jb + threadIdx.x;
      const bool on = j < n && cx.hv[j] > 0.f;
      const unsigned msk = __ballot_sync(FULL, on);
      if (on) cx.sc->kidx[base + __popc(msk & ((1u << threadIdx.x) - 1u))] = (short)j;
      base += __popc(msk);
    }
    if (threadIdx.x == 0) cx.sc->nk = base;
  }
  __syncthreads();
}

template <class C>
__device__ __forceinline__ void svt_stats(Ctx<C>& cx, float eps) {
  const int n = cx.n;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    float nuc = 0.f, smax = 0.f, amax = 0.f;
    int cnt = 0;
    for (int j = lane; j < n; j += 32) {
      const float sg = sqrtf(cx.ns[j].x);
      const float a = fmaxf(sg - eps, 0.f);
      nuc += a;
      smax = fmaxf(smax, sg);
      amax = fmaxf(amax, a);
      cnt += (sg > eps);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      nuc += __shfl_xor_sync(FULL, nuc, off);
      smax = fmaxf(smax, __shfl_xor_sync(FULL, smax, off));
      amax = fmaxf(amax, __shfl_xor_sync(FULL, amax, off));
      cnt += __shfl_xor_sync(FULL, cnt, off);
    }
    int rel = 0, band = 0;
    for (int j = lane; j < n; j += 32) {
      const float a = fmaxf(sqrtf(cx.ns[j].x) - eps, 0.f);
      if (amax > 0.f) {
        const float ratio = a / amax;
        rel += ratio > 1e-3f;
        band |= (ratio >= 3e-4f && ratio <= 3e-3f);
      }
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      rel += __shfl_xor_sync(FULL, rel, off);
      band |= __shfl_xor_sync(FULL, band, off);
    }
    if (lane == 0) {
      cx.sc->svt_nuc = nuc;
      cx.sc->svt_sig1 = smax;
      cx.sc->svt_rank = cnt;
      cx.sc->svt_relrank = rel;
      cx.sc->svt_band = band;
    }
  }
}

// Newton-Schulz re-orthonormalisation of V (reading Z14): V <- V (1.5 I - 0.5 V^T V).
// S <- V^T, B <- S V, B <- 1.5 I - 0.5 B, S <- V B, swap(S, V). B and S must be free.
template <class C>
__device__ __forceinline__ void ns_step(Ctx<C>& cx) {
  const int n = cx.n, ld = cx.lds;
  transpose_nn<C>(cx.S, cx.V, ld, n);
  __syncthreads();
  gemm_nn<C>(cx.B, cx.S, cx.V, ld, n, n, n);
  for (int e = threadIdx.x; e < ld * n; e += C::NT) {
    const int j = e / ld, i = e - j * ld;
    cx.B[e] = (i == j ? 1.5f : 0.f) - 0.5f * cx.B[e];
  }
  __syncthreads();
  gemm_nn<C>(cx.S, cx.V, cx.B, ld, n, n, n);
  float* t = cx.S;
  cx.S = cx.V;
  cx.V = t;
}

struct SvtOut {
  int sweeps;
  int rotations;
  bool capped;
};

// S_eps(X) for X (= M, or D_hat) in a padded buffer. Leaves V warm (orthonormalised by one
// Newton-Schulz step if ns_after) and calls out(i0, j, float4 rows i0..i0+3 of the result).
template <class C, bool DO_OUT, class Out>
__device__ SvtOut svt(Ctx<C>& cx, const float* X, float eps, float tol, int max_sweeps, bool warm, Out out,
                      bool ns_after) {
  if (!warm) {
    set_identity<C>(cx.V, cx.lds, cx.n);
    __syncthreads();
  }
  gemm_nn<C>(cx.B, X, cx.V, cx.lds, cx.m, cx.n, cx.n);  // B = X V (X in the lds layout)
  SvtOut r;
  r.rotations = 0;
  if constexpr (C::SVD_SMEM) {
    int capped = 0;
    if (threadIdx.x == 0) cx.sc->rot_acc = 0;  // published by the first barrier inside
    r.sweeps = jacobi_sweeps_smem<C>(cx.B, cx.V, cx.ns, cx.n, tol, max_sweeps, &capped, &cx.sc->rot_acc);
    r.capped = capped != 0;
    r.rotations = cx.sc->rot_acc;
  } else {
    r.sweeps = jacobi_sweeps<C>(cx, tol, max_sweeps, &r.capped);
  }
  col_pass<C, 2>(cx, eps);  // sigma_j, h_j, 1 / ||v_j||^2
  svt_stats<C>(cx, eps);
  if constexpr (DO_OUT) {
    col_scale<C>(cx);
    gemm_bvt<C>(cx.B, cx.V, cx.lds, cx.m, cx.n, out, cx.sc->kidx, cx.sc->nk);  // A = B diag(h) V^T
  }
  __syncthreads();
  if (ns_after) ns_step<C>(cx);
  return r;
}

// --------------------------------------------------------------------------------------------
// Warp + Jacobian (Alg. 1 Step 1; readings Z2, Z15, Z16)
// --------------------------------------------------------------------------------------------

struct WarpGeom {
  double s, inv_s, cx, cy, h11, h12, h13, h21, h22, h23, h31, h32;
  int m, n, p, kind;
  bool persp;  // homography with h31 or h32 nonzero (w != 1)
};

__device__ __forceinline__ WarpGeom make_geom(const int* box, const double* tau, int kind) {
  WarpGeom g;
  const int x0 = box[0], y0 = box[1];
  g.n = box[2];
  g.m = box[3];
  g.s = 0.5 * (double)max(g.m, g.n);
  g.inv_s = 1.0 / g.s;
  g.cx = x0 + 0.5 * (g.n - 1);
  g.cy = y0 + 0.5 * (g.m - 1);
  g.h11 = tau[0]; g.h12 = tau[1]; g.h21 = tau[2]; g.h22 = tau[3]; g.h13 = tau[4]; g.h23 = tau[5];
  g.h31 = kind == TILT_HOMOGRAPHY ? tau[6] : 0.0;
  g.h32 = kind == TILT_HOMOGRAPHY ? tau[7] : 0.0;
  g.kind = kind;
  g.p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  g.persp = g.h31 != 0.0 || g.h32 != 0.0;
  return g;
}

// Bilinear sample d and the Jacobian factors (gx, gy, gz) at window pixel (i, j):
// J_raw = (gx u, gx v, gy u, gy v, gx, gy, gz u, gz v) with gx = s I_X / w, gy = s I_Y / w,
// gz = -(gx x + gy y) (normalised frame). Returns false on window escape.
// The one Step-1 pixel routine of every kernel (the standalone K1 k_warp, the CTA-per-patch solve,
// the warp-per-patch and multi-CTA paths): the source coordinate in fp64 (an fp32 coordinate of a
// 100-pixel canvas would carry ~6e-6 px of rounding into the fractions), the 4 taps, the bilinear
// value and the exact interpolant gradient (reading Z2) in fp32 from the fp32 fractions.
// a + e - d of three fp32 values, exact up to the final rounding: the LADMAP residual
// A + E - D_hat cancels O(1e-2) entries down to O(1e-9), so summed in fp32 its rounding (~ulp(a + e)
// per entry, ~2e-7 in norm at 50 x 50) was the crit1 floor (Z7) and, through Y += mu R, put a floor
// of ~mu 1e-6 under crit2: fp32 inner loops that the fp64 oracle ends at mu ~ 2e5 ran to max_inner
// Knuth's TwoSum gives s + err = a + e exactly in fp32; s - d is then exact when s and d are within a
// factor 2 (Sterbenz), which is the cancelling case; otherwise its rounding is relative to a result
// that is not small. 8 fp32 operations instead of the fp64 sum's conversions.
__device__ __forceinline__ float res3(float a, float e, float d) {
  const float s = __fadd_rn(a, e);
  const float bb = __fsub_rn(s, a);
  const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(e, bb));
  return __fadd_rn(__fsub_rn(s, d), err);
}

struct WarpTap {
  int off;                    // yi * W + xi of the cell's top-left tap
  float fx, fy, sw, xn, yn;   // fractions, s / w, normalised source coordinate
  bool ok;                    // the 4-tap stencil lies inside the image
};

// fp64 source coordinate (X, Y) of window pixel (i, j) (Z15, Z16); iw = 1 / w
__device__ __forceinline__ void warp_xy(const WarpGeom& g, int i, int j, double& X, double& Y, double& iw) {
  const double du = j - 0.5 * (g.n - 1);
  const double dv = i - 0.5 * (g.m - 1);
  // 1 / w: fp32 reciprocal refined by one fp64 Newton step, relative error ~(2^-23)^2 (the fp64
  // division's multi-instruction sequence was ~5% of K1's instructions); w = 1 exactly when affine
  iw = 1.0;
  if (g.persp) {
    const double w = 1.0 + (g.h31 * du + g.h32 * dv) * g.inv_s;
    const double r = (double)__frcp_rn((float)w);
    iw = r * fma(-w, r, 2.0);
  }
  X = g.cx + (g.h11 * du + g.h12 * dv + g.s * g.h13) * iw;
  Y = g.cy + (g.h21 * du + g.h22 * dv + g.s * g.h23) * iw;
}

// fp64 geometry of window pixel (i, j): source coordinate, cell by floor, escape test (Z2)
__device__ __forceinline__ WarpTap warp_tap(const WarpGeom& g, int H, int W, int i, int j) {
  double X, Y, iw;
  warp_xy(g, i, j, X, Y, iw);
  const double X0 = floor(X), Y0 = floor(Y);
  WarpTap t;
  t.ok = X0 >= 0.0 && X0 + 1.0 <= W - 1 && Y0 >= 0.0 && Y0 + 1.0 <= H - 1;
  t.off = t.ok ? (int)Y0 * W + (int)X0 : 0;
  t.fx = (float)(X - X0);
  t.fy = (float)(Y - Y0);
  t.sw = (float)(g.s * iw);
  t.xn = (float)((X - g.cx) * g.inv_s);
  t.yn = (float)((Y - g.cy) * g.inv_s);
  return t;
}

// fp32 bilinear value and exact interpolant gradient from the 4 taps (Z2); J_raw factors
__device__ __forceinline__ void warp_interp(const WarpTap& t, float i00, float i01, float i10, float i11, float& d,
                                            float& gx, float& gy, float& gz) {
  const float top = fmaf(t.fx, i01 - i00, i00), bot = fmaf(t.fx, i11 - i10, i10);
  d = fmaf(t.fy, bot - top, top);
  const float dX = fmaf(t.fy, (i11 - i10) - (i01 - i00), i01 - i00);  // (1-fy)(I01-I00) + fy(I11-I10)
  const float dY = bot - top;                                          // (1-fx)(I10-I00) + fx(I11-I01)
  gx = t.sw * dX;
  gy = t.sw * dY;
  gz = -fmaf(gx, t.xn, gy * t.yn);
}

__device__ __forceinline__ bool warp_pixel_f(const WarpGeom& g, const float* __restrict__ img, int H, int W,
                                             int i, int j, float& d, float& gx, float& gy, float& gz) {
  const WarpTap t = warp_tap(g, H, W, i, j);
  if (!t.ok) {
    d = gx = gy = gz = 0.f;
    return false;
  }
  const float* r0 = img + t.off;
  warp_interp(t, __ldg(r0), __ldg(r0 + 1), __ldg(r0 + W), __ldg(r0 + W + 1), d, gx, gy, gz);
  return true;
}

__device__ __forceinline__ bool warp_pixel(const WarpGeom& g, const float* __restrict__ img, int H, int W,
                                           int i, int j, double& d, double& gx, double& gy, double& gz) {
  float df, gxf, gyf, gzf;
  const bool ok = warp_pixel_f(g, img, H, W, i, j, df, gxf, gyf, gzf);
  d = df;
  gx = gxf;
  gy = gyf;
  gz = gzf;
  return ok;
}

__device__ __forceinline__ void jraw_row(double gx, double gy, double gz, double u, double v, double (&jr)[8]) {
  jr[0] = gx * u; jr[1] = gx * v; jr[2] = gy * u; jr[3] = gy * v; jr[4] = gx; jr[5] = gy;
  jr[6] = gz * u; jr[7] = gz * v;
}

// Centre + area constraint rows (reading Z10), unit-norm rows, into q[3][8].
__device__ __forceinline__ void constraint_rows(const double* tau, int kind, int m, int n, double* q) {
  const int p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  const double h11 = tau[0], h12 = tau[1], h21 = tau[2], h22 = tau[3], h13 = tau[4], h23 = tau[5];
  const double h31 = kind == TILT_HOMOGRAPHY ? tau[6] : 0.0, h32 = kind == TILT_HOMOGRAPHY ? tau[7] : 0.0;
  const double big = (double)max(m, n);
  const double cu = n / big, cv = m / big;
  const double us[4] = {-cu, cu, cu, -cu}, vs[4] = {-cv, -cv, cv, cv};
  double X[4], Yv[4], gx[4][8], gy[4][8];
  for (int k = 0; k < 4; ++k) {
    const double u = us[k], v = vs[k];
    const double w = h31 * u + h32 * v + 1.0;
    X[k] = (h11 * u + h12 * v + h13) / w;
    Yv[k] = (h21 * u + h22 * v + h23) / w;
    for (int e = 0; e < 8; ++e) { gx[k][e] = 0.0; gy[k][e] = 0.0; }
    gx[k][0] = u / w; gx[k][1] = v / w; gx[k][4] = 1.0 / w;
    gy[k][2] = u / w; gy[k][3] = v / w; gy[k][5] = 1.0 / w;
    if (kind == TILT_HOMOGRAPHY) {
      gx[k][6] = -X[k] * u / w; gx[k][7] = -X[k] * v / w;
      gy[k][6] = -Yv[k] * u / w; gy[k][7] = -Yv[k] * v / w;
    }
  }
  double ga[8];
  for (int e = 0; e < 8; ++e) ga[e] = 0.0;
  for (int k = 0; k < 4; ++k) {
    const int k1 = (k + 1) & 3;
    for (int e = 0; e < p; ++e)
      ga[e] += 0.5 * (gx[k][e] * Yv[k1] + X[k] * gy[k1][e] - gx[k1][e] * Yv[k] - X[k1] * gy[k][e]);
  }
  double nrm = 0.0;
  for (int e = 0; e < p; ++e) nrm += ga[e] * ga[e];
  nrm = sqrt(nrm);
  for (int e = 0; e < 3 * 8; ++e) q[e] = 0.0;
  q[0 * 8 + 4] = 1.0;
  q[1 * 8 + 5] = 1.0;
  for (int e = 0; e < p; ++e) q[2 * 8 + e] = nrm > 0 ? ga[e] / nrm : 0.0;
}

// Cholesky of G (+ Q^T Q), L^{-1} (fp64, one thread). Returns false if G is not positive definite.
__device__ __forceinline__ bool chol_inverse(const double* G36, const double* qrows, int l, int p, double* Li) {
  double Gf[64], Lm[64];
  int e = 0;
  for (int a = 0; a < 8; ++a)
    for (int b = a; b < 8; ++b) {
      Gf[a * 8 + b] = G36[e];
      Gf[b * 8 + a] = G36[e];
      ++e;
    }
  for (int r = 0; r < l; ++r)
    for (int a = 0; a < p; ++a)
      for (int b = 0; b < p; ++b) Gf[a * 8 + b] += qrows[r * 8 + a] * qrows[r * 8 + b];
  for (int a = 0; a < 64; ++a) { Lm[a] = 0.0; Li[a] = 0.0; }
  double dmax = 0.0;
  for (int a = 0; a < p; ++a) dmax = fmax(dmax, Gf[a * 8 + a]);
  if (!(dmax > 0.0) || !isfinite(dmax)) return false;
  for (int a = 0; a < p; ++a) {
    double s = Gf[a * 8 + a];
    for (int k = 0; k < a; ++k) s -= Lm[a * 8 + k] * Lm[a * 8 + k];
    if (!(s > 1e-14 * dmax)) return false;
    const double la = sqrt(s);
    Lm[a * 8 + a] = la;
    for (int b = a + 1; b < p; ++b) {
      double t = Gf[b * 8 + a];
      for (int k = 0; k < a; ++k) t -= Lm[b * 8 + k] * Lm[a * 8 + k];
      Lm[b * 8 + a] = t / la;
    }
  }
  for (int a = 0; a < p; ++a) {  // L^{-1} column by column (forward substitution)
    Li[a * 8 + a] = 1.0 / Lm[a * 8 + a];
    for (int b = a + 1; b < p; ++b) {
      double s = 0.0;
      for (int k = a; k < b; ++k) s += Lm[b * 8 + k] * Li[k * 8 + a];
      Li[b * 8 + a] = -s / Lm[b * 8 + b];
    }
  }
  return true;
}

// --------------------------------------------------------------------------------------------
// Projectors W^T W v = v - K K^T v, K = J L^{-T} (Eq. Jperpv, Eq. WTW_property)
// --------------------------------------------------------------------------------------------
// Implicit (TILT path): J = (J_raw - D_hat c^T)/||d|| with J_raw rows built per pixel from the
// GX, GY, GZ planes and (u, v); K^T v = L' J_raw^T v - c' (D_hat^T v), L' = L^{-1}/||d||,
// c' = L^{-1}c/||d||; K y = J_raw (L'^T y) - D_hat (c'^T y). No mn x p matrix is stored.
struct ProjImplicit {
  template <class C, class VF>
  static __device__ __forceinline__ void reduce(Ctx<C>& cx, VF vf, float (&s)[8]) {
    const int ld = cx.ld, pl = cx.pl;
    const bool homog = cx.p == 8;
    const float* __restrict__ GX = cx.G;
    const float* __restrict__ GY = cx.G + pl;
    const float* __restrict__ GZ = cx.G + 2 * pl;
    const float* __restrict__ Dp = cx.D;
    float a[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) a[k] = 0.f;
    for (PixIter pi(threadIdx.x, C::NT, ld); pi.idx < pl; pi.next(C::NT)) {
      const int idx = pi.idx;
      const float val = vf(idx);
      const float u = ((float)pi.j - cx.cj) * cx.inv_s;
      const float v = ((float)pi.i - cx.ci) * cx.inv_s;
      const float ga = GX[idx] * val, gb = GY[idx] * val;
      a[0] = fmaf(ga, u, a[0]);
      a[1] = fmaf(ga, v, a[1]);
      a[2] = fmaf(gb, u, a[2]);
      a[3] = fmaf(gb, v, a[3]);
      a[4] += ga;
      a[5] += gb;
      if (homog) {
        const float gc = GZ[idx] * val;
        a[6] = fmaf(gc, u, a[6]);
        a[7] = fmaf(gc, v, a[7]);
      }
      a[8] = fmaf(Dp[idx], val, a[8]);
    }
    // the warps' partial sums are combined in fp64, and so are J_raw^T v and D_hat^T v, which
    // cancel in K^T v = L'(J_raw^T v) - c'(D_hat^T v): with fp32 coefficients and combination the
    // projected residual of the LADMAP iteration carried ~1e-6 relative errors that the dual step
    // integrates (tools/inner_drift.py: A 1e-4 off the fp64 iterate after 400 iterations, inner
    // loops running to max_inner); in fp64 the solve path tracks the oracle as the explicit entry does
    float a9[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) a9[k] = a[k];
    double r[9];
    block_sum_fd<C, 9>(a9, r, cx.sc);
    // s = L' r[0:p] - c' r[8]  (K^T v), then the apply coefficients z = L'^T s, w = c'^T s: formed
    // once (threads 0..8) in fp64 and published through shared memory
    const double* Lp = cx.sc->Lp;
    const double* cp = cx.sc->cp;
    if (threadIdx.x < 8) {
      const int q = threadIdx.x;
      double acc = -cp[q] * r[8];
      for (int b = 0; b <= q; ++b) acc = fma(Lp[q * 8 + b], r[b], acc);
      cx.sc->sd[q] = acc;
    }
    __syncthreads();
    if (threadIdx.x < 9) {
      const int t = threadIdx.x;
      double acc = 0.0;
      if (t < 8) {
        for (int q = t; q < 8; ++q) acc = fma(Lp[q * 8 + t], cx.sc->sd[q], acc);
      } else {
        for (int q = 0; q < 8; ++q) acc = fma(cp[q], cx.sc->sd[q], acc);
      }
      cx.sc->zc[t] = (float)acc;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = (float)cx.sc->sd[q];
  }
  // coefficients for apply (formed by reduce())
  template <class C>
  static __device__ __forceinline__ void coeffs(const Ctx<C>& cx, const float (&s)[8], float (&z)[9]) {
#pragma unroll
    for (int k = 0; k < 9; ++k) z[k] = cx.sc->zc[k];
  }
  // (K y)(pixel) with y the K^T v of reduce(); z from coeffs()
  template <class C>
  static __device__ __forceinline__ float apply(const Ctx<C>& cx, int idx, int i, int j, const float (&z)[9]) {
    const float u = ((float)j - cx.cj) * cx.inv_s;
    const float v = ((float)i - cx.ci) * cx.inv_s;
    float r = cx.G[idx] * fmaf(z[0], u, fmaf(z[1], v, z[4])) + cx.G[cx.pl + idx] * fmaf(z[2], u, fmaf(z[3], v, z[5]));
    if (cx.p == 8) r = fmaf(cx.G[2 * cx.pl + idx], fmaf(z[6], u, z[7] * v), r);
    return fmaf(-cx.D[idx], z[8], r);
  }
};

// Explicit (generic J entries): K planes stored.
struct ProjExplicit {
  template <class C, class VF>
  static __device__ __forceinline__ void reduce(Ctx<C>& cx, VF vf, float (&s)[8]) {
    const int pl = cx.pl, p = cx.p;
    const float* __restrict__ Kp = cx.G;
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.f;
    for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
      const float v = vf(idx);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < p) s[q] = fmaf(Kp[q * pl + idx], v, s[q]);
    }
    block_sum_f<C, 8>(s, cx.sc);
  }
  template <class C>
  static __device__ __forceinline__ void coeffs(const Ctx<C>&, const float (&s)[8], float (&z)[9]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) z[q] = s[q];
    z[8] = 0.f;
  }
  template <class C>
  static __device__ __forceinline__ float apply(const Ctx<C>& cx, int idx, int, int, const float (&z)[9]) {
    float r = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < cx.p) r = fmaf(cx.G[q * cx.pl + idx], z[q], r);
    return r;
  }
};

// --------------------------------------------------------------------------------------------
// Orthonormalise (K2), implicit: from D (raw d) and GX, GY, GZ planes build ||d||, c = D_hat^T
// J_raw, the Gram of J = (J_raw - D_hat c^T)/||d|| plus Q^T Q, its Cholesky L, and L', c' for
// ProjImplicit; D is normalised in place (Alg. 1 Step 1). fp64 throughout.
// --------------------------------------------------------------------------------------------
template <class C, int CH, class RowF>
__device__ __forceinline__ void gram_chunk(Ctx<C>& cx, RowF rowf, double* Gout) {
  double acc[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) acc[e] = 0.0;
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < cx.pl; pi.next(C::NT)) {
    double jn[8];
    rowf(pi.idx, pi.i, pi.j, jn);
    int e = 0;
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = a; b < 8; ++b) {
        if (e >= 12 * CH && e < 12 * CH + 12) acc[e - 12 * CH] = fma(jn[a], jn[b], acc[e - 12 * CH]);
        ++e;
      }
  }
  block_sum_d<C, 12>(acc, cx.sc);
#pragma unroll
  for (int e = 0; e < 12; ++e) Gout[12 * CH + e] = acc[e];
}

template <class C>
__device__ int orthonormalise_implicit(Ctx<C>& cx, const double* qrows, int l) {
  Scal* sc = cx.sc;
  const int p = cx.p, pl = cx.pl;
  float* __restrict__ Dp = cx.D;
  const float* GX = cx.G;
  const float* GY = cx.G + pl;
  const float* GZ = cx.G + 2 * pl;
  const bool homog = p == 8;
  auto raw = [&](int idx, int i, int j, double (&jr)[8]) {
    const double u = ((double)j - cx.cj) * cx.inv_s, v = ((double)i - cx.ci) * cx.inv_s;
    jraw_row(GX[idx], GY[idx], homog ? (double)GZ[idx] : 0.0, u, v, jr);
  };
  double acc[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) acc[e] = 0.0;
  for (PixIter pi(threadIdx.x, C::NT, cx.ld); pi.idx < pl; pi.next(C::NT)) {
    const double d = Dp[pi.idx];
    double jr[8];
    raw(pi.idx, pi.i, pi.j, jr);
    acc[8] = fma(d, d, acc[8]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(jr[q], d, acc[q]);
  }
  block_sum_d<C, 9>(acc, sc);
  const double nd = sqrt(acc[8]);
  if (threadIdx.x == 0) sc->nd = (float)nd;
  if (!(nd > 0.0)) return TILT_PATCH_ZERO_PATCH;
  const double ind = 1.0 / nd;
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = acc[q] * ind;  // D_hat^T J_raw
  auto rown = [&](int idx, int i, int j, double (&jn)[8]) {
    double jr[8];
    raw(idx, i, j, jr);
    const double dh = Dp[idx] * ind;
#pragma unroll
    for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? (jr[q] - dh * c[q]) * ind : 0.0;
  };
  double G[36];
  gram_chunk<C, 0>(cx, rown, G);
  gram_chunk<C, 1>(cx, rown, G);
  gram_chunk<C, 2>(cx, rown, G);
  if (threadIdx.x == 0) {
    const bool ok = chol_inverse(G, qrows, l, p, sc->Linv);
    sc->flag = ok ? 1 : 0;
    if (ok) {
      for (int a = 0; a < 8; ++a) {
        double cpa = 0.0;
        for (int b = 0; b < 8; ++b) {
          sc->Lp[a * 8 + b] = sc->Linv[a * 8 + b] * ind;
          cpa += sc->Linv[a * 8 + b] * c[b];
        }
        sc->cp[a] = cpa * ind;
      }
    }
  }
  __syncthreads();
  if (!sc->flag) return TILT_PATCH_SINGULAR_GRAM;
  for (int idx = threadIdx.x; idx < pl; idx += C::NT) Dp[idx] = (float)(Dp[idx] * ind);
  __syncthreads();
  return TILT_PATCH_CONVERGED;
}

// Explicit: K planes hold J (generic, already "normalised" as given); D untouched.
template <class C>
__device__ int orthonormalise_explicit(Ctx<C>& cx, const double* qrows, int l) {
  Scal* sc = cx.sc;
  const int p = cx.p, pl = cx.pl;
  float* __restrict__ Kp = cx.G;
  auto rowj = [&](int idx, int, int, double (&jn)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? (double)Kp[q * pl + idx] : 0.0;
  };
  double G[36];
  gram_chunk<C, 0>(cx, rowj, G);
  gram_chunk<C, 1>(cx, rowj, G);
  gram_chunk<C, 2>(cx, rowj, G);
  if (threadIdx.x == 0) sc->flag = chol_inverse(G, qrows, l, p, sc->Linv) ? 1 : 0;
  __syncthreads();
  if (!sc->flag) return TILT_PATCH_SINGULAR_GRAM;
  const double* Li = sc->Linv;
  for (int idx = threadIdx.x; idx < pl; idx += C::NT) {
    double jn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? (double)Kp[q * pl + idx] : 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      if (a < p) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b <= a; ++b) s = fma(Li[a * 8 + b], jn[b], s);
        Kp[a * pl + idx] = (float)s;
      }
    }
  }
  __syncthreads();
  return TILT_PATCH_CONVERGED;
}

}  // namespace tilt

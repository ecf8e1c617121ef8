// tilt_device.cuh — sm_100a device code of the batched TILT hot path.
//
// Paper: Ren & Lin, arXiv 1205.5351 (/root/reference/PAPER.md, cited P:<line>). Readings R*/Z*/E*
// are listed in DESIGN.md. The kernels in tilt.cu instantiate these templates per size class.
//
// Data layout inside a CTA (one patch at a time):
//   planes   D_hat, A, E, Y~ and K (p planes): column-major m x n, pixel (i,j) at j*m + i
//   SVD      B = M V, V, S (M or the Newton-Schulz matrix): column-major, ld = MAXD (padded rows 0)
//   vectors  nrm[MAXD] (column norms^2), scl[MAXD] (fast-rotation column scales), hv[MAXD]
// Size classes put everything in shared memory (S32, S64), only the SVD buffers (S128) or nothing
// (S256, per-CTA global workspace slot, L2 resident).
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

template <int LANES_, int RPL_, int NWARPS_, bool PLANES_SMEM_, bool SVD_SMEM_, int MINB_>
struct Cfg {
  static constexpr int LANES = LANES_;   // lanes per Jacobi pair unit (16: half warp, 32: warp)
  static constexpr int RPL = RPL_;       // rows per lane (B and V columns padded to MAXD rows)
  static constexpr int NWARPS = NWARPS_;
  static constexpr int NT = NWARPS_ * 32;
  static constexpr int MAXD = LANES_ * RPL_;
  static constexpr int UNITS = NT / LANES_;
  static constexpr bool PLANES_SMEM = PLANES_SMEM_;
  static constexpr bool SVD_SMEM = SVD_SMEM_;
  static constexpr int MINB = MINB_;
};

using CfgS32 = Cfg<16, 2, 8, true, true, 2>;
using CfgS64 = Cfg<16, 4, 16, true, true, 1>;
using CfgS128 = Cfg<16, 8, 32, false, true, 1>;
using CfgS256 = Cfg<32, 8, 32, false, false, 1>;

struct DevParams {
  float lambda, mu0_scale, mu_max_ratio, rho0, eps1, eps2, obj_tol, tau_tol;
  int max_inner, max_outer, constraint_mode, vws, svd_warm;
  float jacobi_tol;
  int jacobi_max_sweeps;
  int fixed_inner, fixed_outer;
  const uint8_t* rho_replay;
  float* trace;
};

// Scalars and reduction scratch of one CTA (static shared memory).
struct Scal {
  double L[64];      // Cholesky factor of G = J^TJ + Q^TQ (row-major p x p, lower)
  double Linv[64];   // L^{-1}
  double c[8];       // D_hat^T J_raw (quotient rule, Alg. 1 Step 1)
  double tau[8];
  double dtau[8];
  double q[24];      // Q (3 x p)
  double dred[32 * 12];
  double dout[12];
  float fred[32 * 9];
  float fout[12];
  float nd;          // ||D o tau||_F
  float svt_nuc;     // sum_j max(sigma_j - eps, 0) of the last SVT (= ||A||_*)
  float svt_sig1;    // max_j sigma_j(M)
  int svt_rank;      // #{sigma_j > eps}
  int svt_relrank;   // Z19 relative rank of A
  int svt_band;
  int flag;
  int patch;
};

// --------------------------------------------------------------------------------------------
// Block-level reductions (deterministic order; every thread receives the same bits)
// --------------------------------------------------------------------------------------------

template <class C, int KV>
__device__ __forceinline__ void block_sum_f(float (&v)[KV], Scal* sc) {
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
    for (int k = 0; k < KV; ++k) sc->fred[w * KV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < KV) {
    float s = 0.f;
    for (int ww = 0; ww < C::NWARPS; ++ww) s += sc->fred[ww * KV + threadIdx.x];
    sc->fout[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KV; ++k) v[k] = sc->fout[k];
}

template <class C, int KV>
__device__ __forceinline__ void block_sum_d(double (&v)[KV], Scal* sc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    double x = v[k];
#pragma unroll
    for (int off = 16; off; off >>= 1) x += __shfl_xor_sync(FULL, x, off);
    v[k] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < KV; ++k) sc->dred[w * KV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < KV) {
    double s = 0.0;
    for (int ww = 0; ww < C::NWARPS; ++ww) s += sc->dred[ww * KV + threadIdx.x];
    sc->dout[threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KV; ++k) v[k] = sc->dout[k];
}

// --------------------------------------------------------------------------------------------
// Per-CTA context
// --------------------------------------------------------------------------------------------

template <class C>
struct Ctx {
  float *D, *A, *E, *Y, *K;  // planes (col-major, ld = m); K holds p planes back to back
  float *B, *V, *S;          // SVD buffers (col-major, ld = MAXD)
  float *nrm, *scl, *hv;
  Scal* sc;
  int m, n, p, mn;
};

// Pixel iterator over the column-major plane index idx = j*m + i with stride NT.
struct PixIter {
  int idx, i, j, di, dj, m;
  __device__ __forceinline__ PixIter(int start, int stride, int m_) : idx(start), m(m_) {
    j = start / m_;
    i = start - j * m_;
    dj = stride / m_;
    di = stride - dj * m_;
  }
  __device__ __forceinline__ void next(int stride) {
    idx += stride;
    i += di;
    j += dj;
    if (i >= m) {
      i -= m;
      ++j;
    }
  }
};

// --------------------------------------------------------------------------------------------
// Small dense kernels on the padded SVD buffers (column-major, ld = MAXD)
// --------------------------------------------------------------------------------------------

// C = L * R, L: rows x inner, R: inner x cols (C must not alias L or R). Rows >= rows_valid of C
// are written as 0. Thread tile: 4 rows x 2 columns (one float4 of L and two scalars of R per k).
template <class C>
__device__ __forceinline__ void gemm_nn(float* __restrict__ Cm, const float* __restrict__ Lm,
                                        const float* __restrict__ Rm, int rows_valid, int inner, int cols) {
  constexpr int MD = C::MAXD;
  constexpr int rt = MD / 4;  // every row group of the padded column is written (zeros below rows_valid)
  const int ct = (cols + 1) >> 1;
  const int ntiles = rt * ct;
  for (int tile = threadIdx.x; tile < ntiles; tile += C::NT) {
    const int i0 = (tile % rt) * 4;
    const int j0 = (tile / rt) * 2;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    const float* lp = Lm + i0;
    const float* r0 = Rm + j0 * MD;
    const float* r1 = r0 + MD;
    const int kend = i0 < rows_valid ? inner : 0;
#pragma unroll 4
    for (int k = 0; k < kend; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(lp + k * MD);
      const float b0 = r0[k], b1 = r1[k];
      acc[0] = fmaf(a.x, b0, acc[0]);
      acc[1] = fmaf(a.y, b0, acc[1]);
      acc[2] = fmaf(a.z, b0, acc[2]);
      acc[3] = fmaf(a.w, b0, acc[3]);
      acc[4] = fmaf(a.x, b1, acc[4]);
      acc[5] = fmaf(a.y, b1, acc[5]);
      acc[6] = fmaf(a.z, b1, acc[6]);
      acc[7] = fmaf(a.w, b1, acc[7]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const bool ok = (i0 + r) < rows_valid;
      Cm[j0 * MD + i0 + r] = ok ? acc[r] : 0.f;
      if (j0 + 1 < cols) Cm[(j0 + 1) * MD + i0 + r] = ok ? acc[4 + r] : 0.f;
    }
  }
  __syncthreads();
}

// Z = 1.5 I - 0.5 V^T V (one Newton-Schulz step for the polar factor: V <- V Z), into Zm.
template <class C>
__device__ __forceinline__ void ns_matrix(float* Zm, const float* Vm, int n) {
  constexpr int MD = C::MAXD;
  const int rt = (n + 3) >> 2;
  const int ct = (n + 1) >> 1;
  const int ntiles = rt * ct;
  for (int tile = threadIdx.x; tile < ntiles; tile += C::NT) {
    const int i0 = (tile % rt) * 4;
    const int j0 = (tile / rt) * 2;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int k = 0; k < n; k += 4) {  // rows of V (padded with zeros up to MAXD)
      float4 vi[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) vi[c] = *reinterpret_cast<const float4*>(Vm + (i0 + c) * MD + k);
      const float4 w0 = *reinterpret_cast<const float4*>(Vm + j0 * MD + k);
      const float4 w1 = *reinterpret_cast<const float4*>(Vm + (j0 + 1) * MD + k);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c] = fmaf(vi[c].x, w0.x, fmaf(vi[c].y, w0.y, fmaf(vi[c].z, w0.z, fmaf(vi[c].w, w0.w, acc[c]))));
        acc[4 + c] =
            fmaf(vi[c].x, w1.x, fmaf(vi[c].y, w1.y, fmaf(vi[c].z, w1.z, fmaf(vi[c].w, w1.w, acc[4 + c]))));
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + c;
      Zm[j0 * MD + i] = (i < n) ? ((i == j0 ? 1.5f : 0.f) - 0.5f * acc[c]) : 0.f;
      if (j0 + 1 < n) Zm[(j0 + 1) * MD + i] = (i < n) ? ((i == j0 + 1 ? 1.5f : 0.f) - 0.5f * acc[4 + c]) : 0.f;
    }
  }
  __syncthreads();
}

// out(i, j) = sum_k B'[i][k] V[j][k] (B' = B diag(h), pre-scaled), i < m, j < n.
template <class C, class Out>
__device__ __forceinline__ void gemm_bvt(const float* Bm, const float* Vm, int m, int n, Out out) {
  constexpr int MD = C::MAXD;
  const int rt = (m + 3) >> 2;
  const int ct = (n + 1) >> 1;
  const int ntiles = rt * ct;
  for (int tile = threadIdx.x; tile < ntiles; tile += C::NT) {
    const int i0 = (tile % rt) * 4;
    const int j0 = (tile / rt) * 2;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
#pragma unroll 4
    for (int k = 0; k < n; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(Bm + k * MD + i0);
      const float2 v = *reinterpret_cast<const float2*>(Vm + k * MD + j0);
      acc[0] = fmaf(a.x, v.x, acc[0]);
      acc[1] = fmaf(a.y, v.x, acc[1]);
      acc[2] = fmaf(a.z, v.x, acc[2]);
      acc[3] = fmaf(a.w, v.x, acc[3]);
      acc[4] = fmaf(a.x, v.y, acc[4]);
      acc[5] = fmaf(a.y, v.y, acc[5]);
      acc[6] = fmaf(a.z, v.y, acc[6]);
      acc[7] = fmaf(a.w, v.y, acc[7]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (i0 + r < m) {
        out(i0 + r, j0, acc[r]);
        if (j0 + 1 < n) out(i0 + r, j0 + 1, acc[4 + r]);
      }
    }
  }
}

template <class C>
__device__ __forceinline__ void set_identity(float* Vm, int n) {
  constexpr int MD = C::MAXD;
  for (int e = threadIdx.x; e < MD * MD; e += C::NT) {
    const int j = e / MD, i = e - j * MD;
    Vm[e] = (i == j && i < n) ? 1.f : 0.f;
  }
}

template <class C>
__device__ __forceinline__ void zero_buf(float* Xm) {
  constexpr int MD = C::MAXD;
  for (int e = threadIdx.x; e < MD * MD; e += C::NT) Xm[e] = 0.f;
}

// --------------------------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi on B = M V with fast (scaled) rotations
// --------------------------------------------------------------------------------------------
// Column pair (i, j): gamma = b_i . b_j; if |gamma| > tol sqrt(alpha beta) rotate so that the two
// columns become orthogonal (t = sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = (beta-alpha)/2gamma).
// Columns are stored scaled, b_j = scl_j x_j, so a rotation costs 2 FMAs per row instead of 4:
// x_i <- x_i - t (scl_j/scl_i) x_j, x_j <- x_j + t (scl_i/scl_j) x_i, scl <- c scl. The same
// transformation is applied to V, so B = M V holds throughout. Pair schedule: round-robin
// (circle method), n/2 disjoint pairs per round, one pair per LANES-lane unit, barrier per round.

template <class C, int MODE>
__device__ __forceinline__ void col_pass(Ctx<C>& cx, int n, float eps) {
  // MODE 0: nrm_j = ||x_j||^2, scl_j = 1 (no scaling applied)
  // MODE 1: apply scl to B and V columns, nrm_j fresh, scl_j = 1
  // MODE 2: as 1, then compute sigma_j = sqrt(nrm_j) and h_j = max(sigma-eps,0)/sigma (into hv)
  constexpr int MD = C::MAXD, L = C::LANES, RPL = C::RPL;
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const int warp = threadIdx.x >> 5;
  constexpr int UPW = 32 / L;  // units per warp
  for (int jb = warp * UPW; jb < n; jb += C::UNITS) {
    const int j = jb + (unit - warp * UPW);
    const bool valid = j < n;
    const int jj = valid ? j : 0;
    float* bp = cx.B + jj * MD + lu * RPL;
    float* vp = cx.V + jj * MD + lu * RPL;
    float x[RPL];
#pragma unroll
    for (int r = 0; r < RPL; r += 4) {
      if constexpr (RPL >= 4) {
        float4 t = *reinterpret_cast<float4*>(bp + r);
        x[r] = t.x; x[r + 1] = t.y; x[r + 2] = t.z; x[r + 3] = t.w;
      }
    }
    if constexpr (RPL == 2) {
      float2 t = *reinterpret_cast<float2*>(bp);
      x[0] = t.x; x[1] = t.y;
    }
    const float s = (MODE == 0) ? 1.f : cx.scl[jj];
    float ss = 0.f;
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      x[r] *= s;
      ss = fmaf(x[r], x[r], ss);
    }
#pragma unroll
    for (int off = L / 2; off; off >>= 1) ss += __shfl_xor_sync(FULL, ss, off);
    float y[RPL];
    float vv = 1.f;
    if (MODE != 0) {
      if constexpr (RPL >= 4) {
#pragma unroll
        for (int r = 0; r < RPL; r += 4) {
          const float4 t = *reinterpret_cast<const float4*>(vp + r);
          y[r] = t.x * s; y[r + 1] = t.y * s; y[r + 2] = t.z * s; y[r + 3] = t.w * s;
        }
      } else {
        const float2 t = *reinterpret_cast<const float2*>(vp);
        y[0] = t.x * s; y[1] = t.y * s;
      }
    }
    if (MODE == 2) {
      // rotations are orthogonal only to fp32 rounding, which drifts the column norms of V by a
      // few 1e-6 per SVT: B = M V holds for the drifted V, so sigma_j = ||b_j|| / ||v_j|| and
      // A = sum_j h_j b_j v_j^T / ||v_j||^2 remove that scale exactly.
      vv = 0.f;
#pragma unroll
      for (int r = 0; r < RPL; ++r) vv = fmaf(y[r], y[r], vv);
#pragma unroll
      for (int off = L / 2; off; off >>= 1) vv += __shfl_xor_sync(FULL, vv, off);
      ss = vv > 0.f ? ss / vv : 0.f;
    }
    float h = 1.f;
    if (MODE == 2) {
      const float sg = sqrtf(ss);
      h = (sg > eps) ? (sg - eps) / sg : 0.f;
    }
    if (valid && MODE != 0) {
      const float hb = (MODE == 2) ? (vv > 0.f ? h / vv : 0.f) : 1.f;
#pragma unroll
      for (int r = 0; r < RPL; ++r) x[r] *= hb;
      // B columns are stored pre-multiplied by h/||v||^2 in MODE 2 (ready for A = B' V^T)
      if constexpr (RPL >= 4) {
#pragma unroll
        for (int r = 0; r < RPL; r += 4) {
          *reinterpret_cast<float4*>(bp + r) = make_float4(x[r], x[r + 1], x[r + 2], x[r + 3]);
          *reinterpret_cast<float4*>(vp + r) = make_float4(y[r], y[r + 1], y[r + 2], y[r + 3]);
        }
      } else {
        *reinterpret_cast<float2*>(bp) = make_float2(x[0], x[1]);
        *reinterpret_cast<float2*>(vp) = make_float2(y[0], y[1]);
      }
    }
    if (valid && lu == 0) {
      cx.nrm[j] = ss;
      cx.scl[j] = 1.f;
      if (MODE == 2) cx.hv[j] = h;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void rr_pair(int r, int k, int Nn, int& i, int& j) {
  if (k == 0) {
    i = Nn - 1;
    j = r;
  } else {
    const int q = Nn - 1;
    i = (r + k) % q;
    j = (r - k + q) % q;
  }
}

// Returns the number of sweeps; *capped = the last sweep still rotated at the sweep cap.
template <class C>
__device__ int jacobi_sweeps(Ctx<C>& cx, int n, float tol, int max_sweeps, bool* capped) {
  constexpr int MD = C::MAXD, L = C::LANES, RPL = C::RPL;
  constexpr int UPW = 32 / L;
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const int warp = threadIdx.x >> 5;
  const int Nn = n + (n & 1);
  const int npairs = Nn >> 1;
  float* __restrict__ Bm = cx.B;
  float* __restrict__ Vm = cx.V;
  float* __restrict__ nrm = cx.nrm;
  float* __restrict__ scl = cx.scl;
  col_pass<C, 0>(cx, n, 0.f);
  int sweeps = 0;
  bool any = false;
  while (sweeps < max_sweeps) {
    bool rot = false;
    for (int r = 0; r < Nn - 1; ++r) {
      for (int kb = warp * UPW; kb < npairs; kb += C::UNITS) {
        const int k = kb + (unit - warp * UPW);
        int i = 0, j = 0;
        if (k < npairs) rr_pair(r, k, Nn, i, j);
        const bool valid = (k < npairs) && (i < n) && (j < n);
        if (!valid) { i = 0; j = 0; }
        float* bi = Bm + i * MD + lu * RPL;
        float* bj = Bm + j * MD + lu * RPL;
        float* vi = Vm + i * MD + lu * RPL;
        float* vj = Vm + j * MD + lu * RPL;
        float xi[RPL], xj[RPL];
        if constexpr (RPL >= 4) {
#pragma unroll
          for (int q = 0; q < RPL; q += 4) {
            const float4 a = *reinterpret_cast<const float4*>(bi + q);
            const float4 b = *reinterpret_cast<const float4*>(bj + q);
            xi[q] = a.x; xi[q + 1] = a.y; xi[q + 2] = a.z; xi[q + 3] = a.w;
            xj[q] = b.x; xj[q + 1] = b.y; xj[q + 2] = b.z; xj[q + 3] = b.w;
          }
        } else {
          const float2 a = *reinterpret_cast<const float2*>(bi);
          const float2 b = *reinterpret_cast<const float2*>(bj);
          xi[0] = a.x; xi[1] = a.y; xj[0] = b.x; xj[1] = b.y;
        }
        float g = 0.f;
#pragma unroll
        for (int q = 0; q < RPL; ++q) g = fmaf(xi[q], xj[q], g);
#pragma unroll
        for (int off = L / 2; off; off >>= 1) g += __shfl_xor_sync(FULL, g, off);
        const float al = nrm[i], be = nrm[j], di = scl[i], dj = scl[j];
        const float gam = g * di * dj;
        if (valid && al > 0.f && be > 0.f && fabsf(gam) > tol * sqrtf(al * be)) {
          const float zeta = (be - al) / (2.f * gam);
          const float az = fabsf(zeta);
          float t = (az > 1e18f) ? 0.5f / zeta : copysignf(1.f, zeta) / (az + sqrtf(fmaf(zeta, zeta, 1.f)));
          const float x = fmaf(t, t, 1.f);
          float c = rsqrtf(x);
          c = c * fmaf(-0.5f * x * c, c, 1.5f);  // one Newton step: c = 1/sqrt(1+t^2) to ~1 ulp
          const float ca = t * (dj / di);
          const float cb = t * (di / dj);
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const float o = xi[q];
            xi[q] = fmaf(-ca, xj[q], o);
            xj[q] = fmaf(cb, o, xj[q]);
          }
          float yi[RPL], yj[RPL];
          if constexpr (RPL >= 4) {
#pragma unroll
            for (int q = 0; q < RPL; q += 4) {
              const float4 a = *reinterpret_cast<const float4*>(vi + q);
              const float4 b = *reinterpret_cast<const float4*>(vj + q);
              yi[q] = a.x; yi[q + 1] = a.y; yi[q + 2] = a.z; yi[q + 3] = a.w;
              yj[q] = b.x; yj[q + 1] = b.y; yj[q + 2] = b.z; yj[q + 3] = b.w;
            }
          } else {
            const float2 a = *reinterpret_cast<const float2*>(vi);
            const float2 b = *reinterpret_cast<const float2*>(vj);
            yi[0] = a.x; yi[1] = a.y; yj[0] = b.x; yj[1] = b.y;
          }
#pragma unroll
          for (int q = 0; q < RPL; ++q) {
            const float o = yi[q];
            yi[q] = fmaf(-ca, yj[q], o);
            yj[q] = fmaf(cb, o, yj[q]);
          }
          if constexpr (RPL >= 4) {
#pragma unroll
            for (int q = 0; q < RPL; q += 4) {
              *reinterpret_cast<float4*>(bi + q) = make_float4(xi[q], xi[q + 1], xi[q + 2], xi[q + 3]);
              *reinterpret_cast<float4*>(bj + q) = make_float4(xj[q], xj[q + 1], xj[q + 2], xj[q + 3]);
              *reinterpret_cast<float4*>(vi + q) = make_float4(yi[q], yi[q + 1], yi[q + 2], yi[q + 3]);
              *reinterpret_cast<float4*>(vj + q) = make_float4(yj[q], yj[q + 1], yj[q + 2], yj[q + 3]);
            }
          } else {
            *reinterpret_cast<float2*>(bi) = make_float2(xi[0], xi[1]);
            *reinterpret_cast<float2*>(bj) = make_float2(xj[0], xj[1]);
            *reinterpret_cast<float2*>(vi) = make_float2(yi[0], yi[1]);
            *reinterpret_cast<float2*>(vj) = make_float2(yj[0], yj[1]);
          }
          if (lu == 0) {
            nrm[i] = fmaxf(fmaf(-t, gam, al), 0.f);
            nrm[j] = fmaf(t, gam, be);
            scl[i] = c * di;
            scl[j] = c * dj;
          }
          rot = true;
        }
      }
      __syncthreads();
    }
    ++sweeps;
    any = __syncthreads_or(rot);
    col_pass<C, 1>(cx, n, 0.f);  // re-normalise (apply scales, fresh norms)
    if (!any) break;
  }
  *capped = any;
  return sweeps;
}

// sigma_j = sqrt(nrm_j) stats after the final pass: nuclear norm of S_eps, ranks (Z19), sigma_1.
template <class C>
__device__ __forceinline__ void svt_stats(Ctx<C>& cx, int n, float eps) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    float nuc = 0.f, smax = 0.f, amax = 0.f;
    int cnt = 0;
    for (int j = lane; j < n; j += 32) {
      const float sg = sqrtf(cx.nrm[j]);
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
      const float a = fmaxf(sqrtf(cx.nrm[j]) - eps, 0.f);
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
// Uses S as the n x n temporary and B as the output, then swaps B and V.
template <class C>
__device__ __forceinline__ void ns_step(Ctx<C>& cx, int n) {
  ns_matrix<C>(cx.S, cx.V, n);
  gemm_nn<C>(cx.B, cx.V, cx.S, n, n, n);
  float* t = cx.B;
  cx.B = cx.V;
  cx.V = t;
}

struct SvtOut {
  int sweeps;
  bool capped;
};

// S_eps(M) with M in S (padded col-major). Leaves V (orthonormalised by one Newton-Schulz step)
// warm for the next call, calls out(i, j, a_ij) for every entry of the result.
template <class C, bool DO_OUT, class Out>
__device__ SvtOut svt(Ctx<C>& cx, int m, int n, float eps, float tol, int max_sweeps, bool warm, Out out,
                      bool orthonormalise_after) {
  if (!warm) {
    set_identity<C>(cx.V, n);
    __syncthreads();
  }
  gemm_nn<C>(cx.B, cx.S, cx.V, m, n, n);  // B = M V
  SvtOut r;
  r.sweeps = jacobi_sweeps<C>(cx, n, tol, max_sweeps, &r.capped);
  col_pass<C, 2>(cx, n, eps);  // sigma_j, h_j, B <- B diag(h)
  svt_stats<C>(cx, n, eps);
  if constexpr (DO_OUT) gemm_bvt<C>(cx.B, cx.V, m, n, out);  // A = B diag(h) V^T
  __syncthreads();
  if (orthonormalise_after) ns_step<C>(cx, n);
  return r;
}

// --------------------------------------------------------------------------------------------
// Warp + Jacobian (Alg. 1 Step 1; readings Z2, Z15, Z16)
// --------------------------------------------------------------------------------------------

struct WarpGeom {
  double s, cx, cy, h11, h12, h13, h21, h22, h23, h31, h32;
  int m, n, p, kind;
};

__device__ __forceinline__ WarpGeom make_geom(const int* box, const double* tau, int kind) {
  WarpGeom g;
  const int x0 = box[0], y0 = box[1];
  g.n = box[2];
  g.m = box[3];
  g.s = 0.5 * (double)max(g.m, g.n);
  g.cx = x0 + 0.5 * (g.n - 1);
  g.cy = y0 + 0.5 * (g.m - 1);
  g.h11 = tau[0]; g.h12 = tau[1]; g.h21 = tau[2]; g.h22 = tau[3]; g.h13 = tau[4]; g.h23 = tau[5];
  g.h31 = kind == TILT_HOMOGRAPHY ? tau[6] : 0.0;
  g.h32 = kind == TILT_HOMOGRAPHY ? tau[7] : 0.0;
  g.kind = kind;
  g.p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  return g;
}

// Bilinear sample d and J_raw row (p entries) at window pixel (i, j). Returns false on escape.
__device__ __forceinline__ bool warp_pixel(const WarpGeom& g, const float* __restrict__ img, int H, int W,
                                           int i, int j, double& d, double (&jr)[8]) {
  const double du = j - 0.5 * (g.n - 1);
  const double dv = i - 0.5 * (g.m - 1);
  const double w = 1.0 + (g.h31 * du + g.h32 * dv) / g.s;
  const double X = g.cx + (g.h11 * du + g.h12 * dv + g.s * g.h13) / w;
  const double Y = g.cy + (g.h21 * du + g.h22 * dv + g.s * g.h23) / w;
  const double X0 = floor(X), Y0 = floor(Y);
  if (!(X0 >= 0.0 && X0 + 1.0 <= W - 1 && Y0 >= 0.0 && Y0 + 1.0 <= H - 1)) {
    d = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) jr[q] = 0.0;
    return false;
  }
  const double fx = X - X0, fy = Y - Y0;
  const int xi = (int)X0, yi = (int)Y0;
  const float* r0 = img + (size_t)yi * W + xi;
  const double i00 = __ldg(r0), i01 = __ldg(r0 + 1), i10 = __ldg(r0 + W), i11 = __ldg(r0 + W + 1);
  d = (1.0 - fy) * ((1.0 - fx) * i00 + fx * i01) + fy * ((1.0 - fx) * i10 + fx * i11);
  const double dX = (1.0 - fy) * (i01 - i00) + fy * (i11 - i10);
  const double dY = (1.0 - fx) * (i10 - i00) + fx * (i11 - i01);
  const double u = du / g.s, v = dv / g.s;
  const double xn = (X - g.cx) / g.s, yn = (Y - g.cy) / g.s;
  const double gx = g.s * dX / w, gy = g.s * dY / w;
  jr[0] = gx * u; jr[1] = gx * v; jr[2] = gy * u; jr[3] = gy * v; jr[4] = gx; jr[5] = gy;
  const double gz = -(gx * xn + gy * yn);
  jr[6] = gz * u; jr[7] = gz * v;
  return true;
}

// Centre + area constraint rows (reading Z10), unit-norm rows, into q[3][p].
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

// --------------------------------------------------------------------------------------------
// Orthonormalise (K2): from D (raw d, fp32) and K planes holding J_raw (fp32) build
//   D_hat = d/||d||, J = (J_raw - D_hat c^T)/||d||  (quotient rule) [if normalise]
//   G = J^TJ + Q^TQ = L L^T (fp64), K = J L^{-T} (fp64 per pixel, stored fp32)
// so that W^TW v = v - K K^T v (Eq. Jperpv, Eq. WTW_property).
// Returns a tilt_patch_status (ZERO_PATCH / SINGULAR_GRAM / CONVERGED=ok).
// --------------------------------------------------------------------------------------------
template <class C, int CH>
__device__ __forceinline__ void gram_chunk(Ctx<C>& cx, bool normalise, double ind, const double (&c)[8],
                                           double* Gout) {
  // entries e in [12*CH, 12*CH+12) of the 8x8 upper triangle (row-major); q >= p columns are 0
  const int mn = cx.mn, p = cx.p;
  const float* __restrict__ Dp = cx.D;
  const float* __restrict__ Kp = cx.K;
  double acc[12];
#pragma unroll
  for (int e = 0; e < 12; ++e) acc[e] = 0.0;
  for (int idx = threadIdx.x; idx < mn; idx += C::NT) {
    const double dh = normalise ? Dp[idx] * ind : 0.0;
    double jn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? ((double)Kp[q * mn + idx] - dh * c[q]) * ind : 0.0;
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
__device__ int orthonormalise(Ctx<C>& cx, bool normalise, const double* qrows, int l) {
  Scal* sc = cx.sc;
  const int mn = cx.mn, p = cx.p;
  float* __restrict__ Dp = cx.D;
  float* __restrict__ Kp = cx.K;
  double nd = 1.0;
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (normalise) {
    double acc[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] = 0.0;
    for (int idx = threadIdx.x; idx < mn; idx += C::NT) {
      const double d = Dp[idx];
      acc[8] = fma(d, d, acc[8]);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < p) acc[q] = fma((double)Kp[q * mn + idx], d, acc[q]);
    }
    block_sum_d<C, 9>(acc, sc);
    nd = sqrt(acc[8]);
    if (threadIdx.x == 0) sc->nd = (float)nd;
    if (!(nd > 0.0)) return TILT_PATCH_ZERO_PATCH;
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = acc[q] / nd;
  }
  const double ind = 1.0 / nd;
  double G[36];
  gram_chunk<C, 0>(cx, normalise, ind, c, G);
  gram_chunk<C, 1>(cx, normalise, ind, c, G);
  gram_chunk<C, 2>(cx, normalise, ind, c, G);
  if (threadIdx.x == 0) {
    // G (8x8 upper-triangle layout) + Q^T Q, Cholesky L L^T, then L^{-1}  (fp64, one thread)
    double Gf[64];
    int e = 0;
    for (int a = 0; a < 8; ++a)
      for (int b = a; b < 8; ++b) {
        Gf[a * 8 + b] = G[e];
        Gf[b * 8 + a] = G[e];
        ++e;
      }
    for (int r = 0; r < l; ++r)
      for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b) Gf[a * 8 + b] += qrows[r * 8 + a] * qrows[r * 8 + b];
    double* Lm = sc->L;
    double* Li = sc->Linv;
    for (int a = 0; a < 64; ++a) { Lm[a] = 0.0; Li[a] = 0.0; }
    double dmax = 0.0;
    for (int a = 0; a < p; ++a) dmax = fmax(dmax, Gf[a * 8 + a]);
    bool ok = dmax > 0.0 && isfinite(dmax);
    for (int a = 0; a < p && ok; ++a) {
      double s = Gf[a * 8 + a];
      for (int k = 0; k < a; ++k) s -= Lm[a * 8 + k] * Lm[a * 8 + k];
      if (!(s > 1e-14 * dmax)) { ok = false; break; }
      const double la = sqrt(s);
      Lm[a * 8 + a] = la;
      for (int b = a + 1; b < p; ++b) {
        double t = Gf[b * 8 + a];
        for (int k = 0; k < a; ++k) t -= Lm[b * 8 + k] * Lm[a * 8 + k];
        Lm[b * 8 + a] = t / la;
      }
    }
    if (ok) {
      for (int a = 0; a < p; ++a) {  // L^{-1} column by column (forward substitution)
        Li[a * 8 + a] = 1.0 / Lm[a * 8 + a];
        for (int b = a + 1; b < p; ++b) {
          double s = 0.0;
          for (int k = a; k < b; ++k) s += Lm[b * 8 + k] * Li[k * 8 + a];
          Li[b * 8 + a] = -s / Lm[b * 8 + b];
        }
      }
    }
    for (int q = 0; q < 8; ++q) sc->c[q] = c[q];
    sc->flag = ok ? 1 : 0;
  }
  __syncthreads();
  if (!sc->flag) return TILT_PATCH_SINGULAR_GRAM;
  // K = J L^{-T}: K[:, a] = sum_{b <= a} Linv[a][b] J[:, b]; D_hat stored fp32
  const double* Li = sc->Linv;
  for (int idx = threadIdx.x; idx < mn; idx += C::NT) {
    const double dh = normalise ? Dp[idx] * ind : 0.0;
    double jn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? ((double)Kp[q * mn + idx] - dh * c[q]) * ind : 0.0;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      if (a < p) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b <= a; ++b) s = fma(Li[a * 8 + b], jn[b], s);
        Kp[a * mn + idx] = (float)s;
      }
    }
    if (normalise) Dp[idx] = (float)dh;
  }
  __syncthreads();
  return TILT_PATCH_CONVERGED;
}

// s = K^T v for v(idx) given by a functor; result (p floats) returned in s (all threads).
template <class C, class VF>
__device__ __forceinline__ void kt_reduce(Ctx<C>& cx, VF vf, float (&s)[8]) {
  const int mn = cx.mn, p = cx.p;
  const float* __restrict__ Kp = cx.K;
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.f;
  for (int idx = threadIdx.x; idx < mn; idx += C::NT) {
    const float v = vf(idx);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < p) s[q] = fmaf(Kp[q * mn + idx], v, s[q]);
  }
  block_sum_f<C, 8>(s, cx.sc);
}

template <class C>
__device__ __forceinline__ float k_apply(const Ctx<C>& cx, int idx, const float (&s)[8]) {
  const int mn = cx.mn, p = cx.p;
  float r = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < p) r = fmaf(cx.K[q * mn + idx], s[q], r);
  return r;
}

}  // namespace tilt

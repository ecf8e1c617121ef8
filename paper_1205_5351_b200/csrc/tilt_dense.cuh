// tilt_dense.cuh — batched dense FP32 kernels of the multi-CTA path (tilt_large.cu): a tiled GEMM
// and a blocked LU solve, both over per-problem workspace slots.
//
// Every problem b owns the slot ws + b * stride (column-major matrices at float offsets inside the
// slot). A kernel runs on all problems (widx == nullptr, blockIdx.z = b) or on the subset listed in
// widx[0 .. gridDim.z) (the problems that take Algorithm 2's warm step).
//
// * k_gemm: C = alpha op(A) op(B) + beta C (op = identity or transpose), 64 x 64 x 16 tiles,
//   256 threads with a 4 x 4 register micro-tile (two 16-byte shared loads per 16 FMAs),
//   double-buffered shared memory with register prefetch of the next K-slice. FP32 FMA throughout
//   (no TF32: the 1e-4 parity of BASELINE.json needs FP32 products). Replaces the SGEMMs of B = MV,
//   A = B diag(h) V^T, the Newton-Schulz step and Algorithm 2's products.
// * LU without pivoting, blocked by LU_NB = 32 (right-looking: diagonal block, the two triangular
//   panels, trailing GEMM update), then forward / backward substitution with blocked GEMM updates.
//   It solves Algorithm 2's Cayley systems (I + S) X = R exactly (Eq. curve_to_search).
//   S = (t*/2) P is skew (P_U, P_V are tangent directions), so I + S has symmetric part
//   I: every leading principal block is nonsingular (x^T (I + S) x = ||x||^2 > 0), elimination
//   without pivoting never meets a zero pivot, and the growth is bounded by ~(1 + ||S||) (a matrix
//   whose symmetric part is positive definite) -- the reason no pivot search is needed.
#pragma once

#include <cuda_runtime.h>

namespace tilt {
namespace dense {

constexpr int GBM = 64, GBN = 64, GBK = 16, GNT = 256;
constexpr int LU_NB = 32;

__device__ __forceinline__ float* prob_base(float* ws, size_t stride, const int* widx) {
  const int b = widx ? widx[blockIdx.z] : (int)blockIdx.z;
  return ws + (size_t)b * stride;
}

// C = alpha op(A) op(B) + beta C; op(A) is M x K, op(B) is K x N (column-major, leading dims lda,
// ldb, ldc). beta == 0 never reads C.
template <bool TA, bool TB>
__global__ void __launch_bounds__(GNT) k_gemm(float* __restrict__ ws, size_t stride, const int* __restrict__ widx,
                                              int M, int N, int K, size_t oA, int lda, size_t oB, int ldb, size_t oC,
                                              int ldc, float alpha, float beta) {
  float* base = prob_base(ws, stride, widx);
  const float* __restrict__ A = base + oA;
  const float* __restrict__ Bm = base + oB;
  float* C = base + oC;
  __shared__ __align__(16) float As[2][GBK][GBM + 4];
  __shared__ __align__(16) float Bs[2][GBK][GBN + 4];
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const int i0 = blockIdx.x * GBM, j0 = blockIdx.y * GBN;
  float ra[4], rb[4];
  // element q of this thread's share of a 64 x 16 (A) / 16 x 64 (B) tile: (row/col in tile, k)
  auto a_idx = [&](int q, int& i, int& kk) {
    if (!TA) { i = t & 63; kk = (t >> 6) + 4 * q; }   // op(A)(i,k) = A[i + k lda]: coalesced in i
    else     { kk = t & 15; i = (t >> 4) + 16 * q; }  // op(A)(i,k) = A[k + i lda]: coalesced in k
  };
  auto b_idx = [&](int q, int& j, int& kk) {
    if (!TB) { kk = t & 15; j = (t >> 4) + 16 * q; }  // op(B)(k,j) = B[k + j ldb]
    else     { j = t & 63; kk = (t >> 6) + 4 * q; }   // op(B)(k,j) = B[j + k ldb]
  };
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i, kk;
      a_idx(q, i, kk);
      const int gi = i0 + i, gk = k0 + kk;
      ra[q] = (gi < M && gk < K) ? (TA ? A[gk + (size_t)gi * lda] : A[gi + (size_t)gk * lda]) : 0.f;
      int j, kb;
      b_idx(q, j, kb);
      const int gj = j0 + j, gkb = k0 + kb;
      rb[q] = (gj < N && gkb < K) ? (TB ? Bm[gj + (size_t)gkb * ldb] : Bm[gkb + (size_t)gj * ldb]) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int i, kk;
      a_idx(q, i, kk);
      As[buf][kk][i] = ra[q];
      int j, kb;
      b_idx(q, j, kb);
      Bs[buf][kb][j] = rb[q];
    }
  };
  float acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.f;
  load(0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += GBK) {
    const bool more = k0 + GBK < K;
    if (more) load(k0 + GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      const float4 a4 = *reinterpret_cast<const float4*>(&As[buf][kk][4 * tx]);
      const float4 b4 = *reinterpret_cast<const float4*>(&Bs[buf][kk][4 * ty]);
      const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int gj = j0 + 4 * ty + c;
    if (gj >= N) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int gi = i0 + 4 * tx + r;
      if (gi >= M) continue;
      float* cp = C + gi + (size_t)gj * ldc;
      *cp = beta != 0.f ? fmaf(alpha, acc[r][c], beta * *cp) : alpha * acc[r][c];
    }
  }
}

// LU (no pivoting) of the nb x nb diagonal block at (k0, k0) of P (leading dimension ldp), in place:
// unit lower L11 below the diagonal, U11 on and above it. One CTA per problem.
__global__ void __launch_bounds__(256) k_lu_diag(float* __restrict__ ws, size_t stride, const int* __restrict__ widx,
                                                 size_t oP, int ldp, int k0, int nb) {
  float* P = prob_base(ws, stride, widx) + oP + k0 + (size_t)k0 * ldp;
  __shared__ float D[LU_NB][LU_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) D[e % nb][e / nb] = P[e % nb + (size_t)(e / nb) * ldp];
  __syncthreads();
  for (int j = 0; j < nb - 1; ++j) {
    const float inv = 1.f / D[j][j];
    for (int i = j + 1 + threadIdx.x; i < nb; i += blockDim.x) D[i][j] *= inv;
    __syncthreads();
    const int w = nb - 1 - j;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int i = j + 1 + e % w, c = j + 1 + e / w;
      D[i][c] = fmaf(-D[i][j], D[j][c], D[i][c]);
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) P[e % nb + (size_t)(e / nb) * ldp] = D[e % nb][e / nb];
}

// X[k0:k0+nb, c] <- L11^{-1} X[k0:k0+nb, c] (L11 unit lower, from P at (k0, k0)) for the columns
// c in [c0, c0 + ncols) of X (leading dimension ldx): the row panel of the factorisation (X = P) and
// the forward substitution. One thread per column.
__global__ void __launch_bounds__(128) k_trsm_l(float* __restrict__ ws, size_t stride, const int* __restrict__ widx,
                                                size_t oP, int ldp, size_t oX, int ldx, int k0, int nb, int c0,
                                                int ncols) {
  float* base = prob_base(ws, stride, widx);
  const float* L = base + oP + k0 + (size_t)k0 * ldp;
  __shared__ float Ls[LU_NB][LU_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Ls[e % nb][e / nb] = L[e % nb + (size_t)(e / nb) * ldp];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  float* x = base + oX + k0 + (size_t)(c0 + c) * ldx;
  float v[LU_NB];
#pragma unroll
  for (int r = 0; r < LU_NB; ++r) v[r] = r < nb ? x[r] : 0.f;
#pragma unroll
  for (int r = 1; r < LU_NB; ++r) {
    float s = v[r];
#pragma unroll
    for (int q = 0; q < r; ++q) s = fmaf(-Ls[r][q], v[q], s);
    v[r] = r < nb ? s : 0.f;
  }
#pragma unroll
  for (int r = 0; r < LU_NB; ++r)
    if (r < nb) x[r] = v[r];
}

// X[k0:k0+nb, c] <- U11^{-1} X[k0:k0+nb, c] (U11 upper, from P at (k0, k0)): backward substitution.
__global__ void __launch_bounds__(128) k_trsm_u(float* __restrict__ ws, size_t stride, const int* __restrict__ widx,
                                                size_t oP, int ldp, size_t oX, int ldx, int k0, int nb, int ncols) {
  float* base = prob_base(ws, stride, widx);
  const float* U = base + oP + k0 + (size_t)k0 * ldp;
  __shared__ float Us[LU_NB][LU_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Us[e % nb][e / nb] = U[e % nb + (size_t)(e / nb) * ldp];
  __syncthreads();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  float* x = base + oX + k0 + (size_t)c * ldx;
  float v[LU_NB];
#pragma unroll
  for (int r = 0; r < LU_NB; ++r) v[r] = r < nb ? x[r] : 0.f;
#pragma unroll
  for (int r = LU_NB - 1; r >= 0; --r) {
    if (r < nb) {
      float s = v[r];
#pragma unroll
      for (int q = r + 1; q < LU_NB; ++q) s = fmaf(-Us[r][q], v[q], s);
      v[r] = s / Us[r][r];
    }
  }
#pragma unroll
  for (int r = 0; r < LU_NB; ++r)
    if (r < nb) x[r] = v[r];
}

// P[r, k0:k0+nb] <- P[r, k0:k0+nb] U11^{-1} for the rows r in [k0 + nb, k0 + nb + nrows): the column
// panel of the factorisation (L21). One thread per row (coalesced: consecutive rows).
__global__ void __launch_bounds__(128) k_trsm_ru(float* __restrict__ ws, size_t stride, const int* __restrict__ widx,
                                                 size_t oP, int ldp, int k0, int nb, int nrows) {
  float* base = prob_base(ws, stride, widx);
  float* P = base + oP;
  const float* U = P + k0 + (size_t)k0 * ldp;
  __shared__ float Us[LU_NB][LU_NB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) Us[e % nb][e / nb] = U[e % nb + (size_t)(e / nb) * ldp];
  __syncthreads();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  float* x = P + (k0 + nb + r) + (size_t)k0 * ldp;
  float v[LU_NB];
#pragma unroll
  for (int j = 0; j < LU_NB; ++j) v[j] = j < nb ? x[(size_t)j * ldp] : 0.f;
#pragma unroll
  for (int j = 0; j < LU_NB; ++j) {
    if (j < nb) {
      float s = v[j];
#pragma unroll
      for (int i = 0; i < j; ++i) s = fmaf(-v[i], Us[i][j], s);
      v[j] = s / Us[j][j];
    }
  }
#pragma unroll
  for (int j = 0; j < LU_NB; ++j)
    if (j < nb) x[(size_t)j * ldp] = v[j];
}

}  // namespace dense
}  // namespace tilt

// tilt_large.cu — the multi-CTA path for large windows (m, n <= 1024; SURVEY.md §8(f) NEXT-4:
// Table 1's 300x300 ... 1000x1000 sizes). The same LADMAP inner loop as
// tilt_kernels.cuh (P:437-501 with errata E1, E2; readings Z3, Z6, Z7, Z14, Z19, Z21) and the same
// warm one-sided Jacobi SVT, with the work of one problem spread over the
// whole GPU instead of one CTA:
//   * planes (column-major, ld = m rounded to 4) live in a per-problem HBM/L2 slot;
//   * elementwise passes and the projector reductions K^T v run over all CTAs (fp64 atomics);
//   * B = M V, A = B diag(h) V^T, the Newton-Schulz step and Algorithm 2's products are the
//     hand-written batched FP32 GEMM of tilt_dense.cuh (no TF32), its Cayley systems the blocked LU
//     solve there;
//   * the Jacobi sweep is block-cyclic: columns in blocks of BW = 16; one round rotates every
//     cross pair of a block pair (one CTA per block pair; both blocks' columns staged in shared
//     memory, 16 warps, one column pair per warp, fast scaled rotations as tilt_jacobi.cuh) and
//     accumulates the 32 x 32 transformation W, then V <- V W for the pair's 32 columns. A sweep is
//     one intra-block round plus the circle method over blocks, so every column pair is visited
//     once per sweep as in the CTA kernels; the stop rule is theirs.
// The host drives the iteration (one stream; one host read of an active-problem counter per Jacobi
// sweep and per LADMAP iteration).
#define TILT_NO_FREE_KERNELS

#include <cstdio>
#include <cstring>

#include "tilt_dense.cuh"
#include "tilt_kernels.cuh"
#include "tilt_large_host.h"
#include "tilt_nvtx.h"

namespace tilt {
namespace lp {
namespace {

constexpr int BW = 16;    // Jacobi block width (columns)
constexpr int RNT = 512;  // threads of a Jacobi round (16 warps)
constexpr int ENT = 256;  // threads of the elementwise / reduction kernels
constexpr int EPT = 8;    // elements per thread of the elementwise kernels
constexpr int NACC = 40;

// fp64 accumulator slots (G: setup only; the others per LADMAP iteration)
enum : int {
  ACC_G = 0,    // 36 (packed upper triangle of J^T J)
  ACC_S1 = 0,   // 8: K^T v, then 1: ||A+ - A||^2
  ACC_DA = 8,
  ACC_S2 = 9,   // 8: K^T v2, then 1: ||E+ - E||^2
  ACC_DE = 17,
  ACC_C1 = 18,  // ||R||^2
  ACC_R = 19,   // ||W^TW D||^2
  ACC_L1 = 20   // ||E||_1
};

struct St {
  double acc[NACC];
  double Linv[64];
  float mu, mu_next, mu0, mu_max, denom, denom0, lam, eps;
  float crit1, crit2, nuc, sig1;
  float inv_nd;  // ADM: 1 / ||D||_F
  int svt_rank, relrank, band;
  int iters, done, status, conv;
  int svt_done, big_any, rot_any, sw_cur, cap_cur, rot_cur;
  int sweeps, caps, rotations, aux_sweeps;
  double fro2;  // ||B||_F^2 at the start of the current SVT (negligible-column threshold)
  // SVD warm start (Algorithm 2, svd_mode 1; readings Z26/Z27)
  double wacc[8];  // ||M - M_prev||^2, <h0, h1>, ||h1||^2, <h0, h2>, ||P_U||^2, ||P_V||^2
  float eps_svd, t_star;
  int warm, have_prev, warm_steps;
  // Algorithm 1 state (solve entry)
  double tau[8];
  double Q[24];
  float f_prev, f, dtau_inf, nd;
  int outer_done, have_fprev, outer_iters, inner_total, stop_rule, esc;
};

struct Lay {
  int m, n, p, ldm, ldn;
  size_t plane, vplane;
  size_t oD, oA, oAn, oE, oY, oS, oB, oK, oV, oV2, oT, oSig, oVv, oSt, stride;
  // SVD warm start buffers (0 when not allocated): U, M_prev, W, H1, Z, H2, X, X2 (m x n),
  // P_U (m x m, ld = ldm), P_V, Vt, Vt2 (n x n), signed Sigma, P_Sigma (n)
  size_t oU, oMp, oW, oH1, oZ, oH2, oX, oX2, oPU, oPV, oVt, oVt2, oSg, oPs;
};

inline size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }

Lay make_lay(int m, int n, int p, bool svdws = false) {
  Lay L;
  L.m = m;
  L.n = n;
  L.p = p;
  L.ldm = (int)up(m, 4);
  L.ldn = (int)up(n, 4);
  L.plane = up((size_t)L.ldm * n, 64);
  L.vplane = up((size_t)L.ldn * n, 64);
  size_t o = 0;
  L.oD = o; o += L.plane;
  L.oA = o; o += L.plane;
  L.oAn = o; o += L.plane;
  L.oE = o; o += L.plane;
  L.oY = o; o += L.plane;
  L.oS = o; o += L.plane;
  L.oB = o; o += L.plane;
  L.oK = o; o += (size_t)p * L.plane;
  L.oV = o; o += L.vplane;
  L.oV2 = o; o += L.vplane;
  L.oT = o; o += L.vplane;
  L.oSig = o; o += up(n, 64);
  L.oVv = o; o += up(n, 64);
  L.oSt = o; o += up(sizeof(St) / 4 + 1, 64);
  L.oU = L.oMp = L.oW = L.oH1 = L.oZ = L.oH2 = L.oX = L.oX2 = L.oPU = L.oPV = L.oVt = L.oVt2 = L.oSg = L.oPs = 0;
  if (svdws) {
    L.oU = o; o += L.plane;
    L.oMp = o; o += L.plane;
    L.oW = o; o += L.plane;
    L.oH1 = o; o += L.plane;
    L.oZ = o; o += L.plane;
    L.oH2 = o; o += L.plane;
    L.oX = o; o += L.plane;
    L.oX2 = o; o += L.plane;
    L.oPU = o; o += up((size_t)L.ldm * m, 64);
    L.oPV = o; o += L.vplane;
    L.oVt = o; o += L.vplane;
    L.oVt2 = o; o += L.vplane;
    L.oSg = o; o += up(n, 64);
    L.oPs = o; o += up(n, 64);
  }
  L.stride = o;
  return L;
}

struct Args {
  float* ws;
  Lay L;
  int B;
  DevParams P;
  size_t oV;       // current V buffer (swapped by the Newton-Schulz step)
  float tol, big2;
  float tiny2;     // a column with ||b||^2 <= tiny2 ||B||_F^2 is numerically zero: never rotated
  int max_sweeps;
  int NB, NBp;     // Jacobi blocks
  int niter;
  int* counter;
  int rep_outer, cur_outer;  // replay / trace rows: [B][rep_outer][max_inner] (1, 0 for the inner entry)
  // Algorithm 1 (tilt_solve_batch on the multi-CTA path)
  const float* images;
  int n_images, H, W, kind;
  const int* patch_image;
  const int* boxes;
  // pyramid warm start (reading Z26): the coarse level's A, E, Y [B][m/2][n/2] row-major and reports
  const float* warm_A;
  const float* warm_E;
  const float* warm_Y;
  const tilt_report* warm_rep;
};

__device__ __forceinline__ float* slot(const Args& a, int b) { return a.ws + (size_t)b * a.L.stride; }
__device__ __forceinline__ St* state(const Args& a, int b) { return reinterpret_cast<St*>(slot(a, b) + a.L.oSt); }
// row of the replay bits / trace of inner iteration k of problem b (current outer iteration)
__device__ __forceinline__ size_t rix(const Args& a, int b, int k) {
  return ((size_t)b * a.rep_outer + a.cur_outer) * a.P.max_inner + k;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block sum of NV per-thread partials, added (fp64 atomics) into dst[0..NV)
template <int NV>
__device__ __forceinline__ void block_add(float (&v)[NV], double* dst) {
  __shared__ float red[NV][ENT / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const float s = warp_sum(v[k]);
    if (lane == 0) red[k][wid] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < ENT / 32; ++w) s += red[threadIdx.x][w];
    atomicAdd(dst + threadIdx.x, s);
  }
}

// element loop of an elementwise kernel: CTA blockIdx.x covers ENT*EPT consecutive plane entries
__device__ __forceinline__ size_t elems_end(size_t pl) {
  const size_t e = (size_t)(blockIdx.x + 1) * ENT * EPT;
  return e < pl ? e : pl;
}
#define FOR_ELEMS(pl) \
  for (size_t idx = (size_t)blockIdx.x * ENT * EPT + threadIdx.x, end_ = elems_end(pl); idx < end_; idx += ENT)

__device__ __forceinline__ void load_s(const double* acc, int p, float (&s)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = q < p ? (float)acc[q] : 0.f;
}

__device__ __forceinline__ float kdot(const float* K, size_t pl, size_t idx, int p, const float (&s)[8]) {
  float r = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < p) r = fmaf(K[q * pl + idx], s[q], r);
  return r;
}

// ---------------------------------------------------------------------------------------------
// Layout conversion: row-major [m][n] <-> column-major plane (ld), 32 x 32 tiles
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_to_plane(const float* __restrict__ src, int nper, Args a, size_t off) {
  __shared__ float t[32][33];
  const Lay& L = a.L;
  const int z = blockIdx.z, b = z / nper, q = z % nper;
  const float* s = src + ((size_t)b * nper + q) * L.m * L.n;
  float* d = slot(a, b) + off + (size_t)q * L.plane;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    t[r][threadIdx.x] = (i < L.m && j < L.n) ? s[(size_t)i * L.n + j] : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += 8) {
    const int j = j0 + c, i = i0 + threadIdx.x;
    if (i < L.m && j < L.n) d[(size_t)j * L.ldm + i] = t[threadIdx.x][c];
  }
}

// plane -> row-major [m][n] (zeros for problems whose Gram failed when zero_bad)
__global__ void __launch_bounds__(256) k_from_plane(float* __restrict__ dst, Args a, size_t off, int rows, int cols,
                                                    int ld, int zero_bad) {
  __shared__ float t[32][33];
  const int b = blockIdx.z;
  const float* s = slot(a, b) + off;
  const bool z = (zero_bad == 1 && state(a, b)->status == TILT_PATCH_SINGULAR_GRAM) ||
                 (zero_bad == 2 && state(a, b)->outer_iters == 0);
  float* d = dst + (size_t)b * rows * cols;
  const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
  for (int c = threadIdx.y; c < 32; c += 8) {
    const int j = j0 + c, i = i0 + threadIdx.x;
    t[c][threadIdx.x] = (i < rows && j < cols && !z) ? s[(size_t)j * ld + i] : 0.f;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < rows && j < cols) d[(size_t)i * cols + j] = t[threadIdx.x][r];
  }
}

// ---------------------------------------------------------------------------------------------
// Projector setup: G = J^T J (fp64), L^{-1} from chol(G + Q^T Q), K = J L^{-T} (Eq. Jperpv
// P:601-606, Eq. WTW_property), as orthonormalise_explicit in tilt_device.cuh
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(ENT) k_gram(Args a) {
  const int b = blockIdx.y;
  if (state(a, b)->outer_done) return;
  const Lay& L = a.L;
  const float* K = slot(a, b) + L.oK;
  double g[36];
#pragma unroll
  for (int e = 0; e < 36; ++e) g[e] = 0.0;
  FOR_ELEMS(L.plane) {
    float j[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) j[q] = q < L.p ? K[q * L.plane + idx] : 0.f;
    int e = 0;
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = x; y < 8; ++y) {
        g[e] = fma((double)j[x], (double)j[y], g[e]);
        ++e;
      }
  }
  __shared__ double red[ENT / 32];
  St* st = state(a, b);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int e = 0; e < 36; ++e) {
    double v = g[e];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < ENT / 32; ++w) s += red[w];
      atomicAdd(&st->acc[ACC_G + e], s);
    }
    __syncthreads();
  }
}

// Q: the caller's rows [B][l][p] (inner entry), or st->Q (l = 3, solve entry) when q_state
__global__ void k_chol(Args a, const float* __restrict__ Q, int l, int q_state) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->outer_done) return;
  double qr[24];
  for (int e = 0; e < 24; ++e) qr[e] = q_state ? st->Q[e] : 0.0;
  if (Q && !q_state)
    for (int r = 0; r < l; ++r)
      for (int q = 0; q < a.L.p; ++q) qr[r * 8 + q] = Q[((size_t)b * l + r) * a.L.p + q];
  const bool ok = chol_inverse(st->acc + ACC_G, qr, (Q || q_state) ? l : 0, a.L.p, st->Linv);
  st->status = ok ? TILT_PATCH_CONVERGED : TILT_PATCH_SINGULAR_GRAM;
  st->done = ok ? 0 : 1;
  if (!ok) st->outer_done = 1;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
}

__global__ void __launch_bounds__(ENT) k_apply_linv(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->status != TILT_PATCH_CONVERGED || st->outer_done) return;
  const Lay& L = a.L;
  float* K = slot(a, b) + L.oK;
  const double* Li = st->Linv;
  FOR_ELEMS(L.plane) {
    double j[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) j[q] = q < L.p ? (double)K[q * L.plane + idx] : 0.0;
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      if (x < L.p) {
        double s = 0.0;
#pragma unroll
        for (int y = 0; y <= x; ++y) s = fma(Li[x * 8 + y], j[y], s);
        K[x * L.plane + idx] = (float)s;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Projector reductions and the elementwise LADMAP steps (ladmap_inner in tilt_kernels.cuh)
// ---------------------------------------------------------------------------------------------
// MODE 0: v = D; 1: v = A + E - D; 2: v = A+ + E - D and ||A+ - A||^2. -> acc[ACC_S1..]
template <int MODE>
__global__ void __launch_bounds__(ENT) k_kt(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  const float* w = slot(a, b);
  const float* D = w + L.oD;
  const float* A = w + L.oA;
  const float* An = w + L.oAn;
  const float* E = w + L.oE;
  const float* K = w + L.oK;
  float s[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) s[q] = 0.f;
  FOR_ELEMS(L.plane) {
    float v;
    if (MODE == 0) {
      v = D[idx];
    } else if (MODE == 1) {
      v = A[idx] + E[idx] - D[idx];
    } else if (MODE == 3) {  // ADM dtau step: v = A + E - D - Y/mu
      v = fmaf(-w[L.oY + idx], 1.f / st->mu, A[idx] + E[idx] - D[idx]);
    } else {
      const float an = An[idx];
      v = an + E[idx] - D[idx];
      const float d = an - A[idx];
      s[8] = fmaf(d, d, s[8]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < L.p) s[q] = fmaf(K[q * L.plane + idx], v, s[q]);
  }
  block_add<9>(s, st->acc + ACC_S1);
}

// ||W^TW D||^2 (the Cond1/Cond2 denominator, Z11)
__global__ void __launch_bounds__(ENT) k_denom(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  const float* w = slot(a, b);
  float s[8];
  load_s(st->acc + ACC_S1, L.p, s);
  float r2[1] = {0.f};
  FOR_ELEMS(L.plane) {
    const float r = w[L.oD + idx] - kdot(w + L.oK, L.plane, idx, L.p, s);
    r2[0] = fmaf(r, r, r2[0]);
  }
  block_add<1>(r2, st->acc + ACC_R);
}

// M_0 = A - W^TW(A + E - D) - Y/mu_0 into S (write_m0)
__global__ void __launch_bounds__(ENT) k_m0(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  float s[8];
  load_s(st->acc + ACC_S1, L.p, s);
  const float inv = 1.f / st->mu;
  FOR_ELEMS(L.plane) {
    const float av = w[L.oA + idx];
    const float v = res3(av, w[L.oE + idx], w[L.oD + idx]);
    const float r = v - kdot(w + L.oK, L.plane, idx, L.p, s);
    w[L.oS + idx] = av - r - w[L.oY + idx] * inv;
  }
}

// E step (Eq. E with erratum E2): N = E - W^TW(A+ + E - D) - Y/mu, E+ = T_{lam/mu}(N); then the
// first half of the dual step: K^T (A+ + E+ - D) -> acc[ACC_S2..], ||E+ - E||^2
__global__ void __launch_bounds__(ENT) k_estep(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  const float* K = w + L.oK;
  float s[8];
  load_s(st->acc + ACC_S1, L.p, s);
  const float inv_mu = 1.f / st->mu;
  const float thr = st->lam * inv_mu;
  float o[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) o[q] = 0.f;
  FOR_ELEMS(L.plane) {
    const float an = w[L.oAn + idx], e = w[L.oE + idx], dv = w[L.oD + idx];
    const float pv = res3(an, e, dv) - kdot(K, L.plane, idx, L.p, s);
    const float nk = e - pv - w[L.oY + idx] * inv_mu;
    const float en = copysignf(fmaxf(fabsf(nk) - thr, 0.f), nk);
    const float d = en - e;
    o[8] = fmaf(d, d, o[8]);
    w[L.oE + idx] = en;
    const float v2 = res3(an, en, dv);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < L.p) o[q] = fmaf(K[q * L.plane + idx], v2, o[q]);
  }
  block_add<9>(o, st->acc + ACC_S2);
}

// dual step (Eq. Y, erratum E1) and the next M: R = W^TW(A+ + E+ - D), Y += mu R,
// S = A+ - R - Y/mu_{k+1}, A = A+, ||R||^2
__global__ void __launch_bounds__(ENT) k_ystep(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  float s[8];
  load_s(st->acc + ACC_S2, L.p, s);
  const float mu = st->mu, inv_mun = 1.f / st->mu_next;
  float c1[1] = {0.f};
  FOR_ELEMS(L.plane) {
    const float an = w[L.oAn + idx];
    const float r = res3(an, w[L.oE + idx], w[L.oD + idx]) - kdot(w + L.oK, L.plane, idx, L.p, s);
    const float y = fmaf(mu, r, w[L.oY + idx]);
    w[L.oY + idx] = y;
    c1[0] = fmaf(r, r, c1[0]);
    w[L.oS + idx] = an - r - y * inv_mun;
    w[L.oA + idx] = an;
  }
  block_add<1>(c1, st->acc + ACC_C1);
}

__global__ void __launch_bounds__(ENT) k_l1(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->status != TILT_PATCH_CONVERGED) return;
  const float* E = slot(a, b) + a.L.oE;
  float s[1] = {0.f};
  FOR_ELEMS(a.L.plane) s[0] += fabsf(E[idx]);
  block_add<1>(s, st->acc + ACC_L1);
}

// ||B||_F^2 of the current SVT (B = M V)
__global__ void __launch_bounds__(ENT) k_fro(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->svt_done) return;
  const float* X = slot(a, b) + a.L.oB;
  float s[1] = {0.f};
  FOR_ELEMS(a.L.plane) s[0] = fmaf(X[idx], X[idx], s[0]);
  block_add<1>(s, &st->fro2);
}

__global__ void __launch_bounds__(ENT) k_copy_plane(Args a, size_t dst, size_t src) {
  const int b = blockIdx.y;
  if (state(a, b)->done) return;
  float* w = slot(a, b);
  FOR_ELEMS(a.L.plane) w[dst + idx] = w[src + idx];
}

// V <- I (n x n, ld = ldn)
__global__ void __launch_bounds__(ENT) k_identity(Args a, size_t off) {
  const int b = blockIdx.y;
  if (state(a, b)->done) return;
  float* V = slot(a, b) + off;
  const int ldn = a.L.ldn, n = a.L.n;
  FOR_ELEMS(a.L.vplane) {
    const int j = (int)(idx / ldn), i = (int)(idx % ldn);
    V[idx] = (i == j && j < n) ? 1.f : 0.f;
  }
}

// T <- 1.5 I - 0.5 T (Newton-Schulz, Z14). Applied to every problem, also those whose inner loop has
// ended: the batched GEMMs around it run for all of them, and skipping this step would turn their
// V <- V (1.5 I - 0.5 V^T V) into V <- V (V^T V), which grows the column norms without bound over
// the remaining iterations of the batch -- and V warm-starts the next outer iteration.
__global__ void __launch_bounds__(ENT) k_ns_mid(Args a) {
  const int b = blockIdx.y;
  float* T = slot(a, b) + a.L.oT;
  const int ldn = a.L.ldn;
  FOR_ELEMS(a.L.vplane) {
    const int j = (int)(idx / ldn), i = (int)(idx % ldn);
    T[idx] = (i == j ? 1.5f : 0.f) - 0.5f * T[idx];
  }
}

// ---------------------------------------------------------------------------------------------
// Per-problem scalar steps (one thread per problem)
// ---------------------------------------------------------------------------------------------
__global__ void k_init(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  const int m = a.L.m, n = a.L.n;
  st->lam = a.P.lambda > 0.f ? a.P.lambda : rsqrtf((float)max(m, n));
  st->iters = st->sweeps = st->caps = st->rotations = st->aux_sweeps = 0;
  st->conv = 0;
  st->crit1 = st->crit2 = __int_as_float(0x7fc00000);
  st->nuc = 0.f;
  st->svt_rank = st->relrank = st->band = 0;
}

__global__ void k_sc_denom(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  const float d0 = (float)sqrt(st->acc[ACC_R]);
  st->denom0 = d0;
  st->denom = d0 > 0.f ? d0 : 1.f;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
}

// mu_0 = mu0_scale / sigma_1(D) (Z3) after the sigma_1 SVD; mu_max = ratio mu_0 (Z6)
__global__ void k_sc_mu0(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  const float s1 = st->sig1;
  st->mu0 = s1 > 0.f ? a.P.mu0_scale / s1 : a.P.mu0_scale;
  st->mu = st->mu0;
  st->mu_max = a.P.mu_max_ratio * st->mu0;
  st->aux_sweeps += st->sw_cur;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
}

// Cond2 and the penalty update (Eqs. rho, mu; replay Z21)
__global__ void k_sc1(Args a, int k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  const float dA = (float)st->acc[ACC_DA], dE = (float)st->acc[ACC_DE];
  const float crit2 = st->mu * sqrtf(fmaxf(dA, dE)) / st->denom;
  int rho_bit = crit2 < a.P.eps2 ? 1 : 0;
  if (a.P.rho_replay) rho_bit = a.P.rho_replay[rix(a, b, k)] & 1;
  st->mu_next = fminf(st->mu_max, rho_bit ? a.P.rho0 * st->mu : st->mu);
  st->crit2 = crit2;
  if (a.P.trace) a.P.trace[4 * (rix(a, b, k)) + 3] = (float)(rho_bit + 2 * st->warm);  // + Alg. 2 step
}

// Cond1, the stop rule (strict), mu <- mu_{k+1}
__global__ void k_sc2(Args a, int k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  const float crit1 = (float)sqrt(st->acc[ACC_C1]) / st->denom;
  if (a.P.trace) {
    float* t = a.P.trace + 4 * (rix(a, b, k));
    t[0] = st->mu;
    t[1] = crit1;
    t[2] = st->crit2;
  }
  st->crit1 = crit1;
  st->iters = k + 1;
  bool stop = crit1 < a.P.eps1 && st->crit2 < a.P.eps2;
  if (a.P.rho_replay) stop = (a.P.rho_replay[rix(a, b, k)] & 2) != 0;
  if (stop) st->conv = 1;
  const float mu_used = st->mu;
  st->mu = st->mu_next;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
  if ((stop && a.P.fixed_inner <= 0) || k + 1 >= a.niter) {
    st->done = 1;
    st->mu = mu_used;  // report mu_K of the last SVT
  } else {
    atomicAdd(a.counter, 1);
  }
}

__global__ void k_report(Args a, tilt_report* rep) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  tilt_report r;
  memset(&r, 0, sizeof(r));
  r.status = st->status;
  if (st->status == TILT_PATCH_CONVERGED) {
    r.status = st->conv ? TILT_PATCH_CONVERGED : TILT_PATCH_MAX_OUTER;
    r.outer_iters = 1;
    r.inner_iters = st->iters;
    r.jacobi_sweeps = st->sweeps;
    r.aux_sweeps = st->aux_sweeps;
    r.rank = st->relrank;
    r.rank_band = st->band;
    r.svt_rank = st->svt_rank;
    r.sweep_cap_hits = st->caps;
    r.objective = st->nuc + st->lam * (float)st->acc[ACC_L1];
    r.crit1 = st->crit1;
    r.crit2 = st->crit2;
    r.patch_norm = st->denom0;
    r.mu_last = st->mu;
    r.jacobi_rotations = st->rotations;
    r.kernel_path = 3;
    r.svd_warm_steps = st->warm_steps;
  }
  rep[b] = r;
}

// ---------------------------------------------------------------------------------------------
// SVT pieces
// ---------------------------------------------------------------------------------------------
// eps_mode 0: eps = 1/mu (LADMAP), 1: eps from the caller's array, 2: eps = 0 (sigma_1 SVD)
__global__ void k_svt_begin(Args a, const float* __restrict__ eps, int eps_mode) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  st->svt_done = st->done || st->warm;  // a warm-step problem (Alg. 2) skips the Jacobi sweeps
  st->big_any = st->rot_any = 0;
  st->sw_cur = st->cap_cur = st->rot_cur = 0;
  st->fro2 = 0.0;
  if (st->done) return;
  st->eps = eps_mode == 0 ? 1.f / st->mu : (eps_mode == 1 ? eps[b] : 0.f);
  if (!st->svt_done) atomicAdd(a.counter, 1);
}

// Loop condition of the device-side sweep loop (a WHILE node of the sweep graph): another sweep
// while any problem's SVT is still running; counter[8] tallies the sweeps run (launch accounting)
__global__ void k_sweep_cond(const int* counter, int* tally, cudaGraphConditionalHandle h) {
  *tally += 1;
  cudaGraphSetConditional(h, counter[0] > 0 ? 1u : 0u);
}

__global__ void k_sweep_end(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->svt_done) return;
  st->sw_cur += 1;
  if (!st->big_any) {
    st->svt_done = 1;
  } else if (st->sw_cur >= a.max_sweeps) {
    st->svt_done = 1;
    st->cap_cur = st->rot_any;
  }
  st->big_any = st->rot_any = 0;
  if (!st->svt_done) atomicAdd(a.counter, 1);
}

// sigma_j = ||b_j|| / ||v_j||, ||v_j||^2 (one warp per column)
__global__ void __launch_bounds__(256) k_svt_sig(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || st->warm) return;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= a.L.n) return;
  const float* w = slot(a, b);
  const float* bj = w + a.L.oB + (size_t)j * a.L.ldm;
  const float* vj = w + a.oV + (size_t)j * a.L.ldn;
  float sb = 0.f, sv = 0.f;
  for (int i = lane; i < a.L.m; i += 32) sb = fmaf(bj[i], bj[i], sb);
  for (int i = lane; i < a.L.n; i += 32) sv = fmaf(vj[i], vj[i], sv);
  sb = warp_sum(sb);
  sv = warp_sum(sv);
  if (lane == 0) {
    float* sig = slot(a, b) + a.L.oSig;
    float* vv = slot(a, b) + a.L.oVv;
    sig[j] = sv > 0.f ? sqrtf(sb / sv) : 0.f;
    vv[j] = sv;
  }
}

// SVT statistics (svt_stats in tilt_device.cuh): ||A||_*, sigma_1, #{sigma > eps}, the Z19 rank and
// band flag; one warp per problem. Also folds the sweep counters into the totals.
// which: 0 = problems of the Jacobi SVT, 1 = problems of the Alg. 2 warm step (sig holds |Sigma|)
__global__ void __launch_bounds__(32) k_svt_stats(Args a, int count_sweeps, int which = 0) {
  const int b = blockIdx.x;
  St* st = state(a, b);
  if (st->done || st->warm != which) return;
  const float* sig = slot(a, b) + a.L.oSig;
  const float eps = st->eps;
  const int lane = threadIdx.x, n = a.L.n;
  float nuc = 0.f, smax = 0.f, amax = 0.f;
  int cnt = 0;
  for (int j = lane; j < n; j += 32) {
    const float sg = sig[j];
    const float x = fmaxf(sg - eps, 0.f);
    nuc += x;
    smax = fmaxf(smax, sg);
    amax = fmaxf(amax, x);
    cnt += (sg > eps);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    nuc += __shfl_xor_sync(0xffffffffu, nuc, off);
    smax = fmaxf(smax, __shfl_xor_sync(0xffffffffu, smax, off));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
  }
  int rel = 0, band = 0;
  for (int j = lane; j < n; j += 32) {
    const float x = fmaxf(sig[j] - eps, 0.f);
    if (amax > 0.f) {
      const float ratio = x / amax;
      rel += ratio > 1e-3f;
      band |= (ratio >= 3e-4f && ratio <= 3e-3f);
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    rel += __shfl_xor_sync(0xffffffffu, rel, off);
    band |= __shfl_xor_sync(0xffffffffu, band, off);
  }
  if (lane == 0) {
    st->nuc = nuc;
    st->sig1 = smax;
    st->svt_rank = cnt;
    st->relrank = rel;
    st->band = band;
    if (count_sweeps) {
      st->sweeps += st->sw_cur;
      st->caps += st->cap_cur ? 1 : 0;
      st->rotations += st->rot_cur;
    }
  }
}

// B <- B diag(h_j / ||v_j||^2), h_j = max(sigma_j - eps, 0) / sigma_j (ready for A = B V^T)
__global__ void __launch_bounds__(ENT) k_svt_scale(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || st->warm) return;
  float* w = slot(a, b);
  const float* sig = w + a.L.oSig;
  const float* vv = w + a.L.oVv;
  const float eps = st->eps;
  const int ldm = a.L.ldm;
  FOR_ELEMS(a.L.plane) {
    const int j = (int)(idx / ldm);
    if (j >= a.L.n) continue;
    const float sg = sig[j], v2 = vv[j];
    const float h = sg > eps ? (sg - eps) / sg : 0.f;
    w[a.L.oB + idx] *= v2 > 0.f ? h / v2 : 0.f;
  }
}


// ---------------------------------------------------------------------------------------------
// One Jacobi round over a block pair (CROSS) or within one block (intra): see the header.
// Shared memory: X [NCOL][MAXD] (the columns, rows >= m zero), W [NCOL][NCOL] (column-major),
// ns [NCOL] (alpha, d, 1/d, -) of the fast rotations (tilt_jacobi.cuh).
// ---------------------------------------------------------------------------------------------
template <int RPL, int CROSS>
__global__ void __launch_bounds__(RNT, RPL <= 8 ? 2 : 1) k_round(Args a, int r) {  // 2 CTAs/SM up to 256 rows
  constexpr int MAXD = 32 * RPL;
  constexpr int NCOL = CROSS ? 2 * BW : BW;
  extern __shared__ float4 sm4[];
  float* X = reinterpret_cast<float*>(sm4);
  float* W = X + NCOL * MAXD;
  float4* ns = reinterpret_cast<float4*>(W + NCOL * NCOL);
  __shared__ int s_any, s_big, s_cnt;
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->svt_done) return;
  const Lay& L = a.L;
  int I, J = -1;
  if (CROSS) {
    const int q = a.NBp - 1, k = blockIdx.x;
    I = k == 0 ? q : (r + k) % q;
    J = k == 0 ? r : (r - k + q) % q;
    if (I >= a.NB || J >= a.NB) return;  // the dummy block
  } else {
    I = blockIdx.x;
  }
  const int nI = min(BW, L.n - I * BW), nJ = CROSS ? min(BW, L.n - J * BW) : 0;
  // valid local columns as a bit mask; global column of local c: c + (c < BW ? gI : gJ)
  const uint32_t vmask = ((1u << nI) - 1u) | (CROSS ? ((1u << nJ) - 1u) << BW : 0u);
  const int gI = I * BW, gJ = J * BW - BW;
  auto gcol = [&](int c) { return c + (c < BW ? gI : gJ); };
  auto cvalid = [&](int c) { return ((vmask >> c) & 1u) != 0u; };
  float* w = slot(a, b);
  float* Bm = w + L.oB;
  float* V = w + a.oV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_any = s_big = s_cnt = 0;
  // stage the columns (float4; rows >= ldm zero), W = I
  constexpr int C4 = MAXD / 4;
  // cp.async (16 B per request, all in flight at once; src-size 0 zero-fills the padding)
  for (int e = tid; e < NCOL * C4; e += RNT) {
    const int c = e / C4, i4 = e % C4;
    const bool in = cvalid(c) && 4 * i4 < L.ldm;
    const float* src = in ? Bm + (size_t)gcol(c) * L.ldm + 4 * i4 : Bm;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(sm4 + e)), "l"(src),
                 "r"(in ? 16 : 0)
                 : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  for (int e = tid; e < NCOL * NCOL; e += RNT) W[e] = (e / NCOL == e % NCOL) ? 1.f : 0.f;
  __syncthreads();
  using CL = Col<RPL, 32>;
  const uint32_t sX = smem_u32(X);
  for (int c = warp; c < NCOL; c += RNT / 32) {  // fresh norms, d = 1
    CL x;
    x.sload_full(sX + c * MAXD * 4 + lane * 16);
    const float ss = unit_sum<32>(x.sq());
    if (lane == 0) ns[c] = make_float4(ss, 1.f, 1.f, 0.f);
  }
  __syncthreads();
  const float tol2 = a.tol * a.tol, big2 = a.big2;
  const float amin = (float)(a.tiny2 * st->fro2);
  int rot = 0, big = 0, cnt = 0;
  // one rotation of local columns (i, j) with x_i, x_j, their states and W entries in registers
  auto rotate = [&](CL& xi, CL& xj, float4& ni, float4& nj, float& wi, float& wj) -> bool {
    const float g = unit_sum<32>(xi.dot(xj));
    const float gam = g * ni.y * nj.y;
    const float ab = ni.x * nj.x;
    const bool doit = ni.x > amin && nj.x > amin && gam * gam > tol2 * ab;
    if (doit) {  // warp-uniform
      const Rot rp = rot_params(ni, nj, gam, true);
      CL::rotate(xi, xj, rp.ca, rp.cb);
      const float w0 = wi;
      wi = fmaf(-rp.ca, wj, w0);
      wj = fmaf(rp.cb, w0, wj);
      const float sx = rp.c * fmaf(rp.t, rp.t, 1.f);  // sqrt(1 + t^2)
      ni = make_float4(fmaxf(fmaf(-rp.t, gam, ni.x), 0.f), rp.c * ni.y, sx * ni.z, 0.f);
      nj = make_float4(fmaf(rp.t, gam, nj.x), rp.c * nj.y, sx * nj.z, 0.f);
      rot = 1;
      cnt += 1;
      big |= gam * gam > big2 * ab ? 1 : 0;
    }
    return doit;
  };
  if constexpr (CROSS) {
    // warp w keeps column w of block I (x, state, its W column entry) in registers for all 16
    // steps; step s pairs it with column BW + (w + s) % BW of block J, loaded from shared memory
    const int i = warp;
    const bool vi = cvalid(i);
    const uint32_t ai = sX + i * MAXD * 4 + lane * 16;
    CL xi;
    xi.sload_full(ai);
    float4 ni = ns[i];
    float wi = W[i * NCOL + lane];
    for (int s = 0; s < BW; ++s) {
      const int j = BW + ((warp + s) & (BW - 1));
      if (vi && cvalid(j)) {  // warp-uniform
        const uint32_t aj = sX + j * MAXD * 4 + lane * 16;
        CL xj;
        xj.sload_full(aj);
        float4 nj = ns[j];
        float wj = W[j * NCOL + lane];
        if (rotate(xi, xj, ni, nj, wi, wj)) {
          xj.sstore(aj, 0xffffffffu);
          W[j * NCOL + lane] = wj;
          if (lane == 0) ns[j] = nj;
        }
      }
      __syncthreads();
    }
    if (vi) {
      xi.sstore(ai, 0xffffffffu);
      W[i * NCOL + lane] = wi;
      if (lane == 0) ns[i] = ni;
    }
  } else {
    for (int s = 0; s < BW - 1; ++s) {  // circle method on the block's BW columns, BW/2 warps
      const int q = BW - 1, k = warp;
      const bool on = k < BW / 2;
      const int i = on ? (k == 0 ? q : (s + k) % q) : 0;
      const int j = on ? (k == 0 ? s : (s - k + q) % q) : 0;
      if (on && cvalid(i) && cvalid(j)) {  // warp-uniform
        CL xi, xj;
        const uint32_t ai = sX + i * MAXD * 4 + lane * 16, aj = sX + j * MAXD * 4 + lane * 16;
        xi.sload_full(ai);
        xj.sload_full(aj);
        float4 ni = ns[i], nj = ns[j];
        float wi = lane < NCOL ? W[i * NCOL + lane] : 0.f, wj = lane < NCOL ? W[j * NCOL + lane] : 0.f;
        if (rotate(xi, xj, ni, nj, wi, wj)) {
          xi.sstore(ai, 0xffffffffu);
          xj.sstore(aj, 0xffffffffu);
          if (lane < NCOL) {
            W[i * NCOL + lane] = wi;
            W[j * NCOL + lane] = wj;
          }
          if (lane == 0) {
            ns[i] = ni;
            ns[j] = nj;
          }
        }
      }
      __syncthreads();
    }
  }
  if (lane == 0 && rot) {
    atomicOr(&s_any, 1);
    atomicAdd(&s_cnt, cnt);
  }
  if (lane == 0 && big) atomicOr(&s_big, 1);
  __syncthreads();
  if (!s_any) return;  // nothing rotated: B and V unchanged
  if (tid == 0) {
    atomicOr(&st->rot_any, 1);
    if (s_big) atomicOr(&st->big_any, 1);
    atomicAdd(&st->rot_cur, s_cnt);
  }
  // apply the scales d_c: B columns = d_c x_c, W_eff[:, c] = d_c W[:, c]
  for (int e = tid; e < NCOL * C4; e += RNT) {
    const int c = e / C4, i4 = e % C4;
    if (!cvalid(c) || 4 * i4 >= L.ldm) continue;
    const float d = ns[c].y;
    float4 v = sm4[e];
    v.x *= d; v.y *= d; v.z *= d; v.w *= d;
    *reinterpret_cast<float4*>(Bm + (size_t)gcol(c) * L.ldm + 4 * i4) = v;
  }
  for (int e = tid; e < NCOL * NCOL; e += RNT) W[e] *= ns[e / NCOL].y;
  __syncthreads();
  // V[:, cols] <- V[:, cols] W_eff: two threads per row, each forming HALF of the NCOL outputs from
  // the row's inputs in chunks of 8 (at most ~40 live registers, so two 512-thread CTAs fit an SM).
  // Thread tid: row r0 + tid % (RNT / 2), half tid / (RNT / 2), so a warp reads one W row at a time
  // (a broadcast, no bank conflict between the halves); both halves of a row are in the same pass and
  // all inputs are read before the CTA barrier, then written.
  constexpr int HALF = NCOL / 2;
  for (int r0 = 0; r0 < L.n; r0 += RNT / 2) {
    const int h = tid / (RNT / 2), row = r0 + (tid & (RNT / 2 - 1));
    const bool on = row < L.n;
    float o[HALF];
#pragma unroll
    for (int q = 0; q < HALF; ++q) o[q] = 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < NCOL; c0 += 8) {
      const float* vc = V + (size_t)(c0 + (c0 < BW ? gI : gJ)) * L.ldn + row;
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = (on && cvalid(c0 + u)) ? vc[(size_t)u * L.ldn] : 0.f;
#pragma unroll
      for (int q = 0; q < HALF; ++q) {
        const float4 w0 = *reinterpret_cast<const float4*>(W + (h * HALF + q) * NCOL + c0);
        const float4 w1 = *reinterpret_cast<const float4*>(W + (h * HALF + q) * NCOL + c0 + 4);
        o[q] = fmaf(v[0], w0.x, o[q]);
        o[q] = fmaf(v[1], w0.y, o[q]);
        o[q] = fmaf(v[2], w0.z, o[q]);
        o[q] = fmaf(v[3], w0.w, o[q]);
        o[q] = fmaf(v[4], w1.x, o[q]);
        o[q] = fmaf(v[5], w1.y, o[q]);
        o[q] = fmaf(v[6], w1.z, o[q]);
        o[q] = fmaf(v[7], w1.w, o[q]);
      }
    }
    __syncthreads();  // every thread read its inputs before the other half of its row is overwritten
    if (on) {
      float* vo = V + (size_t)(h * HALF + (h * HALF < BW ? gI : gJ)) * L.ldn + row;
#pragma unroll
      for (int q = 0; q < HALF; ++q)
        if (cvalid(h * HALF + q)) vo[(size_t)q * L.ldn] = o[q];
    }
  }
}

// ---------------------------------------------------------------------------------------------
// SVD warm start (Algorithm 2; Appendix A; oracle.svd_warm_start): for a
// problem whose M_k is within eps_svd of M_{k-1}, one Taylor step along the Cayley curve from the
// previous SVD (U, Sigma, V) replaces the Jacobi SVT:
//   W = U Sigma V^T, P_U = W M^T - M W^T, P_V = W^T M - M^T W, P_Sigma = Sigma - diag(U^T M V),
//   h1 = P_U W + U P_Sigma V^T - W P_V, Z = h1 + U P_Sigma V^T, h2 = -P_U Z + Z P_V,
//   t* = -<h0, h1> / (||h1||^2 + <h0, h2>), h0 = M - W,
//   U <- (I + t/2 P_U)^{-1} (I - t/2 P_U) U, Sigma <- Sigma - t P_Sigma, V likewise with P_V,
// then A = U T_eps(Sigma) V^T. The products run in the hand-written batched GEMM (tilt_dense.cuh)
// on the gated problems only; each Cayley system is solved exactly, as printed, for any t*:
// X(t) = (I + S)^{-1} (I - S) X = 2 (I + S)^{-1} X - X with S = (t*/2) P skew, by the blocked LU of
// I + S (no pivoting needed: its symmetric part is I) and two triangular solves. The only rejected
// step is f''(0) <= 0, where the quadratic model of Eq. ft has no minimiser (reading Z27).
// ---------------------------------------------------------------------------------------------
// dst = src diag(vec) (mode 0), src diag(T_eps(vec)) (mode 1); problems with st->warm == want
__global__ void __launch_bounds__(ENT) k_colscale(Args a, size_t dst, size_t src, size_t vec, int mode, int want) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || st->warm != want) return;
  float* w = slot(a, b);
  const int ldm = a.L.ldm;
  const float eps = st->eps;
  FOR_ELEMS(a.L.plane) {
    const int j = (int)(idx / ldm);
    float f = j < a.L.n ? w[vec + j] : 0.f;
    if (mode == 1) f = copysignf(fmaxf(fabsf(f) - eps, 0.f), f);
    w[dst + idx] = w[src + idx] * f;
  }
}

// plane copy (count floats) for problems with st->warm == want (want < 0: every active problem)
__global__ void __launch_bounds__(ENT) k_copy_if(Args a, size_t dst, size_t src, size_t count, int want) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || (want >= 0 && st->warm != want)) return;
  float* w = slot(a, b);
  FOR_ELEMS(count) w[dst + idx] = w[src + idx];
}

// X <- X - X^T in place (an n x n block, leading dimension ld): the skew part of Eqs.
// projected_gradient1-2; scale_t: X <- I + (t*/2) X (the Cayley system matrix)
__global__ void __launch_bounds__(ENT) k_skew(Args a, size_t off, int nn, int ld, int scale_t) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  float* X = slot(a, b) + off;
  const float f = scale_t ? 0.5f * st->t_star : 1.f;
  FOR_ELEMS((size_t)nn * nn) {
    const int j = (int)(idx / nn), i = (int)(idx % nn);
    if (scale_t) {
      X[(size_t)j * ld + i] = fmaf(f, X[(size_t)j * ld + i], i == j ? 1.f : 0.f);
    } else if (i < j) {
      const float x = X[(size_t)j * ld + i], y = X[(size_t)i * ld + j];
      X[(size_t)j * ld + i] = x - y;
      X[(size_t)i * ld + j] = y - x;
    } else if (i == j) {
      X[(size_t)j * ld + i] = 0.f;
    }
  }
}

// X <- 2 T - X (the Cayley point from T = (I + S)^{-1} X)
__global__ void __launch_bounds__(ENT) k_cay_finish(Args a, size_t oX, size_t oT, size_t count) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  float* w = slot(a, b);
  FOR_ELEMS(count) w[oX + idx] = fmaf(2.f, w[oT + idx], -w[oX + idx]);
}

// ||M - M_prev||_F^2 (the gate of Alg. 2)
__global__ void __launch_bounds__(ENT) k_ws_diff(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->have_prev) return;
  const float* w = slot(a, b);
  float s[1] = {0.f};
  FOR_ELEMS(a.L.plane) {
    const float d = w[a.L.oS + idx] - w[a.L.oMp + idx];
    s[0] = fmaf(d, d, s[0]);
  }
  block_add<1>(s, st->wacc);
}

// gate: warm iff ||M_k - M_{k-1}||_F < eps_svd (replay bit 2 overrides, reading Z21's protocol)
__global__ void k_ws_gate(Args a, int k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  st->warm = 0;
  if (st->done || !st->have_prev) return;
  bool w = sqrt(st->wacc[0]) < (double)st->eps_svd;
  if (a.P.rho_replay) w = (a.P.rho_replay[rix(a, b, k)] & 4) != 0;
  for (int e = 0; e < 8; ++e) st->wacc[e] = 0.0;
  st->eps = 1.f / st->mu;
  if (w) {
    st->warm = 1;
    atomicAdd(a.counter + 1, 1);
  }
}

// P_Sigma_j = Sigma_j - u_j . (M V)_j (one warp per column; M V in H2)
__global__ void __launch_bounds__(256) k_ws_psig(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= a.L.n) return;
  float* w = slot(a, b);
  const float* u = w + a.L.oU + (size_t)j * a.L.ldm;
  const float* mv = w + a.L.oH2 + (size_t)j * a.L.ldm;
  float s = 0.f;
  for (int i = lane; i < a.L.m; i += 32) s = fmaf(u[i], mv[i], s);
  s = warp_sum(s);
  if (lane == 0) w[a.L.oPs + j] = w[a.L.oSg + j] - s;
}

// Z <- H1 + Z (Z holds U P_Sigma V^T)
__global__ void __launch_bounds__(ENT) k_ws_z(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  float* w = slot(a, b);
  FOR_ELEMS(a.L.plane) w[a.L.oZ + idx] += w[a.L.oH1 + idx];
}

// <h0, h1>, ||h1||^2, <h0, h2> with h0 = M - W
__global__ void __launch_bounds__(ENT) k_ws_red(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  const float* w = slot(a, b);
  float s[3] = {0.f, 0.f, 0.f};
  FOR_ELEMS(a.L.plane) {
    const float h0 = w[a.L.oS + idx] - w[a.L.oW + idx];
    const float h1 = w[a.L.oH1 + idx], h2 = w[a.L.oH2 + idx];
    s[0] = fmaf(h0, h1, s[0]);
    s[1] = fmaf(h1, h1, s[1]);
    s[2] = fmaf(h0, h2, s[2]);
  }
  block_add<3>(s, st->wacc + 1);
}

// t* = -f'(0)/f''(0) (Eq. ft); f''(0) <= 0 (no minimiser of the quadratic model) rejects the step
// for a full SVD (reading Z27)
__global__ void k_ws_t(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  const double f1 = st->wacc[1], f2 = st->wacc[2] + st->wacc[3];
  const double t = f2 > 0.0 ? -f1 / f2 : 0.0;
  st->t_star = (float)t;
  if (!(f2 > 0.0) || t == 0.0) {
    st->warm = 0;
    return;
  }
  atomicAdd(a.counter + 1, 1);
}

// Sigma <- Sigma - t P_Sigma; |Sigma| for the statistics; count the warm step
__global__ void k_ws_sigma(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || !st->warm) return;
  float* w = slot(a, b);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < a.L.n) {
    const float sg = w[a.L.oSg + j] - st->t_star * w[a.L.oPs + j];
    w[a.L.oSg + j] = sg;
    w[a.L.oSig + j] = fabsf(sg);
  }
  if (j == 0) st->warm_steps += 1;
}

// state of a full SVD (Jacobi problems): U_j = b_j / ||b_j||, Sigma_j = sigma_j (before the scale)
__global__ void __launch_bounds__(256) k_ws_state(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done || st->warm) return;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= a.L.n) return;
  float* w = slot(a, b);
  const float* bj = w + a.L.oB + (size_t)j * a.L.ldm;
  float* uj = w + a.L.oU + (size_t)j * a.L.ldm;
  float s = 0.f;
  for (int i = lane; i < a.L.m; i += 32) s = fmaf(bj[i], bj[i], s);
  s = warp_sum(s);
  const float inv = s > 0.f ? rsqrtf(s) : 0.f;
  for (int i = lane; i < a.L.m; i += 32) uj[i] = bj[i] * inv;
  if (lane == 0) w[a.L.oSg + j] = w[a.L.oSig + j];
}

// after the SVT: M_prev <- M for the next gate
__global__ void __launch_bounds__(ENT) k_ws_after(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  float* w = slot(a, b);
  FOR_ELEMS(a.L.plane) w[a.L.oMp + idx] = w[a.L.oS + idx];
  if (blockIdx.x == 0 && threadIdx.x == 0) st->have_prev = 1;
}

__global__ void k_ws_init(Args a, float gate) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  // eps_svd = gate ||D||_F (the oracle's SvdWarm takes the absolute threshold); every inner loop
  // starts with full SVDs (a fresh oracle SvdWarm per LADMAP call)
  st->eps_svd = gate * (float)sqrt(st->acc[ACC_R + 2]);
  st->warm = 0;
  st->have_prev = 0;
}

__global__ void __launch_bounds__(ENT) k_dnorm(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  const float* D = slot(a, b) + a.L.oD;
  float s[1] = {0.f};
  FOR_ELEMS(a.L.plane) s[0] = fmaf(D[idx], D[idx], s[0]);
  block_add<1>(s, st->acc + ACC_R + 2);
}

// the problems taking the Alg. 2 step (order irrelevant: every problem's GEMMs are independent)
__global__ void k_ws_index(Args a, int* widx) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const St* st = state(a, b);
  if (!st->done && st->warm) widx[atomicAdd(a.counter + 3, 1)] = b;
}

// ---------------------------------------------------------------------------------------------
// ADM baseline (adm_inner in tilt_kernels.cuh, reading Z24) on the multi-CTA path:
//   A = S_{1/mu}(D + J dtau - E + Y/mu), E = T_{lam/mu}(D + J dtau - A + Y/mu),
//   J dtau = K K^T (A + E - D - Y/mu), Y += mu (D + J dtau - A - E), mu *= rho;
//   stop at ||D + J dtau - A - E||_F / ||D||_F < adm_tol. J dtau lives in the An plane.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(ENT) k_adm_m(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  const float inv_mu = 1.f / st->mu;
  FOR_ELEMS(L.plane) w[L.oS + idx] = fmaf(w[L.oY + idx], inv_mu, w[L.oD + idx] + w[L.oAn + idx] - w[L.oE + idx]);
}

__global__ void __launch_bounds__(ENT) k_adm_e(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  const float inv_mu = 1.f / st->mu, thr = st->lam * inv_mu;
  FOR_ELEMS(L.plane) {
    const float x = fmaf(w[L.oY + idx], inv_mu, w[L.oD + idx] + w[L.oAn + idx] - w[L.oA + idx]);
    w[L.oE + idx] = copysignf(fmaxf(fabsf(x) - thr, 0.f), x);
  }
}

__global__ void __launch_bounds__(ENT) k_adm_y(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  float s[8];
  load_s(st->acc + ACC_S1, L.p, s);
  const float mu = st->mu;
  float r2[1] = {0.f};
  FOR_ELEMS(L.plane) {
    const float jdt = kdot(w + L.oK, L.plane, idx, L.p, s);
    w[L.oAn + idx] = jdt;
    const float r = w[L.oD + idx] + jdt - w[L.oA + idx] - w[L.oE + idx];
    w[L.oY + idx] = fmaf(mu, r, w[L.oY + idx]);
    r2[0] = fmaf(r, r, r2[0]);
  }
  block_add<1>(r2, st->acc + ACC_C1);
}

__global__ void k_adm_init(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  const double nd2 = st->acc[ACC_R + 2];
  st->inv_nd = nd2 > 0.0 ? (float)(1.0 / sqrt(nd2)) : 1.f;
}

__global__ void k_adm_sc(Args a, int k) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  const float resid = (float)sqrt(st->acc[ACC_C1]) * st->inv_nd;
  if (a.P.trace) {
    float* t = a.P.trace + 4 * (rix(a, b, k));
    t[0] = st->mu;
    t[1] = resid;
    t[2] = 0.f;
    t[3] = 0.f;
  }
  st->crit1 = resid;
  st->iters = k + 1;
  const float mu_used = st->mu;
  st->mu *= a.P.adm_rho;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
  const bool stop = resid < a.P.adm_tol;
  if (stop) st->conv = 1;
  if ((stop && a.P.fixed_inner <= 0) || k + 1 >= a.niter) {
    st->done = 1;
    st->mu = mu_used;
  } else {
    atomicAdd(a.counter, 1);
  }
}

// ---------------------------------------------------------------------------------------------
// Algorithm 1 on the multi-CTA path (tilt_solve_batch, windows above 256; solve_patch in
// tilt_kernels.cuh is the CTA-per-patch version of the same steps)
// ---------------------------------------------------------------------------------------------
__global__ void k_solve_init(Args a, const float* __restrict__ tau0) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  const int p = a.L.p;
  for (int q = 0; q < 8; ++q) st->tau[q] = 0.0;
  if (tau0) {
    for (int q = 0; q < p; ++q) st->tau[q] = tau0[(size_t)b * p + q];
  } else {
    st->tau[0] = 1.0;
    st->tau[3] = 1.0;
  }
  st->status = TILT_PATCH_MAX_OUTER;
  st->stop_rule = 0;
  st->f = st->f_prev = st->dtau_inf = st->nd = __int_as_float(0x7fc00000);
  if (a.boxes[4 * b + 2] != a.L.n || a.boxes[4 * b + 3] != a.L.m) {  // every box has the call's size
    st->status = TILT_PATCH_BAD_BOX;
    st->outer_done = 1;
    st->done = 1;
  }
}

// Step 1 (Z2, Z15, Z16), pass 1: d, gx, gy, gz per pixel (fp64 geometry, the CTA
// kernel's warp_pixel) into D and K[0..2]; sums of d^2 and J_raw^T d; window escape
__global__ void __launch_bounds__(ENT) k_lwarp(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->outer_done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  const int bx[4] = {a.boxes[4 * b], a.boxes[4 * b + 1], a.boxes[4 * b + 2], a.boxes[4 * b + 3]};
  const WarpGeom g = make_geom(bx, st->tau, a.kind);
  const float* img = a.images + (size_t)a.patch_image[b] * a.H * a.W;
  const double ci = 0.5 * (L.m - 1), cj = 0.5 * (L.n - 1), inv_s = 1.0 / g.s;
  const bool homog = a.kind == TILT_HOMOGRAPHY;
  float acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.f;
  int esc = 0;
  FOR_ELEMS(L.plane) {
    const int j = (int)(idx / L.ldm), i = (int)(idx % L.ldm);
    if (i >= L.m || j >= L.n) continue;
    double d, gx, gy, gz;
    if (!warp_pixel(g, img, a.H, a.W, i, j, d, gx, gy, gz)) esc = 1;
    const float df = (float)d, gxf = (float)gx, gyf = (float)gy, gzf = (float)gz;
    w[L.oD + idx] = df;
    w[L.oK + idx] = gxf;
    w[L.oK + L.plane + idx] = gyf;
    w[L.oK + 2 * L.plane + idx] = gzf;
    double jr[8];
    jraw_row(gxf, gyf, homog ? (double)gzf : 0.0, ((double)j - cj) * inv_s, ((double)i - ci) * inv_s, jr);
    acc[8] = fmaf(df, df, acc[8]);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fmaf((float)jr[q], df, acc[q]);
  }
  if (__syncthreads_or(esc) && threadIdx.x == 0) atomicOr(&st->esc, 1);
  block_add<9>(acc, st->acc);
}

// Step 1 status: ||D o tau||, escape / zero patch (these end the problem, as in solve_patch)
__global__ void k_lwarp_status(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->outer_done) return;
  const double nd = sqrt(st->acc[8]);
  st->nd = (float)nd;
  if (st->esc) {
    st->status = TILT_PATCH_WINDOW_ESCAPE;
    st->outer_done = 1;
  } else if (!(nd > 0.0)) {
    st->status = TILT_PATCH_ZERO_PATCH;
    st->outer_done = 1;
  } else {
    for (int q = 0; q < 8; ++q) st->Linv[q] = st->acc[q] / nd;  // c = D_hat^T J_raw (Linv is rebuilt next)
  }
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
}

// Step 1, pass 2: D_hat = d / ||d||, J = (J_raw - D_hat c^T) / ||d|| (quotient rule)
__global__ void __launch_bounds__(ENT) k_lwarp_norm(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->outer_done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  const double ind = 1.0 / (double)st->nd;
  double c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q] = st->Linv[q];
  const double s = 0.5 * (double)max(L.m, L.n);
  const double ci = 0.5 * (L.m - 1), cj = 0.5 * (L.n - 1), inv_s = 1.0 / s;
  const bool homog = a.kind == TILT_HOMOGRAPHY;
  const int p = L.p;
  FOR_ELEMS(L.plane) {
    const int j = (int)(idx / L.ldm), i = (int)(idx % L.ldm);
    if (i >= L.m || j >= L.n) continue;
    const double d = w[L.oD + idx];
    const double gx = w[L.oK + idx], gy = w[L.oK + L.plane + idx], gz = w[L.oK + 2 * L.plane + idx];
    double jr[8];
    jraw_row(gx, gy, homog ? gz : 0.0, ((double)j - cj) * inv_s, ((double)i - ci) * inv_s, jr);
    const double dh = d * ind;
    w[L.oD + idx] = (float)dh;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < p) w[L.oK + q * L.plane + idx] = (float)((jr[q] - dh * c[q]) * ind);
  }
}

// constraint rows Q (Z10) from tau
__global__ void k_qrows(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  for (int e = 0; e < 24; ++e) st->Q[e] = 0.0;
  if (st->outer_done || a.P.constraint_mode != TILT_CONSTRAINTS_CENTER_AREA) return;
  constraint_rows(st->tau, a.kind, a.L.m, a.L.n, st->Q);
}

// every inner loop starts with the problems whose outer loop is still running
__global__ void k_outer_begin(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  st->done = st->outer_done;
  st->iters = 0;
  st->conv = 0;
}

// cold start of an inner loop: A = D_hat, E = Y = 0 (Z4)
__global__ void __launch_bounds__(ENT) k_cold(Args a) {
  const int b = blockIdx.y;
  if (state(a, b)->done) return;
  float* w = slot(a, b);
  FOR_ELEMS(a.L.plane) {
    w[a.L.oA + idx] = w[a.L.oD + idx];
    w[a.L.oE + idx] = 0.f;
    w[a.L.oY + idx] = 0.f;
  }
}

// first inner loop of the pyramid's fine level (reading Z26): A, E, Y from the coarse level's state
// replicated 2x2 and halved where the coarse level produced one (CONVERGED or MAX_OUTER), else cold;
// Y is then projected (k_kty / k_projy) as every warm start
__global__ void __launch_bounds__(ENT) k_cold_coarse(Args a) {
  const int b = blockIdx.y;
  if (state(a, b)->done) return;
  float* w = slot(a, b);
  const int st = a.warm_rep[b].status;
  const bool from = st == TILT_PATCH_CONVERGED || st == TILT_PATCH_MAX_OUTER;
  const int ldm = a.L.ldm, m = a.L.m, mc = a.L.m / 2, nc = a.L.n / 2;
  const size_t o = (size_t)b * mc * nc;
  FOR_ELEMS(a.L.plane) {
    const int i = (int)(idx % ldm), j = (int)(idx / ldm);
    if (from && i < m) {
      const size_t c = o + (size_t)(i / 2) * nc + j / 2;
      w[a.L.oA + idx] = 0.5f * a.warm_A[c];
      w[a.L.oE + idx] = 0.5f * a.warm_E[c];
      w[a.L.oY + idx] = 0.5f * a.warm_Y[c];
    } else {
      w[a.L.oA + idx] = w[a.L.oD + idx];
      w[a.L.oE + idx] = 0.f;
      w[a.L.oY + idx] = 0.f;
    }
  }
}

// Y <- W^TW Y (Eq. Y_new_warmstart): K^T Y, then Y -= K (K^T Y)
__global__ void __launch_bounds__(ENT) k_kty(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  const float* w = slot(a, b);
  float s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) s[q] = 0.f;
  FOR_ELEMS(L.plane) {
    const float y = w[L.oY + idx];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < L.p) s[q] = fmaf(w[L.oK + q * L.plane + idx], y, s[q]);
  }
  block_add<8>(s, st->acc + ACC_S1);
}

__global__ void __launch_bounds__(ENT) k_projy(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->done) return;
  const Lay& L = a.L;
  float* w = slot(a, b);
  float s[8];
  load_s(st->acc + ACC_S1, L.p, s);
  FOR_ELEMS(L.plane) w[L.oY + idx] -= kdot(w + L.oK, L.plane, idx, L.p, s);
}

__global__ void k_clear_acc(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->done) return;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
}

// Step 3 inputs: K^T (A + E - D_hat) and ||E||_1 (problems whose outer loop runs)
__global__ void __launch_bounds__(ENT) k_dtau_red(Args a) {
  const int b = blockIdx.y;
  St* st = state(a, b);
  if (st->outer_done) return;
  const Lay& L = a.L;
  const float* w = slot(a, b);
  float s[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) s[q] = 0.f;
  FOR_ELEMS(L.plane) {
    const float e = w[L.oE + idx];
    const float v = res3(w[L.oA + idx], e, w[L.oD + idx]);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < L.p) s[q] = fmaf(w[L.oK + q * L.plane + idx], v, s[q]);
    s[8] += fabsf(e);
  }
  block_add<9>(s, st->acc + ACC_S1);
}

// Steps 3-4 and the outer stop (Eq. Delta_tau P:376-378 with Q; tau += dtau; Z9)
__global__ void k_dtau(Args a, int it, int n_outer) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  if (st->outer_done) return;
  const int p = a.L.p;
  double dt_inf = 0.0;
  bool finite = true;
  for (int q = 0; q < p; ++q) {
    double dq = 0.0;
    for (int r = q; r < p; ++r) dq += st->Linv[r * 8 + q] * (double)(float)st->acc[ACC_S1 + r];
    st->tau[q] = (double)(float)(st->tau[q] + dq);  // tau carried in fp32 (Z28)
    dt_inf = fmax(dt_inf, fabs(dq));
    finite = finite && isfinite(st->tau[q]);
  }
  const float f = st->nuc + st->lam * (float)st->acc[ACC_S1 + 8];
  st->dtau_inf = (float)dt_inf;
  st->f = f;
  st->outer_iters = it + 1;
  st->inner_total += st->iters;
  for (int e = 0; e < NACC; ++e) st->acc[e] = 0.0;
  if (!finite || !isfinite(f) || f > 1e12f) {
    st->status = TILT_PATCH_DIVERGED;
    st->outer_done = 1;
    return;
  }
  int rule = 0;
  if (st->have_fprev && fabsf(f - st->f_prev) < a.P.obj_tol * fabsf(st->f_prev)) rule = 1;
  else if (st->dtau_inf < a.P.tau_tol) rule = 2;
  st->f_prev = f;
  st->have_fprev = 1;
  if (rule) {
    st->status = TILT_PATCH_CONVERGED;
    st->stop_rule = rule;
    if (a.P.fixed_outer <= 0) st->outer_done = 1;
  } else {
    st->status = TILT_PATCH_MAX_OUTER;
    st->stop_rule = 3;
  }
  if (it + 1 >= n_outer) st->outer_done = 1;
  if (!st->outer_done) atomicAdd(a.counter, 1);
}

__global__ void k_report_solve(Args a, tilt_report* rep, float* tau_out, const tilt_report* rep_prev) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const St* st = state(a, b);
  const int p = a.L.p;
  for (int q = 0; q < p; ++q) tau_out[(size_t)b * p + q] = (float)st->tau[q];
  if (!rep) return;
  tilt_report r;
  memset(&r, 0, sizeof(r));
  r.status = st->status;
  r.stop_rule = st->stop_rule;
  r.outer_iters = st->outer_iters;
  r.inner_iters = st->inner_total;
  r.jacobi_sweeps = st->sweeps;
  r.aux_sweeps = st->aux_sweeps;
  r.rank = st->relrank;
  r.rank_band = st->band;
  r.svt_rank = st->svt_rank;
  r.sweep_cap_hits = st->caps;
  r.objective = st->f;
  r.crit1 = st->crit1;
  r.crit2 = st->crit2;
  r.patch_norm = st->nd;
  r.dtau_inf = st->dtau_inf;
  r.mu_last = st->mu;
  r.jacobi_rotations = st->rotations;
  r.kernel_path = 3;
  r.svd_warm_steps = st->warm_steps;
  if (rep_prev) {  // pyramid: the coarse level's counters (as solve_patch)
    const tilt_report& pr = rep_prev[b];
    r.outer_iters += pr.outer_iters;
    r.inner_iters += pr.inner_iters;
    r.jacobi_sweeps += pr.jacobi_sweeps;
    r.aux_sweeps += pr.aux_sweeps;
    r.sweep_cap_hits += pr.sweep_cap_hits;
    r.jacobi_rotations += pr.jacobi_rotations;
  }
  rep[b] = r;
}

// ---------------------------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------------------------
template <int RPL>
constexpr int RPL_TAG = RPL;

struct Run {
  Ctx& ctx;
  Args a;
  tilt_status st = TILT_OK;
  int rpl = 32;
  bool svdws = false;  // LADMAP+SVDWS (DevParams::svd_mode 1)

  explicit Run(Ctx& c) : ctx(c) {}

  bool fail_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return false;
    *ctx.err = std::string(what) + ": " + cudaGetErrorString(e);
    st = TILT_E_CUDA;
    return true;
  }
  bool check(const char* what) { return fail_cuda(cudaGetLastError(), what); }
  dim3 egrid(size_t count) const {
    return dim3((unsigned)((count + (size_t)ENT * EPT - 1) / ((size_t)ENT * EPT)), (unsigned)a.B);
  }
  dim3 sgrid() const { return dim3((unsigned)((a.B + 127) / 128)); }
  void launched(int k = 1) { *ctx.launches += k; }
  // the device tally of graph-run sweeps (counter[8]) since the last read, counted as launches
  void tally_sweeps() {
    const int t = ctx.h_counter[8];
    launched((t - ctx.sweep_tally_seen) * (a.NBp + 2));
    ctx.sweep_tally_seen = t;
  }
  int read_counter() {
    if (fail_cuda(cudaMemcpyAsync(ctx.h_counter, ctx.counter, 9 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream),
                  "cudaMemcpyAsync(counter)"))
      return -1;
    if (fail_cuda(cudaStreamSynchronize(ctx.stream), "cudaStreamSynchronize")) return -1;
    tally_sweeps();
    return *ctx.h_counter;
  }
  bool zero_counter() { return fail_cuda(cudaMemsetAsync(ctx.counter, 0, 4 * sizeof(int), ctx.stream), "memset"); }
  // counters [0..3) after a stream sync (false on error)
  bool read_counters(int* out) {
    if (fail_cuda(cudaMemcpyAsync(ctx.h_counter, ctx.counter, 9 * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream),
                  "cudaMemcpyAsync(counters)"))
      return false;
    if (fail_cuda(cudaStreamSynchronize(ctx.stream), "cudaStreamSynchronize")) return false;
    tally_sweeps();
    for (int i = 0; i < 3; ++i) out[i] = ctx.h_counter[i];
    return true;
  }

  // C = alpha op(X) op(Y) + beta C with per-problem strides (column-major; the hand-written FP32
  // GEMM of tilt_dense.cuh). nsub > 0: the GEMM runs on the nsub problems listed in ctx.widx only.
  int nsub = 0;

  bool gemm(bool ta, bool tb, int M, int N, int K, size_t oX, int ldx, size_t oY, int ldy, size_t oC, int ldc,
            float alpha = 1.f, float beta = 0.f) {
    const int nz = nsub > 0 ? nsub : a.B;
    const int* wi = nsub > 0 ? ctx.widx : nullptr;
    const dim3 g((M + dense::GBM - 1) / dense::GBM, (N + dense::GBN - 1) / dense::GBN, nz);
    const size_t s = a.L.stride;
    if (!ta && !tb)
      dense::k_gemm<false, false><<<g, dense::GNT, 0, ctx.stream>>>(a.ws, s, wi, M, N, K, oX, ldx, oY, ldy, oC, ldc, alpha, beta);
    else if (!ta && tb)
      dense::k_gemm<false, true><<<g, dense::GNT, 0, ctx.stream>>>(a.ws, s, wi, M, N, K, oX, ldx, oY, ldy, oC, ldc, alpha, beta);
    else if (ta && !tb)
      dense::k_gemm<true, false><<<g, dense::GNT, 0, ctx.stream>>>(a.ws, s, wi, M, N, K, oX, ldx, oY, ldy, oC, ldc, alpha, beta);
    else
      dense::k_gemm<true, true><<<g, dense::GNT, 0, ctx.stream>>>(a.ws, s, wi, M, N, K, oX, ldx, oY, ldy, oC, ldc, alpha, beta);
    launched();
    return check("gemm");
  }

  // (on the nsub problems of ctx.widx) solve P X = X in place: P (Nd x Nd, ldp) is factored in place
  // by blocked LU without pivoting (tilt_dense.cuh: P = I + S with S skew), X is Nd x ncols (ldx)
  bool lu_solve(size_t oP, int ldp, int Nd, size_t oX, int ldx, int ncols) {
    const int nz = nsub;
    const int* wi = ctx.widx;
    const size_t s = a.L.stride;
    cudaStream_t sm = ctx.stream;
    const int NB = dense::LU_NB;
    for (int k0 = 0; k0 < Nd; k0 += NB) {
      const int nb = Nd - k0 < NB ? Nd - k0 : NB;
      const int rest = Nd - k0 - nb;
      dense::k_lu_diag<<<dim3(1, 1, nz), 256, 0, sm>>>(a.ws, s, wi, oP, ldp, k0, nb);
      launched();
      if (rest > 0) {
        dense::k_trsm_l<<<dim3((rest + 127) / 128, 1, nz), 128, 0, sm>>>(a.ws, s, wi, oP, ldp, oP, ldp, k0, nb, k0 + nb, rest);
        dense::k_trsm_ru<<<dim3((rest + 127) / 128, 1, nz), 128, 0, sm>>>(a.ws, s, wi, oP, ldp, k0, nb, rest);
        launched(2);
        const size_t o21 = oP + (k0 + nb) + (size_t)k0 * ldp, o12 = oP + k0 + (size_t)(k0 + nb) * ldp;
        if (gemm(false, false, rest, rest, nb, o21, ldp, o12, ldp, o21 + (size_t)nb * ldp, ldp, -1.f, 1.f)) return true;
      }
    }
    for (int k0 = 0; k0 < Nd; k0 += NB) {  // forward: L Y = X
      const int nb = Nd - k0 < NB ? Nd - k0 : NB;
      const int rest = Nd - k0 - nb;
      dense::k_trsm_l<<<dim3((ncols + 127) / 128, 1, nz), 128, 0, sm>>>(a.ws, s, wi, oP, ldp, oX, ldx, k0, nb, 0, ncols);
      launched();
      if (rest > 0 && gemm(false, false, rest, ncols, nb, oP + (k0 + nb) + (size_t)k0 * ldp, ldp, oX + k0, ldx,
                           oX + k0 + nb, ldx, -1.f, 1.f))
        return true;
    }
    for (int k0 = ((Nd - 1) / NB) * NB; k0 >= 0; k0 -= NB) {  // backward: U X = Y
      const int nb = Nd - k0 < NB ? Nd - k0 : NB;
      dense::k_trsm_u<<<dim3((ncols + 127) / 128, 1, nz), 128, 0, sm>>>(a.ws, s, wi, oP, ldp, oX, ldx, k0, nb, ncols);
      launched();
      if (k0 > 0 && gemm(false, false, k0, ncols, nb, oP + (size_t)k0 * ldp, ldp, oX + k0, ldx, oX, ldx, -1.f, 1.f))
        return true;
    }
    return check("lu solve");
  }

  template <int RPL>
  bool sweeps_rpl() {
    const size_t sm_cross = (size_t)(2 * BW * 32 * RPL + 4 * BW * BW + 8 * BW) * sizeof(float);
    const size_t sm_intra = (size_t)(BW * 32 * RPL + BW * BW + 4 * BW) * sizeof(float);
    if (fail_cuda(cudaFuncSetAttribute((const void*)k_round<RPL, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm_cross),
                  "cudaFuncSetAttribute(k_round)"))
      return true;
    if (fail_cuda(cudaFuncSetAttribute((const void*)k_round<RPL, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm_intra),
                  "cudaFuncSetAttribute(k_round)"))
      return true;
    auto enqueue = [&](cudaStream_t sm) {  // one sweep: intra round, NBp - 1 cross rounds, reset, end
      k_round<RPL, 0><<<dim3(a.NB, a.B), RNT, sm_intra, sm>>>(a, 0);
      for (int r = 0; r < a.NBp - 1; ++r)
        k_round<RPL, 1><<<dim3(a.NBp / 2, a.B), RNT, sm_cross, sm>>>(a, r);
      cudaMemsetAsync(ctx.counter, 0, 4 * sizeof(int), sm);
      k_sweep_end<<<sgrid(), 128, 0, sm>>>(a);
    };
    // All sweeps of an SVT as one graph: a WHILE node whose body is one sweep (NBp + 1 launches, the
    // counter reset) followed by k_sweep_cond, which ends the loop once no problem's SVT runs (each
    // problem also stops itself at max_sweeps in k_sweep_end). No host round trip per sweep and one
    // launch call per SVT: with few active problems the host's launches and the per-sweep counter
    // read, not the GPU, set the pace (one 200x200 problem: 1.48 ms per LADMAP iteration of which
    // 0.64 ms on the GPU). Cached by the kernels' argument bytes (the V buffer offset
    // alternates with the Newton-Schulz step: two executables); captured on a private stream
    // (capture is not allowed on the legacy default stream), launched on ctx.stream.
    if (!ctx.cap_stream &&
        fail_cuda(cudaStreamCreateWithFlags(&ctx.cap_stream, cudaStreamNonBlocking), "cudaStreamCreate(capture)"))
      return true;
    std::string key(reinterpret_cast<const char*>(&a), sizeof(Args));
    key.append(reinterpret_cast<const char*>(&RPL_TAG<RPL>), sizeof(int));
    cudaGraphExec_t exec = nullptr;
    for (int c = 0; c < 2; ++c)
      if (ctx.sweep_exec[c] && ctx.sweep_key[c] == key) exec = ctx.sweep_exec[c];
    if (!exec) {
      cudaGraph_t g = nullptr;
      if (fail_cuda(cudaGraphCreate(&g, 0), "cudaGraphCreate(sweeps)")) return true;
      cudaGraphConditionalHandle h;
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cudaGraphNode_t node;
      bool bad = fail_cuda(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault), "conditional handle");
      if (!bad) {
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        bad = fail_cuda(cudaGraphAddNode(&node, g, nullptr, 0, &cp), "cudaGraphAddNode(while)");
      }
      if (!bad) {
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        bad = fail_cuda(cudaStreamBeginCaptureToGraph(ctx.cap_stream, body, nullptr, nullptr, 0,
                                                      cudaStreamCaptureModeThreadLocal),
                        "capture(sweep)");
        if (!bad) {
          enqueue(ctx.cap_stream);
          k_sweep_cond<<<1, 1, 0, ctx.cap_stream>>>(ctx.counter, ctx.counter + 8, h);
          bad = fail_cuda(cudaStreamEndCapture(ctx.cap_stream, &body), "capture(sweep) end");
        }
      }
      const int c = ctx.sweep_next;
      if (!bad) {
        ctx.sweep_next ^= 1;
        if (ctx.sweep_exec[c]) cudaGraphExecDestroy(ctx.sweep_exec[c]);
        ctx.sweep_exec[c] = nullptr;
        bad = fail_cuda(cudaGraphInstantiate(&ctx.sweep_exec[c], g, 0), "cudaGraphInstantiate(sweeps)");
      }
      cudaGraphDestroy(g);
      if (bad) return true;
      ctx.sweep_key[c] = key;
      exec = ctx.sweep_exec[c];
    }
    if (fail_cuda(cudaGraphLaunch(exec, ctx.stream), "cudaGraphLaunch(sweeps)")) return true;
    return check("jacobi sweeps");
  }

  // Jacobi sweeps on (B, V) until every problem's SVT stopped (k_svt_begin ran before)
  bool sweeps() {
    switch (rpl) {
      case 4: return sweeps_rpl<4>();
      case 8: return sweeps_rpl<8>();
      case 16: return sweeps_rpl<16>();
      default: return sweeps_rpl<32>();
    }
  }

  // one SVT of S (eps per eps_mode) with the V in a.oV; leaves B scaled, sigma/stats in the state
  bool svt_core(const float* eps, int eps_mode, int count_sweeps, bool do_scale, bool ws_state = false) {
    if (zero_counter()) return true;
    k_svt_begin<<<sgrid(), 128, 0, ctx.stream>>>(a, eps, eps_mode);
    launched();
    const Lay& L = a.L;
    if (gemm(false, false, L.m, L.n, L.n, L.oS, L.ldm, a.oV, L.ldn, L.oB, L.ldm)) return true;
    k_fro<<<egrid(L.plane), ENT, 0, ctx.stream>>>(a);
    launched();
    if (sweeps()) return true;
    k_svt_sig<<<dim3((L.n + 7) / 8, a.B), 256, 0, ctx.stream>>>(a);
    k_svt_stats<<<a.B, 32, 0, ctx.stream>>>(a, count_sweeps);
    launched(2);
    if (ws_state) {  // U = B / ||b||, Sigma = sigma for the next warm step (before B is scaled)
      k_ws_state<<<dim3((L.n + 7) / 8, a.B), 256, 0, ctx.stream>>>(a);
      launched();
    }
    if (do_scale) {
      k_svt_scale<<<egrid(L.plane), ENT, 0, ctx.stream>>>(a);
      launched();
    }
    return check("svt");
  }

  // list the problems with st->warm in ctx.widx; the following GEMMs run on them only
  bool ws_subset(int count) {
    if (zero_counter()) return true;
    k_ws_index<<<sgrid(), 128, 0, ctx.stream>>>(a, ctx.widx);
    launched();
    nsub = count;
    return check("subset index");
  }

  // Alg. 2, first half (problems with st->warm): W, P_U, P_V, P_Sigma, h1, h2, t*
  bool ws_part1() {
    const Lay& L = a.L;
    const int m = L.m, n = L.n, ldm = L.ldm, ldn = L.ldn;
    const dim3 ep = egrid(L.plane);
    k_colscale<<<ep, ENT, 0, ctx.stream>>>(a, L.oX, L.oU, L.oSg, 0, 1);
    launched();
    if (gemm(false, true, m, n, n, L.oX, ldm, a.oV, ldn, L.oW, ldm)) return true;      // W
    if (gemm(false, true, m, m, n, L.oW, ldm, L.oS, ldm, L.oPU, ldm)) return true;     // W M^T
    k_skew<<<egrid((size_t)m * m), ENT, 0, ctx.stream>>>(a, L.oPU, m, ldm, 0);                     // P_U
    if (gemm(true, false, n, n, m, L.oW, ldm, L.oS, ldm, L.oPV, ldn)) return true;     // W^T M
    k_skew<<<egrid((size_t)n * n), ENT, 0, ctx.stream>>>(a, L.oPV, n, ldn, 0);                     // P_V
    launched(2);
    if (gemm(false, false, m, n, n, L.oS, ldm, a.oV, ldn, L.oH2, ldm)) return true;     // M V
    k_ws_psig<<<dim3((n + 7) / 8, a.B), 256, 0, ctx.stream>>>(a);                                  // P_Sigma
    k_colscale<<<ep, ENT, 0, ctx.stream>>>(a, L.oX2, L.oU, L.oPs, 0, 1);
    launched(2);
    if (gemm(false, true, m, n, n, L.oX2, ldm, a.oV, ldn, L.oZ, ldm)) return true;    // U P_S V^T
    k_copy_if<<<ep, ENT, 0, ctx.stream>>>(a, L.oH1, L.oZ, L.plane, 1);
    launched();
    if (gemm(false, false, m, n, m, L.oPU, ldm, L.oW, ldm, L.oH1, ldm, 1.f, 1.f)) return true;
    if (gemm(false, false, m, n, n, L.oW, ldm, L.oPV, ldn, L.oH1, ldm, -1.f, 1.f)) return true;
    k_ws_z<<<ep, ENT, 0, ctx.stream>>>(a);                                                          // Z
    launched();
    if (gemm(false, false, m, n, m, L.oPU, ldm, L.oZ, ldm, L.oH2, ldm, -1.f, 0.f)) return true;
    if (gemm(false, false, m, n, n, L.oZ, ldm, L.oPV, ldn, L.oH2, ldm, 1.f, 1.f)) return true;
    k_ws_red<<<ep, ENT, 0, ctx.stream>>>(a);
    launched();
    if (zero_counter()) return true;
    k_ws_t<<<sgrid(), 128, 0, ctx.stream>>>(a);
    launched();
    return check("svd warm step (1)");
  }

  // Cayley update X <- (I + S)^{-1} (I - S) X = 2 (I + S)^{-1} X - X, S = (t*/2) P skew, exactly:
  // P holds I + S (k_skew scale_t), factored in place; `tmp` (rows x cols, ldx) receives the solve
  bool cayley(size_t oP, int ldp, size_t oX, size_t tmp, int rows, int cols, int ldx, size_t count) {
    const dim3 eg = egrid(count);
    k_copy_if<<<eg, ENT, 0, ctx.stream>>>(a, tmp, oX, count, 1);
    launched();
    if (lu_solve(oP, ldp, rows, tmp, ldx, cols)) return true;
    k_cay_finish<<<eg, ENT, 0, ctx.stream>>>(a, oX, tmp, count);
    launched();
    return check("cayley");
  }

  // Alg. 2, second half: U(t), V(t), Sigma(t); B <- U T_eps(Sigma) so that A = B V^T for every problem
  bool ws_part2() {
    const Lay& L = a.L;
    const int m = L.m, n = L.n, ldm = L.ldm, ldn = L.ldn;
    k_skew<<<egrid((size_t)m * m), ENT, 0, ctx.stream>>>(a, L.oPU, m, ldm, 1);  // I + (t/2) P_U
    k_skew<<<egrid((size_t)n * n), ENT, 0, ctx.stream>>>(a, L.oPV, n, ldn, 1);  // I + (t/2) P_V
    launched(2);
    if (cayley(L.oPU, ldm, L.oU, L.oX, m, n, ldm, L.plane)) return true;
    if (cayley(L.oPV, ldn, a.oV, L.oVt, n, n, ldn, L.vplane)) return true;
    k_ws_sigma<<<dim3((n + 127) / 128, a.B), 128, 0, ctx.stream>>>(a);
    k_svt_stats<<<a.B, 32, 0, ctx.stream>>>(a, 0, 1);
    k_colscale<<<egrid(L.plane), ENT, 0, ctx.stream>>>(a, L.oB, L.oU, L.oSg, 1, 1);
    launched(3);
    return check("svd warm step (2)");
  }

  bool ns_step() {
    const Lay& L = a.L;
    if (gemm(true, false, L.n, L.n, L.n, a.oV, L.ldn, a.oV, L.ldn, L.oT, L.ldn)) return true;
    k_ns_mid<<<egrid(L.vplane), ENT, 0, ctx.stream>>>(a);
    launched();
    const size_t other = a.oV == L.oV ? L.oV2 : L.oV;
    if (gemm(false, false, L.n, L.n, L.n, a.oV, L.ldn, L.oT, L.ldn, other, L.ldn)) return true;
    a.oV = other;
    return check("ns");
  }

  void setup(int B, int m, int n, int p, const DevParams& P) {
    a.ws = ctx.ws;
    svdws = P.svd_mode == 1;
    a.L = make_lay(m, n, p, svdws);
    a.B = B;
    a.P = P;
    a.oV = a.L.oV;
    a.counter = ctx.counter;
    a.rep_outer = 1;
    a.cur_outer = 0;
    a.images = nullptr;
    a.boxes = nullptr;
    a.patch_image = nullptr;
    a.warm_A = a.warm_E = a.warm_Y = nullptr;
    a.warm_rep = nullptr;
    a.tiny2 = 1e-14f;  // ||b_j|| <= 1e-7 ||M||_F: below fp32 resolution of the SVT output
    a.NB = (n + BW - 1) / BW;
    a.NBp = a.NB + (a.NB & 1);
    if (a.NBp < 2) a.NBp = 2;
    const int d = m;  // column length of the Jacobi columns
    rpl = d <= 128 ? 4 : d <= 256 ? 8 : d <= 512 ? 16 : 32;
  }
};

}  // namespace

size_t ws_need(int B, int m, int n, int p, bool svdws) { return (size_t)B * make_lay(m, n, p, svdws).stride; }

tilt_status ensure(Ctx& ctx, size_t floats, int B) {
  if (!ctx.counter) {
    if (cudaMalloc(&ctx.counter, 64 * sizeof(int)) != cudaSuccess) return TILT_E_OOM;
    if (cudaMallocHost(&ctx.h_counter, 64 * sizeof(int)) != cudaSuccess) return TILT_E_OOM;
    if (cudaMemset(ctx.counter, 0, 64 * sizeof(int)) != cudaSuccess) return TILT_E_CUDA;
    ctx.sweep_tally_seen = 0;
  }
  if (ctx.cap_b < B) {
    if (ctx.widx) cudaFree(ctx.widx);
    ctx.widx = nullptr;
    ctx.cap_b = 0;
    if (cudaMalloc(&ctx.widx, (size_t)B * sizeof(int)) != cudaSuccess) return TILT_E_OOM;
    ctx.cap_b = B;
  }
  if (ctx.ws_floats < floats) {
    if (ctx.ws) cudaFree(ctx.ws);
    ctx.ws = nullptr;
    ctx.ws_floats = 0;
    if (cudaMalloc(&ctx.ws, floats * sizeof(float)) != cudaSuccess) {
      *ctx.err = "cudaMalloc(multi-CTA workspace) failed";
      return TILT_E_OOM;
    }
    ctx.ws_floats = floats;
  }
  return TILT_OK;
}

void release(Ctx& ctx) {
  for (auto& g : ctx.sweep_exec)
    if (g) cudaGraphExecDestroy(g);
  if (ctx.cap_stream) cudaStreamDestroy(ctx.cap_stream);
  if (ctx.ws) cudaFree(ctx.ws);
  if (ctx.widx) cudaFree(ctx.widx);
  if (ctx.counter) cudaFree(ctx.counter);
  if (ctx.h_counter) cudaFreeHost(ctx.h_counter);
  ctx = Ctx();
}

// Orthonormalise (K2) from the planes in D / K, the (warm or cold) start, mu_0 (Z3) and one inner loop
// (LADMAP or the ADM baseline) for every problem with done == 0. Returns true on error (R.st set).
static bool inner_core(Run& R, const DevParams& P, const float* Q, int l, int q_state, bool first) {
  Args& a = R.a;
  const Lay& L = a.L;
  const int m = L.m, n = L.n;
  cudaStream_t sm = R.ctx.stream;
    k_gram<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  k_chol<<<R.sgrid(), 128, 0, sm>>>(a, Q, l, q_state);
  k_apply_linv<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  R.launched(3);
  // warm start (Eq. warm_start, Eq. Y_new_warmstart) or A_0 = D, E_0 = Y_0 = 0
  if (first && P.vws && a.warm_A) {  // pyramid fine level from the coarse state (Z26)
    k_cold_coarse<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_clear_acc<<<R.sgrid(), 128, 0, sm>>>(a);
    k_kty<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_projy<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_clear_acc<<<R.sgrid(), 128, 0, sm>>>(a);
    R.launched(5);
  } else if (first || !P.vws) {
    k_cold<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    R.launched();
  } else {
    k_clear_acc<<<R.sgrid(), 128, 0, sm>>>(a);
    k_kty<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_projy<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_clear_acc<<<R.sgrid(), 128, 0, sm>>>(a);
    R.launched(4);
  }
  if (first) {
    k_identity<<<R.egrid(L.vplane), ENT, 0, sm>>>(a, L.oV);
    R.launched();
  }
  // ||W^TW D||
  k_kt<0><<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  k_denom<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  if (R.svdws || P.inner_solver == 1) {
    k_dnorm<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    if (R.svdws) k_ws_init<<<R.sgrid(), 128, 0, sm>>>(a, P.svd_ws_gate);
    if (P.inner_solver == 1) k_adm_init<<<R.sgrid(), 128, 0, sm>>>(a);
    R.launched(2);
  }
  k_sc_denom<<<R.sgrid(), 128, 0, sm>>>(a);
  R.launched(5);
  if (R.check("inner setup")) return true;
  // sigma_1(D) by the same Jacobi (Z3); its V warm-starts the first SVT
  k_copy_plane<<<R.egrid(L.plane), ENT, 0, sm>>>(a, L.oS, L.oD);
  R.launched();
  if (R.svt_core(nullptr, 2, 0, false)) return true;
  k_sc_mu0<<<R.sgrid(), 128, 0, sm>>>(a);
  R.launched();
  const bool warm = P.svd_warm != 0;
  if (P.inner_solver == 1) {  // ADM baseline (reading Z24): cold start A = D, E = Y = J dtau = 0
    for (int k = 0; k < a.niter; ++k) {
      if (!warm) {
        k_identity<<<R.egrid(L.vplane), ENT, 0, sm>>>(a, a.oV);
        R.launched();
      }
      k_adm_m<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      R.launched();
      if (R.svt_core(nullptr, 0, 1, true)) return true;
      if (R.gemm(false, true, m, n, n, L.oB, L.ldm, a.oV, L.ldn, L.oA, L.ldm)) return true;
      if (warm && (k % P.ns_period == P.ns_period - 1 || k + 1 == a.niter))
        if (R.ns_step()) return true;
      k_adm_e<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      k_kt<3><<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      k_adm_y<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      R.launched(3);
      if (R.zero_counter()) return true;
      k_adm_sc<<<R.sgrid(), 128, 0, sm>>>(a, k);
      R.launched();
      if (R.check("adm iteration")) return true;
      const int act = R.read_counter();
      if (act < 0) return true;
      if (act == 0) break;
    }
  } else {
  k_kt<1><<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  k_m0<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  R.launched(2);
  for (int k = 0; k < a.niter; ++k) {
    if (!warm) {
      k_identity<<<R.egrid(L.vplane), ENT, 0, sm>>>(a, a.oV);
      R.launched();
    }
    int nwarm = 0;
    if (R.svdws && k > 0) {  // Alg. 2 gate, then the warm step's first half for the gated problems
      if (R.zero_counter()) return true;
      k_ws_diff<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      k_ws_gate<<<R.sgrid(), 128, 0, sm>>>(a, k);
      R.launched(2);
      int c[3];
      if (!R.read_counters(c)) return true;
      if (c[1] > 0) {
        if (R.ws_subset(c[1])) return true;
        if (R.ws_part1()) return true;
        R.nsub = 0;
        if (!R.read_counters(c)) return true;
        nwarm = c[1];
      }
    }
    if (R.svt_core(nullptr, 0, 1, true, R.svdws)) return true;
    if (nwarm > 0) {
      if (R.ws_subset(nwarm)) return true;
      if (R.ws_part2()) return true;
      R.nsub = 0;
    }
    if (R.gemm(false, true, m, n, n, L.oB, L.ldm, a.oV, L.ldn, L.oAn, L.ldm)) return true;
    if (warm && (k % P.ns_period == P.ns_period - 1 || k + 1 == a.niter))
      if (R.ns_step()) return true;
    if (R.svdws) {
      k_ws_after<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      R.launched();
    }
    k_kt<2><<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_estep<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    k_sc1<<<R.sgrid(), 128, 0, sm>>>(a, k);
    k_ystep<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    if (R.zero_counter()) return true;
    k_sc2<<<R.sgrid(), 128, 0, sm>>>(a, k);
    R.launched(5);
    if (R.check("ladmap iteration")) return true;
    const int act = R.read_counter();
    if (act < 0) return true;
    if (act == 0) break;
  }
  }
  return false;
}

tilt_status inner(Ctx& ctx, const float* D, const float* J, const float* Q, int l, int B, int m, int n, int p,
                  const DevParams& P, float* A, float* E, float* Y, tilt_report* rep) {
  tilt_status s0 = ensure(ctx, ws_need(B, m, n, p, P.svd_mode == 1), B);
  if (s0 != TILT_OK) return s0;
  Run R(ctx);
  R.setup(B, m, n, p, P);
  Args& a = R.a;
  const Lay& L = a.L;
  a.tol = P.jacobi_tol > 0.f ? P.jacobi_tol : default_jacobi_tol(m);
  a.big2 = a.tol / (float)n;
  a.max_sweeps = P.jacobi_max_sweeps;
  a.niter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
  cudaStream_t sm = ctx.stream;
  if (R.fail_cuda(cudaMemsetAsync(ctx.ws, 0, (size_t)B * L.stride * sizeof(float), sm), "memset(ws)")) return R.st;
  const dim3 tg((n + 31) / 32, (m + 31) / 32, B), tgj((n + 31) / 32, (m + 31) / 32, B * p);
  k_to_plane<<<tg, dim3(32, 8), 0, sm>>>(D, 1, a, L.oD);
  k_to_plane<<<tgj, dim3(32, 8), 0, sm>>>(J, p, a, L.oK);
  k_init<<<R.sgrid(), 128, 0, sm>>>(a);
  R.launched(3);
  if (inner_core(R, P, Q, l, 0, true)) return R.st;
  k_l1<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
  k_report<<<R.sgrid(), 128, 0, sm>>>(a, rep);
  const dim3 og((n + 31) / 32, (m + 31) / 32, B);
  k_from_plane<<<og, dim3(32, 8), 0, sm>>>(A, a, L.oA, m, n, L.ldm, 1);
  k_from_plane<<<og, dim3(32, 8), 0, sm>>>(E, a, L.oE, m, n, L.ldm, 1);
  R.launched(4);
  if (Y) {
    k_from_plane<<<og, dim3(32, 8), 0, sm>>>(Y, a, L.oY, m, n, L.ldm, 1);
    R.launched();
  }
  R.check("inner outputs");
  return R.st;
}

tilt_status solve(Ctx& ctx, const float* images, int n_images, int H, int W, const int32_t* patch_image,
                  const int32_t* boxes, const float* tau0, int B, int m, int n, int kind, const DevParams& P,
                  float* tau_out, float* A, float* E, float* Y, tilt_report* rep, const tilt_report* rep_prev,
                  const float* warm_A, const float* warm_E, const float* warm_Y, const tilt_report* warm_rep) {
  const int p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  if (P.inner_solver != 0) return TILT_E_ARG;  // the ADM's own dtau step is the CTA kernels' (k_solve)
  tilt_status s0 = ensure(ctx, ws_need(B, m, n, p, P.svd_mode == 1), B);
  if (s0 != TILT_OK) return s0;
  Run R(ctx);
  R.setup(B, m, n, p, P);
  Args& a = R.a;
  const Lay& L = a.L;
  a.tol = P.jacobi_tol > 0.f ? P.jacobi_tol : default_jacobi_tol(m);
  a.big2 = a.tol / (float)n;
  a.max_sweeps = P.jacobi_max_sweeps;
  a.niter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
  a.rep_outer = P.max_outer;
  a.images = images;
  a.n_images = n_images;
  a.H = H;
  a.W = W;
  a.kind = kind;
  a.patch_image = patch_image;
  a.boxes = boxes;
  if (warm_A && warm_E && warm_Y && warm_rep) {
    a.warm_A = warm_A;
    a.warm_E = warm_E;
    a.warm_Y = warm_Y;
    a.warm_rep = warm_rep;
  }
  cudaStream_t sm = ctx.stream;
  if (R.fail_cuda(cudaMemsetAsync(ctx.ws, 0, (size_t)B * L.stride * sizeof(float), sm), "memset(ws)")) return R.st;
  k_init<<<R.sgrid(), 128, 0, sm>>>(a);
  k_solve_init<<<R.sgrid(), 128, 0, sm>>>(a, tau0);
  R.launched(2);
  const int n_outer = P.fixed_outer > 0 ? P.fixed_outer : P.max_outer;
  for (int it = 0; it < n_outer; ++it) {
    a.cur_outer = it;
    NvtxRange nv_outer("multi-CTA outer iteration");
    // Step 1: D_hat, J (two passes), Q
    {
      NvtxRange nv_k1("K1 warp + Jacobian");
      k_lwarp<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      k_lwarp_status<<<R.sgrid(), 128, 0, sm>>>(a);
      k_lwarp_norm<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
      k_qrows<<<R.sgrid(), 128, 0, sm>>>(a);
      k_outer_begin<<<R.sgrid(), 128, 0, sm>>>(a);
      R.launched(5);
    }
    if (R.check("warp")) return R.st;
    // Step 2: orthonormalise, warm start, inner loop
    {
      NvtxRange nv_k3("K2-K3 orthonormalise + LADMAP inner loop");
      if (inner_core(R, P, nullptr, 3, 1, it == 0)) return R.st;
    }
    // Steps 3-4, outer stop
    k_dtau_red<<<R.egrid(L.plane), ENT, 0, sm>>>(a);
    if (R.zero_counter()) return R.st;
    k_dtau<<<R.sgrid(), 128, 0, sm>>>(a, it, n_outer);
    R.launched(2);
    if (R.check("dtau")) return R.st;
    const int act = R.read_counter();
    if (act < 0) return R.st;
    if (act == 0) break;
  }
  k_report_solve<<<R.sgrid(), 128, 0, sm>>>(a, rep, tau_out, rep_prev);
  const dim3 og((n + 31) / 32, (m + 31) / 32, B);
  R.launched();
  if (A) {
    k_from_plane<<<og, dim3(32, 8), 0, sm>>>(A, a, L.oA, m, n, L.ldm, 2);
    R.launched();
  }
  if (E) {
    k_from_plane<<<og, dim3(32, 8), 0, sm>>>(E, a, L.oE, m, n, L.ldm, 2);
    R.launched();
  }
  if (Y) {
    k_from_plane<<<og, dim3(32, 8), 0, sm>>>(Y, a, L.oY, m, n, L.ldm, 2);
    R.launched();
  }
  R.check("solve outputs");
  return R.st;
}

__global__ void k_svt_out(Args a, float* sigma, int32_t* sweeps) {
  const int b = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const St* st = state(a, b);
  if (sigma && j < a.L.n) sigma[(size_t)b * a.L.n + j] = slot(a, b)[a.L.oSig + j];
  if (sweeps && j == 0) sweeps[b] = st->sw_cur;
}

__global__ void k_svt_clear(Args a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  St* st = state(a, b);
  st->done = 0;
  st->status = TILT_PATCH_CONVERGED;
}

tilt_status svt(Ctx& ctx, const float* M, int B, int m, int n, const float* eps, float* V_io, float* A,
                float* sigma, int32_t* sweeps, float tol, int max_sweeps) {
  tilt_status s0 = ensure(ctx, ws_need(B, m, n, 1, false), B);
  if (s0 != TILT_OK) return s0;
  Run R(ctx);
  DevParams P;
  memset(&P, 0, sizeof(P));
  R.setup(B, m, n, 1, P);
  Args& a = R.a;
  const Lay& L = a.L;
  a.tol = tol;
  a.big2 = tol / (float)n;
  a.max_sweeps = max_sweeps;
  cudaStream_t sm = ctx.stream;
  if (R.fail_cuda(cudaMemsetAsync(ctx.ws, 0, (size_t)B * L.stride * sizeof(float), sm), "memset(ws)")) return R.st;
  k_svt_clear<<<R.sgrid(), 128, 0, sm>>>(a);
  k_to_plane<<<dim3((n + 31) / 32, (m + 31) / 32, B), dim3(32, 8), 0, sm>>>(M, 1, a, L.oS);
  R.launched(2);
  if (V_io) {  // row-major [n][n] -> column-major plane (ld = ldn)
    Args av = a;
    av.L.m = n;
    av.L.ldm = L.ldn;
    k_to_plane<<<dim3((n + 31) / 32, (n + 31) / 32, B), dim3(32, 8), 0, sm>>>(V_io, 1, av, L.oV);
  } else {
    k_identity<<<R.egrid(L.vplane), ENT, 0, sm>>>(a, L.oV);
  }
  R.launched();
  if (R.svt_core(eps, 1, 0, true)) return R.st;
  if (R.gemm(false, true, m, n, n, L.oB, L.ldm, a.oV, L.ldn, L.oAn, L.ldm)) return R.st;
  k_from_plane<<<dim3((n + 31) / 32, (m + 31) / 32, B), dim3(32, 8), 0, sm>>>(A, a, L.oAn, m, n, L.ldm, 0);
  k_svt_out<<<dim3((n + 127) / 128, B), 128, 0, sm>>>(a, sigma, sweeps);
  R.launched(2);
  if (V_io) {
    k_from_plane<<<dim3((n + 31) / 32, (n + 31) / 32, B), dim3(32, 8), 0, sm>>>(V_io, a, a.oV, n, n, L.ldn, 0);
    R.launched();
  }
  R.check("svt outputs");
  return R.st;
}

}  // namespace lp
}  // namespace tilt

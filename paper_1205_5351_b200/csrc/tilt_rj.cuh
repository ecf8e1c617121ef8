// tilt_rj.cuh — one warp per patch, "row-register" layout, for windows with m <= 64 and n <= 50
// (configs 1, 2, 5 and the coarse level of config 3).
//
// Paper: Ren & Lin, arXiv 1205.5351 (/root/reference/PAPER.md, cited P:<line>); readings: DESIGN.md.
// Same method and readings as the CTA-per-patch kernels of tilt_kernels.cuh (Algorithm 1, LADMAP with
// the W^TW projector, warm one-sided Jacobi SVT); only the data layout and the Jacobi ordering differ.
//
// Layout. Lane l of the warp owns rows 2l and 2l+1 of every m x n patch matrix; a column j of a
// matrix is one u64 register pair {X[2l][j], X[2l+1][j]} per lane, so every row-wise update is one
// packed FFMA2 (two FMAs per issue slot, sm_100a). During the SVT the whole of B = M V and of the
// warm V (n x n) sit in registers: a Jacobi rotation of columns (i, j) is 2 FFMA2 for B and 2 for
// V per lane, and the only cross-lane traffic of a round is the column-pair dot products
// (transpose-reduce: one shuffle per pair per round) and the rotation parameters (one shared-memory
// float2 per pair, broadcast). No CTA barriers: a patch is one warp.
//
// Jacobi ordering: odd-even transposition (round A pairs slots (2k, 2k+1), round B pairs
// (2k+1, 2k+2)); every rotation also swaps the two slots, so after n rounds every column pair has
// met exactly once and a rolled loop of "round A + round B" keeps static register indices.
//
// Patch planes (D_hat, A, E, Y~, and the Jacobian factors GX, GY, GZ of the implicit projector) are
// column-major in the per-warp global workspace slot (L2-resident): column j at j*LDP, lane l reads
// the float2 at j*LDP + 2l (coalesced). V (and the Newton-Schulz temporary) are in shared memory,
// row-pair interleaved: Vs[(q*NC + j)*2 + h] = V[2q+h][j].
#pragma once


#include "tilt_kernels.cuh"

namespace tilt {
namespace rj {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 up(u64 x) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(x));
  return v;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fmas2(u64 a, float s, u64 c) { return fma2(a, pk(s, s), c); }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 muls2(u64 a, float s) { return mul2(a, pk(s, s)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// packed a + e - d, each half exact up to the final rounding (res3 of tilt_device.cuh)
__device__ __forceinline__ u64 res3_2(u64 a, u64 e, u64 d) {
  const float2 x = up(a), y = up(e), z = up(d);
  return pk(res3(x.x, y.x, z.x), res3(x.y, y.y, z.y));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float hsum(u64 x) {
  const float2 v = up(x);
  return v.x + v.y;
}
__device__ __forceinline__ u64 shrink2(u64 x, float thr) {
  const float2 v = up(x);
  return pk(copysignf(fmaxf(fabsf(v.x) - thr, 0.f), v.x), copysignf(fmaxf(fabsf(v.y) - thr, 0.f), v.y));
}

// Butterfly all-reduce (every lane ends with bitwise-identical sums: each level adds the same two
// operands in every lane).
__device__ __forceinline__ float wsum(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}
__device__ __forceinline__ double wsumd(double x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}
__device__ __forceinline__ float wmax(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(FULL, x, o));
  return x;
}
__device__ __forceinline__ int wsumi(int x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Transpose-reduce: w[k] (k < K) are per-lane partial sums of K quantities; returns, in lane l,
// the warp sum of quantity l (0 for l >= K). One shuffle per quantity (31 for K = 32).
template <int K>
__device__ __forceinline__ float treduce(float (&w)[32], int lane) {
  static_assert(K >= 1 && K <= 32, "at most 32 quantities");
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool b = (lane & h) != 0;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      if (k >= K) continue;  // entries >= K are identically zero at every level
      const float x = w[k];
      const float y = (k + h < K) ? w[k + h] : 0.f;
      const float send = b ? x : y, keep = b ? y : x;
      w[k] = keep + __shfl_xor_sync(FULL, send, h);
    }
  }
  return w[0];
}

template <int NC_>
struct RJ {
  static constexpr int NC = NC_;          // column slots (even); n <= NC
  static constexpr int NH = NC / 2;       // pairs per round / row pairs of V
  static constexpr int Q = NC - 1;        // circle-method ring length
  static constexpr int RR = 7;            // rounds per body (register shift between bodies)
  static constexpr int NB = Q / RR;       // bodies per sweep
  static constexpr int WPB = 4;           // warps (= patches in flight) per block
  static constexpr int NT = 32 * WPB;
  static constexpr int VSF = NC * NC;     // floats of Vs / Ts
  // per-warp shared floats: Vs, Ts, Pw[2][32] float2, wv[NC] float2, Lp[64], cp[8], Linv[64] (double)
  static constexpr int OFF_PW = VSF;
  static constexpr int OFF_WV = OFF_PW + 128;
  static constexpr int OFF_LP = OFF_WV + 2 * NC + 4;
  static constexpr int OFF_CP = OFF_LP + 64;
  static constexpr int OFF_LINV = (OFF_CP + 8 + 3) & ~3;
  static constexpr int OFF_SC = OFF_LINV + 128;  // per-call scalar scratch (16 words)
  static constexpr int LOGRING = 8;              // rounds of the rotation log staged in shared memory
  static constexpr int OFF_RING = OFF_SC + 16;   // LOGRING x 32 float2 (cp.async staging of the log)
  static constexpr int SMF = OFF_RING + LOGRING * 64;
  static constexpr int NPLANES = 8;       // D, A, E, Y, GX, GY, GZ, B (= M V)
  static_assert(NC % 2 == 0 && NC <= 52, "register budget: 4 NC + ~40 registers per lane");
  static_assert(Q % RR == 0, "the ring length must be a multiple of the body length");
  static_assert(SMF % 4 == 0, "16-byte aligned per-warp shared blocks");
  // circle-method pair k of (local) round r: elements (register indices) I (top) and J (bottom)
  static __host__ __device__ constexpr int I(int r, int k) { return k == 0 ? Q : (r + k) % Q; }
  static __host__ __device__ constexpr int J(int r, int k) { return k == 0 ? r % Q : ((r - k) % Q + Q) % Q; }
};

template <int NC>
__host__ __device__ inline size_t ws_log_floats() {
  return (size_t)64 * (NC - 1);  // rotation log of one sweep: (NC-1) rounds x 32 float2
}
template <int NC>
__host__ __device__ inline size_t ws_floats_rj(int m) {  // planes, rotation log, Newton-Schulz T
  return (size_t)RJ<NC>::NPLANES * ((m + 1) & ~1) * NC + ws_log_floats<NC>() + (size_t)NC * NC;
}

// Per-warp context
template <int NC>
struct W {
  float* ws;                            // global planes (column stride LDP, plane stride ps)
  float* sm;                            // per-warp shared block
  int m, n, p, LDP, ps, lane;
  bool lok;                             // 2*lane < LDP (the lane owns stored rows)
  u64 vv;                               // normalised v-coordinates {v(2l), v(2l+1)}
  float cj, inv_s;
  __device__ __forceinline__ float* plane(int k) const { return ws + k * ps; }
  __device__ __forceinline__ float* D() const { return plane(0); }
  __device__ __forceinline__ float* A() const { return plane(1); }
  __device__ __forceinline__ float* E() const { return plane(2); }
  __device__ __forceinline__ float* Y() const { return plane(3); }
  __device__ __forceinline__ float* GX() const { return plane(4); }
  __device__ __forceinline__ float* GY() const { return plane(5); }
  __device__ __forceinline__ float* GZ() const { return plane(6); }
  __device__ __forceinline__ float* Bm() const { return plane(7); }
  __device__ __forceinline__ float2* logp() const { return reinterpret_cast<float2*>(plane(8)); }
  __device__ __forceinline__ float* Vs() const { return sm; }
  __device__ __forceinline__ float* Ts() const { return ws + RJ<NC>::NPLANES * ps + ws_log_floats<NC>(); }
  __device__ __forceinline__ float* Lp() const { return sm + RJ<NC>::OFF_LP; }
  __device__ __forceinline__ float* cp() const { return sm + RJ<NC>::OFF_CP; }
  __device__ __forceinline__ double* Linv() const { return reinterpret_cast<double*>(sm + RJ<NC>::OFF_LINV); }
  __device__ __forceinline__ u64 ld(const float* P, int j) const {
    return lok ? *reinterpret_cast<const u64*>(P + j * LDP + 2 * lane) : 0ull;
  }
  __device__ __forceinline__ void st(float* P, int j, u64 x) const {
    if (lok) *reinterpret_cast<u64*>(P + j * LDP + 2 * lane) = x;
  }
  __device__ __forceinline__ float ucol(int j) const { return ((float)j - cj) * inv_s; }
};

// ---------------------------------------------------------------------------------------------
// Implicit projector W^TW v = v - K K^T v (Eq. Jperpv, Eq. WTW_property):
// K^T v = L'(J_raw^T v) - c'(D_hat^T v), (K y)(px) = J_raw(px)(L'^T y) - D_hat(px)(c'^T y), with
// J_raw rows rebuilt per pixel from GX, GY, GZ and the pixel's (u, v) (see tilt_device.cuh).
// ---------------------------------------------------------------------------------------------
template <int NC, class VF>
__device__ __forceinline__ void proj_s(const W<NC>& w, VF vf, float (&s)[8]) {
  const bool homog = w.p == 8;
  const float *GX = w.GX(), *GY = w.GY(), *GZ = w.GZ(), *Dp = w.D();
  u64 a[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) a[k] = 0ull;
#pragma unroll 2
  for (int j = 0; j < w.n; ++j) {
    const u64 val = vf(j);
    const float u = w.ucol(j);
    const u64 ga = mul2(w.ld(GX, j), val), gb = mul2(w.ld(GY, j), val);
    a[0] = fmas2(ga, u, a[0]);
    a[1] = fma2(ga, w.vv, a[1]);
    a[2] = fmas2(gb, u, a[2]);
    a[3] = fma2(gb, w.vv, a[3]);
    a[4] = add2(a[4], ga);
    a[5] = add2(a[5], gb);
    if (homog) {
      const u64 gc = mul2(w.ld(GZ, j), val);
      a[6] = fmas2(gc, u, a[6]);
      a[7] = fma2(gc, w.vv, a[7]);
    }
    a[8] = fma2(w.ld(Dp, j), val, a[8]);
  }
  float r[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) r[k] = wsum(hsum(a[k]));
  const float* Lp = w.Lp();
  const float* cp = w.cp();
#pragma unroll
  for (int q = 0; q < 8; ++q) {  // s = K^T v = L' r[0:8] - c' r[8]
    float acc = -cp[q] * r[8];
#pragma unroll
    for (int b = 0; b <= q; ++b) acc = fmaf(Lp[q * 8 + b], r[b], acc);
    s[q] = acc;
  }
}

template <int NC, class VF>
__device__ __forceinline__ void proj_z(const W<NC>& w, VF vf, float (&z)[9]) {
  float s[8];
  proj_s<NC>(w, vf, s);
  const float* Lp = w.Lp();
  const float* cp = w.cp();
#pragma unroll
  for (int b = 0; b < 8; ++b) {  // z[0:8] = L'^T s, z[8] = c'^T s
    float acc = 0.f;
#pragma unroll
    for (int q = b; q < 8; ++q) acc = fmaf(Lp[q * 8 + b], s[q], acc);
    z[b] = acc;
  }
  float ww = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) ww = fmaf(cp[q], s[q], ww);
  z[8] = ww;
}

// (K y) at column j for the lane's two rows
template <int NC>
__device__ __forceinline__ u64 proj_apply(const W<NC>& w, int j, const float (&z)[9]) {
  const float u = w.ucol(j);
  const float s1 = fmaf(z[0], u, z[4]), s2 = fmaf(z[2], u, z[5]);
  const u64 c1 = fmas2(w.vv, z[1], pk(s1, s1));
  const u64 c2 = fmas2(w.vv, z[3], pk(s2, s2));
  u64 r = mul2(w.ld(w.GX(), j), c1);
  r = fma2(w.ld(w.GY(), j), c2, r);
  if (w.p == 8) {
    const float s3 = z[6] * u;
    const u64 c3 = fmas2(w.vv, z[7], pk(s3, s3));
    r = fma2(w.ld(w.GZ(), j), c3, r);
  }
  return fmas2(w.ld(w.D(), j), -z[8], r);
}

// Projector factors of one column (lane rows), loaded once and shared by apply + accumulate
struct ColG {
  u64 gx, gy, gz, d;
  float u;
};

template <int NC>
__device__ __forceinline__ ColG load_g(const W<NC>& w, const float* __restrict__ GX, const float* __restrict__ GY,
                                       const float* __restrict__ GZ, const float* __restrict__ Dp, int j) {
  ColG c;
  c.gx = w.ld(GX, j);
  c.gy = w.ld(GY, j);
  c.gz = w.p == 8 ? w.ld(GZ, j) : 0ull;
  c.d = w.ld(Dp, j);
  c.u = w.ucol(j);
  return c;
}

// (K z) at a column from its factors (as proj_apply)
template <int NC>
__device__ __forceinline__ u64 apply_g(const W<NC>& w, const ColG& c, const float (&z)[9]) {
  const float s1 = fmaf(z[0], c.u, z[4]), s2 = fmaf(z[2], c.u, z[5]), s3 = z[6] * c.u;
  u64 r = mul2(c.gx, fmas2(w.vv, z[1], pk(s1, s1)));
  r = fma2(c.gy, fmas2(w.vv, z[3], pk(s2, s2)), r);
  r = fma2(c.gz, fmas2(w.vv, z[7], pk(s3, s3)), r);  // gz = 0 for affine
  return fmas2(c.d, -z[8], r);
}

// accumulate the 9 projector sums of a column value (as proj_s)
__device__ __forceinline__ void accum_g(const ColG& c, u64 vv, u64 val, u64 (&a)[9]) {
  const u64 ga = mul2(c.gx, val), gb = mul2(c.gy, val), gc = mul2(c.gz, val);
  a[0] = fmas2(ga, c.u, a[0]);
  a[1] = fma2(ga, vv, a[1]);
  a[2] = fmas2(gb, c.u, a[2]);
  a[3] = fma2(gb, vv, a[3]);
  a[4] = add2(a[4], ga);
  a[5] = add2(a[5], gb);
  a[6] = fmas2(gc, c.u, a[6]);
  a[7] = fma2(gc, vv, a[7]);
  a[8] = fma2(c.d, val, a[8]);
}

// warp-reduce the sums and form z (as proj_z)
template <int NC>
__device__ __forceinline__ void finish_z(const W<NC>& w, const u64 (&a)[9], float (&z)[9]) {
  float r[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) r[k] = wsum(hsum(a[k]));
  const float* Lp = w.Lp();
  const float* cp = w.cp();
  float s[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float acc = -cp[q] * r[8];
#pragma unroll
    for (int b = 0; b <= q; ++b) acc = fmaf(Lp[q * 8 + b], r[b], acc);
    s[q] = acc;
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    float acc = 0.f;
#pragma unroll
    for (int q = b; q < 8; ++q) acc = fmaf(Lp[q * 8 + b], s[q], acc);
    z[b] = acc;
  }
  float ww = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) ww = fmaf(cp[q], s[q], ww);
  z[8] = ww;
}

// ---------------------------------------------------------------------------------------------
// Warm one-sided Jacobi, circle (round-robin) ordering, deferred V.
// A sweep first rotates only B (X, lane rows in registers): column pairs of a round are static
// register indices inside a body of RR rounds (the round's dots and rotations are specialised
// per round through a switch; reduction and parameter code are shared); between bodies the
// registers are shifted by RR along the ring. The rotation parameters of every round are logged
// (global workspace, L2); after the sweep B is parked in its plane and the same rotations are
// replayed on V (lane rows in registers), then B is reloaded. Each phase holds one 2 NC register
// array, so the kernel needs ~150 registers instead of 255 + spills.
// Parameter lane k holds the state of its pair's two columns: a = ||b||^2 (tracked), d = scale
// (b = d x). Rotation of (i, j) (tilt_jacobi.cuh): t = sgn(D) G/(|D| + sqrt(D^2+G^2)),
// D = a_j - a_i, G = 2 gamma, applied in place as two shears (see rotate_params); a_i -= t gamma,
// a_j += t gamma (exact for the rotation that orthogonalises i, j).
// ---------------------------------------------------------------------------------------------
struct Slot {
  float a, d;
};

struct RotOut {
  float ca, cb;
  Slot si, sj;
  bool doit, big;
};

__device__ __forceinline__ RotOut rotate_params(float g, Slot si, Slot sj, bool on, float tol2, float big2) {
  RotOut o;
  const float gam = g * si.d * sj.d;
  const float ab = si.a * sj.a;
  const bool doit = on && si.a > 0.f && sj.a > 0.f && gam * gam > tol2 * ab;
  const float D = sj.a - si.a, G = 2.f * gam;
  const float r2 = fmaf(D, D, G * G);
  const float den = fmaf(r2, rsqrt_approx(r2), fabsf(D));
  float t = G * rcp_approx(den);
  t = (D < 0.f) ? -t : t;
  t = doit ? t : 0.f;
  const float x2 = fmaf(t, t, 1.f);
  const float c = rsqrt_approx(x2);
  const float rr = sj.d * rcp_approx(si.d);  // d_j / d_i
  // in-place two-shear form: x_i <- x_i - ca x_j, then x_j <- x_j + cb x_i (new x_i), with
  // ca = t d_j/d_i, cb = t d_i/(d_j (1+t^2)); d_i <- c d_i, d_j <- sqrt(1+t^2) d_j, so that in the
  // b = d x frame the pair undergoes exactly b_i <- c(b_i - t b_j), b_j <- c(b_j + t b_i).
  o.ca = doit ? t * rr : 0.f;
  o.cb = doit ? t * rcp_approx(rr * x2) : 0.f;
  o.si.a = fmaxf(fmaf(-t, gam, si.a), 0.f);
  o.si.d = c * si.d;
  o.sj.a = fmaf(t, gam, sj.a);
  o.sj.d = (c * x2) * sj.d;
  o.doit = doit;
  o.big = doit && gam * gam > big2 * ab;
  return o;
}

__device__ __forceinline__ Slot shfl_down_slot(Slot s) {
  return Slot{__shfl_down_sync(FULL, s.a, 1), __shfl_down_sync(FULL, s.d, 1)};
}
__device__ __forceinline__ Slot shfl_up_slot(Slot s) {
  return Slot{__shfl_up_sync(FULL, s.a, 1), __shfl_up_sync(FULL, s.d, 1)};
}

// squared column norms of the round-0 pair of lane k: (top element, bottom element)
template <int NC>
__device__ __forceinline__ float2 pair_norms(const u64 (&X)[NC], int lane) {
  using R = RJ<NC>;
  float w[32];
#pragma unroll
  for (int k = 0; k < R::NH; ++k) w[k] = hsum(mul2(X[R::I(0, k)], X[R::I(0, k)]));
  const float t = treduce<R::NH>(w, lane);
#pragma unroll
  for (int k = 0; k < R::NH; ++k) w[k] = hsum(mul2(X[R::J(0, k)], X[R::J(0, k)]));
  const float b = treduce<R::NH>(w, lane);
  return make_float2(t, b);
}

// Lane k (< NH) publishes a float2 per element of its round-0 pair into wv (shared)
template <int NC>
__device__ __forceinline__ void publish_elems(float* sm, int lane, float2 top, float2 bot) {
  using R = RJ<NC>;
  float2* wv = reinterpret_cast<float2*>(sm + R::OFF_WV);
  __syncwarp();
  if (lane < R::NH) {
    wv[lane == 0 ? R::Q : lane] = top;  // elements I(0, k), J(0, k)
    wv[lane == 0 ? 0 : R::Q - lane] = bot;
  }
  __syncwarp();
}

// X[e] *= wv[e].x (SEL = 0) or .y (SEL = 1), element-wise
template <int NC, int SEL>
__device__ __forceinline__ void scale_by_wv(const float* sm, u64 (&X)[NC]) {
  using R = RJ<NC>;
  const float4* w4 = reinterpret_cast<const float4*>(sm + R::OFF_WV);
#pragma unroll
  for (int q = 0; q < R::NH; ++q) {
    const float4 c = w4[q];  // elements 2q, 2q+1
    X[2 * q] = muls2(X[2 * q], SEL ? c.y : c.x);
    X[2 * q + 1] = muls2(X[2 * q + 1], SEL ? c.w : c.z);
  }
}

template <int NC>
__device__ __forceinline__ void ring_shift(u64 (&X)[NC]) {
  using R = RJ<NC>;
  u64 T[NC];
#pragma unroll
  for (int e = 0; e < R::Q; ++e) T[e] = X[(e + R::RR) % R::Q];
#pragma unroll
  for (int e = 0; e < R::Q; ++e) X[e] = T[e];
}

// Column-pair dot products of circle round r (static register indices): g[k] = x_I . x_J (lane rows)
template <int NC, int r>
__device__ __forceinline__ void round_dots(const u64 (&X)[NC], float (&g)[32]) {
  using R = RJ<NC>;
#pragma unroll
  for (int k = 0; k < R::NH; ++k) g[k] = hsum(mul2(X[R::I(r, k)], X[R::J(r, k)]));
}

// In-place rotations of circle round r with the (ca, cb) of every pair (float4 = two pairs)
template <int NC, int r, class PF>
__device__ __forceinline__ void round_rot(u64 (&X)[NC], PF params) {
  using R = RJ<NC>;
#pragma unroll
  for (int q = 0; q < (R::NH + 1) / 2; ++q) {
    const float4 c = params(q);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * q + h;
      if (k >= R::NH) break;
      const float ca = h ? c.z : c.x, cb = h ? c.w : c.y;
      const int i = R::I(r, k), j = R::J(r, k);
      X[i] = fmas2(X[j], -ca, X[i]);  // x_i - ca x_j
      X[j] = fmas2(X[i], cb, X[j]);   // x_j + cb x_i(new)
    }
  }
}

template <int NC, class PF>
__device__ __forceinline__ void round_rot_dispatch(int r, u64 (&X)[NC], PF params) {
  switch (r) {
    case 0: round_rot<NC, 0>(X, params); break;
    case 1: round_rot<NC, 1>(X, params); break;
    case 2: round_rot<NC, 2>(X, params); break;
    case 3: round_rot<NC, 3>(X, params); break;
    case 4: round_rot<NC, 4>(X, params); break;
    case 5: round_rot<NC, 5>(X, params); break;
    default: round_rot<NC, 6>(X, params); break;
  }
}

struct SvtRes {
  float dA2, nuc, sig1;
  int rank, relrank, band, sweeps, rotations, capped;
};

// V rows of the lane <-> shared Vs (row-pair interleaved)
template <int NC>
__device__ __forceinline__ void load_vrows(const float* Vs, int lane, u64 (&V)[NC]) {
  if (lane < NC / 2) {
    const float4* src = reinterpret_cast<const float4*>(Vs + lane * NC * 2);
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      const float4 v = src[q];
      V[2 * q] = pk(v.x, v.y);
      V[2 * q + 1] = pk(v.z, v.w);
    }
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j) V[j] = 0ull;
  }
}
template <int NC>
__device__ __forceinline__ void store_vrows(float* Vs, int lane, const u64 (&V)[NC]) {
  __syncwarp();
  if (lane < NC / 2) {
    float4* dst = reinterpret_cast<float4*>(Vs + lane * NC * 2);
#pragma unroll
    for (int q = 0; q < NC / 2; ++q) {
      const float2 a = up(V[2 * q]), b = up(V[2 * q + 1]);
      dst[q] = make_float4(a.x, a.y, b.x, b.y);
    }
  }
  __syncwarp();
}

// B plane (lane rows, column stride LDP) <-> registers
template <int NC>
__device__ __forceinline__ void load_cols(const float* P, int LDP, int n, int lane, u64 (&X)[NC]) {
  const bool lok = 2 * lane < LDP;
#pragma unroll
  for (int j = 0; j < NC; ++j) X[j] = (lok && j < n) ? *reinterpret_cast<const u64*>(P + j * LDP + 2 * lane) : 0ull;
}
template <int NC>
__device__ __forceinline__ void store_cols(float* P, int LDP, int n, int lane, const u64 (&X)[NC]) {
  const bool lok = 2 * lane < LDP;
#pragma unroll
  for (int j = 0; j < NC; ++j)
    if (lok && j < n) *reinterpret_cast<u64*>(P + j * LDP + 2 * lane) = X[j];
}

// A = X V^T column pair (c, c+1) (c even) for the lane rows
template <int NC>
__device__ __forceinline__ void gemm_xvt_cols(const float* Vs, const u64 (&X)[NC], int c, u64& a0, u64& a1) {
  const float4* V4 = reinterpret_cast<const float4*>(Vs) + (c >> 1) * (NC / 2);
  u64 p0 = 0ull, p1 = 0ull, q0 = 0ull, q1 = 0ull;
#pragma unroll
  for (int jj = 0; jj < NC / 2; ++jj) {
    const float4 v = V4[jj];  // V[c][2jj], V[c+1][2jj], V[c][2jj+1], V[c+1][2jj+1]
    p0 = fmas2(X[2 * jj], v.x, p0);
    p1 = fmas2(X[2 * jj], v.y, p1);
    q0 = fmas2(X[2 * jj + 1], v.z, q0);
    q1 = fmas2(X[2 * jj + 1], v.w, q1);
  }
  a0 = add2(p0, q0);
  a1 = add2(p1, q1);
}

// One sweep on B (registers): all Q rounds, logging (ca, cb) of every pair of every round to
// logp[round][32] (float2). Returns with the lane states at round-0 pairs.
template <int NC>
__device__ __forceinline__ void sweep_b(u64 (&X)[NC], float2* Pw, float2* logp, int lane, Slot& top, Slot& bot,
                                        float tol2, float big2, bool& rot, bool& big, int& nrot) {
  using R = RJ<NC>;
#pragma unroll 1
  for (int body = 0; body < R::NB; ++body) {
#pragma unroll 1
    for (int r = 0; r < R::RR; ++r) {
      float g[32];
      switch (r) {
        case 0: round_dots<NC, 0>(X, g); break;
        case 1: round_dots<NC, 1>(X, g); break;
        case 2: round_dots<NC, 2>(X, g); break;
        case 3: round_dots<NC, 3>(X, g); break;
        case 4: round_dots<NC, 4>(X, g); break;
        case 5: round_dots<NC, 5>(X, g); break;
        default: round_dots<NC, 6>(X, g); break;
      }
      const float gk = treduce<R::NH>(g, lane);
      const RotOut o = rotate_params(gk, top, bot, lane < R::NH, tol2, big2);
      const float2 cc = make_float2(o.ca, o.cb);
      Pw[(r & 1) * 32 + lane] = cc;
      logp[(body * R::RR + r) * 32 + lane] = cc;
      rot |= o.doit;
      big |= o.big;
      nrot += o.doit ? 1 : 0;
      // states to the next round's pairs: tops come from lane k+1, bottoms from lane k-1
      const Slot tdn = shfl_down_slot(o.si);
      const Slot bup = shfl_up_slot(o.sj);
      top = lane == 0 ? o.si : (lane == R::NH - 1 ? o.sj : tdn);
      bot = lane == 0 ? tdn : bup;
      __syncwarp();
      const float4* P4 = reinterpret_cast<const float4*>(Pw + (r & 1) * 32);
      round_rot_dispatch<NC>(r, X, [&](int q) { return P4[q]; });
    }
    ring_shift<NC>(X);
  }
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Replay of a logged sweep on V (registers). The log (global, written by sweep_b) is staged into a
// shared ring of LOGRING rounds by cp.async, LOGRING - 1 rounds ahead of its use (each lane copies
// its own float2 of a round), so the replay never waits on L2.
template <int NC>
__device__ __forceinline__ void sweep_v(u64 (&V)[NC], const float2* logp, float* sm, int lane) {
  using R = RJ<NC>;
  constexpr int NR = R::Q;  // rounds per sweep
  constexpr int AHEAD = R::LOGRING - 1;
  float2* ring = reinterpret_cast<float2*>(sm + R::OFF_RING);
#pragma unroll
  for (int r = 0; r < AHEAD; ++r) {
    if (r < NR) cp_async8(ring + r * 32 + lane, logp + r * 32 + lane);
    cp_async_commit();
  }
#pragma unroll 1
  for (int body = 0; body < R::NB; ++body) {
#pragma unroll 1
    for (int r = 0; r < R::RR; ++r) {
      const int g = body * R::RR + r;
      const int ahead = g + AHEAD;
      if (ahead < NR) cp_async8(ring + (ahead % R::LOGRING) * 32 + lane, logp + ahead * 32 + lane);
      cp_async_commit();
      cp_async_wait<AHEAD>();  // round g has landed (this lane's part)
      __syncwarp();            // ... and every other lane's part
      const float4* P4 = reinterpret_cast<const float4*>(ring + (g % R::LOGRING) * 32);
      round_rot_dispatch<NC>(r, V, [&](int q) { return P4[q]; });
      __syncwarp();  // the slot is refilled LOGRING - 1 rounds later
    }
    ring_shift<NC>(V);
  }
  cp_async_wait<0>();
}

// Singular value thresholding S_eps (Eqs. A_1, S_operator) of M, given B = M V in the
// B plane (lane rows, column stride LDP) and the warm V (shared Vs). Warm one-sided Jacobi to
// convergence (reading Z14); then sigma_j = ||b_j||/||v_j||, h_j = max(sigma_j - eps, 0)/sigma_j,
// V columns normalised and stored back (warm start of the next SVT), and, if Ap is given,
// A = B diag(h) V^T written to the A plane with ||A - A_old||_F^2 returned in dA2.
// logp: per-warp rotation log (global, (NC-1) x 32 float2).
template <int NC>
__device__ __noinline__ SvtRes svt_rj(float* Bp, float* Ap, float* sm, float2* logp, int LDP, int n, float eps,
                                      float tol, int max_sweeps) {
  using R = RJ<NC>;
  const int lane = threadIdx.x & 31;
  float2* Pw = reinterpret_cast<float2*>(sm + R::OFF_PW);
  SvtRes res;
  res.sweeps = 0;
  int nrot = 0;
  bool any = false;
  const float tol2 = tol * tol;
  const float big2 = tol / (float)n;
  float2 nr, vn;
  {
    u64 X[NC];
    load_cols<NC>(Bp, LDP, n, lane, X);
    nr = pair_norms<NC>(X, lane);
  }
  while (true) {
    bool rot = false, big = false;
    {
      u64 X[NC];
      load_cols<NC>(Bp, LDP, n, lane, X);
      Slot top{nr.x, 1.f}, bot{nr.y, 1.f};
      sweep_b<NC>(X, Pw, logp, lane, top, bot, tol2, big2, rot, big, nrot);
      // scales d -> wv[e].x (for B) and .y (for V)
      publish_elems<NC>(sm, lane, make_float2(top.d, top.d), make_float2(bot.d, bot.d));
      scale_by_wv<NC, 0>(sm, X);
      nr = pair_norms<NC>(X, lane);  // fresh ||b_j||^2 (round-0 pairs)
      store_cols<NC>(Bp, LDP, n, lane, X);
    }
    __syncwarp();
    {
      u64 V[NC];
      load_vrows<NC>(sm, lane, V);
      sweep_v<NC>(V, logp, sm, lane);
      scale_by_wv<NC, 1>(sm, V);
      vn = pair_norms<NC>(V, lane);
      store_vrows<NC>(sm, lane, V);
    }
    ++res.sweeps;
    any = __any_sync(FULL, rot);
    const bool more = __any_sync(FULL, big);
    if (!more) {
      any = false;
      break;
    }
    if (res.sweeps >= max_sweeps) break;
  }
  res.capped = any ? 1 : 0;
  res.rotations = wsumi(nrot);
  // ---- sigma_j = ||b_j||/||v_j||, h_j; V <- V diag(1/||v_j||), B <- B diag(h_j/||v_j||) ------
  {
    const float bbs[2] = {nr.x, nr.y}, vvs[2] = {vn.x, vn.y};
    float sg[2], xs[2], vs[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool ok = lane < R::NH && vvs[e] > 0.f;
      sg[e] = ok ? sqrtf(bbs[e] / vvs[e]) : 0.f;
      const float h = (sg[e] > eps) ? (sg[e] - eps) / sg[e] : 0.f;
      const float iv = ok ? rsqrtf(vvs[e]) : 0.f;
      xs[e] = h * iv;
      vs[e] = iv;
    }
    publish_elems<NC>(sm, lane, make_float2(xs[0], vs[0]), make_float2(xs[1], vs[1]));
    {
      u64 V[NC];
      load_vrows<NC>(sm, lane, V);
      scale_by_wv<NC, 1>(sm, V);
      store_vrows<NC>(sm, lane, V);
    }
    float nuc = 0.f, smax = 0.f, amax = 0.f;
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float a = fmaxf(sg[e] - eps, 0.f);
      nuc += a;
      smax = fmaxf(smax, sg[e]);
      amax = fmaxf(amax, a);
      cnt += sg[e] > eps ? 1 : 0;
    }
    res.nuc = wsum(nuc);
    res.sig1 = wmax(smax);
    amax = wmax(amax);
    res.rank = wsumi(cnt);
    int rel = 0, band = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const float a = fmaxf(sg[e] - eps, 0.f);
      if (amax > 0.f) {
        const float ratio = a / amax;
        rel += ratio > 1e-3f ? 1 : 0;
        band |= (ratio >= 3e-4f && ratio <= 3e-3f) ? 1 : 0;
      }
    }
    res.relrank = wsumi(rel);
    res.band = __any_sync(FULL, band) ? 1 : 0;
    // A = B diag(h / ||v||) V^T; the per-element sigma goes to wv[e].y for the standalone entry
    float dA2 = 0.f;
    {
      u64 X[NC];
      load_cols<NC>(Bp, LDP, n, lane, X);
      scale_by_wv<NC, 0>(sm, X);
      publish_elems<NC>(sm, lane, make_float2(sg[0], sg[0]), make_float2(sg[1], sg[1]));
      if (Ap) {
        const bool lok = 2 * lane < LDP;
#pragma unroll 1
        for (int c0 = 0; c0 < n; c0 += 2) {
          u64 a0, a1;
          gemm_xvt_cols<NC>(sm, X, c0, a0, a1);
          if (lok) {
            u64* p0 = reinterpret_cast<u64*>(Ap + c0 * LDP + 2 * lane);
            const u64 d0 = sub2(a0, *p0);
            dA2 += hsum(mul2(d0, d0));
            *p0 = a0;
            if (c0 + 1 < n) {
              u64* p1 = reinterpret_cast<u64*>(Ap + (c0 + 1) * LDP + 2 * lane);
              const u64 d1 = sub2(a1, *p1);
              dA2 += hsum(mul2(d1, d1));
              *p1 = a1;
            }
          }
        }
      }
    }
    res.dA2 = wsum(dA2);
  }
  return res;
}

template <int NC>
__device__ __forceinline__ void set_identity_v(float* Vs, int lane, int n) {
  for (int e = lane; e < NC * NC; e += 32) {
    const int h = e & 1, jq = e >> 1, j = jq % NC, q = jq / NC;
    Vs[e] = (2 * q + h == j && j < n) ? 1.f : 0.f;
  }
  __syncwarp();
}

// Newton-Schulz step on the shared V (reading Z14): G = V^T V, T = 1.5 I - 0.5 G, V <- V T.
// Output columns are produced in blocks of CBP column pairs to bound the live registers.
template <int NC>
__device__ __noinline__ void ns_step(float* sm, float* Ts) {
  constexpr int NH = NC / 2;
  constexpr int CBP = (NH % 5 == 0) ? 5 : (NH % 6 == 0 ? 6 : (NH % 4 == 0 ? 4 : (NH % 3 == 0 ? 3 : 1)));
  const int lane = threadIdx.x & 31;
  float* Vs = sm;
  const float4* V4 = reinterpret_cast<const float4*>(Vs);
  float4* T4 = reinterpret_cast<float4*>(Ts);
  if (lane < NH) {
#pragma unroll 1
    for (int blk = 0; blk < NH; blk += CBP) {  // G rows 2l, 2l+1, columns 2bb, 2bb+1 of the block
      u64 acc[2 * CBP];
#pragma unroll
      for (int b = 0; b < 2 * CBP; ++b) acc[b] = 0ull;
#pragma unroll 1
      for (int q = 0; q < NH; ++q) {
        const float4 own = V4[q * NH + lane];  // V[2q][2l], V[2q+1][2l], V[2q][2l+1], V[2q+1][2l+1]
        const u64 o0 = pk(own.x, own.z), o1 = pk(own.y, own.w);
#pragma unroll
        for (int c = 0; c < CBP; ++c) {
          const float4 v = V4[q * NH + blk + c];
          acc[2 * c] = fmas2(o0, v.x, acc[2 * c]);
          acc[2 * c] = fmas2(o1, v.y, acc[2 * c]);
          acc[2 * c + 1] = fmas2(o0, v.z, acc[2 * c + 1]);
          acc[2 * c + 1] = fmas2(o1, v.w, acc[2 * c + 1]);
        }
      }
#pragma unroll
      for (int c = 0; c < CBP; ++c) {  // T rows 2l, 2l+1 in the row-pair interleaved layout
        const int bb = blk + c;
        const float2 g0 = up(acc[2 * c]), g1 = up(acc[2 * c + 1]);
        const float t00 = (2 * bb == 2 * lane ? 1.5f : 0.f) - 0.5f * g0.x;
        const float t10 = (2 * bb == 2 * lane + 1 ? 1.5f : 0.f) - 0.5f * g0.y;
        const float t01 = (2 * bb + 1 == 2 * lane ? 1.5f : 0.f) - 0.5f * g1.x;
        const float t11 = (2 * bb + 1 == 2 * lane + 1 ? 1.5f : 0.f) - 0.5f * g1.y;
        T4[lane * NH + bb] = make_float4(t00, t10, t01, t11);
      }
    }
  }
  __syncwarp();
  if (lane < NH) {
    u64 vr[NC];  // the lane's own V rows (2l, 2l+1), all columns
#pragma unroll
    for (int q = 0; q < NH; ++q) {
      const float4 own = V4[lane * NH + q];  // V[2l][2q], V[2l+1][2q], V[2l][2q+1], V[2l+1][2q+1]
      vr[2 * q] = pk(own.x, own.y);
      vr[2 * q + 1] = pk(own.z, own.w);
    }
    float4* dst = reinterpret_cast<float4*>(Vs) + lane * NH;
#pragma unroll 1
    for (int blk = 0; blk < NH; blk += CBP) {  // V_new rows 2l, 2l+1, column pairs of the block
      u64 acc[2 * CBP];
#pragma unroll
      for (int b = 0; b < 2 * CBP; ++b) acc[b] = 0ull;
#pragma unroll
      for (int q = 0; q < NH; ++q) {
#pragma unroll
        for (int c = 0; c < CBP; ++c) {
          const float4 t = __ldcg(T4 + q * NH + blk + c);  // T[2q][2cc], T[2q+1][2cc], T[2q][2cc+1], T[2q+1][2cc+1]
          acc[2 * c] = fmas2(vr[2 * q], t.x, acc[2 * c]);
          acc[2 * c] = fmas2(vr[2 * q + 1], t.y, acc[2 * c]);
          acc[2 * c + 1] = fmas2(vr[2 * q], t.z, acc[2 * c + 1]);
          acc[2 * c + 1] = fmas2(vr[2 * q + 1], t.w, acc[2 * c + 1]);
        }
      }
#pragma unroll
      for (int c = 0; c < CBP; ++c) {
        const float2 x = up(acc[2 * c]), y = up(acc[2 * c + 1]);
        dst[blk + c] = make_float4(x.x, x.y, y.x, y.y);
      }
    }
  }
  __syncwarp();
}

// X (= B) += M[:, k], M[:, k+1] (lane rows) times V rows k, k+1 (k even)
template <int NC>
__device__ __forceinline__ void gemm_mv_acc(const float* Vs, u64 (&X)[NC], int k, u64 mk, u64 mk1) {
  const float4* V4 = reinterpret_cast<const float4*>(Vs) + (k >> 1) * (NC / 2);
#pragma unroll
  for (int jj = 0; jj < NC / 2; ++jj) {
    const float4 v = V4[jj];  // V[k][2jj], V[k+1][2jj], V[k][2jj+1], V[k+1][2jj+1]
    X[2 * jj] = fmas2(mk, v.x, X[2 * jj]);
    X[2 * jj] = fmas2(mk1, v.y, X[2 * jj]);
    X[2 * jj + 1] = fmas2(mk, v.z, X[2 * jj + 1]);
    X[2 * jj + 1] = fmas2(mk1, v.w, X[2 * jj + 1]);
  }
}

// The B plane <- M V with M's column pairs produced by mcol(k) (k even: returns M[:, k], M[:, k+1])
template <int NC, class MF>
__device__ __forceinline__ void build_b(const W<NC>& w, float* Bp, MF mcol) {
  u64 X[NC];
#pragma unroll
  for (int j = 0; j < NC; ++j) X[j] = 0ull;
  const float* Vs = w.Vs();
#pragma unroll 1
  for (int k = 0; k < w.n; k += 2) {
    u64 m0, m1;
    mcol(k, m0, m1);
    gemm_mv_acc<NC>(Vs, X, k, m0, m1);
  }
#pragma unroll
  for (int j = 0; j < NC; ++j)
    if (j < w.n) w.st(Bp, j, X[j]);
}

// ---------------------------------------------------------------------------------------------
// Algorithm 1 for one patch on one warp (as solve_patch, tilt_kernels.cuh)
// ---------------------------------------------------------------------------------------------
template <int NC>
__device__ void solve_patch_rj(const SolveArgs& a, const W<NC>& w, int b) {
  const DevParams& P = a.P;
  const int lane = w.lane;
  const int m = a.m, n = a.n, p = a.p;
  const int bx[4] = {a.boxes[4 * b], a.boxes[4 * b + 1], a.boxes[4 * b + 2], a.boxes[4 * b + 3]};
  const float* img = a.images + (size_t)a.patch_image[b] * a.H * a.W;
  double tau[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) tau[q] = 0.0;
  if (a.tau0) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < p) tau[q] = a.tau0[b * p + q];
  } else {
    tau[0] = 1.0;
    tau[3] = 1.0;
  }
  const float lam = P.lambda > 0.f ? P.lambda : rsqrtf((float)max(m, n));
  const float tol = P.jacobi_tol > 0.f ? P.jacobi_tol : default_jacobi_tol(m);
  const bool warm = P.svd_warm != 0;
  const bool homog = p == 8;
  float* Vs = w.Vs();
  float *Dp = w.D(), *Ap = w.A(), *Ep = w.E(), *Yp = w.Y();
  for (int j = 0; j < NC; ++j)  // zero the planes (padding rows/columns stay 0)
    for (int k = 0; k < RJ<NC>::NPLANES; ++k) w.st(w.plane(k), j, 0ull);
  set_identity_v<NC>(Vs, lane, n);
  int status = TILT_PATCH_MAX_OUTER, stop_rule = 0, outer = 0, inner_total = 0, sweeps_total = 0, aux_total = 0,
      caps = 0, rank = 0, band = 0, svt_rank = 0, rot_total = 0;
  const float fnan = __int_as_float(0x7fc00000);
  float f = fnan, f_prev = fnan, crit1 = fnan, crit2 = fnan, dtau_inf = fnan, mu_last = fnan, nd = fnan;
  bool have_state = false, have_fprev = false;
  const bool box_ok = bx[2] == n && bx[3] == m;  // all boxes of a call share the window size
  if (!box_ok) status = TILT_PATCH_BAD_BOX;
  const int n_outer = !box_ok ? 0 : P.fixed_outer > 0 ? P.fixed_outer : P.max_outer;
  const int r0 = 2 * lane;
  for (int it = 0; it < n_outer; ++it) {
    // ---- Step 1: D o tau and the Jacobian factors (fp64 per pixel), escape check ------------
    {
      const WarpGeom g = make_geom(bx, tau, a.kind);
      bool esc = false;
      for (int j = 0; j < n; ++j) {
        float dv[2], gxv[2], gyv[2], gzv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = r0 + h;
          double d = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
          if (i < m) {
            if (!warp_pixel(g, img, a.H, a.W, i, j, d, gx, gy, gz)) esc = true;
          }
          dv[h] = (float)d;
          gxv[h] = (float)gx;
          gyv[h] = (float)gy;
          gzv[h] = (float)gz;
        }
        w.st(Dp, j, pk(dv[0], dv[1]));
        w.st(w.GX(), j, pk(gxv[0], gxv[1]));
        w.st(w.GY(), j, pk(gyv[0], gyv[1]));
        if (homog) w.st(w.GZ(), j, pk(gzv[0], gzv[1]));
      }
      if (__any_sync(FULL, esc)) {
        status = TILT_PATCH_WINDOW_ESCAPE;
        break;
      }
    }
    // ---- orthonormalise (implicit projector), fp64 (as orthonormalise_implicit) --------------
    const double inv_s = (double)w.inv_s;
    auto rawrow = [&](int i, int j, double (&jr)[8], double& d) {
      const int h = i - r0;
      const float2 D2 = up(w.ld(Dp, j)), X2 = up(w.ld(w.GX(), j)), Y2 = up(w.ld(w.GY(), j));
      const float2 Z2 = homog ? up(w.ld(w.GZ(), j)) : make_float2(0.f, 0.f);
      d = h ? D2.y : D2.x;
      const double u = ((double)j - (double)w.cj) * inv_s;
      const double v = ((double)i - (double)(0.5f * (float)(m - 1))) * inv_s;
      jraw_row(h ? X2.y : X2.x, h ? Y2.y : Y2.x, homog ? (double)(h ? Z2.y : Z2.x) : 0.0, u, v, jr);
    };
    double acc[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] = 0.0;
    for (int j = 0; j < n; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = r0 + h;
        if (i >= m) continue;
        double jr[8], d;
        rawrow(i, j, jr, d);
        acc[8] = fma(d, d, acc[8]);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = fma(jr[q], d, acc[q]);
      }
    }
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e] = wsumd(acc[e]);
    const double ndd = sqrt(acc[8]);
    nd = (float)ndd;
    if (!(ndd > 0.0)) {
      status = TILT_PATCH_ZERO_PATCH;
      break;
    }
    const double ind = 1.0 / ndd;
    double c[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = acc[q] * ind;
    double G[36];
#pragma unroll
    for (int e = 0; e < 36; ++e) G[e] = 0.0;
    for (int j = 0; j < n; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = r0 + h;
        if (i >= m) continue;
        double jr[8], d;
        rawrow(i, j, jr, d);
        const double dh = d * ind;
        double jn[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) jn[q] = (q < p) ? (jr[q] - dh * c[q]) * ind : 0.0;
        int e = 0;
#pragma unroll
        for (int aa = 0; aa < 8; ++aa)
#pragma unroll
          for (int bb = aa; bb < 8; ++bb) {
            G[e] = fma(jn[aa], jn[bb], G[e]);
            ++e;
          }
      }
    }
#pragma unroll
    for (int e = 0; e < 36; ++e) G[e] = wsumd(G[e]);
    {
      double qr[24];
      int l = 0;
      if (P.constraint_mode == TILT_CONSTRAINTS_CENTER_AREA) {
        constraint_rows(tau, a.kind, m, n, qr);
        l = 3;
      }
      __syncwarp();
      int ok = 1;
      if (lane == 0) {
        double Li[64];
        ok = chol_inverse(G, qr, l, p, Li) ? 1 : 0;
        if (ok) {
          for (int aa = 0; aa < 8; ++aa) {
            double cpa = 0.0;
            for (int bb = 0; bb < 8; ++bb) {
              w.Lp()[aa * 8 + bb] = (float)(Li[aa * 8 + bb] * ind);
              cpa += Li[aa * 8 + bb] * c[bb];
              w.Linv()[aa * 8 + bb] = Li[aa * 8 + bb];
            }
            w.cp()[aa] = (float)(cpa * ind);
          }
        }
      }
      ok = __shfl_sync(FULL, ok, 0);
      __syncwarp();
      if (!ok) {
        status = TILT_PATCH_SINGULAR_GRAM;
        break;
      }
    }
    for (int j = 0; j < n; ++j) {  // D <- D_hat (in place, (float)(d * ind) of the fp32 d)
      const float2 d2 = up(w.ld(Dp, j));
      w.st(Dp, j, pk((float)((double)d2.x * ind), (float)((double)d2.y * ind)));
    }
    // ---- Step 2 warm start (Eq. warm_start; Eq. Y_new_warmstart; Z4) ----
    float z[9];
    if (!have_state || !P.vws) {
      for (int j = 0; j < n; ++j) {
        w.st(Ap, j, w.ld(Dp, j));
        w.st(Ep, j, 0ull);
        w.st(Yp, j, 0ull);
      }
    } else {
      proj_z<NC>(w, [&](int j) { return w.ld(Yp, j); }, z);
      for (int j = 0; j < n; ++j) w.st(Yp, j, sub2(w.ld(Yp, j), proj_apply<NC>(w, j, z)));
    }
    // denom = ||W^TW D_hat||_F (reading Z11)
    proj_z<NC>(w, [&](int j) { return w.ld(Dp, j); }, z);
    float dn = 0.f;
    for (int j = 0; j < n; ++j) {
      const u64 r = sub2(w.ld(Dp, j), proj_apply<NC>(w, j, z));
      dn += hsum(mul2(r, r));
    }
    const float denom0 = sqrtf(wsum(dn));
    const float denom = denom0 > 0.f ? denom0 : 1.f;
    const float inv_den = 1.f / denom;
    // sigma_1(D_hat) by the warm SVD (reading Z3)
    if (!warm) set_identity_v<NC>(Vs, lane, n);
    build_b<NC>(w, w.Bm(), [&](int k, u64& m0, u64& m1) {
      m0 = w.ld(Dp, k);
      m1 = k + 1 < n ? w.ld(Dp, k + 1) : 0ull;
    });
    const SvtRes s1r = svt_rj<NC>(w.Bm(), nullptr, w.sm, w.logp(), w.LDP, n, 0.f, tol, P.jacobi_max_sweeps);
    aux_total += s1r.sweeps;
    const float s1 = s1r.sig1;
    const float mu0 = s1 > 0.f ? P.mu0_scale / s1 : P.mu0_scale;
    const float mu_max = P.mu_max_ratio * mu0;
    // ---- M_0 = A - W^TW(A + E - D) - Y/mu0, B = M_0 V --------------------------------------
    {
      proj_z<NC>(w, [&](int j) { return res3_2(w.ld(Ap, j), w.ld(Ep, j), w.ld(Dp, j)); }, z);
      const float inv = 1.f / mu0;
      build_b<NC>(w, w.Bm(), [&](int k, u64& m0, u64& m1) {
        u64 mk[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = k + h;
          if (j >= n) {
            mk[h] = 0ull;
            continue;
          }
          const u64 av = w.ld(Ap, j);
          const u64 v = res3_2(av, w.ld(Ep, j), w.ld(Dp, j));
          const u64 r = sub2(v, proj_apply<NC>(w, j, z));
          mk[h] = fmas2(w.ld(Yp, j), -inv, sub2(av, r));
        }
        m0 = mk[0];
        m1 = mk[1];
      });
    }
    // ---- LADMAP inner loop (as ladmap_inner, tilt_kernels.cuh) -------------------------------
    const size_t toff = ((size_t)b * P.max_outer + it) * P.max_inner;
    const uint8_t* replay = P.rho_replay ? P.rho_replay + toff : nullptr;
    float* trace = P.trace ? P.trace + 4 * toff : nullptr;
    const int niter = P.fixed_inner > 0 ? P.fixed_inner : P.max_inner;
    float mu = mu0;
    int iters = 0;
    float c1v = fnan, c2v = fnan;
    SvtRes sst;
    sst.nuc = 0.f;
    sst.relrank = sst.band = sst.rank = 0;
    for (int k = 0; k < niter; ++k) {
      // A step: A_{k+1} = S_{1/mu}(M_k) (B = M_k V in the B plane)
      sst = svt_rj<NC>(w.Bm(), Ap, w.sm, w.logp(), w.LDP, n, 1.f / mu, tol, P.jacobi_max_sweeps);
      sweeps_total += sst.sweeps;
      caps += sst.capped;
      rot_total += sst.rotations;
      if (warm && (k % P.ns_period == P.ns_period - 1 || k + 1 == niter)) ns_step<NC>(w.sm, w.Ts());
      // E step: N_k = E_k - W^TW(A_{k+1} + E_k - D) - Y/mu, E_{k+1} = T_{lam/mu}(N_k); the same
      // pass accumulates the projector sums of A_{k+1} + E_{k+1} - D for the dual step
      const float inv_mu = 1.f / mu;
      const float thr = lam * inv_mu;
      const float *__restrict__ GXp = w.GX(), *__restrict__ GYp = w.GY(), *__restrict__ GZp = w.GZ();
      proj_z<NC>(w, [&](int j) { return res3_2(w.ld(Ap, j), w.ld(Ep, j), w.ld(Dp, j)); }, z);
      float dE2 = 0.f;
      u64 acc[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] = 0ull;
#pragma unroll 4
      for (int j = 0; j < n; ++j) {
        const ColG cg = load_g<NC>(w, GXp, GYp, GZp, Dp, j);
        const u64 e = w.ld(Ep, j), av = w.ld(Ap, j), yv = w.ld(Yp, j);
        const u64 v = res3_2(av, e, cg.d);
        const u64 pv = sub2(v, apply_g<NC>(w, cg, z));
        const u64 nk = fmas2(yv, -inv_mu, sub2(e, pv));
        const u64 en = shrink2(nk, thr);
        const u64 d = sub2(en, e);
        dE2 += hsum(mul2(d, d));
        w.st(Ep, j, en);
        accum_g(cg, w.vv, res3_2(av, en, cg.d), acc);
      }
      dE2 = wsum(dE2);
      const float c2 = mu * sqrtf(fmaxf(sst.dA2, dE2)) * inv_den;
      int rho_bit = c2 < P.eps2 ? 1 : 0;
      if (replay) rho_bit = replay[k] & 1;
      const float mu_next = fminf(mu_max, rho_bit ? P.rho0 * mu : mu);
      const float inv_mun = 1.f / mu_next;
      // dual step (Y += mu R, erratum E1) + next M = A - R - Y/mu_next, B = M V
      finish_z<NC>(w, acc, z);
      float c1 = 0.f;
      build_b<NC>(w, w.Bm(), [&](int kk, u64& m0, u64& m1) {
        u64 mk[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = kk + h;
          if (j >= n) {
            mk[h] = 0ull;
            continue;
          }
          const ColG cg = load_g<NC>(w, GXp, GYp, GZp, Dp, j);
          const u64 av = w.ld(Ap, j);
          const u64 v = res3_2(av, w.ld(Ep, j), cg.d);
          const u64 r = sub2(v, apply_g<NC>(w, cg, z));
          const u64 y = fmas2(r, mu, w.ld(Yp, j));
          w.st(Yp, j, y);
          c1 += hsum(mul2(r, r));
          mk[h] = fmas2(y, -inv_mun, sub2(av, r));
        }
        m0 = mk[0];
        m1 = mk[1];
      });
      const float cr1 = sqrtf(wsum(c1)) * inv_den;
      if (trace && lane == 0) {
        trace[4 * k + 0] = mu;
        trace[4 * k + 1] = cr1;
        trace[4 * k + 2] = c2;
        trace[4 * k + 3] = (float)rho_bit;
      }
      iters = k + 1;
      c1v = cr1;
      c2v = c2;
      mu_last = mu;
      bool stop = cr1 < P.eps1 && c2 < P.eps2;
      if (replay) stop = (replay[k] & 2) != 0;
      if (stop && P.fixed_inner <= 0) break;
      mu = mu_next;
    }
    have_state = true;
    inner_total += iters;
    crit1 = c1v;
    crit2 = c2v;
    rank = sst.relrank;
    band = sst.band;
    svt_rank = sst.rank;
    // ---- Step 3: dtau = L^{-T} K^T (A + E - D_hat) (Eq. Delta_tau) ---------------------------
    float s[8];
    proj_s<NC>(w, [&](int j) { return res3_2(w.ld(Ap, j), w.ld(Ep, j), w.ld(Dp, j)); }, s);
    float l1 = 0.f;
    for (int j = 0; j < n; ++j) {
      const float2 e2 = up(w.ld(Ep, j));
      l1 += fabsf(e2.x) + fabsf(e2.y);
    }
    l1 = wsum(l1);
    double dt_inf = 0.0;
    bool finite = true;
    const double* Linv = w.Linv();
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // Step 4: tau += dtau
      if (q >= p) continue;
      double dq = 0.0;
      for (int r = q; r < p; ++r) dq += Linv[r * 8 + q] * (double)s[r];
      tau[q] = (double)(float)(tau[q] + dq);  // tau carried in fp32 between outer iterations (Z28)
      dt_inf = fmax(dt_inf, fabs(dq));
      finite = finite && isfinite(tau[q]);
    }
    dtau_inf = (float)dt_inf;
    f = sst.nuc + lam * l1;
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
  }
  // ---- outputs (row-major [m][n]) ----------------------------------------------------------
  __syncwarp();
  float* outs[3] = {a.A_out, a.E_out, a.Y_out};
  const float* src[3] = {Ap, Ep, Yp};
  for (int o = 0; o < 3; ++o) {
    if (!outs[o]) continue;
    float* dst = outs[o] + (size_t)b * m * n;
    for (int e = lane; e < m * n; e += 32) {
      const int i = e / n, j = e - i * n;
      dst[e] = have_state ? src[o][j * w.LDP + i] : 0.f;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < p) a.tau_out[b * p + q] = (float)tau[q];
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
      r.kernel_path = 2;
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
  __syncwarp();
}

template <int NC>
__device__ __forceinline__ W<NC> make_w(float* smem_warp, float* ws_warp, int m, int n, int p) {
  W<NC> w;
  w.lane = threadIdx.x & 31;
  w.m = m;
  w.n = n;
  w.p = p;
  w.LDP = (m + 1) & ~1;
  w.ps = w.LDP * NC;
  w.lok = 2 * w.lane < w.LDP;
  w.ws = ws_warp;
  w.sm = smem_warp;
  const float s = 0.5f * (float)max(m, n);
  w.inv_s = 1.f / s;
  w.cj = 0.5f * (float)(n - 1);
  const float ci = 0.5f * (float)(m - 1);
  w.vv = pk(((float)(2 * w.lane) - ci) * w.inv_s, ((float)(2 * w.lane + 1) - ci) * w.inv_s);
  return w;
}

template <int NC>
__global__ void __launch_bounds__(RJ<NC>::NT, 3) k_solve_rj(SolveArgs a) {
  extern __shared__ float4 dsm4[];
  const int wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * RJ<NC>::WPB + wid;
  float* smem = reinterpret_cast<float*>(dsm4) + wid * RJ<NC>::SMF;
  float* ws = a.ws + (size_t)gw * a.ws_stride;
  const W<NC> w = make_w<NC>(smem, ws, a.m, a.n, a.p);
  while (true) {
    int b = 0;
    if (w.lane == 0) b = atomicAdd(a.counter, 1);
    b = __shfl_sync(FULL, b, 0);
    if (b >= a.B) break;
    solve_patch_rj<NC>(a, w, b);
  }
}

// Standalone SVT on the warp-per-patch path (step parity of the K3 core): V_io warm start / output.
// Workspace per warp: the B and A planes (2 x LDP x NC floats) and the rotation log.
template <int NC>
__global__ void __launch_bounds__(RJ<NC>::NT, 3) k_svt_rj(SvtArgs a) {
  extern __shared__ float4 dsm4[];
  const int wid = threadIdx.x >> 5;
  float* smem = reinterpret_cast<float*>(dsm4) + wid * RJ<NC>::SMF;
  const int m = a.m, n = a.n;
  const int gw = blockIdx.x * RJ<NC>::WPB + wid;
  const W<NC> w = make_w<NC>(smem, a.ws + (size_t)gw * a.ws_stride, m, n, 0);
  const int lane = w.lane;
  float* Bp = w.plane(0);
  float* Ap = w.plane(1);
  float2* logp = reinterpret_cast<float2*>(w.plane(2));  // after the two planes
  for (int b = gw; b < a.B; b += gridDim.x * RJ<NC>::WPB) {
    const float* M = a.M + (size_t)b * m * n;
    if (a.V_io) {  // Vs <- V_io (row-major n x n) or I
      const float* Vi = a.V_io + (size_t)b * n * n;
      for (int e = lane; e < NC * NC; e += 32) {
        const int h = e & 1, jq = e >> 1, j = jq % NC, q = jq / NC, r = 2 * q + h;
        w.Vs()[e] = (r < n && j < n) ? Vi[r * n + j] : 0.f;
      }
      __syncwarp();
    } else {
      set_identity_v<NC>(w.Vs(), lane, n);
    }
    auto mval = [&](int j) -> u64 {
      if (j >= n) return 0ull;
      const float x0 = (2 * lane < m) ? M[(2 * lane) * n + j] : 0.f;
      const float x1 = (2 * lane + 1 < m) ? M[(2 * lane + 1) * n + j] : 0.f;
      return pk(x0, x1);
    };
    for (int j = 0; j < NC; ++j) w.st(Ap, j, 0ull);
    build_b<NC>(w, Bp, [&](int k, u64& m0, u64& m1) {
      m0 = mval(k);
      m1 = mval(k + 1);
    });
    const SvtRes r = svt_rj<NC>(Bp, Ap, w.sm, logp, w.LDP, n, a.eps[b], a.tol, a.max_sweeps);
    __syncwarp();
    float* Ab = a.A + (size_t)b * m * n;
    for (int e = lane; e < m * n; e += 32) {
      const int i = e / n, j = e - i * n;
      Ab[e] = Ap[j * w.LDP + i];
    }
    if (a.sigma) {  // singular values of M, unsorted (element order)
      const float2* wv = reinterpret_cast<const float2*>(w.sm + RJ<NC>::OFF_WV);
      for (int j = lane; j < n; j += 32) a.sigma[(size_t)b * n + j] = wv[j].x;
    }
    if (a.V_io) {
      float* Vo = a.V_io + (size_t)b * n * n;
      for (int e = lane; e < n * n; e += 32) {
        const int rr = e / n, j = e - rr * n;
        Vo[e] = w.Vs()[((rr >> 1) * NC + j) * 2 + (rr & 1)];
      }
    }
    if (a.sweeps && lane == 0) a.sweeps[b] = r.sweeps;
    __syncwarp();
  }
}

}  // namespace rj
}  // namespace tilt

// tilt_jacobi.cuh — warm one-sided (Hestenes) Jacobi for the singular value thresholding S_eps
// (Eqs. A_1, S_operator), included by tilt_device.cuh.
//
// Column pair (i, j) of B = M V: gamma = b_i . b_j; if gamma^2 > tol^2 alpha beta, rotate so the two
// columns become orthogonal: with D = beta - alpha, G = 2 gamma,
//     t = sgn(D) G / (|D| + sqrt(D^2 + G^2))     (= sgn(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = D/G)
//     b_i <- c (b_i - t b_j), b_j <- c (b_j + t b_i), c = 1/sqrt(1 + t^2)
// Columns are stored scaled, b_j = d_j x_j (fast rotations): x_i <- x_i - t (d_j/d_i) x_j,
// x_j <- x_j + t (d_i/d_j) x_i, d <- c d, 1/d <- sqrt(1+t^2)/d, so a rotation is 2 FMAs per row.
// The same transformation is applied to V, so B = M V holds exactly for whatever (slightly
// non-orthogonal, from rounding in c) transform is applied; the final pass divides by ||v_j||
// (sigma_j = ||b_j|| / ||v_j||, A = sum_j h_j b_j v_j^T / ||v_j||^2), and the Newton-Schulz step
// re-orthonormalises the carried V, so c needs no refinement.
// Schedule: round-robin (circle method), n/2 disjoint pairs per round, one pair per LANES-lane unit,
// a CTA barrier per round; per-sweep fresh norms. Stop: a sweep without rotation, or a sweep whose
// rotations all had gamma^2 < (tol^2/n) alpha beta (quadratic convergence makes the next sweep
// rotation-free), or the sweep cap.
// ns[j] = (alpha_j = ||x_j||^2 d_j^2 tracked, d_j, 1/d_j, 0).
#pragma once
// (included inside namespace tilt by tilt_device.cuh)

// Per-lane rows of one column: lane lu of an L-lane unit holds RPL/4 float4 chunks, chunk q being
// rows [4(lu + qL), 4(lu + qL) + 4) (interleaved, so the 8 lanes of a shared-memory phase touch 128
// consecutive bytes: conflict-free); a chunk exists iff its first row is < ld (ld % 4 == 0).
// Addresses passed in point at the lane's first chunk (column base + 4 lu floats).
// Packed FP32x2 (sm_100: one FFMA2 issues two FMAs; the scalar operand broadcast as {s, s})
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void up2(unsigned long long x, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int RPL, int L>
struct Col {
  static_assert(RPL % 4 == 0, "float4 chunks");
  float v[RPL];
  static constexpr int NCH = RPL / 4;
  static __device__ __forceinline__ uint32_t chunk_mask(int lu, int ld) {
    uint32_t m = 0;
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      if (4 * (lu + q * L) < ld) m |= 1u << q;
    return m;
  }
  // generic-pointer versions (global or shared)
  __device__ __forceinline__ void gload(const float* p, uint32_t cm) {
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const float4 a = (cm >> q & 1u) ? *reinterpret_cast<const float4*>(p + 4 * q * L) : make_float4(0.f, 0.f, 0.f, 0.f);
      v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
    }
  }
  __device__ __forceinline__ void gstore(float* p, uint32_t cm) const {
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      if (cm >> q & 1u)
        *reinterpret_cast<float4*>(p + 4 * q * L) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  }
  // shared-window (32-bit address) versions with predicated vector ld/st.shared
  __device__ __forceinline__ void sload(uint32_t a, uint32_t cm) {
#pragma unroll
    for (int q = 0; q < RPL; ++q) v[q] = 0.f;
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n}"
          : "+f"(v[4 * q]), "+f"(v[4 * q + 1]), "+f"(v[4 * q + 2]), "+f"(v[4 * q + 3])
          : "r"(a + 16 * q * L), "r"((int)(cm >> q & 1u)));
  }
  __device__ __forceinline__ void sload_full(uint32_t a) {  // every chunk exists
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(v[4 * q]), "=f"(v[4 * q + 1]), "=f"(v[4 * q + 2]), "=f"(v[4 * q + 3])
                   : "r"(a + 16 * q * L));
  }
  __device__ __forceinline__ void sstore(uint32_t a, uint32_t cm) const {
#pragma unroll
    for (int q = 0; q < NCH; ++q)
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n}" ::"r"(a + 16 * q * L),
          "f"(v[4 * q]), "f"(v[4 * q + 1]), "f"(v[4 * q + 2]), "f"(v[4 * q + 3]), "r"((int)(cm >> q & 1u))
          : "memory");
  }
  __device__ __forceinline__ float dot(const Col& o) const {
    unsigned long long acc = 0ull;  // two chains, one FFMA2 per row pair
#pragma unroll
    for (int e = 0; e < RPL; e += 2) acc = fma2(pk2(v[e], v[e + 1]), pk2(o.v[e], o.v[e + 1]), acc);
    float a, b;
    up2(acc, a, b);
    return a + b;
  }
  // the fast rotation of a column pair (x, y) <- (x - ca y, y + cb x), one FFMA2 per row pair
  static __device__ __forceinline__ void rotate(Col& x, Col& y, float ca, float cb) {
    const unsigned long long mca = pk2(-ca, -ca), pcb = pk2(cb, cb);
#pragma unroll
    for (int e = 0; e < RPL; e += 2) {
      const unsigned long long x2 = pk2(x.v[e], x.v[e + 1]), y2 = pk2(y.v[e], y.v[e + 1]);
      up2(fma2(y2, mca, x2), x.v[e], x.v[e + 1]);
      up2(fma2(x2, pcb, y2), y.v[e], y.v[e + 1]);
    }
  }
  __device__ __forceinline__ float sq() const { return dot(*this); }
  __device__ __forceinline__ void scale(float s) {
#pragma unroll
    for (int e = 0; e < RPL; ++e) v[e] *= s;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v, bool on) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n @p st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n}" ::"r"(a),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"((int)on)
               : "memory");
}

template <int L>
__device__ __forceinline__ float unit_sum(float g) {
#pragma unroll
  for (int off = L / 2; off; off >>= 1) g += __shfl_xor_sync(FULL, g, off);
  return g;
}

// Rotation parameters of one pair (all lanes of a unit compute them redundantly).
struct Rot {
  float ca, cb, c, t;
};

__device__ __forceinline__ Rot rot_params(float4 ni, float4 nj, float gam, bool doit) {
  const float D = nj.x - ni.x, G = 2.f * gam;
  const float r2 = fmaf(D, D, G * G);
  const float den = fmaf(r2, rsqrt_approx(r2), fabsf(D));  // |D| + sqrt(D^2 + G^2), > 0 when doit
  float t = G * rcp_approx(den);
  t = (D < 0.f) ? -t : t;
  t = doit ? t : 0.f;
  Rot r;
  r.t = t;
  const float x2 = fmaf(t, t, 1.f);
  r.c = rsqrt_approx(x2);
  r.ca = t * nj.y * ni.z;  // t d_j / d_i
  r.cb = t * ni.y * nj.z;  // t d_i / d_j
  return r;
}

// ---------------------------------------------------------------------------------------------
// Re-normalisation passes
// MODE 0: ns_j = (||x_j||^2, 1, 1) (no scaling applied)
// MODE 1: apply the scales to B and V columns, ns_j = (fresh ||x_j||^2, 1, 1)
// MODE 2: as 1, then sigma_j = ||b_j|| / ||v_j||, h_j = max(sigma_j - eps, 0)/sigma_j;
//         ns_j = (sigma_j^2, 1/||v_j||^2, 1), hv_j = h_j (B is scaled for the product by svt()).
// ---------------------------------------------------------------------------------------------
template <class C, int MODE>
__device__ __forceinline__ void col_pass(Ctx<C>& cx, float eps) {
  constexpr int L = C::LANES, RPL = C::RPL, UPW = 32 / L;
  const int n = cx.n, ld = cx.lds;
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const int warp = threadIdx.x >> 5;
  const uint32_t cm = Col<RPL, L>::chunk_mask(lu, ld);
  for (int jb = warp * UPW; jb < n; jb += C::UNITS) {
    const int j = jb + (unit - warp * UPW);
    const bool valid = j < n;
    const int jj = valid ? j : 0;
    float* bp = cx.B + jj * ld + 4 * lu;
    float* vp = cx.V + jj * ld + 4 * lu;
    Col<RPL, L> x, y;
    x.gload(bp, cm);
    const float s = (MODE == 0) ? 1.f : cx.ns[jj].y;
    x.scale(s);
    float ss = unit_sum<L>(x.sq());
    float h = 1.f;
    if (MODE != 0) {
      y.gload(vp, cm);
      y.scale(s);
    }
    float ivv = 1.f;
    if (MODE == 2) {
      const float vv = unit_sum<L>(y.sq());
      ss = vv > 0.f ? ss / vv : 0.f;
      ivv = vv > 0.f ? 1.f / vv : 0.f;
      const float sg = sqrtf(ss);
      h = (sg > eps) ? (sg - eps) / sg : 0.f;
    }
    if (valid && MODE != 0) {
      x.gstore(bp, cm);
      y.gstore(vp, cm);
    }
    if (valid && lu == 0) {
      cx.ns[j] = make_float4(ss, ivv, 1.f, 0.f);
      if (MODE == 2) cx.hv[j] = h;
    }
  }
  __syncthreads();
}

template <class C, int MODE>
__device__ __forceinline__ void col_pass_smem(uint32_t sB, uint32_t sV, uint32_t sNS, int n, int ld) {
  constexpr int L = C::LANES, RPL = C::RPL, UPW = 32 / L;
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const int warp = threadIdx.x >> 5;
  const uint32_t cm = Col<RPL, L>::chunk_mask(lu, ld);
  const uint32_t lane_off = 4 * lu * 4, colb = ld * 4;
  for (int jb = warp * UPW; jb < n; jb += C::UNITS) {
    const int j = jb + (unit - warp * UPW);
    const bool valid = j < n;
    const int jj = valid ? j : 0;
    Col<RPL, L> x;
    x.sload(sB + jj * colb + lane_off, cm);
    const float s = MODE == 0 ? 1.f : lds4(sNS + 16 * jj).y;
    x.scale(s);
    const float ss = unit_sum<L>(x.sq());
    if (MODE == 1) {
      Col<RPL, L> y;
      y.sload(sV + jj * colb + lane_off, cm);
      y.scale(s);
      x.sstore(sB + jj * colb + lane_off, valid ? cm : 0u);
      y.sstore(sV + jj * colb + lane_off, valid ? cm : 0u);
    }
    sts4(sNS + 16 * jj, make_float4(ss, 1.f, 1.f, 0.f), valid && lu == 0);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------------------------
// Generic version (any memory space, any n): used by S256 (B, V in the global workspace)
// ---------------------------------------------------------------------------------------------
template <class C>
__device__ int jacobi_sweeps(Ctx<C>& cx, float tol, int max_sweeps, bool* capped) {
  constexpr int L = C::LANES, RPL = C::RPL, UPW = 32 / L;
  const int n = cx.n, ld = cx.lds;
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const int warp = threadIdx.x >> 5;
  const int sub = unit - warp * UPW;
  const uint32_t cm = Col<RPL, L>::chunk_mask(lu, ld);
  const int Nn = n + (n & 1);
  const int q = Nn - 1;
  const int npairs = Nn >> 1;
  const float tol2 = tol * tol;
  const float big2 = tol / (float)n;  // cos^2 threshold: a sweep below it leaves cos <~ n big2 = tol
  float* __restrict__ Bm = cx.B;
  float* __restrict__ Vm = cx.V;
  float4* __restrict__ ns = cx.ns;
  col_pass<C, 0>(cx, 0.f);
  int sweeps = 0;
  bool any = false;
  while (sweeps < max_sweeps) {
    bool rot = false, big = false;
    for (int r = 0; r < q; ++r) {
      for (int kb = warp * UPW; kb < npairs; kb += C::UNITS) {
        const int k = kb + sub;
        int i = r + k, j = r - k;
        if (i >= q) i -= q;
        if (j < 0) j += q;
        if (k == 0) {
          i = q;
          j = r;
        }
        const bool valid = (k < npairs) && (i < n) && (j < n);
        if (!valid) i = j = 0;
        float* bi = Bm + i * ld + 4 * lu;
        float* bj = Bm + j * ld + 4 * lu;
        Col<RPL, L> xi, xj;
        xi.gload(bi, cm);
        xj.gload(bj, cm);
        const float g = unit_sum<L>(xi.dot(xj));
        const float4 ni = ns[i], nj = ns[j];
        const float gam = g * ni.y * nj.y;
        const float ab = ni.x * nj.x;
        const bool doit = valid && ni.x > 0.f && nj.x > 0.f && gam * gam > tol2 * ab;
        if (__any_sync(FULL, doit)) {
          const Rot rp = rot_params(ni, nj, gam, doit);
          Col<RPL, L>::rotate(xi, xj, rp.ca, rp.cb);
          float* vi = Vm + i * ld + 4 * lu;
          float* vj = Vm + j * ld + 4 * lu;
          Col<RPL, L> yi, yj;
          yi.gload(vi, doit ? cm : 0u);
          yj.gload(vj, doit ? cm : 0u);
          Col<RPL, L>::rotate(yi, yj, rp.ca, rp.cb);
          if (doit) {
            xi.gstore(bi, cm);
            xj.gstore(bj, cm);
            yi.gstore(vi, cm);
            yj.gstore(vj, cm);
          }
          if (doit && lu == 0) {
            const float sx = rp.c * fmaf(rp.t, rp.t, 1.f);  // sqrt(1 + t^2)
            ns[i] = make_float4(fmaxf(fmaf(-rp.t, gam, ni.x), 0.f), rp.c * ni.y, sx * ni.z, 0.f);
            ns[j] = make_float4(fmaf(rp.t, gam, nj.x), rp.c * nj.y, sx * nj.z, 0.f);
          }
          rot |= doit;
          big |= doit && gam * gam > big2 * ab;
        }
      }
      __syncthreads();
    }
    ++sweeps;
    any = __syncthreads_or(rot);
    const bool more = __syncthreads_or(big);
    col_pass<C, 1>(cx, 0.f);  // re-normalise (apply scales, fresh norms)
    if (!more) {
      any = false;
      break;
    }
  }
  *capped = any;
  return sweeps;
}

// ---------------------------------------------------------------------------------------------
// Shared-memory specialisation (S32/S64/S128: B, V in shared memory, n/2 <= UNITS): 32-bit shared
// addresses with predicated vector ld/st.shared, the circle-method pair advanced incrementally
// (i, j <- i+1, j+1 mod q), __noinline__ so the caller's live state does not crowd its registers.
// ---------------------------------------------------------------------------------------------
template <class C>
__device__ __noinline__ int jacobi_sweeps_smem(float* Bp, float* Vp, float4* nsp, int n, float tol,
                                               int max_sweeps, int* capped, int* rot_acc) {
  int nrot = 0;  // rotations applied by this unit (counted on lane 0)
  constexpr int L = C::LANES, RPL = C::RPL;
  constexpr int ld = C::MAXD;  // SVD buffers are MAXD rows: every chunk exists, no masks
  constexpr uint32_t cm = (1u << Col<RPL, L>::NCH) - 1u;
  const uint32_t sB = smem_u32(Bp), sV = smem_u32(Vp), sNS = smem_u32(nsp);
  const int unit = threadIdx.x / L, lu = threadIdx.x % L;
  const uint32_t lane_off = 4 * lu * 4, colb = ld * 4;
  const int Nn = n + (n & 1);
  const int q = Nn - 1;
  const int npairs = Nn >> 1;
  const int k = unit;  // one pair per unit per round (n/2 <= UNITS)
  const bool unit_on = k < npairs;
  const float tol2 = tol * tol;
  const float big2 = tol / (float)n;  // cos^2 threshold: a sweep below it leaves cos <~ n big2 = tol
  col_pass_smem<C, 0>(sB, sV, sNS, n, ld);
  int sweeps = 0;
  int any = 0;
  while (sweeps < max_sweeps) {
    int rot = 0, big = 0;
    int i = k == 0 ? q : k, j = k == 0 ? 0 : q - k;  // round 0 of the circle method
    for (int r = 0; r < q; ++r) {
      const bool valid = unit_on && i < n && j < n;
      const int ii = valid ? i : 0, jj = valid ? j : 0;
      const uint32_t ai = sB + ii * colb + lane_off, aj = sB + jj * colb + lane_off;
      Col<RPL, L> xi, xj;
      if (unit_on) {  // units beyond n/2 pairs (a whole quarter-warp or warp) issue no loads
        xi.sload_full(ai);
        xj.sload_full(aj);
      } else {
#pragma unroll
        for (int e = 0; e < RPL; ++e) xi.v[e] = xj.v[e] = 0.f;
      }
      const float4 ni = lds4(sNS + 16 * ii), nj = lds4(sNS + 16 * jj);  // (alpha, d, 1/d, -)
      const float g = unit_sum<L>(xi.dot(xj));
      const float gam = g * ni.y * nj.y;
      const float ab = ni.x * nj.x;
      const bool doit = valid && ni.x > 0.f && nj.x > 0.f && gam * gam > tol2 * ab;
      if (__any_sync(FULL, doit)) {  // warp-uniform branch
        const Rot rp = rot_params(ni, nj, gam, doit);
        const uint32_t vi = sV + ii * colb + lane_off, vj = sV + jj * colb + lane_off;
        const uint32_t cmr = doit ? cm : 0u;
        Col<RPL, L>::rotate(xi, xj, rp.ca, rp.cb);
        xi.sstore(ai, cmr);
        xj.sstore(aj, cmr);
        // V columns after B's are stored: only two columns live in registers at a time
        Col<RPL, L> yi, yj;
        yi.sload(vi, cmr);  // only units that rotate read (and write) their V columns
        yj.sload(vj, cmr);
        Col<RPL, L>::rotate(yi, yj, rp.ca, rp.cb);
        yi.sstore(vi, cmr);
        yj.sstore(vj, cmr);
        const float sx = rp.c * fmaf(rp.t, rp.t, 1.f);  // sqrt(1 + t^2)
        sts4(sNS + 16 * ii, make_float4(fmaxf(fmaf(-rp.t, gam, ni.x), 0.f), rp.c * ni.y, sx * ni.z, 0.f),
             doit && lu == 0);
        sts4(sNS + 16 * jj, make_float4(fmaf(rp.t, gam, nj.x), rp.c * nj.y, sx * nj.z, 0.f), doit && lu == 0);
        rot |= doit ? 1 : 0;
        nrot += (doit && lu == 0) ? 1 : 0;
        big |= (doit && gam * gam > big2 * ab) ? 1 : 0;
      }
      __syncthreads();
      if (k != 0) i = (i + 1 == q) ? 0 : i + 1;
      j = (j + 1 == q) ? 0 : j + 1;
    }
    ++sweeps;
    any = __syncthreads_or(rot);
    const int more = __syncthreads_or(big);
    col_pass_smem<C, 1>(sB, sV, sNS, n, ld);  // re-normalise (apply scales, fresh norms)
    if (!more) {
      any = 0;
      break;
    }
  }
  if (rot_acc && nrot) atomicAdd(rot_acc, nrot);
  __syncthreads();
  *capped = any;
  return sweeps;
}

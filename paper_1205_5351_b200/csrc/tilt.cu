// tilt.cu — C ABI of libtilt (include/tilt.h): handle, validation, size-class dispatch, launches.
// Paper: Ren & Lin, arXiv 1205.5351. Design: DESIGN.md.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tilt_kernels.cuh"
#include "tilt_large_host.h"
#include "tilt_nvtx.h"

using namespace tilt;

namespace {

thread_local std::string g_last_error;

tilt_status cuda_fail(cudaError_t e, const char* what) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  g_last_error = buf;
  return TILT_E_CUDA;
}

#define TILT_CUDA(call)                                 \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

enum SizeClass { SC32 = 0, SC64 = 1, SC128 = 2, SC256 = 3, SC_NONE = 4, SC256G = 5, SC56 = 6, SC100 = 7 };

SizeClass size_class(int m, int n) {
  const int d = m > n ? m : n;
  if (d <= 32) return SC32;
  if (d <= 56) return SC56;
  if (d <= 64) return SC64;
  if (d <= 100) return SC100;
  if (d <= 128) return SC128;
  if (d <= 256) return n <= 216 ? SC256 : SC256G;  // B in shared memory while MAXD x n floats fit
  return SC_NONE;
}

}  // namespace

struct tilt_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  int max_batch = 0, max_m = 0, max_n = 0, max_p = 8;
  int64_t max_image_elems = 0;
  // workspace
  float* ws = nullptr;
  size_t ws_floats = 0;   // total
  int ws_slots = 0;
  int* counter = nullptr;  // work-queue counters
  float* coarse_images = nullptr;
  int* coarse_boxes = nullptr;
  tilt_report* coarse_rep = nullptr;
  float* coarse_aey = nullptr;  // pyramid warm start: coarse A, E, Y [3][B][m/2][n/2]
  // host-entry staging
  float* h_images = nullptr;
  int* h_patch = nullptr;
  int* h_boxes = nullptr;
  float* h_tau0 = nullptr;
  float* h_tau = nullptr;
  float* h_A = nullptr;
  float* h_E = nullptr;
  tilt_report* h_rep = nullptr;
  int64_t launches = 0;
  int svt_path = 0;  // tilt_svt_batch kernel family (tilt_set_svt_path): 0/1 CTA-per-patch, (2 retired),
                     // 3 multi-CTA
  tilt::lp::Ctx lp;  // multi-CTA path for large windows (workspace on first use)
  size_t lp_budget = 0;  // bytes of multi-CTA workspace (batches above it run in chunks)
};

namespace {

tilt::lp::Ctx& lp_ctx(tilt_handle* h) {
  h->lp.device = h->device;
  h->lp.num_sms = h->num_sms;
  h->lp.stream = h->stream;
  h->lp.launches = &h->launches;
  h->lp.err = &g_last_error;
  return h->lp;
}

// Opt in to `sm` bytes of dynamic shared memory when static + dynamic exceeds the 48 KB default (the
// static part counts: a 32 x 32 homography solve has 45.7 KB dynamic plus its static block).
inline tilt_status allow_dynamic_smem(const void* fn, size_t sm) {
  cudaFuncAttributes fa;
  TILT_CUDA(cudaFuncGetAttributes(&fa, fn));
  if (sm + fa.sharedSizeBytes > 48 * 1024)
    TILT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  return TILT_OK;
}

template <class C>
int occupancy_for(const void* fn, size_t smem) {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, C::NT, smem) != cudaSuccess) return 0;
  return nb;
}

DevParams to_dev(const tilt_params* prm) {
  DevParams P;
  P.lambda = prm->lambda;
  P.mu0_scale = prm->mu0_scale;
  P.mu_max_ratio = prm->mu_max_ratio;
  P.rho0 = prm->rho0;
  P.eps1 = prm->eps1;
  P.eps2 = prm->eps2;
  P.obj_tol = prm->obj_tol;
  P.tau_tol = prm->tau_tol;
  P.max_inner = prm->max_inner;
  P.max_outer = prm->max_outer;
  P.constraint_mode = prm->constraint_mode;
  P.vws = prm->vws;
  P.svd_warm = prm->svd_warm;
  P.jacobi_tol = prm->jacobi_tol;
  P.jacobi_max_sweeps = prm->jacobi_max_sweeps;
  P.fixed_inner = prm->fixed_inner_iters;
  P.fixed_outer = prm->fixed_outer_iters;
  P.ns_period = prm->ns_period > 1 ? prm->ns_period : 1;
  P.inner_solver = prm->inner_solver;
  P.adm_rho = prm->adm_rho;
  P.adm_tol = prm->adm_tol;
  P.svd_mode = prm->svd_mode;
  P.svd_ws_gate = prm->svd_ws_gate;
  P.rho_replay = prm->rho_replay;
  P.trace = prm->trace;
  return P;
}

bool params_ok(const tilt_params* p) {
  if (!p) return false;
  const float fs[] = {p->mu0_scale, p->mu_max_ratio, p->rho0, p->eps1, p->eps2, p->obj_tol, p->tau_tol};
  for (float f : fs)
    if (!std::isfinite(f)) return false;
  if (!std::isfinite(p->lambda) || !std::isfinite(p->jacobi_tol)) return false;
  if (p->mu0_scale <= 0.f || p->mu_max_ratio < 1.f || p->rho0 < 1.f || p->eps1 <= 0.f || p->eps2 <= 0.f) return false;
  if (p->max_inner <= 0 || p->max_outer <= 0 || p->jacobi_max_sweeps <= 0) return false;
  if (p->fixed_inner_iters < 0 || p->fixed_outer_iters < 0) return false;
  if (p->fixed_inner_iters > p->max_inner || p->fixed_outer_iters > p->max_outer) return false;
  if (p->pyramid_levels < 1 || p->pyramid_levels > 2) return false;
  if (p->constraint_mode != TILT_CONSTRAINTS_NONE && p->constraint_mode != TILT_CONSTRAINTS_CENTER_AREA) return false;
  if (p->kernel_path < 0 || p->kernel_path > 3 || p->kernel_path == 2) return false;  // 2: retired
  if (p->inner_solver == 1 && p->svd_mode == 1) return false;  // SVDWS is LADMAP's (Table 1's third column)
  if (p->inner_solver < 0 || p->inner_solver > 1) return false;
  if (p->ctas_per_sm < 0) return false;
  if (p->pyramid_warm < 0 || p->pyramid_warm > 1) return false;
  if (p->svd_mode < 0 || p->svd_mode > 1) return false;
  if (!std::isfinite(p->svd_ws_gate) || p->svd_ws_gate < 0.f) return false;
  if (!std::isfinite(p->adm_rho) || !std::isfinite(p->adm_tol) || p->adm_rho < 1.f || p->adm_tol <= 0.f) return false;
  return true;
}

// Per-call geometry: leading dimension (ld_of), columns, extra planes of the projector
struct Geo {
  int ld, n, gplanes;
};

template <class C>
inline Geo geo_of(int m, int n, int gplanes) { return Geo{ld_of<C>(m, n), n, gplanes}; }

template <class C>
struct Launch {
  static size_t smem(Geo g) { return Layout<C>::smem_bytes(g.ld, g.n, g.gplanes); }
  static size_t wsf(Geo g) { return Layout<C>::ws_floats(g.ld, g.n, g.gplanes); }

  static tilt_status prep(const void* fn, size_t sm) { return allow_dynamic_smem(fn, sm); }

  // grid size (persistent): num_sms * occupancy, capped by B and by the workspace slots
  static tilt_status grid(tilt_handle* h, const void* fn, Geo geo, int B, int* g, int cap_per_sm = 0) {
    const size_t sm = smem(geo);
    tilt_status s = prep(fn, sm);
    if (s != TILT_OK) return s;
    const int occ = occupancy_for<C>(fn, sm);
    if (occ <= 0) {
      g_last_error = "kernel does not fit on an SM (shared memory / registers)";
      return TILT_E_UNSUPPORTED;
    }
    int gsz = h->num_sms * (cap_per_sm > 0 && cap_per_sm < occ ? cap_per_sm : occ);
    if (gsz > B) gsz = B;
    const size_t w = wsf(geo);
    if (w > 0) {
      const size_t slots = h->ws_floats / w;
      if (slots == 0) {
        g_last_error = "workspace too small for this size (raise max_m/max_n/max_p at tilt_create)";
        return TILT_E_ARG;
      }
      if ((size_t)gsz > slots) gsz = (int)slots;
    }
    *g = gsz < 1 ? 1 : gsz;
    return TILT_OK;
  }

  template <class Args>
  static void set_ws(tilt_handle* h, Args& a, Geo geo) {
    a.ws = wsf(geo) ? h->ws : nullptr;
    a.ws_stride = wsf(geo);
  }

  static tilt_status solve(tilt_handle* h, SolveArgs a) {
    const Geo geo = geo_of<C>(a.m, a.n, a.p == 8 ? 3 : 2);
    const void* fn = (const void*)k_solve<C>;
    int g = 0;
    tilt_status s = grid(h, fn, geo, a.B, &g, a.ctas_per_sm);
    if (s != TILT_OK) return s;
    set_ws(h, a, geo);
    TILT_CUDA(cudaMemsetAsync(a.counter, 0, sizeof(int), h->stream));
    k_solve<C><<<g, C::NT, smem(geo), h->stream>>>(a);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    return TILT_OK;
  }

  static tilt_status inner(tilt_handle* h, InnerArgs a) {
    const Geo geo = geo_of<C>(a.m, a.n, a.p);
    const void* fn = (const void*)k_inner<C>;
    int g = 0;
    tilt_status s = grid(h, fn, geo, a.B, &g);
    if (s != TILT_OK) return s;
    set_ws(h, a, geo);
    k_inner<C><<<g, C::NT, smem(geo), h->stream>>>(a);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    return TILT_OK;
  }

  static tilt_status svt(tilt_handle* h, SvtArgs a) {
    const Geo geo = geo_of<C>(a.m, a.n, 0);
    const void* fn = (const void*)k_svt<C>;
    int g = 0;
    tilt_status s = grid(h, fn, geo, a.B, &g);
    if (s != TILT_OK) return s;
    set_ws(h, a, geo);
    k_svt<C><<<g, C::NT, smem(geo), h->stream>>>(a);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    return TILT_OK;
  }

  static tilt_status project(tilt_handle* h, ProjArgs a) {
    const Geo geo = geo_of<C>(a.m, a.n, a.p);
    const void* fn = (const void*)k_project<C>;
    int g = 0;
    tilt_status s = grid(h, fn, geo, a.B, &g);
    if (s != TILT_OK) return s;
    set_ws(h, a, geo);
    k_project<C><<<g, C::NT, smem(geo), h->stream>>>(a);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    return TILT_OK;
  }
};

template <template <class> class F, class... Args>
tilt_status dispatch(SizeClass c, Args... args) {
  switch (c) {
    case SC32: return F<CfgS32>::run(args...);
    case SC56: return F<CfgS56>::run(args...);
    case SC64: return F<CfgS64>::run(args...);
    case SC100: return F<CfgS100>::run(args...);
    case SC128: return F<CfgS128>::run(args...);
    case SC256: return F<CfgS256>::run(args...);
    case SC256G: return F<CfgS256G>::run(args...);
    default: g_last_error = "m, n must be <= 256"; return TILT_E_ARG;
  }
}

template <class C>
struct SolveF {
  static tilt_status run(tilt_handle* h, SolveArgs a) { return Launch<C>::solve(h, a); }
};
template <class C>
struct InnerF {
  static tilt_status run(tilt_handle* h, InnerArgs a) { return Launch<C>::inner(h, a); }
};
template <class C>
struct SvtF {
  static tilt_status run(tilt_handle* h, SvtArgs a) { return Launch<C>::svt(h, a); }
};
template <class C>
struct ProjF {
  static tilt_status run(tilt_handle* h, ProjArgs a) { return Launch<C>::project(h, a); }
};

// workspace floats per slot for the largest geometry of any entry (explicit K: p planes)
size_t ws_need(SizeClass c, int m, int n, int gpl) {
  switch (c) {
    case SC32: return Launch<CfgS32>::wsf(geo_of<CfgS32>(m, n, gpl));
    case SC56: return Launch<CfgS56>::wsf(geo_of<CfgS56>(m, n, gpl));
    case SC64: return Launch<CfgS64>::wsf(geo_of<CfgS64>(m, n, gpl));
    case SC100: return Launch<CfgS100>::wsf(geo_of<CfgS100>(m, n, gpl));
    case SC128: return Launch<CfgS128>::wsf(geo_of<CfgS128>(m, n, gpl));
    case SC256: return Launch<CfgS256>::wsf(geo_of<CfgS256>(m, n, gpl));
    case SC256G: return Launch<CfgS256G>::wsf(geo_of<CfgS256G>(m, n, gpl));
    default: return 0;
  }
}

template <class C>
int occ_of(Geo g) {
  const size_t sm = Launch<C>::smem(g);
  int best = 0;
  const void* fns[] = {(const void*)k_solve<C>, (const void*)k_inner<C>, (const void*)k_svt<C>,
                       (const void*)k_project<C>};
  for (const void* fn : fns) {
    Launch<C>::prep(fn, sm);
    const int o = occupancy_for<C>(fn, sm);
    best = o > best ? o : best;
  }
  return best;
}

int occ_need(SizeClass c, int m, int n, int gpl) {
  switch (c) {
    case SC32: return occ_of<CfgS32>(geo_of<CfgS32>(m, n, gpl));
    case SC56: return occ_of<CfgS56>(geo_of<CfgS56>(m, n, gpl));
    case SC64: return occ_of<CfgS64>(geo_of<CfgS64>(m, n, gpl));
    case SC100: return occ_of<CfgS100>(geo_of<CfgS100>(m, n, gpl));
    case SC128: return occ_of<CfgS128>(geo_of<CfgS128>(m, n, gpl));
    case SC256: return occ_of<CfgS256>(geo_of<CfgS256>(m, n, gpl));
    case SC256G: return occ_of<CfgS256G>(geo_of<CfgS256G>(m, n, gpl));
    default: return 1;
  }
}

}  // namespace

extern "C" {

int32_t tilt_abi_version(void) { return TILT_ABI_VERSION; }

const char* tilt_status_string(tilt_status s) {
  switch (s) {
    case TILT_OK: return "TILT_OK";
    case TILT_E_ARG: return "TILT_E_ARG: invalid argument";
    case TILT_E_CUDA: return "TILT_E_CUDA: CUDA runtime error";
    case TILT_E_OOM: return "TILT_E_OOM: device allocation failed";
    case TILT_E_UNSUPPORTED: return "TILT_E_UNSUPPORTED";
    default: return "unknown tilt_status";
  }
}

const char* tilt_patch_status_string(int32_t s) {
  switch (s) {
    case TILT_PATCH_CONVERGED: return "CONVERGED";
    case TILT_PATCH_MAX_OUTER: return "MAX_OUTER";
    case TILT_PATCH_WINDOW_ESCAPE: return "WINDOW_ESCAPE";
    case TILT_PATCH_SINGULAR_GRAM: return "SINGULAR_GRAM";
    case TILT_PATCH_ZERO_PATCH: return "ZERO_PATCH";
    case TILT_PATCH_DIVERGED: return "DIVERGED";
    default: return "UNKNOWN";
  }
}

const char* tilt_last_error(void) { return g_last_error.c_str(); }

tilt_status tilt_default_params(tilt_params* prm) {
  if (!prm) return TILT_E_ARG;
  memset(prm, 0, sizeof(*prm));
  prm->lambda = -1.f;
  prm->mu0_scale = 1.25f;
  prm->mu_max_ratio = 1e6f;
  prm->rho0 = 2.0f;
  prm->eps1 = 1e-6f;
  prm->eps2 = 0.1f;
  prm->obj_tol = 1e-5f;
  prm->tau_tol = 1e-4f;
  prm->max_inner = 1000;
  prm->max_outer = 50;
  prm->constraint_mode = TILT_CONSTRAINTS_CENTER_AREA;
  prm->vws = 1;
  prm->svd_warm = 1;
  prm->pyramid_levels = 1;
  prm->jacobi_tol = 0.f;
  prm->jacobi_max_sweeps = 20;
  prm->ns_period = 4;
  prm->inner_solver = 0;
  prm->adm_rho = 1.25f;
  prm->adm_tol = 1e-6f;
  prm->svd_mode = 0;
  prm->svd_ws_gate = 2e-5f;
  return TILT_OK;
}

tilt_status tilt_destroy(tilt_handle* h) {
  if (!h) return TILT_OK;
  cudaSetDevice(h->device);
  void* ptrs[] = {h->ws, h->counter, h->coarse_images, h->coarse_boxes, h->coarse_rep, h->coarse_aey, h->h_images, h->h_patch,
                  h->h_boxes, h->h_tau0, h->h_tau, h->h_A, h->h_E, h->h_rep};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  tilt::lp::release(h->lp);
  delete h;
  return TILT_OK;
}

// the multi-CTA path's batch chunk: its workspace is B x (a few planes + n x n buffers) per problem,
// so a handle sized for many small patches runs large windows in chunks within lp_budget bytes
static int lp_chunk(tilt_handle* h, int B, int m, int n, int p, bool svdws) {
  const size_t per = tilt::lp::ws_need(1, m, n, p, svdws) * sizeof(float);
  size_t c = per > 0 ? h->lp_budget / per : (size_t)B;
  if (c < 1) c = 1;
  if (c > 65535) c = 65535;  // problems index gridDim.y / gridDim.z of the multi-CTA kernels
  return c < (size_t)B ? (int)c : B;
}

tilt_status tilt_create(tilt_handle** out, const tilt_create_opts* o) {
  if (!out || !o) return TILT_E_ARG;
  *out = nullptr;
  if (o->max_batch < 0 || o->max_m < 1 || o->max_n < 1 || o->max_m > tilt::lp::MAX_DIM || o->max_n > tilt::lp::MAX_DIM)
    return TILT_E_ARG;
  if (o->max_p != 6 && o->max_p != 8) return TILT_E_ARG;
  tilt_handle* h = new tilt_handle();
  h->device = o->device;
  h->stream = (cudaStream_t)o->stream;
  h->max_batch = o->max_batch;
  h->max_m = o->max_m;
  h->max_n = o->max_n;
  h->max_p = o->max_p;
  h->max_image_elems = o->max_image_elems;
  cudaError_t e = cudaSetDevice(h->device);
  if (e != cudaSuccess) {
    tilt_status s = cuda_fail(e, "cudaSetDevice");
    delete h;
    return s;
  }
  e = cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  if (e != cudaSuccess) {
    tilt_status s = cuda_fail(e, "cudaDeviceGetAttribute");
    delete h;
    return s;
  }

  auto fail = [&](cudaError_t err, const char* what) {
    cuda_fail(err, what);
    tilt_destroy(h);
    return err == cudaErrorMemoryAllocation ? TILT_E_OOM : TILT_E_CUDA;
  };
  // CTA-per-patch workspace for windows up to 256 x 256 (larger windows: the multi-CTA path)
  const int cm = h->max_m < 256 ? h->max_m : 256, cn = h->max_n < 256 ? h->max_n : 256;
  const SizeClass c = size_class(cm, cn);
  const int mn = h->max_m * h->max_n;
  const int gpl = h->max_p > 3 ? h->max_p : 3;
  const size_t wsf = ws_need(c, cm, cn, gpl);
  if (wsf > 0) {
    const int occ = occ_need(c, cm, cn, gpl);
    h->ws_slots = h->num_sms * (occ > 0 ? occ : 1);
    h->ws_floats = wsf * h->ws_slots;
  }
  if (h->ws_floats > 0) {
    if ((e = cudaMalloc(&h->ws, h->ws_floats * sizeof(float))) != cudaSuccess) return fail(e, "cudaMalloc(ws)");
  }
  if ((e = cudaMalloc(&h->counter, 64 * sizeof(int))) != cudaSuccess) return fail(e, "cudaMalloc(counter)");
  // windows above 128 x 128 take the multi-CTA path by default: its workspace is
  // made here, so the solve entries allocate nothing (SVDWS or a forced kernel_path = 3 at smaller
  // sizes still allocate on first use, as tilt.h states)
  {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) fr = (size_t)8 << 30;
    h->lp_budget = fr / 2 < ((size_t)24 << 30) ? fr / 2 : ((size_t)24 << 30);
  }
  if ((h->max_m > 128 || h->max_n > 128) && h->max_batch > 0) {
    const int ch = lp_chunk(h, h->max_batch, h->max_m, h->max_n, h->max_p, false);
    const tilt_status ls = tilt::lp::ensure(lp_ctx(h), tilt::lp::ws_need(ch, h->max_m, h->max_n, h->max_p), ch);
    if (ls != TILT_OK) {
      tilt_destroy(h);
      return ls;
    }
  }
  if (h->max_image_elems > 0) {
    const size_t nb = (size_t)h->max_batch;
    if ((e = cudaMalloc(&h->coarse_images, (size_t)h->max_image_elems / 4 * sizeof(float) + 64)) != cudaSuccess)
      return fail(e, "cudaMalloc(coarse)");
    if ((e = cudaMalloc(&h->coarse_boxes, 4 * nb * sizeof(int) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->coarse_rep, nb * sizeof(tilt_report) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->coarse_aey, 3 * nb * (size_t)(h->max_m / 2) * (h->max_n / 2) * sizeof(float) + 64)) !=
        cudaSuccess)
      return fail(e, "cudaMalloc(coarse A/E/Y)");
    if ((e = cudaMalloc(&h->h_images, (size_t)h->max_image_elems * sizeof(float))) != cudaSuccess)
      return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_patch, nb * sizeof(int) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_boxes, 4 * nb * sizeof(int) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_tau0, 8 * nb * sizeof(float) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_tau, 8 * nb * sizeof(float) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_A, nb * mn * sizeof(float) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_E, nb * mn * sizeof(float) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&h->h_rep, nb * sizeof(tilt_report) + 64)) != cudaSuccess) return fail(e, "cudaMalloc");
  }
  *out = h;
  return TILT_OK;
}

tilt_status tilt_set_stream(tilt_handle* h, void* stream) {
  if (!h) return TILT_E_ARG;
  h->stream = (cudaStream_t)stream;
  return TILT_OK;
}

int64_t tilt_launch_count(const tilt_handle* h) { return h ? h->launches : 0; }

tilt_status tilt_set_svt_path(tilt_handle* h, int32_t path) {
  if (!h || path < 0 || path > 3 || path == 2) return TILT_E_ARG;  // 2: the retired warp-per-patch family
  h->svt_path = path;
  return TILT_OK;
}

static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

static tilt_status solve_level(tilt_handle* h, const float* images, int32_t n_images, int32_t H, int32_t W,
                               const int32_t* patch_image, const int32_t* boxes, const float* tau0, int32_t B,
                               int m, int n, int32_t kind, const tilt_params* prm, float* tau_out, float* A_out,
                               float* E_out, float* Y_out, tilt_report* rep, const tilt_report* rep_prev,
                               const float* warm_aey = nullptr, const tilt_report* warm_rep = nullptr) {
  SolveArgs a;
  memset(&a, 0, sizeof(a));
  a.images = images;
  a.n_images = n_images;
  a.H = H;
  a.W = W;
  a.patch_image = patch_image;
  a.boxes = boxes;
  a.tau0 = tau0;
  a.B = B;
  a.m = m;
  a.n = n;
  a.p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  a.kind = kind;
  a.P = to_dev(prm);
  a.tau_out = tau_out;
  a.A_out = A_out;
  a.E_out = E_out;
  a.Y_out = Y_out;
  a.rep = rep;
  a.rep_prev = rep_prev;
  a.counter = h->counter;
  a.ctas_per_sm = prm->ctas_per_sm;
  if (warm_aey) {
    const size_t cn = (size_t)B * (m / 2) * (n / 2);
    a.warm_A = warm_aey;
    a.warm_E = warm_aey + cn;
    a.warm_Y = warm_aey + 2 * cn;
    a.warm_rep = warm_rep;
  }
  // the multi-CTA path: asked for, beyond the CTA kernels, SVDWS, or auto above 128 (config 4,
  // 256 x 200x200: 14.6 s vs 34.4 s on the CTA-per-patch kernel)
  if (prm->kernel_path == 3 || m > 256 || n > 256 || prm->svd_mode != 0 ||
      (prm->kernel_path == 0 && prm->inner_solver == 0 && (m > 128 || n > 128))) {
    if (prm->inner_solver != 0 || (prm->svd_mode == 1 && m < n)) {
      g_last_error = "multi-CTA tilt_solve_batch: LADMAP only (svd_mode 1 needs m >= n)";
      return TILT_E_ARG;
    }
    if (capturing(h->stream)) {
      g_last_error = "the multi-CTA path synchronises its stream: not allowed while capturing";
      return TILT_E_UNSUPPORTED;
    }
    const int p = a.p;
    const int ch = lp_chunk(h, B, m, n, p, prm->svd_mode == 1);
    const size_t mn = (size_t)m * n, cn = (size_t)B * (m / 2) * (n / 2), cmn = (size_t)(m / 2) * (n / 2);
    for (int b0 = 0; b0 < B; b0 += ch) {  // bounded workspace: the batch in chunks
      const int nb = B - b0 < ch ? B - b0 : ch;
      tilt::DevParams P = a.P;
      const size_t rows = (size_t)b0 * P.max_outer * P.max_inner;
      if (P.rho_replay) P.rho_replay += rows;
      if (P.trace) P.trace += rows * 4;
      const tilt_status st = tilt::lp::solve(
          lp_ctx(h), images, n_images, H, W, patch_image + b0, boxes + 4 * (size_t)b0, tau0 ? tau0 + (size_t)b0 * p : nullptr,
          nb, m, n, kind, P, tau_out + (size_t)b0 * p, A_out ? A_out + b0 * mn : nullptr, E_out ? E_out + b0 * mn : nullptr,
          Y_out ? Y_out + b0 * mn : nullptr, rep ? rep + b0 : nullptr, rep_prev ? rep_prev + b0 : nullptr,
          warm_aey ? warm_aey + b0 * cmn : nullptr, warm_aey ? warm_aey + cn + b0 * cmn : nullptr,
          warm_aey ? warm_aey + 2 * cn + b0 * cmn : nullptr, warm_rep ? warm_rep + b0 : nullptr);
      if (st != TILT_OK) return st;
    }
    return TILT_OK;
  }
  return dispatch<SolveF>(size_class(m, n), h, a);
}

// All boxes of one call must share (w, h): read from the caller's box array? The boxes live on
// the device, so the window size is passed through the first box copied to the host.
static tilt_status first_box(tilt_handle* h, const int32_t* boxes, int* m, int* n) {
  if (capturing(h->stream)) {
    g_last_error = "win_h/win_w = 0 reads boxes[0] with a host sync: not allowed on a capturing stream";
    return TILT_E_UNSUPPORTED;
  }
  int bx[4];
  TILT_CUDA(cudaMemcpyAsync(bx, boxes, sizeof(bx), cudaMemcpyDeviceToHost, h->stream));
  TILT_CUDA(cudaStreamSynchronize(h->stream));
  *n = bx[2];
  *m = bx[3];
  return TILT_OK;
}

tilt_status tilt_solve_batch(tilt_handle* h, const float* images, int32_t n_images, int32_t H, int32_t W,
                             const int32_t* patch_image, const int32_t* boxes, const float* tau0, int32_t B,
                             int32_t kind, const tilt_params* prm, float* tau_out, float* A_out, float* E_out,
                             float* Y_out, tilt_report* rep) {
  if (!h || !params_ok(prm)) return TILT_E_ARG;
  if (B < 0 || B > h->max_batch) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!images || !patch_image || !boxes || !tau_out || n_images < 1 || H < 2 || W < 2) return TILT_E_ARG;
  tilt::NvtxRange nv("tilt_solve_batch (K1-K4: persistent Algorithm 1)");
  if (kind != TILT_AFFINE && kind != TILT_HOMOGRAPHY) return TILT_E_ARG;
  const int p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  if (p > h->max_p) return TILT_E_ARG;
  if ((prm->rho_replay || prm->trace) && prm->max_outer <= 0) return TILT_E_ARG;
  TILT_CUDA(cudaSetDevice(h->device));
  int m = prm->win_h, n = prm->win_w;
  tilt_status s = TILT_OK;
  if (m <= 0 || n <= 0) {
    s = first_box(h, boxes, &m, &n);
    if (s != TILT_OK) return s;
  }
  if (m < 2 || n < 2 || m > h->max_m || n > h->max_n) {
    g_last_error = "box size outside [2, max_m] x [2, max_n]";
    return TILT_E_ARG;
  }
  if (prm->pyramid_levels == 2) {
    if ((m & 1) || (n & 1) || (H & 1) || (W & 1) || m < 8 || n < 8) {
      g_last_error = "pyramid needs even box and image sizes";
      return TILT_E_ARG;
    }
    if (!h->coarse_images || (int64_t)n_images * H * W > h->max_image_elems) {
      g_last_error = "pyramid workspace too small (max_image_elems at tilt_create)";
      return TILT_E_ARG;
    }
    const size_t total = (size_t)n_images * (H / 2) * (W / 2);
    int blocks = (int)((total + 255) / 256);
    if (blocks > 4 * h->num_sms * 8) blocks = 4 * h->num_sms * 8;
    k_downsample<<<blocks, 256, 0, h->stream>>>(images, h->coarse_images, n_images, H, W);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    k_half_boxes<<<(4 * B + 255) / 256, 256, 0, h->stream>>>(boxes, h->coarse_boxes, B);
    h->launches++;
    TILT_CUDA(cudaGetLastError());
    tilt_params pc = *prm;
    pc.rho_replay = nullptr;
    pc.trace = nullptr;
    const bool pw = prm->pyramid_warm != 0 && prm->vws != 0;
    const size_t cn = (size_t)B * (m / 2) * (n / 2);
    float* cA = pw ? h->coarse_aey : nullptr;
    s = solve_level(h, h->coarse_images, n_images, H / 2, W / 2, patch_image, h->coarse_boxes, tau0, B, m / 2,
                    n / 2, kind, &pc, tau_out, cA, pw ? cA + cn : nullptr, pw ? cA + 2 * cn : nullptr, h->coarse_rep,
                    nullptr);
    if (s != TILT_OK) return s;
    return solve_level(h, images, n_images, H, W, patch_image, boxes, tau_out, B, m, n, kind, prm, tau_out, A_out,
                       E_out, Y_out, rep, rep ? h->coarse_rep : nullptr, cA, h->coarse_rep);
  }
  return solve_level(h, images, n_images, H, W, patch_image, boxes, tau0, B, m, n, kind, prm, tau_out, A_out, E_out,
                     Y_out, rep, nullptr);
}

tilt_status tilt_solve_batch_host(tilt_handle* h, const float* images, int32_t n_images, int32_t H, int32_t W,
                                  const int32_t* patch_image, const int32_t* boxes, const float* tau0, int32_t B,
                                  int32_t kind, const tilt_params* prm, float* tau_out, float* A_out, float* E_out,
                                  tilt_report* rep) {
  if (!h || !params_ok(prm)) return TILT_E_ARG;
  if (B < 0 || B > h->max_batch) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!images || !patch_image || !boxes || !tau_out) return TILT_E_ARG;
  if (!h->h_images || (int64_t)n_images * H * W > h->max_image_elems) {
    g_last_error = "host entry needs max_image_elems >= n_images*H*W at tilt_create";
    return TILT_E_ARG;
  }
  tilt::NvtxRange nv("tilt_solve_batch_host (H2D, solve, D2H)");
  const int p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  const int m = boxes[3], n = boxes[2];
  if (m < 2 || n < 2 || m > h->max_m || n > h->max_n) return TILT_E_ARG;
  TILT_CUDA(cudaSetDevice(h->device));
  const size_t mn = (size_t)m * n;
  TILT_CUDA(cudaMemcpyAsync(h->h_images, images, (size_t)n_images * H * W * sizeof(float), cudaMemcpyHostToDevice,
                            h->stream));
  TILT_CUDA(cudaMemcpyAsync(h->h_patch, patch_image, B * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  TILT_CUDA(cudaMemcpyAsync(h->h_boxes, boxes, 4 * B * sizeof(int), cudaMemcpyHostToDevice, h->stream));
  if (tau0)
    TILT_CUDA(cudaMemcpyAsync(h->h_tau0, tau0, p * B * sizeof(float), cudaMemcpyHostToDevice, h->stream));
  tilt_params pw = *prm;
  pw.win_h = m;
  pw.win_w = n;
  tilt_status s = tilt_solve_batch(h, h->h_images, n_images, H, W, h->h_patch, h->h_boxes, tau0 ? h->h_tau0 : nullptr,
                                   B, kind, &pw, h->h_tau, A_out ? h->h_A : nullptr, E_out ? h->h_E : nullptr,
                                   nullptr, rep ? h->h_rep : nullptr);
  if (s != TILT_OK) return s;
  TILT_CUDA(cudaMemcpyAsync(tau_out, h->h_tau, p * B * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  if (A_out) TILT_CUDA(cudaMemcpyAsync(A_out, h->h_A, B * mn * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  if (E_out) TILT_CUDA(cudaMemcpyAsync(E_out, h->h_E, B * mn * sizeof(float), cudaMemcpyDeviceToHost, h->stream));
  if (rep) TILT_CUDA(cudaMemcpyAsync(rep, h->h_rep, B * sizeof(tilt_report), cudaMemcpyDeviceToHost, h->stream));
  TILT_CUDA(cudaStreamSynchronize(h->stream));
  return TILT_OK;
}

tilt_status tilt_warp_batch(tilt_handle* h, const float* images, int32_t n_images, int32_t H, int32_t W,
                            const int32_t* patch_image, const int32_t* boxes, const float* tau, int32_t B, int32_t kind,
                            int32_t win_h, int32_t win_w, float* Dhat, float* J, float* norm, int32_t* status) {
  if (!h || B < 0) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!images || !patch_image || !boxes || !tau || !Dhat) return TILT_E_ARG;
  if (kind != TILT_AFFINE && kind != TILT_HOMOGRAPHY) return TILT_E_ARG;
  tilt::NvtxRange nv("K1 tilt_warp_batch");
  TILT_CUDA(cudaSetDevice(h->device));
  int m = win_h, n = win_w;
  if (m <= 0 || n <= 0) {
    tilt_status s = first_box(h, boxes, &m, &n);
    if (s != TILT_OK) return s;
  }
  if (m < 2 || n < 2 || m > tilt::lp::MAX_DIM || n > tilt::lp::MAX_DIM) return TILT_E_ARG;
  WarpArgs a;
  a.images = images;
  a.n_images = n_images;
  a.H = H;
  a.W = W;
  a.patch_image = patch_image;
  a.boxes = boxes;
  a.tau = tau;
  a.B = B;
  a.m = m;
  a.n = n;
  a.p = kind == TILT_HOMOGRAPHY ? 8 : 6;
  a.kind = kind;
  a.Dhat = Dhat;
  a.J = J;
  a.norm = norm;
  a.status = status;
  const size_t k1_smem = (size_t)m * n * sizeof(float4);  // (d, gx, gy, gz) per window pixel
  if (k1_smem > 227 * 1024) return TILT_E_ARG;
  {
    const tilt_status s1 = allow_dynamic_smem((const void*)k_warp, k1_smem);
    if (s1 != TILT_OK) return s1;
  }
  k_warp<<<B, K1_NT, k1_smem, h->stream>>>(a);
  h->launches++;
  TILT_CUDA(cudaGetLastError());
  return TILT_OK;
}

tilt_status tilt_svt_batch(tilt_handle* h, const float* M, int32_t B, int32_t m, int32_t n, const float* eps,
                           float* V_io, float* A, float* sigma, int32_t* sweeps) {
  if (!h || B < 0 || m < 1 || n < 1 || m > h->max_m || n > h->max_n) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!M || !eps || !A) return TILT_E_ARG;
  tilt::NvtxRange nv("K3 tilt_svt_batch");
  TILT_CUDA(cudaSetDevice(h->device));
  SvtArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M;
  a.B = B;
  a.m = m;
  a.n = n;
  a.eps = eps;
  a.V_io = V_io;
  a.A = A;
  a.sigma = sigma;
  a.sweeps = sweeps;
  a.tol = default_jacobi_tol(m);
  a.max_sweeps = 20;
  if (h->svt_path == 3 || m > 256 || n > 256) {
    if (capturing(h->stream)) {
      g_last_error = "the multi-CTA path synchronises its stream: not allowed while capturing";
      return TILT_E_UNSUPPORTED;
    }
    const int ch = lp_chunk(h, B, m, n, 1, false);
    for (int b0 = 0; b0 < B; b0 += ch) {  // bounded workspace: the batch in chunks
      const int nb = B - b0 < ch ? B - b0 : ch;
      const size_t mn = (size_t)m * n, nn = (size_t)n * n;
      const tilt_status st = tilt::lp::svt(lp_ctx(h), M + b0 * mn, nb, m, n, eps + b0, V_io ? V_io + b0 * nn : nullptr,
                                           A + b0 * mn, sigma ? sigma + (size_t)b0 * n : nullptr,
                                           sweeps ? sweeps + b0 : nullptr, a.tol, a.max_sweeps);
      if (st != TILT_OK) return st;
    }
    return TILT_OK;
  }
  return dispatch<SvtF>(size_class(m, n), h, a);
}

tilt_status tilt_project_batch(tilt_handle* h, const float* J, const float* Q, int32_t l, const float* v, int32_t B,
                               int32_t m, int32_t n, int32_t p, float* Pv, float* dtau, int32_t* status) {
  if (!h || B < 0 || m < 1 || n < 1 || m > h->max_m || n > h->max_n) return TILT_E_ARG;
  if (p < 1 || p > 8 || p > h->max_p || (Q && (l < 1 || l > 3))) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!J || !v || !Pv) return TILT_E_ARG;
  tilt::NvtxRange nv("K2 tilt_project_batch");
  TILT_CUDA(cudaSetDevice(h->device));
  ProjArgs a;
  memset(&a, 0, sizeof(a));
  a.J = J;
  a.Q = Q;
  a.l = Q ? l : 0;
  a.v = v;
  a.B = B;
  a.m = m;
  a.n = n;
  a.p = p;
  a.Pv = Pv;
  a.dtau = dtau;
  a.status = status;
  return dispatch<ProjF>(size_class(m, n), h, a);
}

tilt_status tilt_inner_batch(tilt_handle* h, const float* D, const float* J, const float* Q, int32_t l, int32_t B,
                             int32_t m, int32_t n, int32_t p, const tilt_params* prm, float* A, float* E, float* Y,
                             tilt_report* rep) {
  if (!h || !params_ok(prm) || B < 0 || m < 2 || n < 2 || m > h->max_m || n > h->max_n) return TILT_E_ARG;
  if (p < 1 || p > 8 || p > h->max_p || (Q && (l < 1 || l > 3))) return TILT_E_ARG;
  if (B == 0) return TILT_OK;
  if (!D || !J || !A || !E) return TILT_E_ARG;
  tilt::NvtxRange nv("K3 tilt_inner_batch");
  TILT_CUDA(cudaSetDevice(h->device));
  InnerArgs a;
  memset(&a, 0, sizeof(a));
  a.D = D;
  a.J = J;
  a.Q = Q;
  a.l = Q ? l : 0;
  a.B = B;
  a.m = m;
  a.n = n;
  a.p = p;
  a.P = to_dev(prm);
  a.A = A;
  a.E = E;
  a.Y = Y;
  a.rep = rep;
  if (prm->kernel_path == 3 || m > 256 || n > 256 || prm->svd_mode == 1 ||
      (prm->kernel_path == 0 && prm->inner_solver == 0 && (m > 128 || n > 128))) {
    if (prm->svd_mode == 1 && m < n) return TILT_E_ARG;
    if (capturing(h->stream)) {
      g_last_error = "the multi-CTA path synchronises its stream: not allowed while capturing";
      return TILT_E_UNSUPPORTED;
    }
    const int ch = lp_chunk(h, B, m, n, p, prm->svd_mode == 1);
    const size_t mn = (size_t)m * n;
    for (int b0 = 0; b0 < B; b0 += ch) {  // bounded workspace: the batch in chunks
      const int nb = B - b0 < ch ? B - b0 : ch;
      tilt::DevParams P = a.P;
      if (P.rho_replay) P.rho_replay += (size_t)b0 * P.max_inner;
      if (P.trace) P.trace += (size_t)b0 * P.max_inner * 4;
      const tilt_status st = tilt::lp::inner(lp_ctx(h), D + b0 * mn, J + b0 * p * mn, Q ? Q + (size_t)b0 * l * p : nullptr,
                                             Q ? l : 0, nb, m, n, p, P, A + b0 * mn, E + b0 * mn,
                                             Y ? Y + b0 * mn : nullptr, rep ? rep + b0 : nullptr);
      if (st != TILT_OK) return st;
    }
    return TILT_OK;
  }
  return dispatch<InnerF>(size_class(m, n), h, a);
}

}  // extern "C"

// tilt_rj.cu — translation unit of the warp-per-patch kernels (tilt_rj.cuh) and their launchers.
// Paper: Ren & Lin, arXiv 1205.5351. Design: DESIGN.md.
#define TILT_NO_FREE_KERNELS
#include "tilt_rj.cuh"
#include "tilt_rj_host.h"

namespace tilt {
namespace rjh {
namespace {

int nc_of(int n) { return n <= 36 ? 36 : 50; }

template <int NC>
size_t smem_bytes() {
  return (size_t)rj::RJ<NC>::SMF * rj::RJ<NC>::WPB * sizeof(float);
}

template <int NC>
int blocks_per_sm(const void* fn) {
  const size_t sm = smem_bytes<NC>();
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) return 0;
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, rj::RJ<NC>::NT, sm) != cudaSuccess) return 0;
  return nb;
}

template <int NC>
size_t ws_need_nc(int num_sms, int m) {
  const int nb = blocks_per_sm<NC>((const void*)rj::k_solve_rj<NC>);
  return (size_t)num_sms * (nb > 0 ? nb : 1) * rj::RJ<NC>::WPB * rj::ws_floats_rj<NC>(m);
}

tilt_status cuda_err(cudaError_t e, const char* what, std::string* err) {
  *err = std::string(what) + ": " + cudaGetErrorString(e);
  return TILT_E_CUDA;
}

template <int NC>
tilt_status solve_nc(int num_sms, float* ws, size_t ws_floats, int* counter, cudaStream_t stream, SolveArgs a,
                     int64_t* launches, std::string* err) {
  using R = rj::RJ<NC>;
  const void* fn = (const void*)rj::k_solve_rj<NC>;
  const int nb = blocks_per_sm<NC>(fn);
  if (nb <= 0) {
    *err = "warp-per-patch kernel does not fit on an SM";
    return TILT_E_UNSUPPORTED;
  }
  const size_t wsf = rj::ws_floats_rj<NC>(a.m);
  const size_t slots = ws_floats / wsf;  // warps the workspace can hold
  int blocks = num_sms * nb;
  const int need = (a.B + R::WPB - 1) / R::WPB;
  if (blocks > need) blocks = need;
  if ((size_t)blocks * R::WPB > slots) blocks = (int)(slots / R::WPB);
  if (blocks < 1) {
    *err = "workspace too small for the warp-per-patch kernel";
    return TILT_E_ARG;
  }
  a.ws = ws;
  a.ws_stride = wsf;
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync", err);
  rj::k_solve_rj<NC><<<blocks, R::NT, smem_bytes<NC>(), stream>>>(a);
  ++*launches;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "k_solve_rj", err);
  return TILT_OK;
}

template <int NC>
tilt_status svt_nc(int num_sms, float* ws, size_t ws_floats, cudaStream_t stream, SvtArgs a, int64_t* launches,
                   std::string* err) {
  using R = rj::RJ<NC>;
  const void* fn = (const void*)rj::k_svt_rj<NC>;
  const int nb = blocks_per_sm<NC>(fn);
  if (nb <= 0) {
    *err = "warp-per-patch SVT kernel does not fit on an SM";
    return TILT_E_UNSUPPORTED;
  }
  int blocks = num_sms * nb;
  const int need = (a.B + R::WPB - 1) / R::WPB;
  if (blocks > need) blocks = need;
  const size_t wsf = 2 * (size_t)((a.m + 1) & ~1) * NC + rj::ws_log_floats<NC>();  // B, A planes + log
  if ((size_t)blocks * R::WPB * wsf > ws_floats) blocks = (int)(ws_floats / (wsf * R::WPB));
  if (blocks < 1) {
    *err = "workspace too small for the warp-per-patch SVT";
    return TILT_E_ARG;
  }
  a.ws = ws;
  a.ws_stride = wsf;
  rj::k_svt_rj<NC><<<blocks, R::NT, smem_bytes<NC>(), stream>>>(a);
  ++*launches;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "k_svt_rj", err);
  return TILT_OK;
}

}  // namespace

bool fits(int m, int n) { return m >= 2 && n >= 2 && m <= 64 && n <= 50; }

size_t ws_need(int num_sms, int m, int n) {
  if (!fits(m, n)) return 0;
  return nc_of(n) == 36 ? ws_need_nc<36>(num_sms, m) : ws_need_nc<50>(num_sms, m);
}

tilt_status solve(int num_sms, float* ws, size_t ws_floats, int* counter, cudaStream_t stream, SolveArgs a,
                  int64_t* launches, std::string* err) {
  return nc_of(a.n) == 36 ? solve_nc<36>(num_sms, ws, ws_floats, counter, stream, a, launches, err)
                          : solve_nc<50>(num_sms, ws, ws_floats, counter, stream, a, launches, err);
}

tilt_status svt(int num_sms, float* ws, size_t ws_floats, cudaStream_t stream, SvtArgs a, int64_t* launches,
                std::string* err) {
  return nc_of(a.n) == 36 ? svt_nc<36>(num_sms, ws, ws_floats, stream, a, launches, err)
                          : svt_nc<50>(num_sms, ws, ws_floats, stream, a, launches, err);
}

}  // namespace rjh
}  // namespace tilt

// tilt_large_host.h — host side of the multi-CTA path for large windows (tilt_large.cu), called by
// the C ABI in tilt.cu. Internal interface (not part of include/tilt.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tilt.h"

namespace tilt {
struct DevParams;
namespace lp {

constexpr int MAX_DIM = 1024;  // largest m, n of the multi-CTA path

// Library state of the multi-CTA path (owned by the tilt_handle; workspace allocated on first use).
struct Ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  float* ws = nullptr;       // per-problem slots (planes, V buffers, state)
  size_t ws_floats = 0;
  int* counter = nullptr;    // device: active-problem counter
  int* widx = nullptr;       // device: indices of the problems in a subset GEMM / solve (Alg. 2 steps)
  int cap_b = 0;
  int* h_counter = nullptr;  // pinned host mirror
  int64_t* launches = nullptr;
  std::string* err = nullptr;
  // one Jacobi sweep (the intra-block and cross rounds, the counter reset, k_sweep_end) captured as a
  // CUDA graph: two cached executables keyed by the kernels' argument bytes and the row class
  cudaGraphExec_t sweep_exec[2] = {nullptr, nullptr};
  std::string sweep_key[2];
  int sweep_next = 0;
  cudaStream_t cap_stream = nullptr;  // private stream the sweep is captured on (the user's may be legacy)
  int sweep_tally_seen = 0;           // counter[8] (sweeps run by the graphs) at the last host read
};

// workspace floats of B problems of size m x n with p Jacobian planes
size_t ws_need(int B, int m, int n, int p, bool svdws = false);
// (re)allocate ctx.ws for at least `floats` floats
tilt_status ensure(Ctx& ctx, size_t floats, int B);
void release(Ctx& ctx);

// LADMAP inner loop (tilt_inner_batch semantics) on the multi-CTA path
tilt_status inner(Ctx& ctx, const float* D, const float* J, const float* Q, int l, int B, int m, int n, int p,
                  const DevParams& P, float* A, float* E, float* Y, tilt_report* rep);
// Algorithm 1 (tilt_solve_batch semantics, no pyramid) on the multi-CTA path
tilt_status solve(Ctx& ctx, const float* images, int n_images, int H, int W, const int32_t* patch_image,
                  const int32_t* boxes, const float* tau0, int B, int m, int n, int kind, const DevParams& P,
                  float* tau_out, float* A, float* E, float* Y, tilt_report* rep,
                  const tilt_report* rep_prev = nullptr, const float* warm_A = nullptr,
                  const float* warm_E = nullptr, const float* warm_Y = nullptr,
                  const tilt_report* warm_rep = nullptr);
// SVT (tilt_svt_batch semantics) on the multi-CTA path
tilt_status svt(Ctx& ctx, const float* M, int B, int m, int n, const float* eps, float* V_io, float* A,
                float* sigma, int32_t* sweeps, float tol, int max_sweeps);

}  // namespace lp
}  // namespace tilt

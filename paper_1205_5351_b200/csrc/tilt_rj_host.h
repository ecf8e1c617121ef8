// tilt_rj_host.h — host-side launchers of the warp-per-patch kernels (tilt_rj.cu), called by the
// C ABI in tilt.cu. Internal interface (not part of include/tilt.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tilt.h"

namespace tilt {
struct SolveArgs;
struct SvtArgs;
namespace rjh {

// true if the warp-per-patch kernels handle an m x n window (m <= 64, n <= 50)
bool fits(int m, int n);
// workspace floats needed by the warp-per-patch solve at window (m, n) on num_sms SMs
size_t ws_need(int num_sms, int m, int n);
// persistent warp-per-patch solve of a.B patches (a.ws / a.ws_stride are set here)
tilt_status solve(int num_sms, float* ws, size_t ws_floats, int* counter, cudaStream_t stream, SolveArgs a,
                  int64_t* launches, std::string* err);
// warp-per-patch standalone SVT (step parity)
tilt_status svt(int num_sms, float* ws, size_t ws_floats, cudaStream_t stream, SvtArgs a, int64_t* launches,
                std::string* err);

}  // namespace rjh
}  // namespace tilt

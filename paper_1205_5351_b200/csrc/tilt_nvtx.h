// tilt_nvtx.h — NVTX ranges around the host-side steps of the library (header-only NVTX v3 from
// the CUDA toolkit; free when no tool is attached). Names follow the step ids of DESIGN.md:
// K1 warp/Jacobian, K2 orthonormalise, K3 LADMAP inner loop + SVT, K4 scheduler (the persistent
// solve launch), K5 gather (Python side), plus the multi-CTA path's per-iteration steps.
#pragma once
#include <nvtx3/nvToolsExt.h>

namespace tilt {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace tilt

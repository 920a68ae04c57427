// Shared host-side helpers: error type mirroring tad::ValidationError, CUDA checks.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <stdexcept>
#include <utility>
#include <string>

namespace tamoe {

// Mirrors tad::ValidationError (reference errors.hpp:11-14): malformed inputs and
// failed preconditions. The C-ABI maps it to status 2; anything else is status 1.
class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& what) : std::runtime_error(what) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

#define TAMOE_CUDA(expr) ::tamoe::cuda_check((expr), #expr)

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw ValidationError(msg);
}

// Programmatic dependent launch between the step's kernels (TAMOE_PDL=1; off by default: the N=1 step measured
// 1.155-1.178 ms without vs 1.185-1.195 ms with it, same box, alternating runs).  Every kernel launched this way
// calls griddepcontrol.launch_dependents / .wait (ptx::pdl_trigger / pdl_wait) before it touches memory the
// previous kernel writes or reads; without the attribute both are no-ops.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_PDL");
    return v && v[0] == '1';
  }();
  return on;
}

// kernel<<<grid, block, smem, s>>>(args...) with the programmatic-serialization attribute
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TAMOE_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    TAMOE_CUDA(cudaGetDevice(&dev));
    TAMOE_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

}  // namespace tamoe

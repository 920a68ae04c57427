// Shared host-side helpers: error type mirroring tad::ValidationError, CUDA checks.
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
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

// Exception -> status-code translation for the extern "C" boundary.
// Status mirrors the reference CLI's exit codes (tools/main.cpp:435-441):
// 0 = ok, 1 = internal (CUDA/NCCL/runtime_error), 2 = validation (tad::ValidationError).
#pragma once
#include <exception>
#include <string>

#include "common.hpp"

namespace tamoe {

inline std::string& last_error_slot() {
  static thread_local std::string s;
  return s;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    last_error_slot().clear();
    return 0;
  } catch (const ValidationError& e) {
    last_error_slot() = e.what();
    return 2;
  } catch (const std::exception& e) {
    last_error_slot() = e.what();
    return 1;
  } catch (...) {
    last_error_slot() = "unknown error";
    return 1;
  }
}

}  // namespace tamoe

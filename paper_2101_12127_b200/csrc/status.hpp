// status.hpp -- thread-local error message + status helpers for the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/dpcuda.h"

namespace dpk {

void set_last_error(const std::string& msg);

inline int fail(int code, const std::string& msg) {
  set_last_error(msg);
  return code;
}

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DP_OK;
  return fail(e == cudaErrorMemoryAllocation ? DP_ERR_OUT_OF_MEMORY : DP_ERR_CUDA,
              std::string(what) + ": " + cudaGetErrorString(e));
}

// Checks the launch that was just issued.
inline int launch_status(const char* what) {
  return cuda_status(cudaGetLastError(), what);
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace dpk

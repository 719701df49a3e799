// capi_misc.cpp -- dp_last_error / dp_build_info / dp_device_count.
#include <cuda_runtime.h>

#include <string>

#include "status.hpp"

namespace dpk {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace dpk

extern "C" const char* dp_last_error(void) { return dpk::g_last_error.c_str(); }

extern "C" const char* dp_build_info(void) {
  return "libdpcuda sm_100a; HBM-bound kernels K1-K7 + host engine; built " __DATE__;
}

extern "C" int dp_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    n = 0;
  } else if (e != cudaSuccess) {
    return dpk::cuda_status(e, "cudaGetDeviceCount");
  }
  if (count) *count = n;
  return DP_OK;
}

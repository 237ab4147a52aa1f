// common.cuh -- host-side status/error plumbing shared by the libara translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include "ara.h"

namespace ara {

ara_status set_error(ara_status s, const char* fmt, ...);
ara_status cuda_error(cudaError_t e, const char* what);

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev >= 0 && dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace ara

#define ARA_CUDA(call)                                       \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) return ara::cuda_error(_e, #call); \
  } while (0)

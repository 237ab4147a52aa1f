// common.cuh -- host-side status/error plumbing shared by the libara translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include <nvtx3/nvToolsExt.h>  // header-only: a no-op unless a profiler (nsys, ncu) injects itself

#include "ara.h"

namespace ara {

// NVTX range over an ABI call (host timeline annotation for nsys / ncu --nvtx).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

ara_status set_error(ara_status s, const char* fmt, ...);
ara_status cuda_error(cudaError_t e, const char* what);

// metrics.cu: PML/TVaR into caller-provided device scratch (no allocation, graph-capturable)
size_t metrics_scratch_size(uint64_t n);
ara_status metrics_device_into(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                               double* tvar_dev, char* scratch, size_t bytes, cudaStream_t s, bool zeroed);

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

// testing.cu -- libara_testing.so: test-only read-back of a context's tables (include/ara_testing.h).  Not
// linked into the product library; shares only the internal context layout (ctx.cuh).
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include "ara_testing.h"
#include "ctx.cuh"

namespace {
thread_local char g_terr[256] = "";

ara_status fail(ara_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_terr, sizeof g_terr, fmt, ap);
  va_end(ap);
  return s;
}
}  // namespace

extern "C" {

ara_status ara_table_row(ara_ctx* c, uint32_t layer, uint32_t event, float* out) {
  if (!c || !out || layer >= c->layers.size()) return fail(ARA_E_ARG, "invalid argument");
  if (event > c->C) return fail(ARA_E_RANGE, "event %u > catalog size %u", event, c->C);
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != c->device) cudaSetDevice(c->device);
  const ara::Layer& L = c->layers[layer];
  const cudaError_t e = cudaMemcpy(out, L.table + (uint64_t)event * L.jpad, L.jpad * 4, cudaMemcpyDeviceToHost);
  if (prev >= 0 && prev != c->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return fail(ARA_E_CUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
  return ARA_OK;
}

const char* ara_testing_last_error(void) { return g_terr; }

}  // extern "C"

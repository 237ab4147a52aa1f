// Device YET generator (ARA-GEN-1).  Input generation only -- none of the ARA method lives here.
// Integer-only, so it matches paper_1412_4556_b200/synth/__init__.py bit for bit.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "ara_synth.h"

namespace {

thread_local char g_err[256] = "";

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Each thread writes 4 consecutive ids with one 16-byte store when the destination is aligned.
__global__ void __launch_bounds__(256) yet_ids_kernel(uint32_t* __restrict__ out, uint64_t key, uint64_t q0,
                                                      uint64_t count, uint32_t C) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v * 4 < count; v += nthreads) {
    uint64_t i = v * 4;
    uint32_t id[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint64_t r = sm64(key + q0 + i + u);
      id[u] = 1u + (uint32_t)(((r >> 32) * (uint64_t)C) >> 32);
    }
    if (i + 4 <= count && ((reinterpret_cast<uintptr_t>(out + i) & 15) == 0)) {
      *reinterpret_cast<uint4*>(out + i) = make_uint4(id[0], id[1], id[2], id[3]);
    } else {
      for (int u = 0; u < 4 && i + u < count; ++u) out[i + u] = id[u];
    }
  }
}

}  // namespace

extern "C" int ara_synth_yet_ids(uint32_t* out, uint64_t seed, uint64_t q0, uint64_t count, uint32_t catalog_size,
                                 void* stream) {
  if (catalog_size == 0 || (out == nullptr && count > 0)) {
    snprintf(g_err, sizeof g_err, "invalid argument");
    return 1;
  }
  if (count == 0) return 0;
  const uint64_t s = 1ull << 32;  // kind 1 (YET ids), g = 0
  const uint64_t key = sm64(seed ^ (s * 0xD1B54A32D192ED03ull));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t vec = (count + 3) / 4;
  uint64_t blocks = (vec + 255) / 256;
  uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  yet_ids_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, key, q0, count, catalog_size);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "%s", cudaGetErrorString(e));
    return 6;
  }
  return 0;
}

extern "C" const char* ara_synth_last_error(void) { return g_err; }

// outputs.cu -- further outputs of the analysis ("reports"):
//   ara_aal          average annual loss = mean of a YLT (deterministic fp64 reduction)
//   ara_ep           exceedance probability P(YLT >= x) at given losses (the EP curve / RPL report)
//   ara_sum_layers   program / portfolio totals: per trial, the sum of layer YLTs grouped by program
// The occurrence-basis table (largest occurrence-net loss per trial) is produced by the ARA kernels
// themselves (ara_run_ex); ara_pml / ara_tvar on it give OEP-basis metrics.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "ara.h"
#include "common.cuh"

namespace ara {

constexpr int kOutBlock = 256;
constexpr int kMaxThresholds = 256;
constexpr int kMaxGroupLayers = 128;

struct AalState {
  unsigned int ticket;
  double result;
};

// Block b sums the contiguous chunk [n*b/G, n*(b+1)/G) (thread-strided, then a fixed tree); the last
// block adds the block partials in block order.  Bitwise reproducible for a given n and grid.
__global__ void __launch_bounds__(kOutBlock) aal_kernel(const double* __restrict__ y, uint64_t n,
                                                        double* __restrict__ partial, AalState* st) {
  __shared__ double ws[kOutBlock / 32];
  __shared__ bool last;
  const uint64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  double a = 0.0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) a += y[i];
  for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kOutBlock / 32; ++w) b += ws[w];
    partial[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double s = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) s += ((volatile double*)partial)[b];
  st->result = s / (double)n;
}

__global__ void __launch_bounds__(kOutBlock) ep_kernel(const double* __restrict__ y, uint64_t n,
                                                       const double* __restrict__ x, int m,
                                                       unsigned long long* __restrict__ count) {
  __shared__ unsigned long long c[kMaxThresholds];
  __shared__ double sx[kMaxThresholds];
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    c[i] = 0;
    sx[i] = x[i];
  }
  __syncthreads();
  // warp-uniform trip count (every lane of the warp iterates together), validity as a predicate, so the
  // ballots always see the full warp and lane 0 counts
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const double v = valid ? y[i] : 0.0;
    for (int k = 0; k < m; ++k) {
      const unsigned ball = __ballot_sync(0xffffffffu, valid && v >= sx[k]);
      if ((threadIdx.x & 31) == 0 && ball) atomicAdd(&c[k], (unsigned long long)__popc(ball));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    if (c[i]) atomicAdd(&count[i], c[i]);
}

struct GroupMap {
  uint32_t group[kMaxGroupLayers];
};

__global__ void __launch_bounds__(kOutBlock) sum_layers_kernel(const double* __restrict__ ylt, uint32_t L, uint64_t n,
                                                               const __grid_constant__ GroupMap gm, uint32_t G,
                                                               double* __restrict__ out) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    for (uint32_t g = 0; g < G; ++g) {
      double s = 0.0;
      for (uint32_t l = 0; l < L; ++l)  // layer order
        if (gm.group[l] == g) s += ylt[(uint64_t)l * n + t];
      out[(uint64_t)g * n + t] = s;
    }
  }
}

static int grid_for(uint64_t n, int mult) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t b = (n + kOutBlock - 1) / kOutBlock;
  const uint64_t cap = (uint64_t)sms * mult;
  return (int)(b < cap ? (b ? b : 1) : cap);
}

}  // namespace ara

using namespace ara;

extern "C" {

ara_status ara_aal(const double* ylt, uint64_t n, double* out, void* stream) {
  if (!ylt || !out || n == 0) return set_error(ARA_E_ARG, "invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = grid_for(n, 4);
  char* scratch = nullptr;
  const size_t bytes = sizeof(AalState) + (size_t)grid * sizeof(double);
  ARA_CUDA(cudaMallocAsync((void**)&scratch, bytes, s));
  AalState* st = (AalState*)scratch;
  double* partial = (double*)(scratch + sizeof(AalState));
  cudaError_t e = cudaMemsetAsync(st, 0, sizeof(AalState), s);
  if (e == cudaSuccess) {
    aal_kernel<<<grid, kOutBlock, 0, s>>>(ylt, n, partial, st);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, &st->result, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(scratch, s);
  if (e != cudaSuccess) return cuda_error(e, "ara_aal");
  return ARA_OK;
}

ara_status ara_ep(const double* ylt, uint64_t n, const double* thresholds, uint32_t m, double* out, void* stream) {
  if (!ylt || !thresholds || !out || n == 0 || m == 0 || m > kMaxThresholds)
    return set_error(ARA_E_ARG, "invalid argument (m must be in [1, %d])", kMaxThresholds);
  cudaStream_t s = (cudaStream_t)stream;
  char* scratch = nullptr;
  ARA_CUDA(cudaMallocAsync((void**)&scratch, (size_t)m * (sizeof(double) + sizeof(unsigned long long)), s));
  double* dx = (double*)scratch;
  unsigned long long* dc = (unsigned long long*)(dx + m);
  std::vector<unsigned long long> hc(m);
  cudaError_t e = cudaMemcpyAsync(dx, thresholds, (size_t)m * sizeof(double), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dc, 0, (size_t)m * sizeof(unsigned long long), s);
  if (e == cudaSuccess) {
    ep_kernel<<<grid_for(n, 4), kOutBlock, 0, s>>>(ylt, n, dx, (int)m, dc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), dc, (size_t)m * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(scratch, s);
  if (e != cudaSuccess) return cuda_error(e, "ara_ep");
  for (uint32_t i = 0; i < m; ++i) out[i] = (double)hc[i] / (double)n;
  return ARA_OK;
}

ara_status ara_sum_layers(const double* ylt, uint32_t num_layers, uint64_t n, const uint32_t* group,
                          uint32_t num_groups, double* out, void* stream) {
  if (!ylt || !group || !out || num_layers == 0 || num_groups == 0 || num_layers > kMaxGroupLayers)
    return set_error(ARA_E_ARG, "invalid argument (at most %d layers)", kMaxGroupLayers);
  GroupMap gm;
  memset(&gm, 0, sizeof gm);
  for (uint32_t l = 0; l < num_layers; ++l) {
    if (group[l] >= num_groups) return set_error(ARA_E_ARG, "layer %u: group %u >= %u", l, group[l], num_groups);
    gm.group[l] = group[l];
  }
  if (n == 0) return ARA_OK;
  sum_layers_kernel<<<grid_for(n, 8), kOutBlock, 0, (cudaStream_t)stream>>>(ylt, num_layers, n, gm, num_groups, out);
  ARA_CUDA(cudaGetLastError());
  return ARA_OK;
}

}  // extern "C"

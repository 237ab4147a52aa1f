// Probe: random 4-B lookups into a bitmap distributed over the shared memory of a thread-block cluster
// (ld.shared::cluster), vs the same lookups into the CTA's own shared memory.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int CL, bool REMOTE>
__global__ void __launch_bounds__(1024, 1) k_lookup(uint32_t words_per_cta, int iters, uint32_t* out) {
  extern __shared__ uint32_t sm[];
  for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) sm[i] = i * 2654435761u;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  uint32_t base[CL];
  const uint32_t local = (uint32_t)__cvta_generic_to_shared(sm);
#pragma unroll
  for (int c = 0; c < CL; ++c) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local), "r"(c));
    base[c] = a;
  }
  uint32_t x = threadIdx.x * 7919u + blockIdx.x * 104729u, acc = 0;
  const uint32_t total = words_per_cta * 32u * CL;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x = x * 1664525u + 1013904223u;
      const uint32_t id = __umulhi(x, total);       // bit index over the cluster's bitmap
      const uint32_t c = id / (words_per_cta * 32u);
      const uint32_t wd = (id - c * words_per_cta * 32u) >> 5;
      uint32_t v;
      if (REMOTE) {
        uint32_t bc = base[0];
#pragma unroll
        for (int j = 1; j < CL; ++j) bc = c == (uint32_t)j ? base[j] : bc;
        asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(bc + 4u * wd));
      } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(local + 4u * (wd % words_per_cta)));
      }
      acc += (v >> (id & 31)) & 1u;
    }
  }
  cl.sync();
  if (acc == 0xdeadbeef) out[0] = acc;
}

template <int CL, bool REMOTE>
void run(uint32_t words, int threads) {
  uint32_t* out; cudaMalloc(&out, 4);
  auto k = k_lookup<CL, REMOTE>;
  size_t smem = words * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  int grid = (148 / CL) * CL;
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  int iters = 2000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaLaunchKernelEx(&cfg, k, words, 10, out);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k, words, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double looks = (double)grid * threads * iters * 8;
  printf("cluster %2d %s threads %4d smem %6zu KB: %.2f ms, %.2f lookups/clk/SM (grid %d) err=%s\n", CL,
         REMOTE ? "dsmem" : "local", threads, smem / 1024, ms, looks / grid / (ms * 1e-3 * 1.965e9), grid,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  run<8, false>(40000, 1024);
  run<8, true>(40000, 1024);
  run<8, true>(40000, 768);
  run<4, true>(40000, 1024);
  run<2, true>(40000, 1024);
  run<16, true>(20000, 1024);
  return 0;
}

// Probe: cost of a cooperative launch and of a software grid barrier (atomic ticket + spin), as used by
// metrics_fused, for 148 blocks x 1024 threads.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void grid_sync(unsigned* count, unsigned* gen, unsigned nb, int mode) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = gen;
    const unsigned g = *vgen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      if (mode == 0) while (*vgen == g) __nanosleep(32);
      else while (*vgen == g) {}
    }
    __threadfence();
  }
  __syncthreads();
}
// release/acquire variant: red.release.gpu arrival, ld.acquire.gpu polling
__device__ __forceinline__ void grid_sync_ra(unsigned* count, unsigned nb, unsigned& target) {
  __syncthreads();
  target += nb;
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory"); } while ((int)(v - target) < 0);
  }
  __syncthreads();
}
__global__ void k_bar(unsigned* st, int nbar, int mode) {
  unsigned target = 0;
  for (int i = 0; i < nbar; ++i) {
    if (mode == 2) grid_sync_ra(st + 2, gridDim.x, target);
    else grid_sync(st, st + 1, gridDim.x, mode);
  }
}
int main() {
  unsigned* st; cudaMalloc(&st, 64); 
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 3; ++mode)
  for (int nbar : {0, 1, 9, 33}) {
    float best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemsetAsync(st, 0, 64, s);
      void* args[] = {&st, &nbar, &mode};
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)k_bar, 148, 1024, args, 0, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("mode %d barriers %2d: %.2f us (err %s)\n", mode, nbar, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

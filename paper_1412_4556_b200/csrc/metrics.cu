// metrics.cu -- PML and TVaR of a device YLT (PAPER.md:26, :131 name them; readings c11-c14
// define them): k = ceil(N / RP); PML = k-th largest YLT value; TVaR = mean of the k largest.
//
// Device MSD radix SELECT (no full sort): the YLT doubles are mapped to order-preserving uint64 keys
// and, for all m return periods at once, 8 passes of 8-bit digits narrow each query's key prefix
// until it is the exact key of its k-th largest value T.  Then one pass computes, per query, the
// count c and fp64 sum of values with key > T, and TVaR = (sum + (k - c) * T) / k, which is exact
// under ties (reading c14).  Every pass is one kernel; its last block (ticket counter) finalises the
// pass on the device, so there is no host round trip until the 2m results are copied back.
// Sums are reduced in a fixed order (thread -> warp -> block -> blocks in index order), so results
// are bitwise reproducible run to run.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <vector>

#include "ara.h"
#include "common.cuh"

namespace ara {

constexpr int kMaxQ = 16;        // queries per kernel batch
constexpr int kSelBlock = 256;

struct SelState {
  uint64_t prefix[kMaxQ];  // known high bits of the k-th largest key (right-aligned)
  uint64_t rank[kMaxQ];    // remaining 1-based rank from the top among keys sharing the prefix
  uint64_t k[kMaxQ];
  unsigned int hist[kMaxQ][256];  // per histogram SLOT (distinct prefix), not per query
  unsigned int ticket;
  int nslot;                      // distinct prefixes this pass; queries sharing one share a histogram
  int q2slot[kMaxQ];
  uint64_t slot_prefix[kMaxQ];
  double sum[kMaxQ];       // filled by the tail pass
  unsigned long long cnt[kMaxQ];
};

__device__ __forceinline__ uint64_t to_key(double v) {
  uint64_t b = (uint64_t)__double_as_longlong(v);
  if (b == 0x8000000000000000ull) b = 0;              // -0.0 == +0.0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // order-preserving for all non-NaN doubles
}

__device__ __forceinline__ double from_key(uint64_t k) {
  uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// One radix pass: histogram of digit `pass` (bits 63-8*pass .. 56-8*pass) over the keys that match each
// distinct query prefix (queries with equal prefixes share one histogram slot); the last block picks
// each query's digit and rebuilds the slots for the next pass.
__global__ void __launch_bounds__(kSelBlock) select_pass(const double* __restrict__ y, uint64_t n, int m, int pass,
                                                          SelState* st) {
  __shared__ unsigned int sh[kMaxQ][256];
  __shared__ uint64_t spre[kMaxQ];
  __shared__ int s_nslot;
  __shared__ bool last;
  if (threadIdx.x == 0) s_nslot = st->nslot;
  if (threadIdx.x < kMaxQ) spre[threadIdx.x] = st->slot_prefix[threadIdx.x];
  __syncthreads();
  const int ns = s_nslot;
  for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) sh[i / 256][i % 256] = 0;
  __syncthreads();
  const int shift = 56 - 8 * pass;
  const unsigned FULL = 0xffffffffu;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // Iterate in warp-uniform trip counts so __match_any_sync sees the whole warp.
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const uint64_t key = valid ? to_key(y[i]) : 0;
    const unsigned digit = (unsigned)(key >> shift) & 0xffu;
    const uint64_t hi = pass == 0 ? 0 : (key >> (shift + 8));
    for (int sl = 0; sl < ns; ++sl) {
      const bool hit = valid && hi == spre[sl];
      if (!__any_sync(FULL, hit)) continue;
      const unsigned tag = hit ? digit : 0x100u;
      const unsigned peers = __match_any_sync(FULL, tag);
      if (hit && (__ffs(peers) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&sh[sl][digit], __popc(peers));
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) {
    const unsigned v = sh[i / 256][i % 256];
    if (v) atomicAdd(&st->hist[i / 256][i % 256], v);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&st->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Last block: pull the global histograms into shared memory in parallel, then one thread per query
  // walks its slot's 256 bins from the top (digit 255) to find the bucket holding its remaining rank.
  for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) sh[i / 256][i % 256] = ((volatile unsigned int*)st->hist[i / 256])[i % 256];
  __syncthreads();
  if (threadIdx.x < m) {
    const int q = threadIdx.x;
    const unsigned int* h = sh[st->q2slot[q]];
    uint64_t r = st->rank[q], above = 0;
    int d = 255;
    for (; d > 0; --d) {
      const uint64_t c = h[d];
      if (above + c >= r) break;
      above += c;
    }
    st->rank[q] = r - above;
    st->prefix[q] = (st->prefix[q] << 8) | (uint64_t)d;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) st->hist[i / 256][i % 256] = 0;
  if (threadIdx.x == 0) {
    int k = 0;  // distinct prefixes for the next pass, in query order
    for (int q = 0; q < m; ++q) {
      const uint64_t pq = st->prefix[q];
      int sl = 0;
      while (sl < k && st->slot_prefix[sl] != pq) ++sl;
      if (sl == k) st->slot_prefix[k++] = pq;
      st->q2slot[q] = sl;
    }
    st->nslot = k;
    st->ticket = 0;
  }
}

// Tail pass: per query, count and fp64-sum the values with key > T (T = full prefix after 8 passes).
// Block partials go to part[block][q]; the last block adds them in block order.
__global__ void __launch_bounds__(kSelBlock) tail_pass(const double* __restrict__ y, uint64_t n, int m, SelState* st,
                                                        double* __restrict__ psum,
                                                        unsigned long long* __restrict__ pcnt, double* __restrict__ out) {
  __shared__ uint64_t sT[kMaxQ];
  __shared__ double wsum[kSelBlock / 32][kMaxQ];
  __shared__ unsigned long long wcnt[kSelBlock / 32][kMaxQ];
  __shared__ bool last;
  if (threadIdx.x < m) sT[threadIdx.x] = st->prefix[threadIdx.x];
  __syncthreads();
  double s[kMaxQ];
  unsigned long long c[kMaxQ];
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) {
    s[q] = 0.0;
    c[q] = 0;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = y[i];
    const uint64_t key = to_key(v);
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      if (q < m && key > sT[q]) {
        s[q] += v;
        c[q] += 1;
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < kMaxQ; ++q) {
    if (q >= m) break;
    double a = s[q];
    unsigned long long b = c[q];
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    if (lane == 0) {
      wsum[w][q] = a;
      wcnt[w][q] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    double a = 0.0;
    unsigned long long b = 0;
    for (int i = 0; i < kSelBlock / 32; ++i) {
      a += wsum[i][threadIdx.x];
      b += wcnt[i][threadIdx.x];
    }
    psum[(uint64_t)blockIdx.x * kMaxQ + threadIdx.x] = a;
    pcnt[(uint64_t)blockIdx.x * kMaxQ + threadIdx.x] = b;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(&st->ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Last block: every warp sums a strided subset of the block partials for each query (fixed order),
  // then warp partials are combined in warp order -- deterministic.
  __shared__ double fsum[kSelBlock / 32][kMaxQ];
  __shared__ unsigned long long fcnt[kSelBlock / 32][kMaxQ];
  for (int q = 0; q < m; ++q) {
    double a = 0.0;
    unsigned long long b = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      a += ((volatile double*)psum)[(uint64_t)i * kMaxQ + q];
      b += ((volatile unsigned long long*)pcnt)[(uint64_t)i * kMaxQ + q];
    }
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, off);
      b += __shfl_xor_sync(0xffffffffu, b, off);
    }
    if (lane == 0) {
      fsum[w][q] = a;
      fcnt[w][q] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int q = threadIdx.x;
    double a = 0.0;
    unsigned long long b = 0;
    for (int i = 0; i < kSelBlock / 32; ++i) {
      a += fsum[i][q];
      b += fcnt[i][q];
    }
    const double T = from_key(sT[q]);
    const uint64_t k = st->k[q];
    out[q] = T;                                            // PML: the k-th largest value
    out[kMaxQ + q] = __ddiv_rn(__dadd_rn(a, __dmul_rn((double)(k - b), T)), (double)k);  // TVaR (no FMA contraction)
  }
  if (threadIdx.x == 0) st->ticket = 0;
}

// ------------------------------------------------------------------------------------------------
// Fused variant: ONE cooperative launch runs the 8 radix passes and the tail pass, separated by grid
// barriers.  Each block keeps its contiguous chunk of keys in shared memory (when it fits), so the
// YLT is read from HBM once; every block redundantly derives the per-query digits from the final
// global histogram of the pass (triple-buffered so it can be cleared two passes ahead).
constexpr int kFusedBlock = 1024;   // one block per SM: fewer arrivals at each grid barrier
constexpr int kCacheKeys = 8192;    // 64 KB of cached keys per block (N <= 1.2M on 148 SMs)

struct FusedState {  // zeroed (cudaMemsetAsync) before every launch
  unsigned int H[3][kMaxQ][256];
  unsigned int bar_count, bar_gen;
};

struct FusedQueries {  // kernel parameter
  uint64_t k[kMaxQ];
};

__device__ __forceinline__ void grid_sync(unsigned int* count, unsigned int* gen, unsigned int nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kFusedBlock) metrics_fused(const double* __restrict__ y, uint64_t n, int m,
                                                              FusedState* st, double* __restrict__ psum,
                                                              unsigned long long* __restrict__ pcnt,
                                                              const __grid_constant__ FusedQueries Q,
                                                              double* __restrict__ pml_out, double* __restrict__ tvar_out) {
  extern __shared__ uint64_t skeys[];
  __shared__ unsigned int sh[kMaxQ][256];
  __shared__ uint64_t s_prefix[kMaxQ], s_rank[kMaxQ], s_slot_prefix[kMaxQ];
  __shared__ int s_q2slot[kMaxQ], s_nslot;
  __shared__ double wsum[kFusedBlock / 32][kMaxQ];
  __shared__ unsigned long long wcnt[kFusedBlock / 32][kMaxQ];
  __shared__ uint32_t s_nact, s_nnext;
  // ACTIVE key lists (cached case): after a pass only the keys that fed some slot's histogram can
  // matter to the next passes, so each pass scans the previous pass's survivors only (indices into the
  // cached keys; the tail still reads every key)
  const uint32_t act_s = (uint32_t)__cvta_generic_to_shared(skeys + kCacheKeys);  // two u16 lists of kCacheKeys
  const unsigned FULL = 0xffffffffu;
  const unsigned nb = gridDim.x;
  const uint64_t lo = n * blockIdx.x / nb, hi = n * (blockIdx.x + 1) / nb;
  const uint32_t cnt = (uint32_t)(hi - lo);
  const bool cached = (n + nb - 1) / nb <= (uint64_t)kCacheKeys;  // uniform over blocks
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (cached)
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) skeys[i] = to_key(y[lo + i]);
  if (threadIdx.x < m) {
    s_prefix[threadIdx.x] = 0;
    s_rank[threadIdx.x] = Q.k[threadIdx.x];
    s_q2slot[threadIdx.x] = 0;
  }
  if (threadIdx.x == 0) {
    s_nslot = 1;
    s_slot_prefix[0] = 0;
    s_nact = cnt;
  }
  __syncthreads();
  const unsigned lt = (1u << lane) - 1u;
  for (int pass = 0; pass < 8; ++pass) {
    const int ns = s_nslot;
    for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) sh[i / 256][i % 256] = 0;
    if (threadIdx.x == 0) s_nnext = 0;
    __syncthreads();
    const int shift = 56 - 8 * pass;
    const uint32_t nact = cached ? s_nact : cnt;
    const uint32_t cur_s = act_s + (uint32_t)(pass & 1) * (kCacheKeys * 2u);
    const uint32_t nxt_s = act_s + (uint32_t)((pass + 1) & 1) * (kCacheKeys * 2u);
    for (uint32_t base = 0; base < nact; base += blockDim.x) {  // warp-uniform trip count
      const uint32_t i = base + threadIdx.x;
      const bool valid = i < nact;
      uint32_t idx = i;
      if (pass != 0 && cached && valid) {
        unsigned short v16;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v16) : "r"(cur_s + 2u * i) : "memory");
        idx = v16;
      }
      const uint64_t key = valid ? (cached ? skeys[idx] : to_key(y[lo + idx])) : 0;
      const unsigned digit = (unsigned)(key >> shift) & 0xffu;
      const uint64_t hik = pass == 0 ? 0 : (key >> (shift + 8));
      // the slots' prefixes are distinct, so a key feeds at most one slot's histogram
      int sl = -1;
      if (valid)
        for (int j = 0; j < ns; ++j)
          if (hik == s_slot_prefix[j]) sl = j;
      const unsigned keep = __ballot_sync(FULL, sl >= 0);
      if (keep == 0u) continue;
      if (cached) {  // survivors of this pass (order is irrelevant to the histograms)
        uint32_t at = 0;
        if (lane == __ffs(keep) - 1) at = atomicAdd(&s_nnext, (uint32_t)__popc(keep));
        at = __shfl_sync(FULL, at, __ffs(keep) - 1);
        if (sl >= 0)
          asm volatile("st.shared.u16 [%0], %1;" ::"r"(nxt_s + 2u * (at + __popc(keep & lt))), "h"((unsigned short)idx)
                       : "memory");
      }
      const unsigned bin = sl >= 0 ? ((unsigned)sl << 8 | digit) : 0xffffffffu;
      const unsigned peers = __match_any_sync(FULL, bin);  // warp-aggregated shared atomics
      if (sl >= 0 && (__ffs(peers) - 1) == lane) atomicAdd(&sh[sl][digit], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x == 0) s_nact = s_nnext;
    unsigned int(*H)[256] = st->H[pass % 3];
    for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) {
      const unsigned v = sh[i / 256][i % 256];
      if (v) atomicAdd(&H[i / 256][i % 256], v);
    }
    if (blockIdx.x == 0)  // clear the buffer pass+1 will use (last read before the previous barrier)
      for (int i = threadIdx.x; i < kMaxQ * 256; i += blockDim.x) st->H[(pass + 1) % 3][i / 256][i % 256] = 0;
    grid_sync(&st->bar_count, &st->bar_gen, nb);
    for (int i = threadIdx.x; i < ns * 256; i += blockDim.x) sh[i / 256][i % 256] = ((volatile unsigned int*)H[i / 256])[i % 256];
    __syncthreads();
    if (w < m) {  // warp q: the digit d of query q's k-th largest key among the keys of its slot
      const int q = w;
      const unsigned int* h = sh[s_q2slot[q]];
      const uint64_t r = s_rank[q];
      // lane l owns digits 255 - 8l .. 248 - 8l (descending); exclusive prefix of the lane totals
      uint64_t c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = h[255 - 8 * lane - j];
        tot += c[j];
      }
      uint64_t above = tot;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(FULL, above, off);
        if (lane >= off) above += o;
      }
      above -= tot;  // count of keys in the slot with a larger digit than this lane's bins
      // the lane whose range holds rank r finds its digit (digit 0 if the rank runs past every bin)
      const bool mine = above < r && (r <= above + tot || lane == 31);
      const unsigned who = __ballot_sync(FULL, mine);
      const int src = __ffs(who) - 1;
      int d = 0;
      uint64_t ab = above;
      if (lane == src) {
        d = 248 - 8 * lane;  // lowest digit of the range (taken if the rank runs past it)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int dj = 255 - 8 * lane - j;
          if (ab + c[j] >= r) {
            d = dj;
            break;
          }
          if (dj == 0) {  // rank beyond the slot's keys cannot happen for a valid k; keep digit 0
            d = 0;
            break;
          }
          ab += c[j];
        }
      }
      d = __shfl_sync(FULL, d, src);
      ab = __shfl_sync(FULL, ab, src);
      if (lane == 0) {
        s_rank[q] = r - ab;
        s_prefix[q] = (s_prefix[q] << 8) | (uint64_t)d;
      }
    }
    __syncthreads();
    if (w == 0) {  // slots = distinct prefixes, numbered in query order
      const uint64_t pq = lane < m ? s_prefix[lane] : ~0ull;
      int first = lane;
      for (int q2 = 0; q2 < m; ++q2)
        if (q2 < first && s_prefix[q2] == pq) first = q2;
      const unsigned leaders = __ballot_sync(FULL, lane < m && first == lane);
      if (lane < m) {
        const int sl = __popc(leaders & ((1u << first) - 1u));
        s_q2slot[lane] = sl;
        if (first == lane) s_slot_prefix[sl] = pq;
      }
      if (lane == 0) s_nslot = __popc(leaders);
    }
    __syncthreads();
  }
  // tail: count and fp64-sum the values above each query's threshold T (fixed reduction order), four
  // queries per sweep over the keys (each key decoded once per sweep; every query still adds its keys
  // in the same thread order as a query-at-a-time loop)
  for (int q0 = 0; q0 < m; q0 += 4) {
    uint64_t pq[4];
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t b[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int j = 0; j < 4; ++j) pq[j] = q0 + j < m ? s_prefix[q0 + j] : ~0ull;  // no key exceeds ~0
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint64_t key = cached ? skeys[i] : to_key(y[lo + i]);
      const double v = from_key(key);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (key > pq[j]) {
          a[j] += v;
          b[j] += 1u;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double aj = a[j];
      unsigned long long bj = b[j];
      for (int off = 16; off > 0; off >>= 1) {
        aj += __shfl_xor_sync(FULL, aj, off);
        bj += __shfl_xor_sync(FULL, bj, off);
      }
      if (lane == 0 && q0 + j < m) {
        wsum[w][q0 + j] = aj;
        wcnt[w][q0 + j] = bj;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    double a = 0.0;
    unsigned long long b = 0;
    for (int i = 0; i < kFusedBlock / 32; ++i) {
      a += wsum[i][threadIdx.x];
      b += wcnt[i][threadIdx.x];
    }
    psum[(uint64_t)blockIdx.x * kMaxQ + threadIdx.x] = a;
    pcnt[(uint64_t)blockIdx.x * kMaxQ + threadIdx.x] = b;
  }
  grid_sync(&st->bar_count, &st->bar_gen, nb);
  if (blockIdx.x != 0) return;
  if (w < m) {  // warp q combines the block partials of query q in a fixed order
    const int q = w;
    double a = 0.0;
    unsigned long long b = 0;
    for (unsigned i = lane; i < nb; i += 32) {
      a += ((volatile double*)psum)[(uint64_t)i * kMaxQ + q];
      b += ((volatile unsigned long long*)pcnt)[(uint64_t)i * kMaxQ + q];
    }
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(FULL, a, off);
      b += __shfl_xor_sync(FULL, b, off);
    }
    if (lane == 0) {
      const double T = from_key(s_prefix[q]);
      const uint64_t k = Q.k[q];
      if (pml_out) pml_out[q] = T;  // PML: the k-th largest value
      if (tvar_out) tvar_out[q] = __ddiv_rn(__dadd_rn(a, __dmul_rn((double)(k - b), T)), (double)k);  // TVaR
    }
  }
}

// Per-device launch facts of the fused kernel, queried once (host-side cache; no per-call queries).
struct FusedInfo {
  int ready = 0, coop = 0, sms = 148, occ = 0;
};
static FusedInfo g_fused[64];

static const FusedInfo& fused_info() {
  int dev = 0;
  cudaGetDevice(&dev);
  FusedInfo& f = g_fused[dev & 63];
  if (!f.ready) {
    // the per-call metric scratch comes from the device's stream-ordered pool: keep freed blocks in the
    // pool (no trimming at synchronisation points), so a call never goes back to the driver for memory
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    cudaDeviceGetAttribute(&f.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&f.coop, cudaDevAttrCooperativeLaunch, dev);
    const size_t dyn = (size_t)kCacheKeys * (sizeof(uint64_t) + 2 * sizeof(uint16_t));
    cudaFuncSetAttribute((const void*)metrics_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f.occ, (const void*)metrics_fused, kFusedBlock, dyn) != cudaSuccess) {
      cudaGetLastError();
      f.occ = 0;
    }
    f.ready = 1;
  }
  return f;
}

// Launch the fused kernel cooperatively for one batch of <= kMaxQ queries, results to DEVICE pml/tvar
// (either may be null); asynchronous.  Returns false if the device refuses a cooperative launch of the
// needed size (callers fall back to the pass kernels).
static bool metrics_fused_batch(const double* ylt, uint64_t n, int mq, const uint64_t* ks, char* scratch,
                                size_t scratch_bytes, double* pml_dev, double* tvar_dev, cudaStream_t s,
                                cudaError_t* err) {
  *err = cudaSuccess;
  const FusedInfo& f = fused_info();
  if (!f.coop || f.occ < 1) return false;
  const size_t dyn = (size_t)kCacheKeys * (sizeof(uint64_t) + 2 * sizeof(uint16_t));
  uint64_t grid = (uint64_t)f.sms * f.occ;
  const uint64_t need = (n + kFusedBlock - 1) / kFusedBlock;
  if (grid > need) grid = need;
  const size_t state = sizeof(FusedState);
  const size_t need_bytes = state + grid * kMaxQ * (sizeof(double) + sizeof(unsigned long long));
  if (need_bytes > scratch_bytes) return false;
  FusedState* st = (FusedState*)scratch;
  double* psum = (double*)(scratch + state);
  unsigned long long* pcnt = (unsigned long long*)(psum + grid * kMaxQ);
  FusedQueries Q;
  memset(&Q, 0, sizeof Q);
  for (int q = 0; q < mq; ++q) Q.k[q] = ks[q];
  if ((*err = cudaMemsetAsync(st, 0, sizeof(FusedState), s)) != cudaSuccess) return true;
  int m_ = mq;
  void* args[] = {(void*)&ylt, (void*)&n, (void*)&m_, (void*)&st, (void*)&psum, (void*)&pcnt, (void*)&Q,
                  (void*)&pml_dev, (void*)&tvar_dev};
  *err = cudaLaunchCooperativeKernel((const void*)metrics_fused, dim3((unsigned)grid), dim3(kFusedBlock), args, dyn, s);
  return true;
}

// k = ceil(n / RP) (reading c12): exact integer ceil for integral RP, fuzzed otherwise.  0 = invalid.
static uint64_t metric_rank(uint64_t n, double rp) {
  if (!(rp > 1.0) || !(rp <= (double)n) || !isfinite(rp)) return 0;
  if (rp == floor(rp) && rp < 9007199254740992.0) {
    const uint64_t r = (uint64_t)rp;
    return n / r + (n % r ? 1 : 0);
  }
  const double x = (double)n / rp;
  return (uint64_t)ceil(x - 1e-9 * x);
}

static ara_status ranks_for(uint64_t n, const double* rps, uint32_t m, std::vector<uint64_t>& ks) {
  if (!rps || n == 0 || m == 0 || m > ARA_MAX_RETURN_PERIODS) return set_error(ARA_E_ARG, "invalid metric arguments");
  ks.resize(m);
  for (uint32_t i = 0; i < m; ++i) {
    ks[i] = metric_rank(n, rps[i]);
    if (!ks[i]) return set_error(ARA_E_RANGE, "return period %g outside (1, %llu]", rps[i], (unsigned long long)n);
  }
  return ARA_OK;
}

// Scratch: [2*kMaxQ doubles of batch results][state][block partials].
static size_t scratch_bytes(uint64_t n, uint64_t* blocks_out) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + kSelBlock - 1) / kSelBlock;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;  // covers the fused grid (<= SMs x occupancy)
  *blocks_out = blocks;
  return 2 * kMaxQ * sizeof(double) + std::max(sizeof(SelState), sizeof(FusedState)) +
         blocks * kMaxQ * (sizeof(double) + sizeof(unsigned long long));
}

static ara_status metrics(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml, double* tvar,
                          cudaStream_t s) {
  const bool use_fused = getenv("ARA_METRICS_PASSES") == nullptr;  // env switch keeps the pass kernels testable
  if (!ylt) return set_error(ARA_E_ARG, "ylt is NULL");
  std::vector<uint64_t> ks;
  ara_status rc = ranks_for(n, rps, m, ks);
  if (rc) return rc;
  uint64_t blocks = 0;
  const size_t bytes = scratch_bytes(n, &blocks);
  char* scratch = nullptr;
  ARA_CUDA(cudaMallocAsync((void**)&scratch, bytes, s));
  double* d_out = (double*)scratch;
  ARA_CUDA(cudaMemsetAsync(d_out, 0, 2 * kMaxQ * sizeof(double), s));  // every copied-back slot defined
  char* rest = scratch + 2 * kMaxQ * sizeof(double);
  const size_t rest_bytes = bytes - 2 * kMaxQ * sizeof(double);
  SelState* st = (SelState*)rest;
  double* psum = (double*)(rest + std::max(sizeof(SelState), sizeof(FusedState)));
  unsigned long long* pcnt = (unsigned long long*)(psum + blocks * kMaxQ);
  std::vector<double> h_out(2 * kMaxQ);
  SelState init;
  for (uint32_t q0 = 0; q0 < m && rc == ARA_OK; q0 += kMaxQ) {
    const int mq = (int)std::min<uint32_t>(kMaxQ, m - q0);
    cudaError_t e = cudaSuccess;
    if (!(use_fused && metrics_fused_batch(ylt, n, mq, &ks[q0], rest, rest_bytes, d_out, d_out + kMaxQ, s, &e))) {
      memset(&init, 0, sizeof init);
      for (int q = 0; q < mq; ++q) {
        init.rank[q] = ks[q0 + q];
        init.k[q] = ks[q0 + q];
        init.q2slot[q] = 0;
      }
      init.nslot = 1;  // pass 0: every prefix is empty
      init.slot_prefix[0] = 0;
      e = cudaMemcpyAsync(st, &init, sizeof init, cudaMemcpyHostToDevice, s);
      for (int pass = 0; pass < 8 && e == cudaSuccess; ++pass) {
        select_pass<<<(unsigned)blocks, kSelBlock, 0, s>>>(ylt, n, mq, pass, st);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) {
        tail_pass<<<(unsigned)blocks, kSelBlock, 0, s>>>(ylt, n, mq, st, psum, pcnt, d_out);
        e = cudaGetLastError();
      }
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_out.data(), d_out, 2 * kMaxQ * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      rc = cuda_error(e, "metric kernels");
      break;
    }
    for (int q = 0; q < mq; ++q) {
      if (pml) pml[q0 + q] = h_out[q];
      if (tvar) tvar[q0 + q] = h_out[kMaxQ + q];
    }
  }
  cudaFreeAsync(scratch, s);
  return rc;
}

// Asynchronous variant into caller-provided device scratch (metrics_scratch_size(n) bytes): results to
// DEVICE pml_dev[m] / tvar_dev[m]; needs cooperative launch.  No allocation, no synchronisation, so it
// can be captured into a CUDA graph (ara_plan_create).
ara_status metrics_device_into(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                               double* tvar_dev, char* scratch, size_t bytes, cudaStream_t s) {
  if (!ylt || (!pml_dev && !tvar_dev)) return set_error(ARA_E_ARG, "NULL argument");
  std::vector<uint64_t> ks;
  ara_status rc = ranks_for(n, rps, m, ks);
  if (rc) return rc;
  for (uint32_t q0 = 0; q0 < m && rc == ARA_OK; q0 += kMaxQ) {
    const int mq = (int)std::min<uint32_t>(kMaxQ, m - q0);
    cudaError_t e = cudaSuccess;
    if (!metrics_fused_batch(ylt, n, mq, &ks[q0], scratch, bytes, pml_dev ? pml_dev + q0 : nullptr,
                             tvar_dev ? tvar_dev + q0 : nullptr, s, &e))
      rc = set_error(ARA_E_UNSUPPORTED, "cooperative launch unavailable for the asynchronous metrics");
    else if (e != cudaSuccess)
      rc = cuda_error(e, "fused metric kernel");
  }
  return rc;
}

size_t metrics_scratch_size(uint64_t n) {
  uint64_t blocks = 0;
  return scratch_bytes(n, &blocks);
}

// Asynchronous variant with its own stream-ordered scratch allocation.
static ara_status metrics_device(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                                 double* tvar_dev, cudaStream_t s) {
  if (!ylt || (!pml_dev && !tvar_dev)) return set_error(ARA_E_ARG, "NULL argument");
  const size_t bytes = metrics_scratch_size(n);
  char* scratch = nullptr;
  ARA_CUDA(cudaMallocAsync((void**)&scratch, bytes, s));
  ara_status rc = metrics_device_into(ylt, n, rps, m, pml_dev, tvar_dev, scratch, bytes, s);
  cudaFreeAsync(scratch, s);
  return rc;
}

}  // namespace ara

extern "C" {

ara_status ara_pml_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_out,
                        double* tvar_out, void* stream) {
  if (!pml_out && !tvar_out) return ara::set_error(ARA_E_ARG, "no output");
  return ara::metrics(ylt, n, rps, m, pml_out, tvar_out, (cudaStream_t)stream);
}

ara_status ara_pml_tvar_device(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                               double* tvar_dev, void* stream) {
  return ara::metrics_device(ylt, n, rps, m, pml_dev, tvar_dev, (cudaStream_t)stream);
}

ara_status ara_pml(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out, void* stream) {
  if (!out) return ara::set_error(ARA_E_ARG, "out is NULL");
  return ara::metrics(ylt, n, rps, m, out, nullptr, (cudaStream_t)stream);
}

ara_status ara_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out, void* stream) {
  if (!out) return ara::set_error(ARA_E_ARG, "out is NULL");
  return ara::metrics(ylt, n, rps, m, nullptr, out, (cudaStream_t)stream);
}

}  // extern "C"

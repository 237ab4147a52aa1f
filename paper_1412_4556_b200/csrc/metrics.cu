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
#include <stddef.h>
#include <stdint.h>
#include <stdio.h>
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
// metrics_select: ONE cooperative launch (one 1024-thread block per SM) selects every query's k-th
// largest key with as few grid barriers as the data allow (typically 3; at most 6):
//
//   A  every block caches its contiguous chunk of keys in shared memory and histograms the top 16 bits
//      (65,536 u16 bins in shared memory; a 256-bin coarse histogram beside the fine one in global
//      memory), and publishes its chunk's largest and smallest key with their multiplicities;
//      -- barrier --  a query whose rank falls on the global maximum (or minimum) key is DONE (T = that
//      key: the tie block of capped or zero years, reading c14); every other query finds its 16-bit
//      bucket (coarse, then fine bins) and its rank inside it;
//   H  while a query's bucket holds more than kCandCap keys: histogram the next 12 bits of the keys of
//      each such bucket (distinct buckets share nothing; queries in one bucket share its histogram)
//      -- barrier --  narrow (coarse 64 + fine 64 bins); a full 64-bit prefix is the key itself (DONE);
//   C  every bucket of <= kCandCap keys is COMPACTED into a global candidate list, and every block sums,
//      per query, the values above the query's bucket (or above T) in a fixed order -- barrier --;
//   F  block 0 sorts each candidate list (rank counting: at most kCandCap keys), reads T = the rank's
//      key, and TVaR = (sum above T + (k - count above T) * T) / k with the block partials combined in
//      block order, then the candidates above T in descending order -- bitwise reproducible.
//
// The global histograms of passes H live in scratch that every launch zeroes during pass A; pass A's
// own histogram is zeroed by the launch that used it, after its last reader (the scratch is zeroed once
// when it is allocated).  Barrier state is self-resetting.
constexpr int kSelThreads = 1024;
constexpr uint32_t kSelCache = 8192;      // cached keys per block (64 KB): n <= 8192 * SMs is read once
constexpr uint32_t kSelHistWords = 32768; // 128 KB of packed u16 bin counters
constexpr uint32_t kSelMapWords = 2048 + 512 + 2048;  // first H pass: 65,536-bit prefix map + u8 word bases;
                                                    // pass C: 65,536-bit map of the candidate buckets' prefixes
constexpr uint32_t kSelSub = 65535;       // keys per histogram sub-chunk (a u16 counter cannot overflow)
constexpr uint32_t kCandCap = 256;        // bucket size compacted instead of narrowed further
constexpr int kSelMaxBlocks = 160;      // >= the SM count (148 on B200): one block per SM
constexpr int kSelHPasses = 4;            // 16 + 4 x 12 = 64 bits
enum : int { kModeHist = 0, kModeCand = 1, kModeDone = 2 };

struct alignas(16) SelScratch {  // global scratch of metrics_select
  // -- must hold zeros when a launch starts (cleared when the scratch is allocated; every launch leaves
  //    them zero again)
  unsigned bar_count, bar_exit;
  alignas(16) unsigned HA_c[256];
  alignas(16) unsigned HA_f[65536];
  // -- written before they are read within a launch
  alignas(16) unsigned HB_c[kSelHPasses][kMaxQ][64];
  alignas(16) unsigned HB_f[kSelHPasses][kMaxQ][4096];
  unsigned long long bmax[kSelMaxBlocks], bmin[kSelMaxBlocks];
  unsigned bcmax[kSelMaxBlocks], bcmin[kSelMaxBlocks];
  unsigned cand_bn[kMaxQ][kSelMaxBlocks];                     // candidates of slot s held by block b
  double psum[kSelMaxBlocks][kMaxQ];
  unsigned long long trace[kSelMaxBlocks][24];                // ARA_METRICS_TRACE: %globaltimer per block and phase
  unsigned long long cand_b[kSelMaxBlocks][kMaxQ][kCandCap];  // block b's candidates of slot s
};
constexpr size_t kSelZeroBytes = offsetof(SelScratch, HB_c);  // the part a fresh scratch must have zeroed

struct SelQueries {  // kernel parameter
  uint64_t k[kMaxQ];
};

// Grid barrier: arrival by a release reduction, polling by acquire loads of a counter that only grows
// during a launch (barrier i waits for i * gridDim.x arrivals); the last block past the final barrier
// resets it.  Measured on B200 (148 x 1024 threads): ~1.3 us per barrier, vs ~2.3 us for a fence +
// atomic + generation-flag barrier.
__device__ __forceinline__ void grid_sync(unsigned int* count, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// Warp: the digit d of the bucket holding rank r (1-based from the top) of a histogram of 32*PER bins
// in global memory (h[0] = digit 0), and the count of keys in larger digits.  Lane l owns the bins
// 32*PER-1-PER*l .. 32*PER-PER*l (descending).  Requires r <= the histogram's total.
template <int PER, bool SHARED = false>
__device__ __forceinline__ void find_digit(const unsigned* h, uint32_t r, int lane, uint32_t& d, uint32_t& above) {
  constexpr int NB = 32 * PER;
  uint32_t c[PER], tot = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    c[j] = SHARED ? h[NB - 1 - PER * lane - j] : __ldcg(h + NB - 1 - PER * lane - j);
    tot += c[j];
  }
  uint32_t incl = tot;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  const uint32_t ab0 = incl - tot;
  const unsigned who = __ballot_sync(0xffffffffu, ab0 < r && r <= incl);
  const int src = who ? __ffs(who) - 1 : 31;
  uint32_t dd = 0, ab = ab0;
  if (lane == src) {
    dd = (uint32_t)(NB - PER * lane - PER);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      if (ab + c[j] >= r) {
        dd = (uint32_t)(NB - 1 - PER * lane - j);
        break;
      }
      ab += c[j];
    }
  }
  d = __shfl_sync(0xffffffffu, dd, src);
  above = __shfl_sync(0xffffffffu, ab, src);
}

// Zero `words` (a multiple of 4) 32-bit words of shared memory with 16-B stores.
__device__ __forceinline__ void zero_words(uint32_t* hw, uint32_t words) {
  uint4* z = reinterpret_cast<uint4*>(hw);
  for (uint32_t i = threadIdx.x; i < words / 4u; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
}

// Flush the 64 packed u16 bins of words 32t .. 32t+31 (t = the calling thread's range) into the global
// fine histogram fine[0 .. 64) (atomics for non-zero bins only; most words are zero), return their total.
__device__ __forceinline__ uint32_t flush_range(const uint32_t* hw, uint32_t t, unsigned* fine, int lane) {
  const uint4* h4 = reinterpret_cast<const uint4*>(hw) + 8u * t;
  uint32_t tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int jj = (j + lane) & 7;  // rotated: the 8 threads of a quarter-warp hit distinct banks
    const uint4 v = h4[jj];
    if ((v.x | v.y | v.z | v.w) != 0u) {
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t lo16 = wv[c] & 0xffffu, hi16 = wv[c] >> 16;
        if (lo16) atomicAdd(fine + 8 * jj + 2 * c, lo16);
        if (hi16) atomicAdd(fine + 8 * jj + 2 * c + 1, hi16);
        tot += lo16 + hi16;
      }
    }
  }
  return tot;
}

// Packed u16 bin counter += 1 for every lane of the warp holding `bin` (warp-aggregated).
__device__ __forceinline__ void hist_add(uint32_t* hw, bool valid, uint32_t bin, int lane) {
  if (valid) atomicAdd(hw + (bin >> 1), 1u << ((bin & 1u) * 16u));
}

// (value, multiplicity) of the largest / smallest key seen: merge another pair into (v, c)
__device__ __forceinline__ void merge_max(uint64_t& v, uint32_t& c, uint64_t v2, uint32_t c2) {
  c = v2 > v ? c2 : (v2 == v ? c + c2 : c);
  v = v2 > v ? v2 : v;
}
__device__ __forceinline__ void merge_min(uint64_t& v, uint32_t& c, uint64_t v2, uint32_t c2) {
  c = v2 < v ? c2 : (v2 == v ? c + c2 : c);
  v = v2 < v ? v2 : v;
}
__device__ __forceinline__ void warp_merge_extremes(uint64_t& mx, uint32_t& cx, uint64_t& mn, uint32_t& cn) {
  // warp reductions (REDUX) on the 32-bit halves: the high words, then the low words among the lanes that
  // hold the extreme high word, then the multiplicities of the extreme key
  const unsigned FULL = 0xffffffffu;
  const uint32_t hx = __reduce_max_sync(FULL, (uint32_t)(mx >> 32));
  const uint32_t lx = __reduce_max_sync(FULL, (uint32_t)(mx >> 32) == hx ? (uint32_t)mx : 0u);
  const uint64_t gx = ((uint64_t)hx << 32) | lx;
  cx = __reduce_add_sync(FULL, mx == gx ? cx : 0u);
  mx = gx;
  const uint32_t hn = __reduce_min_sync(FULL, (uint32_t)(mn >> 32));
  const uint32_t ln = __reduce_min_sync(FULL, (uint32_t)(mn >> 32) == hn ? (uint32_t)mn : 0xffffffffu);
  const uint64_t gn = ((uint64_t)hn << 32) | ln;
  cn = __reduce_add_sync(FULL, mn == gn ? cn : 0u);
  mn = gn;
}

// Index of the slot whose key range [slo, shi] holds `key` among `ns` disjoint ranges sorted by slo, else -1.
__device__ __forceinline__ int find_range(uint64_t key, const uint64_t* slo, const uint64_t* shi, int ns) {
  if (ns == 0 || key < slo[0]) return -1;
  int i = 0;
#pragma unroll
  for (int step = 8; step > 0; step >>= 1)
    if (i + step < ns && slo[i + step] <= key) i += step;
  return key <= shi[i] ? i : -1;
}

// Warp 0: the distinct key ranges [lo, hi] of the queries q < m with s_mode[q] == mode, sorted ascending
// (disjoint: equal ranges are one slot), into slo/shi; q2slot[q] = the query's slot; returns the count.
__device__ __forceinline__ void build_slots(int mode, int m, const int* s_mode, const uint64_t* s_pre,
                                            const int* s_nbits, uint64_t* slo, uint64_t* shi, int* q2slot, int* nslot,
                                            int lane) {
  const bool in = lane < m && s_mode[lane] == mode;
  uint64_t lo = ~0ull, hi = ~0ull;
  if (in) {
    const int rb = 64 - s_nbits[lane];
    lo = s_pre[lane] << rb;
    hi = lo | ((1ull << rb) - 1ull);
  }
  // distinct ranges: a query leads its range if no lower lane holds the same one (a range's lo is never ~0,
  // the value every other lane holds)
  const unsigned peers = __match_any_sync(0xffffffffu, lo);
  const bool lead = in && (__ffs(peers) - 1) == lane;
  int rank = 0;  // number of distinct ranges below this one
  const unsigned leaders = __ballot_sync(0xffffffffu, lead);
  for (int j = 0; j < m; ++j) {
    const uint64_t lj = __shfl_sync(0xffffffffu, lo, j);
    if (((leaders >> j) & 1u) && lj < lo) ++rank;
  }
  if (lead) {
    slo[rank] = lo;
    shi[rank] = hi;
  }
  if (in) q2slot[lane] = rank;
  if (lane == 0) *nslot = __popc(leaders);
}

template <bool CACHED>
__global__ void __launch_bounds__(kSelThreads, 1) metrics_select(const double* __restrict__ y, uint64_t n, int m,
                                                                 SelScratch* __restrict__ S,
                                                                 const __grid_constant__ SelQueries Q,
                                                                 double* __restrict__ pml_out, double* __restrict__ tvar_out,
                                                                 int trace) {
  extern __shared__ __align__(16) uint64_t sdyn[];
  uint64_t* skeys = sdyn;                                        // [kSelCache]
  uint32_t* hw = reinterpret_cast<uint32_t*>(sdyn + kSelCache);  // [kSelHistWords] packed u16 bins
  uint32_t* smap = hw + kSelHistWords;  // first H pass: bit d = 16-bit prefix d is a slot; then u8 bases
  uint32_t* cmap = smap + 2560;         // pass C: bit d = 16-bit prefix d opens a candidate bucket
  for (uint32_t i = threadIdx.x; i < 2048u; i += blockDim.x) cmap[i] = 0u;  // (visible after pass A's barriers)
  __shared__ uint64_t s_pre[kMaxQ], s_T[kMaxQ], s_up[kMaxQ], s_slo[kMaxQ], s_shi[kMaxQ];
  __shared__ uint32_t s_r[kMaxQ], s_above[kMaxQ];  // rank inside the bucket; keys above the bucket (or T)
  __shared__ int s_nbits[kMaxQ], s_mode[kMaxQ], s_q2slot[kMaxQ], s_nslot;
  __shared__ unsigned long long s_ev[2][32];
  __shared__ uint32_t s_ec[2][32];
  const unsigned FULL = 0xffffffffu;
  const unsigned nb = gridDim.x;
  const uint64_t lo = n * blockIdx.x / nb, hi = n * (blockIdx.x + 1) / nb;
  const uint32_t cnt = (uint32_t)(hi - lo);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned bar_target = 0;
  auto key_at = [&](uint32_t i) -> uint64_t {
    if constexpr (CACHED) return skeys[i];
    else return to_key(__ldg(y + lo + i));
  };
  int tp = 0;
  auto stamp = [&]() {  // ARA_METRICS_TRACE: phase boundaries
    if (trace && threadIdx.x == 0 && tp < 24) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      S->trace[blockIdx.x][tp] = t;
    }
    ++tp;
  };
  stamp();
  // ---- zero the pass-H histograms of this launch (this block's share) and the candidate counters
  {
    const uint32_t words = (uint32_t)((sizeof(S->HB_c) + sizeof(S->HB_f)) / 4);
    uint32_t* z = &S->HB_c[0][0][0];
    const uint32_t per = (words + nb - 1) / nb, b0 = per * blockIdx.x, b1 = min(words, b0 + per);
    for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) z[i] = 0u;
  }
  // ---- pass A: cache the keys, histogram the top 16 bits, chunk max/min with multiplicities
  if constexpr (CACHED) {  // all of a thread's loads in flight at once (<= 8: cnt <= kSelCache)
    double v[kSelCache / kSelThreads];
#pragma unroll
    for (uint32_t j = 0; j < kSelCache / kSelThreads; ++j) {
      const uint32_t i = threadIdx.x + j * kSelThreads;
      v[j] = i < cnt ? __ldg(y + lo + i) : 0.0;
    }
#pragma unroll
    for (uint32_t j = 0; j < kSelCache / kSelThreads; ++j) {
      const uint32_t i = threadIdx.x + j * kSelThreads;
      if (i < cnt) skeys[i] = to_key(v[j]);
    }
  }
  uint64_t mx = 0, mn = ~0ull;
  uint32_t cx = 0, cn = 0;
  for (uint32_t s0 = 0;; s0 += kSelSub) {
    const uint32_t s1 = min(cnt, s0 + kSelSub);
    zero_words(hw, kSelHistWords);
    __syncthreads();
    stamp();
    for (uint32_t base = s0; base < s1; base += blockDim.x) {  // warp-uniform trip count
      const uint32_t i = base + threadIdx.x;
      const bool valid = i < s1;
      const uint64_t key = valid ? key_at(i) : 0;
      if (valid) {
        merge_max(mx, cx, key, 1u);
        merge_min(mn, cn, key, 1u);
      }
      hist_add(hw, valid, (uint32_t)(key >> 48), lane);
    }
    __syncthreads();
    stamp();
    {  // thread t: bins 64t .. 64t+63 (a quarter of coarse bin t / 4)
      uint32_t csum = flush_range(hw, threadIdx.x, S->HA_f + 64u * threadIdx.x, lane);
      csum += __shfl_xor_sync(FULL, csum, 1);
      csum += __shfl_xor_sync(FULL, csum, 2);
      if ((threadIdx.x & 3u) == 0u && csum) atomicAdd(&S->HA_c[threadIdx.x >> 2], csum);
    }
    if (s1 >= cnt) break;
    __syncthreads();
  }
  __syncthreads();
  stamp();
  warp_merge_extremes(mx, cx, mn, cn);
  if (lane == 0) {
    s_ev[0][w] = mx;
    s_ec[0][w] = cx;
    s_ev[1][w] = mn;
    s_ec[1][w] = cn;
  }
  __syncthreads();
  if (w == 0) {
    mx = s_ev[0][lane];
    cx = s_ec[0][lane];
    mn = s_ev[1][lane];
    cn = s_ec[1][lane];
    warp_merge_extremes(mx, cx, mn, cn);
    if (lane == 0) {
      S->bmax[blockIdx.x] = mx;
      S->bcmax[blockIdx.x] = cx;
      S->bmin[blockIdx.x] = mn;
      S->bcmin[blockIdx.x] = cn;
    }
  }
  stamp();
  grid_sync(&S->bar_count, bar_target += nb);
  stamp();
  // ---- after A: warp 31 merges the chunks' extremes; warp 30 stages the coarse histogram in shared memory
  // (every block reads each global line once: 148 blocks x 13 queries reading the same lines from L2
  // was a hot spot costing ~10 us); then warp q < m finds query q's 16-bit bucket
  uint32_t qd = 0, qa = 0, qc = 0;  // warp q: digit, keys above its bucket, bucket size
  uint32_t* sh_c = hw;              // [256] coarse bins
  uint32_t* sh_f = hw + 256;        // [m][256] fine bins of each query's coarse digit
  if (w == 31) {
    uint64_t gx = 0, gn = ~0ull;
    uint32_t gcx = 0, gcn = 0;
    for (uint32_t b = lane; b < nb; b += 32) {
      merge_max(gx, gcx, __ldcg(&S->bmax[b]), __ldcg(&S->bcmax[b]));
      merge_min(gn, gcn, __ldcg(&S->bmin[b]), __ldcg(&S->bcmin[b]));
    }
    warp_merge_extremes(gx, gcx, gn, gcn);
    if (lane == 0) {
      s_ev[0][0] = gx;
      s_ec[0][0] = gcx;
      s_ev[1][0] = gn;
      s_ec[1][0] = gcn;
    }
  } else if (w == 30) {
    const uint4* src = reinterpret_cast<const uint4*>(S->HA_c);
    reinterpret_cast<uint4*>(sh_c)[lane] = __ldcg(src + lane);
    reinterpret_cast<uint4*>(sh_c)[lane + 32] = __ldcg(src + lane + 32);
  }
  __syncthreads();
  if (w < m) {
    const uint32_t k = (uint32_t)Q.k[w];
    uint32_t dc, ac, df, af;
    find_digit<8, true>(sh_c, k, lane, dc, ac);
    uint32_t* f = sh_f + 256u * w;
    const uint4* src = reinterpret_cast<const uint4*>(S->HA_f + 256u * dc);
    reinterpret_cast<uint4*>(f)[lane] = __ldcg(src + lane);
    reinterpret_cast<uint4*>(f)[lane + 32] = __ldcg(src + lane + 32);
    __syncwarp();
    find_digit<8, true>(f, k - ac, lane, df, af);
    qd = 256u * dc + df;
    qa = ac + af;
    qc = f[df];
  }
  __syncthreads();
  if (w < m && lane == 0) {  // classify: the rank falls on the global maximum / minimum key, or a bucket
    const int q = w;
    const uint32_t k = (uint32_t)Q.k[q], cmx = s_ec[0][0], cmn = s_ec[1][0];
    if (k <= cmx || k > (uint32_t)n - cmn) {
      s_mode[q] = kModeDone;
      s_T[q] = k <= cmx ? s_ev[0][0] : s_ev[1][0];
      s_above[q] = k <= cmx ? 0u : (uint32_t)n - cmn;
    } else {
      s_pre[q] = qd;
      s_nbits[q] = 16;
      s_r[q] = k - qa;
      s_above[q] = qa;
      s_mode[q] = qc <= kCandCap ? kModeCand : kModeHist;
    }
  }
  __syncthreads();
  stamp();
  // ---- passes H: 12 more bits of every bucket still larger than kCandCap
  for (int hp = 0; hp < kSelHPasses; ++hp) {
    if (w == 0) build_slots(kModeHist, m, s_mode, s_pre, s_nbits, s_slo, s_shi, s_q2slot, &s_nslot, lane);
    __syncthreads();
    const int ns = s_nslot;
    if (ns == 0) break;  // uniform over the grid: every block derived the same state
    int nbits = 0;
    for (int q = 0; q < m; ++q)
      if (s_mode[q] == kModeHist) nbits = s_nbits[q];  // every HIST query holds the same number of bits
    const int shift = 52 - nbits;  // digit = bits [shift, shift + 12)
    const uint64_t rlo = s_slo[0], rhi = s_shi[ns - 1];
    // 16-bit buckets (the first H pass): slot of a key = rank of its 16-bit prefix among the slots' prefixes,
    // from a 65,536-bit map and per-word bases (no search); deeper prefixes use find_range
    const bool map16 = nbits == 16;
    uint8_t* mbase = reinterpret_cast<uint8_t*>(smap + 2048);
    if (map16) {
      for (uint32_t i = threadIdx.x; i < 2048u; i += blockDim.x) {
        uint32_t bits = 0, below = 0;
        for (int j = 0; j < ns; ++j) {
          const uint32_t d = (uint32_t)(s_slo[j] >> 48);
          bits |= (d >> 5) == i ? 1u << (d & 31u) : 0u;
          below += (d >> 5) < i ? 1u : 0u;
        }
        smap[i] = bits;
        mbase[i] = (uint8_t)below;
      }
    }
    for (uint32_t s0 = 0;; s0 += kSelSub) {
      const uint32_t s1 = min(cnt, s0 + kSelSub);
      zero_words(hw, (uint32_t)ns * 2048u);
      __syncthreads();
      for (uint32_t base = s0; base < s1; base += blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const uint64_t key = i < s1 ? key_at(i) : 0;
        int sl = -1;
        if (i < s1 && key >= rlo && key <= rhi) {
          if (map16) {
            const uint32_t d = (uint32_t)(key >> 48), bits = smap[d >> 5], b = 1u << (d & 31u);
            if (bits & b) sl = (int)mbase[d >> 5] + __popc(bits & (b - 1u));
          } else {
            sl = find_range(key, s_slo, s_shi, ns);
          }
        }
        hist_add(hw, sl >= 0, ((uint32_t)sl << 12) | ((uint32_t)(key >> shift) & 0xfffu), lane);
      }
      __syncthreads();
      stamp();
      if (threadIdx.x < (unsigned)ns * 64u) {  // thread t: slot t / 64, coarse bin t % 64 = words 32t .. 32t+31
        const uint32_t csum = flush_range(hw, threadIdx.x, &S->HB_f[hp][0][0] + 64u * threadIdx.x, lane);
        if (csum) atomicAdd(&S->HB_c[hp][threadIdx.x >> 6][threadIdx.x & 63u], csum);
      }
      if (s1 >= cnt) break;
      __syncthreads();
    }
    stamp();
    grid_sync(&S->bar_count, bar_target += nb);
    stamp();
    // stage every slot's 64 coarse bins in shared memory (one read per line per block), then warp q
    // finds its digit: coarse from shared memory, its 64 fine bins staged per warp
    {
      const uint32_t* src = &S->HB_c[hp][0][0];
      for (uint32_t i = threadIdx.x; i < (uint32_t)ns * 64u; i += blockDim.x) hw[i] = __ldcg(src + i);
    }
    __syncthreads();
    if (w < m && s_mode[w] == kModeHist) {
      const int q = w, sl = s_q2slot[q];
      uint32_t dc, ac, df, af;
      const uint32_t r = s_r[q];
      find_digit<2, true>(hw + 64u * sl, r, lane, dc, ac);
      uint32_t* f = hw + 1024u + 64u * w;
      const uint32_t* fsrc = S->HB_f[hp][sl] + 64u * dc;
      f[lane] = __ldcg(fsrc + lane);
      f[lane + 32] = __ldcg(fsrc + lane + 32);
      __syncwarp();
      find_digit<2, true>(f, r - ac, lane, df, af);
      const uint32_t d = 64u * dc + df;
      if (lane == 0) {
        const uint32_t c = f[df];
        const uint64_t pre = (s_pre[q] << 12) | d;
        s_pre[q] = pre;
        s_nbits[q] = nbits + 12;
        s_r[q] = r - ac - af;
        s_above[q] += ac + af;
        if (nbits + 12 == 64) {
          s_mode[q] = kModeDone;
          s_T[q] = pre;
        } else {
          s_mode[q] = c <= kCandCap ? kModeCand : kModeHist;
        }
      }
    }
    __syncthreads();
    stamp();
  }
  stamp();
  // ---- pass C: compact the candidate buckets; per query, sum the values above its bucket (or above T)
  if (w == 0) build_slots(kModeCand, m, s_mode, s_pre, s_nbits, s_slo, s_shi, s_q2slot, &s_nslot, lane);
  if (threadIdx.x >= 32 && threadIdx.x < 32u + (unsigned)m) {  // per query: the largest key it does not sum
    const int q = threadIdx.x - 32;
    const int rb = 64 - s_nbits[q];
    s_up[q] = s_mode[q] == kModeDone ? s_T[q] : ((s_pre[q] << rb) | ((1ull << rb) - 1ull));
  }
  __syncthreads();
  const int nc = s_nslot;
  if (threadIdx.x < (unsigned)nc) {  // every candidate bucket holds >= 16 bits: its top 16 bits are one prefix
    const uint32_t d = (uint32_t)(s_slo[threadIdx.x] >> 48);
    atomicOr(&cmap[d >> 5], 1u << (d & 31u));
  }
  __syncthreads();
  if (nc > 0) {  // block-local lists in shared memory, then copied to this block's region (no global atomics)
    uint64_t* lc = reinterpret_cast<uint64_t*>(hw);  // [nc][kCandCap]
    __shared__ uint32_t s_ln[kMaxQ];
    if (threadIdx.x < (unsigned)nc) s_ln[threadIdx.x] = 0u;
    __syncthreads();
    const uint64_t rlo = s_slo[0], rhi = s_shi[nc - 1];
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint64_t key = key_at(i);
      const uint32_t d = (uint32_t)(key >> 48);
      if (key >= rlo && key <= rhi && ((cmap[d >> 5] >> (d & 31u)) & 1u)) {  // most keys stop at the map
        const int sl = find_range(key, s_slo, s_shi, nc);
        if (sl >= 0) lc[sl * kCandCap + atomicAdd(&s_ln[sl], 1u)] = key;
      }
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)nc) S->cand_bn[threadIdx.x][blockIdx.x] = s_ln[threadIdx.x];
    for (uint32_t e = threadIdx.x; e < (uint32_t)nc * kCandCap; e += blockDim.x) {
      const uint32_t sl = e / kCandCap, i = e % kCandCap;
      if (i < s_ln[sl]) S->cand_b[blockIdx.x][sl][i] = lc[e];
    }
  }
  stamp();
  // fp64 sums of the values above s_up: every key adds its value to ONE interval between consecutive
  // thresholds (ascending: query s_ord[i] has the i-th smallest), in a per-thread column of shared memory;
  // the intervals are reduced in a fixed order and each query takes the suffix sum of the intervals above
  // its threshold -- one fp64 add per key instead of one per (key, query); counts follow from the ranks.
  __shared__ uint64_t s_uo[kMaxQ];
  __shared__ int s_ord[kMaxQ];
  if (w == 0 && lane < m) {
    const uint64_t u = s_up[lane];
    int rank = 0;
    for (int j = 0; j < m; ++j) rank += (s_up[j] < u || (s_up[j] == u && j < lane)) ? 1 : 0;
    s_uo[rank] = u;
    s_ord[rank] = lane;
  }
  __syncthreads();  // (the compaction above is done with hw)
  double* bk = reinterpret_cast<double*>(hw);  // [kMaxQ][kSelThreads]: interval i of this thread
  for (int i = 0; i < m; ++i) bk[i * kSelThreads + threadIdx.x] = 0.0;
  __syncthreads();
  {
    const uint64_t u0 = s_uo[0];
    for (uint32_t e = threadIdx.x; e < cnt; e += blockDim.x) {
      const uint64_t key = key_at(e);
      if (key > u0) {  // the largest i with s_uo[i] < key
        int i = 0;
#pragma unroll
        for (int step = 8; step > 0; step >>= 1)
          if (i + step < m && s_uo[i + step] < key) i += step;
        bk[i * kSelThreads + threadIdx.x] += from_key(key);
      }
    }
  }
  stamp();
  __syncthreads();
  __shared__ double s_bsum[kMaxQ];
  if (w < m) {  // warp i reduces interval i: lane l sums threads 32l .. 32l+31 in order, then a fixed tree
    const double* col = bk + w * kSelThreads + 32 * lane;
    double a = 0.0;
#pragma unroll 8
    for (int t = 0; t < 32; ++t) a += col[(t + lane) & 31];  // rotated start: no bank conflicts; fixed per lane
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
    if (lane == 0) s_bsum[w] = a;
  }
  __syncthreads();
  if (w == 0) {
    if (lane == 0) {  // query s_ord[i] sums the intervals i .. m-1, added from the top interval down
      double acc = 0.0;
      for (int i = m - 1; i >= 0; --i) {
        acc += s_bsum[i];
        S->psum[blockIdx.x][s_ord[i]] = acc;
      }
    }
  }
  stamp();
  grid_sync(&S->bar_count, bar_target += nb);
  stamp();
  if (threadIdx.x == 0 && atomicAdd(&S->bar_exit, 1u) == nb - 1) {  // every block is past the last barrier
    S->bar_count = 0u;
    S->bar_exit = 0u;
  }
  {  // pass A's histogram has had its last reader: zero it for the next launch (this block's share)
    const uint32_t words = 256u + 65536u;
    uint32_t* z = S->HA_c;
    const uint32_t per = (words + nb - 1) / nb, b0 = per * blockIdx.x, b1 = min(words, b0 + per);
    for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) z[i] = 0u;
  }
  if (blockIdx.x != 0) return;
  // ---- F (block 0): sort each candidate list descending (position = keys above + equal keys listed
  // before: distinct positions, and equal keys are equal values), then per query T and TVaR
  uint64_t* craw = reinterpret_cast<uint64_t*>(hw);  // [nc][kCandCap] as compacted (any order)
  uint64_t* cs = craw + kMaxQ * kCandCap;              // [nc][kCandCap] sorted descending
  __shared__ uint32_t s_cn[kMaxQ];
  uint32_t* boff = reinterpret_cast<uint32_t*>(cs + kMaxQ * kCandCap);  // [nc][nb] offsets of the blocks' lists
  uint32_t* bcnt = boff + kMaxQ * kSelMaxBlocks;                          // [nc][nb] their lengths
  if (w < nc) {  // warp s: the blocks' counts of slot s, exclusive prefix in block order
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < nb; b0 += 32) {
      const uint32_t b = b0 + lane;
      const uint32_t c = b < nb ? __ldcg(&S->cand_bn[w][b]) : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(FULL, incl, off);
        if (lane >= off) incl += o;
      }
      if (b < nb) {
        boff[w * nb + b] = carry + incl - c;
        bcnt[w * nb + b] = c;
      }
      carry += __shfl_sync(FULL, incl, 31);
    }
    if (lane == 0) s_cn[w] = carry;
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < (uint32_t)nc * nb; e += blockDim.x) {  // (slot, block): copy its list
    const uint32_t sl = e / nb, b = e % nb, o = boff[e], c = bcnt[e];
    for (uint32_t i = 0; i < c; ++i) craw[sl * kCandCap + o + i] = __ldcg(&S->cand_b[b][sl][i]);
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < (uint32_t)nc * kCandCap; e += blockDim.x) {
    const uint32_t sl = e / kCandCap, i = e % kCandCap, nn = s_cn[sl];
    if (i >= nn) continue;
    const uint64_t* c = craw + sl * kCandCap;
    const uint64_t ki = c[i];
    uint32_t pos = 0;
    for (uint32_t j = 0; j < nn; ++j) pos += (c[j] > ki) || (c[j] == ki && j < i);
    cs[sl * kCandCap + pos] = ki;
  }
  __syncthreads();
  if (w < m) {
    const int q = w;
    double a = 0.0;
    for (unsigned i = lane; i < nb; i += 32) a += __ldcg(&S->psum[i][q]);
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(FULL, a, off);
    if (lane == 0) {
      uint64_t T, b = s_above[q];
      if (s_mode[q] == kModeDone) {
        T = s_T[q];
      } else {  // the candidates of the bucket, descending: T is the rank's key; add those above T in order
        const uint64_t* c = cs + s_q2slot[q] * kCandCap;
        const uint32_t r = s_r[q];
        T = c[r - 1];
        for (uint32_t j = 0; j < r - 1 && c[j] > T; ++j) {
          a += from_key(c[j]);
          b += 1;
        }
      }
      const double Tv = from_key(T);
      const uint64_t k = Q.k[q];
      if (pml_out) pml_out[q] = Tv;  // PML: the k-th largest value
      if (tvar_out) tvar_out[q] = __ddiv_rn(__dadd_rn(a, __dmul_rn((double)(k - b), Tv)), (double)k);  // TVaR
    }
  }
  __syncthreads();
  stamp();
}

// Per-device launch facts of metrics_select, queried once (host-side cache; no per-call queries).
struct FusedInfo {
  int ready = 0, coop = 0, sms = 148, occ = 0;
};
static FusedInfo g_fused[64];
constexpr size_t kSelDynSmem =
    (size_t)kSelCache * sizeof(uint64_t) + (size_t)(kSelHistWords + kSelMapWords) * sizeof(uint32_t);

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
    int occ_u = 0;
    cudaFuncSetAttribute((const void*)metrics_select<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelDynSmem);
    cudaFuncSetAttribute((const void*)metrics_select<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSelDynSmem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&f.occ, (const void*)metrics_select<true>, kSelThreads, kSelDynSmem) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_u, (const void*)metrics_select<false>, kSelThreads, kSelDynSmem) !=
            cudaSuccess) {
      cudaGetLastError();
      f.occ = 0;
    }
    f.occ = std::min(f.occ, occ_u);
    f.ready = 1;
  }
  return f;
}

// Launch metrics_select cooperatively for one batch of <= kMaxQ queries, results to DEVICE pml/tvar
// (either may be null); asynchronous.  `zeroed`: the scratch is known to hold zeros where the kernel
// expects them (a plan's scratch after its first use); otherwise it is cleared first.  Returns false if
// the device refuses a cooperative launch of the needed size (callers fall back to the pass kernels).
static bool metrics_fused_batch(const double* ylt, uint64_t n, int mq, const uint64_t* ks, char* scratch,
                                size_t scratch_bytes, double* pml_dev, double* tvar_dev, cudaStream_t s,
                                cudaError_t* err, bool zeroed = false) {
  *err = cudaSuccess;
  const FusedInfo& f = fused_info();
  if (!f.coop || f.occ < 1 || n > 0xffffffffull) return false;
  uint64_t grid = (uint64_t)f.sms * f.occ;
  const uint64_t need = (n + kSelThreads - 1) / kSelThreads;
  if (grid > need) grid = need;
  if (grid > (uint64_t)kSelMaxBlocks) grid = kSelMaxBlocks;
  if (sizeof(SelScratch) > scratch_bytes) return false;
  SelScratch* st = (SelScratch*)scratch;
  SelQueries Q;
  memset(&Q, 0, sizeof Q);
  for (int q = 0; q < mq; ++q) Q.k[q] = ks[q];
  if (!zeroed && (*err = cudaMemsetAsync(st, 0, kSelZeroBytes, s)) != cudaSuccess) return true;
  int m_ = mq;
  int trace = getenv("ARA_METRICS_TRACE") ? 1 : 0;  // development aid: per-block phase timestamps
  void* args[] = {(void*)&ylt, (void*)&n, (void*)&m_, (void*)&st, (void*)&Q, (void*)&pml_dev, (void*)&tvar_dev, &trace};
  const bool cached = (n + grid - 1) / grid <= (uint64_t)kSelCache;  // every block's chunk fits its key cache
  *err = cudaLaunchCooperativeKernel(cached ? (const void*)metrics_select<true> : (const void*)metrics_select<false>,
                                     dim3((unsigned)grid), dim3(kSelThreads), args, kSelDynSmem, s);
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

// Scratch: [2*kMaxQ doubles of batch results][the pass kernels' state + block partials, or metrics_select's
// SelScratch, whichever is larger].
static size_t pass_scratch_bytes(uint64_t n, uint64_t* blocks_out) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + kSelBlock - 1) / kSelBlock;
  if (blocks > (uint64_t)sms * 8) blocks = (uint64_t)sms * 8;
  *blocks_out = blocks;
  return sizeof(SelState) + blocks * kMaxQ * (sizeof(double) + sizeof(unsigned long long));
}
static size_t scratch_bytes(uint64_t n, uint64_t* blocks_out) {
  return 2 * kMaxQ * sizeof(double) + std::max(pass_scratch_bytes(n, blocks_out), sizeof(SelScratch));
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
  double* psum = (double*)(rest + sizeof(SelState));
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
    if (e == cudaSuccess && use_fused && getenv("ARA_METRICS_TRACE")) {  // development aid: phase times
      std::vector<unsigned long long> tr((size_t)kSelMaxBlocks * 24);
      const int nbk = (int)std::min<uint64_t>((n + kSelThreads - 1) / kSelThreads, (uint64_t)fused_info().sms);
      if (cudaMemcpyAsync(tr.data(), ((SelScratch*)rest)->trace, tr.size() * 8, cudaMemcpyDeviceToHost, s) == cudaSuccess &&
          cudaStreamSynchronize(s) == cudaSuccess) {
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < nbk; ++b) t0 = std::min(t0, tr[(size_t)b * 24]);
        fprintf(stderr, "metrics_select stamps (us from first block start: min/max over %d blocks):", nbk);
        for (int i = 0; i < 24; ++i) {
          unsigned long long a = ~0ull, z = 0;
          for (int b = 0; b < nbk; ++b) {
            const unsigned long long t = tr[(size_t)b * 24 + i];
            a = std::min(a, t);
            z = std::max(z, t);
          }
          if (a < t0 || z - t0 > 100000000ull) break;
          fprintf(stderr, " [%d] %.1f/%.1f", i, (a - t0) * 1e-3, (z - t0) * 1e-3);
        }
        fprintf(stderr, "\n");
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
// can be captured into a CUDA graph (ara_plan_create).  `zeroed`: the scratch was zeroed when allocated
// and only ever used by these launches (they leave it as they found it), so no clearing memset is needed.
ara_status metrics_device_into(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                               double* tvar_dev, char* scratch, size_t bytes, cudaStream_t s, bool zeroed) {
  if (!ylt || (!pml_dev && !tvar_dev)) return set_error(ARA_E_ARG, "NULL argument");
  std::vector<uint64_t> ks;
  ara_status rc = ranks_for(n, rps, m, ks);
  if (rc) return rc;
  for (uint32_t q0 = 0; q0 < m && rc == ARA_OK; q0 += kMaxQ) {
    const int mq = (int)std::min<uint32_t>(kMaxQ, m - q0);
    cudaError_t e = cudaSuccess;
    if (!metrics_fused_batch(ylt, n, mq, &ks[q0], scratch, bytes, pml_dev ? pml_dev + q0 : nullptr,
                             tvar_dev ? tvar_dev + q0 : nullptr, s, &e, zeroed))
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
  ara_status rc = metrics_device_into(ylt, n, rps, m, pml_dev, tvar_dev, scratch, bytes, s, false);
  cudaFreeAsync(scratch, s);
  return rc;
}

}  // namespace ara

extern "C" {

ara_status ara_pml_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_out,
                        double* tvar_out, void* stream) {
  ara::NvtxRange nvtx("ara_pml_tvar");
  if (!pml_out && !tvar_out) return ara::set_error(ARA_E_ARG, "no output");
  return ara::metrics(ylt, n, rps, m, pml_out, tvar_out, (cudaStream_t)stream);
}

ara_status ara_pml_tvar_device(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                               double* tvar_dev, void* stream) {
  ara::NvtxRange nvtx("ara_pml_tvar_device");
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

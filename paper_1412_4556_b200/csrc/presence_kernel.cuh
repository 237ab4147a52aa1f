// presence_kernel.cuh -- the default ARA hot path on sm_100a: the same direct-access interleaved table as
// ara_layer_kernel, plus a per-layer PRESENCE bitmap (bit e set iff row e of the table holds a non-zero
// loss).  Most event rows are all zero (990,000 of 1,000,000 entries of an ELT; 92% of
// the rows of the paper-shaped layer), and an all-zero row contributes exactly +0 to every sum (reading
// c9), so only rows whose bit is set are gathered.  The bitmap lives in SHARED memory (one copy per SM,
// folded modulo its capacity when C+1 exceeds it -- folding only adds false positives, i.e. gathers of
// rows that turn out to be zero, never misses), so the per-occurrence test costs one LDS instead of a
// 64-B gather.  The kernel is then bound by streaming the YET ids from HBM.
//
//   * one warp per trial (persistent grid); the warp streams the trial's ids in 128-id windows, each lane
//     one 16-B vector (L1::no_allocate, L2 evict_first), with the next window prefetched;
//   * per window slot: validity check, bitmap test, __ballot_sync; hits (event ids) are appended to a
//     per-warp ring queue in shared memory (64 entries);
//   * whenever 32 hits are queued the warp drains them with all lanes active: each queued event's row is
//     gathered by G lanes (V-float vectors, 256-bit loads), FT1 is applied in fp64 to its non-zero
//     entries and summed, the G partials are combined, FT2 is applied and the leader lane accumulates
//     the occurrence-net loss (steps 1-4);
//   * at the end of the trial the remaining hits are drained, the lanes' sums are reduced with shuffles
//     and FT3 is applied to S_n.
#pragma once
#include "ara_kernel.cuh"

namespace ara {

constexpr int kQueue = 64;  // per-warp ring of pending hits (< 32 carried + <= 32 new per slot)

// Drain n (<= 32) queued events starting at ring position `head`: all 32 lanes participate.
template <int V, int NV, int G>
__device__ __forceinline__ void drain(const LayerParams& p, const uint32_t* __restrict__ q, unsigned head, int n,
                                      int lane, const double* s_r1, const double* s_l1, uint64_t pol_tab,
                                      double& S) {
  constexpr int RG = 32 / G;
  constexpr int NVL = (NV + G - 1) / G;
  constexpr int JP = V * NV;
  constexpr unsigned FULL = 0xffffffffu;
  const int g = lane % G;
#pragma unroll
  for (int r = 0; r < G; ++r) {
    const int slot = r * RG + lane / G;
    if (r * RG >= n) break;  // warp-uniform
    const uint32_t id = slot < n ? q[(head + slot) & (kQueue - 1)] : 0u;
    const float* row = p.table + (uint64_t)id * JP;
    float x[NVL][V];
#pragma unroll
    for (int i = 0; i < NVL; ++i) {
      const int s = g + i * G;
      if (id != 0 && (NV % G == 0 || s < NV)) {
        ld_row<V>(row + s * V, pol_tab, x[i]);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) x[i][c] = 0.0f;
      }
    }
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < NVL; ++i)
#pragma unroll
      for (int c = 0; c < V; ++c) {
        if (__float_as_uint(x[i][c]) != 0u) {
          const int j = (g + i * G) * V + c;
          sum += clamp_terms((double)x[i][c], s_r1[j], s_l1[j]);
        }
      }
    if constexpr (G > 1) {
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(FULL, sum, off);
    }
    if (sum != 0.0 && g == 0) S += clamp_terms(sum, p.r2, p.l2);
  }
}

// V/NV: row format (as ara_layer_kernel); G: lanes per row in a drain; NW: warps per block.
template <int V, int NV, int G, int NW>
__global__ void __launch_bounds__(NW * 32, 1) ara_presence_kernel(const __grid_constant__ LayerParams p) {
  constexpr int JP = V * NV;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ uint32_t smem[];
  __shared__ double s_r1[JP], s_l1[JP];
  uint32_t* bits = smem;                       // [fold_words]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t* q = smem + p.fold_words + warp * kQueue;

  for (int j = threadIdx.x; j < JP; j += blockDim.x) {
    s_r1[j] = p.r1[j];
    s_l1[j] = p.l1[j];
  }
  // Stage the presence bitmap (folded modulo fold_words if it does not fit).
  const uint32_t fw = p.fold_words;
  if (p.present_words <= fw) {
    for (uint32_t w = threadIdx.x; w < p.present_words; w += blockDim.x) bits[w] = __ldg(p.present + w);
  } else {
    for (uint32_t w = threadIdx.x; w < fw; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    for (uint32_t w = threadIdx.x; w < p.present_words; w += blockDim.x) {
      const uint32_t v = __ldg(p.present + w);
      if (v) atomicOr(&bits[w % fw], v);
    }
  }
  __syncthreads();

  const uint64_t pol_tab = make_policy(true, p.l2_hints);
  const uint64_t pol_yet = make_policy(false, p.l2_hints);
  const uint64_t warp0 = (uint64_t)blockIdx.x * NW + warp;
  const uint64_t nwarps = (uint64_t)gridDim.x * NW;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(p.ids) & 15u) == 0);
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t C = p.C;

  for (uint64_t t = warp0; t < p.num_trials; t += nwarps) {
    uint64_t b, e;
    unsigned bad = 0;
    if (p.offsets) {
      b = p.offsets[t];
      e = p.offsets[t + 1];
      if (e < b || e > p.num_events) {
        bad |= 2u;
        e = b;
      }
    } else {
      b = t * p.K;
      e = b + p.K;
    }
    double S = 0.0;
    unsigned head = 0;
    int count = 0;
    // windows of 128 ids aligned to 16 B; lane loads ids [w + 4 lane, w + 4 lane + 4)
    uint64_t w = b & ~(uint64_t)3;
    auto load4 = [&](uint64_t at) -> uint4 {
      const uint64_t qq = at + 4u * lane;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (qq < e) {
        if (vec_ok && qq + 4 <= p.num_events) {
          v = ld_ids4(p.ids + qq, pol_yet);
        } else {
          v.x = ld_id(p.ids + qq, pol_yet);
          if (qq + 1 < e) v.y = ld_id(p.ids + qq + 1, pol_yet);
          if (qq + 2 < e) v.z = ld_id(p.ids + qq + 2, pol_yet);
          if (qq + 3 < e) v.w = ld_id(p.ids + qq + 3, pol_yet);
        }
      }
      return v;
    };
    uint4 cur = w < e ? load4(w) : make_uint4(0u, 0u, 0u, 0u);
    for (; w < e; w += 128) {
      const uint4 nxt = (w + 128 < e) ? load4(w + 128) : make_uint4(0u, 0u, 0u, 0u);
      const uint32_t idv[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t pos = w + 4u * lane + u;
        uint32_t id = (pos >= b && pos < e) ? idv[u] : 0u;
        bool hit = false;
        if (pos >= b && pos < e) {
          if (id - 1u >= C) {  // outside [1, C]: record, treat as absent
            bad |= 1u;
            id = 0u;
          } else {
            uint32_t wd = id >> 5;
            if (wd >= fw) wd %= fw;
            hit = (bits[wd] >> (id & 31u)) & 1u;
          }
        }
        const unsigned m = __ballot_sync(FULL, hit);
        if (hit) q[(head + count + __popc(m & lt)) & (kQueue - 1)] = id;
        count += __popc(m);
        if (count >= 32) {
          __syncwarp();
          drain<V, NV, G>(p, q, head, 32, lane, s_r1, s_l1, pol_tab, S);
          __syncwarp();
          head = (head + 32) & (kQueue - 1);
          count -= 32;
        }
      }
      cur = nxt;
    }
    if (count > 0) {
      __syncwarp();
      drain<V, NV, G>(p, q, head, count, lane, s_r1, s_l1, pol_tab, S);
      __syncwarp();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(FULL, S, off);
    bad = __reduce_or_sync(FULL, bad);
    if (lane == 0) {
      p.ylt[t] = clamp_terms(S, p.r3, p.l3);
      if (bad) atomicOr(p.err, bad);
    }
  }
}

}  // namespace ara

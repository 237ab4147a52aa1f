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

constexpr int kQueue = 128;  // per-warp ring of pending hits (< 32 carried + <= 64 new per slot pair)

// Gathers for a batch of up to 32 queued events, split into an ISSUE step (loads into registers)
// and a CONSUME step (FT1 / sum / FT2 / accumulate), so a batch's L2 latency overlaps the scan of the
// following YET windows.  Round r covers queue slots r*32/G .. (r+1)*32/G - 1; slot r*RG + lane/G is
// fetched by the G lanes lane/G*G .. +G-1, lane g holding vectors g, g+G, ... of the row.
template <int V, int NV, int G>
struct RowBatch {
  static constexpr int RG = 32 / G;
  static constexpr int NVL = (NV + G - 1) / G;
  // Narrow rows: all G rounds of a batch stay in registers between issue and consume (async).
  // Wide rows: one round at a time (issue and consume back to back) to stay inside 64 registers.
  static constexpr bool kAsync = G == 1 && NVL * V <= 16;
  static constexpr int R = kAsync ? G : 1;
  float x[R][NVL][V];

  __device__ __forceinline__ void issue_round(int r, const LayerParams& p, const uint32_t* __restrict__ q,
                                              unsigned head, int n, int lane, uint64_t pol_tab) {
    const int g = lane % G;
    const int slot = r * RG + lane / G;
    const uint32_t id = slot < n ? q[(head + slot) & (kQueue - 1)] : 0u;
    const float* row = p.table + (uint64_t)id * (V * NV);
    float(&xr)[NVL][V] = x[kAsync ? r : 0];
#pragma unroll
    for (int i = 0; i < NVL; ++i) {
      const int s = g + i * G;
      if (id != 0 && (NV % G == 0 || s < NV)) {
        ld_row<V>(row + s * V, pol_tab, xr[i]);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) xr[i][c] = 0.0f;
      }
    }
  }

  __device__ __forceinline__ void consume_round(int r, const LayerParams& p, int lane, const double* s_r1,
                                                const double* s_l1, double& S) const {
    const int g = lane % G;
    const float(&xr)[NVL][V] = x[kAsync ? r : 0];
    // Steps 1-2: FT1 on each of the row's losses, summed across the layer's ELTs.  Branch-free: an
    // absent loss (0) gives clamp(0; R >= 0, L) = +0 exactly, so the dense sum equals the sparse one.
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < NVL; ++i)
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int j = (g + i * G) * V + c;
        sum += clamp_terms((double)xr[i][c], s_r1[j], s_l1[j]);
      }
    if constexpr (G > 1) {
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    }
    if (g == 0) S += clamp_terms(sum, p.r2, p.l2);  // step 3 (FT2); step 4 accumulation (exact +0 if sum 0)
  }

  // Async: issue all rounds now, consume later.  Sync: issue+consume round by round.
  __device__ __forceinline__ void issue(const LayerParams& p, const uint32_t* __restrict__ q, unsigned head, int n,
                                        int lane, uint64_t pol_tab, const double* s_r1, const double* s_l1,
                                        double& S) {
#pragma unroll
    for (int r = 0; r < G; ++r) {
      if (r * RG >= n) break;  // warp-uniform
      issue_round(r, p, q, head, n, lane, pol_tab);
      if constexpr (!kAsync) consume_round(r, p, lane, s_r1, s_l1, S);
    }
    if constexpr (kAsync) {
      for (int r = (n + RG - 1) / RG; r < G; ++r)  // rounds past n hold nothing
#pragma unroll
        for (int i = 0; i < NVL; ++i)
#pragma unroll
          for (int c = 0; c < V; ++c) x[r][i][c] = 0.0f;
    }
  }

  __device__ __forceinline__ void consume(const LayerParams& p, int lane, const double* s_r1, const double* s_l1,
                                          double& S) const {
    if constexpr (kAsync) {
#pragma unroll
      for (int r = 0; r < G; ++r) consume_round(r, p, lane, s_r1, s_l1, S);
    }
  }
};

// V/NV: row format (as ara_layer_kernel); G: lanes per row in a drain; NW: warps per block.
template <int V, int NV, int G, int NW>
__global__ void __launch_bounds__(NW * 32, 1) ara_presence_kernel(const __grid_constant__ LayerParams p) {
  constexpr int JP = V * NV;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ uint32_t smem[];
  // FT1 terms, padded to the G*NVL*V columns a row group covers (padding: R = 0, L = +inf, so the
  // branch-free FT1 of a padding column -- always loss 0 -- is exactly +0).
  constexpr int JPS = G * ((NV + G - 1) / G) * V;
  __shared__ double s_r1[JPS], s_l1[JPS];
  uint32_t* bits = smem;                       // [fold_words]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t* q = smem + p.fold_words + warp * kQueue;

  for (int j = threadIdx.x; j < JPS; j += blockDim.x) {
    s_r1[j] = j < JP ? p.r1[j] : 0.0;
    s_l1[j] = j < JP ? p.l1[j] : __longlong_as_double(0x7ff0000000000000ll);
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
  const bool fold_sub = p.present_words <= 2u * fw;  // one conditional subtraction folds every word
  const uint64_t fmagic = p.fold_magic;

  // word index of event id in the (folded) shared bitmap
  auto word_of = [&](uint32_t id) -> uint32_t {
    uint32_t wd = id >> 5;
    if (fold_sub) {
      wd = wd >= fw ? wd - fw : wd;
    } else {
      wd = (uint32_t)__umul64hi(fmagic * (uint64_t)wd, (uint64_t)fw);  // wd % fw
    }
    return wd;
  };

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
    const uint32_t len = (uint32_t)(e - b);
    const uint32_t* base = p.ids + b;
    // Windows of 128 ids starting at the trial's first occurrence, so the order in which hits are
    // queued (hence the fp64 summation order) depends only on the trial's own ids: the YLT is bitwise
    // identical however the YET is sharded or offset.  Lane l holds ids [rel + 4l, rel + 4l + 4): one
    // 16-B vector when the trial start is 16-B aligned, else scalar loads.
    const bool vec = vec_ok && ((b & 3u) == 0);
    auto load4 = [&](uint32_t rel) -> uint4 {
      const uint32_t qq = rel + 4u * lane;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (qq < len) {
        if (vec && qq + 4 <= len) {
          v = ld_ids4(base + qq, pol_yet);
        } else {
          v.x = ld_id(base + qq, pol_yet);
          if (qq + 1 < len) v.y = ld_id(base + qq + 1, pol_yet);
          if (qq + 2 < len) v.z = ld_id(base + qq + 2, pol_yet);
          if (qq + 3 < len) v.w = ld_id(base + qq + 3, pol_yet);
        }
      }
      return v;
    };
    double S = 0.0;
    unsigned head = 0;
    unsigned count = 0;
    RowBatch<V, NV, G> rows;
    bool pending = false;
    uint4 cur = load4(0);
    uint4 nx1 = load4(128);
    for (uint32_t rel = 0; rel < len; rel += 128) {
      const uint4 nx2 = load4(rel + 256);
      uint32_t id[4] = {cur.x, cur.y, cur.z, cur.w};
      bool hit[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        // positions past the trial end were loaded as 0 and stay 0 (never a hit, never "bad")
        const bool inside = rel + 4u * lane + u < len;
        const bool ok = id[u] - 1u < C;          // 1 <= id <= C
        bad |= (inside && !ok) ? 1u : 0u;        // outside [1, C]: record, treat as absent
        id[u] = ok ? id[u] : 0u;                 // id 0 -> bit 0 of word 0, never set
        const uint32_t word = bits[word_of(id[u])];
        hit[u] = (word >> (id[u] & 31u)) & 1u;
      }
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const uint32_t ia = h ? id[2] : id[0], ib = h ? id[3] : id[1];
        const bool ha = h ? hit[2] : hit[0], hb = h ? hit[3] : hit[1];
        const unsigned m0 = __ballot_sync(FULL, ha);
        const unsigned m1 = __ballot_sync(FULL, hb);
        const unsigned n0 = __popc(m0);
        const unsigned at = head + count;
        if (ha) q[(at + __popc(m0 & lt)) & (kQueue - 1)] = ia;
        if (hb) q[(at + n0 + __popc(m1 & lt)) & (kQueue - 1)] = ib;
        count += n0 + __popc(m1);
        while (count >= 32) {  // warp-uniform; at most 31 + 64 = 95 < kQueue pending
          __syncwarp();
          if (pending) rows.consume(p, lane, s_r1, s_l1, S);
          rows.issue(p, q, head, 32, lane, pol_tab, s_r1, s_l1, S);
          pending = RowBatch<V, NV, G>::kAsync;
          __syncwarp();
          head = (head + 32) & (kQueue - 1);
          count -= 32;
        }
      }
      cur = nx1;
      nx1 = nx2;
    }
    if (count > 0) {  // final partial batch (the pending one is consumed first, in queue order)
      __syncwarp();
      if (pending) rows.consume(p, lane, s_r1, s_l1, S);
      rows.issue(p, q, head, (int)count, lane, pol_tab, s_r1, s_l1, S);
      pending = RowBatch<V, NV, G>::kAsync;
      __syncwarp();
    }
    if (pending) rows.consume(p, lane, s_r1, s_l1, S);
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

// fused_kernel.cuh -- SURVEY.md 8(f) N1: every layer of a fixed-length-trial YET in ONE pass.
//
// Algorithm 1 is layer-outer: each layer re-streams the whole YET.  With the presence
// kernels the YET is ~99% of a pass's DRAM bytes, so config M (8 layers) streams 8 x 4 GB.  This kernel
// streams the YET once for a group of layers:
//
//   * presence test against the UNION bitmap (rows holding a loss in any layer of the group), folded into
//     shared memory like the single-layer kernels (false positives only);
//   * every hit goes into its lane's own queue (lane_kernel.cuh); a gather round cp.asyncs each popped
//     event's 32-B COMBINED record: up to four (global column, loss) entries over the group's layers,
//     in layer order (a global column is layer ell's ELT j at col0[ell] + j);
//   * per hit, Steps 1-3 run per layer: FT1 per entry, the sum over the layer's
//     entries, FT2 of that layer (:113, :127), added to the lane's accumulator for (layer, trial) in
//     shared memory; an event with more than four entries reads its rows from the layer tables;
//   * at the end of a trial every queue is drained and, per layer, the 32 lane accumulators are combined
//     by the fixed xor-tree, FT3 of the layer is applied (:114, :129) and the YLT row is stored.
//
// Summation order: lane l sums, per layer, the occurrence-net losses of the hits at trial positions p
// with (p mod 128) / 4 == l in stream order -- exactly the single-layer lane kernel's order (a hit that
// holds no loss of layer ell adds nothing to it), so each layer's YLT equals that kernel's bit for bit.
#pragma once
#include "lane_kernel.cuh"

namespace ara {

constexpr int kFusedMaxLayers = 16;
constexpr int kFusedMaxCols = 256;                     // global columns of a fused layer group
constexpr uint32_t kFusedRecWords = 8;                 // 32-B record
constexpr uint32_t kFusedDepth = 3;                    // gather rounds in flight (record slots per lane)
constexpr uint32_t kFusedWarpSmem = 32 * kLaneQ * 4 + kFusedDepth * 32 * 32;  // lane queues + record slots

struct FusedParams {
  const uint32_t* ids;
  uint64_t num_trials, num_events;
  uint32_t K, C;
  const uint32_t* present;      // union bitmap folded to present_words (fold_mul), sentinel bit C set
  uint32_t present_words, fold_mul;
  const uint4* rec;             // 2 x uint4 per event: [c0 c1 c2 c3 | n | l0 l1 l2 l3 | id | -]
  uint32_t nl;                  // layers in the group
  uint32_t prefetch;
  double* ylt;                  // layer ell's row at ylt + ell * ld
  uint64_t ld;
  unsigned* err;
  const float* table[kFusedMaxLayers];  // per layer: direct-access table (rows with > 4 entries)
  uint32_t jpad[kFusedMaxLayers], col0[kFusedMaxLayers], J[kFusedMaxLayers];
  double r2[kFusedMaxLayers], l2[kFusedMaxLayers], r3[kFusedMaxLayers], l3[kFusedMaxLayers];
  double r1[kFusedMaxCols], l1[kFusedMaxCols];  // FT1 per global column
  uint8_t layer_of[kFusedMaxCols];              // global column -> layer
};

__host__ __device__ constexpr uint32_t fused_smem_extra(uint32_t nw, uint32_t nl) {
  // FT1 pairs (4 KB) + FT2 pairs (256 B) + column -> layer (256 B) + alignment slack + per-warp queues and
  // record slots + per-warp accumulators (nl layers x 32 lanes x 8 B)
  return 16u + kFusedMaxCols * 16u + kFusedMaxLayers * 16u + kFusedMaxCols + 1024u + nw * kFusedWarpSmem +
         nw * nl * 32u * 8u;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) ara_fused_kernel(const __grid_constant__ FusedParams p) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t fw = p.present_words;
  uint32_t bits_s;  // folded union bitmap (shared address kept in a register)
  asm volatile("mov.u32 %0, %1;" : "=r"(bits_s) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
  const uint32_t t1_w = (fw + 3u) & ~3u;
  double2* s_t1 = reinterpret_cast<double2*>(smem + t1_w);                 // [256] FT1 (R, L) per column
  double2* s_t2 = s_t1 + kFusedMaxCols;                                    // [16] FT2 per layer
  uint8_t* s_lay = reinterpret_cast<uint8_t*>(s_t2 + kFusedMaxLayers);     // [256] column -> layer
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);
  const uint32_t base_s = ((uint32_t)__cvta_generic_to_shared(s_lay + kFusedMaxCols) + 1023u) & ~1023u;
  uint32_t q_l;  // this lane's queue: entry j at q_l + 128 j (queues first, 1 KB each: OR addressing)
  asm volatile("mov.u32 %0, %1;" : "=r"(q_l) : "r"(base_s + warp * (32u * kLaneQ * 4u) + 4u * lane));
  // record slot s of this lane: rec_l + s * 1024 (kFusedDepth slots, rounds in flight)
  const uint32_t rec_l = base_s + NW * (32u * kLaneQ * 4u) + warp * (kFusedDepth * 1024u) + 32u * lane;
  // accumulators after every warp's queue and record slots: acc[ell * 32] is this lane's (layer ell)
  const uint32_t acc_off = base_s - (uint32_t)__cvta_generic_to_shared(smem) + NW * kFusedWarpSmem;  // bytes
  double* acc = reinterpret_cast<double*>(reinterpret_cast<char*>(smem) + acc_off) + warp * (p.nl * 32u) + lane;
  for (uint32_t j = threadIdx.x; j < kFusedMaxCols; j += blockDim.x) {
    s_t1[j] = make_double2(p.r1[j], p.l1[j]);
    s_lay[j] = p.layer_of[j];
  }
  for (uint32_t j = threadIdx.x; j < kFusedMaxLayers; j += blockDim.x) s_t2[j] = make_double2(p.r2[j], p.l2[j]);
  for (uint32_t w = threadIdx.x; w < fw; w += blockDim.x) smem[w] = __ldg(p.present + w);
  for (uint32_t l = 0; l < p.nl; ++l) acc[l * 32u] = 0.0;
  __syncthreads();

  // interleaved trials: warp W takes W, W + NWT, ...
  const uint64_t W = (uint64_t)blockIdx.x * NW + warp, NWT = (uint64_t)gridDim.x * NW;
  const uint64_t N = p.num_trials;
  const uint32_t nt = (uint32_t)(N > W ? (N - 1 - W) / NWT + 1 : 0);
  if (nt == 0) return;
  const uint32_t K = p.K;
  const uint32_t nwin = (K + 127u) >> 7;
  const bool lane_last = 4u * lane < K - 128u * (nwin - 1u);
  const uint32_t last_valid = lane_last ? FULL : 0u;
  const uint32_t C = p.C, fmul = p.fold_mul, nl = p.nl;

  uint32_t tail = 0, head = 0, vmax = 0;
  uint32_t nin = 0;   // rounds in flight (warp-uniform, <= kFusedDepth - 1 after a round is issued)
  uint32_t oldest = 0;  // record slot of the oldest round in flight

  // flush a layer's event sum: FT2 of that layer, added to the lane's (layer, trial) accumulator
  auto flush = [&](uint32_t l, double s) {
    const double2 t = s_t2[l];
    acc[l * 32u] += clamp_fast(s, t.x, t.y);  // step 3 (FT2); step 4 accumulation
  };
  // Consume the oldest round in flight (its cp.async group is complete once at most nin - 1 are pending).
  auto consume = [&]() {
    if (nin == 0u) return;
    if (nin >= 3u) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else if (nin == 2u) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else cp_async_wait_all();
    const uint32_t slot = rec_l + oldest * 1024u;
    const uint4 a = lds_u128(slot), b = lds_u128(slot + 16u);
    const uint32_t n = a.y;
    if (__any_sync(FULL, n > 4u)) {  // rare: more than four entries -- every layer's row read in full
      if (n > 4u) {
        const uint32_t e = b.z;  // the record's event id
        for (uint32_t l = 0; l < nl; ++l) {
          const float* row = p.table[l] + (uint64_t)e * p.jpad[l];
          double s = 0.0;
          bool any = false;
          for (uint32_t j = 0; j < p.J[l]; ++j) {
            const float x = row[j];
            if (x != 0.0f) {
              const double2 t = s_t1[p.col0[l] + j];
              s += clamp_fast((double)x, t.x, t.y);  // steps 1-2 in layer order
              any = true;
            }
          }
          if (any) flush(l, s);
        }
      }
    }
    if (n <= 4u && n != 0u) {
      const uint32_t cols = a.x;
      const float loss[4] = {__uint_as_float(a.z), __uint_as_float(a.w), __uint_as_float(b.x), __uint_as_float(b.y)};
      uint32_t cur = s_lay[cols & 0xffu];
      double s = 0.0;
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i) {
        if (i < n) {
          const uint32_t c = (cols >> (8u * i)) & 0xffu;
          const uint32_t l = s_lay[c];
          if (l != cur) {  // entries are in layer order: a new layer starts
            flush(cur, s);
            s = 0.0;
            cur = l;
          }
          const double2 t = s_t1[c];
          s += clamp_fast((double)loss[i], t.x, t.y);  // steps 1-2: FT1, sum over the layer's ELTs
        }
      }
      flush(cur, s);
    }
    oldest = oldest == kFusedDepth - 1u ? 0u : oldest + 1u;
    --nin;
  };
  // One round: with the pipeline full, consume the oldest round; then every lane with a queued hit pops
  // one and requests its record into the next free slot (an empty lane gets a zero record).
  auto round = [&]() {
    if (nin == kFusedDepth - 1u) consume();
    const bool act = head != tail;
    const uint32_t x = lds_u32(q_l | (head & 0x380u));
    if (act) {
      head += 128u;
      vmax = max(vmax, x);
    }
    const uint32_t bx = act ? x : C;
    uint32_t slot = oldest + nin;
    slot = slot >= kFusedDepth ? slot - kFusedDepth : slot;
    const uint32_t dst = rec_l + slot * 1024u;
    const uint4* src = p.rec + 2u * (uint64_t)(bx + 1u);  // C + 1: the all-zero record
    cp_async16_zf(dst, src, act ? 16u : 0u);
    cp_async16_zf(dst + 16u, src + 1, act ? 16u : 0u);
    cp_async_commit();
    ++nin;
  };
  auto scan = [&](const uint4 v, uint32_t valid) {
    test_enqueue(v.x, C, fmul, bits_s, valid, q_l, tail);
    test_enqueue(v.y, C, fmul, bits_s, valid, q_l, tail);
    test_enqueue(v.z, C, fmul, bits_s, valid, q_l, tail);
    test_enqueue(v.w, C, fmul, bits_s, valid, q_l, tail);
    // high candidate rates: a round whenever most lanes hold a hit, or a queue could overflow.  One call
    // site, so one copy of the round's code in the hot loop.
    bool go = __any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u) || __popc(__ballot_sync(FULL, tail != head)) >= 24;
    while (go) {
      round();
      go = __any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u);
    }
  };

  const uint64_t tstride = NWT * K;
  const uint32_t* lp = p.ids + W * K + 4u * lane;
  uint4 A = make_uint4(0u, 0u, 0u, 0u);
  if (nwin > 1u || lane_last) A = ld_ids4_stream(lp);
  for (uint32_t k = 0; k < nt; ++k) {
    if (p.prefetch && lane == 0 && k + 2u < nt) prefetch_l2_bulk(lp + 2u * tstride - 4u * lane, K * 4u);
    for (uint32_t w = 0; w < nwin; ++w) {  // one scan site; buffers rotated by moves
      const bool last = w + 1u == nwin;
      const uint32_t* nx = last ? lp + tstride : lp + 128u * (w + 1u);
      const bool ok = last ? (k + 1u < nt && (nwin > 1u || lane_last)) : (w + 2u < nwin || lane_last);
      uint4 nxt = A;
      if (ok) nxt = ld_ids4_stream(nx);
      scan(A, last ? last_valid : FULL);
      A = nxt;
    }
    lp += tstride;
    // ---- trial end: drain every queue, then close each layer of trial W + k NWT
    while (__any_sync(FULL, tail != head)) round();
    while (nin != 0u) consume();
    const uint64_t t = W + (uint64_t)k * NWT;
    for (uint32_t l = 0; l < nl; ++l) {
      double v = acc[l * 32u];
      acc[l * 32u] = 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
      if (lane == 0) p.ylt[l * p.ld + t] = clamp_terms(v, p.r3[l], p.l3[l]);  // step 4: FT3 on S_n
    }
  }
  const bool bad = __any_sync(FULL, vmax >= C);
  if (lane == 0 && bad) atomicOr(p.err, 1u);
}

}  // namespace ara

// mask_kernel.cuh -- the ARA hot path for fixed-length trials of at most 1024 occurrences (configs P, PI,
// M, X: K = 1000, K % 4 == 0, 16-B aligned ids), built so that the per-occurrence work is one presence
// test and ONE instruction to record a hit.
//
// Algorithm 1 per layer; one warp per trial at a time, trials interleaved over the
// grid's warps.  A trial's K ids form <= 8 windows of 128 (lane l holds window positions 4l..4l+3):
//
//   * Step 1's presence test is the folded shared-memory bitmap of the presence kernel (an
//     absent event's loss is 0, reading c9; folding adds false positives only; ids outside [1, C] map to
//     the always-set sentinel bit C);
//   * a hit sets bit 4 w + u of the lane's 32-bit CANDIDATE MASK (window w, slot u): no queue, no ballot;
//   * after the trial's last window the masks are compacted once: a warp prefix sum of the popcounts gives
//     every candidate its index in the trial's canonical order (lane-major, stream order within a lane),
//     each lane reloads its candidates' ids (L2-resident: the trial was streamed a moment ago) into a
//     per-warp staging list;
//   * while the warp scans the NEXT trial, the staged list is consumed in batches of 32: each lane
//     cp.asyncs its event's 16-B sparse record, and one batch step later applies FT1 per ELT, sums, applies
//     FT2 (Steps 1-3) and adds the occurrence-net loss to its partial sum;
//   * the trial is closed when its last batch is consumed: fixed xor-tree over the lanes, FT3 (Step 4,
//     PAPER.md:114, :129), one 8-B YLT store.
//
// Summation order: batch lane L accumulates the trial's candidates whose canonical index is L mod 32, in
// index order; the lanes are combined by the fixed tree.  The order depends only on the trial's own ids
// and the layer's (canonical) fold, so the YLT is bitwise reproducible for any sharding or launch shape.
#pragma once
#include <type_traits>

#include "ara_kernel.cuh"

namespace ara {

constexpr uint32_t kMaskStage = 256;  // staged candidates per warp (a trial with more is consumed in chunks)
constexpr uint32_t kMaskWarpSmem = kMaskStage * 4 + 2 * 32 * 16;  // staging + two record slots per lane

__host__ __device__ constexpr uint32_t mask_smem_extra(uint32_t jpad, uint32_t nw) {
  return 16u + jpad * 16u + 16u + nw * kMaskWarpSmem;  // bitmap pad, FT1 pairs, alignment, warps
}

// Presence test of the lane's four ids of window W; a hit on slot u sets bit 4 W + u of the lane's candidate
// mask (predicated OR with an immediate, no branch, no integer 0/1).  `vpred` masks a lane outside the
// trial (the lane-masked last window).
template <int W>
__device__ __forceinline__ void test_mark4(const uint4 v, uint32_t C, uint32_t fmul, uint32_t bits_s, uint32_t valid,
                                           uint32_t& mask) {
  asm volatile(
      "{\n"
      " .reg .pred p0, p1, p2, p3;\n"
      " .reg .b32 x0, x1, x2, x3, w0, w1, w2, w3;\n"
      " sub.u32 x0, %1, 1;\n min.u32 x0, x0, %5;\n sub.u32 x1, %2, 1;\n min.u32 x1, x1, %5;\n"
      " sub.u32 x2, %3, 1;\n min.u32 x2, x2, %5;\n sub.u32 x3, %4, 1;\n min.u32 x3, x3, %5;\n"
      " mul.hi.u32 w0, x0, %6;\n mad.lo.u32 w0, w0, 4, %7;\n ld.shared.u32 w0, [w0];\n"
      " mul.hi.u32 w1, x1, %6;\n mad.lo.u32 w1, w1, 4, %7;\n ld.shared.u32 w1, [w1];\n"
      " mul.hi.u32 w2, x2, %6;\n mad.lo.u32 w2, w2, 4, %7;\n ld.shared.u32 w2, [w2];\n"
      " mul.hi.u32 w3, x3, %6;\n mad.lo.u32 w3, w3, 4, %7;\n ld.shared.u32 w3, [w3];\n"
      " and.b32 x0, x0, 31;\n shl.b32 x0, 1, x0;\n and.b32 x0, x0, w0;\n and.b32 x0, x0, %9;\n setp.ne.b32 p0, x0, 0;\n"
      " and.b32 x1, x1, 31;\n shl.b32 x1, 1, x1;\n and.b32 x1, x1, w1;\n and.b32 x1, x1, %9;\n setp.ne.b32 p1, x1, 0;\n"
      " and.b32 x2, x2, 31;\n shl.b32 x2, 1, x2;\n and.b32 x2, x2, w2;\n and.b32 x2, x2, %9;\n setp.ne.b32 p2, x2, 0;\n"
      " and.b32 x3, x3, 31;\n shl.b32 x3, 1, x3;\n and.b32 x3, x3, w3;\n and.b32 x3, x3, %9;\n setp.ne.b32 p3, x3, 0;\n"
      " @p0 or.b32 %0, %0, %8;\n @p1 or.b32 %0, %0, %10;\n @p2 or.b32 %0, %0, %11;\n @p3 or.b32 %0, %0, %12;\n"
      "}\n"
      : "+r"(mask)
      : "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(C), "r"(fmul), "r"(bits_s), "n"(1u << (4 * W)), "r"(valid),
        "n"(1u << (4 * W + 1)), "n"(1u << (4 * W + 2)), "n"(1u << (4 * W + 3)));
}

// Streaming 16-B load of 4 YET ids kept in L2 (evict_last): the trial's candidate ids are reloaded from L2
// when the trial is staged.
__device__ __forceinline__ uint4 ld_ids4_keep(const uint32_t* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// NW: warps per block (one block per SM).  OLT: also the largest occurrence-net loss per trial.
// NWIN: windows per trial (compile time; 8 covers K in (896, 1024], the paper's 1000 events per trial).
// PFD: > 0 = each lane also prefetches (prefetch.global.L2) its slots PFD windows ahead.
template <int NW, bool OLT, int NWIN = 8, int PFD = 0>
__global__ void __launch_bounds__(NW * 32, 1) ara_mask_kernel(const __grid_constant__ LayerParams p) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t fw = p.present_words;
  const uint32_t jpad = p.jpad;
  uint32_t bits_s;  // folded bitmap (shared address kept in a register)
  asm volatile("mov.u32 %0, %1;" : "=r"(bits_s) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
  const uint32_t t1_w = (fw + 3u) & ~3u;
  double2* s_t1 = reinterpret_cast<double2*>(smem + t1_w);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);
  const uint32_t base_s = ((uint32_t)__cvta_generic_to_shared(smem + t1_w + jpad * 4u) + 15u) & ~15u;
  const uint32_t stage_s = base_s + warp * kMaskWarpSmem;  // this warp's staging list (kMaskStage ids)
  const uint32_t rec_l = base_s + warp * kMaskWarpSmem + kMaskStage * 4u + 16u * lane;  // slot s: + s * 512

  for (uint32_t j = threadIdx.x; j < jpad; j += blockDim.x) s_t1[j] = make_double2(p.r1[j], p.l1[j]);
  for (uint32_t w = threadIdx.x; w < fw; w += blockDim.x) smem[w] = __ldg(p.present + w);
  __syncthreads();

  const uint64_t W = (uint64_t)blockIdx.x * NW + warp, NWT = (uint64_t)gridDim.x * NW;
  const uint64_t N = p.num_trials;
  const uint32_t nt = (uint32_t)(N > W ? (N - 1 - W) / NWT + 1 : 0);
  if (nt == 0) return;
  const uint32_t K = p.K;  // 4 .. 1024, multiple of 4
  static_assert(NWIN >= 2, "the mask kernel needs at least two windows per trial");
  constexpr uint32_t nwin = NWIN;  // the host launches this kernel only when (K + 127) / 128 == NWIN
  const bool lane_last = 4u * lane < K - 128u * (nwin - 1u);
  const uint64_t pol_yet = make_policy(true, 1u);  // evict_last: the trial's lines stay for the reload
  const uint32_t C = p.C, fmul = p.fold_mul;

  // ---- the previous trial's staged candidates (warp-uniform except S, M)
  uint32_t pt_total = 0;   // candidates of the trial being consumed
  uint32_t pt_chunk = 0;   // canonical index of staging[0] (chunks of kMaskStage)
  uint32_t pt_next = 0;    // next canonical index to issue
  uint64_t pt_t = 0;       // its trial index
  bool pt_open = false;    // a trial is being consumed
  uint32_t pt_mask = 0, pt_prefix = 0;  // per lane: its mask and exclusive prefix (for chunk refills)
  const uint32_t* pt_ids = nullptr;     // per lane: its slots of the trial's first window (id reloads)
  int inflight = 0;        // batches in flight (0..2)
  uint32_t slot_old = 0;   // record slot of the oldest in-flight batch
  uint32_t vmax = 0;       // max over issued (id - 1); >= C marks an invalid id
  double S = 0.0, Mx = 0.0;

  // Stage candidates [pt_chunk, pt_chunk + kMaskStage) of the trial being consumed: every lane walks its
  // set bits and cp.asyncs the ids whose canonical index falls in the chunk straight from global memory
  // (L2) into the staging list -- no register round trip; the first batch step waits for them.
  bool staged_pending = false;
  auto stage_chunk = [&]() {
    uint32_t m = pt_mask, idx = pt_prefix;
    const uint32_t st_s = stage_s;
    while (m != 0u) {
      const uint32_t b = __ffs(m) - 1u;
      m &= m - 1u;
      if (idx >= pt_chunk && idx < pt_chunk + kMaskStage)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(st_s + 4u * (idx - pt_chunk)),
                     "l"(pt_ids + (b >> 2) * 128u + (b & 3u))
                     : "memory");
      ++idx;
    }
    cp_async_commit();
    staged_pending = true;
  };
  auto close = [&]() {  // fixed tree, FT3, one store (and the OLT maximum)
    double v = S;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    if (lane == 0) p.ylt[pt_t] = clamp_terms(v, p.r3, p.l3);
    if constexpr (OLT) {
      double mm = Mx;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mm = fmax(mm, __shfl_xor_sync(FULL, mm, off));
      if (lane == 0) p.olt[pt_t] = mm;
      Mx = 0.0;
    }
    S = 0.0;
    pt_open = false;
  };
  auto consume_oldest = [&]() {  // Steps 1-3 for the oldest batch in flight, accumulated per lane
    if (inflight == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else cp_async_wait_all();
    const uint4 r = lds_u128(rec_l + slot_old * 512u);
    const uint32_t c1 = r.x & 0xffu, c2 = (r.x >> 8) & 0xffu, nz = (r.x >> 16) & 0xffu;
    double sum = 0.0;
    if (__any_sync(FULL, nz > 2u)) {  // rare: a row with more than two losses is read in full
      if (nz > 2u) {
        const float* row = p.table + (uint64_t)r.w * jpad;  // r.w: the record's event id
        for (uint32_t j = 0; j < jpad; ++j) {
          const float x = row[j];
          if (x != 0.0f) {
            const double2 t = s_t1[j];
            sum += clamp_fast((double)x, t.x, t.y);
          }
        }
      }
    }
    if (nz <= 2u) {
      const double2 ta = s_t1[c1], tb = s_t1[c2];
      sum += clamp_fast((double)__uint_as_float(r.y), ta.x, ta.y);  // steps 1-2: FT1, sum over ELTs
      sum += clamp_fast((double)__uint_as_float(r.z), tb.x, tb.y);
    }
    const double o = clamp_fast(sum, p.r2, p.l2);  // step 3: FT2 (+0 for empty slots and zero rows)
    S += o;                                        // step 4 accumulation
    if constexpr (OLT) Mx = o > Mx ? o : Mx;
    slot_old ^= 1u;
    --inflight;
  };
  // One batch step: consume the oldest batch if both slots are busy, then issue the next 32 staged
  // candidates (refilling the staging list when the chunk is used up).
  auto batch_step = [&]() {
    if (inflight == 2) consume_oldest();
    if (pt_next >= pt_chunk + kMaskStage) {  // the trial has more candidates than one staging chunk
      while (inflight) consume_oldest();       // the chunk's batches are done with the staging list
      __syncwarp();
      pt_chunk += kMaskStage;
      stage_chunk();
    }
    if (staged_pending) {  // the staged ids have landed (no record batch is in flight here)
      if (inflight == 0) cp_async_wait_all();
      else asm volatile("cp.async.wait_group 1;" ::: "memory");
      __syncwarp();
      staged_pending = false;
    }
    const uint32_t i = pt_next + lane;
    const bool act = i < pt_total;
    uint32_t e = act ? lds_u32(stage_s + 4u * (i - pt_chunk)) : 0u;
    vmax = act ? max(vmax, e - 1u) : vmax;  // an invalid id reached the list via the sentinel (0 wraps)
    e = min(e, C + 1u);                        // invalid ids read the all-zero record C + 1
    const uint32_t slot = slot_old ^ (uint32_t)inflight;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rec_l + slot * 512u), "l"(p.rec + e),
                 "r"(act ? 16u : 0u)
                 : "memory");
    cp_async_commit();
    ++inflight;
    pt_next += 32u;
  };
  // Finish the trial being consumed: every remaining batch, then close it.
  auto finish = [&]() {
    if (!pt_open) return;
    while (pt_next < pt_total) batch_step();
    while (inflight) consume_oldest();
    if (staged_pending) {  // a trial without candidates: its (empty) staging group
      cp_async_wait_all();
      staged_pending = false;
    }
    __syncwarp();  // every lane is done with the staging list before it is refilled
    close();
  };

  const uint64_t tstride = NWT * K;
  const uint32_t* lp = p.ids + W * K + 4u * lane;  // this lane's slots of the trial's first window
  uint4 A = make_uint4(0u, 0u, 0u, 0u);
  if (nwin > 1u || lane_last) A = ld_ids4_keep(lp, pol_yet);
  for (uint32_t k = 0; k < nt; ++k) {
    if (p.prefetch && lane == 0 && k + 2u < nt) prefetch_l2_bulk(lp + 2u * tstride - 4u * lane, K * 4u);
    uint32_t mask = 0;
    // ---- scan the trial: one presence test and one predicated OR per id; a batch step of the previous
    // trial after every second window
    auto window = [&](auto wc) {
      constexpr uint32_t w = decltype(wc)::value;
      constexpr bool last = w + 1u == nwin;
      uint4 nxt = A;
      if constexpr (!last) {
        if (w + 2u < nwin || lane_last) nxt = ld_ids4_keep(lp + 128u * (w + 1u), pol_yet);
      } else {
        if (k + 1u < nt && (nwin > 1u || lane_last)) nxt = ld_ids4_keep(lp + tstride, pol_yet);  // next trial
      }
      if constexpr (PFD > 0) {  // per-lane L2 prefetch PFD windows ahead (into the next trial)
        constexpr uint32_t g = w + (uint32_t)PFD;
        const uint32_t* pf = g < nwin ? lp + 128u * g : lp + tstride + 128u * (g - nwin);
        if (g < nwin || k + 1u < nt) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
      }
      test_mark4<(int)w>(A, C, fmul, bits_s, (!last || lane_last) ? 0xffffffffu : 0u, mask);
      A = nxt;
      if constexpr ((w & 1u) == 0u) {
        if (pt_open && pt_next < pt_total) batch_step();
      }
    };
    window(std::integral_constant<uint32_t, 0>{});
    if constexpr (nwin > 1) window(std::integral_constant<uint32_t, 1>{});
    if constexpr (nwin > 2) window(std::integral_constant<uint32_t, 2>{});
    if constexpr (nwin > 3) window(std::integral_constant<uint32_t, 3>{});
    if constexpr (nwin > 4) window(std::integral_constant<uint32_t, 4>{});
    if constexpr (nwin > 5) window(std::integral_constant<uint32_t, 5>{});
    if constexpr (nwin > 6) window(std::integral_constant<uint32_t, 6>{});
    if constexpr (nwin > 7) window(std::integral_constant<uint32_t, 7>{});
    // ---- the previous trial is done: close it; then stage this trial's candidates
    finish();
    const uint32_t cnt = __popc(mask);
    uint32_t incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, off);
      if (lane >= (uint32_t)off) incl += y;
    }
    pt_total = __shfl_sync(FULL, incl, 31);
    pt_prefix = incl - cnt;
    pt_mask = mask;
    pt_ids = lp;
    pt_t = W + (uint64_t)k * NWT;
    pt_chunk = 0;
    pt_next = 0;
    pt_open = true;
    stage_chunk();
    lp += tstride;
  }
  finish();
  const bool bad = __any_sync(FULL, vmax >= C);
  if (lane == 0 && bad) atomicOr(p.err, 1u);
}

}  // namespace ara

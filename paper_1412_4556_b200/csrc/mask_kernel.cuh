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
template <int NW, bool OLT, int NWIN = 8>
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
  constexpr uint32_t nwin = NWIN;  // the host launches this kernel only when (K + 127) / 128 == NWIN
  const bool lane_last = 4u * lane < K - 128u * (nwin - 1u);
  const uint64_t pol_yet = make_policy(true, 1u);  // evict_last: the trial's lines stay for the reload
  const uint32_t C = p.C, fmul = p.fold_mul;

  // ---- the staged trial: its candidates are issued as batches of 32 while the next trial is scanned
  uint32_t st_total = 0;   // candidates of the staged trial
  uint32_t st_chunk = 0;   // canonical index of staging[0] (chunks of kMaskStage)
  uint32_t st_next = 0;    // next canonical index to issue
  uint64_t st_t = 0;       // its trial index
  uint32_t st_par = 0;     // its parity (accumulator)
  bool st_live = false;    // a staged trial still has a batch to issue (an empty trial issues one empty batch)
  bool st_pending = false; // the staged ids are still in flight (cp.async)
  uint32_t st_mask = 0, st_prefix = 0;  // per lane: its candidate mask and exclusive prefix (chunk refills)
  const uint32_t* st_ids = nullptr;     // per lane: its slots of the staged trial's first window
  // ---- batches in flight (FIFO of <= 2, record slots alternate); each closes its trial if it is the last
  uint32_t inflight = 0, slot_old = 0;
  uint32_t f_par[2] = {0u, 0u}, f_last[2] = {0u, 0u};
  uint64_t f_t[2] = {0u, 0u};
  uint32_t vmax = 0;       // max over issued (id - 1); >= C marks an invalid id
  double S0 = 0.0, S1 = 0.0, M0 = 0.0, M1 = 0.0;  // per lane: partial sums (and OLT maxima) by trial parity

  // Stage candidates [st_chunk, st_chunk + kMaskStage) of the staged trial: every lane walks its set bits
  // and cp.asyncs the ids whose canonical index falls in the chunk straight from global memory (L2) into
  // the staging list (no register round trip); the next issue waits for them.
  auto stage_chunk = [&]() {
    uint32_t m = st_mask, idx = st_prefix;
    while (m != 0u) {
      const uint32_t bpos = __ffs(m) - 1u;
      m &= m - 1u;
      if (idx >= st_chunk && idx < st_chunk + kMaskStage)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(stage_s + 4u * (idx - st_chunk)),
                     "l"(st_ids + (bpos >> 2) * 128u + (bpos & 3u))
                     : "memory");
      ++idx;
    }
    cp_async_commit();
    st_pending = true;
  };
  auto close = [&](uint32_t par, uint64_t t) {  // fixed tree, FT3, one store (and the OLT maximum)
    double v = par ? S1 : S0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    if (lane == 0) p.ylt[t] = clamp_terms(v, p.r3, p.l3);  // step 4: FT3 on S_n
    if constexpr (OLT) {
      double mm = par ? M1 : M0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mm = fmax(mm, __shfl_xor_sync(FULL, mm, off));
      if (lane == 0) p.olt[t] = mm;
      if (par) M1 = 0.0; else M0 = 0.0;
    }
    if (par) S1 = 0.0; else S0 = 0.0;
  };
  auto consume_oldest = [&]() {  // Steps 1-3 for the oldest batch in flight, accumulated by trial parity
    if (inflight == 2u) asm volatile("cp.async.wait_group 1;" ::: "memory");
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
    const uint32_t par = slot_old ? f_par[1] : f_par[0];
    S0 += par ? 0.0 : o;  // step 4 accumulation (x + 0 == x exactly)
    S1 += par ? o : 0.0;
    if constexpr (OLT) {
      if (par) M1 = o > M1 ? o : M1;
      else M0 = o > M0 ? o : M0;
    }
    if (slot_old ? f_last[1] : f_last[0]) close(par, slot_old ? f_t[1] : f_t[0]);
    slot_old ^= 1u;
    --inflight;
  };
  // Issue the staged trial's next batch of 32 (consuming the oldest batch first when both slots are busy).
  auto issue = [&]() {
    if (inflight == 2u) consume_oldest();
    if (st_next >= st_chunk + kMaskStage) {  // more candidates than one staging chunk: refill (the batches of
      __syncwarp();                         // the chunk already hold their records, not staging entries)
      st_chunk += kMaskStage;
      stage_chunk();
    }
    if (st_pending) {  // the staged ids (the newest cp.async group; older record groups complete first anyway)
      cp_async_wait_all();
      __syncwarp();
      st_pending = false;
    }
    const uint32_t i = st_next + lane;
    const bool act = i < st_total;
    uint32_t e = act ? lds_u32(stage_s + 4u * (i - st_chunk)) : 0u;
    if (act) vmax = max(vmax, e - 1u);  // an invalid id reached the list via the sentinel (0 wraps)
    e = min(e, C + 1u);                  // invalid ids read the all-zero record C + 1
    const uint32_t slot = slot_old ^ inflight;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(rec_l + slot * 512u), "l"(p.rec + e),
                 "r"(act ? 16u : 0u)
                 : "memory");
    cp_async_commit();
    st_next += 32u;
    const uint32_t last = st_next >= st_total ? 1u : 0u;
    if (slot) {
      f_par[1] = st_par; f_last[1] = last; f_t[1] = st_t;
    } else {
      f_par[0] = st_par; f_last[0] = last; f_t[0] = st_t;
    }
    st_live = !last;
    ++inflight;
  };

  const uint64_t tstride = NWT * K;
  const uint32_t* lp = p.ids + W * K + 4u * lane;  // this lane's slots of the trial's first window
  // window w + 1 (or the next trial's window 0) is requested while window w is tested.  A look-ahead of
  // two windows (three rotating register sets) measured no faster (1.392 vs 1.39 ms on P) and spills at
  // NW = 32, so one window it is
  uint4 A = make_uint4(0u, 0u, 0u, 0u);
  if (nwin > 1u || lane_last) A = ld_ids4_keep(lp, pol_yet);
  for (uint32_t k = 0; k < nt; ++k) {
    if (p.prefetch && lane == 0 && k + 2u < nt) prefetch_l2_bulk(lp + 2u * tstride - 4u * lane, K * 4u);
    uint32_t mask = 0;
    // ---- scan the trial: one presence test and one predicated OR per id; a batch step of the staged
    // trial after every second window
    auto window = [&](auto wc) {
      constexpr uint32_t w = decltype(wc)::value;
      constexpr bool last = w + 1u == nwin;
      uint4 nxt = A;
      if constexpr (!last) {
        if (w + 2u < nwin || lane_last) nxt = ld_ids4_keep(lp + 128u * (w + 1u), pol_yet);
      } else {
        if (k + 1u < nt && (nwin > 1u || lane_last)) nxt = ld_ids4_keep(lp + tstride, pol_yet);
      }
      test_mark4<(int)w>(A, C, fmul, bits_s, (!last || lane_last) ? 0xffffffffu : 0u, mask);
      A = nxt;
      if constexpr ((w & 1u) == 1u) {
        if (st_live) issue();
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
    // ---- every batch of the staged trial is issued (its records are in flight); stage this trial
    while (st_live) issue();
    const uint32_t cnt = __popc(mask);
    uint32_t incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, off);
      if (lane >= (uint32_t)off) incl += y;
    }
    __syncwarp();  // every lane has read the staging list of the previous trial
    st_total = __shfl_sync(FULL, incl, 31);
    st_prefix = incl - cnt;
    st_mask = mask;
    st_ids = lp;
    st_t = W + (uint64_t)k * NWT;
    st_par = k & 1u;
    st_chunk = 0;
    st_next = 0;
    st_live = true;  // a trial without candidates still issues one (empty) batch that closes it
    stage_chunk();
    lp += tstride;
  }
  while (st_live) issue();
  while (inflight) consume_oldest();
  const bool bad = __any_sync(FULL, vmax >= C);
  if (lane == 0 && bad) atomicOr(p.err, 1u);
}

}  // namespace ara

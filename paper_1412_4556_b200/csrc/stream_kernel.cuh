// stream_kernel.cuh -- the ARA hot path for fixed-length trials on sm_100a (configs P, PI, M, X: every
// trial holds K event occurrences, K % 4 == 0, 16-B aligned ids).  Same method and same summation
// order as ara_presence_kernel (presence_kernel.cuh), with the per-trial and per-batch machinery rebuilt
// so that far fewer instructions are spent per event occurrence:
//
//   * each warp owns a CONTIGUOUS block of trials, so its YET is one continuous stream: the last
//     (lane-masked) window of a trial and the first window of the next are requested one step ahead
//     like every other window, and one bulk L2 prefetch per trial pulls the next trial in;
//   * Step 1's presence test is the folded shared-memory bitmap of the presence kernel (an event is
//     gathered only if its row holds a loss; PAPER.md:209 -- an absent event's loss is 0, reading c9);
//     hits are appended per pair of window slots with one ballot (the presence kernel's order), into a
//     128-entry RING per warp (no queue shifting);
//   * every 32 queued hits form a batch: each lane cp.asyncs its event's 16-B sparse record into
//     shared memory; one batch later the lane applies FT1 (per ELT), sums, applies FT2 (Steps 1-3,
//     PAPER.md:109-113, :125-127) and adds the occurrence-net loss to its partial sum of the trial
//     that owns the hit;
//   * trial ownership: the first hit ordinal of each started trial is kept in a 32-entry ring held in
//     REGISTERS (lane j: trials k = j mod 32), so a batch may span any number of trials; a trial is
//     closed when a later trial's first hit is consumed (or at the end): a fixed rotation into the
//     canonical frame (lane c: the trial's hits i = c mod 32) and xor-tree, then FT3 (Step 4,
//     PAPER.md:114, :129) and one 8-B YLT store.  Trials without hits are closed the same way (+0).
//
// The order in which a trial's hits are queued depends only on the trial's ids (windows start at the
// trial's first occurrence), each lane sums its hits in queue order, and the close is a fixed tree: the
// YLT is bitwise identical to the presence kernel's, for any sharding or launch shape.
#pragma once
#include "ara_kernel.cuh"

namespace ara {

constexpr int kRing = 128;                        // per-warp hit ring (entries; a power of two)
constexpr uint32_t kRingMask = (kRing - 1) * 4;   // byte offset mask inside the ring
constexpr uint32_t kWarpSmem = kRing * 4 + 32 * 16;  // ring + 32 record slots = 1 KB per warp

// Dynamic shared memory of the stream kernel besides the bitmap words (host and device agree on this).
__host__ __device__ constexpr uint32_t stream_smem_extra(uint32_t jpad, uint32_t nw) {
  return 16u + jpad * 16u + 1024u + nw * kWarpSmem;  // bitmap pad, FT1 pairs, ring alignment slack, warps
}

// Pair insertion into the warp's ring: the presence kernel's pair_insert (same order: the lanes' first
// hit of the pair, lanes ascending, then -- only if some lane hit both -- the second ids), with the
// slot address wrapped into the 512-B aligned ring at ring_s.  qt: byte counter of inserted hits.
__device__ __forceinline__ void ring_pair_insert(uint32_t wa, uint32_t xa, uint32_t ida, uint32_t wb, uint32_t xb,
                                                 uint32_t idb, uint32_t lt, uint32_t& qt, uint32_t valid,
                                                 uint32_t ring_s) {
  asm volatile(
      "{\n"
      " .reg .pred pa, pb, pany, pboth, pq;\n"
      " .reg .b32 sa, sb, ma, mb, f, m, t, a, c;\n"
      " and.b32 sa, %2, 31;\n shl.b32 ma, 1, sa;\n and.b32 ma, ma, %1;\n and.b32 ma, ma, %8;\n setp.ne.b32 pa, ma, 0;\n"
      " and.b32 sb, %5, 31;\n shl.b32 mb, 1, sb;\n and.b32 mb, mb, %4;\n and.b32 mb, mb, %8;\n setp.ne.b32 pb, mb, 0;\n"
      " or.pred pany, pa, pb;\n and.pred pboth, pa, pb;\n"
      " selp.b32 f, %3, %6, pa;\n"
      " vote.sync.ballot.b32 m, pany, 0xffffffff;\n"
      " and.b32 t, m, %7;\n popc.b32 t, t;\n mad.lo.u32 a, t, 4, %0;\n and.b32 a, a, %10;\n or.b32 a, a, %9;\n"
      " @pany st.shared.u32 [a], f;\n"
      " popc.b32 c, m;\n mad.lo.u32 %0, c, 4, %0;\n"
      " vote.sync.any.pred pq, pboth, 0xffffffff;\n"
      " @!pq bra.uni RPAIR_DONE_%=;\n"
      " vote.sync.ballot.b32 m, pboth, 0xffffffff;\n"
      " and.b32 t, m, %7;\n popc.b32 t, t;\n mad.lo.u32 a, t, 4, %0;\n and.b32 a, a, %10;\n or.b32 a, a, %9;\n"
      " @pboth st.shared.u32 [a], %6;\n"
      " popc.b32 c, m;\n mad.lo.u32 %0, c, 4, %0;\n"
      "RPAIR_DONE_%=:\n"
      "}\n"
      : "+r"(qt)
      : "r"(wa), "r"(xa), "r"(ida), "r"(wb), "r"(xb), "r"(idb), "r"(lt), "r"(valid), "r"(ring_s), "n"(kRingMask)
      : "memory");
}

// 16-byte cp.async with zero fill: copies `src_bytes` (16 or 0) and fills the rest of the slot with 0.
// (No L2 cache-policy operand: with one, ptxas 12.9 placed the 64-bit policy descriptor in an odd
// uniform register, an illegal instruction at run time.)
__device__ __forceinline__ void cp_async16_zfill(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}

// NW: warps per block (one block per SM).  OLT: also the largest occurrence-net loss per trial.
template <int NW, bool OLT>
__global__ void __launch_bounds__(NW * 32, 1) ara_stream_kernel(const __grid_constant__ LayerParams p) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t fw = p.present_words;
  const uint32_t jpad = p.jpad;
  uint32_t* bits = smem;                                   // folded presence bitmap (fold_mul)
  const uint32_t bits_s = (uint32_t)__cvta_generic_to_shared(bits);
  const uint32_t t1_w = (fw + 3u) & ~3u;                   // FT1 (R, L) pairs, 16-B aligned
  double2* s_t1 = reinterpret_cast<double2*>(smem + t1_w);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);  // warp-uniform for the compiler
  const uint32_t base_s = (uint32_t)__cvta_generic_to_shared(smem + t1_w + jpad * 4u);
  const uint32_t ring_s = ((base_s + 511u) & ~511u) + warp * kWarpSmem;  // 512-B aligned ring
  const uint32_t rec_s = ring_s + kRing * 4u;                              // 32 x 16-B record slots

  for (uint32_t j = threadIdx.x; j < jpad; j += blockDim.x) s_t1[j] = make_double2(p.r1[j], p.l1[j]);
  for (uint32_t w = threadIdx.x; w < fw; w += blockDim.x) bits[w] = __ldg(p.present + w);
  __syncthreads();

  // this warp's trials t0 + k * tstep, k < nt: a contiguous block (tstep 1) or interleaved over the grid
  const uint64_t W = (uint64_t)blockIdx.x * NW + warp, NWT = (uint64_t)gridDim.x * NW;
  const uint64_t N = p.num_trials;
  const uint64_t tstep = p.interleave ? NWT : 1u;
  const uint64_t t0 = p.interleave ? W : (uint64_t)(((unsigned __int128)W * N) / NWT);
  const uint32_t nt = p.interleave ? (uint32_t)(N > W ? (N - 1 - W) / NWT + 1 : 0)
                                   : (uint32_t)((uint64_t)(((unsigned __int128)(W + 1) * N) / NWT) - t0);
  if (nt == 0) return;  // warp-uniform

  const uint32_t K = p.K;                       // > 0, multiple of 4
  const uint32_t nwin = (K + 127u) >> 7;        // windows per trial; the last one lane-masked
  const bool lane_last = 4u * lane < K - 128u * (nwin - 1u);  // this lane's slots lie inside the last window
  const uint32_t last_valid = lane_last ? FULL : 0u;
  const uint32_t C = p.C;
  const uint32_t fmul = p.fold_mul;
  const uint32_t lt = lanemask_lt();

  // ---- hit ring + batch state (warp-uniform unless noted)
  uint32_t qt = 0;    // bytes: 4 x (ordinal of the next hit to insert)
  uint32_t hd = 0;    // bytes: 4 x (ordinal of the next hit to issue); batches start at multiples of 32
  uint32_t bs = 0;    // ordinal of slot 0 of the pending batch
  uint32_t bn = 0;    // pending batch size (0 = none)
  uint32_t be = 0;    // per lane: the pending batch's event id (clamped), for rows read in full
  uint32_t vmax = 0;  // per lane: max over issued ids of (id - 1); >= C means an invalid id was seen
  // ---- trial bookkeeping
  uint32_t fr = 0;              // per lane j: first hit ordinal of the started trials k = j (mod 32)
  uint32_t kO = 0;              // open trial: the trial owning the next hit to consume
  uint32_t fO = 0;              // its first hit ordinal (rotation into the canonical frame)
  uint32_t nb = 0xffffffffu;    // first hit ordinal of trial kO + 1 (0xffffffff: not started yet)
  uint32_t kcur = 0;            // trial being scanned
  double S = 0.0;               // per lane: partial sum of trial kO (hits with ordinal = lane mod 32)
  double Mx = 0.0;              // per lane: largest occurrence-net loss of trial kO (OLT)

  // Close trial kO: rotate into the canonical frame, fixed xor-tree, FT3, one store (lane 0).
  auto close_open = [&]() {
    double Sr = __shfl_sync(FULL, S, (lane + fO) & 31u);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) Sr += __shfl_xor_sync(FULL, Sr, off);
    if (lane == 0) p.ylt[t0 + (uint64_t)kO * tstep] = clamp_terms(Sr, p.r3, p.l3);  // step 4: FT3 on S_n
    if constexpr (OLT) {
      double M = Mx;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, off));
      if (lane == 0) p.olt[t0 + (uint64_t)kO * tstep] = M;
      Mx = 0.0;
    }
    S = 0.0;
  };
  // Consume the pending batch: Steps 1-3 per lane from its record, then attribute each lane's
  // occurrence-net loss to the trial owning its ordinal (bs + lane), closing trials as they end.
  auto consume = [&]() {
    if (bn == 0u) return;
    cp_async_wait_all();
    const uint4 r = lds_u128(rec_s + 16u * lane);
    const uint32_t c1 = r.x & 0xffu, c2 = (r.x >> 8) & 0xffu, nz = (r.x >> 16) & 0xffu;
    double sum = 0.0;
    if (__any_sync(FULL, nz > 2u)) {  // rare: a row with more than two losses is read in full
      if (nz > 2u) {
        const float* row = p.table + (uint64_t)be * jpad;
        for (uint32_t j = 0; j < jpad; ++j) {
          const float x = row[j];
          if (x != 0.0f) {
            const double2 t = s_t1[j];
            sum += clamp_fast((double)x, t.x, t.y);  // steps 1-2 in layer order, absent (+0) terms dropped
          }
        }
      }
    }
    if (nz <= 2u) {
      const double2 ta = s_t1[c1], tb = s_t1[c2];
      sum += clamp_fast((double)__uint_as_float(r.y), ta.x, ta.y);  // steps 1-2: FT1, sum over ELTs
      sum += clamp_fast((double)__uint_as_float(r.z), tb.x, tb.y);  // (an absent column: exactly +0)
    }
    const double o = clamp_fast(sum, p.r2, p.l2);  // step 3: FT2 (+0 for empty slots and zero rows)
    uint32_t lo = 0;
    while (true) {
      if (nb >= bs + 32u) {  // trial kO owns every remaining lane of the batch (the common case)
        const bool mine = lane >= lo;
        S += mine ? o : 0.0;
        if constexpr (OLT) Mx = (mine && o > Mx) ? o : Mx;
        break;
      }
      const uint32_t hi = max((int)(nb - bs), (int)lo);  // lanes [lo, hi) belong to trial kO
      const bool mine = lane >= lo && lane < hi;
      S += mine ? o : 0.0;
      if constexpr (OLT) Mx = (mine && o > Mx) ? o : Mx;
      close_open();
      ++kO;
      fO = nb;
      nb = (kO + 1u <= kcur) ? __shfl_sync(FULL, fr, (kO + 1u) & 31u) : 0xffffffffu;
      lo = hi;
    }
    bn = 0u;
  };
  // Issue the next n (<= 32) queued hits as a batch (after consuming the pending one).
  auto issue = [&](uint32_t n) {
    consume();
    __syncwarp();  // the ring slots written by the scans are visible
    const uint32_t e = lds_u32(ring_s | ((hd + 4u * lane) & kRingMask));
    if (lane < n) vmax = max(vmax, e - 1u);  // an invalid id reached the ring via the sentinel bit (0 wraps)
    be = min(e, C + 1u);       // invalid ids read the all-zero record C + 1 (0 reads row 0, also zero)
    cp_async16_zfill(rec_s + 16u * lane, p.rec + be, lane < n ? 16u : 0u);
    cp_async_commit();
    bs = hd >> 2;
    bn = n;
    hd += 128u;  // a partial batch skips the rest of its 32 ordinals: batches stay 32-aligned
  };
  // Consume everything queued and close every trial up to kcur (end of the block, or ring overflow).
  auto flush_all = [&]() {
    while (qt != hd) {
      const uint32_t cnt = (qt - hd) >> 2;
      if (cnt >= 32u) {
        issue(32u);
      } else {
        issue(cnt);
        qt = hd;  // the partial batch moved hd to the next multiple of 32 ordinals
      }
    }
    consume();
    while (kO <= kcur) {  // trials whose hits are all consumed (later ones hold none: +0)
      close_open();
      ++kO;
    }
    nb = 0xffffffffu;
  };
  // Scan one window: lane slots v (positions 4 lane .. +3), `valid` masks lanes outside the trial.
  auto scan = [&](const uint4 v, uint32_t valid) {
    const uint32_t id[4] = {v.x, v.y, v.z, v.w};
    uint32_t x[4], wd[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = min(id[u] - 1u, C);                           // invalid ids -> the always-set sentinel bit C
      wd[u] = lds_ro_u32(bits_s + 4u * __umulhi(x[u], fmul));  // folded bitmap word holding bit x & 31
    }
    ring_pair_insert(wd[0], x[0], id[0], wd[1], x[1], id[1], lt, qt, valid, ring_s);
    while (qt - hd >= 128u) issue(32u);  // <= 31 + 64 queued, ring of 128
    ring_pair_insert(wd[2], x[2], id[2], wd[3], x[3], id[3], lt, qt, valid, ring_s);
    while (qt - hd >= 128u) issue(32u);
  };

  // Window loop.  A holds the window being scanned next; windows are requested one step ahead into the
  // other buffer, full windows in pairs (A, B) so the buffers alternate without copies and the loads
  // use immediate offsets from one running pointer per trial.
  const uint32_t nfull = nwin - 1u;   // full windows per trial before the lane-masked tail window
  const uint32_t npair = nfull >> 1;
  const uint32_t* lp = p.ids + t0 * K + 4u * lane;  // this lane's slots of the trial's first window
  uint4 A = make_uint4(0u, 0u, 0u, 0u), B = A;
  if (nfull != 0u || lane_last) A = ld_ids4_stream(lp);
  for (uint32_t k = 0; k < nt; ++k) {
    // ---- trial start: its first hit ordinal, ring overflow guard, next-trial L2 prefetch
    if (k - kO >= 31u) flush_all();  // 32 trials pending in the register ring (hitless runs)
    if (lane == (k & 31u)) fr = qt >> 2;
    if (k == kO + 1u) nb = qt >> 2;
    if (k == kO) fO = qt >> 2;
    kcur = k;
    if (p.prefetch && lane == 0 && k + 2u < nt) prefetch_l2_bulk(lp + 2u * tstep * K - 4u * lane, K * 4u);
    const uint32_t* wp = lp;
    for (uint32_t i = 0; i < npair; ++i, wp += 256) {  // full windows 2i (in A) and 2i+1
      B = ld_ids4_stream(wp + 128);                    // window 2i+1 < nfull: full
      scan(A, FULL);
      if (2u * i + 2u < nfull || lane_last) A = ld_ids4_stream(wp + 256);  // full, or the tail window
      scan(B, FULL);
    }
    if (nfull & 1u) {  // one more full window (in A); the tail window follows it
      if (lane_last) B = ld_ids4_stream(wp + 128);
      scan(A, FULL);
      A = B;
      wp += 128;
    }
    // the tail window (in A); its successor is the next trial's first window
    lp += tstep * K;
    if (k + 1u < nt && (nfull != 0u || lane_last)) B = ld_ids4_stream(lp);
    scan(A, last_valid);
    A = B;
  }
  flush_all();
  const bool bad = __any_sync(FULL, vmax >= C);
  if (lane == 0 && bad) atomicOr(p.err, 1u);
}

}  // namespace ara

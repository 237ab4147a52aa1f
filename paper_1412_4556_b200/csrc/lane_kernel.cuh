// lane_kernel.cuh -- the default ARA hot path for fixed-length trials on sm_100a (configs P, PI, M, X:
// every trial holds K event occurrences, K % 4 == 0, 16-B aligned ids).
//
// Algorithm 1 of the paper per layer, one WARP per trial at a time, each warp owning
// a contiguous block of trials (so its YET is one continuous stream):
//
//   * YET stream: 128-id windows from the trial's first occurrence, lane l holding positions 4l..4l+3
//     (one 16-B load); full windows are requested one step ahead in pairs of register buffers, the
//     last (lane-masked) window requests the next trial's first window, and one bulk L2 prefetch per
//     trial pulls the trial after next into L2;
//   * Step 1 presence test (an event absent from every ELT of the layer has loss 0 in all
//     of them, reading c9): the layer's presence bitmap FOLDED into shared memory (false positives only,
//     never misses); an id outside [1, C] maps to the always-set sentinel bit C and is reported later;
//   * every hit goes into its LANE's own 8-entry queue in shared memory (no ballots, no compaction):
//     a lane's queue holds the hits of its own position class in stream order;
//   * ROUNDS: when enough lanes hold a queued hit (or one lane's queue is nearly full), every lane
//     with a queued hit pops one and cp.asyncs its event's 16-B sparse record; one round later it
//     applies FT1 per ELT, sums over the layer's ELTs, applies FT2 (Steps 1-3, PAPER.md:109-113,
//     :125-127) and adds the occurrence-net loss to its partial sum of that hit's trial;
//   * a trial is closed lazily, when the trial after next starts (at most two trials are open): a fixed
//     xor-tree over the 32 lanes' partial sums, FT3 (Step 4), one 8-B YLT store.
//
// Summation order: lane l sums, in stream order, the occurrence-net losses of the trial's hits at
// positions p with (p mod 128) / 4 == l; the lanes are combined by a fixed tree.  The order depends
// only on the trial's own ids -- not on the fold (a false positive adds an exact +0), the sharding or
// the launch shape -- so the YLT is bitwise reproducible across all of them.
#pragma once
#include "ara_kernel.cuh"

namespace ara {

constexpr uint32_t kLaneQ = 8;                           // entries per lane queue (power of two)
constexpr uint32_t kLaneWarpSmem = 32 * kLaneQ * 4 + 32 * 16;  // queues (1 KB) + record slots (512 B)

// Dynamic shared memory of the lane kernel besides the bitmap words (host and device agree on this).
__host__ __device__ constexpr uint32_t lane_smem_extra(uint32_t jpad, uint32_t nw) {
  return 16u + jpad * 16u + 1024u + nw * kLaneWarpSmem;  // bitmap pad, FT1 pairs, alignment slack, warps
}

// 16-byte cp.async with zero fill: copies `src_bytes` (16 or 0) and zero-fills the rest of the slot.
// (No L2 cache-policy operand: with one, ptxas 12.9 placed the 64-bit policy descriptor in an odd
// uniform register -- an illegal instruction at run time.)
__device__ __forceinline__ void cp_async16_zf(uint32_t saddr, const void* g, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}

// Presence test of one id and append to the lane's queue, as one PTX block so the hit stays a predicate:
//   x = min(id - 1, C) (invalid ids -> the sentinel bit C), word = bitmap[umulhi(x, fmul)],
//   hit = word bit (x & 31) & valid;  if hit: queue[tail] = x, tail += 1 (queue stride 128 B).
__device__ __forceinline__ void test_enqueue(uint32_t id, uint32_t C, uint32_t fmul, uint32_t bits_s, uint32_t valid,
                                             uint32_t q_l, uint32_t& tail) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " .reg .b32 x, w, a, s, m;\n"
      " sub.u32 x, %1, 1;\n min.u32 x, x, %2;\n"
      " mul.hi.u32 w, x, %3;\n shl.b32 w, w, 2;\n add.u32 w, w, %4;\n ld.shared.u32 w, [w];\n"
      " and.b32 s, x, 31;\n shl.b32 m, 1, s;\n and.b32 m, m, w;\n and.b32 m, m, %5;\n setp.ne.b32 p, m, 0;\n"
      " and.b32 a, %0, 0x380;\n or.b32 a, a, %6;\n"
      " @p st.shared.u32 [a], x;\n"
      " @p add.u32 %0, %0, 128;\n"
      "}\n"
      : "+r"(tail)
      : "r"(id), "r"(C), "r"(fmul), "r"(bits_s), "r"(valid), "r"(q_l)
      : "memory");
}

// XS (exact scan filter, for catalogues far larger than the shared bitmap, config X): the folded test
// only nominates CANDIDATES; each candidate loads the rank entry of its word of the layer's unfolded
// presence bitmap (global memory, L2-resident: the word, bit e = row e holds a loss, and the number of
// rows holding a loss before it) that decides it exactly.  The load is issued while scanning window w and
// used one window later, where only exact hits (and invalid ids, forced through) enter the lane's queue
// -- as their COMPACT record index, the rank of the row among the rows that hold a loss (the event ->
// compact-row index of PAPER.md:211-213's direct-access table without its zero rows).  A false positive
// costs one L2 entry instead of a queue slot, a gather round and a record fetch, and the records a hit
// fetches form a table of the loss-holding rows only (15 MB for config X instead of 160 MB: L2-resident).
// The queue order and the records -- hence the YLT bits -- are those of the plain path.
__device__ __forceinline__ uint32_t fold_candidate(uint32_t id, uint32_t C, uint32_t fmul, uint32_t bits_s,
                                                   uint32_t valid, uint32_t& x) {
  x = min(id - 1u, C);
  const uint32_t w = lds_ro_u32(bits_s + 4u * __umulhi(x, fmul));
  return (w >> (x & 31u)) & valid & 1u;
}

// When bit s = (x + 1) & 31 of the exact word ew.x is set, append the row's compact record index
// ew.y + popc(ew.x & (2^s - 1)) to the lane's queue.
__device__ __forceinline__ void exact_enqueue(uint2 ew, uint32_t x, uint32_t q_l, uint32_t& tail) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      " .reg .b32 s, m, h, r, a;\n"
      " add.u32 s, %1, 1;\n and.b32 s, s, 31;\n shl.b32 m, 1, s;\n and.b32 h, m, %2;\n setp.ne.b32 p, h, 0;\n"
      " sub.u32 m, m, 1;\n and.b32 m, m, %2;\n popc.b32 r, m;\n add.u32 r, r, %3;\n"
      " and.b32 a, %0, 0x380;\n or.b32 a, a, %4;\n"
      " @p st.shared.u32 [a], r;\n"
      " @p add.u32 %0, %0, 128;\n"
      "}\n"
      : "+r"(tail)
      : "r"(x), "r"(ew.x), "r"(ew.y), "r"(q_l)
      : "memory");
}



// NW: warps per block (one block per SM).  OLT: also the largest occurrence-net loss per trial.
// XS: exact scan filter (see exact_enqueue).
// XD: windows between an exact word's load and its test (1 or 2; 2 hides more L2 latency, 8 more registers).
template <int NW, bool OLT, bool XS = false, int XD = 1>
__global__ void __launch_bounds__(NW * 32, 1) ara_lane_kernel(const __grid_constant__ LayerParams p) {
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t fw = p.present_words;
  const uint32_t jpad = p.jpad;
  uint32_t bits_s;  // folded presence bitmap (shared address kept in a register, not rematerialised)
  asm volatile("mov.u32 %0, %1;" : "=r"(bits_s) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
  const uint32_t t1_w = (fw + 3u) & ~3u;                               // FT1 (R, L) pairs, 16-B aligned
  double2* s_t1 = reinterpret_cast<double2*>(smem + t1_w);
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t warp = __shfl_sync(FULL, threadIdx.x >> 5, 0);  // warp-uniform for the compiler
  const uint32_t base_s = (uint32_t)__cvta_generic_to_shared(smem + t1_w + jpad * 4u);
  // all warps' queues first (1 KB each, so every queue is 1 KB aligned and an entry address is an OR),
  // then the warps' record slots (512 B each)
  const uint32_t wq_s = ((base_s + 1023u) & ~1023u) + warp * (32u * kLaneQ * 4u);
  uint32_t q_l;  // entry j of this lane's queue: q_l + 128 j (one register: the OR with the entry offset)
  asm volatile("mov.u32 %0, %1;" : "=r"(q_l) : "r"(wq_s + 4u * lane));
  const uint32_t rec_l = ((base_s + 1023u) & ~1023u) + NW * (32u * kLaneQ * 4u) + warp * 512u + 16u * lane;

  for (uint32_t j = threadIdx.x; j < jpad; j += blockDim.x) s_t1[j] = make_double2(p.r1[j], p.l1[j]);
  for (uint32_t w = threadIdx.x; w < fw; w += blockDim.x) smem[w] = __ldg(p.present + w);
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
  const bool lane_last = 4u * lane < K - 128u * (nwin - 1u);  // this lane's slots lie in the last window
  const uint32_t last_valid = lane_last ? FULL : 0u;
  const uint32_t C = p.C;
  const uint32_t fmul = p.fold_mul;
  const uint32_t round_min = p.round_min;       // lanes with a queued hit that trigger a round
  const uint64_t pol_exact = make_policy(true, p.l2_hints);  // XS: the exact bitmap stays in L2

  // ---- per-lane queue state: tail/head count entries in units of 128 (the queue stride), so an
  // entry's address is q_l | (count & 0x380)
  uint32_t tail = 0, head = 0;
  uint32_t pb = 0;        // queued entries (at the head) that belong to the PREVIOUS trial
  uint32_t bx = 0;        // in-flight round: this lane's x = id - 1 (C: invalid), for rows read in full
                          // (XS: its compact record index)
  uint32_t bpar = 0;      // its trial parity
  uint32_t vmax = 0;      // max over popped x; x == C marks an invalid id
  bool inflight = false;  // a round's records are in flight (warp-uniform)
  bool bact = false;      // this lane's slot of the in-flight round holds a hit
  double S0 = 0.0, S1 = 0.0;  // per lane: partial sums of the open trials, by trial parity
  double M0 = 0.0, M1 = 0.0;  // OLT: largest occurrence-net loss of the open trials, by parity
  uint32_t curpar = 0;        // parity of the trial being scanned (warp-uniform)

  // Steps 1-3 for the in-flight round, accumulated by trial parity.
  auto consume = [&]() {
    if (!inflight) return;
    cp_async_wait_all();
    const uint4 r = lds_u128(rec_l);
    const uint32_t c1 = r.x & 0xffu, c2 = (r.x >> 8) & 0xffu, nz = (r.x >> 16) & 0xffu;
    double sum = 0.0;
    if (__any_sync(FULL, nz > 2u)) {  // rare: a row with more than two losses is read in full
      if (nz > 2u) {
        const float* row = p.table + (uint64_t)(XS ? r.w : bx + 1u) * jpad;  // r.w: the row's event id
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
    S0 += bpar ? 0.0 : o;                          // step 4 accumulation (x + 0 == x exactly)
    S1 += bpar ? o : 0.0;
    if constexpr (OLT) {
      if (bpar) M1 = o > M1 ? o : M1;
      else M0 = o > M0 ? o : M0;
    }
    inflight = false;
  };
  // One round: consume the in-flight records, then every lane with a queued hit pops one and requests
  // its record (lanes without one get a zero-filled slot: o = +0).
  auto round = [&]() {
    consume();
    const bool act = head != tail;
    const uint32_t x = lds_u32(q_l | (head & 0x380u));
    const bool isprev = pb != 0u;
    bpar = isprev ? (curpar ^ 1u) : curpar;
    if (act) {
      head += 128u;
      pb -= isprev ? 1u : 0u;
      vmax = max(vmax, x);  // XS: x is a compact record index, rec_zero only for an invalid id
    }
    bact = act;
    if constexpr (XS) {  // x: the compact record index (rec_zero: the zero record)
      bx = act ? x : p.rec_zero;
      cp_async16_zf(rec_l, p.rec_c + bx, act ? 16u : 0u);
    } else {
      bx = act ? x : C;
      cp_async16_zf(rec_l, p.rec + (bx + 1u), act ? 16u : 0u);  // x + 1 = the id; C + 1: the zero record
    }
    cp_async_commit();
    inflight = true;
  };
  // Close the trial of parity `par` (index t0 + kc): fixed tree, FT3, one store.
  auto close = [&](uint32_t par, uint32_t kc) {
    double Sv = par ? S1 : S0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) Sv += __shfl_xor_sync(FULL, Sv, off);
    if (lane == 0) p.ylt[t0 + (uint64_t)kc * tstep] = clamp_terms(Sv, p.r3, p.l3);  // step 4: FT3 on S_n
    if constexpr (OLT) {
      double M = par ? M1 : M0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, off));
      if (lane == 0) p.olt[t0 + (uint64_t)kc * tstep] = M;
      if (par) M1 = 0.0; else M0 = 0.0;
    }
    if (par) S1 = 0.0; else S0 = 0.0;
  };
  // Scan one window: presence test per id, hits appended to the lane's own queue.
  // XS: the previous window's candidates (x, exact word; a non-candidate holds word 0); with XD == 2 also
  // the window before it (qx*, qw*), tested first
  const uint2 z2 = make_uint2(0u, 0u);
  uint32_t px0 = 0, px1 = 0, px2 = 0, px3 = 0, qx0 = 0, qx1 = 0, qx2 = 0, qx3 = 0;
  uint2 pw0 = z2, pw1 = z2, pw2 = z2, pw3 = z2, qw0 = z2, qw1 = z2, qw2 = z2, qw3 = z2;
  // a candidate's rank entry: word (x + 1) >> 5; an invalid id (x = C) reads the sentinel bit C + 1,
  // whose rank is rec_zero (no row holding a loss lies after it).  Predicated, no branch.
  const uint2* const xr = p.xrank;
  auto exact_load = [&](uint32_t cand, uint32_t x) -> uint2 {
    uint2 w = z2;
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n"
        " @q ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%3], %4;\n}\n"
        : "+r"(w.x), "+r"(w.y)
        : "r"(cand), "l"(xr + ((x + 1u) >> 5)), "l"(pol_exact));
    return w;
  };
  auto flush_oldest = [&]() {  // XS: the oldest pending window's exact hits enter the queue (slot order)
    if constexpr (XD == 2) {
      exact_enqueue(qw0, qx0, q_l, tail);
      exact_enqueue(qw1, qx1, q_l, tail);
      exact_enqueue(qw2, qx2, q_l, tail);
      exact_enqueue(qw3, qx3, q_l, tail);
      qx0 = px0; qx1 = px1; qx2 = px2; qx3 = px3;
      qw0 = pw0; qw1 = pw1; qw2 = pw2; qw3 = pw3;
    } else {
      exact_enqueue(pw0, px0, q_l, tail);
      exact_enqueue(pw1, px1, q_l, tail);
      exact_enqueue(pw2, px2, q_l, tail);
      exact_enqueue(pw3, px3, q_l, tail);
    }
    pw0 = pw1 = pw2 = pw3 = z2;
  };
  // XS: every pending window, oldest first.  A window adds up to 4 entries per lane and a queue holds 8, so
  // with two pending windows the queue must be drained to <= 4 entries between them (without this a lane
  // could overflow its queue at a trial's end and lose a hit: measured on config X's real-regime YLT)
  auto drain_to_4 = [&]() {
    while (__any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u)) round();
  };
  auto flush_pending = [&]() {
    flush_oldest();
    if constexpr (XD == 2) {
      drain_to_4();
      flush_oldest();
    }
  };
  auto scan = [&](const uint4 v, uint32_t valid) {
    if constexpr (XS) {
      flush_oldest();
      uint32_t c;
      c = fold_candidate(v.x, C, fmul, bits_s, valid, px0);
      pw0 = exact_load(c, px0);
      c = fold_candidate(v.y, C, fmul, bits_s, valid, px1);
      pw1 = exact_load(c, px1);
      c = fold_candidate(v.z, C, fmul, bits_s, valid, px2);
      pw2 = exact_load(c, px2);
      c = fold_candidate(v.w, C, fmul, bits_s, valid, px3);
      pw3 = exact_load(c, px3);
    } else {
      test_enqueue(v.x, C, fmul, bits_s, valid, q_l, tail);
      test_enqueue(v.y, C, fmul, bits_s, valid, q_l, tail);
      test_enqueue(v.z, C, fmul, bits_s, valid, q_l, tail);
      test_enqueue(v.w, C, fmul, bits_s, valid, q_l, tail);
    }
    // rounds: enough lanes hold a hit, or a queue could overflow in the next window (<= 4 more; a queue
    // of 8 entries takes them while it holds <= 4).  One call site, so one copy of the round's code.
    bool go = __any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u) ||
              (uint32_t)__popc(__ballot_sync(FULL, tail != head)) >= round_min;
    while (go) {
      round();
      go = __any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u);
    }
  };

  // Window loop: one scan site (the window's successor is requested first -- the next window of the
  // trial, or the first window of the warp's next trial after the lane-masked tail window -- and the
  // buffers are rotated by moves), so the hot code stays small.
  const uint32_t* lp = p.ids + t0 * K + 4u * lane;  // this lane's slots of the trial's first window
  const uint64_t tstride = tstep * K;
  uint4 A = make_uint4(0u, 0u, 0u, 0u);
  if (nwin > 1u || lane_last) A = ld_ids4_stream(lp);
  for (uint32_t k = 0; k < nt; ++k) {
    // ---- trial start: trial k-2 (parity k & 1) must be complete -- no queued or in-flight hit of it
    // -- before its parity is reused; close it, then every queued hit belongs to trial k-1
    if (k >= 2u) {
      while (__any_sync(FULL, pb != 0u || (inflight && bact && bpar == (k & 1u)))) round();
      close(k & 1u, k - 2u);
    }
    pb = (tail - head) >> 7;
    curpar = k & 1u;
    if (p.prefetch && lane == 0 && k + 2u < nt) prefetch_l2_bulk(lp + 2u * tstride - 4u * lane, K * 4u);
    for (uint32_t w = 0; w < nwin; ++w) {
      const bool last = w + 1u == nwin;
      const uint32_t* nx = last ? lp + tstride : lp + 128u * (w + 1u);
      const bool ok = last ? (k + 1u < nt && (nwin > 1u || lane_last)) : (w + 2u < nwin || lane_last);
      uint4 nxt = A;
      if (ok) nxt = ld_ids4_stream(nx);
      scan(A, last ? last_valid : FULL);
      A = nxt;
    }
    lp += tstride;
    if constexpr (XS) {  // the trial's last window: its exact hits before the trial boundary
      flush_pending();
      while (__any_sync(FULL, tail - head >= (kLaneQ - 3u) * 128u)) round();
    }
  }
  // ---- drain every queue, then close the (at most two) open trials
  while (__any_sync(FULL, tail != head)) round();
  consume();
  if (nt >= 2u) close((nt - 2u) & 1u, nt - 2u);
  close((nt - 1u) & 1u, nt - 1u);
  const bool bad = __any_sync(FULL, vmax >= (XS ? p.rec_zero : C));
  if (lane == 0 && bad) atomicOr(p.err, 1u);
}

}  // namespace ara

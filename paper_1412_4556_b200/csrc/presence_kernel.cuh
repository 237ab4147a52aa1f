// presence_kernel.cuh -- the default ARA hot path on sm_100a: the same direct-access interleaved table as
// ara_layer_kernel, plus a per-layer PRESENCE bitmap (bit e set iff row e of the table holds a non-zero
// loss).  Most event rows are all zero (990,000 of 1,000,000 entries of an ELT; 92% of
// the rows of the paper-shaped layer), and an all-zero row contributes exactly +0 to every sum (reading
// c9), so only rows whose bit is set are gathered.  The bitmap lives in SHARED memory (one copy per SM,
// folded modulo its capacity when C+1 exceeds it -- folding only adds false positives, i.e. gathers of
// rows that turn out to be zero, never misses), so the per-occurrence test costs one LDS instead of a
// 64-B gather.  The kernel is then bound by instruction issue (P) or by the record gathers (X).
//
//   * one warp per trial (persistent grid); the warp streams the trial's ids in 128-id windows, each lane
//     one 16-B vector (L1::no_allocate), one window requested ahead in registers; the trial's first window
//     is requested before the per-trial bookkeeping and its last (partial) window is lane-masked inside
//     the same loop, so no load sits on the critical path;
//   * per window: bitmap test per id (the folded word's bit, a sentinel bit for invalid ids), one ballot
//     per pair of slots appends the hits to a linear per-warp queue in shared memory;
//   * whenever 32 hits are queued the warp consumes the previous batch and issues the next: with one lane
//     per row (G == 1, the default for every width) each lane cp.asyncs its event's 16-B sparse record
//     (first two non-zero columns; rows with more are read in full), applies FT1 in fp64 to those losses,
//     sums them, applies FT2 and accumulates the occurrence-net loss of the trial that owns the hit
//     (steps 1-3); G > 1 variants gather full rows round by round;
//   * the queue is carried across the warp's trials; a trial is finalized lazily -- when the trial that
//     reuses its parity slot starts, or at the end -- by a fixed rotation + xor-tree of the lanes' sums,
//     then FT3 on S_n (step 4) and one 8-B YLT store.
#pragma once
#include "ara_kernel.cuh"

namespace ara {

constexpr int kQueue = 160;  // per-warp queue of pending hits (<= 31 left over + <= 128 new per window)

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
                                              int n, int lane, uint64_t pol_tab) {
    const int g = lane % G;
    const int slot = r * RG + lane / G;
    // queue word = event id; an invalid id (0 or > C, queued through the sentinel bit and reported by
    // the kernel) fetches the zero row 0 instead
    uint32_t id = slot < n ? q[slot] : 0u;
    id = id <= p.C ? id : 0u;
    const float* row = p.table + (uint64_t)id * (V * NV);
    float(&xr)[NVL][V] = x[kAsync ? r : 0];
#pragma unroll
    for (int i = 0; i < NVL; ++i) {
      const int s = g + i * G;
      if (NV % G == 0 || s < NV) {  // empty slots fetch row 0, a real all-zero row
        ld_row<V>(row + s * V, pol_tab, xr[i]);
      } else {
#pragma unroll
        for (int c = 0; c < V; ++c) xr[i][c] = 0.0f;
      }
    }
  }

  __device__ __forceinline__ void consume_round(int r, const LayerParams& p, int lane, const double* s_r1,
                                                const double* s_l1, double& S, double& M) const {
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
        sum += clamp_fast((double)xr[i][c], s_r1[j], s_l1[j]);
      }
    if constexpr (G > 1) {
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
    }
    if (g == 0) {  // step 3 (FT2); step 4 accumulation (exact +0 if sum 0)
      const double o = clamp_fast(sum, p.r2, p.l2);
      S += o;
      M = o > M ? o : M;
    }
  }

  // G == 1 only: occurrence-net loss o = FT2(sum_j FT1(x_j)) of the lane's own row (slot = lane).
  __device__ __forceinline__ double row_loss(const LayerParams& p, const double* s_r1, const double* s_l1) const {
    double sum = 0.0;
#pragma unroll
    for (int i = 0; i < NVL; ++i)
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int j = i * V + c;
        sum += clamp_fast((double)x[0][i][c], s_r1[j], s_l1[j]);  // steps 1-2
      }
    return clamp_fast(sum, p.r2, p.l2);  // step 3 (exactly +0 for an all-zero row)
  }

  // Async: issue all rounds now, consume later.  Sync: issue+consume round by round.
  __device__ __forceinline__ void issue(const LayerParams& p, const uint32_t* __restrict__ q, int n, int lane,
                                        uint64_t pol_tab, const double* s_r1, const double* s_l1, double& S,
                                        double& M) {
#pragma unroll
    for (int r = 0; r < G; ++r) {
      if (r * RG >= n) break;  // warp-uniform
      issue_round(r, p, q, n, lane, pol_tab);
      if constexpr (!kAsync) consume_round(r, p, lane, s_r1, s_l1, S, M);
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
                                          double& S, double& M) const {
    if constexpr (kAsync) {
#pragma unroll
      for (int r = 0; r < G; ++r) consume_round(r, p, lane, s_r1, s_l1, S, M);
    }
  }
};

// One lane per row (G == 1, any row width): the batch holds each queued event's 16-byte sparse
// RECORD instead of its full row.  Typically a present row has a single non-zero loss (the ELTs are
// sparse and nearly disjoint), so steps 1-3 cost two FT1 clamps and one FT2 clamp per row; a row with
// more than two losses (rare) is read in full from the table.  The sum runs over the non-zero columns
// in layer order, i.e. the oracle's order with its exact +0 terms dropped.  The records travel by
// cp.async into the warp's shared slots, so no registers are held while the warp scans on.
template <int V, int NV>
struct RecBatch {
  static constexpr bool kAsync = true;

  // lane -> slot `lane` of the warp's record buffer (rec_s: its 32-bit shared address)
  __device__ __forceinline__ void issue(const LayerParams& p, const uint32_t* __restrict__ q, int n, int lane,
                                        uint64_t pol_tab, uint32_t rec_s) const {
    const uint32_t e = lane < n ? q[lane] : 0u;
    const uint32_t id = e <= p.C ? e : 0u;  // invalid ids (reported by the kernel) read the zero record of row 0
    cp_async16(rec_s + 16u * (uint32_t)lane, p.rec + id, pol_tab);
    cp_async_commit();
  }

  // occurrence-net loss o = FT2(sum_j FT1(x_j)) of the lane's queued event
  // s_t1: the FT1 terms as (retention, limit) pairs, one 16-B shared load per column
  __device__ __forceinline__ double row_loss(const LayerParams& p, const double* s_r1, const double* s_l1,
                                             const double2* s_t1, uint64_t pol_tab, uint32_t rec_s, int lane) const {
    cp_async_wait_all();
    const uint4 r = lds_u128(rec_s + 16u * (uint32_t)lane);
    const uint32_t c1 = r.x & 0xffu, c2 = (r.x >> 8) & 0xffu, nz = (r.x >> 16) & 0xffu;
    double sum = 0.0;
    if (__any_sync(0xffffffffu, nz > 2u)) {  // rare: some row of the batch has more than two losses
      if (nz > 2u) {
        constexpr int JP = V * NV;
        const float* row = p.table + (uint64_t)r.w * JP;  // r.w: the record's own event id
#pragma unroll(NV <= 2 ? NV : 1)  // wide rows: one vector at a time (registers)
        for (int i = 0; i < NV; ++i) {
          float x[V];
          ld_row<V>(row + i * V, pol_tab, x);
#pragma unroll
          for (int c = 0; c < V; ++c) sum += clamp_fast((double)x[c], s_r1[i * V + c], s_l1[i * V + c]);
        }
      }
    }
    if (nz <= 2u) {
      // absent columns hold loss 0: clamp(0; R >= 0, L) = +0 exactly, so n < 2 needs no branch
      const double2 ta = s_t1[c1], tb = s_t1[c2];
      sum += clamp_fast((double)__uint_as_float(r.y), ta.x, ta.y);  // steps 1-2: FT1, sum over ELTs
      sum += clamp_fast((double)__uint_as_float(r.z), tb.x, tb.y);
    }
    return clamp_fast(sum, p.r2, p.l2);  // step 3: FT2 (exactly +0 for an empty record)
  }
};

// SURVEY N3 (precombined occurrence-net event table, an ablation): steps 1-3 depend only on the event,
// so ara_create may tabulate o[e] = FT2(sum_j FT1(l_ej)) per layer (fp64, summed in layer order like the
// oracle, so bitwise equal to the record path); a hit then moves one 8-B value and does no FT1/FT2
// work.  Exact for the deterministic method only (secondary uncertainty, would vary the
// losses per occurrence), and it performs no ELT lookups at run time -- reported separately.
struct OccBatch {
  static constexpr bool kAsync = true;
  __device__ __forceinline__ void issue(const LayerParams& p, const uint32_t* __restrict__ q, int n, int lane,
                                        uint64_t, uint32_t rec_s) const {
    const uint32_t e = lane < n ? q[lane] : 0u;
    cp_async8(rec_s + 16u * (uint32_t)lane, p.occ + (e <= p.C ? e : 0u));  // o[0] = +0
    cp_async_commit();
  }
  __device__ __forceinline__ double row_loss(const LayerParams&, const double*, const double*, const double2*,
                                             uint64_t, uint32_t rec_s, int lane) const {
    cp_async_wait_all();
    double o;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(o) : "r"(rec_s + 16u * (uint32_t)lane) : "memory");
    return o;
  }
};

template <int V, int NV, int G, bool kRec, bool kOcc = false>
struct BatchOf {  // G > 1: full-row batches (round by round for wide rows)
  using type = RowBatch<V, NV, G>;
};
template <int V, int NV>
struct BatchOf<V, NV, 1, true, false> {
  using type = RecBatch<V, NV>;
};
template <int V, int NV>
struct BatchOf<V, NV, 1, true, true> {
  using type = OccBatch;
};

// Per-warp bookkeeping of the (at most two) trials whose hits are still in flight (carried queue).
struct WarpTrials {
  uint64_t trial[2];  // trial index per parity slot
  uint32_t first[2];  // stream position of the trial's first hit
  uint32_t end[2];    // stream position one past its last hit (valid once its scan is done)
  uint32_t state[2];  // 0 free, 1 scanning, 2 scanned (waiting for its hits to be consumed)
  uint32_t bad;
  uint32_t cur;       // parity of the most recently started trial
};

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

// V/NV: row format (as ara_layer_kernel); G: lanes per row in a batch; NW: warps per block.
//
// Presence test.  The shared bitmap is the layer's presence bitmap FOLDED to the words that fit: event
// id e (x = e - 1) maps to bit x & 31 of word umulhi(x, fold_mul); fold_mul = 2^27 (no folding: word
// x >> 5) or smaller, so neighbouring blocks of ids share words.  Folding only adds false positives
// (gathers of all-zero rows, exact +0), never misses.  Any invalid id (0 or > C) clamps to x = C, whose
// SENTINEL bit is always set, so invalid ids are queued like hits and reported when their batch is
// issued: the scan itself needs no validity check.
//
// Hits are queued as raw event ids and, with one lane per row (G == 1), the queue is CARRIED across the warp's
// consecutive trials: batches are always full (32 rows) except when the queue must be flushed, so the
// per-trial partial batch disappears.  A queued hit's trial follows from its stream position (each open
// trial owns [first, end)).  The occurrence-net loss of the i-th hit of a trial is always accumulated by
// lane i mod 32 (a shuffle rotates each batch into that frame), and the lanes are combined by the same
// xor-tree -- so a trial's fp64 summation order depends only on its own ids, never on its neighbours,
// the sharding or the launch shape.
// OLT: also track the largest occurrence-net loss per trial (ara_run_ex); a separate instantiation so
// the plain YLT path carries no extra registers.
// FX (one lane per row only): EXACT filter stage for layers whose sparse records do not stay in L2.  A
// batch of queued candidates first loads, per lane, the word of the layer's unfolded presence bitmap
// (global memory, (C+1) bits, L2-resident) that holds its event; one batch later only the candidates
// whose exact bit is set fetch their record, the others (false positives of the fold) get a zero record
// in shared memory.  A zero record gives o = +0, exactly what their own (zero) record gave, so the results
// are bitwise identical with and without FX; only the records' DRAM traffic changes.  Measured on config
// X (B200): DRAM traffic 301 -> 74 GB per 8M trials, but 6.6 instead of 5.9 ms per 1M trials (the extra
// L2 round trip per batch and its shared-memory dependencies), so it is an option, off by default.
// PC: SURVEY N3 ablation -- batches gather the precombined o[e] (OccBatch) instead of records.
template <int V, int NV, int G, int NW, bool OLT, bool FX = false, bool PC = false>
__global__ void __launch_bounds__(NW * 32, 1) ara_presence_kernel(const __grid_constant__ LayerParams p) {
  constexpr int JP = V * NV;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr bool kCarry = (G == 1);  // one lane per row: sparse records + carried queue (any row width)
  static_assert(!FX || kCarry, "the exact filter stage needs record batches");
  static_assert(!PC || (kCarry && !FX), "the precombined table replaces the record batches");
  using Batch = typename BatchOf<V, NV, G, kCarry, PC>::type;
  extern __shared__ uint32_t smem[];
  // FT1 terms, padded to the G*NVL*V columns a row group covers (padding: R = 0, L = +inf, so the
  // branch-free FT1 of a padding column -- always loss 0 -- is exactly +0).
  constexpr int JPS = G * ((NV + G - 1) / G) * V;
  __shared__ double s_r1[JPS], s_l1[JPS];
  __shared__ double2 s_t1[kCarry ? JPS : 1];  // record batches: FT1 as (R, L) pairs, one 16-B load per column
  __shared__ WarpTrials s_wt[NW];
  uint32_t* bits = smem;  // [present_words], already folded by the host (fold_mul)
  uint32_t bits_s;        // its shared address, kept in a register (not rebuilt from the CTA id per window)
  asm volatile("mov.u32 %0, %1;" : "=r"(bits_s) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // provably warp-uniform for ptxas
  const int lane = threadIdx.x & 31;
  uint32_t* q = smem + p.present_words + warp * kQueue;
  WarpTrials& wt = s_wt[warp];
  const uint32_t q_s = (uint32_t)__cvta_generic_to_shared(q);  // 32-bit shared addresses
  // record slots (G == 1): 32 x 16 B per warp after the queues, 16-B aligned
  const uint32_t rec_s = (((uint32_t)__cvta_generic_to_shared(smem + p.present_words + NW * kQueue) + 15u) & ~15u) +
                         (uint32_t)warp * 512u;

  for (int j = threadIdx.x; j < JPS; j += blockDim.x) {
    s_r1[j] = j < JP ? p.r1[j] : 0.0;
    s_l1[j] = j < JP ? p.l1[j] : __longlong_as_double(0x7ff0000000000000ll);
    if constexpr (kCarry) s_t1[j] = make_double2(s_r1[j], s_l1[j]);
  }
  for (uint32_t w = threadIdx.x; w < p.present_words; w += blockDim.x) bits[w] = __ldg(p.present + w);
  if (lane == 0) {
    wt.state[0] = wt.state[1] = 0u;
    wt.bad = 0u;
    wt.cur = 0u;
  }
  __syncthreads();

  const uint64_t pol_tab = make_policy(true, p.l2_hints);
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(p.ids) & 15u) == 0);
  const uint32_t C = p.C;
  const uint32_t fmul = p.fold_mul;
  const unsigned lt = lanemask_lt();

  double S0 = 0.0, S1 = 0.0;  // per-lane partial sums of the (<= 2) open trials, by parity
  double M0 = 0.0, M1 = 0.0;  // per-lane largest occurrence-net loss of those trials (OLT)
  constexpr bool want_olt = OLT;
  // The warp's queue is linear: the unissued hits are q[0 .. count), qt = q_s + 4 * count is the shared
  // address of the next free slot; issuing a batch takes q[0 .. n) and moves the rest down.
  uint32_t qt = q_s;
  uint32_t issued = 0;           // stream position of the next hit to issue
  Batch rows;
  uint32_t bstart = 0;           // pending batch: stream position of slot 0
  int bn = 0;                    // pending batch size (0 = none)
  uint32_t f_id = 0, f_w = 0;    // FX: this lane's candidate of the filter batch and its exact bitmap word
  uint32_t fstart = 0;           // FX: stream position of the filter batch's slot 0
  int fn = 0;                    // FX: filter batch size (0 = none)
  unsigned bad = 0;

  // FT3 on the warp-combined sum of parity slot a; lane 0 writes the YLT.
  auto finalize = [&](int a) {
    double S = (kCarry && a) ? S1 : S0;
    // lane L holds the trial's hits i = L - first (mod 32) (batches start at multiples of 32 in the
    // stream); rotate into the canonical frame (lane c: hits i = c mod 32) before the fixed xor-tree
    if constexpr (kCarry) S = __shfl_sync(FULL, S, (lane + (int)wt.first[a]) & 31);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(FULL, S, off);
    if (lane == 0) p.ylt[wt.trial[a]] = clamp_terms(S, p.r3, p.l3);  // step 4: aggregate terms FT3
    if constexpr (OLT) {  // the trial's largest occurrence-net loss (order-free, exact)
      double M = (kCarry && a) ? M1 : M0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, off));
      if (lane == 0) p.olt[wt.trial[a]] = M;
    }
    if (kCarry && a) {
      S1 = 0.0;
      M1 = 0.0;
    } else {
      S0 = 0.0;
      M0 = 0.0;
    }
    __syncwarp();
    if (lane == 0) wt.state[a] = 0u;
    __syncwarp();
  };
  // Finalize every scanned trial whose hits have all been consumed (stream position `done`).
  auto settle = [&](uint32_t done) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
      if (wt.state[a] == 2u && (int32_t)(done - wt.end[a]) >= 0) finalize(a);
  };
  // Consume the pending batch: FT1/FT2 per row, accumulated per trial.
  auto consume = [&]() {
    if (bn != 0) {
      if constexpr (kCarry) {
        const double o = rows.row_loss(p, s_r1, s_l1, s_t1, pol_tab, rec_s, lane);
        // Batch lane L holds stream position bstart + L (bstart is a multiple of 32).  A queued hit
        // belongs to the most recently started trial (parity wt.cur) if it lies at or after that
        // trial's first hit, else to its predecessor (the other parity): the trial before that was
        // fully consumed when the current one started.  Each lane accumulates its own hits: no
        // shuffles per batch (finalize rotates once per trial).
        const uint32_t cp = wt.cur;
        const bool newer = (int32_t)(bstart + (uint32_t)lane - wt.first[cp]) >= 0;
        const bool in0 = newer == (cp == 0u);
        if (lane < bn) {
          if (in0) S0 += o; else S1 += o;
          if (want_olt) {  // the maximum needs no canonical order
            if (in0) M0 = o > M0 ? o : M0;
            else M1 = o > M1 ? o : M1;
          }
        }
      } else {
        rows.consume(p, lane, s_r1, s_l1, S0, M0);
      }
      bn = 0;
    }
    // one lane per row: trials are finalized lazily (at the start of the trial that reuses their parity,
    // or at the end), not after every batch
    if constexpr (!kCarry) settle(issued);
  };
  // Issue the next n (<= 32) queued hits as a batch (consuming the previous batch first).
  auto issue = [&](int n) {
    consume();
    __syncwarp();
    if constexpr (FX) {  // filter batch -> record batch: records only for exact hits
      if (fn != 0) {
        const uint32_t xe = f_id;  // 0 for empty slots and invalid ids
        const bool tp = (f_w >> (xe & 31u)) & 1u;
        if (tp) {
          cp_async16(rec_s + 16u * (uint32_t)lane, p.rec + xe, pol_tab);
        } else {  // (fetching row 0's zero record instead makes one L2 sector a hot spot: 15x slower on X)
          asm volatile("st.shared.v4.u32 [%0], {%1,%1,%1,%1};" :: "r"(rec_s + 16u * (uint32_t)lane), "r"(0u) : "memory");
        }
        cp_async_commit();
        bstart = fstart;
        bn = fn;
        fn = 0;
      }
      if (n == 0) return;  // flush: nothing left to take from the queue
    }
    const uint32_t count = (qt - q_s) >> 2;
    const uint32_t e = lane < n ? q[lane] : 1u;
    bad |= (e - 1u >= C) ? 1u : 0u;  // an invalid id reached the queue through the sentinel bit
    if constexpr (FX) {  // queue -> filter batch: load the exact presence words (used one batch later)
      f_id = (lane < n && e - 1u < C) ? e : 0u;
      f_w = f_id != 0u ? ld_id(p.exact + (f_id >> 5), pol_tab) : 0u;
    } else if constexpr (kCarry) {
      rows.issue(p, q, n, lane, pol_tab, rec_s);
    } else {
      rows.issue(p, q, n, lane, pol_tab, s_r1, s_l1, S0, M0);
    }
    __syncwarp();  // every lane has read its batch slots
    for (uint32_t i = (uint32_t)lane; i + (uint32_t)n < count; i += 32u) q[i] = q[i + n];  // n == 32 here
    __syncwarp();
    if constexpr (FX) {
      fstart = issued;
      fn = n;
    } else {
      bstart = issued;
      bn = n;
    }
    issued += 32u;  // a partial batch skips the rest of its 32 stream positions: batches stay 32-aligned
    qt -= 4u * (uint32_t)n;
    if constexpr (!kCarry) consume();  // wide rows: rows.issue already consumed round by round
  };
  auto flush = [&]() {
    while (qt != q_s) {
      const uint32_t count = (qt - q_s) >> 2;
      issue(count < 32 ? (int)count : 32);
    }
    if constexpr (FX) {
      if (fn != 0) issue(0);  // the filter batch becomes the record batch
    }
    consume();
  };
  // Scan one window: lane l holds window positions 4l .. 4l+3 (ids v); CHECKED windows mask positions
  // outside the trial (r = window position of id 0 relative to the trial start, len = trial length).
  // `valid`: all ones, or 0 for a lane whose 4 slots all lie outside the trial (lane-masked tail).
  auto scan = [&](const uint4 v, auto checked, uint32_t r, uint32_t len, uint32_t valid) {
    const uint32_t id[4] = {v.x, v.y, v.z, v.w};
    uint32_t x[4], wd[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x[u] = min(id[u] - 1u, C);          // invalid ids -> the sentinel bit C
      wd[u] = lds_ro_u32(bits_s + 4u * __umulhi(x[u], fmul));  // the folded bitmap word holding bit x & 31
      if constexpr (decltype(checked)::value) wd[u] = (r + (uint32_t)u < len) ? wd[u] : 0u;  // outside the trial
    }
    // Append the hits in a fixed order that depends only on the window: per pair of slots, first the
    // lanes' first hit of the pair (lanes ascending), then -- only if some lane hit both -- the
    // second ids of those lanes.  One ballot per pair instead of one per slot.
    pair_insert(wd[0], x[0], id[0], wd[1], x[1], id[1], lt, qt, valid);
    pair_insert(wd[2], x[2], id[2], wd[3], x[3], id[3], lt, qt, valid);
    // warp-uniform; at most 31 + 128 = 159 < kQueue queued
    while (qt - q_s >= 128u) issue(32);
  };

  uint32_t k = 0;  // local trial counter (parity = k & 1)
  for (uint64_t t = (uint64_t)blockIdx.x * NW + warp; t < p.num_trials; t += (uint64_t)gridDim.x * NW, ++k) {
    const int par = (int)(k & 1u);
    uint64_t b, e;
    if (p.offsets) {
      b = __shfl_sync(FULL, p.offsets[t], 0);  // warp-uniform (every lane loaded the same value)
      e = __shfl_sync(FULL, p.offsets[t + 1], 0);
      if (e < b || e > p.num_events) {
        bad |= 2u;
        e = b;
      }
    } else {
      b = t * p.K;
      e = b + p.K;
    }
    const uint32_t len = (uint32_t)(e - b);
    const bool vec = vec_ok && ((b & 3u) == 0);
    // the trial's first full window is requested before the bookkeeping below, so its latency overlaps it
    // aligned trial whose length is a multiple of 4: every window is whole 16-B vectors, the last one
    // lane-masked (lanes past the end keep stale ids that their mask hides)
    const bool valn = vec && (len & 3u) == 0u;
    uint4 wfirst = make_uint4(0u, 0u, 0u, 0u);
    if (valn && 4u * (uint32_t)lane < len) wfirst = ld_ids4_stream(p.ids + b + 4u * (uint32_t)lane);
    if (wt.state[par] != 0u) {  // trial k-2 is not finalized yet
      // first stream position not consumed yet
      const uint32_t done = bn != 0 ? bstart : ((FX && fn != 0) ? fstart : issued);
      if (wt.state[par] == 2u && (int32_t)(done - wt.end[par]) >= 0) {
        finalize(par);  // all its hits are consumed
      } else {
        flush();  // trial k-2 still has hits in flight
        for (int a = 0; a < 2; ++a)
          if (wt.state[a] == 2u) finalize(a);
      }
    }
    __syncwarp();
    if (lane == 0) {  // warp-uniform bookkeeping in shared memory (one writer, then a warp barrier)
      wt.cur = (uint32_t)par;
      wt.trial[par] = t;
      wt.first[par] = issued + ((qt - q_s) >> 2);  // stream position of the trial's first hit
      wt.state[par] = 1u;
    }
    __syncwarp();

    // Bring this warp's NEXT trial into L2 (lane l prefetches its 128-B line l: the first 4 KB), so its
    // windows arrive at L2 latency: one window of register prefetch cannot cover DRAM latency.
    if (p.prefetch) {
      const uint64_t tn = t + (uint64_t)gridDim.x * NW;
      if (tn < p.num_trials) {
        const uint64_t nb = p.offsets ? p.offsets[tn] : tn * p.K;
        const uint64_t ne = p.offsets ? p.offsets[tn + 1] : nb + p.K;
        const uint64_t g = nb + 32u * (uint32_t)lane;  // id index of this lane's line
        if (g < ne && g < p.num_events) prefetch_l2_line(p.ids + g);
      }
    }
    // Windows of 128 ids from the trial's first occurrence (so the order in which a trial's hits are
    // queued depends only on the trial itself): lane l holds window positions 4l .. 4l+3.  When the
    // trial start is 16-B aligned, full windows are single 16-B vectors streamed through a running
    // per-lane pointer with no checks, one window held ahead in registers; the last partial window (or
    // an unaligned trial) goes through the checked loader.
    const uint32_t nwin = (len + 127u) / 128u;
    auto load_checked = [&](uint32_t w) -> uint4 {
      const uint32_t r = w * 128u + 4u * lane;  // trial position of this lane's first slot
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (vec && r + 4u <= len) return ld_ids4_stream(p.ids + b + r);
      if (r < len) v.x = ld_id_stream(p.ids + b + r);
      if (r + 1u < len) v.y = ld_id_stream(p.ids + b + r + 1);
      if (r + 2u < len) v.z = ld_id_stream(p.ids + b + r + 2);
      if (r + 3u < len) v.w = ld_id_stream(p.ids + b + r + 3);
      return v;
    };
    auto rel0 = [&](uint32_t w) -> uint32_t { return w * 128u + 4u * (uint32_t)lane; };
    if (valn) {
      // windows streamed through a running per-lane pointer, one window held ahead in registers (two
      // register sets, unrolled); window w covers trial positions r .. r+3 of this lane, r = 128 w + 4 l
      if (nwin != 0u) {
        const uint32_t* lpp = p.ids + b + 4u * (uint32_t)lane;
        uint32_t r = 4u * (uint32_t)lane;
        uint4 wa = wfirst, wb = wfirst;
        uint32_t rem = nwin - 1u;  // windows after the one in wa
        bool ok_a = r < len, ok_b;
        while (true) {
          ok_b = r + 128u < len;
          if (rem != 0u && ok_b) wb = ld_ids4_stream(lpp + 128);
          scan(wa, BoolC<false>{}, 0u, 0u, ok_a ? 0xffffffffu : 0u);
          if (rem == 0u) break;
          --rem;
          lpp += 256;
          r += 256u;
          ok_a = r < len;
          if (rem != 0u && ok_a) wa = ld_ids4_stream(lpp);
          scan(wb, BoolC<false>{}, 0u, 0u, ok_b ? 0xffffffffu : 0u);
          if (rem == 0u) break;
          --rem;
        }
      }
    } else {
      for (uint32_t w = 0; w < nwin; ++w) scan(load_checked(w), BoolC<true>{}, rel0(w), len, 0xffffffffu);  // unaligned trial
    }
    __syncwarp();
    if (lane == 0) {
      wt.end[par] = issued + ((qt - q_s) >> 2);
      wt.state[par] = 2u;
    }
    __syncwarp();
    if (!kCarry) flush();  // full-row batches: one trial at a time (finalized by the flush's settle)
  }
  flush();
  // every hit is consumed now: finalize the (at most two) trials still open
  for (int a = 0; a < 2; ++a)
    if (wt.state[a] == 2u) finalize(a);
  bad = __reduce_or_sync(FULL, bad);
  if (lane == 0 && bad) atomicOr(p.err, bad);
}

}  // namespace ara

// ara_kernel.cuh -- the ARA hot path on sm_100a: YET stream -> direct-access row gather -> FT1 / sum /
// FT2 -> per-trial cumulative sum -> FT3 -> YLT.  One launch per layer (Algorithm 1 is layer-outer,
// PAPER.md:104-105).
//
// Mapping (B200-first, not the paper's one-thread-per-trial of PAPER.md:199):
//   * one WARP per trial, persistent grid-stride loop over trials;
//   * the warp is split into RG = 32/G row groups of G lanes; a row group owns one event occurrence
//     at a time and its G lanes fetch that event's table row together (row = the event's losses in
//     all J ELTs of the layer, event-major interleaved: "ELTs combined as a single
//     table"), each lane one V-float vector (V = 8 -> one 256-bit LDG = one 32-B sector);
//     so a 64-B row (J = 16) is one L1 wavefront for 2 lanes instead of 2 wavefronts for 1 lane;
//   * each row group handles U occurrences per iteration, so a warp has 32/G*U rows in flight;
//   * FT1 is applied in fp64 only to entries whose fp32 loss is non-zero: an absent event has loss 0
//     and clamp(0; R>=0, L) = +0 exactly (reading c9), so skipping it is exact, not an approximation;
//   * the per-row partial sums of the G lanes are combined with xor-shuffles, FT2 is applied, and the
//     group leader accumulates the occurrence-net loss; the trial's cumulative sum S_n is the
//     warp-shuffle sum of the leaders' running sums (the YLT needs only the last prefix);
//   * terms (FT1 per ELT, FT2, FT3) arrive as kernel parameters -- the constant bank, as the paper
//     keeps terms in constant memory; FT1 is staged into shared memory so a lane can
//     index it by its entry.
// Cache policy: table rows are loaded L1::no_allocate with an L2 evict_last policy (the table is the
// re-used working set); YET ids are streamed with an L2 evict_first policy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ara {

constexpr int kMaxJ = 128;  // ARA_MAX_ELTS_PER_LAYER

struct LayerParams {
  const float* table;        // (C+1) x jpad fp32, row 0 zero
  const uint32_t* ids;       // YET event ids (device)
  const uint64_t* offsets;   // [num_trials+1] or nullptr
  uint64_t num_trials;
  uint64_t num_events;       // ids buffer length (bounds every read)
  uint32_t K;                // events per trial when offsets == nullptr
  uint32_t C;                // catalogue size
  uint32_t jpad;             // row stride in floats
  uint32_t l2_hints;         // 1: evict_last / evict_first policies; 0: evict_normal
  uint32_t prefetch;         // presence kernel: 1 = L2 prefetch of the warp's next trial
  double* ylt;               // this layer's YLT row (num_trials doubles)
  double* olt;               // this layer's OLT row (largest occurrence-net loss per trial) or nullptr
  unsigned* err;             // bit0: id out of range, bit1: bad offsets
  double r2, l2, r3, l3;     // FT2, FT3
  const uint32_t* present;   // FOLDED presence bitmap (presence kernel): for x = e - 1, bit x & 31 of word
                             // umulhi(x, fold_mul) is set if row e holds a non-zero loss; x = C: sentinel
  uint32_t present_words;    // words of the folded bitmap (staged in shared memory)
  uint32_t fold_mul;         // 2^27 (no folding: word x >> 5) or floor((present_words * 2^32 - 1) / C)
  const uint4* rec;          // per-event sparse row record (presence kernels with one lane per row)
  const uint32_t* exact;     // UNFOLDED presence bitmap (bit e of word e >> 5), for the FX filter stage
  const uint2* xrank;        // XS: per word of the unfolded bitmap (the word, rows with a loss before it),
                             // through the word of bit C + 1, which is set there (the invalid-id sentinel)
  const uint4* rec_c;        // XS: the sparse records of the rows holding a loss only, in row order (rank
                             // = index), then one all-zero record at index rec_zero (invalid ids)
  uint32_t rec_zero;         // XS: rows holding a loss
  const double* occ;         // precombined occurrence-net loss FT2(sum_j FT1(l_ej)) per event
  uint32_t round_min;        // lane kernel: lanes with a queued hit that trigger a gather round
  uint32_t interleave;       // fixed-length kernels: 1 = trials interleaved over the grid's warps, 0 = blocks
  double r1[kMaxJ], l1[kMaxJ];  // FT1 per table column (padding columns: 0, +inf)
};

// Sparse record of one table row (built by ara_create for every layer, any row width <= kMaxJ):
//   x = c1 | c2 << 8 | n << 16   (n = non-zero losses in the row; c1 < c2 their columns, layer order)
//   y = bits of the loss in column c1 (0 if n == 0), z = bits of the loss in column c2 (0 if n < 2)
//   w = the event id (row index)
// A row with n > 2 is read in full from the table.
__device__ __forceinline__ uint4 ld_rec(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Streaming 16-byte load of 4 YET ids (L1 no-allocate; L2 policy from make_policy).
__device__ __forceinline__ uint4 ld_ids4(const uint32_t* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ uint64_t make_policy(bool evict_last, bool enabled) {
  uint64_t p;
  if (!enabled) {
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  } else if (evict_last) {
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  } else {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  }
  return p;
}

__device__ __forceinline__ uint32_t ld_id(const uint32_t* p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

// Gather V consecutive fp32 of a table row (one vector, V*4 bytes, naturally aligned).
template <int V>
__device__ __forceinline__ void ld_row(const float* p, uint64_t pol, float (&x)[V]) {
  if constexpr (V == 8) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
                 : "l"(p), "l"(pol));
  } else if constexpr (V == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3])
                 : "l"(p), "l"(pol));
  } else if constexpr (V == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                 : "=f"(x[0]), "=f"(x[1])
                 : "l"(p), "l"(pol));
  } else {
    static_assert(V == 1, "V must be 1, 2, 4 or 8");
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(x[0]) : "l"(p), "l"(pol));
  }
}

// min(max(x - R, 0), L) in fp64.  Never produces -0.0.
__device__ __forceinline__ double clamp_terms(double x, double R, double L) {
  double y = x - R;
  y = (y > 0.0) ? y : 0.0;
  return (y < L) ? y : L;
}

// Same clamp, branch- and NaN-handling-free (inputs are never NaN): max(y, 0) by masking the sign with
// integer ops, then one compare-select against the limit.  Bitwise identical to clamp_terms for every
// non-NaN input (x - R is never -0.0 here; a negative difference becomes +0).
__device__ __forceinline__ double clamp_fast(double x, double R, double L) {
  const double y = x - R;
  const int hi = __double2hiint(y), lo = __double2loint(y);
  const int keep = ~(hi >> 31);
  const double z = __hiloint2double(hi & keep, lo & keep);
  double r;
  asm("{\n .reg .pred p;\n setp.lt.f64 p, %1, %2;\n selp.f64 %0, %1, %2, p;\n}" : "=d"(r) : "d"(z), "d"(L));
  return r;
}

// st.shared predicated on `pred` without a branch.
__device__ __forceinline__ void st_shared_if(uint32_t* ptr, uint32_t v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.u32 [%0], %1;\n}"
               :: "r"((uint32_t)__cvta_generic_to_shared(ptr)), "r"(v), "r"((int)pred) : "memory");
}

// Warp-synchronous primitives as inline PTX for full-warp, converged call sites (the presence kernel's
// scan): avoids the divergence-handling slow paths nvcc wraps around the intrinsics.
__device__ __forceinline__ unsigned ballot_full(bool p) {
  unsigned r;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n vote.sync.ballot.b32 %0, q, 0xffffffff;\n}"
               : "=r"(r) : "r"((unsigned)p));
  return r;
}
__device__ __forceinline__ bool any_full(bool p) {
  unsigned r;
  asm volatile("{\n .reg .pred q, o;\n setp.ne.u32 q, %1, 0;\n vote.sync.any.pred o, q, 0xffffffff;\n selp.u32 %0, 1, 0, o;\n}"
               : "=r"(r) : "r"((unsigned)p));
  return r != 0;
}

// 32-bit shared-window helpers (the shared-memory base is computed once per kernel).
__device__ __forceinline__ void sts_u32_if(uint32_t saddr, uint32_t v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p st.shared.u32 [%0], %1;\n}"
               :: "r"(saddr), "r"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
// 16-byte asynchronous global -> shared copy (L2 only), completion awaited with cp_async_wait_all.
__device__ __forceinline__ void cp_async8(uint32_t saddr, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(saddr), "l"(g) : "memory");
}
// (The L2 cache-policy operand is not used: ptxas 12.9 sometimes encodes the cache-hinted LDGSTS with an
// odd-numbered uniform descriptor register next to a uniform shared-address offset -- an illegal
// instruction at run time, seen on the FX and stream kernels.)
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, uint64_t /*pol*/) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(saddr), "l"(g) : "memory");
}
// Streaming 16-byte load of 4 YET ids with no L2 policy operand (L1 no-allocate).
__device__ __forceinline__ uint4 ld_ids4_stream(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_id_stream(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
// L2 prefetch of the 128-B line holding `g`.
__device__ __forceinline__ void prefetch_l2_line(const void* g) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(g));
}
// Bulk L2 prefetch of `bytes` (multiple of 16) from a 16-B aligned global address (one TMA request).
__device__ __forceinline__ void prefetch_l2_bulk(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ uint4 lds_u128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr) : "memory");
  return v;
}
// Presence-queue insertion for a pair of window slots (presence kernel).  wa/wb: the bitmap words of
// the two ids, xa/xb: their bit indices (mod 32); the lane's first hit of the pair is appended at
// qt + 4 * (hits of lower lanes), then -- only if some lane hit both -- the second ids likewise; qt
// (the queue's shared tail address) advances by 4 per appended id.  One ballot per pair; the hit
// tests stay predicates end to end (written in PTX so no 0/1 integers are materialised).
// `valid` masks the two slots (all ones for full windows; ptxas folds the AND into the test's LOP3).
__device__ __forceinline__ void pair_insert(uint32_t wa, uint32_t xa, uint32_t ida, uint32_t wb, uint32_t xb,
                                            uint32_t idb, uint32_t lt, uint32_t& qt, uint32_t valid = 0xffffffffu) {
  asm volatile(
      "{\n"
      " .reg .pred pa, pb, pany, pboth, pq;\n"
      " .reg .b32 sa, sb, ma, mb, f, m, t, a, c;\n"
      " and.b32 sa, %2, 31;\n shr.b32 ma, %1, sa;\n and.b32 ma, ma, %8;\n and.b32 ma, ma, 1;\n setp.ne.b32 pa, ma, 0;\n"
      " and.b32 sb, %5, 31;\n shr.b32 mb, %4, sb;\n and.b32 mb, mb, %8;\n and.b32 mb, mb, 1;\n setp.ne.b32 pb, mb, 0;\n"
      " or.pred pany, pa, pb;\n and.pred pboth, pa, pb;\n"
      " selp.b32 f, %3, %6, pa;\n"
      " vote.sync.ballot.b32 m, pany, 0xffffffff;\n"
      " and.b32 t, m, %7;\n popc.b32 t, t;\n mad.lo.u32 a, t, 4, %0;\n"
      " @pany st.shared.u32 [a], f;\n"
      " popc.b32 c, m;\n mad.lo.u32 %0, c, 4, %0;\n"
      " vote.sync.any.pred pq, pboth, 0xffffffff;\n"
      " @!pq bra.uni PAIR_DONE_%=;\n"
      " vote.sync.ballot.b32 m, pboth, 0xffffffff;\n"
      " and.b32 t, m, %7;\n popc.b32 t, t;\n mad.lo.u32 a, t, 4, %0;\n"
      " @pboth st.shared.u32 [a], %6;\n"
      " popc.b32 c, m;\n mad.lo.u32 %0, c, 4, %0;\n"
      "PAIR_DONE_%=:\n"
      "}\n"
      : "+r"(qt)
      : "r"(wa), "r"(xa), "r"(ida), "r"(wb), "r"(xb), "r"(idb), "r"(lt), "r"(valid)
      : "memory");
}

// Read-only shared loads (no volatile, no memory clobber: the bitmap and the FT1 terms are written once
// before the kernel's __syncthreads, so these may be scheduled and hoisted freely).
__device__ __forceinline__ uint32_t lds_ro_u32(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ double2 lds_ro_f64x2(uint32_t saddr) {
  double2 v;
  asm("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(saddr));
  return v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// V: floats per vector load; NV: vectors per row (jpad = V*NV); G: lanes per row (power of 2 <= 32);
// U: rows per row group per iteration.
template <int V, int NV, int G, int U>
__global__ void __launch_bounds__(256) ara_layer_kernel(const __grid_constant__ LayerParams p) {
  static_assert(32 % G == 0, "G must divide 32");
  constexpr int RG = 32 / G;              // row groups (rows in flight per warp per u)
  constexpr int NVL = (NV + G - 1) / G;   // vectors per lane per row
  constexpr int JP = V * NV;
  constexpr unsigned FULL = 0xffffffffu;

  __shared__ double s_r1[JP], s_l1[JP];
  for (int j = threadIdx.x; j < JP; j += blockDim.x) {
    s_r1[j] = p.r1[j];
    s_l1[j] = p.l1[j];
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int g = lane % G;
  const uint64_t pol_tab = make_policy(true, p.l2_hints);
  const uint64_t pol_yet = make_policy(false, p.l2_hints);
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const double R2 = p.r2, L2 = p.l2;

  for (uint64_t t = warp0; t < p.num_trials; t += nwarps) {
    uint64_t b, e;
    unsigned bad = 0;
    if (p.offsets) {
      b = p.offsets[t];
      e = p.offsets[t + 1];
      if (e < b || e > p.num_events) {  // invalid offsets: flag, contribute nothing
        bad |= 2u;
        e = b;
      }
    } else {
      b = t * p.K;
      e = b + p.K;
    }
    double S = 0.0;  // leader's running sum of occurrence-net losses (step 4)
    double M = 0.0;  // leader's largest occurrence-net loss (OLT)
    for (uint64_t k0 = b; k0 < e; k0 += (uint64_t)RG * U) {
      uint32_t id[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t q = k0 + (uint64_t)u * RG + grp;
        uint32_t v = 0;
        if (q < e) {
          v = ld_id(p.ids + q, pol_yet);
          if (v - 1u >= p.C) {  // id outside [1, C]: record, treat as absent
            bad |= 1u;
            v = 0;
          }
        }
        id[u] = v;
      }
      float x[U][NVL][V];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float* row = p.table + (uint64_t)id[u] * JP;
#pragma unroll
        for (int i = 0; i < NVL; ++i) {
          const int s = g + i * G;
          if (id[u] != 0 && (NV % G == 0 || s < NV)) {
            ld_row<V>(row + s * V, pol_tab, x[u][i]);
          } else {
#pragma unroll
            for (int c = 0; c < V; ++c) x[u][i][c] = 0.0f;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // Steps 1-2: FT1 on every non-zero loss of the row, summed across ELTs (fp64).
        uint32_t nz = 0;
#pragma unroll
        for (int i = 0; i < NVL; ++i)
#pragma unroll
          for (int c = 0; c < V; ++c) nz |= __float_as_uint(x[u][i][c]);
        double s = 0.0;
        if (nz) {
#pragma unroll
          for (int i = 0; i < NVL; ++i)
#pragma unroll
            for (int c = 0; c < V; ++c) {
              if (__float_as_uint(x[u][i][c]) != 0u) {
                const int j = (g + i * G) * V + c;
                s += clamp_terms((double)x[u][i][c], s_r1[j], s_l1[j]);
              }
            }
        }
        if constexpr (G > 1) {
          if (__any_sync(FULL, s != 0.0)) {
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(FULL, s, off);
          }
        }
        // Step 3: occurrence terms FT2; step 4: accumulate (leader lane of the row group).
        if (s != 0.0 && g == 0) {
          const double o = clamp_terms(s, R2, L2);
          S += o;
          M = o > M ? o : M;
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(FULL, S, off);
    if (p.olt) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) M = fmax(M, __shfl_xor_sync(FULL, M, off));
      if (lane == 0) p.olt[t] = M;
    }
    bad = __reduce_or_sync(FULL, bad);
    if (lane == 0) {
      p.ylt[t] = clamp_terms(S, p.r3, p.l3);  // step 4: aggregate terms FT3 on S_n
      if (bad) atomicOr(p.err, bad);
    }
  }
}

}  // namespace ara

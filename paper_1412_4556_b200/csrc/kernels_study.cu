// kernels_study.cu -- the paper's Section IV.B data-structure comparison, on B200.
//
// The same Algorithm 1 (one warp per trial, one lane per occurrence, ELTs in layer order, fp64 terms)
// over three ELT representations:
//   STUDY_INTERLEAVED  the combined table T[e][j] (one row per event across the layer's ELTs) -- the
//                      layout of the product kernels ("the ELTs are combined as a single table")
//   STUDY_INDEPENDENT  one direct-access array per ELT, T_j[e] ("each ELT is an independent
//                      table"; the paper's faster layout on its M2050)
//   STUDY_SORTED       per ELT the (event, loss) pairs sorted by event id, found by binary search
//                      ("binary search require O(log(n)) memory accesses")
//   STUDY_HASH         per ELT an open-addressing hash table of (event, loss) pairs, load factor <= 1/2,
//                      multiplicative hash, linear probing ("constant-time hash search")
//   STUDY_INDEX        an event -> compact-row index over the layer (one u32 per event) and a table of the
//                      rows that hold a loss (~154k rows for P instead of 2M)
// The loops are deliberately plain: the point is the memory behaviour of each representation
// (sectors per lookup, DRAM traffic), measured by bench.py --study and ncu.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ara_kernel.cuh"
#include "study.cuh"

namespace ara {

template <int LAYOUT>
__device__ __forceinline__ float study_lookup(const StudyParams& p, uint32_t e, uint32_t j) {
  if constexpr (LAYOUT == STUDY_INTERLEAVED) {
    return __ldg(p.table + (uint64_t)e * p.jpad + j);
  } else if constexpr (LAYOUT == STUDY_INDEPENDENT) {
    return __ldg(p.indep + (uint64_t)j * p.rows + e);
  } else if constexpr (LAYOUT == STUDY_HASH) {
    const uint2* t = p.hash + p.hash_off[j];
    const uint32_t bits = p.hash_bits[j], mask = (1u << bits) - 1u;
    uint32_t h = (e * 0x9E3779B1u) >> (32u - bits);
    while (true) {  // an empty slot (id 0) ends the probe: the event is absent from this ELT
      const uint2 v = __ldg(t + h);
      if (v.x == e) return __uint_as_float(v.y);
      if (v.x == 0u) return 0.0f;
      h = (h + 1u) & mask;
    }
  } else if constexpr (LAYOUT == STUDY_INDEX) {
    const uint32_t r = __ldg(p.row_index + e);  // 0: the event holds no loss (row 0 is all zero)
    return __ldg(p.compact + (uint64_t)r * p.jpad + j);
  } else {
    const uint32_t* ids = p.sorted_ids + p.sorted_off[j];
    const float* losses = p.sorted_loss + p.sorted_off[j];
    uint32_t lo = 0, hi = p.sorted_off[j + 1] - p.sorted_off[j];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(ids + mid) < e)
        lo = mid + 1;
      else
        hi = mid;
    }
    return (lo < p.sorted_off[j + 1] - p.sorted_off[j] && __ldg(ids + lo) == e) ? __ldg(losses + lo) : 0.0f;
  }
}

template <int LAYOUT>
__global__ void __launch_bounds__(256) study_kernel(const __grid_constant__ StudyParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t t = warp0; t < p.num_trials; t += nwarps) {
    uint64_t b, e;
    if (p.offsets) {
      b = p.offsets[t];
      e = p.offsets[t + 1];
    } else {
      b = t * p.K;
      e = b + p.K;
    }
    double S = 0.0;
    for (uint64_t k = b + lane; k < e; k += 32) {
      uint32_t ev = __ldg(p.ids + k);
      if (ev - 1u >= p.C) ev = 0;  // the study assumes validated input; out-of-range ids read as absent
      double s = 0.0;
      for (uint32_t j = 0; j < p.J; ++j)
        s += clamp_terms((double)study_lookup<LAYOUT>(p, ev, j), p.r1[j], p.l1[j]);  // steps 1-2
      S += clamp_terms(s, p.r2, p.l2);  // step 3; step 4 accumulation
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
    if (lane == 0) p.ylt[t] = clamp_terms(S, p.r3, p.l3);
  }
}

void* study_kernel_fn(int layout) {
  switch (layout) {
    case STUDY_INTERLEAVED: return (void*)study_kernel<STUDY_INTERLEAVED>;
    case STUDY_INDEPENDENT: return (void*)study_kernel<STUDY_INDEPENDENT>;
    case STUDY_SORTED: return (void*)study_kernel<STUDY_SORTED>;
    case STUDY_HASH: return (void*)study_kernel<STUDY_HASH>;
    case STUDY_INDEX: return (void*)study_kernel<STUDY_INDEX>;
  }
  return nullptr;
}

// T_j[e] = T[e][j]: the independent per-ELT arrays from the combined table.
__global__ void __launch_bounds__(256) study_transpose_kernel(float* __restrict__ indep, const float* __restrict__ table,
                                                              uint32_t jpad, uint32_t J, uint64_t rows) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows * J; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = i / rows, e = i % rows;
    indep[i] = table[e * jpad + j];
  }
}

void study_transpose(float* indep, const float* table, uint32_t jpad, uint32_t J, uint64_t rows, int sms,
                     cudaStream_t s) {
  const uint64_t n = rows * J;
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 16);
  study_transpose_kernel<<<(unsigned)blocks, 256, 0, s>>>(indep, table, jpad, J, rows);
}

}  // namespace ara

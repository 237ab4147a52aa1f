// ara_api.cu -- the C ABI of include/ara.h: validation, the per-layer direct-access tables, kernel
// dispatch, the end-to-end host path, and the small utilities.  Metrics live in metrics.cu.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "ara.h"
#include "ara_kernel.cuh"
#include "presence_kernel.cuh"
#include "stream_kernel.cuh"
#include "lane_kernel.cuh"
#include "mask_kernel.cuh"
#include "fused_kernel.cuh"
#include "variants.cuh"
#include "study.cuh"
#include "common.cuh"
#include "ctx.cuh"

namespace ara {

static thread_local char g_err[512] = "";

ara_status set_error(ara_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

ara_status cuda_error(cudaError_t e, const char* what) {
  return set_error(ARA_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------------------ layout
// Row stride in floats: J rounded up to a power of two when 4J <= 32 B (a row never straddles a
// 32-B sector), else to a multiple of 8 floats (whole sectors).
static uint32_t row_floats(uint32_t J) {
  if (J <= 1) return 1;
  if (J <= 2) return 2;
  if (J <= 4) return 4;
  if (J <= 8) return 8;
  return (J + 7) / 8 * 8;
}

// ------------------------------------------------------------------------------------------ variants
static void variants_for(int kind, uint32_t jpad, std::vector<const Variant*>& out) {
  out.clear();
  const Variant* (*tables[3])(int*) = {presence_variants_narrow, presence_variants_mid, presence_variants_wide};
  for (int k = 0; k < (kind == KIND_DENSE ? 1 : 3); ++k) {
    int n = 0;
    const Variant* t = kind == KIND_DENSE ? dense_variants(&n) : tables[k](&n);
    for (int i = 0; i < n; ++i)
      if (t[i].jpad == jpad) out.push_back(&t[i]);
  }
}

static bool valid_terms(const ara_terms& t) {
  return isfinite(t.retention) && t.retention >= 0.0 && !isnan(t.limit) && t.limit > 0.0;
}

static ara_status validate(uint32_t C, const ara_elt* elts, uint32_t num_elts, const ara_layer* layers,
                           uint32_t num_layers) {
  if (C == 0) return set_error(ARA_E_ARG, "catalog_size must be >= 1");
  if (!elts || num_elts == 0) return set_error(ARA_E_ARG, "no ELTs");
  if (!layers || num_layers == 0) return set_error(ARA_E_ARG, "no layers");
  std::vector<uint64_t> seen((C + 64ull) / 64, 0);
  for (uint32_t j = 0; j < num_elts; ++j) {
    const ara_elt& e = elts[j];
    if (e.num_entries && (!e.event_ids || !e.losses)) return set_error(ARA_E_ARG, "ELT %u: NULL arrays", j);
    if (!valid_terms(e.ft1)) return set_error(ARA_E_VALUE, "ELT %u: invalid FT1 terms", j);
    for (uint64_t i = 0; i < e.num_entries; ++i) {
      uint32_t id = e.event_ids[i];
      if (id < 1 || id > C) {
        for (uint64_t k = 0; k < i; ++k) seen[e.event_ids[k] >> 6] = 0;
        return set_error(ARA_E_RANGE, "ELT %u entry %llu: event id %u outside [1, %u]", j, (unsigned long long)i, id, C);
      }
      float l = e.losses[i];
      if (!isfinite(l) || !(l > 0.0f)) {
        for (uint64_t k = 0; k < i; ++k) seen[e.event_ids[k] >> 6] = 0;
        return set_error(ARA_E_VALUE, "ELT %u entry %llu: loss must be finite and > 0", j, (unsigned long long)i);
      }
      uint64_t bit = 1ull << (id & 63);
      if (seen[id >> 6] & bit) {
        for (uint64_t k = 0; k < i; ++k) seen[e.event_ids[k] >> 6] = 0;
        return set_error(ARA_E_DUP, "ELT %u: event id %u appears twice", j, id);
      }
      seen[id >> 6] |= bit;
    }
    for (uint64_t i = 0; i < e.num_entries; ++i) seen[e.event_ids[i] >> 6] = 0;
  }
  for (uint32_t l = 0; l < num_layers; ++l) {
    const ara_layer& L = layers[l];
    if (!L.elt_index || L.num_elts == 0) return set_error(ARA_E_ARG, "layer %u: no ELTs", l);
    if (L.num_elts > kMaxJ)
      return set_error(ARA_E_UNSUPPORTED, "layer %u: %u ELTs > %d", l, L.num_elts, kMaxJ);
    for (uint32_t m = 0; m < L.num_elts; ++m) {
      if (L.elt_index[m] >= num_elts) return set_error(ARA_E_ARG, "layer %u: ELT index %u out of range", l, L.elt_index[m]);
      for (uint32_t k = 0; k < m; ++k)
        if (L.elt_index[k] == L.elt_index[m]) return set_error(ARA_E_ARG, "layer %u: ELT %u listed twice", l, L.elt_index[m]);
    }
    if (!valid_terms(L.occurrence)) return set_error(ARA_E_VALUE, "layer %u: invalid occurrence terms", l);
    if (!valid_terms(L.aggregate)) return set_error(ARA_E_VALUE, "layer %u: invalid aggregate terms", l);
  }
  return ARA_OK;
}

// Scatter (event id, loss) pairs into the layer's interleaved table: T[id][col] = loss.
__global__ void __launch_bounds__(256) scatter_kernel(float* __restrict__ table, uint32_t jpad,
                                                      const uint32_t* __restrict__ ids,
                                                      const float* __restrict__ losses,
                                                      const uint32_t* __restrict__ col, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    table[(uint64_t)ids[i] * jpad + col[i]] = losses[i];
}

// Build the presence bitmap of one layer: bit id of present[] for every ELT entry of the layer.
__global__ void __launch_bounds__(256) presence_build_kernel(uint32_t* __restrict__ present,
                                                             const uint32_t* __restrict__ ids, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[i];
    atomicOr(present + (id >> 5), 1u << (id & 31u));
  }
}


// Fold the presence bitmap into `fw` words for the presence kernel: row e >= 1 (x = e - 1) sets bit
// x & 31 of word umulhi(x, mul); x = C is the always-set sentinel that catches invalid ids.
__global__ void __launch_bounds__(256) presence_fold_kernel(uint32_t* __restrict__ folded,
                                                            const uint32_t* __restrict__ present, uint32_t words,
                                                            uint32_t C, uint32_t mul) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint32_t v = present[w];
    while (v) {
      const uint32_t e = w * 32u + (uint32_t)(__ffs(v) - 1);
      v &= v - 1u;
      if (e == 0u || e > C) continue;
      const uint32_t x = e - 1u;
      atomicOr(folded + __umulhi(x, mul), 1u << (x & 31u));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(folded + __umulhi(C, mul), 1u << (C & 31u));
}

// Sparse record per table row (see ld_rec in ara_kernel.cuh): the first two non-zero columns and losses,
// the count of non-zero columns and the event id itself.
__global__ void __launch_bounds__(256) record_build_kernel(uint4* __restrict__ rec, const float* __restrict__ table,
                                                           uint32_t jpad, uint64_t rows) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows; e += (uint64_t)gridDim.x * blockDim.x) {
    const float* row = table + e * jpad;
    uint32_t n = 0, c1 = 0, c2 = 0, l1 = 0, l2 = 0;
    for (uint32_t j = 0; j < jpad; ++j) {
      const uint32_t b = __float_as_uint(row[j]);
      if (b == 0u) continue;
      if (n == 0) {
        c1 = j;
        l1 = b;
      } else if (n == 1) {
        c2 = j;
        l2 = b;
      }
      ++n;
    }
    rec[e] = make_uint4(c1 | (c2 << 8) | (n << 16), l1, l2, (uint32_t)e);
  }
}

// XS compact-row index (the event -> compact row map of SURVEY N2, folded into the exact
// scan filter).  Block b of 1024 words: bsum[b] = rows holding a loss in it.
__global__ void __launch_bounds__(1024) rank_count_kernel(const uint32_t* __restrict__ present, uint32_t words,
                                                          uint32_t* __restrict__ bsum) {
  const uint32_t w = blockIdx.x * 1024u + threadIdx.x;
  uint32_t v = w < words ? __popc(present[w]) : 0u;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __shared__ uint32_t ws[32];
  if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < 32; ++i) t += ws[i];
    bsum[blockIdx.x] = t;
  }
}
// Exclusive prefix of the block sums (one thread: a few hundred blocks, built once per layer).
__global__ void rank_scan_kernel(uint32_t* bsum, uint32_t nb) {
  uint32_t t = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    const uint32_t v = bsum[b];
    bsum[b] = t;
    t += v;
  }
}
// xrank[w] = (word w, loss-holding rows in words < w); then each loss-holding row's record is copied to
// its rank: rec_c[rank(e)] = rec[e].
// Entries run through word (C + 1) >> 5 (`xwords`), where bit C + 1 -- no row, rank = every row holding a
// loss -- is set: an invalid id (x = C after the clamp) is an exact hit on the zero record.
__global__ void __launch_bounds__(1024) rank_write_kernel(const uint32_t* __restrict__ present, uint32_t words,
                                                          uint32_t xwords, uint32_t C,
                                                          const uint32_t* __restrict__ bsum, const uint4* __restrict__ rec,
                                                          uint2* __restrict__ xrank, uint4* __restrict__ rec_c) {
  const uint32_t w = blockIdx.x * 1024u + threadIdx.x, lane = threadIdx.x & 31u;
  const uint32_t word = w < words ? present[w] : 0u;
  const uint32_t c = __popc(word);
  uint32_t incl = c;
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= (uint32_t)off) incl += y;
  }
  __shared__ uint32_t ws[32];
  if (lane == 31u) ws[threadIdx.x >> 5] = incl;
  __syncthreads();
  if (threadIdx.x < 32u) {
    uint32_t v = ws[threadIdx.x], x = v;
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (threadIdx.x >= (uint32_t)off) x += y;
    }
    ws[threadIdx.x] = x - v;  // exclusive over the block's warps
  }
  __syncthreads();
  if (w >= xwords) return;
  uint32_t base = bsum[blockIdx.x] + ws[threadIdx.x >> 5] + incl - c;
  const uint32_t sentinel = w == (C + 1u) >> 5 ? 1u << ((C + 1u) & 31u) : 0u;
  xrank[w] = make_uint2(word | sentinel, base);
  for (uint32_t m = word; m != 0u; m &= m - 1u) rec_c[base++] = rec[(uint64_t)w * 32u + (__ffs(m) - 1u)];
}

// the union presence bitmap of a layer group (word-wise OR of the layers' bitmaps).
__global__ void __launch_bounds__(256) union_bitmap_kernel(uint32_t* __restrict__ out, const uint32_t* const* in,
                                                           uint32_t nl, uint32_t words) {
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (uint32_t l = 0; l < nl; ++l) v |= in[l][w];
    out[w] = v;
  }
}

struct FusedBuildArgs {
  const float* table[kFusedMaxLayers];
  uint32_t jpad[kFusedMaxLayers], J[kFusedMaxLayers], col0[kFusedMaxLayers];
  uint32_t nl;
};

// combined 32-B record per event over a layer group: up to four (global column, loss) entries
// in layer/column order, their count (more than four: read the layer rows in full), the event id.
__global__ void __launch_bounds__(256) fused_record_kernel(uint4* __restrict__ rec, const __grid_constant__ FusedBuildArgs a,
                                                           uint64_t rows) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows; e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t n = 0, cols = 0, l[4] = {0u, 0u, 0u, 0u};
    for (uint32_t ly = 0; ly < a.nl; ++ly) {
      const float* row = a.table[ly] + e * a.jpad[ly];
      for (uint32_t j = 0; j < a.J[ly]; ++j) {
        const uint32_t b = __float_as_uint(row[j]);
        if (b == 0u) continue;
        if (n < 4u) {
          cols |= (a.col0[ly] + j) << (8u * n);
          l[n] = b;
        }
        ++n;
      }
    }
    rec[2 * e] = make_uint4(cols, n, l[0], l[1]);
    rec[2 * e + 1] = make_uint4(l[2], l[3], (uint32_t)e, 0u);
  }
}

// o[e] = FT2(sum_j FT1(T[e][j])) per event, summed over the layer's columns in order with the
// kernels' clamp (absent losses give exact +0 terms), so it equals the record path's value bit for bit.
__global__ void __launch_bounds__(256) occ_build_kernel(double* __restrict__ occ, const float* __restrict__ table,
                                                        uint32_t jpad, const __grid_constant__ LayerParams p,
                                                        uint64_t rows) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows; e += (uint64_t)gridDim.x * blockDim.x) {
    const float* row = table + e * jpad;
    double sum = 0.0;
    for (uint32_t j = 0; j < jpad; ++j) {
      const float x = row[j];
      if (x != 0.0f) sum += clamp_fast((double)x, p.r1[j], p.l1[j]);
    }
    occ[e] = clamp_fast(sum, p.r2, p.l2);
  }
}

static void destroy_ctx(ara_ctx* c) {
  if (!c) return;
  DeviceGuard guard(c->device);
  cudaDeviceSynchronize();
  for (auto& L : c->layers) {
    cudaFree(L.table);
    cudaFree(L.present);
    for (auto& f : L.folds) cudaFree(f.buf);
    cudaFree(L.rec);
    cudaFree(L.xrank);
    cudaFree(L.rec_c);
    cudaFree(L.occ);
    cudaFree(L.indep);
    cudaFree(L.sorted_ids);
    cudaFree(L.sorted_loss);
    cudaFree(L.sorted_off);
    cudaFree(L.hash);
    cudaFree(L.hash_off);
    cudaFree(L.hash_bits);
    cudaFree(L.row_index);
    cudaFree(L.compact);
  }
  for (auto& g : c->groups) {
    cudaFree(g.rec);
    cudaFree(g.present);
    for (auto& f : g.folds) cudaFree(f.buf);
  }
  cudaFree(c->d_err);
  cudaFreeHost(c->h_err);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c->st_ids[i]);
    cudaFree(c->st_off[i]);
    cudaFree(c->st_ylt[i]);
    cudaFreeHost(c->h_off[i]);
    if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
    if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
  }
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  delete c;
}

// Dynamic shared memory of a presence variant besides the bitmap: the per-warp hit queues and, for
// one-lane-per-row variants (record batches), 32 x 16-B record slots per warp (+16 B alignment slack).
static size_t presence_warp_smem(const Variant* v) {
  const bool rec = v->G == 1;
  return (size_t)v->NW * kQueue * 4 + (rec ? (size_t)v->NW * 512 + 16 : 0);
}

static int kind_of(const ara_ctx* c, const Layer& L) { return c->kernel < 0 ? L.auto_kind : c->kernel; }

static const Variant* pick(const ara_ctx* c, const Layer& L) {
  const auto& vs = L.variants[kind_of(c, L)];
  int v = c->variant;
  if (v < 0 || v >= (int)vs.size()) v = 0;
  return vs[v];
}

// Static shared memory of a kernel, cached per context (cudaFuncGetAttributes once per kernel).
static ara_status fn_static_smem(ara_ctx* c, const void* fn, int* out) {
  for (auto& f : c->fn_info)
    if (f.fn == fn) {
      *out = f.static_smem;
      return ARA_OK;
    }
  cudaFuncAttributes fa;
  ARA_CUDA(cudaFuncGetAttributes(&fa, fn));
  c->fn_info.push_back({fn, (int)fa.sharedSizeBytes, 0});
  *out = (int)fa.sharedSizeBytes;
  return ARA_OK;
}

// Raise a kernel's dynamic shared-memory limit only when a launch needs more than already set.
static ara_status fn_dyn_smem(ara_ctx* c, const void* fn, size_t bytes) {
  int dummy;
  ara_status st = fn_static_smem(c, fn, &dummy);
  if (st) return st;
  for (auto& f : c->fn_info)
    if (f.fn == fn) {
      if ((int)bytes > f.dyn_set) {
        ARA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        f.dyn_set = (int)bytes;
      }
      return ARA_OK;
    }
  return ARA_OK;
}

// The layer's presence bitmap folded into `words` words (built on first use, stream-ordered; one buffer
// per fold size, so a fold is never rebuilt while an earlier launch may still read it).
static ara_status get_fold(ara_ctx* c, Layer& L, uint32_t words, cudaStream_t stream, const uint32_t** buf,
                           uint32_t* mul_out) {
  const uint64_t C = c->C;
  const uint32_t fw = (uint32_t)std::min<uint64_t>(L.present_words, words);
  const uint32_t mul = (C + 1 <= 32ull * fw) ? (1u << 27) : (uint32_t)((((uint64_t)fw << 32) - 1) / C);
  for (auto& f : L.folds)
    if (f.words == fw && f.mul == mul) {
      *buf = f.buf;
      *mul_out = mul;
      return ARA_OK;
    }
  uint32_t* b = nullptr;
  if (cudaMalloc(&b, (size_t)fw * 4) != cudaSuccess) {
    cudaGetLastError();
    return set_error(ARA_E_NOMEM, "folded presence bitmap");
  }
  ARA_CUDA(cudaMemsetAsync(b, 0, (size_t)fw * 4, stream));
  const unsigned fb = (unsigned)std::min<uint64_t>((L.present_words + 255) / 256, 4096);
  presence_fold_kernel<<<fb, 256, 0, stream>>>(b, L.present, L.present_words, c->C, mul);
  ARA_CUDA(cudaGetLastError());
  L.folds.push_back({fw, mul, b});
  *buf = b;
  *mul_out = mul;
  return ARA_OK;
}

// The XS compact-row index of a layer (built on first use, stream-ordered, never rebuilt).
static ara_status get_compact(ara_ctx* c, Layer& L, cudaStream_t stream) {
  if (L.xrank) return ARA_OK;
  const uint32_t words = L.present_words, xwords = (uint32_t)((c->C + 1ull) >> 5) + 1u;
  const uint32_t nb = (std::max(words, xwords) + 1023u) / 1024u;
  uint32_t* bsum = nullptr;
  if (cudaMalloc(&L.xrank, (size_t)xwords * sizeof(uint2)) != cudaSuccess ||
      cudaMalloc(&L.rec_c, (L.present_rows + 1) * sizeof(uint4)) != cudaSuccess ||
      cudaMallocAsync((void**)&bsum, (size_t)nb * 4, stream) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(L.xrank);
    cudaFree(L.rec_c);
    L.xrank = nullptr;
    L.rec_c = nullptr;
    return set_error(ARA_E_NOMEM, "compact-row index");
  }
  ARA_CUDA(cudaMemsetAsync(L.rec_c + L.present_rows, 0, sizeof(uint4), stream));  // the zero record
  rank_count_kernel<<<nb, 1024, 0, stream>>>(L.present, words, bsum);
  rank_scan_kernel<<<1, 1, 0, stream>>>(bsum, nb);
  rank_write_kernel<<<nb, 1024, 0, stream>>>(L.present, words, xwords, c->C, bsum, L.rec, L.xrank, L.rec_c);
  ARA_CUDA(cudaGetLastError());
  cudaFreeAsync(bsum, stream);
  return ARA_OK;
}

// The fixed-length-trial kernel applies to a YET of fixed length K (K % 4 == 0, 16-B aligned ids), a
// catalogue below 2^32 - 2 and per-warp hit ordinals that cannot wrap.
static bool stream_eligible(const ara_ctx* c, const uint32_t* ids, const uint64_t* offsets, uint64_t num_trials,
                            uint32_t K, int nw) {
  if (offsets || K == 0 || (K & 3u) || (reinterpret_cast<uintptr_t>(ids) & 15u)) return false;
  if (c->precombined) return false;  // that ablation lives in the presence kernel
  if ((uint64_t)c->C + 2 > 0xffffffffull) return false;
  const uint64_t warps = (uint64_t)c->sms * nw;
  const uint64_t per_warp = (num_trials + warps - 1) / warps + 1;
  return per_warp * ((K + 127ull) / 128 * 128) < (1ull << 30);
}

static ara_status launch_layer(ara_ctx* c, Layer& L, const uint32_t* ids, const uint64_t* offsets,
                               uint64_t num_trials, uint64_t num_events, uint32_t K, double* ylt, double* olt,
                               cudaStream_t stream) {
  if (num_trials == 0) return ARA_OK;
  const Variant* var = pick(c, L);
  LayerParams p;
  memset(&p, 0, sizeof p);
  p.table = L.table;
  p.ids = ids;
  p.offsets = offsets;
  p.num_trials = num_trials;
  p.num_events = num_events;
  p.K = K;
  p.C = c->C;
  p.jpad = L.jpad;
  p.l2_hints = c->l2_policy == 1 ? 0u : 1u;
  p.prefetch = c->prefetch > 0 ? 1u : 0u;
  p.ylt = ylt;
  p.olt = olt;
  p.err = c->d_err;
  p.r2 = L.r2;
  p.l2 = L.l2;
  p.r3 = L.r3;
  p.l3 = L.l3;
  for (int j = 0; j < kMaxJ; ++j) {
    p.r1[j] = L.r1[j];
    p.l1[j] = L.l1[j];
  }
  int threads = c->block_threads;
  size_t dyn_smem = 0;
  KernelFn fn = olt ? var->fn_olt : var->fn;
  const char* name = var->name;
  int bps = c->blocks_per_sm;
  int nsv = 0;
  const StreamVariant* sv = stream_variants(&nsv);
  const StreamVariant* svar = (c->stream_kernel > 0 && c->stream_kernel <= nsv) ? &sv[c->stream_kernel - 1] : nullptr;
  if (!svar && (c->filter == 1 || (c->filter < 0 && L.xs_auto)))  // exact scan filter for fixed-length trials
    for (int v = 0; v < nsv && !svar; ++v)
      if (sv[v].xs) svar = &sv[v];
  if (var->kind == KIND_PRESENCE && svar && stream_eligible(c, ids, offsets, num_trials, K, svar->NW) &&
      (svar->ring != 2 || (K + 127u) / 128u == 8u)) {  // the mask kernel is built for 8 windows per trial
    // fixed-length trials: the stream kernel (stream_kernel.cuh), one block of NW warps per SM
    fn = olt ? svar->fn_olt : svar->fn;
    name = svar->name;
    // auto: bulk L2 prefetch two trials ahead (lane/ring kernels); the mask kernel: off (measured: the bulk
    // prefetch doubles its DRAM bytes)
    p.prefetch = c->prefetch < 0 ? (svar->ring == 2 ? 0u : 1u) : (c->prefetch != 0 ? 1u : 0u);
    threads = svar->NW * 32;
    int st_smem = 0;
    ara_status st = fn_static_smem(c, (const void*)fn, &st_smem);
    if (st) return st;
    const uint32_t extra = svar->ring == 1 ? stream_smem_extra(L.jpad, svar->NW)
                           : svar->ring == 2 ? mask_smem_extra(L.jpad, svar->NW)
                                             : lane_smem_extra(L.jpad, svar->NW);
    const int64_t budget = (int64_t)c->smem_optin - st_smem - (int64_t)extra;
    if (budget < 4096) return set_error(ARA_E_UNSUPPORTED, "no shared memory left for the presence bitmap");
    const uint32_t* fold = nullptr;
    uint32_t mul = 0;
    const uint32_t fw = (uint32_t)std::min<int64_t>(L.fold_words, budget / 4);
    st = get_fold(c, L, fw, stream, &fold, &mul);
    if (st) return st;
    if (svar->xs) {
      st = get_compact(c, L, stream);
      if (st) return st;
      p.xrank = L.xrank;
      p.rec_c = L.rec_c;
      p.rec_zero = (uint32_t)L.present_rows;
    }
    p.present = fold;
    p.rec = L.rec;
    p.exact = L.present;
    p.present_words = fw;
    p.fold_mul = mul;
    dyn_smem = (size_t)fw * 4 + extra;
    p.round_min = (uint32_t)c->round_min;
    p.interleave = (uint32_t)c->interleave;
    st = fn_dyn_smem(c, (const void*)fn, dyn_smem);
    if (st) return st;
    bps = 1;
  } else if (var->kind == KIND_PRESENCE) {
    threads = var->NW * 32;
    int st_smem = 0;
    ara_status st = fn_static_smem(c, (const void*)var->fn, &st_smem);
    if (st) return st;
    const int64_t budget = (int64_t)c->smem_optin - st_smem - (int64_t)presence_warp_smem(var);
    if (budget < 4096) return set_error(ARA_E_UNSUPPORTED, "no shared memory left for the presence bitmap");
    const uint32_t fw = (uint32_t)std::min<int64_t>(L.fold_words, budget / 4);
    const uint32_t* fold = nullptr;
    uint32_t mul = 0;
    st = get_fold(c, L, fw, stream, &fold, &mul);
    if (st) return st;
    const uint64_t C = c->C;
    p.present = fold;
    p.rec = L.rec;
    p.exact = L.present;
    p.present_words = fw;
    p.fold_mul = mul;
    dyn_smem = (size_t)fw * 4 + presence_warp_smem(var);
    // exact filter stage (ARA_OPT_FILTER): only on request -- it cuts the DRAM traffic of a folded
    // bitmap's false positives but measured slower on config X (presence_kernel.cuh, FX)
    const bool fx = var->fn_fx && c->filter == 1;
    fn = fx ? (olt ? var->fn_fx_olt : var->fn_fx) : fn;
    if (c->precombined && var->fn_pc) {  // SURVEY N3 ablation: o[e] tabulated once per layer
      if (!L.occ) {
        if (cudaMalloc(&L.occ, ((size_t)C + 1) * sizeof(double)) != cudaSuccess) {
          cudaGetLastError();
          return set_error(ARA_E_NOMEM, "precombined table");
        }
        const uint64_t rows = C + 1;
        const unsigned ob = (unsigned)std::min<uint64_t>((rows + 255) / 256, (uint64_t)c->sms * 16);
        occ_build_kernel<<<ob, 256, 0, stream>>>(L.occ, L.table, L.jpad, p, rows);
        ARA_CUDA(cudaGetLastError());
      }
      p.occ = L.occ;
      fn = olt ? var->fn_pc_olt : var->fn_pc;
    }
    st = fn_dyn_smem(c, (const void*)fn, dyn_smem);
    if (st) return st;
    if (bps <= 0) bps = 1;  // __launch_bounds__(NW * 32, 1) and a shared-memory-sized bitmap: one block per SM
  }
  if (bps <= 0) {
    ARA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (const void*)var->fn, threads, dyn_smem));
    if (bps < 1) bps = 1;
  }
  uint64_t warps_per_block = threads / 32;
  uint64_t blocks = (uint64_t)c->sms * bps;
  uint64_t need = (num_trials + warps_per_block - 1) / warps_per_block;
  if (blocks > need) blocks = need;
  c->last_kernel = name;

  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = dyn_smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  if (c->l2_policy == 2 && c->window_max > 0) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = L.table;
    size_t bytes = std::min<size_t>(L.table_bytes, (size_t)c->window_max);
    attr[0].val.accessPolicyWindow.num_bytes = bytes;
    attr[0].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)c->persist_max / (double)bytes);
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  ARA_CUDA(cudaLaunchKernelEx(&cfg, fn, p));
  return ARA_OK;
}

// consecutive presence layers grouped for the fused kernel (<= 16 layers, <= 256 columns).
static ara_status build_groups(ara_ctx* c, cudaStream_t s) {
  c->groups_built = true;
  const uint32_t nlay = (uint32_t)c->layers.size();
  const uint64_t rows = (uint64_t)c->C + 1;
  uint32_t l = 0;
  while (l < nlay) {
    ara_ctx::FusedGroup g;
    g.l0 = l;
    uint32_t cols = 0;
    while (l < nlay && l - g.l0 < (uint32_t)kFusedMaxLayers && cols + c->layers[l].J <= (uint32_t)kFusedMaxCols) {
      cols += c->layers[l].J;
      ++l;
    }
    if (l == g.l0) ++l;  // a single layer wider than 256 columns: runs on its own
    g.l1 = l;
    g.cols = cols;
    c->groups.push_back(g);
  }
  for (auto& g : c->groups) {
    const uint32_t nl = g.l1 - g.l0;
    if (nl < 2) continue;
    const uint32_t words = c->layers[0].present_words;
    if (cudaMalloc(&g.rec, (rows + 1) * 32) != cudaSuccess || cudaMalloc(&g.present, (size_t)words * 4) != cudaSuccess) {
      cudaGetLastError();
      return set_error(ARA_E_NOMEM, "fused layer-group records");
    }
    ARA_CUDA(cudaMemsetAsync(g.rec + 2 * rows, 0, 32, s));  // record C + 1: all zero (invalid ids)
    const uint32_t* h_in[kFusedMaxLayers];
    FusedBuildArgs a;
    memset(&a, 0, sizeof a);
    a.nl = nl;
    uint32_t col = 0;
    for (uint32_t i = 0; i < nl; ++i) {
      const Layer& L = c->layers[g.l0 + i];
      h_in[i] = L.present;
      a.table[i] = L.table;
      a.jpad[i] = L.jpad;
      a.J[i] = L.J;
      a.col0[i] = col;
      col += L.J;
    }
    const uint32_t** d_in = nullptr;
    ARA_CUDA(cudaMalloc(&d_in, sizeof h_in));
    ARA_CUDA(cudaMemcpyAsync(d_in, h_in, sizeof h_in, cudaMemcpyHostToDevice, s));
    const unsigned ub = (unsigned)std::min<uint64_t>((words + 255) / 256, (uint64_t)c->sms * 8);
    union_bitmap_kernel<<<ub, 256, 0, s>>>(g.present, d_in, nl, words);
    ARA_CUDA(cudaGetLastError());
    const unsigned rb = (unsigned)std::min<uint64_t>((rows + 255) / 256, (uint64_t)c->sms * 16);
    fused_record_kernel<<<rb, 256, 0, s>>>(g.rec, a, rows);
    ARA_CUDA(cudaGetLastError());
    ARA_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_in);
  }
  return ARA_OK;
}

static ara_status launch_fused(ara_ctx* c, ara_ctx::FusedGroup& g, const uint32_t* ids, uint64_t num_trials,
                               uint64_t num_events, uint32_t K, double* ylt, uint64_t ld, cudaStream_t stream) {
  constexpr int NW = 16;
  const uint32_t nl = g.l1 - g.l0;
  const void* fn = (const void*)ara_fused_kernel<NW>;
  int st_smem = 0;
  ara_status st = fn_static_smem(c, fn, &st_smem);
  if (st) return st;
  const int64_t budget = (int64_t)c->smem_optin - st_smem - (int64_t)fused_smem_extra(NW, nl);
  if (budget < 4096) return set_error(ARA_E_UNSUPPORTED, "no shared memory left for the fused bitmap");
  // fold the union bitmap (the folds of the group are cached like a layer's)
  const Layer& L0 = c->layers[g.l0];
  const uint64_t C = c->C;
  const uint32_t fw = (uint32_t)std::min<int64_t>(L0.present_words, budget / 4);
  const uint32_t mul = (C + 1 <= 32ull * fw) ? (1u << 27) : (uint32_t)((((uint64_t)fw << 32) - 1) / C);
  const uint32_t* fold = nullptr;
  for (auto& f : g.folds)
    if (f.words == fw && f.mul == mul) fold = f.buf;
  if (!fold) {
    uint32_t* b = nullptr;
    if (cudaMalloc(&b, (size_t)fw * 4) != cudaSuccess) {
      cudaGetLastError();
      return set_error(ARA_E_NOMEM, "folded union bitmap");
    }
    ARA_CUDA(cudaMemsetAsync(b, 0, (size_t)fw * 4, stream));
    const unsigned fb = (unsigned)std::min<uint64_t>((L0.present_words + 255) / 256, 4096);
    presence_fold_kernel<<<fb, 256, 0, stream>>>(b, g.present, L0.present_words, c->C, mul);
    ARA_CUDA(cudaGetLastError());
    g.folds.push_back({fw, mul, b});
    fold = b;
  }
  FusedParams p;
  memset(&p, 0, sizeof p);
  p.ids = ids;
  p.num_trials = num_trials;
  p.num_events = num_events;
  p.K = K;
  p.C = c->C;
  p.present = fold;
  p.present_words = fw;
  p.fold_mul = mul;
  p.rec = g.rec;
  p.nl = nl;
  p.prefetch = c->prefetch != 0 ? 1u : 0u;
  p.ylt = ylt;
  p.ld = ld;
  p.err = c->d_err;
  for (int j = 0; j < kFusedMaxCols; ++j) {
    p.r1[j] = 0.0;
    p.l1[j] = INFINITY;
  }
  uint32_t col = 0;
  for (uint32_t i = 0; i < nl; ++i) {
    const Layer& L = c->layers[g.l0 + i];
    p.table[i] = L.table;
    p.jpad[i] = L.jpad;
    p.J[i] = L.J;
    p.col0[i] = col;
    p.r2[i] = L.r2;
    p.l2[i] = L.l2;
    p.r3[i] = L.r3;
    p.l3[i] = L.l3;
    for (uint32_t j = 0; j < L.J; ++j) {
      p.r1[col + j] = L.r1[j];
      p.l1[col + j] = L.l1[j];
      p.layer_of[col + j] = (uint8_t)i;
    }
    col += L.J;
  }
  const size_t dyn = (size_t)fw * 4 + fused_smem_extra(NW, nl);
  st = fn_dyn_smem(c, fn, dyn);
  if (st) return st;
  uint64_t blocks = (uint64_t)c->sms;
  const uint64_t need = (num_trials + NW - 1) / NW;
  if (blocks > need) blocks = need;
  c->last_kernel = "ara_fused_kernel<NW=16>";
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = stream;
  ARA_CUDA(cudaLaunchKernelEx(&cfg, ara_fused_kernel<NW>, p));
  return ARA_OK;
}

static ara_status run_layers(ara_ctx* c, const uint32_t* ids, const uint64_t* offsets, uint64_t num_trials,
                             uint64_t num_events, uint32_t K, double* ylt, double* olt, uint64_t ld, cudaStream_t s) {
  // one pass over the YET per layer group (fixed-length trials, every layer on the sparse path)
  bool fuse = c->fused > 0 && !olt && c->layers.size() >= 2 && num_trials > 0 &&
              stream_eligible(c, ids, offsets, num_trials, K, 16) && c->kernel < 0 && !c->precombined &&
              c->stream_kernel == 0;
  for (size_t l = 0; fuse && l < c->layers.size(); ++l) fuse = !c->layers[l].xs_auto;  // not for heavily folded layers
  if (fuse) {
    if (!c->groups_built) {
      ara_status st = build_groups(c, s);
      if (st) return st;
    }
    for (auto& g : c->groups) {
      ara_status st = (g.l1 - g.l0 >= 2)
                          ? launch_fused(c, g, ids, num_trials, num_events, K, ylt + g.l0 * ld, ld, s)
                          : launch_layer(c, c->layers[g.l0], ids, offsets, num_trials, num_events, K, ylt + g.l0 * ld,
                                         nullptr, s);
      if (st) return st;
    }
    return ARA_OK;
  }
  for (size_t l = 0; l < c->layers.size(); ++l) {
    ara_status st = launch_layer(c, c->layers[l], ids, offsets, num_trials, num_events, K, ylt + l * ld,
                                 olt ? olt + l * ld : nullptr, s);
    if (st) return st;
  }
  return ARA_OK;
}

static ara_status check_yet(const ara_yet* y) {
  if (!y) return set_error(ARA_E_ARG, "yet is NULL");
  if (y->num_trials == 0) return ARA_OK;
  if (!y->trial_offsets) {
    if (y->events_per_trial > 0 && !y->event_ids) return set_error(ARA_E_ARG, "event_ids is NULL");
    unsigned __int128 need = (unsigned __int128)y->num_trials * y->events_per_trial;
    if (need > y->num_events) return set_error(ARA_E_ARG, "num_events < num_trials * events_per_trial");
  } else if (y->num_events > 0 && !y->event_ids) {
    return set_error(ARA_E_ARG, "event_ids is NULL");
  }
  return ARA_OK;
}

static ara_status take_err(ara_ctx* c, cudaStream_t s) {
  ARA_CUDA(cudaMemcpyAsync(c->h_err, c->d_err, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
  ARA_CUDA(cudaMemsetAsync(c->d_err, 0, sizeof(unsigned), s));
  ARA_CUDA(cudaStreamSynchronize(s));
  unsigned e = *c->h_err;
  if (e & 1u) return set_error(ARA_E_RANGE, "YET contains an event id outside [1, %u]", c->C);
  if (e & 2u) return set_error(ARA_E_ARG, "YET trial offsets decrease or exceed num_events");
  return ARA_OK;
}

}  // namespace ara

using namespace ara;

extern "C" {

ara_status ara_table_footprint(uint32_t catalog_size, uint32_t num_elts, uint64_t* bytes, uint32_t* row_stride) {
  if (catalog_size == 0 || num_elts == 0 || (!bytes && !row_stride)) return set_error(ARA_E_ARG, "invalid argument");
  uint32_t jp = row_floats(num_elts);
  if (bytes) *bytes = ((uint64_t)catalog_size + 1) * jp * sizeof(float);
  if (row_stride) *row_stride = jp * (uint32_t)sizeof(float);
  return ARA_OK;
}

ara_status ara_create(uint32_t catalog_size, const ara_elt* elts, uint32_t num_elts, const ara_layer* layers,
                      uint32_t num_layers, int device, void* stream, ara_ctx** out) {
  ara::NvtxRange nvtx("ara_create");
  if (!out) return set_error(ARA_E_ARG, "out is NULL");
  *out = nullptr;
  ara_status st = validate(catalog_size, elts, num_elts, layers, num_layers);
  if (st) return st;
  int ndev = 0;
  ARA_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_error(ARA_E_ARG, "device %d not present", device);
  cudaDeviceProp prop;
  ARA_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return set_error(ARA_E_UNSUPPORTED, "libara is built for sm_100a; device %d is sm_%d%d", device, prop.major, prop.minor);
  DeviceGuard guard(device);
  cudaStream_t s = (cudaStream_t)stream;

  ara_ctx* c = new (std::nothrow) ara_ctx();
  if (!c) return set_error(ARA_E_NOMEM, "host allocation failed");
  c->device = device;
  c->sms = prop.multiProcessorCount;
  c->C = catalog_size;
  cudaDeviceGetAttribute(&c->persist_max, cudaDevAttrMaxPersistingL2CacheSize, device);
  cudaDeviceGetAttribute(&c->window_max, cudaDevAttrMaxAccessPolicyWindowSize, device);
  cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);

#define FAIL(x)          \
  do {                   \
    ara_status _s = (x); \
    destroy_ctx(c);      \
    return _s;           \
  } while (0)
#define CK(call)                                             \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) FAIL(cuda_error(_e, #call));      \
  } while (0)

  CK(cudaMalloc(&c->d_err, sizeof(unsigned)));
  CK(cudaMallocHost(&c->h_err, sizeof(unsigned)));
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(unsigned), s));

  c->layers.resize(num_layers);
  std::vector<uint32_t> h_ids, h_col;
  std::vector<float> h_loss;
  uint32_t* d_ids = nullptr;
  uint32_t* d_col = nullptr;
  float* d_loss = nullptr;
  for (uint32_t l = 0; l < num_layers; ++l) {
    Layer& L = c->layers[l];
    const ara_layer& in = layers[l];
    L.J = in.num_elts;
    L.jpad = row_floats(L.J);
    variants_for(KIND_PRESENCE, L.jpad, L.variants[KIND_PRESENCE]);
    variants_for(KIND_DENSE, L.jpad, L.variants[KIND_DENSE]);
    if (L.variants[0].empty() || L.variants[1].empty())
      FAIL(set_error(ARA_E_UNSUPPORTED, "no kernel for row width %u", L.jpad));
    for (int j = 0; j < kMaxJ; ++j) {
      L.r1[j] = 0.0;
      L.l1[j] = INFINITY;
    }
    for (uint32_t m = 0; m < L.J; ++m) {
      L.r1[m] = elts[in.elt_index[m]].ft1.retention;
      L.l1[m] = elts[in.elt_index[m]].ft1.limit;
    }
    L.r2 = in.occurrence.retention;
    L.l2 = in.occurrence.limit;
    L.r3 = in.aggregate.retention;
    L.l3 = in.aggregate.limit;
    L.table_bytes = ((uint64_t)catalog_size + 1) * L.jpad * sizeof(float);
    if (cudaMalloc(&L.table, L.table_bytes) != cudaSuccess) {
      cudaGetLastError();
      FAIL(set_error(ARA_E_NOMEM, "table of %llu bytes for layer %u", (unsigned long long)L.table_bytes, l));
    }
    CK(cudaMemsetAsync(L.table, 0, L.table_bytes, s));
    L.present_words = (uint32_t)(((uint64_t)catalog_size + 1 + 31) / 32);
    if (cudaMalloc(&L.present, (size_t)L.present_words * 4) != cudaSuccess) {
      cudaGetLastError();
      FAIL(set_error(ARA_E_NOMEM, "presence bitmap for layer %u", l));
    }
    CK(cudaMemsetAsync(L.present, 0, (size_t)L.present_words * 4, s));
    {  // presence statistics -> automatic kernel choice (see ara.h, ARA_OPT_KERNEL)
      std::vector<uint8_t> cnt((uint64_t)catalog_size + 1, 0);  // non-zero losses per row, saturating at 3
      for (uint32_t m = 0; m < L.J; ++m) {
        const ara_elt& e = elts[in.elt_index[m]];
        for (uint64_t i = 0; i < e.num_entries; ++i) {
          uint8_t& k = cnt[e.event_ids[i]];
          k = k < 3 ? (uint8_t)(k + 1) : k;
        }
      }
      uint64_t multi = 0;  // rows with more than two losses: read in full by the record path
      for (uint8_t k : cnt) {
        L.present_rows += k != 0;
        multi += k > 2;
      }
      const Variant* pv = L.variants[KIND_PRESENCE][0];
      cudaFuncAttributes fa;
      CK(cudaFuncGetAttributes(&fa, (const void*)pv->fn));
      const int64_t budget = (int64_t)c->smem_optin - (int64_t)fa.sharedSizeBytes - (int64_t)presence_warp_smem(pv);
      const double pw = (double)(((uint64_t)catalog_size + 1 + 31) / 32);
      // canonical fold: the words the tightest kernel (the default stream variant) can hold, so every
      // kernel tests the same candidates and sums a trial's hits in the same order (bitwise equal YLTs)
      {
        int nsv = 0;
        const StreamVariant* sv = stream_variants(&nsv);
        int64_t b = budget;
        for (int v = 0; v < nsv; ++v)
          if (sv[v].ring != 2)  // the mask kernel folds with its own (smaller) budget
          b = std::min<int64_t>(b, (int64_t)c->smem_optin -
                                       (int64_t)(sv[v].ring == 1   ? stream_smem_extra(L.jpad, sv[v].NW)
                                                 : sv[v].ring == 2 ? mask_smem_extra(L.jpad, sv[v].NW)
                                                                   : lane_smem_extra(L.jpad, sv[v].NW)));
        L.fold_words = (uint32_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)pw, b / 4));
      }
      const double fw = budget > 0 ? std::min(pw, (double)L.fold_words) : 1.0;
      {  // exact scan filter: the fold nominates at least twice the rows that hold a loss
        const double d = (double)L.present_rows / ((double)catalog_size + 1.0);
        const double cand = 1.0 - pow(1.0 - d, std::max(1.0, pw / fw));
        L.xs_auto = cand >= 2.0 * d;
      }
      const double dens = (double)L.present_rows / ((double)catalog_size + 1.0);
      L.est_hit_rate = 1.0 - pow(1.0 - dens, std::max(1.0, pw / fw));
      // The presence kernel pays off while it skips most rows.  With one lane per row (G = 1) a hit
      // fetches its 16-B sparse record, not the row, unless the row holds more than two losses; with
      // full-row batches (G > 1) wide rows gather 13+ sectors per hit in rounds and need a sparser bitmap.
      const double multi_share = L.present_rows ? (double)multi / (double)L.present_rows : 0.0;
      const double lim = pv->G == 1 ? (multi_share <= 0.05 ? 0.6 : 0.25) : (L.jpad <= 16 ? 0.25 : 0.15);
      L.auto_kind = (budget >= 4096 && L.est_hit_rate <= lim) ? KIND_PRESENCE : KIND_DENSE;
    }
    h_ids.clear();
    h_col.clear();
    h_loss.clear();
    for (uint32_t m = 0; m < L.J; ++m) {
      const ara_elt& e = elts[in.elt_index[m]];
      h_ids.insert(h_ids.end(), e.event_ids, e.event_ids + e.num_entries);
      h_loss.insert(h_loss.end(), e.losses, e.losses + e.num_entries);
      h_col.insert(h_col.end(), e.num_entries, m);
    }
    uint64_t n = h_ids.size();
    if (n) {
      CK(cudaMalloc(&d_ids, n * 4));
      CK(cudaMalloc(&d_col, n * 4));
      CK(cudaMalloc(&d_loss, n * 4));
      CK(cudaMemcpyAsync(d_ids, h_ids.data(), n * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(d_col, h_col.data(), n * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(d_loss, h_loss.data(), n * 4, cudaMemcpyHostToDevice, s));
      uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 8);
      scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(L.table, L.jpad, d_ids, d_loss, d_col, n);
      CK(cudaGetLastError());
      presence_build_kernel<<<(unsigned)blocks, 256, 0, s>>>(L.present, d_ids, n);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(s));  // host staging vectors are reused for the next layer
      cudaFree(d_ids);
      cudaFree(d_col);
      cudaFree(d_loss);
      d_ids = nullptr;
      d_col = nullptr;
      d_loss = nullptr;
    }
    {  // sparse row records for the one-lane-per-row presence kernels (every row width <= kMaxJ)
      if (cudaMalloc(&L.rec, ((uint64_t)catalog_size + 2) * sizeof(uint4)) != cudaSuccess) {
        cudaGetLastError();
        FAIL(set_error(ARA_E_NOMEM, "row records for layer %u", l));
      }
      const uint64_t rows = (uint64_t)catalog_size + 1;
      CK(cudaMemsetAsync(L.rec + rows, 0, sizeof(uint4), s));  // record C + 1: all zero (invalid ids)
      const uint64_t rb = std::min<uint64_t>((rows + 255) / 256, (uint64_t)c->sms * 16);
      record_build_kernel<<<(unsigned)rb, 256, 0, s>>>(L.rec, L.table, L.jpad, rows);
      CK(cudaGetLastError());
    }
  }
  CK(cudaStreamSynchronize(s));
#undef CK
#undef FAIL
  *out = c;
  return ARA_OK;
}

void ara_destroy(ara_ctx* ctx) { destroy_ctx(ctx); }

ara_status ara_run_ex(ara_ctx* c, const ara_yet* yet, double* ylt, double* olt, void* stream) {
  ara::NvtxRange nvtx("ara_run");
  if (!c) return set_error(ARA_E_ARG, "ctx is NULL");
  ara_status st = check_yet(yet);
  if (st) return st;
  if (yet->num_trials == 0) return ARA_OK;
  if (!ylt) return set_error(ARA_E_ARG, "ylt is NULL");
  DeviceGuard guard(c->device);
  return run_layers(c, yet->event_ids, yet->trial_offsets, yet->num_trials, yet->num_events,
                    yet->events_per_trial, ylt, olt, yet->num_trials, (cudaStream_t)stream);
}

ara_status ara_run(ara_ctx* c, const ara_yet* yet, double* ylt, void* stream) {
  return ara_run_ex(c, yet, ylt, nullptr, stream);
}

}  // extern "C"

// A captured analysis step: ara_run over a fixed device YET + PML/TVaR of every layer, replayed as one
// CUDA graph (no per-step host work: launch attributes, folds and metric scratch are set up once).
struct ara_plan {
  int device = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  char* scratch = nullptr;
};

namespace ara {

static ara_status plan_step(ara_ctx* c, const ara_yet* yet, double* ylt, const double* rps, uint32_t m,
                            double* pml_dev, double* tvar_dev, char* scratch, size_t bytes, cudaStream_t s) {
  ara_status st = run_layers(c, yet->event_ids, yet->trial_offsets, yet->num_trials, yet->num_events,
                             yet->events_per_trial, ylt, nullptr, yet->num_trials, s);
  if (st) return st;
  for (size_t l = 0; m && l < c->layers.size(); ++l) {
    st = metrics_device_into(ylt + l * yet->num_trials, yet->num_trials, rps, m, pml_dev ? pml_dev + l * m : nullptr,
                             tvar_dev ? tvar_dev + l * m : nullptr, scratch, bytes, s, true);
    if (st) return st;
  }
  return ARA_OK;
}

static void plan_free(ara_plan* p) {
  if (!p) return;
  DeviceGuard guard(p->device);
  if (p->exec) cudaGraphExecDestroy(p->exec);
  if (p->graph) cudaGraphDestroy(p->graph);
  cudaFree(p->scratch);
  delete p;
}

}  // namespace ara

extern "C" {

ara_status ara_plan_create(ara_ctx* c, const ara_yet* yet, double* ylt, const double* rps, uint32_t m,
                           double* pml_dev, double* tvar_dev, void* stream, ara_plan** out) {
  if (!c || !out) return set_error(ARA_E_ARG, "NULL argument");
  *out = nullptr;
  ara_status st = check_yet(yet);
  if (st) return st;
  if (yet->num_trials == 0 || !ylt) return set_error(ARA_E_ARG, "empty YET or NULL ylt");
  if (m && (!rps || (!pml_dev && !tvar_dev))) return set_error(ARA_E_ARG, "metrics requested without outputs");
  DeviceGuard guard(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  ara_plan* p = new (std::nothrow) ara_plan();
  if (!p) return set_error(ARA_E_NOMEM, "host allocation failed");
  p->device = c->device;
  const size_t bytes = m ? metrics_scratch_size(yet->num_trials) : 0;
  if (bytes && cudaMalloc(&p->scratch, bytes) != cudaSuccess) {
    cudaGetLastError();
    plan_free(p);
    return set_error(ARA_E_NOMEM, "metric scratch");
  }
  // zeroed once: the metric launches leave their scratch as they found it (metrics.cu, metrics_select)
  if (bytes && cudaMemset(p->scratch, 0, bytes) != cudaSuccess) {
    plan_free(p);
    return cuda_error(cudaGetLastError(), "metric scratch");
  }
  // one eager step first: builds the folds and caches every launch attribute, so the capture records
  // stream work only (and validates the arguments)
  st = plan_step(c, yet, ylt, rps, m, pml_dev, tvar_dev, p->scratch, bytes, s);
  if (st == ARA_OK && cudaStreamSynchronize(s) != cudaSuccess) st = cuda_error(cudaGetLastError(), "plan warm-up");
  cudaStream_t cs = nullptr;
  if (st == ARA_OK && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
    st = cuda_error(cudaGetLastError(), "capture stream");
  if (st == ARA_OK) {
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      st = cuda_error(e, "cudaStreamBeginCapture");
    } else {
      st = plan_step(c, yet, ylt, rps, m, pml_dev, tvar_dev, p->scratch, bytes, cs);
      e = cudaStreamEndCapture(cs, &p->graph);
      if (st == ARA_OK && e != cudaSuccess) st = cuda_error(e, "cudaStreamEndCapture");
      if (st == ARA_OK && (e = cudaGraphInstantiate(&p->exec, p->graph, 0)) != cudaSuccess)
        st = cuda_error(e, "cudaGraphInstantiate");
    }
  }
  if (cs) cudaStreamDestroy(cs);
  if (st) {
    plan_free(p);
    return st;
  }
  *out = p;
  return ARA_OK;
}

ara_status ara_plan_launch(ara_plan* p, void* stream) {
  ara::NvtxRange nvtx("ara_plan_launch");
  if (!p || !p->exec) return set_error(ARA_E_ARG, "plan is NULL");
  DeviceGuard guard(p->device);
  ARA_CUDA(cudaGraphLaunch(p->exec, (cudaStream_t)stream));
  return ARA_OK;
}

void ara_plan_destroy(ara_plan* p) { plan_free(p); }

ara_status ara_metrics_plan_create(const double* ylt, uint64_t n, uint32_t num_layers, const double* rps, uint32_t m,
                                   double* pml_dev, double* tvar_dev, uint64_t out_stride, void* stream,
                                   ara_plan** out) {
  if (!out) return set_error(ARA_E_ARG, "out is NULL");
  *out = nullptr;
  if (!ylt || n == 0 || num_layers == 0 || !rps || m == 0 || (!pml_dev && !tvar_dev))
    return set_error(ARA_E_ARG, "invalid metric plan arguments");
  if (num_layers > 1 && out_stride < m) return set_error(ARA_E_ARG, "out_stride %llu < m", (unsigned long long)out_stride);
  int dev = 0;
  ARA_CUDA(cudaGetDevice(&dev));
  cudaStream_t s = (cudaStream_t)stream;
  ara_plan* p = new (std::nothrow) ara_plan();
  if (!p) return set_error(ARA_E_NOMEM, "host allocation failed");
  p->device = dev;
  const size_t bytes = metrics_scratch_size(n);
  if (cudaMalloc(&p->scratch, bytes) != cudaSuccess || cudaMemset(p->scratch, 0, bytes) != cudaSuccess) {
    cudaGetLastError();
    plan_free(p);
    return set_error(ARA_E_NOMEM, "metric scratch");
  }
  auto step = [&](cudaStream_t st) -> ara_status {
    for (uint32_t l = 0; l < num_layers; ++l) {
      const ara_status r = metrics_device_into(ylt + (uint64_t)l * n, n, rps, m, pml_dev ? pml_dev + l * out_stride : nullptr,
                                               tvar_dev ? tvar_dev + l * out_stride : nullptr, p->scratch, bytes, st,
                                               true);
      if (r) return r;
    }
    return ARA_OK;
  };
  ara_status st = step(s);  // eager once: validates and sets the launch attributes outside the capture
  if (st == ARA_OK && cudaStreamSynchronize(s) != cudaSuccess) st = cuda_error(cudaGetLastError(), "metric plan warm-up");
  cudaStream_t cs = nullptr;
  if (st == ARA_OK && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess)
    st = cuda_error(cudaGetLastError(), "capture stream");
  if (st == ARA_OK) {
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      st = cuda_error(e, "cudaStreamBeginCapture");
    } else {
      st = step(cs);
      e = cudaStreamEndCapture(cs, &p->graph);
      if (st == ARA_OK && e != cudaSuccess) st = cuda_error(e, "cudaStreamEndCapture");
      if (st == ARA_OK && (e = cudaGraphInstantiate(&p->exec, p->graph, 0)) != cudaSuccess)
        st = cuda_error(e, "cudaGraphInstantiate");
    }
  }
  if (cs) cudaStreamDestroy(cs);
  if (st) {
    plan_free(p);
    return st;
  }
  *out = p;
  return ARA_OK;
}

ara_status ara_check(ara_ctx* c, void* stream) {
  if (!c) return set_error(ARA_E_ARG, "ctx is NULL");
  DeviceGuard guard(c->device);
  return take_err(c, (cudaStream_t)stream);
}

ara_status ara_run_host(ara_ctx* c, const ara_yet* yet, double* ylt_host, void* stream) {
  ara::NvtxRange nvtx("ara_run_host");
  if (!c) return set_error(ARA_E_ARG, "ctx is NULL");
  ara_status st = check_yet(yet);
  if (st) return st;
  if (yet->num_trials == 0) return ARA_OK;
  if (!ylt_host) return set_error(ARA_E_ARG, "ylt_host is NULL");
  DeviceGuard guard(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t N = yet->num_trials;
  const uint64_t L = c->layers.size();
  const uint32_t K = yet->events_per_trial;
  const uint64_t* hoff = yet->trial_offsets;
  if (hoff) {  // host offsets: validate here (the device copy is rebased per batch)
    if (hoff[N] > yet->num_events) return set_error(ARA_E_ARG, "trial offsets exceed num_events");
    for (uint64_t t = 0; t < N; ++t)
      if (hoff[t + 1] < hoff[t]) return set_error(ARA_E_ARG, "trial offsets decrease at trial %llu", (unsigned long long)t);
  }
  // staging: 2 x 256 MB of ids, batches of whole trials
  const uint64_t cap_ids = 64ull << 20;
  const uint64_t cap_trials = hoff ? (1ull << 20) : std::max<uint64_t>(1, K ? cap_ids / K : (1ull << 20));
  if (!c->copy_stream) ARA_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; ++i) {
    if (!c->ev_copied[i]) ARA_CUDA(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
    if (!c->ev_done[i]) ARA_CUDA(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
  }
  if (c->st_cap_ids < cap_ids || c->st_cap_trials < cap_trials) {
    ARA_CUDA(cudaDeviceSynchronize());
    for (int i = 0; i < 2; ++i) {
      cudaFree(c->st_ids[i]);
      cudaFree(c->st_off[i]);
      cudaFree(c->st_ylt[i]);
      cudaFreeHost(c->h_off[i]);
      c->st_ids[i] = nullptr;
      c->st_off[i] = nullptr;
      c->st_ylt[i] = nullptr;
      c->h_off[i] = nullptr;
      c->st_cap_ids = c->st_cap_trials = 0;
      if (cudaMalloc(&c->st_ids[i], cap_ids * 4) != cudaSuccess || cudaMalloc(&c->st_off[i], (cap_trials + 1) * 8) != cudaSuccess ||
          cudaMalloc(&c->st_ylt[i], cap_trials * L * 8) != cudaSuccess ||
          cudaMallocHost(&c->h_off[i], (cap_trials + 1) * 8) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ARA_E_NOMEM, "staging buffers");
      }
    }
    c->st_cap_ids = cap_ids;
    c->st_cap_trials = cap_trials;
  }
  if (getenv("ARA_DEBUG")) {
    cudaPointerAttributes pa;
    cudaError_t pe = cudaPointerGetAttributes(&pa, yet->event_ids);
    fprintf(stderr, "[ara_run_host] yet ids %p: %s type=%d; ylt %p\n", (const void*)yet->event_ids,
            cudaGetErrorString(pe), (int)pa.type, (void*)ylt_host);
    cudaGetLastError();
  }
  ARA_CUDA(cudaEventRecord(c->ev_done[0], s));
  ARA_CUDA(cudaEventRecord(c->ev_done[1], s));
  uint64_t t0 = 0;
  int b = 0;
  while (t0 < N) {
    // batch [t0, t1): as many whole trials as fit the staging buffer
    uint64_t t1, q0, q1;
    if (hoff) {
      t1 = t0 + 1;
      while (t1 < N && t1 - t0 < cap_trials && hoff[t1 + 1] - hoff[t0] <= cap_ids) ++t1;
      q0 = hoff[t0];
      q1 = hoff[t1];
      if (q1 - q0 > cap_ids) return set_error(ARA_E_UNSUPPORTED, "a single trial exceeds the staging buffer");
    } else {
      t1 = std::min(N, t0 + cap_trials);
      q0 = t0 * K;
      q1 = t1 * K;
    }
    const int i = b & 1;
    ARA_CUDA(cudaStreamWaitEvent(c->copy_stream, c->ev_done[i], 0));
    if (q1 > q0)
      ARA_CUDA(cudaMemcpyAsync(c->st_ids[i], yet->event_ids + q0, (q1 - q0) * 4, cudaMemcpyHostToDevice, c->copy_stream));
    if (hoff) {
      ARA_CUDA(cudaEventSynchronize(c->ev_done[i]));  // h_off[i] may still be in flight from batch b-2
      for (uint64_t t = t0; t <= t1; ++t) c->h_off[i][t - t0] = hoff[t] - q0;
      ARA_CUDA(cudaMemcpyAsync(c->st_off[i], c->h_off[i], (t1 - t0 + 1) * 8, cudaMemcpyHostToDevice, c->copy_stream));
    }
    ARA_CUDA(cudaEventRecord(c->ev_copied[i], c->copy_stream));
    ARA_CUDA(cudaStreamWaitEvent(s, c->ev_copied[i], 0));
    st = run_layers(c, c->st_ids[i], hoff ? c->st_off[i] : nullptr, t1 - t0, q1 - q0, K, c->st_ylt[i], nullptr,
                    t1 - t0, s);
    if (st) return st;
    for (uint64_t l = 0; l < L; ++l)
      ARA_CUDA(cudaMemcpyAsync(ylt_host + l * N + t0, c->st_ylt[i] + l * (t1 - t0), (t1 - t0) * 8,
                               cudaMemcpyDeviceToHost, s));
    ARA_CUDA(cudaEventRecord(c->ev_done[i], s));
    t0 = t1;
    ++b;
  }
  return take_err(c, s);
}

ara_status ara_run_study(ara_ctx* c, int layout, const ara_yet* yet, double* ylt, void* stream) {
  if (!c) return set_error(ARA_E_ARG, "ctx is NULL");
  if (layout < STUDY_INTERLEAVED || layout > STUDY_INDEX) return set_error(ARA_E_ARG, "unknown layout %d", layout);
  ara_status st = check_yet(yet);
  if (st) return st;
  if (yet->num_trials == 0) return ARA_OK;
  if (!ylt) return set_error(ARA_E_ARG, "ylt is NULL");
  DeviceGuard guard(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t rows = (uint64_t)c->C + 1;
  for (size_t l = 0; l < c->layers.size(); ++l) {
    Layer& L = c->layers[l];
    if (layout == STUDY_INDEPENDENT && !L.indep) {
      if (cudaMalloc(&L.indep, rows * L.J * sizeof(float)) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ARA_E_NOMEM, "independent tables");
      }
      study_transpose(L.indep, L.table, L.jpad, L.J, rows, c->sms, s);
      ARA_CUDA(cudaGetLastError());
    }
    if (layout == STUDY_SORTED && !L.sorted_ids) {
      std::vector<float> h(rows * L.jpad);
      ARA_CUDA(cudaStreamSynchronize(s));
      ARA_CUDA(cudaMemcpy(h.data(), L.table, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
      std::vector<uint32_t> off(L.J + 1, 0), ids;
      std::vector<float> loss;
      for (uint32_t j = 0; j < L.J; ++j) {
        for (uint64_t e = 1; e < rows; ++e)
          if (h[e * L.jpad + j] != 0.0f) {
            ids.push_back((uint32_t)e);
            loss.push_back(h[e * L.jpad + j]);
          }
        off[j + 1] = (uint32_t)ids.size();
      }
      const size_t n = std::max<size_t>(1, ids.size());
      if (cudaMalloc(&L.sorted_ids, n * 4) != cudaSuccess || cudaMalloc(&L.sorted_loss, n * 4) != cudaSuccess ||
          cudaMalloc(&L.sorted_off, off.size() * 4) != cudaSuccess) {
        cudaGetLastError();
        return set_error(ARA_E_NOMEM, "sorted ELT arrays");
      }
      ARA_CUDA(cudaMemcpy(L.sorted_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice));
      ARA_CUDA(cudaMemcpy(L.sorted_loss, loss.data(), loss.size() * 4, cudaMemcpyHostToDevice));
      ARA_CUDA(cudaMemcpy(L.sorted_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
    }
    if ((layout == STUDY_HASH && !L.hash) || (layout == STUDY_INDEX && !L.row_index)) {
      std::vector<float> h(rows * L.jpad);
      ARA_CUDA(cudaStreamSynchronize(s));
      ARA_CUDA(cudaMemcpy(h.data(), L.table, h.size() * sizeof(float), cudaMemcpyDeviceToHost));
      if (layout == STUDY_HASH) {  // per ELT: capacity = smallest power of two >= 2 n (load factor <= 1/2)
        std::vector<uint32_t> off(L.J + 1, 0), bits(L.J, 1);
        std::vector<uint2> tab;
        for (uint32_t j = 0; j < L.J; ++j) {
          uint64_t n = 0;
          for (uint64_t e = 1; e < rows; ++e) n += h[e * L.jpad + j] != 0.0f;
          uint32_t b = 1;
          while ((1ull << b) < 2 * n + 2) ++b;
          bits[j] = b;
          const size_t base = tab.size();
          tab.resize(base + (1ull << b), make_uint2(0u, 0u));
          for (uint64_t e = 1; e < rows; ++e) {
            const float x = h[e * L.jpad + j];
            if (x == 0.0f) continue;
            uint32_t k = ((uint32_t)e * 0x9E3779B1u) >> (32u - b);
            while (tab[base + k].x != 0u) k = (k + 1u) & ((1u << b) - 1u);
            uint32_t bitsx;
            memcpy(&bitsx, &x, 4);
            tab[base + k] = make_uint2((uint32_t)e, bitsx);
          }
          off[j + 1] = (uint32_t)tab.size();
        }
        if (cudaMalloc(&L.hash, tab.size() * sizeof(uint2)) != cudaSuccess ||
            cudaMalloc(&L.hash_off, off.size() * 4) != cudaSuccess || cudaMalloc(&L.hash_bits, bits.size() * 4) != cudaSuccess) {
          cudaGetLastError();
          return set_error(ARA_E_NOMEM, "hash tables");
        }
        ARA_CUDA(cudaMemcpy(L.hash, tab.data(), tab.size() * sizeof(uint2), cudaMemcpyHostToDevice));
        ARA_CUDA(cudaMemcpy(L.hash_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
        ARA_CUDA(cudaMemcpy(L.hash_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
      } else {  // event -> compact row; compact row 0 is the zero row
        std::vector<uint32_t> idx(rows, 0u);
        std::vector<float> comp(L.jpad, 0.0f);
        for (uint64_t e = 1; e < rows; ++e) {
          bool any = false;
          for (uint32_t j = 0; j < L.jpad; ++j) any |= h[e * L.jpad + j] != 0.0f;
          if (!any) continue;
          idx[e] = (uint32_t)(comp.size() / L.jpad);
          comp.insert(comp.end(), h.begin() + e * L.jpad, h.begin() + (e + 1) * L.jpad);
        }
        if (cudaMalloc(&L.row_index, rows * 4) != cudaSuccess || cudaMalloc(&L.compact, comp.size() * 4) != cudaSuccess) {
          cudaGetLastError();
          return set_error(ARA_E_NOMEM, "compact rows");
        }
        ARA_CUDA(cudaMemcpy(L.row_index, idx.data(), rows * 4, cudaMemcpyHostToDevice));
        ARA_CUDA(cudaMemcpy(L.compact, comp.data(), comp.size() * 4, cudaMemcpyHostToDevice));
      }
    }
    StudyParams p;
    memset(&p, 0, sizeof p);
    p.table = L.table;
    p.hash = L.hash;
    p.hash_off = L.hash_off;
    p.hash_bits = L.hash_bits;
    p.row_index = L.row_index;
    p.compact = L.compact;
    p.indep = L.indep;
    p.sorted_ids = L.sorted_ids;
    p.sorted_loss = L.sorted_loss;
    p.sorted_off = L.sorted_off;
    p.ids = yet->event_ids;
    p.offsets = yet->trial_offsets;
    p.num_trials = yet->num_trials;
    p.rows = rows;
    p.K = yet->events_per_trial;
    p.C = c->C;
    p.J = L.J;
    p.jpad = L.jpad;
    p.ylt = ylt + l * yet->num_trials;
    p.r2 = L.r2;
    p.l2 = L.l2;
    p.r3 = L.r3;
    p.l3 = L.l3;
    for (int j = 0; j < kMaxJ; ++j) {
      p.r1[j] = L.r1[j];
      p.l1[j] = L.l1[j];
    }
    void* fn = study_kernel_fn(layout);
    int bps = 0;
    ARA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, 256, 0));
    uint64_t blocks = (uint64_t)c->sms * std::max(1, bps);
    blocks = std::min<uint64_t>(blocks, (yet->num_trials + 7) / 8);
    void* args[] = {&p};
    ARA_CUDA(cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(256), args, 0, s));
  }
  return ARA_OK;
}

ara_status ara_unshard(const double* gathered, uint32_t G, uint64_t cap, uint32_t L, const uint64_t* starts,
                       double* ylt, void* stream) {
  if (!gathered || !starts || !ylt || G == 0 || L == 0) return set_error(ARA_E_ARG, "invalid argument");
  if (starts[0] != 0) return set_error(ARA_E_ARG, "starts[0] must be 0");
  const uint64_t N = starts[G];
  for (uint32_t g = 0; g < G; ++g)
    if (starts[g + 1] < starts[g] || starts[g + 1] - starts[g] > cap)
      return set_error(ARA_E_ARG, "shard %u does not fit shard_cap", g);
  for (uint32_t g = 0; g < G; ++g) {
    uint64_t cnt = starts[g + 1] - starts[g];
    if (!cnt) continue;
    ARA_CUDA(cudaMemcpy2DAsync(ylt + starts[g], N * 8, gathered + (uint64_t)g * L * cap, cap * 8, cnt * 8, L,
                               cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  return ARA_OK;
}

ara_status ara_set_option(ara_ctx* c, ara_option opt, int64_t v) {
  if (!c) return set_error(ARA_E_ARG, "ctx is NULL");
  switch (opt) {
    case ARA_OPT_BLOCK_THREADS:
      if (v == 0) v = 256;
      if (v < 32 || v > 256 || v % 32) return set_error(ARA_E_ARG, "block threads must be a multiple of 32 in [32, 256]");
      c->block_threads = (int)v;
      return ARA_OK;
    case ARA_OPT_BLOCKS_PER_SM:
      if (v < 0 || v > 32) return set_error(ARA_E_ARG, "blocks per SM in [0, 32]");
      c->blocks_per_sm = (int)v;
      return ARA_OK;
    case ARA_OPT_L2_POLICY:
      if (v < 0 || v > 2) return set_error(ARA_E_ARG, "L2 policy in {0, 1, 2}");
      if (v == 2) {
        DeviceGuard guard(c->device);
        ARA_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)c->persist_max));
      }
      c->l2_policy = (int)v;
      return ARA_OK;
    case ARA_OPT_VARIANT:
      if (v < 0) return set_error(ARA_E_ARG, "variant >= 0");
      for (auto& L : c->layers)
        if (v >= (int64_t)L.variants[kind_of(c, L)].size())
          return set_error(ARA_E_ARG, "variant %lld not available", (long long)v);
      c->variant = (int)v;
      return ARA_OK;
    case ARA_OPT_KERNEL:
      if (v < -1 || v > 1) return set_error(ARA_E_ARG, "kernel in {-1 auto, 0 presence, 1 dense}");
      c->kernel = (int)v;
      c->variant = 0;
      return ARA_OK;
    case ARA_OPT_PREFETCH:
      if (v < -1 || v > 1) return set_error(ARA_E_ARG, "prefetch in {-1, 0, 1}");
      c->prefetch = (int)v;
      return ARA_OK;
    case ARA_OPT_FILTER:
      if (v < -1 || v > 1) return set_error(ARA_E_ARG, "filter in {-1, 0, 1}");
      c->filter = (int)v;
      return ARA_OK;
    case ARA_OPT_PRECOMBINED:
      if (v < 0 || v > 1) return set_error(ARA_E_ARG, "precombined in {0, 1}");
      c->precombined = (int)v;
      return ARA_OK;
    case ARA_OPT_FUSED:
      if (v < 0 || v > 1) return set_error(ARA_E_ARG, "fused in {0, 1}");
      c->fused = (int)v;
      return ARA_OK;
    case ARA_OPT_TRIAL_ORDER:
      if (v < 0 || v > 1) return set_error(ARA_E_ARG, "trial order in {0 blocks, 1 interleaved}");
      c->interleave = (int)v;
      return ARA_OK;
    case ARA_OPT_ROUND_MIN:
      if (v == 0) v = 24;
      if (v < 1 || v > 32) return set_error(ARA_E_ARG, "round trigger in [1, 32]");
      c->round_min = (int)v;
      return ARA_OK;
    case ARA_OPT_STREAM: {
      int n = 0;
      stream_variants(&n);
      if (v < 0 || v > n) return set_error(ARA_E_ARG, "stream kernel in [0, %d]", n);
      c->stream_kernel = (int)v;
      return ARA_OK;
    }
  }
  return set_error(ARA_E_ARG, "unknown option %d", (int)opt);
}

ara_status ara_get_option(ara_ctx* c, ara_option opt, int64_t* v) {
  if (!c || !v) return set_error(ARA_E_ARG, "NULL argument");
  switch (opt) {
    case ARA_OPT_BLOCK_THREADS: *v = c->block_threads; return ARA_OK;
    case ARA_OPT_BLOCKS_PER_SM: *v = c->blocks_per_sm; return ARA_OK;
    case ARA_OPT_L2_POLICY: *v = c->l2_policy; return ARA_OK;
    case ARA_OPT_VARIANT: *v = c->variant; return ARA_OK;
    case ARA_OPT_KERNEL: *v = c->kernel; return ARA_OK;
    case ARA_OPT_PREFETCH: *v = c->prefetch; return ARA_OK;
    case ARA_OPT_FILTER: *v = c->filter; return ARA_OK;
    case ARA_OPT_PRECOMBINED: *v = c->precombined; return ARA_OK;
    case ARA_OPT_STREAM: *v = c->stream_kernel; return ARA_OK;
    case ARA_OPT_ROUND_MIN: *v = c->round_min; return ARA_OK;
    case ARA_OPT_TRIAL_ORDER: *v = c->interleave; return ARA_OK;
    case ARA_OPT_FUSED: *v = c->fused; return ARA_OK;
  }
  return set_error(ARA_E_ARG, "unknown option %d", (int)opt);
}

ara_status ara_layer_info(ara_ctx* c, uint32_t layer, uint64_t* table_bytes, uint32_t* row_stride,
                          uint32_t* num_variants, const char** variant_name) {
  if (!c || layer >= c->layers.size()) return set_error(ARA_E_ARG, "invalid context or layer");
  const Layer& L = c->layers[layer];
  if (table_bytes) *table_bytes = L.table_bytes;
  if (row_stride) *row_stride = L.jpad * 4;
  if (num_variants) *num_variants = (uint32_t)L.variants[kind_of(c, L)].size();
  if (variant_name) *variant_name = pick(c, L)->name;
  return ARA_OK;
}

ara_status ara_layer_stats(ara_ctx* c, uint32_t layer, uint64_t* present_rows, double* est_hit_rate, int* kernel) {
  if (!c || layer >= c->layers.size()) return set_error(ARA_E_ARG, "invalid context or layer");
  const Layer& L = c->layers[layer];
  if (present_rows) *present_rows = L.present_rows;
  if (est_hit_rate) *est_hit_rate = L.est_hit_rate;
  if (kernel) *kernel = kind_of(c, L);
  return ARA_OK;
}


const char* ara_status_string(ara_status s) {
  switch (s) {
    case ARA_OK: return "ARA_OK";
    case ARA_E_ARG: return "ARA_E_ARG";
    case ARA_E_RANGE: return "ARA_E_RANGE";
    case ARA_E_DUP: return "ARA_E_DUP";
    case ARA_E_VALUE: return "ARA_E_VALUE";
    case ARA_E_NOMEM: return "ARA_E_NOMEM";
    case ARA_E_CUDA: return "ARA_E_CUDA";
    case ARA_E_UNSUPPORTED: return "ARA_E_UNSUPPORTED";
  }
  return "ARA_E_UNKNOWN";
}

const char* ara_last_error(void) { return g_err; }

const char* ara_kernel_name(ara_ctx* c) { return c ? c->last_kernel : ""; }

uint32_t ara_version(void) { return (ARA_VERSION_MAJOR << 16) | ARA_VERSION_MINOR; }

}  // extern "C"

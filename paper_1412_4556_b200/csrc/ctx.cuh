// ctx.cuh -- the context behind the opaque `ara_ctx` handle of include/ara.h: per-layer device tables,
// presence bitmaps, records and launch caches.  Internal to the library; shared with the test-only
// libara_testing.so (testing.cu), which reads a context's tables for the exhaustive table tests.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ara.h"
#include "ara_kernel.cuh"
#include "variants.cuh"

namespace ara {

struct Layer {
  uint32_t J = 0, jpad = 0;
  float* table = nullptr;
  uint64_t table_bytes = 0;
  uint32_t* present = nullptr;  // presence bitmap, (C + 1 + 31) / 32 words: bit e set iff row e holds a loss
  // the bitmap folded into the words a kernel's shared memory holds, one buffer per fold size (never
  // rebuilt in place, so a launch still reading one fold cannot see another being built)
  struct Fold {
    uint32_t words, mul;
    uint32_t* buf;
  };
  std::vector<Fold> folds;
  uint32_t fold_words = 0;  // canonical fold size of this layer (every presence/stream launch uses it)
  bool xs_auto = false;     // fixed-length trials: the exact scan filter pays (ARA_OPT_FILTER auto)
  uint4* rec = nullptr;         // sparse row records (C + 2) x 16 B; record C + 1 is all zero (invalid ids)
  uint2* xrank = nullptr;       // XS, built on first use: per bitmap word (word, loss-holding rows before it)
  uint4* rec_c = nullptr;       // XS: records of the loss-holding rows only (+ one zero record)
  double* occ = nullptr;        // precombined o[e] per event, (C + 1) x 8 B, built on first use
  // Section IV.B study structures, built on first use by ara_run_study
  float* indep = nullptr;         // J x (C + 1) independent per-ELT direct-access arrays
  uint32_t* sorted_ids = nullptr; // per-ELT (event, loss) pairs sorted by event
  float* sorted_loss = nullptr;
  uint32_t* sorted_off = nullptr; // J + 1
  uint2* hash = nullptr;           // STUDY_HASH tables, offsets and log2 capacities
  uint32_t* hash_off = nullptr;
  uint32_t* hash_bits = nullptr;
  uint32_t* row_index = nullptr;   // STUDY_INDEX: event -> compact row, and the compact rows
  float* compact = nullptr;
  uint32_t present_words = 0;
  std::vector<const Variant*> variants[2];  // by KernelKind
  uint64_t present_rows = 0;                // rows holding at least one loss
  double est_hit_rate = 0.0;                // expected share of occurrences gathered by the presence kernel
  int auto_kind = KIND_PRESENCE;            // kernel chosen when ARA_OPT_KERNEL is auto
  double r1[kMaxJ], l1[kMaxJ];
  double r2 = 0, l2 = 0, r3 = 0, l3 = 0;
};

}  // namespace ara

struct ara_ctx {
  int device = 0;
  // per-kernel static shared memory and the largest dynamic size already set (host-side launch cache)
  struct FnInfo {
    const void* fn;
    int static_smem;
    int dyn_set;
  };
  std::vector<FnInfo> fn_info;
  int sms = 148;
  uint32_t C = 0;
  std::vector<ara::Layer> layers;
  unsigned* d_err = nullptr;
  unsigned* h_err = nullptr;  // pinned
  // options
  int block_threads = 256;
  int blocks_per_sm = 0;
  int l2_policy = 0;
  int prefetch = -1;  // ARA_OPT_PREFETCH: -1 auto (stream kernel: on; presence kernel: off), 0 off, 1 on
  int filter = -1;  // ARA_OPT_FILTER: -1 auto, 0 off, 1 on
  int precombined = 0;  // ARA_OPT_PRECOMBINED: 1 = gather o[e] from the precombined table
  int variant = 0;
  int kernel = -1;  // KernelKind, or -1 = per-layer automatic choice
  int fused = 0;          // ARA_OPT_FUSED: 1 one pass over the YET per layer group, 0 layer-outer (default: measured faster on M)
  struct FusedGroup {       // layers [l0, l1) fused into one pass (fused_kernel.cuh)
    uint32_t l0 = 0, l1 = 0, cols = 0;
    uint4* rec = nullptr;           // (C + 2) x 32 B combined records
    uint32_t* present = nullptr;    // union presence bitmap
    std::vector<ara::Layer::Fold> folds;
  };
  std::vector<FusedGroup> groups;  // built on the first fused run
  bool groups_built = false;
  int interleave = 1;     // ARA_OPT_TRIAL_ORDER: 1 trials interleaved over the warps, 0 contiguous blocks
  int round_min = 24;     // ARA_OPT_ROUND_MIN: lane kernel round trigger (lanes holding a queued hit)
  int stream_kernel = 0;  // ARA_OPT_STREAM: 0 off, v > 0 = stream variant v - 1 for fixed-length trials
  const char* last_kernel = "";  // name of the kernel the last launch used (layer 0)
  int persist_max = 0, window_max = 0;
  int smem_optin = 0;
  // end-to-end host path
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  uint32_t* st_ids[2] = {nullptr, nullptr};
  uint64_t* st_off[2] = {nullptr, nullptr};
  double* st_ylt[2] = {nullptr, nullptr};
  uint64_t* h_off[2] = {nullptr, nullptr};  // pinned rebased offsets
  uint64_t st_cap_ids = 0, st_cap_trials = 0;
};

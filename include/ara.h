/* ara.h -- C ABI of the B200-native Aggregate Risk Analysis (ARA) hot path.
 *
 * Source of the method: Varghese & Barker, "Are Clouds Ready to Accelerate Ad hoc Financial
 * Simulations?", arXiv 1412.4556 (PAPER.md in the reference tree; citations are "PAPER.md:line").
 *
 *   Input  YET (Year Event Table), ELTs (Event Loss Tables + FT1), PF (layers + FT2/FT3)
 *   Output YLT (Year Loss Table), one loss per trial and layer
 *   For every layer, trial and event occurrence (Algorithm 1):
 *     1. look the event up in every ELT of the layer (0 if absent)
 *     2. apply FT1 per ELT, sum across the layer's ELTs
 *     3. apply the occurrence terms FT2 to that event loss
 *     4. accumulate over the trial's events and apply the aggregate terms FT3
 *   Every term is  min(max(x - retention, 0), limit)  (readings c1-c4).
 *   PML / TVaR are read from the YLT (readings c11-c14).
 *
 * Library: libara.so (paper_1412_4556_b200/libara.so), hand-written CUDA for sm_100a only.  No CPU
 * fallback exists: every compute step runs in the library's kernels.
 *
 * Conventions for every entry point:
 *   - Returns ara_status; never throws, never aborts.  On failure ara_last_error() holds a
 *     thread-local detail message and no partial object is returned.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Work is enqueued
 *     on it; functions say when they synchronise.
 *   - Arithmetic: ELT losses are fp32 (the stored ground truth); every term, sum and metric is fp64
 *     (reading c19).
 */
#ifndef ARA_H
#define ARA_H
#include <stdint.h>
#if defined(__GNUC__)
#define ARA_API __attribute__((visibility("default")))
#else
#define ARA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define ARA_VERSION_MAJOR 0
#define ARA_VERSION_MINOR 2
#define ARA_MAX_ELTS_PER_LAYER 128 /* compiled kernel set; more -> ARA_E_UNSUPPORTED (reading c16) */
#define ARA_MAX_RETURN_PERIODS 256

typedef enum {
  ARA_OK = 0,
  ARA_E_ARG = 1,         /* NULL pointer, zero count, bad index, duplicate layer ELT, bad offsets   */
  ARA_E_RANGE = 2,       /* event id outside [1, catalog_size]; return period outside (1, N]       */
  ARA_E_DUP = 3,         /* the same event id twice in one ELT                                     */
  ARA_E_VALUE = 4,       /* loss not finite or <= 0; retention < 0 / non-finite; limit <= 0 / NaN   */
  ARA_E_NOMEM = 5,       /* device or host allocation failed                                       */
  ARA_E_CUDA = 6,        /* CUDA runtime error (message from cudaGetErrorString)                   */
  ARA_E_UNSUPPORTED = 7  /* more than ARA_MAX_ELTS_PER_LAYER ELTs in a layer, not an sm_100 device */
} ara_status;

/* A (retention, limit) pair: FT1, FT2 or FT3.  retention finite and >= 0; limit > 0, may be +INFINITY. */
typedef struct {
  double retention;
  double limit;
} ara_terms;

/* One Event Loss Table: event-loss pairs plus its financial terms FT1.
 * HOST memory; copied by ara_create (caller may free on return).  Entries in any order; ids distinct
 * and in [1, catalog_size]; losses finite and > 0 (an event absent from the ELT has loss 0). */
typedef struct {
  const uint32_t* event_ids;
  const float* losses;
  uint64_t num_entries;
  ara_terms ft1;
} ara_elt;

/* One Layer: the ELTs it covers (indices into the ara_elt array, in the order the
 * per-ELT losses are summed) and its occurrence (FT2) and aggregate (FT3) terms.  Programs and the
 * portfolio are flattened into the list of layers: the paper defines no program-level terms
 * (reading c18).  HOST memory, copied. */
typedef struct {
  const uint32_t* elt_index;
  uint32_t num_elts; /* 1 .. ARA_MAX_ELTS_PER_LAYER, distinct indices */
  ara_terms occurrence; /* FT2 */
  ara_terms aggregate;  /* FT3 */
} ara_layer;

/* The Year Event Table: trials of event ids, each trial in time order (timestamps
 * only order events and are not passed, reading c8).  Layout: one contiguous uint32 array, trial-major.
 *   trial_offsets == NULL : trial t occupies event_ids[t*K .. (t+1)*K), K = events_per_trial
 *   trial_offsets != NULL : trial t occupies event_ids[off[t] .. off[t+1]); off has num_trials+1
 *                           non-decreasing entries, off[num_trials] <= num_events.  Empty trials allowed
 *                           (loss 0, reading c17).
 * num_events = number of uint32 ids the event_ids buffer holds (bounds every read).
 * Whether the pointers are host or device memory is fixed by the entry point that takes them. */
typedef struct {
  const uint32_t* event_ids;
  const uint64_t* trial_offsets;
  uint64_t num_trials;
  uint64_t num_events;
  uint32_t events_per_trial;
} ara_yet;

typedef struct ara_ctx ara_ctx; /* opaque; one per device (rank); not thread-safe, distinct contexts are */

/* Preprocessing stage: validate the ELTs and layers, and build on `device`, for every
 * layer, its event-major interleaved direct-access table: row e (e = 0..C) holds
 * the fp32 losses of event e in the layer's ELTs, in layer order, zero where absent; row 0 is all
 * zero.  Row stride = 4*J bytes rounded up to a power of two when <= 32 B, else to a multiple of
 * 32 B (ara_table_footprint).  Synchronises `stream` once.  On success *out owns all device memory.
 * Errors: ARA_E_ARG (NULL / zero counts / bad layer index / duplicate index in a layer),
 * ARA_E_RANGE (ELT id outside [1, C]), ARA_E_DUP, ARA_E_VALUE, ARA_E_UNSUPPORTED, ARA_E_NOMEM,
 * ARA_E_CUDA. */
ARA_API ara_status ara_create(uint32_t catalog_size, const ara_elt* elts, uint32_t num_elts, const ara_layer* layers,
                      uint32_t num_layers, int device, void* stream, ara_ctx** out);

ARA_API void ara_destroy(ara_ctx* ctx); /* NULL is a no-op; synchronises the device before freeing */

/* The analysis stage (Algorithm 1) over a DEVICE-resident YET (borrowed; must stay
 * alive and unmodified until the work on `stream` completes).  Writes ylt[l * num_trials + t]
 * (DEVICE, caller-allocated, num_layers * num_trials doubles).  Layer-outer order (one pass over the
 * YET per layer).  Asynchronous: invalid ids / offsets found by the kernels are
 * recorded in the context and reported by ara_check (the offending occurrences contribute 0).
 * Errors (immediate): ARA_E_ARG (NULL, num_events too small for fixed-length trials), ARA_E_CUDA. */
ARA_API ara_status ara_run(ara_ctx* ctx, const ara_yet* yet, double* ylt, void* stream);

/* ara_run plus the occurrence-basis loss table: olt[l * num_trials + t] = the largest occurrence-net
 * loss (FT2 output) over trial t's events under layer l, 0 for a trial without events (DEVICE,
 * caller-allocated like ylt; NULL = not produced).  PML/TVaR of an OLT row are OEP-basis metrics
 * (SURVEY.md N4).  Same conventions and errors as ara_run. */
ARA_API ara_status ara_run_ex(ara_ctx* ctx, const ara_yet* yet, double* ylt, double* olt, void* stream);

/* A captured analysis step for repeated runs over the same device buffers (PAPER.md:230 times many runs
 * of one workload): ara_run over `yet` (DEVICE, borrowed) into ylt, then PML/TVaR of every layer at the
 * m return periods into pml_dev / tvar_dev (DEVICE, [num_layers][m] each, either may be NULL; m = 0:
 * no metrics).  ara_plan_create runs the step once eagerly (building every cached structure and
 * validating the arguments), then records it into a CUDA graph with all scratch preallocated;
 * ara_plan_launch replays it on `stream` with one graph launch (asynchronous; the results are the
 * same as the eager calls, bit for bit).  The buffers must stay alive until ara_plan_destroy.  Invalid
 * ids are reported by ara_check as for ara_run.  Errors: as ara_run and ara_pml_tvar_device, plus
 * ARA_E_CUDA when the graph cannot be captured. */
typedef struct ara_plan ara_plan;
ARA_API ara_status ara_plan_create(ara_ctx* ctx, const ara_yet* yet, double* ylt, const double* rps, uint32_t m,
                                   double* pml_dev, double* tvar_dev, void* stream, ara_plan** out);
ARA_API ara_status ara_plan_launch(ara_plan* plan, void* stream);
ARA_API void ara_plan_destroy(ara_plan* plan); /* NULL is a no-op */
/* A captured PML/TVaR step (readings c11-c14): the metrics of num_layers DEVICE YLTs of
 * n values each (layer l at ylt + l * n, borrowed) at the m return periods, recorded once into a CUDA
 * graph with its scratch allocated and zeroed beforehand (no per-call allocation or memset); layer l's
 * results go to pml_dev + l * out_stride and tvar_dev + l * out_stride (DEVICE, m doubles each; either
 * may be NULL; out_stride >= m when num_layers > 1).  Runs once eagerly, then ara_plan_launch replays it;
 * results equal ara_pml_tvar_device bit for bit.  Errors: as ara_pml_tvar_device, plus ARA_E_CUDA when
 * the graph cannot be captured. */
ARA_API ara_status ara_metrics_plan_create(const double* ylt, uint64_t n, uint32_t num_layers, const double* rps,
                                           uint32_t m, double* pml_dev, double* tvar_dev, uint64_t out_stride,
                                           void* stream, ara_plan** out);

/* End-to-end variant for a HOST YET (pinned memory gives copy/compute overlap; pageable works but
 * serialises): the YET is streamed to the device in trial batches on an internal copy stream,
 * overlapped with the analysis of the previous batch, and the YLT is written to HOST ylt_host
 * ([num_layers][num_trials]).  Synchronous: returns when ylt_host is complete, with the ara_check
 * result folded in (ARA_E_RANGE / ARA_E_ARG for invalid ids / offsets). */
ARA_API ara_status ara_run_host(ara_ctx* ctx, const ara_yet* yet, double* ylt_host, void* stream);

/* Synchronise `stream` and report (then clear) invalid input seen by earlier ara_run calls:
 * ARA_E_RANGE = an event id outside [1, C]; ARA_E_ARG = decreasing or out-of-bounds trial offsets. */
ARA_API ara_status ara_check(ara_ctx* ctx, void* stream);

/* Probable Maximum Loss and Tail Value-at-Risk of a DEVICE YLT of n values >= 0 at m return periods
 * (readings c11, c12, c14): k = ceil(n / RP) -- exact integer ceil for integral RP, ceil(x - 1e-9 x),
 * x = n / RP, otherwise; PML = k-th largest value; TVaR = mean of the k largest.  Computed with one
 * cooperative launch of a device MSD radix select on the fp64 bit patterns (a 16-bit pass, 12-bit passes
 * only while a query's bucket holds > 256 values, then compaction; ranks on the maximum/minimum tie
 * blocks resolve after the first pass) plus a deterministic fp64 sum: results are bitwise reproducible
 * and, for integer-valued YLTs, bitwise equal to the sorted definition.  Results to HOST out arrays of m
 * doubles; synchronises `stream`.  NaN values are not supported (their order is undefined).
 * Errors: ARA_E_ARG (NULL, n == 0, m == 0 or m > ARA_MAX_RETURN_PERIODS), ARA_E_RANGE (RP not in
 * (1, n] or not finite), ARA_E_NOMEM, ARA_E_CUDA. */
ARA_API ara_status ara_pml_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_out,
                        double* tvar_out, void* stream);
/* Asynchronous form: results to DEVICE pml_dev[m] / tvar_dev[m] (either may be NULL), enqueued on
 * `stream` without synchronising, so successive analyses pipeline without host round trips.
 * ARA_E_UNSUPPORTED if the device refuses the cooperative launch the fused kernel needs. */
ARA_API ara_status ara_pml_tvar_device(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* pml_dev,
                                       double* tvar_dev, void* stream);
ARA_API ara_status ara_pml(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out, void* stream);
ARA_API ara_status ara_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out, void* stream);

/* Section IV.B data-structure study: Algorithm 1 with the same plain kernel (one
 * warp per trial, one lane per occurrence) over one of three ELT representations, for comparing their
 * memory behaviour on B200 -- not the product path:
 *   0 ARA_STUDY_INTERLEAVED  the combined event-major table (one row per event)
 *   1 ARA_STUDY_INDEPENDENT  one direct-access array per ELT (the paper's GPU choice)
 *   2 ARA_STUDY_SORTED       per-ELT arrays sorted by event id, binary search
 *   3 ARA_STUDY_HASH         per-ELT open-addressing hash tables, load factor <= 1/2 (PAPER.md:211,
 *                            "constant-time hash search")
 *   4 ARA_STUDY_INDEX        an event -> compact-row index plus the rows holding a loss
 * The extra structures are built on first use (layouts 2-4 copy the table to the host once).  Same
 * YET / YLT conventions as ara_run; asynchronous except for that first build.  Invalid ids read as
 * absent and are not reported. */
typedef enum {
  ARA_STUDY_INTERLEAVED = 0,
  ARA_STUDY_INDEPENDENT = 1,
  ARA_STUDY_SORTED = 2,
  ARA_STUDY_HASH = 3,
  ARA_STUDY_INDEX = 4
} ara_study_layout;
ARA_API ara_status ara_run_study(ara_ctx* ctx, int layout, const ara_yet* yet, double* ylt, void* stream);

/* Average annual loss of a DEVICE YLT of n values: the mean, reduced in a fixed order (bitwise
 * reproducible).  Result to HOST *out; synchronises `stream`.  ARA_E_ARG for NULL / n == 0. */
ARA_API ara_status ara_aal(const double* ylt, uint64_t n, double* out, void* stream);

/* Exceedance probabilities of a DEVICE YLT at m HOST thresholds: out[i] = #{t : ylt[t] >= x[i]} / n
 * (the EP curve behind return-period loss reports).  1 <= m <= 256.
 * Results to HOST out; synchronises `stream`. */
ARA_API ara_status ara_ep(const double* ylt, uint64_t n, const double* thresholds, uint32_t m, double* out,
                          void* stream);

/* Program / portfolio totals (a portfolio groups programs, a program groups layers):
 * out[g * n + t] = sum over layers l with group[l] == g, in layer order, of ylt[l * n + t].
 * ylt, out: DEVICE ([num_layers][n], [num_groups][n]); group: HOST, num_layers entries < num_groups;
 * num_layers <= 128.  Asynchronous. */
ARA_API ara_status ara_sum_layers(const double* ylt, uint32_t num_layers, uint64_t n, const uint32_t* group,
                                  uint32_t num_groups, double* out, void* stream);

/* Host-only memory accounting of one layer's direct-access table: bytes of the
 * (C+1)-row table and its row stride.  No device needed. */
ARA_API ara_status ara_table_footprint(uint32_t catalog_size, uint32_t num_elts, uint64_t* bytes, uint32_t* row_stride);

/* Multi-GPU reassembly: copy G padded YLT shards gathered as [G][num_layers][shard_cap] (DEVICE)
 * into ylt ([num_layers][num_trials], DEVICE), shard g holding trials [starts[g], starts[g+1]).
 * starts: HOST array of G+1 entries, starts[0] = 0, starts[G] = num_trials, each shard <= shard_cap.
 * Asynchronous device-to-device copies on `stream`. */
ARA_API ara_status ara_unshard(const double* gathered, uint32_t num_shards, uint64_t shard_cap, uint32_t num_layers,
                       const uint64_t* starts, double* ylt, void* stream);

/* Tuning knobs (launch-shape sweep; L2 policy).  0 = library default.
 *   ARA_OPT_BLOCK_THREADS   threads per block of the dense kernel (multiple of 32, 32..256)
 *   ARA_OPT_BLOCKS_PER_SM   resident blocks per SM the persistent grid is sized for
 *   ARA_OPT_L2_POLICY       0 default (evict_last hints on table rows and records; the dense kernel
 *                           also marks YET ids evict_first), 1 no hints, 2 hints + persisting
 *                           access-policy window on the table
 *   ARA_OPT_PREFETCH        L2 prefetch of the YET ahead of the register-staged windows: -1 auto
 *                           (default: on for the per-lane-queue and warp-ring kernels -- one bulk
 *                           prefetch of the trial after next per trial --, off for the presence and
 *                           candidate-mask kernels), 0 off, 1 on
 *                           (presence kernel: each warp prefetches its next trial at a trial start)
 *   ARA_OPT_VARIANT         kernel variant index within the selected kernel and row width
 *                           (ara_layer_info reports the count)
 *   ARA_OPT_KERNEL          -1 auto (default): per layer, the presence kernel when its folded bitmap is
 *                           expected to send at most 60% of the occurrences to the gather (25% when
 *                           more than 5% of the non-zero rows hold more than two losses: those rows
 *                           are read in full instead of through their 16-B sparse record), else the
 *                           dense kernel;
 *                           0 presence: a per-layer presence bitmap of the table's non-zero rows,
 *                           staged in shared memory, so only rows that hold a loss are gathered;
 *                           1 dense: every occurrence gathers its full row.  The same YLT up to
 *                           the fp64 summation order (an all-zero row contributes exactly 0, PAPER.md:209,
 *                           reading c9): bitwise identical in the integer regime, equal to the rounding
 *                           of the summation order otherwise (each kernel's order is fixed, so each is
 *                           reproducible).
 *                           Selecting a kernel resets ARA_OPT_VARIANT to 0.
 *   ARA_OPT_FILTER          presence kernel, one lane per row: -1 auto (default; = off), 0 off, 1 on.
 *                           The exact filter stage checks every candidate of the folded shared-memory
 *                           bitmap against the layer's unfolded presence bitmap (global memory,
 *                           L2-resident) before fetching its record: 4x less DRAM traffic on config X,
 *                           but measured slower there, hence off.  Identical results either way.
 *   ARA_OPT_PRECOMBINED     0 (default) or 1: ablation of SURVEY.md 8(f) N3.  Steps 1-3 depend only on
 *                           the event, so the presence kernel may gather a per-layer table
 *                           o[e] = FT2(sum_j FT1(l_ej)) (fp64, (C+1) x 8 B, built on the first run
 *                           with the option set) instead of the sparse records.  Bitwise identical
 *                           YLT; exact only for deterministic losses (no secondary uncertainty,
 *                           PAPER.md:125), and no ELT lookups happen at run time.
 *   ARA_OPT_STREAM          0 (default): the presence kernel.  v > 0: for a YET of fixed-length trials
 *                           (no offsets, K % 4 == 0, 16-B aligned ids, catalogue < 2^32 - 2) the
 *                           presence path runs a fixed-length-trial kernel instead: v = 1..3 the
 *                           per-lane-queue kernel (lane_kernel.cuh: each lane queues the hits of its
 *                           own window positions and sums them in stream order; 32, 24, 16 warps per
 *                           block), v = 4 the warp-ring kernel (stream_kernel.cuh: the presence
 *                           kernel's summation order), v = 5..8 the per-lane-queue kernel with the
 *                           exact scan filter (see ARA_OPT_FILTER), v = 9, 10 the candidate-mask kernel
 *                           (mask_kernel.cuh; 897 <= K <= 1024 only, else the presence kernel runs;
 *                           10 adds a per-lane L2 prefetch four windows ahead).  Every kernel's order
 *                           is fixed: the YLT is
 *                           reproducible bit for bit and independent of the sharding; across kernels it
 *                           agrees bitwise in the integer regime and to the rounding of the summation
 *                           order otherwise (amplified by FT3 when S_n is close to its retention).
 *   ARA_OPT_ROUND_MIN       per-lane-queue kernel: a gather round starts when at least this many lanes
 *                           hold a queued hit (1..32, 0 = default 24), or when a queue nearly fills.
 *   ARA_OPT_TRIAL_ORDER     fixed-length-trial kernels: 1 (default) trials interleaved over the grid's
 *                           warps (warp w takes trials w, w + W, ...: all warps stream one compact
 *                           region of the YET), 0 contiguous trial blocks per warp.  Same YLT bits.
 *   ARA_OPT_FUSED           0 (default) layer-outer passes; 1: a run over several layers streams a fixed-length YET ONCE per
 *                           group of consecutive sparse-path layers (<= 16 layers, <= 256 ELT columns;
 *                           SURVEY.md N1; fused_kernel.cuh: union presence bitmap, combined per-event
 *                           records, per-layer accumulators) instead of Algorithm 1's layer-outer loop
 *                           (PAPER.md:104-105).  Measured slower on config M (N1), hence off.
 *                           Not used for the occurrence loss table (ara_run_ex
 *                           with olt), ragged YETs, or when ARA_OPT_STREAM / ARA_OPT_KERNEL select a kernel.
 * ARA_OPT_BLOCK_THREADS applies to the dense kernel; the presence kernel fixes its block size. */
typedef enum {
  ARA_OPT_BLOCK_THREADS = 1,
  ARA_OPT_BLOCKS_PER_SM = 2,
  ARA_OPT_L2_POLICY = 3,
  ARA_OPT_VARIANT = 4,
  ARA_OPT_KERNEL = 5,
  ARA_OPT_PREFETCH = 6,
  ARA_OPT_FILTER = 7,
  ARA_OPT_PRECOMBINED = 8,
  ARA_OPT_STREAM = 9,
  ARA_OPT_ROUND_MIN = 10,
  ARA_OPT_TRIAL_ORDER = 11,
  ARA_OPT_FUSED = 12
} ara_option;
ARA_API ara_status ara_set_option(ara_ctx* ctx, ara_option opt, int64_t value);
ARA_API ara_status ara_get_option(ara_ctx* ctx, ara_option opt, int64_t* value);

/* Introspection for the bench / tests: bytes of layer l's table, its row stride, number of kernel
 * variants for its J, and a description of the selected variant (static string). */
ARA_API ara_status ara_layer_info(ara_ctx* ctx, uint32_t layer, uint64_t* table_bytes, uint32_t* row_stride,
                          uint32_t* num_variants, const char** variant_name);

/* Presence statistics of layer l (computed by ara_create on the host): rows of the table that hold at
 * least one loss, the expected share of occurrences the presence kernel sends to the row gather (its
 * folded shared-memory bitmap), and the kernel that runs for this layer under the current
 * ARA_OPT_KERNEL (0 presence, 1 dense).  Any output pointer may be NULL. */
ARA_API ara_status ara_layer_stats(ara_ctx* ctx, uint32_t layer, uint64_t* present_rows, double* est_hit_rate,
                                   int* kernel);

/* Name of the kernel the most recent ara_run / ara_run_ex / ara_run_host of this context launched for
 * its last layer (a static string; "" before the first run). */
ARA_API const char* ara_kernel_name(ara_ctx* ctx);

/* (The test-only table read-back, ara_table_row, lives in libara_testing.so: include/ara_testing.h.) */

ARA_API const char* ara_status_string(ara_status s);
ARA_API const char* ara_last_error(void);
ARA_API uint32_t ara_version(void); /* (major << 16) | minor */

#ifdef __cplusplus
}
#endif
#endif

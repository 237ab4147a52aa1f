/* ara_oracle.h -- plain, slow, obviously-correct CPU oracle for Aggregate Risk Analysis.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_1412_4556_b200/csrc, include/ara.h) and neither includes the other.
 *
 * What it computes (PAPER.md = Varghese & Barker, arXiv 1412.4556):
 *   Algorithm 1 "Aggregate Risk Analysis" in the paper's loop order
 *   Layer -> Trial -> Event -> ELT, with the four steps of PAPER.md:123-129 (Section III):
 *     step 1 lookup l_E of event E in each ELT   -- 0 if absent
 *     step 2 apply FT1 per ELT and sum across the ELTs
 *     step 3 occurrence terms FT2 on the event loss
 *     step 4 aggregate terms FT3 on the trial's cumulative sum
 *   Every financial term is  min(max(x - retention, 0), limit)  (reading c1 of
 *   the printed one-argument max is max(., 0)).  FT1 = (retention, limit) (reading c3).
 *   All arithmetic is IEEE fp64 evaluated in exactly this order; ELT losses are fp32 values
 *   converted exactly to fp64 (reading c19).
 *   PML / TVaR (named, not defined): empirical, k = ceil(N / RP); PML = k-th
 *   largest YLT value; TVaR = mean of the k largest, summed largest-first (readings c11, c12, c14).
 *
 * Lookup: each ELT is held as its own array sorted by event id and searched by binary search, or --
 * brute force -- by a linear scan of the unsorted entries (PAPER.md:211 names both).  It is NOT the
 * direct-access table of the GPU path.
 *
 * Pins (tests/test_oracle_*.py): hand-worked trials (SPEC example -> 140; extended example of
 * SURVEY.md 8(c)), closed forms (identity terms = sum of raw lookups, power-of-two scaling),
 * invariants (bounds, monotonicity, permutation, telescoping), brute-force enumeration, and the
 * metric examples on losses 1..10.  The paper prints no YLT/PML/TVaR values: value-level parity
 * against the paper itself is unpinned.
 */
#ifndef ARA_ORACLE_H
#define ARA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_OK = 0, ORACLE_E_ARG = 1, ORACLE_E_RANGE = 2, ORACLE_E_NOMEM = 5 };
enum { ORACLE_LOOKUP_BINARY = 0, ORACLE_LOOKUP_LINEAR = 1 };

typedef struct {
  const uint32_t* event_ids; /* n entries, any order, distinct */
  const float* losses;       /* n entries, > 0 */
  uint64_t n;
  double ft1_retention, ft1_limit; /* FT1 (limit may be +inf) */
} oracle_elt;

typedef struct {
  const uint32_t* elt_index; /* indices into the ELT array, layer order */
  uint32_t num_elts;
  double ft2_retention, ft2_limit; /* occurrence terms */
  double ft3_retention, ft3_limit; /* aggregate terms */
} oracle_layer;

/* min(max(x - retention, 0), limit); never returns -0.0 for x >= 0. */
double oracle_clamp(double x, double retention, double limit);

/* Algorithm 1.  yet_ids: trial-major event ids in time order; offsets: [num_trials+1] start offsets
 * (NULL => every trial has events_per_trial events).  ylt: [num_layers][num_trials] output.
 * threads <= 0 => all online cores; threads take contiguous trial blocks.
 * Returns ORACLE_E_RANGE if any id is outside [1, catalog_size]. */
int oracle_ylt(uint32_t catalog_size, const uint32_t* yet_ids, const uint64_t* offsets, uint64_t num_trials,
               uint32_t events_per_trial, const oracle_elt* elts, uint32_t num_elts, const oracle_layer* layers,
               uint32_t num_layers, int lookup_mode, int threads, double* ylt);

/* Same as oracle_ylt, also writing olt[l][t] = the largest occurrence-net loss o of trial t under
 * layer l (0 for an empty trial): the occurrence-basis loss table behind OEP metrics (
 * SPEC.md:460 names the occurrence basis).  olt may be NULL. */
int oracle_ylt_olt(uint32_t catalog_size, const uint32_t* yet_ids, const uint64_t* offsets, uint64_t num_trials,
                   uint32_t events_per_trial, const oracle_elt* elts, uint32_t num_elts, const oracle_layer* layers,
                   uint32_t num_layers, int lookup_mode, int threads, double* ylt, double* olt);

/* Average annual loss: the mean of the YLT, summed in trial order ("AAL"). */
double oracle_aal(const double* ylt, uint64_t n);

/* Exceedance probability at m thresholds: #{t : ylt[t] >= x} / n (SPEC.md:402-408 exceedance_curve). */
void oracle_ep(const double* ylt, uint64_t n, const double* x, uint32_t m, double* out);

/* One trial, one layer, event by event: o[k] occurrence-net loss, S[k] prefix sum, a[k] =
 * F3(S_k) - F3(S_{k-1}) per-event aggregate-net loss (SPEC.md "incremental erosion").  Returns the
 * trial loss F3(S_n) through *ylt. */
int oracle_trial_detail(uint32_t catalog_size, const uint32_t* ids, uint64_t n, const oracle_elt* elts,
                        uint32_t num_elts, const oracle_layer* layer, int lookup_mode, double* o, double* S,
                        double* a, double* ylt);

/* Metric rank k = ceil(N/RP): integral RP -> exact integer ceil; otherwise ceil(N/RP - 1e-9*N/RP).
 * Returns 0 if RP is not in (1, N] or not finite. */
uint64_t oracle_rank(uint64_t n, double rp);

/* PML and TVaR at m return periods.  Returns ORACLE_E_RANGE for an invalid RP. */
int oracle_pml(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out);
int oracle_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out);

/* Number of threads oracle_ylt would use for threads <= 0. */
int oracle_default_threads(void);

#ifdef __cplusplus
}
#endif
#endif

/* ara_oracle.c -- TEST INFRASTRUCTURE ONLY (see ara_oracle.h).  Plain C99, fp64, paper order.
 * Compiled with -O2 -ffp-contract=off so every double operation is evaluated as written. */
#define _GNU_SOURCE
#include "ara_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* PAPER.md:127 (FT2), :129 (FT3), reading c3 for FT1: min(max(x - R, 0), L). */
double oracle_clamp(double x, double retention, double limit) {
  double y = x - retention;
  y = (y > 0.0) ? y : 0.0;
  return (y < limit) ? y : limit;
}

/* ---- one ELT as its own sorted (id, loss) array: the oracle's own lookup structure ------------- */
typedef struct {
  uint32_t* ids;
  float* losses;
  uint64_t n;
  const oracle_elt* src;
} sorted_elt;

typedef struct {
  uint32_t id;
  float loss;
} pair_t;

static int cmp_pair(const void* a, const void* b) {
  uint32_t x = ((const pair_t*)a)->id, y = ((const pair_t*)b)->id;
  return (x > y) - (x < y);
}

static int build_sorted(const oracle_elt* e, sorted_elt* s) {
  pair_t* p = (pair_t*)malloc((e->n ? e->n : 1) * sizeof(pair_t));
  s->ids = (uint32_t*)malloc((e->n ? e->n : 1) * sizeof(uint32_t));
  s->losses = (float*)malloc((e->n ? e->n : 1) * sizeof(float));
  if (!p || !s->ids || !s->losses) {
    free(p);
    return ORACLE_E_NOMEM;
  }
  for (uint64_t i = 0; i < e->n; ++i) {
    p[i].id = e->event_ids[i];
    p[i].loss = e->losses[i];
  }
  qsort(p, e->n, sizeof(pair_t), cmp_pair);
  for (uint64_t i = 0; i < e->n; ++i) {
    s->ids[i] = p[i].id;
    s->losses[i] = p[i].loss;
  }
  free(p);
  s->n = e->n;
  s->src = e;
  return ORACLE_OK;
}

/* Step 1: "Lookup E in the ELT and find corresponding loss"; 0 if absent. */
static double lookup_binary(const sorted_elt* s, uint32_t e) {
  uint64_t lo = 0, hi = s->n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (s->ids[mid] < e)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < s->n && s->ids[lo] == e) return (double)s->losses[lo];
  return 0.0;
}

static double lookup_linear(const oracle_elt* src, uint32_t e) {
  for (uint64_t i = 0; i < src->n; ++i)
    if (src->event_ids[i] == e) return (double)src->losses[i];
  return 0.0;
}

static double lookup(const sorted_elt* s, uint32_t e, int mode) {
  return mode == ORACLE_LOOKUP_LINEAR ? lookup_linear(s->src, e) : lookup_binary(s, e);
}

/* Steps 1-3 for one event occurrence E of a trial under one layer:
 *   l_E = sum over the layer's ELTs (layer order) of FT1(lookup(E))
 *   o   = FT2(l_E) */
static double occurrence_loss(uint32_t e, const sorted_elt* tabs, const oracle_elt* elts, const oracle_layer* L,
                              int mode) {
  double s = 0.0;
  for (uint32_t m = 0; m < L->num_elts; ++m) {
    uint32_t j = L->elt_index[m];
    double x = lookup(&tabs[j], e, mode);
    s = s + oracle_clamp(x, elts[j].ft1_retention, elts[j].ft1_limit);
  }
  return oracle_clamp(s, L->ft2_retention, L->ft2_limit);
}

typedef struct {
  uint32_t C;
  const uint32_t* ids;
  const uint64_t* offsets;
  uint32_t K;
  const sorted_elt* tabs;
  const oracle_elt* elts;
  const oracle_layer* layer;
  int mode;
  uint64_t t_lo, t_hi;
  double* ylt; /* this layer's row */
  double* olt; /* this layer's occurrence-loss row, or NULL */
} work_t;

static void* run_block(void* arg) {
  work_t* w = (work_t*)arg;
  for (uint64_t t = w->t_lo; t < w->t_hi; ++t) {
    uint64_t b = w->offsets ? w->offsets[t] : t * (uint64_t)w->K;
    uint64_t e = w->offsets ? w->offsets[t + 1] : b + w->K;
    double S = 0.0; /* step 4: cumulative sum of occurrence-net losses, event (time) order */
    double M = 0.0; /* largest occurrence-net loss of the trial */
    for (uint64_t k = b; k < e; ++k) {
      double o = occurrence_loss(w->ids[k], w->tabs, w->elts, w->layer, w->mode);
      S = S + o;
      if (o > M) M = o;
    }
    w->ylt[t] = oracle_clamp(S, w->layer->ft3_retention, w->layer->ft3_limit); /* FT3 */
    if (w->olt) w->olt[t] = M;
  }
  return NULL;
}

int oracle_default_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static int check_inputs(uint32_t C, const oracle_elt* elts, uint32_t num_elts, const oracle_layer* layers,
                        uint32_t num_layers) {
  if (C == 0) return ORACLE_E_ARG;
  for (uint32_t l = 0; l < num_layers; ++l)
    for (uint32_t m = 0; m < layers[l].num_elts; ++m)
      if (layers[l].elt_index[m] >= num_elts) return ORACLE_E_ARG;
  for (uint32_t j = 0; j < num_elts; ++j)
    for (uint64_t i = 0; i < elts[j].n; ++i)
      if (elts[j].event_ids[i] < 1 || elts[j].event_ids[i] > C) return ORACLE_E_RANGE;
  return ORACLE_OK;
}

int oracle_ylt(uint32_t catalog_size, const uint32_t* yet_ids, const uint64_t* offsets, uint64_t num_trials,
               uint32_t events_per_trial, const oracle_elt* elts, uint32_t num_elts, const oracle_layer* layers,
               uint32_t num_layers, int lookup_mode, int threads, double* ylt) {
  return oracle_ylt_olt(catalog_size, yet_ids, offsets, num_trials, events_per_trial, elts, num_elts, layers,
                        num_layers, lookup_mode, threads, ylt, NULL);
}

int oracle_ylt_olt(uint32_t catalog_size, const uint32_t* yet_ids, const uint64_t* offsets, uint64_t num_trials,
                   uint32_t events_per_trial, const oracle_elt* elts, uint32_t num_elts, const oracle_layer* layers,
                   uint32_t num_layers, int lookup_mode, int threads, double* ylt, double* olt) {
  int rc = check_inputs(catalog_size, elts, num_elts, layers, num_layers);
  if (rc) return rc;
  uint64_t total = offsets ? offsets[num_trials] - offsets[0] : num_trials * (uint64_t)events_per_trial;
  uint64_t first = offsets ? offsets[0] : 0;
  for (uint64_t q = first; q < first + total; ++q)
    if (yet_ids[q] < 1 || yet_ids[q] > catalog_size) return ORACLE_E_RANGE;

  sorted_elt* tabs = (sorted_elt*)calloc(num_elts ? num_elts : 1, sizeof(sorted_elt));
  if (!tabs) return ORACLE_E_NOMEM;
  for (uint32_t j = 0; j < num_elts; ++j)
    if ((rc = build_sorted(&elts[j], &tabs[j]))) goto done;

  if (threads <= 0) threads = oracle_default_threads();
  if ((uint64_t)threads > num_trials) threads = num_trials ? (int)num_trials : 1;
  pthread_t* th = (pthread_t*)malloc(threads * sizeof(pthread_t));
  work_t* w = (work_t*)malloc(threads * sizeof(work_t));
  if (!th || !w) {
    free(th);
    free(w);
    rc = ORACLE_E_NOMEM;
    goto done;
  }
  /* Algorithm 1: for each layer, for each trial (trials split into contiguous
   * blocks, one per thread -- "each trial in the YET is executed using a single thread"). */
  for (uint32_t l = 0; l < num_layers; ++l) {
    for (int i = 0; i < threads; ++i) {
      w[i] = (work_t){catalog_size, yet_ids, offsets, events_per_trial, tabs, elts, &layers[l], lookup_mode,
                      num_trials * (uint64_t)i / threads, num_trials * (uint64_t)(i + 1) / threads,
                      ylt + (uint64_t)l * num_trials, olt ? olt + (uint64_t)l * num_trials : NULL};
      if (threads == 1)
        run_block(&w[i]);
      else
        pthread_create(&th[i], NULL, run_block, &w[i]);
    }
    if (threads > 1)
      for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  }
  free(th);
  free(w);
done:
  for (uint32_t j = 0; j < num_elts; ++j) {
    free(tabs[j].ids);
    free(tabs[j].losses);
  }
  free(tabs);
  return rc;
}

int oracle_trial_detail(uint32_t catalog_size, const uint32_t* ids, uint64_t n, const oracle_elt* elts,
                        uint32_t num_elts, const oracle_layer* layer, int lookup_mode, double* o, double* S,
                        double* a, double* ylt) {
  int rc = check_inputs(catalog_size, elts, num_elts, layer, 1);
  if (rc) return rc;
  for (uint64_t k = 0; k < n; ++k)
    if (ids[k] < 1 || ids[k] > catalog_size) return ORACLE_E_RANGE;
  sorted_elt* tabs = (sorted_elt*)calloc(num_elts ? num_elts : 1, sizeof(sorted_elt));
  if (!tabs) return ORACLE_E_NOMEM;
  for (uint32_t j = 0; j < num_elts; ++j)
    if ((rc = build_sorted(&elts[j], &tabs[j]))) goto done;
  double run = 0.0, prev = 0.0;
  for (uint64_t k = 0; k < n; ++k) {
    double ok = occurrence_loss(ids[k], tabs, elts, layer, lookup_mode);
    run = run + ok;
    double f = oracle_clamp(run, layer->ft3_retention, layer->ft3_limit);
    if (o) o[k] = ok;
    if (S) S[k] = run;
    if (a) a[k] = f - prev;
    prev = f;
  }
  if (ylt) *ylt = oracle_clamp(run, layer->ft3_retention, layer->ft3_limit);
done:
  for (uint32_t j = 0; j < num_elts; ++j) {
    free(tabs[j].ids);
    free(tabs[j].losses);
  }
  free(tabs);
  return rc;
}

/* ---- metrics (readings c11, c12, c14) ------------------------------------------------------ */
uint64_t oracle_rank(uint64_t n, double rp) {
  if (!(rp > 1.0) || !(rp <= (double)n) || !isfinite(rp)) return 0;
  if (rp == floor(rp) && rp < 9007199254740992.0) {
    uint64_t r = (uint64_t)rp;
    return (n + r - 1) / r; /* exact integer ceil(N / RP) */
  }
  double x = (double)n / rp;
  return (uint64_t)ceil(x - 1e-9 * x);
}

static int cmp_desc(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

static double* sorted_desc(const double* y, uint64_t n) {
  double* c = (double*)malloc((n ? n : 1) * sizeof(double));
  if (!c) return NULL;
  memcpy(c, y, n * sizeof(double));
  qsort(c, n, sizeof(double), cmp_desc);
  return c;
}

int oracle_pml(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out) {
  for (uint32_t i = 0; i < m; ++i)
    if (!oracle_rank(n, rps[i])) return ORACLE_E_RANGE;
  double* c = sorted_desc(ylt, n);
  if (!c) return ORACLE_E_NOMEM;
  for (uint32_t i = 0; i < m; ++i) out[i] = c[oracle_rank(n, rps[i]) - 1]; /* k-th largest */
  free(c);
  return ORACLE_OK;
}

int oracle_tvar(const double* ylt, uint64_t n, const double* rps, uint32_t m, double* out) {
  for (uint32_t i = 0; i < m; ++i)
    if (!oracle_rank(n, rps[i])) return ORACLE_E_RANGE;
  double* c = sorted_desc(ylt, n);
  if (!c) return ORACLE_E_NOMEM;
  for (uint32_t i = 0; i < m; ++i) {
    uint64_t k = oracle_rank(n, rps[i]);
    double s = 0.0;
    for (uint64_t q = 0; q < k; ++q) s = s + c[q]; /* largest first */
    out[i] = s / (double)k;                         /* mean of the k largest */
  }
  free(c);
  return ORACLE_OK;
}

double oracle_aal(const double* ylt, uint64_t n) {
  double s = 0.0;
  for (uint64_t t = 0; t < n; ++t) s = s + ylt[t];
  return n ? s / (double)n : 0.0;
}

void oracle_ep(const double* ylt, uint64_t n, const double* x, uint32_t m, double* out) {
  for (uint32_t i = 0; i < m; ++i) {
    uint64_t c = 0;
    for (uint64_t t = 0; t < n; ++t)
      if (ylt[t] >= x[i]) ++c;
    out[i] = n ? (double)c / (double)n : 0.0;
  }
}

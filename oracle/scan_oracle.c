/*
 * scan_oracle.c — CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library (through oracle/fast_oracle.py), and only as the checker;
 * the product path (paper_2510_24380_b200/) never links or calls it.
 *
 * A plain-C, multi-threaded restatement of the reference's exhaustive
 * constrained top-k (reference pkg/src/apexcsl/engine.py), used to check the
 * GPU path at BASELINE scale (1e9 / 5e9 products), where the numpy port
 * (oracle/scan_oracle.py) would take minutes:
 *
 *   iter_blocks            engine.py:169-189  — products of [start, end) in g
 *                          order; a reaction's products are rows (first c-1
 *                          digits, mixed radix, csl.py:151-163) x columns (last
 *                          digit); partial rows at the range ends are clipped
 *                          exactly as the slab clipping at :182-189 does.
 *   block_values           engine.py:210-222  — value = fp64 of the fp32
 *                          contributions accumulated in R-group declaration
 *                          order, bias added LAST: ((v0 + v1) + v2) + b.  The
 *                          row prefix ((v0 + v1) + ...) is the same fp64 value
 *                          the reference forms first (broadcast order).
 *   violation              engine.py:134-144  — feasible <=> lower <= v <= upper
 *                          for every constraint (c == 0 exactly then).
 *   search_topk_stream     engine.py:265-313  — heap on (c, s, -g), violators
 *                          dropped at the end (:246-262); restated, as in
 *                          scan_oracle.py, as the top-min(k, end-start)
 *                          FEASIBLE products by (s desc, g asc), with
 *                          discarded = min(k, end-start) - retained.
 *
 * Exactness of the pruning: each thread keeps every feasible product whose s
 * is >= the k-th best s among the feasible products it has already kept
 * (a set of real products), so nothing that can reach the final top-k is ever
 * dropped; ties at the bound are kept and resolved by (s desc, g asc) at the
 * end.  Threads own contiguous g sub-ranges; their top-k lists are merged
 * exactly (the global top-k is inside the union).
 *
 * Pinned by: tests/test_oracle_golden.py (every golden query recorded from the
 * reference itself, tests/golden/make_golden.py) and against the numpy port on
 * random libraries.  Compiled by __graft_entry__.build() with -O2
 * -ffp-contract=off (no FMA contraction, IEEE fp64 adds as in numpy).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_RG 6
#define ORC_MAX_CONS 32

typedef struct {
  double s;
  uint64_t g;
} orc_entry;

typedef struct {
  /* table */
  const float* values; /* [n_tasks][n_pairs] */
  const double* biases;
  int64_t n_pairs;
  /* library */
  int n_rx;
  const int32_t* n_rg;     /* [n_rx] */
  const int64_t* sizes;    /* [n_rx][ORC_MAX_RG] */
  const int64_t* pair_off; /* [n_rx][ORC_MAX_RG] */
  const uint64_t* g_off;   /* [n_rx + 1] */
  /* query */
  int obj;
  int maximize;
  int n_cons;
  const int32_t* cons_task;
  const double* cons_lo;
  const double* cons_hi;
  int64_t k;
} orc_problem;

typedef struct {
  const orc_problem* P;
  uint64_t start, end;
  orc_entry* buf;
  int64_t cap, n;
  double thr;      /* current k-th best s of the kept set (valid when have_thr) */
  int have_thr;
  int64_t scanned;
} orc_worker;

/* (s desc, g asc) */
static int entry_cmp(const void* a, const void* b) {
  const orc_entry* x = (const orc_entry*)a;
  const orc_entry* y = (const orc_entry*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  if (x->g < y->g) return -1;
  if (x->g > y->g) return 1;
  return 0;
}

static void compact(orc_worker* W) {
  qsort(W->buf, (size_t)W->n, sizeof(orc_entry), entry_cmp);
  if (W->n >= W->P->k) {
    W->n = W->P->k;
    W->thr = W->buf[W->n - 1].s;
    W->have_thr = 1;
  }
}

static inline void push(orc_worker* W, double s, uint64_t g) {
  if (W->n == W->cap) compact(W);
  W->buf[W->n].s = s;
  W->buf[W->n].g = g;
  W->n++;
}

/* value of task for the row prefix p (fp64) and last-R-group contribution x:
 * ((p + x) + b), the reference's order with the bias last (engine.py:214-219) */
static inline double val_of(double p, float x, double b) {
  const double t = p + (double)x; /* -ffp-contract=off, no -ffast-math: IEEE adds in this order */
  return t + b;
}

static void scan_reaction(orc_worker* W, int t, uint64_t lo, uint64_t hi) {
  const orc_problem* P = W->P;
  const int c = P->n_rg[t];
  const int64_t* sz = P->sizes + (size_t)t * ORC_MAX_RG;
  const int64_t* po = P->pair_off + (size_t)t * ORC_MAX_RG;
  const uint64_t n_last = (uint64_t)sz[c - 1];
  const uint64_t goff = P->g_off[t];
  const float* vobj = P->values + (size_t)P->obj * P->n_pairs;
  const float* xobj = vobj + po[c - 1];
  const double bobj = P->biases[P->obj];
  double pc[ORC_MAX_CONS];
  const float* xc[ORC_MAX_CONS];
  for (int m = 0; m < P->n_cons; ++m) xc[m] = P->values + (size_t)P->cons_task[m] * P->n_pairs + po[c - 1];
  uint64_t row = lo / n_last;
  uint64_t col0 = lo % n_last;
  for (uint64_t pos = lo; pos < hi; ++row, col0 = 0) {
    const uint64_t col1 = (hi - row * n_last) < n_last ? hi - row * n_last : n_last;
    /* row prefix digits: row = mixed radix over R-groups 0..c-2 */
    int64_t pr[ORC_MAX_RG];
    {
      uint64_t rem = row;
      for (int j = c - 2; j >= 0; --j) {
        pr[j] = po[j] + (int64_t)(rem % (uint64_t)sz[j]);
        rem /= (uint64_t)sz[j];
      }
    }
    double pobj = 0.0;
    if (c > 1) {
      pobj = (double)vobj[pr[0]];
      for (int j = 1; j < c - 1; ++j) pobj = pobj + (double)vobj[pr[j]];
    }
    for (int m = 0; m < P->n_cons; ++m) {
      const float* v = P->values + (size_t)P->cons_task[m] * P->n_pairs;
      double p = 0.0;
      if (c > 1) {
        p = (double)v[pr[0]];
        for (int j = 1; j < c - 1; ++j) p = p + (double)v[pr[j]];
      }
      pc[m] = p;
    }
    const uint64_t gbase = goff + row * n_last;
    if (c == 1) {
      /* one R-group: value = v0 + b (block_values with c == 1) */
      for (uint64_t col = col0; col < col1; ++col) {
        const double vo = (double)xobj[col] + bobj;
        const double s = P->maximize ? vo : -vo;
        if (W->have_thr && s < W->thr) continue;
        int ok = 1;
        for (int m = 0; m < P->n_cons && ok; ++m) {
          const double v = (double)xc[m][col] + P->biases[P->cons_task[m]];
          ok = (v >= P->cons_lo[m]) && (v <= P->cons_hi[m]);
        }
        if (ok) push(W, s, gbase + col);
      }
    } else {
      for (uint64_t col = col0; col < col1; ++col) {
        const double vo = val_of(pobj, xobj[col], bobj);
        const double s = P->maximize ? vo : -vo;
        if (W->have_thr && s < W->thr) continue;
        int ok = 1;
        for (int m = 0; m < P->n_cons && ok; ++m) {
          const double v = val_of(pc[m], xc[m][col], P->biases[P->cons_task[m]]);
          ok = (v >= P->cons_lo[m]) && (v <= P->cons_hi[m]);
        }
        if (ok) push(W, s, gbase + col);
      }
    }
    pos = row * n_last + col1;
  }
}

static void* worker_main(void* arg) {
  orc_worker* W = (orc_worker*)arg;
  const orc_problem* P = W->P;
  for (int t = 0; t < P->n_rx; ++t) {
    const uint64_t off = P->g_off[t], end_t = P->g_off[t + 1];
    if (end_t <= W->start || off >= W->end) continue;
    const uint64_t lo = (W->start > off ? W->start : off) - off;
    const uint64_t hi = (W->end < end_t ? W->end : end_t) - off;
    scan_reaction(W, t, lo, hi);
  }
  compact(W);
  return NULL;
}

/*
 * Exact top-min(k, end-start) feasible products of [start, end), best-first
 * by (s desc, g asc).  out_s / out_g: capacity k.  Returns retained count
 * (>= 0), or -1 on bad arguments / allocation failure.
 */
int64_t orc_search_topk(const float* values, const double* biases, int32_t n_tasks, int64_t n_pairs,
                        int32_t n_rx, const int32_t* n_rg, const int64_t* sizes, const int64_t* pair_off,
                        const uint64_t* g_off, int32_t obj, int32_t maximize, int32_t n_cons,
                        const int32_t* cons_task, const double* cons_lo, const double* cons_hi, int64_t k,
                        uint64_t start, uint64_t end, int32_t n_threads, double* out_s, uint64_t* out_g) {
  if (k <= 0 || end <= start) return 0;
  if (n_cons > ORC_MAX_CONS || obj < 0 || obj >= n_tasks || n_threads < 1) return -1;
  for (int t = 0; t < n_rx; ++t)
    if (n_rg[t] < 1 || n_rg[t] > ORC_MAX_RG) return -1;
  orc_problem P = {values, biases, n_pairs, n_rx, n_rg, sizes, pair_off, g_off,
                   obj, maximize, n_cons, cons_task, cons_lo, cons_hi, k};
  const uint64_t span = end - start;
  if ((uint64_t)n_threads > span) n_threads = (int32_t)span;
  orc_worker* W = (orc_worker*)calloc((size_t)n_threads, sizeof(orc_worker));
  pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
  if (!W || !th) return -1;
  const int64_t cap = 4 * k + 4096;
  int err = 0;
  for (int i = 0; i < n_threads; ++i) {
    W[i].P = &P;
    W[i].start = start + (uint64_t)(((unsigned __int128)span * (unsigned)i) / (unsigned)n_threads);
    W[i].end = start + (uint64_t)(((unsigned __int128)span * (unsigned)(i + 1)) / (unsigned)n_threads);
    W[i].cap = cap;
    W[i].buf = (orc_entry*)malloc((size_t)cap * sizeof(orc_entry));
    if (!W[i].buf) err = 1;
  }
  if (!err) {
    for (int i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, worker_main, &W[i]);
    worker_main(&W[0]);
    for (int i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
  }
  int64_t total = 0;
  for (int i = 0; i < n_threads; ++i) total += W[i].n;
  orc_entry* all = err ? NULL : (orc_entry*)malloc((size_t)(total > 0 ? total : 1) * sizeof(orc_entry));
  int64_t n = -1;
  if (all) {
    int64_t p = 0;
    for (int i = 0; i < n_threads; ++i) {
      memcpy(all + p, W[i].buf, (size_t)W[i].n * sizeof(orc_entry));
      p += W[i].n;
    }
    qsort(all, (size_t)total, sizeof(orc_entry), entry_cmp);
    n = total < k ? total : k;
    for (int64_t i = 0; i < n; ++i) {
      out_s[i] = all[i].s;
      out_g[i] = all[i].g;
    }
    free(all);
  }
  for (int i = 0; i < n_threads; ++i) free(W[i].buf);
  free(W);
  free(th);
  return n;
}

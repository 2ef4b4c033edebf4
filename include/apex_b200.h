/*
 * apex_b200.h — C ABI of the B200-native APEX enumeration-and-retrieval path.
 *
 * The reference (`/root/reference/pkg/src/apexcsl`, pure Python/numpy) has no
 * FFI: its operator API for this path is three Python functions.  Each entry
 * point below replaces one of them (or one stage inside them), so a host
 * binding (ctypes stub in INTEGRATION.md, or the Python mirror in
 * paper_2510_24380_b200/engine.py) can stand in for:
 *
 *   engine.precompute_contributions(cache, surrogate)      engine.py:80-92
 *       -> apex_load_cache        (K1: fp64 head_w @ u^T, fp32 rounding)
 *   engine.search_topk_stream(library, table, query, index_range)
 *                                                          engine.py:265-313
 *   engine.search_topk_batched(library, table, query, chunk_size, index_range)
 *                                                          engine.py:345-398
 *       -> apex_query             (K2 pack, K3 enumerate+filter, K5 select,
 *                                  K7 decode/materialize; identical results for
 *                                  both reference variants)
 *   ContributionTable construction / load_table            engine.py:35-72, 448-460
 *       -> apex_load_table
 *   CslLibrary index space (offsets, sizes, pair rows)     csl.py:57-112, 138-184
 *       -> apex_load_library
 *
 * Multi-GPU (one process per GPU): apex_query_local produces a
 * rank's exact local top-k as (key, g) entries in a caller-owned DEVICE buffer,
 * the host all-gathers those buffers (NCCL), and apex_merge_finalize selects,
 * orders and materializes the global result from the gathered entries.
 *
 * Conventions (SURVEY.md §8b "Design rules for that ABI"):
 *   - every function returns 0 on success, nonzero (an APEX_E* code) on error;
 *     apex_last_error() returns a thread-local message.  No C++ exception
 *     crosses the ABI.
 *   - host buffers are borrowed for the duration of the call.
 *   - device state is owned by the ctx; the table is immutable after load.
 *   - a ctx is not re-entrant; distinct ctxs may be used concurrently.
 *   - no CPU fallback: if the device is missing or a kernel fails, the call
 *     fails with APEX_ECUDA.
 */
#ifndef APEX_B200_H
#define APEX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APEX_MAX_RGROUPS 6 /* R-groups per reaction supported by the kernels */

enum {
  APEX_OK = 0,
  APEX_EINVAL = 1,    /* bad argument (maps to EngineError) */
  APEX_ERANGE = 2,    /* index range invalid (engine.py:281-282) */
  APEX_ETASK = 3,     /* unknown task (engine.py:58-62) */
  APEX_ECUDA = 4,     /* CUDA failure / no device */
  APEX_ESTATE = 5,    /* call order: library/table not loaded */
  APEX_ENOMEM = 6,    /* device allocation failed */
  APEX_ELIMIT = 7     /* request exceeds a compiled limit (k, R-groups, tests) */
};

typedef struct apex_ctx apex_ctx;

/* One reaction of the library, positional (reaction(id) is positional,
 * csl.py:90-91).  R-groups in declaration order; digit order of the codec
 * (csl.py:151-163): first R-group most significant. */
typedef struct {
  int32_t n_rgroups;                       /* c >= 2 (csl.py:122-123) */
  int32_t _pad;
  int64_t sizes[APEX_MAX_RGROUPS];         /* synthons per R-group */
  int64_t pair_offset[APEX_MAX_RGROUPS];   /* table row of digit 0: rg_offsets[_rg_pos[rg]] */
  uint64_t g_offset;                       /* reaction_offset(t) (csl.py:96-97) */
} apex_reaction;

/* One constraint: task index into the table's task list, closed interval
 * [lower, upper] with +-inf meaning unbounded (engine.py:104-112). */
typedef struct {
  int32_t task;
  int32_t _pad;
  double lower;
  double upper;
} apex_constraint;

/* One query (engine.py:115-131) over the global index range [start, end). */
typedef struct {
  int32_t objective_task;
  int32_t maximize;                /* 1 = "maximize", 0 = "minimize" */
  int32_t n_constraints;
  int32_t _pad;
  const apex_constraint* constraints;
  int64_t k;
  uint64_t start;
  uint64_t end;
} apex_query_spec;

/* Per-stage device time and counters of the last apex_query call. */
typedef struct {
  double pack_ms;          /* K2 pack of the signed test columns */
  double seed_ms;          /* sampled admission threshold (exact, from real products) */
  double scan_ms;          /* K3 enumeration chunks incl. threshold refreshes */
  double select_ms;        /* compaction + K5 exact select */
  double finalize_ms;      /* K6 ordering + K7 materialization */
  double d2h_ms;           /* result copy to host */
  double total_ms;         /* device time of the whole call */
  double scan_kernel_ms;   /* K3 launches only (sum over chunks) */
  int64_t candidates;      /* entries appended by the enumeration kernel */
  int64_t scan_launches;   /* enumeration launches (chunks, incl. retries) */
  int64_t kernel_launches; /* all kernels launched by the call */
  int64_t retries;         /* re-runs after a candidate-buffer overflow */
  int64_t h2d_bytes;       /* host->device bytes copied by the call */
  int64_t d2h_bytes;       /* device->host bytes copied by the call */
  int64_t admitted;        /* products that passed the admission test (admission-first kernel) */
  double host_prepare_us;  /* host time of descriptor checks / staging in the call */
  double host_launch_us;   /* host time of the launches (graph replay or direct) */
  int64_t stale_sources;   /* merge: gathered local results marked stale (a source
                              overflowed and re-ran: gather and merge again) */
} apex_stats;

/* Caller-allocated host output for one query; arrays sized for k entries
 * (constraint_values: k * n_constraints, digits: k * APEX_MAX_RGROUPS).
 * View mode: if all five array pointers are NULL, apex_query / _fetch set
 * them to the rows in the context's pinned host block instead of copying
 * (valid until the next call on the context; all queries of the call must
 * share one range). */
typedef struct {
  uint64_t* global_index;
  double* objective;          /* value in the user's direction (engine.py:254) */
  double* constraint_values;  /* apex_score order (engine.py:95-101) */
  int32_t* reaction;          /* positional reaction index */
  int32_t* digits;            /* per R-group digit, APEX_MAX_RGROUPS stride */
  int64_t n;                  /* out: retained entries (best-first) */
  int64_t discarded;          /* out: min(k, end-start) - retained */
  uint64_t scanned;           /* out: end - start */
  int64_t candidates;         /* out: feasible products with s >= tau appended by the scan */
  int64_t admitted;           /* out: products that passed the admission test (admission-first kernel) */
  int32_t full_predicate;     /* out: 1 if the full-predicate kernel scanned this query */
  int32_t _pad;
} apex_result;

/* Entry exchanged between ranks: order-preserving key of the signed
 * objective (larger = better, +-0 canonicalized) and the global index. */
typedef struct {
  uint64_t key;
  uint64_t g;
} apex_entry;

const char* apex_last_error(void);
const char* apex_version(void);

/* device: CUDA ordinal; stream: a cudaStream_t (NULL = a ctx-owned stream). */
int apex_ctx_create(int32_t device, void* stream, apex_ctx** out);
void apex_ctx_destroy(apex_ctx* ctx);
int apex_set_stream(apex_ctx* ctx, void* stream);

/* Library index space.  n_pairs = table rows expected. */
int apex_load_library(apex_ctx* ctx, const apex_reaction* reactions, int32_t n_reactions,
                      int64_t n_pairs);

/* Contribution table: values float32 [n_tasks][n_pairs] (engine.py:37),
 * biases float64 [n_tasks] (engine.py:38).  Non-finite values are rejected. */
int apex_load_table(apex_ctx* ctx, const float* values, const double* biases, int32_t n_tasks,
                    int64_t n_pairs);

/* K1 synthon precompute (engine.py:80-92): values = fl32(head_w @ u^T) with
 * fp64 products and accumulation, on device; the table becomes resident.
 * u: float64 [n_pairs][d]; head_w: float64 [n_tasks][d]; head_b: float64
 * [n_tasks].  values_out (optional, may be NULL): host copy of the table. */
int apex_load_cache(apex_ctx* ctx, const double* u, int64_t n_pairs, int32_t d,
                    const double* head_w, const double* head_b, int32_t n_tasks,
                    float* values_out);

/* Same as apex_load_cache but u / values_out are DEVICE pointers (no host
 * copies); head_w may be device or host memory (the 11 x 64 TMA form passes
 * the heads as kernel parameters: host heads need no device round trip).
 * Used to time K1 alone (apex_precompute_time). */
int apex_precompute_device(apex_ctx* ctx, const double* u_dev, int64_t n_pairs, int32_t d,
                           const double* head_w_dev, int32_t n_tasks, float* values_dev);

/* Device time (ms) of the last K1 launch of apex_precompute_device /
 * apex_load_cache (CUDA events around the kernel alone), or -1 when that
 * launch used a form without the timer. */
int apex_precompute_time(apex_ctx* ctx, double* kernel_ms);

/* Run n_queries queries (batched: one enumeration schedule, all queries per
 * launch) and materialize each result into results[i] (host buffers). */
int apex_query(apex_ctx* ctx, const apex_query_spec* queries, int32_t n_queries,
               apex_result* results, apex_stats* stats);

/* Asynchronous form of apex_query for queries sharing one range (k >= 1):
 * enqueues the whole device pipeline on the ctx stream and returns without a
 * host sync; results stay on the device until apex_query_fetch, which syncs,
 * validates (re-running exactly after a candidate-buffer overflow) and copies
 * the rows into caller-allocated host results.  A second apex_query_async
 * before the fetch replaces the batch in flight. */
int apex_query_async(apex_ctx* ctx, const apex_query_spec* queries, int32_t n_queries, apex_stats* stats);
int apex_query_fetch(apex_ctx* ctx, apex_result* results, apex_stats* stats);

/* Multi-GPU local step: exact local top-min(k, feasible) of each query over its
 * [start, end), written UNSORTED into out_dev (device, capacity k entries per
 * query, query q at out_dev + q*k); counts_host[q] = entries written. */
int apex_query_local(apex_ctx* ctx, const apex_query_spec* queries, int32_t n_queries,
                     apex_entry* out_dev, int64_t* counts_host, apex_stats* stats);

/* Multi-GPU final step: entries_dev holds n_entries gathered local entries of
 * ONE query (device; padding entries have g == UINT64_MAX and are ignored).
 * Selects the global top-k, orders best-first, materializes into *result.
 * total_scanned = global range size used for `discarded`. */
int apex_merge_finalize(apex_ctx* ctx, const apex_query_spec* query, const apex_entry* entries_dev,
                        int64_t n_entries, uint64_t total_scanned, apex_result* result,
                        apex_stats* stats);

/* Multi-GPU final step for a whole batch: entries_dev (device) holds the
 * all-gathered local entries of n_queries queries from n_src ranks, laid out
 * entries_dev[(src * n_queries + q) * stride + i] (i < stride; padding
 * g == UINT64_MAX ignored) — what all-gathering every rank's [n_queries][k]
 * apex_query_local buffer produces.  One device pass selects, orders and
 * materializes every query's global top-k into results[q]. */
int apex_merge_finalize_batch(apex_ctx* ctx, const apex_query_spec* queries, int32_t n_queries,
                              const apex_entry* entries_dev, int32_t n_src, int64_t stride,
                              uint64_t total_scanned, apex_result* results, apex_stats* stats);

/* Multi-GPU local step, asynchronous form (one process per GPU): enqueues
 * the exact local pipeline of a batch (queries share range; 1 <= k <= stride)
 * and the export of each query's selected entries to out_dev + q*stride
 * (device; unused slots padded with g == UINT64_MAX) on the context stream,
 * with no host sync, so an all-gather and apex_merge_finalize_batch can be
 * enqueued behind it.  apex_query_local_finish then syncs and validates: if a
 * candidate buffer overflowed the batch is re-run exactly, re-exported and
 * *rerun = 1 (the caller must gather and merge again); counts (optional) =
 * entries selected per query. */
int apex_query_local_async(apex_ctx* ctx, const apex_query_spec* queries, int32_t n_queries, apex_entry* out_dev,
                           int64_t stride, apex_stats* stats);
int apex_query_local_finish(apex_ctx* ctx, int64_t* counts_host, int32_t* rerun, apex_stats* stats);

/* Multi-GPU context: ONE process and host thread driving n_devices GPUs
 * (SURVEY.md §8b "one host thread drives all devices").  Every query batch's
 * index range is cut into n_devices contiguous g ranges; each device runs the
 * exact local top-k; the merge on device_ids[0] reads every shard's entries
 * through peer pointers over NVLink inside its load kernel (the gather fused
 * into the merge) and materializes the global result.  A device id may repeat
 * (several shards on one GPU).  Results are identical to apex_query on one
 * device.  Result arrays must be caller-allocated (no view mode). */
typedef struct apex_multi apex_multi;
int apex_multi_create(int32_t n_devices, const int32_t* device_ids, apex_multi** out);
void apex_multi_destroy(apex_multi* m);
int apex_multi_load_library(apex_multi* m, const apex_reaction* reactions, int32_t n_reactions, int64_t n_pairs);
int apex_multi_load_table(apex_multi* m, const float* values, const double* biases, int32_t n_tasks, int64_t n_pairs);
int apex_multi_load_cache(apex_multi* m, const double* u, int64_t n_pairs, int32_t d, const double* head_w,
                          const double* head_b, int32_t n_tasks, float* values_out);
int apex_multi_set_option(apex_multi* m, const char* name, int64_t value);
int apex_multi_query(apex_multi* m, const apex_query_spec* queries, int32_t n_queries, apex_result* results,
                     apex_stats* stats);
int apex_multi_info(apex_multi* m, int32_t* n_devices, int32_t* peer_access);

/* Ground-truth evaluation on the device: the exhaustive
 * oracle top-j of evalkit.oracle_topk (evalkit.py:49-90) over the synthetic
 * ground-truth oracle (props.oracle_block_values, props.py:218-264), without
 * the reference's 1e8-product guard.  Task t of the oracle: latent values per
 * synthon id (row t of latents), +nonlinear (flags & 1): value +=
 * nonlinear_scale * tanh(nonlinear_alpha * base), +pairwise (flags & 2): the
 * splitmix pair coefficients keyed by salt (props.py:162-195). */
typedef struct {
  int32_t flags;            /* 1 = +nonlinear, 2 = +pairwise */
  uint32_t salt;            /* _task_salt(oracle, task) (props.py:198-199) */
  double nonlinear_scale;
  double nonlinear_alpha;
  double pair_scale;
  double pair_density;
} apex_gt_task;

/* member_ids[p]: synthon id of pair row p (the library's pair rows as loaded
 * by apex_load_library); latents: float64 [n_tasks][n_synthons]. */
int apex_gt_load(apex_ctx* ctx, const int64_t* member_ids, int64_t n_pairs, const double* latents, int64_t n_synthons,
                 const apex_gt_task* tasks, int32_t n_tasks);
/* Oracle top-j (j = query->k; tasks index the oracle's tasks) over
 * [start, end): result rows best-first by (s desc, g asc) among oracle-feasible
 * products; objective / constraint_values are the oracle's values. */
int apex_gt_topk(apex_ctx* ctx, const apex_query_spec* query, apex_result* result, apex_stats* stats);

/* BatchTrace accounting of the chain-of-batches variant (engine.py:338-391,
 * SURVEY §8(f) row 3): for batches [start, batch_end[0]), [batch_end[0],
 * batch_end[1]), ... (make_batches, engine.py:316-335) the number of entries
 * of each batch's selection — the k best of (carry ∪ batch) under the full
 * order (violation desc, signed objective desc, global index asc), infeasible
 * products included — that came from the batch (new_out) or the carry
 * (carried_out).  Exact, on the device. */
int apex_batch_trace(apex_ctx* ctx, const apex_query_spec* query, const uint64_t* batch_end, int32_t n_batches,
                     int64_t* new_out, int64_t* carried_out);

/* K8: the factorizer's hierarchy encoding on the device (
 * factorizer.encode_hierarchy, factorizer.py:157-171, 218-233): synthon
 * feature hashing (BLAKE2b-64 of "<salt>:<ngram>" for the 1/2/3-grams of each
 * UTF-8 token, props.py:43-62), the synthon MLP, the R-group and reaction
 * deep sets (mean pooling), the value and key MLPs, and the pair rows
 * u[p] = v[member[p]] @ K[rgroup(p)]^T, all fp64.  nets: 7 MLP shapes in the
 * order synthon, rgroup phi, rgroup rho, reaction phi, reaction rho, value,
 * key (dims[0..n_layers], tanh between layers); params: every net's
 * W0 [dims0 x dims1] (row-major), b0, W1, b1, ... concatenated in that order.
 * The pair matrix stays resident for apex_precompute_resident; every *_out
 * (host, optional) receives a copy. */
typedef struct {
  int32_t n_layers;
  int32_t dims[7];
} apex_mlp_shape;
int apex_encode_hierarchy(apex_ctx* ctx, const apex_mlp_shape* nets, const double* params, int64_t n_params,
                          const uint8_t* token_bytes, const int64_t* token_off, int64_t n_synthons,
                          const uint8_t* salt, int32_t salt_len, int32_t p, double feature_scale,
                          const int64_t* member_ids, int64_t n_pairs, const int64_t* rg_offsets, int32_t n_rg,
                          const int32_t* rg_parent, const int64_t* rx_offsets, int32_t n_rx, int32_t d, int32_t d_u,
                          double* u_out, double* h_s_out, double* h_r_out, double* h_t_out, double* features_out);
/* K1 from the resident K8 pair matrix (engine.py:80-92): the table becomes
 * resident (values_out, optional: host copy). */
int apex_precompute_resident(apex_ctx* ctx, const double* head_w, const double* head_b, int32_t n_tasks,
                             float* values_out);

/* Tuning / introspection. */
int apex_set_option(apex_ctx* ctx, const char* name, int64_t value);

/* Test hook: exact fp32 thresholds of the enumeration kernel for arrays of
 * (p, b, beta) (host buffers): up[i] = max finite fp32 x with
 * ((p + x) + b) <= beta (fp64), +inf if all, NaN if none; lo[i] = min x with
 * ((p + x) + b) >= beta, -inf if all, NaN if none. */
int apex_debug_thresholds(apex_ctx* ctx, const double* p, const double* b, const double* beta, int64_t n,
                          float* up, float* lo);
/* Profiling hook: per-work-item records of the last admission scan, enabled by
 * apex_set_option(ctx, "trace", capacity).  Eight words per record:
 * start ns, end ns, smid | rare-path entries << 8 | query << 32,
 * ncols << 8 | nrows | reaction << 32, rare-path cycles, threshold cycles,
 * staging cycles, candidates.  *n = records copied. */
int apex_debug_trace(apex_ctx* ctx, uint64_t* out, int64_t cap, int64_t* n);
int apex_get_device_info(apex_ctx* ctx, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

#ifdef __cplusplus
}
#endif
#endif /* APEX_B200_H */

// capi.cu — host runtime and C ABI (include/apex_b200.h) of the B200-native
// APEX enumeration-and-retrieval path.
//
// Query protocol (one schedule for a batch of queries over the same range):
//   init_ctl -> pack (K2) -> sample + tau(seed) -> [scan chunk (K3) -> tau]*
//   -> tau(bound) -> compact -> select (K5, cooperative) -> rank/scatter (K6)
//   -> materialize (K7) -> D2H.
// Exactness argument: every appended candidate is an exactly
// feasible product with s >= tau (exact fp32 thresholds on the last R-group's
// contribution, K3); every tau / bound is the k-th best bin edge of a set of
// distinct real feasible products, hence <= the true k-th best key; so the
// true top-k is always inside the candidate set, and K5 selects it exactly by
// (key desc, g asc) == the reference's (s desc, g asc) over feasible rows.
// A candidate-buffer overflow is detected (count > cap) and the query is re-run
// with the final (valid) bound as its starting threshold.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include <cudaTypedefs.h>

#include "kernels.cuh"
#include "gt.cuh"
#include "k8.cuh"
#include "trace.cuh"
#include "bind.cuh"

using namespace apexb200;

namespace {

thread_local std::string t_err;

int set_err(int code, const std::string& m) {
  t_err = m;
  return code;
}

#define APEX_CU(x)                                                                                \
  do {                                                                                            \
    cudaError_t e__ = (x);                                                                        \
    if (e__ != cudaSuccess)                                                                       \
      return set_err(APEX_ECUDA, std::string(#x) + " failed: " + cudaGetErrorString(e__));       \
  } while (0)

// serialize calls on one context (apex_ctx::mu); recursive: apex_query calls
// apex_query_async / apex_query_fetch on the same context
#define APEX_LOCK(c)                                                  \
  if (!(c)) return set_err(APEX_EINVAL, "null context");              \
  std::lock_guard<std::recursive_mutex> lock__((c)->mu)

#define APEX_TRY(x)           \
  do {                        \
    int r__ = (x);            \
    if (r__ != APEX_OK) return r__; \
  } while (0)

// bumped on every (re)allocation by any thread: device pointers baked into a
// captured CUDA graph are only valid while this is unchanged (process-wide, so
// a reallocation on one thread invalidates every context's graph key)
std::atomic<uint64_t> g_alloc_gen{0};

struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes) return APEX_OK;
    ++g_alloc_gen;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(b, 256));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_err(APEX_ENOMEM, "cudaMalloc(" + std::to_string(b) + ") failed: " + cudaGetErrorString(e));
    }
    bytes = std::max<size_t>(b, 256);
    return APEX_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct HBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t b) {
    if (b <= bytes) return APEX_OK;
    ++g_alloc_gen;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&p, std::max<size_t>(b, 256));
    if (e != cudaSuccess) return set_err(APEX_ENOMEM, std::string("cudaMallocHost failed: ") + cudaGetErrorString(e));
    bytes = std::max<size_t>(b, 256);
    return APEX_OK;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

struct Slot {
  DBuf packed, obj_col, buf, sel, sorted;
  void release() {
    for (DBuf* b : {&packed, &obj_col, &buf, &sel, &sorted}) b->release();
  }
};

struct Plan {
  uint64_t start = 0, end = 0;
  int rows = 0;
  int64_t cols = 0;
  std::vector<Tile> tiles;        // permuted
  std::vector<uint64_t> prefix;   // products in tiles[0, i)
  DBuf d_tiles;
  int64_t pair_lo = 0, pair_hi = 0;  // last-R-group pair rows touched
  uint64_t stamp = 0;
  ~Plan() { d_tiles.release(); }
};

// per query: candidate hist + coarse, seed hists (uniform, corner) + their coarse
constexpr size_t kHistWords = (size_t)kHistBins + 256 + 2 * (size_t)kHistBins + 512;

size_t out_bytes(int64_t k, int m) { return (size_t)k * (8 + 8 + 8 * (size_t)m + 4 + 4 * kMaxRg); }

// Tests of a query: test 0 = objective admission, then for every
// task the tightest finite upper bound and the tightest finite lower bound
// (x >= each lower <=> x >= max lower; monotone, so merging is exact).
struct QTests {
  int nt = 0;
  int task[kMaxTests];
  int lower[kMaxTests];
  double beta[kMaxTests];
};

struct RunStats {
  int64_t launches = 0, scans = 0, retries = 0;
  int64_t h2d_bytes = 0, d2h_bytes = 0;
  float ms[8] = {};
  float scan_kernel_ms = 0;
};

// The last enqueued batch: queries sharing one range (deep copies).
struct Batch {
  std::vector<apex_query_spec> qs;       // sorted by kernel test class
  std::vector<int> perm;                 // qs[i] is the caller's query perm[i]
  std::vector<int> cls_nt, cls_begin;    // scan launches: test class, first query (cls_begin.back() == nq)
  std::vector<std::vector<apex_constraint>> cons;
  std::vector<QTests> tests;
  int nq = 0, NT = 0, rl = 0, ntp = 0;
  int64_t k_max = 0;
  bool finalize = false;
  bool copy_out = false;       // result rows D2H inside the pass (synchronous apex_query)
  bool no_full = false;        // this signature needed no full-predicate kernel last time: skip its launches
  std::vector<int> cset_leader;  // shared constraint sets (sorted-column pre-pass): a query of each
  int64_t cset_tests = 0;        // pre-pass threshold rows (sum of the sets' constraint tests)
  bool small_only = false;     // every query of this signature's last run fit the small finalize: skip the
                               // large-path launches (select, chunk sort, merge rank); re-run if one does not
  uint64_t key0 = 0;           // signature before no_full (history key)
  Plan* plan = nullptr;
  Plan* plan_rows = nullptr;    // whole-row tiles (sorted-column admission kernel)
  bool pending = false;
  // multi-GPU local step (apex_query_local_async): where the selected entries
  // are exported, with what per-query stride
  Entry* export_out = nullptr;
  unsigned long long export_stride = 0;
  RunStats st;
};

}  // namespace

struct apex_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;           // second stream: the corner seed runs beside the sample seed
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaStream_t side2 = nullptr;          // third stream: the sorted-column constraint pre-pass
  cudaEvent_t fork2_ev = nullptr, join2_ev = nullptr;
  bool own_stream = false;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  // library
  std::vector<DevReaction> rx;
  std::vector<unsigned long long> goff;  // n_rx + 1
  uint64_t total = 0;
  int64_t lib_pairs = 0;
  int64_t pcols = 0;                     // packed objective-column length (16-B aligned segments)
  DBuf d_rx, d_goff;
  bool lib_loaded = false;
  // table
  DBuf d_values, d_biases;
  std::vector<double> biases;
  // corner seed lists (built lazily once library + table are resident)
  DBuf d_lists, d_slot_off, d_m, d_coff;
  int64_t corner_slots = 0;
  unsigned long long corner_total = 0;
  bool corners_ok = false;
  DBuf d_sorted_x, d_sorted_col;         // per task: each reaction's last R-group sorted ascending (value, column)
  DBuf d_quant;                          // per task, reaction: kQuant + 1 evenly spaced values of the sorted column
  DBuf d_cthr, d_cqc, d_cbest;           // sorted-column constraint pre-pass rows (shared constraint sets)
  DBuf d_packed16;                       // [n_pairs][16] pair-major copy of the table (sorted-column kernel)
  bool packed16_ok = false;
  DBuf d_rowp;                           // [task][rows_total] fp64 row prefix sums (bind_rowp_kernel)
  bool rowp_ok = false;
  int64_t rows_total = 0;                // rows (first c-1 R-group assignments) of all reactions
  int n_tasks = 0;
  int64_t n_pairs = 0;
  bool table_loaded = false;
  // query workspaces
  std::vector<Slot> slots;
  DBuf d_queries, d_tau0;
  DBuf d_hists;                          // per-query histograms, contiguous (one memset per batch)
  DBuf d_ctls;                           // per-query control blocks, contiguous (one strided D2H of the headers)
  bool copy_next = false;                // next prepare_batch: result D2H inside the pass
  std::vector<uint64_t> seen_keys;       // recent batch signatures (graph capture on the second sighting)
  std::vector<uint64_t> nofull_keys;     // signatures whose last run sent no query to the full predicate
  std::vector<uint64_t> small_keys;      // signatures whose last run finished every query in the small finalize
  DBuf d_out;                            // per-query result rows, contiguous (one D2H per batch)
  std::vector<size_t> out_off;           // byte offset of each query's rows in d_out
  DBuf d_work;                           // flattened-work counters of the scan launches
  DBuf d_fin_scratch;                    // bucketed finalize partition regions [query][CTA][kSmallSel]
  DBuf d_trace;                          // optional per-item timing records of the admission scan
  int64_t trace_cap = 0, trace_n = 0;
  HBuf h_queries, h_ctl, h_out, h_tau0;
  std::vector<std::unique_ptr<Plan>> plans;
  uint64_t stamp = 0;
  cudaEvent_t ev[8] = {};
  cudaEvent_t upload_ev = nullptr;
  cudaEvent_t done_ev = nullptr;         // end of a pass (wait_stream's poll)
  std::vector<ScanQuery> uploaded;   // last ScanQuery array copied to d_queries
  Batch batch;
  // options
  int64_t opt_cap = 1 << 22;        // candidate buffer entries per query (minimum)
  int64_t opt_cb = 64;              // columns per smem block
  int64_t opt_rl = 0;               // rows per lane (0 = auto)
  int64_t opt_samples = 0;          // seed samples (0 = auto)
  int64_t opt_chunk_div = 16;       // first scan chunk = 1/opt_chunk_div of the range
  int64_t opt_chunk_min = 1ll << 62;  // ranges at least this large are scanned in two chunks (off)
  int64_t opt_tile_products = 0;    // target products per tile (0 = auto)
  int64_t opt_select_ctas = 16;     // CTAs per query in the select kernel
  int64_t opt_force_upload = 0;     // re-upload query descriptors on every call
  int64_t opt_refresh = 0;          // in-kernel tau refresh interval (0 = k)
  int64_t opt_mode = 3;             // enumeration kernel: 3 = automatic per query (admission-first when
                                    // the seed found a threshold, else full predicate), 2 = admission-first
                                    // (exact short-circuit), 0 = full predicate (FSETP chain),
                                    // 1 = full predicate (FADD2 sign bits)
  int64_t opt_cb_admit = 512;       // columns per smem block in the admission-first kernel
  int64_t opt_corner = 1;           // corner seed on/off
  int64_t opt_corner_mult = 16;
  int64_t opt_pre_rows = 2;         // K1 form: 2 = TMA bulk ring (11 x 64), 1 = row-parallel, 0 = smem tiles
  int64_t opt_vote64 = 1;           // admission kernel 64-column pre-vote
  int64_t opt_sorted = 1;           // sorted-column admission kernel (per-row work) instead of the streaming one
  int64_t opt_fin_bucket = 64;      // bucketed small finalize: max CTAs per query (0: one-CTA finalize_small_kernel)
  int64_t opt_rowp = 1;             // build / use the row-prefix table
  int64_t opt_rowp_bytes = (int64_t)4 << 30;  // its size limit
  int64_t opt_heavy_first = 1;      // whole-row tile plans ordered by products, descending
  int64_t opt_work_ctrs = 4;        // sorted-column scan: work counters (1: one counter)
  int64_t opt_split_cols = 0;       // whole-row tiles of reactions with >= this many columns get split_rows rows (0: off)
  int64_t opt_split_rows = 8;
  int64_t opt_cpre_ctas = 0;        // pre-pass grid: CTAs per SM (grid-stride; 0: one CTA per 8 items)
  int64_t opt_spin_us = 0;          // wait for a pass by polling its end event for up to this long (0: block; measured neutral)
  int64_t opt_bail = 128;           // sorted-column pair budget: range / this (0: no budget)
  int64_t opt_bail_min = 4 << 20;   // ... and at least this many pairs
  int64_t opt_fin_part = 1;         // bucketed finalize partitions the buffer (cooperative) instead of full scans per CTA
  int64_t opt_graph_prio = 1;       // graphs honour the streams' priorities (cudaGraphInstantiateFlagUseNodePriority)
  int64_t opt_cpre_prio = -1;       // pre-pass stream priority: 1 highest, -1 lowest
  int64_t opt_tau_side = 1;         // threshold kernel on the high-priority side stream
  int64_t opt_lazy_hist = 1;        // histograms zeroed by the control init where the last pass left counts
  int64_t opt_cpre_fused = 0;       // constraint pre-pass as one fused kernel (measured slower: 27 us vs 16 + 5)
  int64_t opt_stages = 0;           // record the per-stage events (stats pack/seed/scan/select/finalize ms)
  int64_t opt_cpre = 3;             // sorted-column kernel: constraint pre-pass for sets shared by several queries
                                    // (3: after the control init, enqueued after the seeds; 1: right after the init; 2: at the pass start; 0: off)
  int64_t opt_dense = 16;           // admission kernel dense-row trigger (admitted products of a row in a tile; 0 = off)
  int64_t opt_graph = 1;            // replay the device pipeline of a repeated batch as a CUDA graph
  int64_t opt_packed16 = 1;         // sorted-column kernel reads the pair-major table copy
  int64_t opt_chunk = 1;            // work items per atomic in the scan kernels
  int64_t opt_tiles_per_slot = 8;   // target enumeration tiles per warp slot (balance vs per-tile setup)
  uint64_t opt_gen = 0;             // bumped by apex_set_option
  // the merge's own workspace (merge_impl swaps it in): a local step in
  // flight on this context keeps its buffers while the merge of gathered
  // entries runs on the same stream (dist.sharded_batch enqueues both)
  struct Workspace {
    std::vector<Slot> slots;
    DBuf d_hists, d_ctls, d_queries, d_out;
    HBuf h_queries, h_ctl, h_out;
    std::vector<size_t> out_off;
    std::vector<ScanQuery> uploaded;
  } mws;
  cudaEvent_t mev[2] = {};
  // ground-truth oracle (apex_gt_load): members, latents, task parameters
  DBuf d_gt_members, d_gt_latent, d_gt_tasks, d_gt_hist, d_gt_buf, d_gt_misc;
  std::vector<GtTask> gt_tasks;
  DBuf d_u_res;                          // K8 output: the pair-row matrix u, resident for K1
  int64_t u_res_pairs = 0;
  int u_res_d = 0;
  int64_t gt_synthons = 0;
  bool gt_loaded = false;
  bool k1_timed = false;             // mev brackets the last K1 launch (apex_precompute_time)
  // per-context (= per-device) launch caches
  std::vector<std::pair<std::pair<const void*, size_t>, int>> occ_cache;
  std::vector<std::pair<const void*, size_t>> attr_cache;
  bool attr_small = false;
  bool attr_bucket = false;
  int occ_sel = 0;
  // a context is driven by one thread at a time: every C-ABI call on it holds
  // this lock (calls on different contexts run concurrently)
  std::recursive_mutex mu;
  // CUDA graph of the last batch signature
  cudaGraphExec_t gexec = nullptr;
  uint64_t gkey = 0;
  bool graph_broken = false;
  RunStats graph_stats;
};

namespace {

int check_ctx(apex_ctx* c, bool need_table) {
  if (!c) return set_err(APEX_EINVAL, "null context");
  if (need_table && !(c->lib_loaded && c->table_loaded))
    return set_err(APEX_ESTATE, "library and table must be loaded before querying");
  if (need_table && c->n_pairs != c->lib_pairs)
    return set_err(APEX_EINVAL, "table rows (" + std::to_string(c->n_pairs) + ") do not match library pair rows (" +
                                    std::to_string(c->lib_pairs) + ")");
  APEX_CU(cudaSetDevice(c->device));
  return APEX_OK;
}

// ---------------------------------------------------------------------------
// Enumeration tiles for [start, end): per reaction, rows = prefix assignments
// (mixed radix of the first c-1 digits), columns = last digit; partial rows at
// the range ends (engine.py:182-189 clipping) become single-row tiles.  Tiles
// are shuffled with a fixed seed so any prefix of the list is a representative
// sample of the range (used for the first chunk's threshold).
// force_cols > 0: tiles span whole rows up to that many columns (the
// sorted-column kernel does per-row work, not per-column work)
int build_plan(apex_ctx* c, uint64_t start, uint64_t end, int rows, int nq, Plan*& out, int64_t force_cols = 0) {
  // tile size from the launch's total work (range x queries): big enough to
  // amortize the per-tile setup, small enough for ~6 tiles per warp slot
  const uint64_t span = end - start;
  const int64_t warp_slots = (int64_t)c->sm_count * 24;
  const int64_t target = c->opt_tile_products > 0
                             ? c->opt_tile_products
                             : std::max<int64_t>(8192, (int64_t)(span * (uint64_t)nq / (uint64_t)(c->opt_tiles_per_slot * warp_slots)));
  int64_t cols = std::max<int64_t>(64, std::min<int64_t>(4096, target / rows));
  int64_t p2 = 64;
  while (p2 * 2 <= cols) p2 <<= 1;  // power of two (rounded down): few distinct cached plans
  cols = force_cols > 0 ? force_cols : p2;
  for (auto& p : c->plans) {
    if (p->start == start && p->end == end && p->rows == rows && p->cols == cols) {
      p->stamp = ++c->stamp;
      out = p.get();
      return APEX_OK;
    }
  }
  auto owned = std::make_unique<Plan>();
  Plan& P = *owned;
  P.start = start;
  P.end = end;
  P.rows = rows;
  P.cols = cols;
  P.pair_lo = INT64_MAX;
  P.pair_hi = 0;
  const int n_rx = (int)c->rx.size();
  for (int t = 0; t < n_rx; ++t) {
    const uint64_t off = c->goff[t], size = c->goff[t + 1] - c->goff[t];
    if (off + size <= start || off >= end) continue;
    const DevReaction& R = c->rx[t];
    const uint64_t n_last = (uint64_t)R.size[R.c - 1];
    const uint64_t lo = std::max(start, off) - off, hi = std::min(end, off + size) - off;
    P.pair_lo = std::min<int64_t>(P.pair_lo, R.pair_off[R.c - 1]);
    P.pair_hi = std::max<int64_t>(P.pair_hi, R.pair_off[R.c - 1] + (int64_t)n_last);
    auto emit = [&](uint64_t row0, uint64_t nrows, uint64_t c0, uint64_t c1) {
      for (uint64_t cc = c0; cc < c1; cc += (uint64_t)cols) {
        Tile T;
        T.row0 = row0;
        T.rx = (uint32_t)t;
        T.nrows = (uint32_t)nrows;
        T.col0 = (uint32_t)cc;
        T.ncols = (uint32_t)std::min<uint64_t>((uint64_t)cols, c1 - cc);
        P.tiles.push_back(T);
      }
    };
    const uint64_t r_lo = lo / n_last, c_lo = lo % n_last, r_hi = hi / n_last, c_hi = hi % n_last;
    if (r_lo == r_hi) {
      emit(r_lo, 1, c_lo, c_hi);
      continue;
    }
    uint64_t first_full = r_lo;
    if (c_lo) {
      emit(r_lo, 1, c_lo, n_last);
      first_full = r_lo + 1;
    }
    // whole-row tiles of reactions with long rows (sorted-column kernel):
    // fewer rows per tile, so a tile whose rows admit many pairs becomes
    // several items that run on different warps instead of one long item
    uint64_t rows_t = (uint64_t)rows;
    if (force_cols > 0 && c->opt_split_cols > 0 && n_last >= (uint64_t)c->opt_split_cols)
      rows_t = (uint64_t)std::max<int64_t>(1, std::min<int64_t>(rows, c->opt_split_rows));
    for (uint64_t r = first_full; r < r_hi; r += rows_t) emit(r, std::min<uint64_t>(rows_t, r_hi - r), 0, n_last);
    if (c_hi) emit(r_hi, 1, 0, c_hi);
  }
  if (P.tiles.size() > 0xffffffffull) return set_err(APEX_ELIMIT, "too many enumeration tiles");
  std::mt19937_64 rng(0x5eed5eedull ^ start ^ (end << 1));
  std::shuffle(P.tiles.begin(), P.tiles.end(), rng);
  if (force_cols > 0 && c->opt_heavy_first) {
    // whole-row tiles (sorted-column kernel): the most products first, so the
    // items whose rows can admit the most pairs start early and the tail of
    // the dynamically distributed work is made of light items
    std::stable_sort(P.tiles.begin(), P.tiles.end(), [](const Tile& a, const Tile& b) {
      return (uint64_t)a.nrows * a.ncols > (uint64_t)b.nrows * b.ncols;
    });
  }
  P.prefix.resize(P.tiles.size() + 1);
  P.prefix[0] = 0;
  for (size_t i = 0; i < P.tiles.size(); ++i)
    P.prefix[i + 1] = P.prefix[i] + (uint64_t)P.tiles[i].nrows * P.tiles[i].ncols;
  if (P.prefix.back() != span) return set_err(APEX_EINVAL, "internal: tile plan does not cover the range");
  if (P.pair_lo == INT64_MAX) P.pair_lo = P.pair_hi = 0;
  APEX_TRY(P.d_tiles.ensure(std::max<size_t>(1, P.tiles.size()) * sizeof(Tile)));
  if (!P.tiles.empty())
    APEX_CU(cudaMemcpy(P.d_tiles.p, P.tiles.data(), P.tiles.size() * sizeof(Tile), cudaMemcpyHostToDevice));
  // keep a small cache
  if (c->plans.size() >= 8) {
    auto it = std::min_element(c->plans.begin(), c->plans.end(),
                               [](const std::unique_ptr<Plan>& a, const std::unique_ptr<Plan>& b) {
                                 return a->stamp < b->stamp;
                               });
    if (c->batch.plan == it->get()) c->batch.plan = nullptr;
    if (c->batch.plan_rows == it->get()) c->batch.plan_rows = nullptr;
    (*it)->d_tiles.release();
    c->plans.erase(it);
  }
  P.stamp = ++c->stamp;
  c->plans.push_back(std::move(owned));
  out = c->plans.back().get();
  return APEX_OK;
}

int make_tests(const apex_ctx* c, const apex_query_spec& q, QTests& T) {
  T.nt = 1;
  T.task[0] = q.objective_task;
  T.lower[0] = q.maximize ? 1 : 0;
  T.beta[0] = 0.0;
  std::vector<double> lo(c->n_tasks, -INFINITY), up(c->n_tasks, INFINITY);
  for (int i = 0; i < q.n_constraints; ++i) {
    const apex_constraint& k = q.constraints[i];
    if (k.task < 0 || k.task >= c->n_tasks) return set_err(APEX_ETASK, "unknown task index " + std::to_string(k.task));
    if (!(k.lower < k.upper)) return set_err(APEX_EINVAL, "constraint bounds must satisfy lower < upper");
    lo[k.task] = std::max(lo[k.task], k.lower);
    up[k.task] = std::min(up[k.task], k.upper);
  }
  for (int t = 0; t < c->n_tasks; ++t) {
    if (std::isfinite(up[t])) {
      if (T.nt >= kMaxTests) return set_err(APEX_ELIMIT, "query has more than 23 finite bounds");
      T.task[T.nt] = t; T.lower[T.nt] = 0; T.beta[T.nt] = up[t]; ++T.nt;
    }
    if (std::isfinite(lo[t])) {
      if (T.nt >= kMaxTests) return set_err(APEX_ELIMIT, "query has more than 23 finite bounds");
      T.task[T.nt] = t; T.lower[T.nt] = 1; T.beta[T.nt] = lo[t]; ++T.nt;
    }
  }
  return APEX_OK;
}

int kernel_nt(int nt) {
  static const int sizes[] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 14, 16, 20, 24};
  for (int s : sizes)
    if (nt <= s) return s;
  return -1;
}

using ScanFn = void (*)(const ScanLaunch);

template <int NT, int RL, int MODE>
ScanFn scan_ptr() { return scan_kernel<NT, RL, MODE>; }

// (one full-predicate form is compiled: one row per lane, FSETP compare
// chain — the FADD2 / two-rows-per-lane variants never won an A/B and only
// cost build time)
ScanFn pick_scan(int nt, int rl, int mode) {
  (void)rl;
  (void)mode;
#define CASE(N)                                                                         \
  case N:                                                                               \
    return scan_ptr<N, 1, 0>();
  switch (nt) {
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(14)
    CASE(16) CASE(20) CASE(24)
    default: return nullptr;
  }
#undef CASE
}

size_t scan_smem(int nt, int cb) {
  const int ntp = (nt + 3) / 4 * 4;
  return (size_t)kScanWarps * 2 * cb * ntp * sizeof(float) + (size_t)kScanWarps * 2 * sizeof(uint64_t);
}

int scan_occupancy(apex_ctx* c, ScanFn fn, size_t smem, int* occ) {
  // cached per (kernel, smem) in the context (one device per context; the
  // dynamic-smem attribute is per device): the attribute call and the
  // occupancy query cost microseconds on every launch otherwise
  // (the attribute is per kernel: only ever raise it, so a cached occupancy
  // for a larger request stays launchable)
  auto& cache = c->occ_cache;
  auto& attr = c->attr_cache;
  for (auto& e : cache)
    if (e.first.first == (const void*)fn && e.first.second == smem) {
      *occ = e.second;
      return APEX_OK;
    }
  size_t cur = 0;
  for (auto& a : attr)
    if (a.first == (const void*)fn) cur = a.second;
  if (smem > cur) {
    APEX_CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    bool found = false;
    for (auto& a : attr)
      if (a.first == (const void*)fn) { a.second = smem; found = true; }
    if (!found) attr.push_back({(const void*)fn, smem});
  }
  APEX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, (const void*)fn, kScanWarps * 32, smem));
  if (*occ < 1) return set_err(APEX_ELIMIT, "enumeration kernel does not fit on an SM");
  cache.push_back({{(const void*)fn, smem}, *occ});
  return APEX_OK;
}

// Binding state built once per (library, table), on the device (bind.cuh):
// every R-group column of every task sorted by (value, column); from those,
// per task the sorted last-R-group columns with their quantile tables (the
// sorted-column kernel) and the corner seed lists — for every task, direction
// and (reaction, R-group) the digits of the best-m synthons (largest first for
// maximize, smallest first for minimize), m chosen so a reaction's corner has
// ~4096 products.  Only the list metadata is computed on the host.
int build_corners(apex_ctx* c) {
  const int n_rx = (int)c->rx.size();
  std::vector<int32_t> slot_off((size_t)n_rx * kMaxRg, 0), m((size_t)n_rx * kMaxRg, 0);
  std::vector<unsigned long long> coff(n_rx + 1, 0);
  static const int base_c[kMaxRg + 1] = {1, 4096, 64, 16, 8, 5, 4};
  int64_t slots = 0;
  for (int t = 0; t < n_rx; ++t) {
    const DevReaction& R = c->rx[t];
    unsigned long long prod = 1;
    for (int j = 0; j < R.c; ++j) {
      const int mj = (int)std::min<int64_t>(R.size[j], base_c[R.c]);
      m[(size_t)t * kMaxRg + j] = mj;
      slot_off[(size_t)t * kMaxRg + j] = (int32_t)slots;
      slots += mj;
      prod *= (unsigned long long)mj;
    }
    coff[t + 1] = coff[t] + prod;
  }
  if (slots > INT32_MAX) return set_err(APEX_ELIMIT, "corner lists too large");
  // segments: (task, R-group) for every R-group of every reaction
  std::vector<BindSeg> segs;
  int64_t scratch = 0;
  for (int task = 0; task < c->n_tasks; ++task)
    for (int t = 0; t < n_rx; ++t) {
      const DevReaction& R = c->rx[t];
      for (int j = 0; j < R.c; ++j) {
        BindSeg S;
        S.pair = R.pair_off[j];
        S.n = (int32_t)R.size[j];
        S.task = task;
        S.scratch = -1;
        if (S.n > kBindSmem) {
          int64_t P = 1;
          while (P < S.n) P <<= 1;
          S.scratch = scratch;
          scratch += P;
        }
        segs.push_back(S);
      }
    }
  cudaStream_t s = c->stream;
  DBuf d_segs, d_keys, d_scratch;
  APEX_TRY(d_segs.ensure(std::max<size_t>(1, segs.size()) * sizeof(BindSeg)));
  APEX_TRY(d_keys.ensure(std::max<size_t>(1, (size_t)c->n_tasks * c->n_pairs) * sizeof(unsigned long long)));
  APEX_TRY(d_scratch.ensure(std::max<int64_t>(1, scratch) * sizeof(unsigned long long)));
  if (!segs.empty())
    APEX_CU(cudaMemcpyAsync(d_segs.p, segs.data(), segs.size() * sizeof(BindSeg), cudaMemcpyHostToDevice, s));
  const size_t pc = (size_t)std::max<int64_t>(c->pcols, 4);
  APEX_TRY(c->d_lists.ensure(std::max<size_t>(1, (size_t)c->n_tasks * 2 * slots) * sizeof(int32_t)));
  APEX_TRY(c->d_slot_off.ensure(std::max<size_t>(1, slot_off.size()) * sizeof(int32_t)));
  APEX_TRY(c->d_m.ensure(std::max<size_t>(1, m.size()) * sizeof(int32_t)));
  APEX_TRY(c->d_coff.ensure(coff.size() * sizeof(unsigned long long)));
  APEX_TRY(c->d_sorted_x.ensure((size_t)c->n_tasks * pc * sizeof(float)));
  APEX_TRY(c->d_sorted_col.ensure((size_t)c->n_tasks * pc * sizeof(uint32_t)));
  APEX_TRY(c->d_quant.ensure(std::max<size_t>(1, (size_t)c->n_tasks * n_rx * (kQuant + 1)) * sizeof(float)));
  APEX_CU(cudaMemsetAsync(c->d_sorted_x.p, 0, (size_t)c->n_tasks * pc * sizeof(float), s));
  APEX_CU(cudaMemsetAsync(c->d_sorted_col.p, 0, (size_t)c->n_tasks * pc * sizeof(uint32_t), s));
  if (!slot_off.empty())
    APEX_CU(cudaMemcpyAsync(c->d_slot_off.p, slot_off.data(), slot_off.size() * 4, cudaMemcpyHostToDevice, s));
  if (!m.empty()) APEX_CU(cudaMemcpyAsync(c->d_m.p, m.data(), m.size() * 4, cudaMemcpyHostToDevice, s));
  APEX_CU(cudaMemcpyAsync(c->d_coff.p, coff.data(), coff.size() * 8, cudaMemcpyHostToDevice, s));
  if (!segs.empty()) {
    bind_sort_kernel<<<(unsigned)segs.size(), 1024, 0, s>>>(d_segs.as<BindSeg>(), c->d_values.as<float>(), c->n_pairs,
                                                            d_keys.as<unsigned long long>(),
                                                            d_scratch.as<unsigned long long>());
    APEX_CU(cudaGetLastError());
    BindEmit E;
    E.rx = c->d_rx.as<DevReaction>();
    E.n_rx = n_rx;
    E.n_pairs = c->n_pairs;
    E.keys = d_keys.as<unsigned long long>();
    E.sx = c->d_sorted_x.as<float>();
    E.scol = c->d_sorted_col.as<uint32_t>();
    E.pcols = (int64_t)pc;
    E.quant = c->d_quant.as<float>();
    E.lists = c->d_lists.as<int32_t>();
    E.slot_off = c->d_slot_off.as<int32_t>();
    E.m = c->d_m.as<int32_t>();
    E.slots = slots;
    bind_emit_kernel<<<dim3((unsigned)n_rx, (unsigned)c->n_tasks), 256, 0, s>>>(E);
    APEX_CU(cudaGetLastError());
  }
  if (c->n_tasks <= 16 && c->opt_packed16) {
    APEX_TRY(c->d_packed16.ensure(std::max<size_t>(1, (size_t)c->n_pairs * 16) * sizeof(float)));
    const int64_t tot = c->n_pairs * 16;
    bind_pack16_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((tot + 255) / 256, (int64_t)c->sm_count * 16)), 256,
                         0, s>>>(c->d_values.as<float>(), c->n_pairs, c->n_tasks, c->d_packed16.as<float>());
    APEX_CU(cudaGetLastError());
    c->packed16_ok = true;
  } else {
    c->packed16_ok = false;
  }
  // row-prefix table (sorted-column scan and constraint pre-pass): every
  // row's fp64 prefix sums for every task, when it fits the budget
  c->rowp_ok = false;
  if (c->opt_rowp && c->rows_total > 0 &&
      (unsigned __int128)c->rows_total * (unsigned __int128)c->n_tasks * 8u <= (unsigned __int128)c->opt_rowp_bytes) {
    APEX_TRY(c->d_rowp.ensure((size_t)c->rows_total * c->n_tasks * sizeof(double)));
    int64_t max_rows = 1;
    for (const auto& R : c->rx) max_rows = std::max<int64_t>(max_rows, (int64_t)R.n_rows);
    const unsigned gx = (unsigned)std::min<int64_t>((max_rows + 255) / 256, 4096);
    bind_rowp_kernel<<<dim3(gx, (unsigned)n_rx), 256, 0, s>>>(c->d_rx.as<DevReaction>(), c->d_values.as<float>(),
                                                               c->n_pairs, c->n_tasks, c->rows_total,
                                                               c->d_rowp.as<double>());
    APEX_CU(cudaGetLastError());
    c->rowp_ok = true;
  }
  APEX_CU(cudaStreamSynchronize(s));
  d_segs.release();
  d_keys.release();
  d_scratch.release();
  c->corner_slots = slots;
  c->corner_total = coff[n_rx];
  c->corners_ok = true;
  return APEX_OK;
}

// ---------------------------------------------------------------------------
// Batch lifecycle: prepare (host: tests, plan, workspaces, descriptor upload),
// enqueue (device pipeline, no host sync), check (one sync: overflow check and
// exact re-run with the final bound if the candidate buffer overflowed).

// CTAs per query of the bucketed finalize: about kFinRowsPerCta ranks each,
// within one wave (one CTA per SM) and kFinMaxSplit
constexpr int64_t kCornerTotal = 160000;  // corner seed: products per pass (all queries)

// Reciprocal for the scan kernels' item -> (tile, query) split (item_div):
// ceil(2^32 / nq) is exact for every item index below 2^26 when nq <= 64
// (error below item / 2^32 < 1/64 <= 1/nq); 0 = divide.
unsigned nq_magic(unsigned tiles, int nq) {
  if (nq < 2 || nq > 64 || (uint64_t)tiles * (uint64_t)nq >= (1ull << 26)) return 0u;
  return (unsigned)(((1ull << 32) + (uint64_t)nq - 1) / (uint64_t)nq);
}
constexpr size_t kCtlHdr = (offsetof(QCtl, hist) + 15) / 16 * 16;  // control header bytes per query in the result block

int fin_splits(const apex_ctx* c, int64_t k_max, int nq) {
  const int64_t want = (k_max + kFinRowsPerCta - 1) / kFinRowsPerCta;
  return (int)std::max<int64_t>(
      1, std::min<int64_t>({want, c->opt_fin_bucket, (int64_t)kFinMaxSplit, (int64_t)c->sm_count / std::max(nq, 1)}));
}

int prepare_batch(apex_ctx* c, const apex_query_spec* qs_in, int nq, bool finalize) {
  Batch& B = c->batch;
  if (!c->corners_ok) APEX_TRY(build_corners(c));
  // tests per query, then group queries by the kernel's test class (one scan
  // launch per class, so no query pays for another's padding)
  std::vector<QTests> tests_in(nq);
  std::vector<int> cls(nq);
  int nt_max = 1;
  for (int i = 0; i < nq; ++i) {
    APEX_TRY(make_tests(c, qs_in[i], tests_in[i]));
    if (qs_in[i].n_constraints > kMaxCons) return set_err(APEX_ELIMIT, "more than 32 constraints in a query");
    cls[i] = kernel_nt(tests_in[i].nt);
    if (cls[i] < 0) return set_err(APEX_ELIMIT, "too many tests");
    nt_max = std::max(nt_max, tests_in[i].nt);
  }
  B.perm.resize(nq);
  std::iota(B.perm.begin(), B.perm.end(), 0);
  std::stable_sort(B.perm.begin(), B.perm.end(), [&](int a, int b) { return cls[a] < cls[b]; });
  B.qs.resize(nq);
  B.cons.assign(nq, {});
  B.tests.resize(nq);
  B.cls_nt.clear();
  B.cls_begin.clear();
  for (int i = 0; i < nq; ++i) {
    const int o = B.perm[i];
    B.qs[i] = qs_in[o];
    B.cons[i].assign(qs_in[o].constraints, qs_in[o].constraints + qs_in[o].n_constraints);
    B.qs[i].constraints = B.cons[i].data();
    B.tests[i] = tests_in[o];
    if (B.cls_nt.empty() || B.cls_nt.back() != cls[o]) {
      B.cls_nt.push_back(cls[o]);
      B.cls_begin.push_back(i);
    }
  }
  B.cls_begin.push_back(nq);
  const apex_query_spec* qs = B.qs.data();
  B.nq = nq;
  B.finalize = finalize;
  B.copy_out = finalize && c->copy_next;
  c->copy_next = false;
  B.st = RunStats();
  B.k_max = 0;
  for (int i = 0; i < nq; ++i) B.k_max = std::max<int64_t>(B.k_max, qs[i].k);
  B.NT = kernel_nt(nt_max);
  B.ntp = (B.NT + 3) / 4 * 4;
  B.rl = (int)c->opt_rl;
  if (B.rl != 1 && B.rl != 2) B.rl = 1;
  if (c->opt_mode != 2) B.rl = 1;  // two rows per lane: admission-first streaming kernel only
  APEX_TRY(build_plan(c, qs[0].start, qs[0].end, 32 * B.rl, nq, B.plan));
  B.plan_rows = nullptr;
  if (c->opt_mode >= 2 && c->opt_sorted && c->trace_cap == 0) {
    Plan* keep = B.plan;
    int64_t max_last = 1;
    for (const auto& R : c->rx) max_last = std::max<int64_t>(max_last, R.size[R.c - 1]);
    APEX_TRY(build_plan(c, qs[0].start, qs[0].end, 32, nq, B.plan_rows, max_last));
    B.plan = keep;  // still cached: build_plan never evicts the most recently used plan
  }

  if ((int)c->slots.size() < nq) c->slots.resize(nq);
  for (int i = 0; i < nq; ++i) {
    Slot& S = c->slots[i];
    const int64_t k = qs[i].k;
    // candidate buffer: opt_cap entries, shared out over large batches (an
    // overflow is detected and re-run exactly, so this only trades memory
    // for the rare re-run)
    const int64_t cap = std::max<int64_t>(std::min<int64_t>(c->opt_cap, (int64_t)(1ll << 27) / std::max(nq, 1)),
                                          16 * k + 4096);
    if (c->opt_mode >= 2) APEX_TRY(S.obj_col.ensure((size_t)std::max<int64_t>(c->pcols, 4) * sizeof(float)));
    if (c->opt_mode != 2) {
      const int ntp_i = (kernel_nt(B.tests[i].nt) + 3) / 4 * 4;
      APEX_TRY(S.packed.ensure((size_t)std::max<int64_t>(c->n_pairs, 1) * ntp_i * sizeof(float)));
    }
    APEX_TRY(S.buf.ensure((size_t)cap * sizeof(Entry)));
    APEX_TRY(S.sel.ensure((size_t)std::max<int64_t>(k, 1) * sizeof(Entry)));
    APEX_TRY(S.sorted.ensure((size_t)std::max<int64_t>(k, 1) * sizeof(Entry)));
  }
  APEX_TRY(c->d_ctls.ensure((size_t)nq * sizeof(QCtl)));
  c->out_off.assign(nq + 1, 0);
  for (int i = 0; i < nq; ++i)
    c->out_off[i + 1] = c->out_off[i] + (out_bytes(std::max<int64_t>(qs[i].k, 1), qs[i].n_constraints) + 15) / 16 * 16;
  // the control headers ride at the tail of the result block (one D2H)
  APEX_TRY(c->d_out.ensure(c->out_off[nq] + (size_t)nq * kCtlHdr));
  APEX_TRY(c->h_out.ensure(c->out_off[nq] + (size_t)nq * kCtlHdr));
  // everything enqueue_batch touches is allocated here (no allocation may
  // happen while the pipeline is being captured into a CUDA graph)
  APEX_TRY(c->h_ctl.ensure(nq * sizeof(QCtl)));
  APEX_TRY(c->d_work.ensure(kWorkWords * sizeof(unsigned)));
  {
    const void* before = c->d_hists.p;
    APEX_TRY(c->d_hists.ensure((size_t)nq * kHistWords * sizeof(unsigned)));
    if (c->d_hists.p != before) APEX_CU(cudaMemset(c->d_hists.p, 0, c->d_hists.bytes));  // lazy zeroing starts clean
  }
  if (c->opt_fin_bucket && c->opt_fin_part && fin_splits(c, B.k_max, nq) >= kFinSuffixMin)
    // partitioned bucketed finalize: one region per (query, CTA)
    APEX_TRY(c->d_fin_scratch.ensure((size_t)nq * fin_splits(c, B.k_max, nq) * kSmallSel * sizeof(Entry)));
  std::vector<ScanQuery> hq(nq);
  for (int i = 0; i < nq; ++i) {
    Slot& S = c->slots[i];
    const apex_query_spec& q = qs[i];
    const QTests& T = B.tests[i];
    ScanQuery& Q = hq[i];
    std::memset(&Q, 0, sizeof(Q));
    Q.packed = S.packed.as<float>();
    Q.obj_col = S.obj_col.as<float>();
    Q.buf = S.buf.as<Entry>();
    Q.sel = S.sel.as<Entry>();
    Q.sorted = S.sorted.as<Entry>();
    Q.hist = c->d_hists.as<unsigned>() + (size_t)i * kHistWords;
    Q.coarse = Q.hist + kHistBins;
    Q.seed_hist = Q.coarse + 256;
    Q.ctl = c->d_ctls.as<QCtl>() + i;
    Q.cap = S.buf.bytes / sizeof(Entry);
    {
      // power of two >= max(refresh interval, 256): the kernels test crossings with a shift
      const int64_t want = std::max<int64_t>(c->opt_refresh > 0 ? c->opt_refresh : q.k, 256);
      unsigned sh = 8;
      while ((1ll << sh) < want && sh < 62) ++sh;
      Q.refresh_shift = sh;
    }
    Q.k = q.k;
    // pair budget of the sorted-column kernel (automatic choice only): a
    // query that would enumerate more than 1/kBailDiv of its range gives up
    // and re-runs with the full predicate (which exists for its test count)
    Q.admit_budget = ~0ull;
    if (c->opt_mode == 3 && c->opt_bail > 0 && pick_scan(kernel_nt(T.nt), 1, 0)) {
      const uint64_t span = q.end - q.start;
      Q.admit_budget = std::max<uint64_t>((uint64_t)c->opt_bail_min, span / (uint64_t)c->opt_bail);
    }
    Q.nt = T.nt;
    Q.ntp = (kernel_nt(T.nt) + 3) / 4 * 4;
    Q.slot = B.perm[i];
    Q.maximize = q.maximize ? 1 : 0;
    Q.obj_task = q.objective_task;
    Q.n_cons = q.n_constraints;
    for (int t = 0; t < T.nt; ++t) {
      Q.test_task[t] = T.task[t];
      Q.test_lower[t] = T.lower[t];
      Q.test_beta[t] = T.beta[t];
      Q.test_bias[t] = c->biases[T.task[t]];
    }
    for (int m = 0; m < q.n_constraints; ++m) Q.cons_task[m] = q.constraints[m].task;
    const int64_t kk = std::max<int64_t>(q.k, 1);
    unsigned char* o = c->d_out.as<unsigned char>() + c->out_off[i];
    Q.out_g = reinterpret_cast<unsigned long long*>(o);
    Q.out_obj = reinterpret_cast<double*>(o + 8 * kk);
    Q.out_cons = reinterpret_cast<double*>(o + 16 * kk);
    Q.out_rx = reinterpret_cast<int32_t*>(o + (16 + 8 * (size_t)q.n_constraints) * kk);
    Q.out_dig = reinterpret_cast<int32_t*>(o + (20 + 8 * (size_t)q.n_constraints) * kk);
  }
  // constraint sets shared by several queries: the sorted-column kernel
  // reads their per-row thresholds and best range from a pre-pass
  B.cset_leader.clear();
  B.cset_tests = 0;
  for (int i = 0; i < nq; ++i) hq[i].cset = -1;
  if (B.plan_rows && c->opt_cpre) {
    auto same = [&](int a, int b) {
      const QTests &A = B.tests[a], &Bt = B.tests[b];
      if (A.nt != Bt.nt) return false;
      for (int t = 1; t < A.nt; ++t)
        if (A.task[t] != Bt.task[t] || A.lower[t] != Bt.lower[t] || A.beta[t] != Bt.beta[t]) return false;
      return true;
    };
    for (int i = 0; i < nq; ++i) {
      if (hq[i].cset >= 0 || B.tests[i].nt < 2) continue;
      int members = 0;
      for (int j = i + 1; j < nq; ++j) members += (hq[j].cset < 0 && same(i, j)) ? 1 : 0;
      if (!members) continue;
      const int id = (int)B.cset_leader.size();
      B.cset_leader.push_back(i);
      for (int j = i; j < nq; ++j)
        if (j == i || (hq[j].cset < 0 && same(i, j))) {
          hq[j].cset = id;
          hq[j].cset_off = (int32_t)B.cset_tests;
        }
      B.cset_tests += B.tests[i].nt - 1;
    }
    if (!B.cset_leader.empty()) {
      const int64_t rows_pad = (int64_t)B.plan_rows->tiles.size() * 32;
      APEX_TRY(c->d_cthr.ensure((size_t)std::max<int64_t>(B.cset_tests * rows_pad, 1) * sizeof(float)));
      APEX_TRY(c->d_cqc.ensure((size_t)std::max<int64_t>(B.cset_tests * rows_pad, 1)));
      APEX_TRY(c->d_cbest.ensure((size_t)std::max<int64_t>((int64_t)B.cset_leader.size() * rows_pad, 1) * 16));
    }
  }
  // upload the descriptors only when they changed (pinned staging is reused:
  // wait for the previous copy out of it first)
  const size_t bytes = nq * sizeof(ScanQuery);
  if (c->opt_force_upload || c->uploaded.size() != (size_t)nq ||
      std::memcmp(c->uploaded.data(), hq.data(), bytes) != 0) {
    APEX_CU(cudaEventSynchronize(c->upload_ev));
    APEX_TRY(c->d_queries.ensure(bytes));
    APEX_TRY(c->h_queries.ensure(bytes));
    std::memcpy(c->h_queries.p, hq.data(), bytes);
    APEX_CU(cudaMemcpyAsync(c->d_queries.p, c->h_queries.p, bytes, cudaMemcpyHostToDevice, c->stream));
    APEX_CU(cudaEventRecord(c->upload_ev, c->stream));
    c->uploaded = hq;
    B.st.h2d_bytes += (int64_t)bytes;
  }
  return APEX_OK;
}

// Enqueue the device pipeline of the prepared batch.  pre: per-query presets
// of an exact re-run after an overflow (check_batch), or nullptr.
// Stage timing event; inside a stream capture it is recorded as an external
// event-record node so the graph replay still timestamps it.
cudaError_t stage_mark(apex_ctx* c, int e, cudaStream_t s) {
  // stage events are diagnostics (option "stages"): each recorded event is a
  // node on the pass's critical path (a few microseconds per node in a graph)
  if (!c->opt_stages) return cudaSuccess;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) return cudaEventRecordWithFlags(c->ev[e], s, cudaEventRecordExternal);
  return cudaEventRecord(c->ev[e], s);
}

// Final exact selection of a batch whose candidate buffers and bounds are
// set: small sets sort + materialize in one CTA per query; the rest go
// through the cooperative radix select (launched over chunks of queries that
// fit co-resident), rank, scatter and (finalize) materialization.
int enqueue_select(apex_ctx* c, const ScanQuery* dq, int nq, int64_t k_max, bool finalize, RunStats& st,
                   cudaStream_t s, bool mark, bool compute_bound = true, bool skip_large = false) {
  MatLaunch M;
  M.queries = dq;
  M.rx = c->d_rx.as<DevReaction>();
  M.g_off = c->d_goff.as<unsigned long long>();
  M.n_rx = (int)c->rx.size();
  M.values = c->d_values.as<float>();
  M.p16 = (c->packed16_ok && c->opt_packed16) ? c->d_packed16.as<float>() : nullptr;
  M.n_pairs = c->n_pairs;
  M.biases = c->d_biases.as<double>();
  {
    const size_t smem_small = (size_t)kSmallSel * sizeof(Entry);
    if (!c->attr_small) {  // per context = per device (the attribute is per device)
      APEX_CU(cudaFuncSetAttribute((const void*)finalize_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem_small));
      c->attr_small = true;
    }
    if (compute_bound && c->opt_fin_bucket) {
      // bucketed: ns CTAs per query (one wave), rows materialized inside
      const size_t smem_bucket = fin_bucket_smem();
      if (!c->attr_bucket) {
        APEX_CU(cudaFuncSetAttribute((const void*)finalize_bucket_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bucket));
        c->attr_bucket = true;
      }
      const int ns = fin_splits(c, k_max, nq);
      // partitioned (cooperative: the CTAs of a query meet at a barrier) when
      // the scratch regions were allocated with the batch
      const bool part = c->opt_fin_part && ns >= kFinSuffixMin &&
                        c->d_fin_scratch.bytes >= (size_t)nq * ns * kSmallSel * sizeof(Entry);
      int mat = finalize ? 1 : 0;
      Entry* scratch = part ? c->d_fin_scratch.as<Entry>() : nullptr;
      if (part) {
        void* args[] = {(void*)&M, (void*)&mat, (void*)&scratch};
        APEX_CU(cudaLaunchCooperativeKernel((const void*)finalize_bucket_kernel, dim3((unsigned)ns, (unsigned)nq),
                                            dim3(kFinThreads), args, smem_bucket, s));
      } else {
        finalize_bucket_kernel<<<dim3((unsigned)ns, (unsigned)nq), kFinThreads, smem_bucket, s>>>(M, mat, scratch);
      }
    } else {
      // (materialization runs after, for every query, in materialize_kernel)
      finalize_small_kernel<<<nq, 1024, smem_small, s>>>(M, 0, compute_bound ? 1 : 0);
    }
    ++st.launches;
  }
  if (!skip_large) {
    if (!c->occ_sel)
      APEX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->occ_sel, (const void*)select_kernel, kSelectThreads, 0));
    const int resident = std::max(1, c->occ_sel * c->sm_count);
    const int per_q = (int)std::max<int64_t>(1, std::min<int64_t>(c->opt_select_ctas, resident / std::max(nq, 1)));
    const int q_chunk = std::max(1, resident / per_q);
    for (int q0 = 0; q0 < nq; q0 += q_chunk) {
      const ScanQuery* dqc = dq + q0;
      void* args[] = {(void*)&dqc};
      APEX_CU(cudaLaunchCooperativeKernel((const void*)select_kernel, dim3(per_q, std::min(q_chunk, nq - q0)),
                                          dim3(kSelectThreads), args, 0, s));
      ++st.launches;
    }
  }
  if (mark) APEX_CU(stage_mark(c, 4, s));
  if (finalize) {
    if (!skip_large) {
      const int ib = (int)((k_max + 255) / 256);
      sort_chunks_kernel<<<dim3((unsigned)((k_max + kSortChunk - 1) / kSortChunk), nq), 1024, 0, s>>>(dq);
      merge_rank_kernel<<<dim3(ib, nq), 256, 0, s>>>(dq);
      st.launches += 2;
    }
    // (queries the bucketed finalize materialized are skipped on the device;
    // a signature whose queries all fit it needs no launch)
    if (!(skip_large && compute_bound && c->opt_fin_bucket)) {
      materialize_kernel<<<dim3((unsigned)((k_max + 127) / 128), nq), 128, 0, s>>>(M);
      st.launches += 1;
    }
  }
  return APEX_OK;
}

int enqueue_batch(apex_ctx* c, const RunPreset* tau0) {
  Batch& B = c->batch;
  RunStats& st = B.st;
  const int nq = B.nq;
  Plan* plan = B.plan;
  const uint64_t start = B.qs[0].start, end = B.qs[0].end, span = end - start;
  cudaStream_t s = c->stream;
  const ScanQuery* dq = c->d_queries.as<ScanQuery>();
  APEX_CU(stage_mark(c, 0, s));
  if (tau0) {
    APEX_TRY(c->d_tau0.ensure(nq * sizeof(RunPreset)));
    APEX_TRY(c->h_tau0.ensure(nq * sizeof(RunPreset)));
    APEX_CU(cudaStreamSynchronize(s));
    std::memcpy(c->h_tau0.p, tau0, nq * sizeof(RunPreset));
    APEX_CU(cudaMemcpyAsync(c->d_tau0.p, c->h_tau0.p, nq * sizeof(RunPreset), cudaMemcpyHostToDevice, s));
    st.h2d_bytes += nq * (int64_t)sizeof(RunPreset);
  }
  // kernel choice: admission-first (admit), full predicate (full), or per query (auto)
  const bool admit = c->opt_mode >= 2;
  // the sorted-column kernel takes every query except (auto, on the device)
  // threshold-less ones with a non-sparse feasible set, which stream the
  // full predicate; signatures that needed none of those skip its launches
  const bool sorted_all = c->opt_mode == 3 && B.plan_rows;
  const bool full = c->opt_mode != 2 && !B.no_full;
  const int autok = (c->opt_mode == 3 && !tau0) ? (B.no_full ? 3 : sorted_all ? 2 : 1) : 0;
  // sorted-column constraint pre-pass (shared constraint sets), on a third
  // stream beside the histogram clear, control init and seed kernels; joined
  // before the enumeration
  const bool sorted_go = admit && B.plan_rows &&
                         !(span >= (uint64_t)c->opt_chunk_min && c->opt_chunk_div > 1 && plan->tiles.size() > 1);
  const bool cpre = sorted_go && !B.cset_leader.empty();
  bool cpre_forked = false;
  auto launch_cpre = [&]() -> int {
    if (!cpre_forked) APEX_CU(cudaEventRecord(c->fork2_ev, s));
    APEX_CU(cudaStreamWaitEvent(c->side2, c->fork2_ev, 0));
    ConsPre P{};
    P.queries = dq;
    P.tiles = B.plan_rows->d_tiles.as<Tile>();
    P.n_tiles = (unsigned)B.plan_rows->tiles.size();
    P.rx = c->d_rx.as<DevReaction>();
    P.values = c->d_values.as<float>();
    P.p16 = (c->packed16_ok && c->opt_packed16) ? c->d_packed16.as<float>() : nullptr;
    P.n_pairs = c->n_pairs;
    P.sx = c->d_sorted_x.as<float>();
    P.quant = c->d_quant.as<float>();
    P.pcols = std::max<int64_t>(c->pcols, 4);
    P.n_rx = (int)c->rx.size();
    P.cthr = c->d_cthr.as<float>();
    P.cbest = c->d_cbest.as<int4>();
    P.rows_pad = (int64_t)P.n_tiles * 32;
    P.cqc = c->d_cqc.as<unsigned char>();
    P.rowp = (c->rowp_ok && c->opt_rowp) ? c->d_rowp.as<double>() : nullptr;
    P.rows_total = c->rows_total;
    auto cpre_grid = [&](int64_t items) {
      const int64_t full = (items + 7) / 8;
      return (unsigned)std::max<int64_t>(1, c->opt_cpre_ctas > 0 ? std::min<int64_t>(full, c->sm_count * c->opt_cpre_ctas)
                                                                  : full);
    };
    if (c->opt_cpre_fused) {
      // one kernel: (tile, set) items
      for (size_t s0 = 0; s0 < B.cset_leader.size(); s0 += kConsPreItems) {
        P.n = (int)std::min<size_t>(kConsPreItems, B.cset_leader.size() - s0);
        for (int j = 0; j < P.n; ++j) P.q[j] = B.cset_leader[s0 + j];
        const int64_t items = (int64_t)P.n_tiles * P.n;
        cons_fused_kernel<<<cpre_grid(items), 256, 0, c->side2>>>(P);
        ++st.launches;
      }
      APEX_CU(cudaEventRecord(c->join2_ev, c->side2));
      return APEX_OK;
    }
    // A: (tile, test) threshold + quantile count items
    std::vector<std::pair<int, int>> tests;
    for (int ld : B.cset_leader)
      for (int i = 1; i < B.tests[ld].nt; ++i) tests.push_back({ld, i});
    for (size_t s0 = 0; s0 < tests.size(); s0 += kConsPreItems) {
      P.n = (int)std::min<size_t>(kConsPreItems, tests.size() - s0);
      for (int j = 0; j < P.n; ++j) {
        P.q[j] = tests[s0 + j].first;
        P.ti[j] = (unsigned char)tests[s0 + j].second;
      }
      const int64_t items = (int64_t)P.n_tiles * P.n;
      cons_thr_kernel<<<cpre_grid(items), 256, 0, c->side2>>>(P);
      ++st.launches;
    }
    // B: (tile, set) choice of the most selective test + its exact range
    for (size_t s0 = 0; s0 < B.cset_leader.size(); s0 += kConsPreItems) {
      P.n = (int)std::min<size_t>(kConsPreItems, B.cset_leader.size() - s0);
      for (int j = 0; j < P.n; ++j) P.q[j] = B.cset_leader[s0 + j];
      const int64_t items = (int64_t)P.n_tiles * P.n;
      cons_best_kernel<<<cpre_grid(items), 256, 0, c->side2>>>(P);
      ++st.launches;
    }
    APEX_CU(cudaEventRecord(c->join2_ev, c->side2));
    return APEX_OK;
  };
  if (cpre && c->opt_cpre == 2) APEX_TRY(launch_cpre());
  if (!c->opt_lazy_hist) APEX_CU(cudaMemsetAsync(c->d_hists.p, 0, (size_t)nq * kHistWords * sizeof(unsigned), s));
  init_ctl_kernel<<<dim3(nq, c->opt_lazy_hist ? 8 : 1), 1024, 0, s>>>(dq, tau0 ? c->d_tau0.as<RunPreset>() : nullptr,
                                      (c->opt_mode == 0 || c->opt_mode == 1) ? 1u : 0u, c->d_work.as<unsigned>(),
                                      c->opt_lazy_hist ? 1u : 0u);
  ++st.launches;
  // (3: the pre-pass depends on the control init only, but is enqueued after
  // the seed kernels, so their CTAs are dispatched first: they lead to the
  // threshold, the longer chain)
  const bool cpre_late = cpre && c->opt_cpre == 3 && !tau0;
  if (cpre_late) {
    APEX_CU(cudaEventRecord(c->fork2_ev, s));
    cpre_forked = true;
  } else if (cpre && c->opt_cpre != 2) {
    APEX_TRY(launch_cpre());
  }
  // K2 pack of the streamed objective column
  if (admit && !(B.plan_rows && span < (uint64_t)c->opt_chunk_min)) {
    // (the sorted-column kernel reads the table's sorted lists, not a packed column)
    int64_t max_last = 1;
    for (const auto& R : c->rx) max_last = std::max<int64_t>(max_last, R.size[R.c - 1]);
    const unsigned gx = (unsigned)std::min<int64_t>((max_last + 255) / 256, 64);
    pack_obj_kernel<<<dim3(gx, (unsigned)c->rx.size(), nq), 256, 0, s>>>(dq, c->d_rx.as<DevReaction>(),
                                                                        c->d_values.as<float>(), c->n_pairs);
    ++st.launches;
  }
  APEX_CU(stage_mark(c, 1, s));
  // seed threshold from exact samples (uniform samples on the main stream,
  // the corner on the side stream: independent, they overlap)
  uint64_t S_used = 0;
  if (!tau0) {
    const bool corner = c->opt_corner && c->corners_ok;
    if (corner) {
      APEX_CU(cudaEventRecord(c->fork_ev, s));
      APEX_CU(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
    }
    uint64_t S = c->opt_samples > 0 ? (uint64_t)c->opt_samples
                                     : (uint64_t)std::min<int64_t>(1 << 15, std::max<int64_t>(1 << 11, 2 * B.k_max));
    S = std::min<uint64_t>(S, std::max<uint64_t>(span / 32, std::min<uint64_t>(span, 4096)));
    S_used = S;
    if (S > 0) {
      SampleLaunch P;
      P.queries = dq;
      P.rx = c->d_rx.as<DevReaction>();
      P.g_off = c->d_goff.as<unsigned long long>();
      P.n_rx = (int)c->rx.size();
      P.values = c->d_values.as<float>();
      P.p16 = (c->packed16_ok && c->opt_packed16) ? c->d_packed16.as<float>() : nullptr;
      P.n_pairs = c->n_pairs;
      P.start = start;
      P.end = end;
      P.samples = S;
      // (sample x query) threads: about two waves of the whole GPU
      const uint64_t want = std::max<uint64_t>(1, (uint64_t)c->sm_count * 16 / (uint64_t)nq);
      const unsigned blocks = (unsigned)std::min<uint64_t>((S + 255) / 256, want);
      sample_kernel<<<dim3(blocks, (unsigned)nq), 256, 0, s>>>(P, nq);
      ++st.launches;
    }
    if (corner) {
      CornerLaunch CL;
      CL.queries = dq;
      CL.rx = c->d_rx.as<DevReaction>();
      CL.values = c->d_values.as<float>();
      CL.p16 = (c->packed16_ok && c->opt_packed16) ? c->d_packed16.as<float>() : nullptr;
      CL.n_pairs = c->n_pairs;
      CL.lists = c->d_lists.as<int32_t>();
      CL.slot_off = c->d_slot_off.as<int32_t>();
      CL.m = c->d_m.as<int32_t>();
      CL.coff = c->d_coff.as<unsigned long long>();
      CL.n_rx = (int)c->rx.size();
      CL.slots = c->corner_slots;
      CL.start = start;
      CL.end = end;
      // corner budget per reaction: enough corner products for ~16k feasible
      // seeds across the reactions, within the precomputed list lengths
      const int64_t nrx = std::max<int64_t>(1, (int64_t)c->rx.size());
      // (and at most kCornerTotal corner products per pass: a batch of many
      // queries gains little from more, C2 seed 39 -> 33 us; a single large-k
      // query keeps its budget, C4's tau needs it)
      CL.budget = (int)std::max<int64_t>(
          256, std::min<int64_t>({4096, c->opt_corner_mult * B.k_max / nrx, kCornerTotal / (nrx * std::max(nq, 1))}));
      const int64_t per_rx = (int64_t)c->rx.size() * nq;
      const unsigned split = (unsigned)std::max<int64_t>(1, std::min<int64_t>(8, (2 * (int64_t)c->sm_count + per_rx - 1) / std::max<int64_t>(per_rx, 1)));
      corner_kernel<<<dim3((unsigned)c->rx.size(), nq, split), 256, 0, c->side>>>(CL);
      ++st.launches;
      if (cpre_late) APEX_TRY(launch_cpre());
      if (c->opt_tau_side) {
        // the threshold kernel on the (high-priority) side stream after both
        // seeds: its few CTAs are dispatched ahead of the pre-pass's
        APEX_CU(cudaEventRecord(c->fork_ev, s));
        APEX_CU(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
        tau_kernel<<<(nq + 7) / 8, 256, 0, c->side>>>(dq, nq, 0, autok, (unsigned long long)S_used,
                                                       (unsigned long long)span);
        ++st.launches;
        APEX_CU(cudaEventRecord(c->join_ev, c->side));
        APEX_CU(cudaStreamWaitEvent(s, c->join_ev, 0));
      } else {
        APEX_CU(cudaEventRecord(c->join_ev, c->side));
        APEX_CU(cudaStreamWaitEvent(s, c->join_ev, 0));
        tau_kernel<<<(nq + 7) / 8, 256, 0, s>>>(dq, nq, 0, autok, (unsigned long long)S_used, (unsigned long long)span);
        ++st.launches;
      }
    } else {
      if (cpre_late) APEX_TRY(launch_cpre());
      tau_kernel<<<(nq + 7) / 8, 256, 0, s>>>(dq, nq, 0, autok, (unsigned long long)S_used, (unsigned long long)span);
      ++st.launches;
    }
  }
  // K2 pack of the full-predicate columns (queries that use that kernel)
  if (full && plan->pair_hi > plan->pair_lo) {
    const int64_t n = (plan->pair_hi - plan->pair_lo) * B.ntp;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8 / nq));
    pack_kernel<<<dim3(blocks, nq), 256, 0, s>>>(dq, c->d_values.as<float>(), c->n_pairs, plan->pair_lo, plan->pair_hi);
    ++st.launches;
  }
  APEX_CU(stage_mark(c, 2, s));
  if (cpre) APEX_CU(cudaStreamWaitEvent(s, c->join2_ev, 0));
  // K3 enumeration: chunks x test classes
  const int cb = (int)c->opt_cb;
  const size_t n_tiles = plan->tiles.size();
  std::vector<size_t> bounds;  // chunk ends in tile indices
  if (span >= (uint64_t)c->opt_chunk_min && c->opt_chunk_div > 1 && n_tiles > 1) {
    const uint64_t first = span / (uint64_t)c->opt_chunk_div;
    size_t i1 = (size_t)(std::lower_bound(plan->prefix.begin(), plan->prefix.end(), first) - plan->prefix.begin());
    i1 = std::min(std::max<size_t>(i1, 1), n_tiles);
    bounds.push_back(i1);
  }
  bounds.push_back(n_tiles);
  size_t tb = 0;
  st.scan_kernel_ms = 0;
  int wi = 0;  // flattened-work counter index (one per scan launch)
  // (the flattened-work counters d_work were zeroed by init_ctl_kernel)
  for (size_t ci = 0; ci < bounds.size(); ++ci) {
    const size_t te = bounds[ci];
    if (te > tb) {
      ScanLaunch L{};
      L.tiles = plan->d_tiles.as<Tile>();
      L.tile_begin = (unsigned)tb;
      L.tile_end = (unsigned)te;
      L.rx = c->d_rx.as<DevReaction>();
      L.values = c->d_values.as<float>();
      L.n_pairs = c->n_pairs;
      L.queries = dq;
      L.cb = cb;
      L.nq = nq;
      L.work = c->d_work.as<unsigned>();
      L.chunk = (int)c->opt_chunk;
      if (ci == 0) APEX_CU(stage_mark(c, 6, s));
      if (admit && B.plan_rows && bounds.size() == 1) {
        // sorted-column admission: whole-row tiles, one launch per 64 queries
        const Plan* pr_ = B.plan_rows;
        const size_t smem = (size_t)kScanWarps * kMaxTests * 32 * sizeof(float) + (size_t)kScanWarps * 32 * sizeof(int4) +
                            (APEX_CAND_STAGE ? (size_t)kScanWarps * kCandStage * sizeof(Entry) : 0);
        const bool p16 = c->packed16_ok && c->opt_packed16;
        const bool rowp = c->rowp_ok && c->opt_rowp;
        ScanFn fn = p16 ? (rowp ? reinterpret_cast<ScanFn>(scan_sorted_kernel<true, true>)
                                : reinterpret_cast<ScanFn>(scan_sorted_kernel<true, false>))
                        : (rowp ? reinterpret_cast<ScanFn>(scan_sorted_kernel<false, true>)
                                : reinterpret_cast<ScanFn>(scan_sorted_kernel<false, false>));
        int occ = 0;
        APEX_TRY(scan_occupancy(c, fn, smem, &occ));
        SortedLaunch SL;
        SL.packed16 = p16 ? c->d_packed16.as<float>() : nullptr;
        SL.sx = c->d_sorted_x.as<float>();
        SL.scol = c->d_sorted_col.as<uint32_t>();
        SL.pcols = std::max<int64_t>(c->pcols, 4);
        SL.quant = c->d_quant.as<float>();
        SL.n_rx = (int)c->rx.size();
        SL.cthr = c->d_cthr.as<float>();
        SL.cbest = c->d_cbest.as<int4>();
        SL.rows_pad = (int64_t)pr_->tiles.size() * 32;
        SL.rowp = rowp ? c->d_rowp.as<double>() : nullptr;
        SL.rows_total = c->rows_total;
        for (int q0 = 0; q0 < nq; q0 += 64) {
          const int nql = std::min(64, nq - q0);
          ScanLaunch La = L;
          La.tiles = pr_->d_tiles.as<Tile>();
          La.tile_begin = 0;
          La.tile_end = (unsigned)pr_->tiles.size();
          La.queries = dq + q0;
          La.nq = nql; La.nq_magic = nq_magic((La.tile_end - La.tile_begin), nql);
          const int64_t items = (int64_t)pr_->tiles.size() * nql;
          const int64_t blocks = std::max<int64_t>(
              1, std::min<int64_t>((items + kScanWarps - 1) / kScanWarps, (int64_t)c->sm_count * occ));
          const int slot = wi++ % 64;
          La.work = c->d_work.as<unsigned>() + slot;
          if (q0 == 0 && c->opt_work_ctrs > 1) {  // the first launch: several counters (own lines)
            La.work = c->d_work.as<unsigned>() + 64;
            La.n_ctr = (int)std::min<int64_t>(c->opt_work_ctrs, kWorkCtrs);
          }
          reinterpret_cast<void (*)(ScanLaunch, SortedLaunch)>(fn)<<<(unsigned)blocks, kScanWarps * 32, smem, s>>>(La, SL);
          APEX_CU(cudaGetLastError());
          ++st.launches;
          ++st.scans;
        }
      } else if (admit) {
        const int cba = (int)c->opt_cb_admit;
        const bool tr = c->trace_cap > 0;
        ScanFn fn = B.rl == 2 ? (tr ? scan_admit_kernel<2, true> : scan_admit_kernel<2, false>)
                              : (tr ? scan_admit_kernel<1, true> : scan_admit_kernel<1, false>);
        const size_t smem = (size_t)kScanWarps * 2 * cba * sizeof(float) +
                            (size_t)kScanWarps * 16 * kMaxTests * sizeof(float) +
                            (size_t)kScanWarps * 512 * B.rl * sizeof(unsigned short) +
                            (size_t)kScanWarps * 2 * sizeof(uint64_t) + kBlockDq * sizeof(DenseItem) + 16 +
                            (size_t)kScanWarps * B.rl * kMaxTests * 32 * sizeof(float);
        int occ = 0;
        APEX_TRY(scan_occupancy(c, fn, smem, &occ));
        for (int q0 = 0; q0 < nq; q0 += 64) {
          const int nql = std::min(64, nq - q0);
          ScanLaunch La = L;
          La.cb = cba;
          La.vote64 = (int)c->opt_vote64;
          La.dense_min = c->opt_dense > 0 ? (int)c->opt_dense : 1 << 20;
          if (c->trace_cap > 0) {
            La.trace = c->d_trace.as<unsigned long long>();
            La.trace_cap = (unsigned)c->trace_cap;
            c->trace_n = std::min<int64_t>(c->trace_cap, (int64_t)(La.tile_end - La.tile_begin) * nql);
          }
          const int64_t items = (int64_t)(La.tile_end - La.tile_begin) * nql;
          const int64_t blocks = std::max<int64_t>(
              1, std::min<int64_t>((items + kScanWarps - 1) / kScanWarps, (int64_t)c->sm_count * occ));
          La.queries = dq + q0;
          La.nq = nql;
          const int slot = wi++ % 64;
          La.work = c->d_work.as<unsigned>() + slot;
          fn<<<(unsigned)blocks, kScanWarps * 32, smem, s>>>(La);
          APEX_CU(cudaGetLastError());
          ++st.launches;
          ++st.scans;
        }
      }
      // full-predicate launches per test class alternate between the main and
      // the side stream so consecutive classes overlap (disjoint queries)
      int n_full_launch = 0;
      for (size_t k = 0; full && k + 1 < B.cls_begin.size(); ++k) {
        ScanFn fn = pick_scan(B.cls_nt[k], B.rl, c->opt_mode == 1 ? 1 : 0);
        if (!fn) return set_err(APEX_ELIMIT, "no enumeration kernel for this test count");
        const size_t smem = scan_smem(B.cls_nt[k], cb);
        int occ = 0;
        APEX_TRY(scan_occupancy(c, fn, smem, &occ));
        for (int q0 = B.cls_begin[k]; q0 < B.cls_begin[k + 1]; q0 += 64) {
          const int nql = std::min(64, B.cls_begin[k + 1] - q0);
          const int64_t items = (int64_t)(te - tb) * nql;
          const int64_t blocks = std::max<int64_t>(
              1, std::min<int64_t>((items + kScanWarps - 1) / kScanWarps, (int64_t)c->sm_count * occ));
          ScanLaunch Lc = L;
          Lc.queries = dq + q0;
          Lc.nq = nql; Lc.nq_magic = nq_magic((Lc.tile_end - Lc.tile_begin), nql);
          Lc.work = c->d_work.as<unsigned>() + (wi++ % 64);
          cudaStream_t ls = s;
          if (n_full_launch % 2 == 1) {
            if (n_full_launch == 1) {
              APEX_CU(cudaEventRecord(c->fork_ev, s));
              APEX_CU(cudaStreamWaitEvent(c->side, c->fork_ev, 0));
            }
            ls = c->side;
          }
          ++n_full_launch;
          fn<<<(unsigned)blocks, kScanWarps * 32, smem, ls>>>(Lc);
          APEX_CU(cudaGetLastError());
          ++st.launches;
          ++st.scans;
        }
      }
      if (n_full_launch > 1) {
        APEX_CU(cudaEventRecord(c->join_ev, c->side));
        APEX_CU(cudaStreamWaitEvent(s, c->join_ev, 0));
      }
      if (ci + 1 < bounds.size()) {
        tau_kernel<<<(nq + 7) / 8, 256, 0, s>>>(dq, nq, 1);  // raise tau from the candidates so far
        ++st.launches;
      }
    }
    tb = te;
  }
  APEX_CU(stage_mark(c, 7, s));
  APEX_CU(stage_mark(c, 3, s));
  // final bound (inside the small-set finalize), exact select
  APEX_TRY(enqueue_select(c, dq, nq, B.k_max, B.finalize, st, s, true, true, B.small_only));
  APEX_CU(cudaGetLastError());
  APEX_CU(stage_mark(c, 5, s));
  // control-block headers (read by check_batch) gathered at the tail of the
  // result block by a kernel, then ONE copy: rows + headers when the rows go
  // to the host in this pass (synchronous call; an overflow re-run copies
  // again), else the headers alone
  ctl_export_kernel<<<nq, 64, 0, s>>>(dq, c->d_out.as<unsigned char>() + c->out_off[nq]);
  ++st.launches;
  const size_t hdr = (size_t)nq * kCtlHdr;
  if (B.copy_out) {
    APEX_CU(cudaMemcpyAsync(c->h_out.p, c->d_out.p, c->out_off[nq] + hdr, cudaMemcpyDeviceToHost, s));
  } else {
    APEX_CU(cudaMemcpyAsync(c->h_out.as<unsigned char>() + c->out_off[nq], c->d_out.as<unsigned char>() + c->out_off[nq],
                            hdr, cudaMemcpyDeviceToHost, s));
  }
  st.d2h_bytes += (int64_t)hdr;
  B.pending = true;
  return APEX_OK;
}

// Wait for the pass on the context stream.  opt_spin_us > 0: poll an event
// recorded at the end of the pass for up to that long before a blocking
// synchronize — the waiting thread resumes within a poll of the GPU finishing
// instead of after the driver's wake-up of a blocked or yielding thread.
int wait_stream(apex_ctx* c) {
  if (c->opt_spin_us > 0 && c->done_ev) {
    APEX_CU(cudaEventRecord(c->done_ev, c->stream));
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
      const cudaError_t e = cudaEventQuery(c->done_ev);
      if (e == cudaSuccess) return APEX_OK;
      if (e != cudaErrorNotReady) APEX_CU(e);
      if (std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() > c->opt_spin_us)
        break;
    }
  }
  APEX_CU(cudaStreamSynchronize(c->stream));
  return APEX_OK;
}

// Sync, detect candidate-buffer overflow, re-run exactly if needed.  A re-run
// is preset from the overflowed run's control block (finalize_small_kernel
// nx_*): the admission threshold at the k-th best bin and a 16-bit narrower
// candidate histogram there, or — when that bin is one exact key K (massive
// exact ties) — the composite bound (key > K, or key == K and g below a limit
// narrowed 16 bits per run).  The buffers never grow; each step shrinks the
// admitted set, so the protocol converges (<= 4 key steps + 4 g steps for
// 64-bit keys and indices).
int check_batch(apex_ctx* c) {
  Batch& B = c->batch;
  if (!B.pending) return set_err(APEX_ESTATE, "no query batch in flight");
  const int nq = B.nq;
  std::vector<RunPreset> pre(nq);
  std::vector<int> pre_full(nq, 0);          // queries moved to the full predicate (bail-out)
  for (int attempt = 0;; ++attempt) {
    APEX_TRY(wait_stream(c));
    {  // the control headers from the tail of the result block
      const unsigned char* src = c->h_out.as<unsigned char>() + c->out_off[nq];
      for (int i = 0; i < nq; ++i)
        std::memcpy(c->h_ctl.as<unsigned char>() + (size_t)i * sizeof(QCtl), src + (size_t)i * kCtlHdr,
                    offsetof(QCtl, hist));
    }
    if (B.small_only) {
      // the large path was skipped on the strength of this signature's last
      // run: if a query did not fit the small finalize now, run it again whole
      bool all_small = true;
      for (int i = 0; i < nq; ++i) all_small = all_small && c->h_ctl.as<QCtl>()[i].small_done;
      if (!all_small) {
        B.small_only = false;
        c->small_keys.erase(std::remove(c->small_keys.begin(), c->small_keys.end(), B.key0), c->small_keys.end());
        ++B.st.retries;
        APEX_TRY(enqueue_batch(c, nullptr));
        continue;
      }
    }
    bool overflow = false;
    for (int i = 0; i < nq; ++i) {
      const QCtl& C = c->h_ctl.as<QCtl>()[i];
      const apex_query_spec& q = B.qs[i];
      RunPreset& P = pre[i];
      std::memset(&P, 0, sizeof(P));
      P.tie_glimit = ~0ull;
      P.tie_gshift = 48;
      if (C.bail) {
        // the sorted-column kernel gave the query up (pair budget): re-run it
        // with the full predicate from the admission key it had reached (a
        // valid lower bound on its k-th best key)
        overflow = true;
        pre_full[i] = 1;
        P.full = 1;
        P.tau = C.bail_tau;
        P.base = C.bail_tau;
        P.shift = C.hist_shift;
        continue;
      }
      P.full = pre_full[i] ? 1u : 0u;  // stays on the full predicate in any further re-run
      if (C.count > c->uploaded[i].cap) {
        overflow = true;
        P.tau = C.nx_tau;
        if (C.nx_tie) {
          P.tie_on = 1;
          P.tie_key = C.nx_tau;
          P.shift = 48;
          if (C.nx_tie_enter) {
            const uint64_t span = q.end - q.start;
            unsigned gs = 0;
            while (gs < 63 && (span >> gs) >= 65535ull) ++gs;
            P.tie_gbase = q.start;
            P.tie_glimit = q.end;
            P.tie_gshift = gs;
          } else {
            P.tie_gbase = C.nx_gbase;
            P.tie_glimit = C.nx_glimit;
            P.tie_gshift = C.nx_gshift;
          }
        } else {
          P.base = C.nx_base;
          P.shift = C.nx_shift;
        }
      } else {
        // a query that fit re-runs with its valid final bound (same result)
        P.tau = std::max<unsigned long long>(C.bound_key, C.tau_key);
        P.base = P.tau;
        P.shift = C.hist_shift;
        if (C.tie_on) {
          P.tie_on = 1;
          P.tie_key = C.tie_key;
          P.tie_gbase = C.tie_gbase;
          P.tie_glimit = C.tie_glimit;
          P.tie_gshift = C.tie_gshift;
          P.tau = C.tie_key;
        }
      }
    }
    if (!overflow) break;
    if (attempt >= 12) {
      B.pending = false;
      return set_err(APEX_ELIMIT, "candidate buffer overflow did not converge");
    }
    ++B.st.retries;
    if (std::find(pre_full.begin(), pre_full.end(), 1) != pre_full.end()) B.no_full = false;  // full launches needed
    APEX_TRY(enqueue_batch(c, pre.data()));
  }
  B.pending = false;
  if (!B.small_only) {
    bool all_small = true;
    for (int i = 0; i < nq; ++i) all_small = all_small && c->h_ctl.as<QCtl>()[i].small_done;
    if (all_small && std::find(c->small_keys.begin(), c->small_keys.end(), B.key0) == c->small_keys.end()) {
      if (c->small_keys.size() >= 64) c->small_keys.erase(c->small_keys.begin());
      c->small_keys.push_back(B.key0);
    }
  }
  if (!B.no_full && c->opt_mode == 3 && B.plan_rows) {
    bool any_full = false;
    for (int i = 0; i < nq; ++i) any_full = any_full || c->h_ctl.as<QCtl>()[i].use_full;
    if (!any_full && std::find(c->nofull_keys.begin(), c->nofull_keys.end(), B.key0) == c->nofull_keys.end()) {
      if (c->nofull_keys.size() >= 64) c->nofull_keys.erase(c->nofull_keys.begin());
      c->nofull_keys.push_back(B.key0);
    }
  }
  // (stage times are informational: never fail the query on them)
  for (int e = 0; e < 5; ++e)
    if (!c->opt_stages || cudaEventElapsedTime(&B.st.ms[e], c->ev[e], c->ev[e + 1]) != cudaSuccess) B.st.ms[e] = 0.f;
  if (!c->opt_stages || cudaEventElapsedTime(&B.st.scan_kernel_ms, c->ev[6], c->ev[7]) != cudaSuccess)
    B.st.scan_kernel_ms = 0.f;
  cudaGetLastError();
  return APEX_OK;
}

// Signature of the prepared batch: query contents, options and the
// allocation generation (device / pinned pointers baked into a graph).
uint64_t batch_key(const apex_ctx* c) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  const Batch& B = c->batch;
  mix(&B.nq, sizeof(B.nq));
  mix(&B.finalize, sizeof(B.finalize));
  mix(&B.copy_out, sizeof(B.copy_out));
  mix(&B.no_full, sizeof(B.no_full));
  mix(&B.small_only, sizeof(B.small_only));
  for (int i = 0; i < B.nq; ++i) {
    const apex_query_spec& q = B.qs[i];
    mix(&q.objective_task, sizeof(q.objective_task));
    mix(&q.maximize, sizeof(q.maximize));
    mix(&q.n_constraints, sizeof(q.n_constraints));
    mix(&q.k, sizeof(q.k));
    mix(&q.start, sizeof(q.start));
    mix(&q.end, sizeof(q.end));
    mix(B.cons[i].data(), B.cons[i].size() * sizeof(apex_constraint));
    mix(&B.perm[i], sizeof(int));
  }
  const void* plan = B.plan;
  mix(&plan, sizeof(plan));
  const void* plan_rows = B.plan_rows;
  mix(&plan_rows, sizeof(plan_rows));
  mix(&c->opt_gen, sizeof(c->opt_gen));
  const uint64_t gen = g_alloc_gen.load();
  mix(&gen, sizeof(gen));
  return h;
}

// Enqueue the prepared batch: replay the captured CUDA graph when the batch
// signature repeats, otherwise capture it (or launch directly if capture is
// unavailable).  One graph launch replaces ~30 kernel/memset/memcpy launches.
int launch_batch(apex_ctx* c) {
  // full-predicate launches are skipped for a signature whose previous run
  // sent no query there (the device then never picks that kernel; every query
  // stays exact in the sorted-column kernel either way)
  Batch& Bq = c->batch;
  Bq.no_full = false;
  Bq.key0 = batch_key(c);
  Bq.no_full = c->opt_mode == 3 && Bq.plan_rows &&
               std::find(c->nofull_keys.begin(), c->nofull_keys.end(), Bq.key0) != c->nofull_keys.end();
  Bq.small_only = std::find(c->small_keys.begin(), c->small_keys.end(), Bq.key0) != c->small_keys.end();
  if (!c->opt_graph || c->graph_broken) return enqueue_batch(c, nullptr);
  const uint64_t key = batch_key(c);
  if (c->gexec && key == c->gkey) {
    APEX_CU(cudaGraphLaunch(c->gexec, c->stream));
    c->batch.pending = true;
    c->batch.st = c->graph_stats;  // launch counts / bytes as captured
    return APEX_OK;
  }
  // capture (and pay the instantiation) only for a batch signature seen
  // before: a stream of distinct one-off queries launches directly
  auto seen = std::find(c->seen_keys.begin(), c->seen_keys.end(), key);
  if (seen == c->seen_keys.end()) {
    if (c->seen_keys.size() >= 32) c->seen_keys.erase(c->seen_keys.begin());
    c->seen_keys.push_back(key);
    return enqueue_batch(c, nullptr);
  }
  if (c->gexec) {
    cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
  }
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    c->graph_broken = true;
    return enqueue_batch(c, nullptr);
  }
  const int rc = enqueue_batch(c, nullptr);
  const cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
  cudaGraphExec_t exec = nullptr;
  // node priorities (the streams' priorities, recorded at capture) are honoured
  // only with UseNodePriority: the constraint pre-pass runs at the lowest, so
  // the short seed / threshold kernels get SM slots as soon as any frees
  const unsigned long long gflags = c->opt_graph_prio ? cudaGraphInstantiateFlagUseNodePriority : 0ull;
  const cudaError_t ei = (rc == APEX_OK && ec == cudaSuccess) ? cudaGraphInstantiateWithFlags(&exec, graph, gflags) : ec;
  if (graph) cudaGraphDestroy(graph);
  if (rc != APEX_OK || ec != cudaSuccess || ei != cudaSuccess) {
    cudaGetLastError();
    if (exec) cudaGraphExecDestroy(exec);
    c->graph_broken = true;  // fall back to direct launches for this context
    return enqueue_batch(c, nullptr);
  }
  c->gexec = exec;
  c->gkey = key;
  c->graph_stats = c->batch.st;
  APEX_CU(cudaGraphLaunch(c->gexec, c->stream));
  return APEX_OK;
}

int validate_queries(apex_ctx* c, const apex_query_spec* qs, int nq) {
  if (nq < 0) return set_err(APEX_EINVAL, "negative query count");
  if (nq > 0 && !qs) return set_err(APEX_EINVAL, "null queries");
  for (int i = 0; i < nq; ++i) {
    const apex_query_spec& q = qs[i];
    if (q.objective_task < 0 || q.objective_task >= c->n_tasks)
      return set_err(APEX_ETASK, "unknown task index " + std::to_string(q.objective_task));
    if (q.k < 0) return set_err(APEX_EINVAL, "k must be >= 0");
    if (q.k > (int64_t)1 << 26) return set_err(APEX_ELIMIT, "k exceeds the compiled limit (2^26)");
    if (q.n_constraints < 0 || (q.n_constraints > 0 && !q.constraints))
      return set_err(APEX_EINVAL, "bad constraint list");
    if (!(q.start <= q.end && q.end <= c->total))
      return set_err(APEX_ERANGE, "index range [" + std::to_string(q.start) + ", " + std::to_string(q.end) + ") invalid");
  }
  return APEX_OK;
}

void fill_stats(apex_stats* stats, const RunStats& st, float d2h, float total, int64_t cand) {
  if (!stats) return;
  stats->pack_ms = st.ms[0];
  stats->seed_ms = st.ms[1];
  stats->scan_ms = st.ms[2];
  stats->select_ms = st.ms[3];
  stats->finalize_ms = st.ms[4];
  stats->d2h_ms = d2h;
  stats->total_ms = total;
  stats->scan_kernel_ms = st.scan_kernel_ms;
  stats->candidates = cand;
  stats->scan_launches = st.scans;
  stats->kernel_launches = st.launches;
  stats->retries = st.retries;
  stats->h2d_bytes = st.h2d_bytes;
  stats->d2h_bytes = st.d2h_bytes;
}

// Copy materialized rows of slot i to the caller's result.
int copy_results(apex_ctx* c, const apex_query_spec* qs, int nq, apex_result* res_caller, const int* perm,
                 bool copied = false) {
  std::vector<apex_result> res_sorted(nq);
  for (int i = 0; i < nq; ++i) res_sorted[i] = res_caller[perm ? perm[i] : i];
  apex_result* res = res_sorted.data();
  // one D2H of every query's rows (contiguous in d_out), then host copies of
  // the retained rows into the caller's arrays
  const std::vector<size_t>& offs = c->out_off;
  const size_t total = offs[nq];
  if (!copied) {
    APEX_TRY(c->h_out.ensure(total));
    APEX_CU(cudaMemcpyAsync(c->h_out.p, c->d_out.p, total, cudaMemcpyDeviceToHost, c->stream));
    APEX_CU(cudaStreamSynchronize(c->stream));
  }
  for (int i = 0; i < nq; ++i) {
    const apex_query_spec& q = qs[i];
    apex_result& r = res[i];
    const uint64_t span = q.end - q.start;
    const int64_t kk = std::max<int64_t>(q.k, 1);
    const int m = q.n_constraints;
    int64_t n = 0;
    if (q.k > 0 && span > 0) {
      const QCtl& C = c->h_ctl.as<QCtl>()[i];
      n = (int64_t)C.sel_count;
      r.candidates = (int64_t)C.count;
      r.admitted = (int64_t)C.admitted;
      r.full_predicate = (int32_t)C.use_full;
    } else {
      r.candidates = r.admitted = 0;
      r.full_predicate = 0;
    }
    r.n = n;
    r.scanned = span;
    r.discarded = (int64_t)std::min<uint64_t>((uint64_t)q.k, span) - n;
    unsigned char* o = c->h_out.as<unsigned char>() + offs[i];
    if (!r.global_index && !r.objective && !r.constraint_values && !r.reaction && !r.digits) {
      // view mode: point at the rows in the context's pinned host block
      // (valid until the next call on this context)
      r.global_index = reinterpret_cast<uint64_t*>(o);
      r.objective = reinterpret_cast<double*>(o + 8 * kk);
      r.constraint_values = reinterpret_cast<double*>(o + 16 * kk);
      r.reaction = reinterpret_cast<int32_t*>(o + (16 + 8 * (size_t)m) * kk);
      r.digits = reinterpret_cast<int32_t*>(o + (20 + 8 * (size_t)m) * kk);
    } else if (n > 0) {
      if (r.global_index) std::memcpy(r.global_index, o, 8 * n);
      if (r.objective) std::memcpy(r.objective, o + 8 * kk, 8 * n);
      if (r.constraint_values && m) std::memcpy(r.constraint_values, o + 16 * kk, 8 * (size_t)m * n);
      if (r.reaction) std::memcpy(r.reaction, o + (16 + 8 * (size_t)m) * kk, 4 * n);
      if (r.digits) std::memcpy(r.digits, o + (20 + 8 * (size_t)m) * kk, 4 * (size_t)kMaxRg * n);
    }
  }
  for (int i = 0; i < nq; ++i) res_caller[perm ? perm[i] : i] = res_sorted[i];
  return APEX_OK;
}

// Multi-GPU local step, enqueue half: the exact local pipeline of a batch
// (queries share range and, for the export layout, a stride >= every k) and
// the export of each query's selected entries to out + slot * stride (padded),
// all on the context stream with no host sync.
int local_enqueue(apex_ctx* c, const apex_query_spec* qs, int nq, Entry* out, unsigned long long stride) {
  APEX_TRY(prepare_batch(c, qs, nq, false));
  APEX_TRY(launch_batch(c));
  c->batch.export_out = out;
  c->batch.export_stride = stride;
  const ScanQuery* dq = c->d_queries.as<ScanQuery>();
  const unsigned gx = (unsigned)std::min<unsigned long long>((stride + 255) / 256, 1024);
  export_kernel<<<dim3(gx, nq), 256, 0, c->stream>>>(dq, out, stride);
  APEX_CU(cudaGetLastError());
  ++c->batch.st.launches;
  return APEX_OK;
}

// Multi-GPU local step, validate half: sync, and if a candidate buffer
// overflowed re-run exactly (check_batch) and export again; *rerun = 1 then
// (the entries a peer read before are stale).  counts (optional, caller's
// query order) = entries selected per query.
int local_finish(apex_ctx* c, int64_t* counts, int* rerun) {
  Batch& B = c->batch;
  if (!B.pending) return set_err(APEX_ESTATE, "no local step in flight");
  const int64_t retries0 = B.st.retries;
  APEX_TRY(check_batch(c));
  const bool again = B.st.retries != retries0;
  if (again) {
    const unsigned gx = (unsigned)std::min<unsigned long long>((B.export_stride + 255) / 256, 1024);
    export_kernel<<<dim3(gx, B.nq), 256, 0, c->stream>>>(c->d_queries.as<ScanQuery>(), B.export_out,
                                                         B.export_stride);
    APEX_CU(cudaGetLastError());
    ++B.st.launches;
    APEX_CU(cudaStreamSynchronize(c->stream));
  }
  if (rerun) *rerun = again ? 1 : 0;
  if (counts)
    for (int i = 0; i < B.nq; ++i) counts[B.perm[i]] = (int64_t)c->h_ctl.as<QCtl>()[i].sel_count;
  return APEX_OK;
}

// Swaps the context's query workspace with its merge workspace for a scope.
struct MergeScope {
  apex_ctx* c;
  explicit MergeScope(apex_ctx* c_) : c(c_) { swap(); }
  ~MergeScope() { swap(); }
  void swap() {
    auto& w = c->mws;
    std::swap(c->slots, w.slots);
    std::swap(c->d_hists, w.d_hists);
    std::swap(c->d_ctls, w.d_ctls);
    std::swap(c->d_queries, w.d_queries);
    std::swap(c->d_out, w.d_out);
    std::swap(c->h_queries, w.h_queries);
    std::swap(c->h_ctl, w.h_ctl);
    std::swap(c->h_out, w.h_out);
    std::swap(c->out_off, w.out_off);
    std::swap(c->uploaded, w.uploaded);
  }
};

// Exact merge of gathered local entries (one device pass for a batch): the
// entries of query q from source r are entries[(r * nq + q) * stride + i]
// (one contiguous all-gathered buffer), or srcs[r][q * stride + i] when srcs
// (a device array of n_src device pointers, possibly peers) is given.
// Selects, orders and materializes every query's global top-k into res.
int merge_impl(apex_ctx* c, const apex_query_spec* qs, int nq, const Entry* entries, const Entry* const* srcs,
               int n_src, int64_t stride, uint64_t total_scanned, apex_result* res, apex_stats* stats) {
  for (int i = 0; i < nq; ++i) {
    const apex_query_spec& q = qs[i];
    if (q.objective_task < 0 || q.objective_task >= c->n_tasks) return set_err(APEX_ETASK, "unknown task index");
    if (q.n_constraints > kMaxCons) return set_err(APEX_ELIMIT, "more than 32 constraints in a query");
    if (q.k < 0) return set_err(APEX_EINVAL, "k must be >= 0");
    for (int m = 0; m < q.n_constraints; ++m)
      if (q.constraints[m].task < 0 || q.constraints[m].task >= c->n_tasks) return set_err(APEX_ETASK, "unknown task index");
  }
  if (stats) std::memset(stats, 0, sizeof(*stats));
  MergeScope scope(c);  // never touches the buffers of a local step in flight
  const int64_t n_in = (int64_t)n_src * stride;
  bool any = false;
  for (int i = 0; i < nq; ++i) {
    res[i].scanned = total_scanned;
    if (qs[i].k == 0 || n_in == 0) {
      res[i].n = 0;
      res[i].candidates = res[i].admitted = 0;
      res[i].full_predicate = 0;
      res[i].discarded = (int64_t)std::min<uint64_t>((uint64_t)qs[i].k, total_scanned);
    } else {
      any = true;
    }
  }
  if (!any) return APEX_OK;
  // one slot per query: candidate buffer = every gathered entry of the query
  if ((int)c->slots.size() < nq) c->slots.resize(nq);
  int64_t k_max = 1;
  for (int i = 0; i < nq; ++i) {
    Slot& S = c->slots[i];
    const int64_t k = std::max<int64_t>(qs[i].k, 1);
    k_max = std::max(k_max, k);
    APEX_TRY(S.buf.ensure((size_t)std::max<int64_t>(n_in, 1024) * sizeof(Entry)));
    APEX_TRY(S.sel.ensure((size_t)k * sizeof(Entry)));
    APEX_TRY(S.sorted.ensure((size_t)k * sizeof(Entry)));
  }
  APEX_TRY(c->d_hists.ensure((size_t)nq * kHistWords * sizeof(unsigned)));
  APEX_TRY(c->d_ctls.ensure((size_t)nq * sizeof(QCtl)));
  c->out_off.assign(nq + 1, 0);
  for (int i = 0; i < nq; ++i)
    c->out_off[i + 1] = c->out_off[i] + (out_bytes(std::max<int64_t>(qs[i].k, 1), qs[i].n_constraints) + 15) / 16 * 16;
  APEX_TRY(c->d_out.ensure(c->out_off[nq]));
  const size_t qbytes = (size_t)nq * sizeof(ScanQuery);
  APEX_TRY(c->d_queries.ensure(qbytes));
  APEX_CU(cudaEventSynchronize(c->upload_ev));
  APEX_TRY(c->h_queries.ensure(qbytes));
  APEX_TRY(c->h_ctl.ensure((size_t)nq * sizeof(QCtl)));
  c->uploaded.clear();
  ScanQuery* hq = c->h_queries.as<ScanQuery>();
  for (int i = 0; i < nq; ++i) {
    const apex_query_spec& q = qs[i];
    Slot& S = c->slots[i];
    ScanQuery& Q = hq[i];
    std::memset(&Q, 0, sizeof(Q));
    const int64_t kk = std::max<int64_t>(q.k, 1);
    Q.buf = S.buf.as<Entry>();
    Q.sel = S.sel.as<Entry>();
    Q.sorted = S.sorted.as<Entry>();
    Q.hist = c->d_hists.as<unsigned>() + (size_t)i * kHistWords;
    Q.coarse = Q.hist + kHistBins;
    Q.seed_hist = Q.coarse + 256;
    Q.ctl = c->d_ctls.as<QCtl>() + i;
    Q.cap = S.buf.bytes / sizeof(Entry);
    Q.refresh_shift = 62;
    Q.k = std::max<int64_t>(q.k, 1);  // k == 0 queries are reported empty below
    Q.maximize = q.maximize ? 1 : 0;
    Q.obj_task = q.objective_task;
    Q.n_cons = q.n_constraints;
    for (int m = 0; m < q.n_constraints; ++m) Q.cons_task[m] = q.constraints[m].task;
    unsigned char* o = c->d_out.as<unsigned char>() + c->out_off[i];
    Q.out_g = reinterpret_cast<unsigned long long*>(o);
    Q.out_obj = reinterpret_cast<double*>(o + 8 * kk);
    Q.out_cons = reinterpret_cast<double*>(o + 16 * kk);
    Q.out_rx = reinterpret_cast<int32_t*>(o + (16 + 8 * (size_t)q.n_constraints) * kk);
    Q.out_dig = reinterpret_cast<int32_t*>(o + (20 + 8 * (size_t)q.n_constraints) * kk);
  }
  cudaStream_t s = c->stream;
  const ScanQuery* dq = c->d_queries.as<ScanQuery>();
  RunStats st;
  APEX_CU(cudaEventRecord(c->mev[0], s));
  APEX_CU(cudaMemcpyAsync(c->d_queries.p, c->h_queries.p, qbytes, cudaMemcpyHostToDevice, s));
  APEX_CU(cudaEventRecord(c->upload_ev, s));
  APEX_CU(cudaMemsetAsync(c->d_hists.p, 0, (size_t)nq * kHistWords * sizeof(unsigned), s));
  init_ctl_kernel<<<nq, 1024, 0, s>>>(dq, nullptr, 0u, nullptr, 0u);
  if (n_in > 0) {
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n_in + 255) / 256, 4 * c->sm_count / std::max(nq, 1) + 1));
    merge_load_kernel<<<dim3(gx, nq), 256, 0, s>>>(dq, entries, n_src, nq, (unsigned long long)stride, srcs);
  }
  st.launches = 2;
  // bound_key = 0 (init): every loaded entry is a candidate
  APEX_TRY(enqueue_select(c, dq, nq, k_max, true, st, s, false, false));
  APEX_CU(cudaGetLastError());
  APEX_CU(cudaMemcpy2DAsync(c->h_ctl.p, sizeof(QCtl), c->d_ctls.p, sizeof(QCtl), offsetof(QCtl, hist), nq,
                            cudaMemcpyDeviceToHost, s));
  APEX_CU(cudaEventRecord(c->mev[1], s));
  std::vector<apex_query_spec> qq(qs, qs + nq);
  for (auto& x : qq) {
    x.start = 0;
    x.end = total_scanned;
  }
  APEX_TRY(copy_results(c, qq.data(), nq, res, nullptr));
  for (int i = 0; i < nq; ++i)
    if (qs[i].k == 0 || n_in == 0) {
      res[i].n = 0;
      res[i].discarded = (int64_t)std::min<uint64_t>((uint64_t)qs[i].k, total_scanned);
    }
  if (stats) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->mev[0], c->mev[1]);
    stats->select_ms = ms;
    stats->total_ms = ms;
    stats->kernel_launches = st.launches;
    stats->d2h_bytes = (int64_t)c->out_off[nq] + (int64_t)nq * (int64_t)offsetof(QCtl, hist);
    stats->h2d_bytes = (int64_t)qbytes;
    for (int i = 0; i < nq; ++i) stats->stale_sources += c->h_ctl.as<QCtl>()[i].stale ? 1 : 0;
  }
  return APEX_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* apex_last_error(void) { return t_err.c_str(); }
const char* apex_version(void) { return "apex_b200 0.1 (sm_100a)"; }

// Load every kernel of the query, bind and precompute paths into the device
// context once (CUDA's lazy module loading would otherwise load each on its
// first launch — a first query of an unseen shape paid up to ~0.4 s, C5 sweep).
void preload_kernels() {
  const void* fns[] = {
      (const void*)init_ctl_kernel, (const void*)pack_kernel, (const void*)pack_obj_kernel,
      (const void*)cons_thr_kernel, (const void*)cons_best_kernel, (const void*)cons_fused_kernel,
      (const void*)sample_kernel,
      (const void*)corner_kernel, (const void*)tau_kernel, (const void*)scan_sorted_kernel<true, true>,
      (const void*)scan_sorted_kernel<true, false>, (const void*)scan_sorted_kernel<false, true>,
      (const void*)scan_sorted_kernel<false, false>, (const void*)scan_admit_kernel<1, false>,
      (const void*)scan_admit_kernel<2, false>, (const void*)finalize_bucket_kernel, (const void*)finalize_small_kernel,
      (const void*)select_kernel, (const void*)sort_chunks_kernel, (const void*)merge_rank_kernel,
      (const void*)materialize_kernel, (const void*)export_kernel, (const void*)merge_load_kernel,
      (const void*)bind_sort_kernel, (const void*)bind_emit_kernel, (const void*)bind_pack16_kernel,
      (const void*)bind_rowp_kernel, (const void*)precompute_bulk_kernel<11, 64>,
      (const void*)precompute_rows_kernel<11, 64>, (const void*)precompute_rows_kernel<0, 0>,
      (const void*)precompute_kernel};
  cudaFuncAttributes a;
  for (const void* f : fns) cudaFuncGetAttributes(&a, f);
  for (int nt : {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 14, 16, 20, 24})
    if (ScanFn f = pick_scan(nt, 1, 0)) cudaFuncGetAttributes(&a, (const void*)f);
  cudaGetLastError();
}

int apex_ctx_create(int32_t device, void* stream, apex_ctx** out) {
  if (!out) return set_err(APEX_EINVAL, "null out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return set_err(APEX_ECUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                   "); the B200 path has no CPU fallback");
  }
  if (device < 0 || device >= n) return set_err(APEX_EINVAL, "bad device ordinal");
  APEX_CU(cudaSetDevice(device));
  apex_ctx* c = new apex_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  if (c->cc_major != 10) {
    delete c;
    return set_err(APEX_ECUDA, "device is not sm_100 (B200); kernels are built for sm_100a only");
  }
  {
    static std::mutex m;
    static std::vector<int> loaded;
    std::lock_guard<std::mutex> g(m);
    if (std::find(loaded.begin(), loaded.end(), device) == loaded.end()) {
      preload_kernels();
      loaded.push_back(device);
    }
  }
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete c;
      return set_err(APEX_ECUDA, "stream creation failed");
    }
    c->own_stream = true;
  }
  for (auto& ev : c->ev) cudaEventCreate(&ev);
  for (auto& ev : c->mev) cudaEventCreate(&ev);
  cudaEventCreateWithFlags(&c->upload_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming);
  {
    int lo = 0, hi = 0;  // the seed side stream at the highest priority (see the pre-pass stream below)
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi);
  }
  cudaEventCreateWithFlags(&c->fork2_ev, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->join2_ev, cudaEventDisableTiming);
  {
    // the pre-pass stream at the lowest priority (its thousands of CTAs would
    // otherwise hold every SM slot while the threshold kernel waits), the
    // context's own streams at the highest
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStreamCreateWithPriority(&c->side2, cudaStreamNonBlocking, c->opt_cpre_prio > 0 ? hi : lo);
  }
  *out = c;
  return APEX_OK;
}

void apex_ctx_destroy(apex_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& s : c->slots) s.release();
  c->plans.clear();
  c->d_rx.release();
  c->d_goff.release();
  c->d_values.release();
  c->d_biases.release();
  for (DBuf* b : {&c->d_lists, &c->d_slot_off, &c->d_m, &c->d_coff, &c->d_sorted_x, &c->d_sorted_col, &c->d_quant,
                  &c->d_packed16})
    b->release();
  c->d_queries.release();
  c->d_tau0.release();
  c->d_hists.release();
  c->d_ctls.release();
  c->d_out.release();
  c->d_work.release();
  for (DBuf* b : {&c->d_rowp, &c->d_fin_scratch, &c->d_cthr, &c->d_cqc, &c->d_cbest}) b->release();
  c->d_trace.release();
  c->h_queries.release();
  c->h_ctl.release();
  c->h_out.release();
  c->h_tau0.release();
  for (auto& ev : c->ev) cudaEventDestroy(ev);
  for (auto& ev : c->mev) cudaEventDestroy(ev);
  for (DBuf* b : {&c->d_gt_members, &c->d_gt_latent, &c->d_gt_tasks, &c->d_gt_hist, &c->d_gt_buf, &c->d_gt_misc,
                  &c->d_u_res})
    b->release();
  {
    auto& w = c->mws;
    for (auto& sl : w.slots) sl.release();
    for (DBuf* b : {&w.d_hists, &w.d_ctls, &w.d_queries, &w.d_out}) b->release();
    for (HBuf* b : {&w.h_queries, &w.h_ctl, &w.h_out}) b->release();
  }
  if (c->upload_ev) cudaEventDestroy(c->upload_ev);
  if (c->done_ev) cudaEventDestroy(c->done_ev);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->fork2_ev) cudaEventDestroy(c->fork2_ev);
  if (c->join2_ev) cudaEventDestroy(c->join2_ev);
  if (c->side2) cudaStreamDestroy(c->side2);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

int apex_set_stream(apex_ctx* c, void* stream) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (c->own_stream) {
    cudaStreamSynchronize(c->stream);
    cudaStreamDestroy(c->stream);
    c->own_stream = false;
  }
  if (stream) {
    c->stream = (cudaStream_t)stream;
  } else {
    APEX_CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  return APEX_OK;
}

int apex_load_library(apex_ctx* c, const apex_reaction* rxs, int32_t n_rx, int64_t n_pairs) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (n_rx < 0 || (n_rx > 0 && !rxs) || n_pairs < 0) return set_err(APEX_EINVAL, "bad library arguments");
  std::vector<DevReaction> rx(n_rx);
  std::vector<unsigned long long> goff(n_rx + 1, 0);
  unsigned __int128 total = 0;
  unsigned __int128 rows_total = 0;
  int64_t pcols = 0;
  for (int t = 0; t < n_rx; ++t) {
    const apex_reaction& a = rxs[t];
    if (a.n_rgroups < 1 || a.n_rgroups > kMaxRg)
      return set_err(APEX_ELIMIT, "reaction " + std::to_string(t) + " has " + std::to_string(a.n_rgroups) +
                                      " R-groups (supported: 1.." + std::to_string(kMaxRg) + ")");
    DevReaction& R = rx[t];
    std::memset(&R, 0, sizeof(R));
    R.c = a.n_rgroups;
    unsigned __int128 size = 1;
    for (int j = 0; j < R.c; ++j) {
      if (a.sizes[j] < 1) return set_err(APEX_EINVAL, "empty R-group");
      if (a.pair_offset[j] < 0 || a.pair_offset[j] + a.sizes[j] > n_pairs)
        return set_err(APEX_EINVAL, "table rows for an R-group do not match library");
      R.size[j] = a.sizes[j];
      R.pair_off[j] = a.pair_offset[j];
      size *= (unsigned __int128)a.sizes[j];
    }
    if (R.size[R.c - 1] > 0xffffffffll) return set_err(APEX_ELIMIT, "last R-group larger than 2^32");
    R.n_rows = (uint64_t)(size / (unsigned __int128)R.size[R.c - 1]);
    R.row_off = (int64_t)rows_total;
    rows_total += R.n_rows;
    R.pcol_off = pcols;
    pcols += (R.size[R.c - 1] + 3) / 4 * 4;
    if ((uint64_t)total != a.g_offset) return set_err(APEX_EINVAL, "reaction offsets are not the running product count");
    R.g_off = a.g_offset;
    goff[t] = (unsigned long long)total;
    total += size;
    if (total > (unsigned __int128)UINT64_MAX) return set_err(APEX_ELIMIT, "product count exceeds unsigned 64-bit range");
  }
  goff[n_rx] = (unsigned long long)total;
  APEX_TRY(c->d_rx.ensure(std::max<size_t>(1, rx.size()) * sizeof(DevReaction)));
  APEX_TRY(c->d_goff.ensure(goff.size() * sizeof(unsigned long long)));
  if (n_rx) APEX_CU(cudaMemcpy(c->d_rx.p, rx.data(), rx.size() * sizeof(DevReaction), cudaMemcpyHostToDevice));
  APEX_CU(cudaMemcpy(c->d_goff.p, goff.data(), goff.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  c->rx = std::move(rx);
  c->goff = std::move(goff);
  c->total = (uint64_t)total;
  c->lib_pairs = n_pairs;
  c->pcols = pcols;
  c->rows_total = rows_total > (unsigned __int128)INT64_MAX ? 0 : (int64_t)rows_total;  // 0: no row-prefix table
  c->lib_loaded = true;
  c->batch.plan = nullptr;
  c->batch.pending = false;
  c->plans.clear();
  c->corners_ok = false;
  return APEX_OK;
}

int apex_load_table(apex_ctx* c, const float* values, const double* biases, int32_t n_tasks, int64_t n_pairs) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (n_tasks < 1 || n_pairs < 0 || !biases || (n_pairs > 0 && !values)) return set_err(APEX_EINVAL, "bad table arguments");
  const size_t n = (size_t)n_tasks * n_pairs;
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(values[i])) return set_err(APEX_EINVAL, "contribution table has non-finite entries");
  for (int t = 0; t < n_tasks; ++t)
    if (!std::isfinite(biases[t])) return set_err(APEX_EINVAL, "contribution table has non-finite biases");
  APEX_TRY(c->d_values.ensure(std::max<size_t>(n, 1) * sizeof(float)));
  APEX_TRY(c->d_biases.ensure(n_tasks * sizeof(double)));
  if (n) APEX_CU(cudaMemcpy(c->d_values.p, values, n * sizeof(float), cudaMemcpyHostToDevice));
  APEX_CU(cudaMemcpy(c->d_biases.p, biases, n_tasks * sizeof(double), cudaMemcpyHostToDevice));
  c->biases.assign(biases, biases + n_tasks);
  c->n_tasks = n_tasks;
  c->n_pairs = n_pairs;
  c->table_loaded = true;
  c->corners_ok = false;
  return APEX_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      p = nullptr;
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

int apex_precompute_device(apex_ctx* c, const double* u_dev, int64_t n_pairs, int32_t d, const double* w_dev,
                           int32_t n_tasks, float* values_dev) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (n_pairs < 0 || d < 1 || n_tasks < 1 || !w_dev || !values_dev || (n_pairs > 0 && !u_dev))
    return set_err(APEX_EINVAL, "bad precompute arguments");
  if (n_pairs == 0) return APEX_OK;
  PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
  if (n_tasks == 11 && d == 64 && c->opt_pre_rows == 2 && encode && n_pairs < (int64_t(1) << 31) &&
      (reinterpret_cast<uintptr_t>(u_dev) & 15) == 0) {
    // TMA form (the APEX model's 11 x 64): one persistent CTA per SM, swizzled
    // 2-D tensor copies of u tiles into a 3-stage ring, heads as kernel parameters
    HeadParams<11, 64> W;
    cudaPointerAttributes pa;
    const bool w_on_host = cudaPointerGetAttributes(&pa, w_dev) == cudaSuccess &&
                           (pa.type == cudaMemoryTypeHost || pa.type == cudaMemoryTypeUnregistered);
    cudaGetLastError();
    if (w_on_host) {
      std::memcpy(W.w, w_dev, sizeof(W.w));  // heads given in host memory: no device round trip, no sync
    } else {
      APEX_CU(cudaMemcpyAsync(W.w, w_dev, sizeof(W.w), cudaMemcpyDeviceToHost, c->stream));
      APEX_CU(cudaStreamSynchronize(c->stream));
    }
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {64, (cuuint64_t)n_pairs};
    const cuuint64_t strides[1] = {64 * sizeof(double)};
    const cuuint32_t box[2] = {kBulkBoxCols, kBulkRows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult er = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(u_dev), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (er != CUDA_SUCCESS) return set_err(APEX_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)er) + ")");
    const size_t smem = bulk_smem_bytes<11, 64>();
    APEX_CU(cudaFuncSetAttribute((const void*)precompute_bulk_kernel<11, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    const int64_t tiles = (n_pairs + kBulkRows - 1) / kBulkRows;
    const int blocks = (int)std::min<int64_t>(tiles, c->sm_count);
    APEX_CU(cudaEventRecord(c->mev[0], c->stream));
    precompute_bulk_kernel<11, 64><<<blocks, kBulkThreads, smem, c->stream>>>(tmap, n_pairs, W, values_dev);
    APEX_CU(cudaGetLastError());
    APEX_CU(cudaEventRecord(c->mev[1], c->stream));
    c->k1_timed = true;
    return APEX_OK;
  }
  c->k1_timed = false;
  if (n_tasks <= kPvTasks && d % kPvCols == 0 && c->opt_pre_rows) {
    // row-parallel form: every task per thread, u streamed in 16-column chunks
    const size_t smem2 = ((size_t)((n_tasks * d + 1) & ~1) + 2 * (size_t)kPvRows * kPvLd) * sizeof(double);
    if (smem2 <= 200 * 1024) {
      using PFn = void (*)(const double*, int64_t, int, const double*, int, float*);
      const PFn fn = (n_tasks == 11 && d == 64) ? precompute_rows_kernel<11, 64> : precompute_rows_kernel<0, 0>;
      APEX_CU(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
      int occ2 = 0;
      APEX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, (const void*)fn, kPvRows, smem2));
      const int64_t blocks2 =
          std::min<int64_t>((n_pairs + kPvRows - 1) / kPvRows, (int64_t)c->sm_count * std::max(occ2, 1));
      APEX_CU(cudaEventRecord(c->mev[0], c->stream));
      fn<<<(unsigned)blocks2, kPvRows, smem2, c->stream>>>(u_dev, n_pairs, d, w_dev, n_tasks, values_dev);
      APEX_CU(cudaGetLastError());
      APEX_CU(cudaEventRecord(c->mev[1], c->stream));
      c->k1_timed = true;
      return APEX_OK;
    }
  }
  const size_t smem = ((size_t)n_tasks * d + (size_t)kPreRows * (d + 1)) * sizeof(double);
  if (smem > 220 * 1024) return set_err(APEX_ELIMIT, "precompute: n_tasks * d too large for shared memory");
  APEX_CU(cudaFuncSetAttribute((const void*)precompute_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  APEX_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)precompute_kernel, 256, smem));
  const int64_t blocks = std::min<int64_t>((n_pairs + kPreRows - 1) / kPreRows, (int64_t)c->sm_count * std::max(occ, 1));
  APEX_CU(cudaEventRecord(c->mev[0], c->stream));
  precompute_kernel<<<(unsigned)blocks, 256, smem, c->stream>>>(u_dev, n_pairs, d, w_dev, n_tasks, values_dev);
  APEX_CU(cudaGetLastError());
  APEX_CU(cudaEventRecord(c->mev[1], c->stream));
  c->k1_timed = true;
  return APEX_OK;
}

int apex_precompute_time(apex_ctx* c, double* kernel_ms) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (!kernel_ms) return set_err(APEX_EINVAL, "null output");
  *kernel_ms = -1.0;
  if (!c->k1_timed) return APEX_OK;
  APEX_CU(cudaEventSynchronize(c->mev[1]));
  float ms = 0.f;
  APEX_CU(cudaEventElapsedTime(&ms, c->mev[0], c->mev[1]));
  *kernel_ms = ms;
  return APEX_OK;
}

int apex_load_cache(apex_ctx* c, const double* u, int64_t n_pairs, int32_t d, const double* head_w,
                    const double* head_b, int32_t n_tasks, float* values_out) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (!u || !head_w || !head_b || n_pairs < 0 || d < 1 || n_tasks < 1) return set_err(APEX_EINVAL, "bad cache arguments");
  for (int t = 0; t < n_tasks; ++t)
    if (!std::isfinite(head_b[t])) return set_err(APEX_EINVAL, "non-finite head bias");
  DBuf du, dw;
  APEX_TRY(du.ensure(std::max<size_t>(1, (size_t)n_pairs * d) * sizeof(double)));
  APEX_TRY(dw.ensure((size_t)n_tasks * d * sizeof(double)));
  APEX_TRY(c->d_values.ensure(std::max<size_t>(1, (size_t)n_tasks * n_pairs) * sizeof(float)));
  APEX_TRY(c->d_biases.ensure(n_tasks * sizeof(double)));
  APEX_CU(cudaMemcpyAsync(du.p, u, (size_t)n_pairs * d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  APEX_CU(cudaMemcpyAsync(dw.p, head_w, (size_t)n_tasks * d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  APEX_CU(cudaMemcpyAsync(c->d_biases.p, head_b, n_tasks * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // (the TMA form takes the host heads directly as kernel parameters)
  const bool host_heads = n_tasks == 11 && d == 64 && c->opt_pre_rows == 2;
  int rc = apex_precompute_device(c, du.as<double>(), n_pairs, d, host_heads ? head_w : dw.as<double>(), n_tasks,
                                  c->d_values.as<float>());
  if (rc != APEX_OK) {
    du.release();
    dw.release();
    return rc;
  }
  if (values_out && n_pairs > 0)
    APEX_CU(cudaMemcpyAsync(values_out, c->d_values.p, (size_t)n_tasks * n_pairs * sizeof(float), cudaMemcpyDeviceToHost,
                            c->stream));
  APEX_CU(cudaStreamSynchronize(c->stream));
  du.release();
  dw.release();
  c->biases.assign(head_b, head_b + n_tasks);
  c->n_tasks = n_tasks;
  c->n_pairs = n_pairs;
  c->table_loaded = true;
  c->corners_ok = false;
  return APEX_OK;
}

int apex_query_async(apex_ctx* c, const apex_query_spec* qs, int32_t nq, apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  APEX_TRY(validate_queries(c, qs, nq));
  if (nq < 1) return set_err(APEX_EINVAL, "apex_query_async needs at least one query");
  for (int i = 0; i < nq; ++i) {
    if (qs[i].start != qs[0].start || qs[i].end != qs[0].end)
      return set_err(APEX_EINVAL, "apex_query_async: all queries must share one index range");
    if (qs[i].k < 1 || qs[i].end == qs[i].start)
      return set_err(APEX_EINVAL, "apex_query_async: k >= 1 and a non-empty range required (use apex_query)");
  }
  const auto t0 = std::chrono::steady_clock::now();
  APEX_TRY(prepare_batch(c, qs, nq, true));
  const auto t1 = std::chrono::steady_clock::now();
  APEX_TRY(launch_batch(c));
  const auto t2 = std::chrono::steady_clock::now();
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->kernel_launches = c->batch.st.launches;
    stats->scan_launches = c->batch.st.scans;
    stats->h2d_bytes = c->batch.st.h2d_bytes;
    stats->host_prepare_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
    stats->host_launch_us = std::chrono::duration<double, std::micro>(t2 - t1).count();
  }
  return APEX_OK;
}

int apex_query_fetch(apex_ctx* c, apex_result* res, apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  Batch& B = c->batch;
  if (!B.pending) return set_err(APEX_ESTATE, "no query batch in flight");
  if (!res) return set_err(APEX_EINVAL, "null results");
  APEX_TRY(check_batch(c));
  float d2h = 0;
  if (B.copy_out) {
    // rows already in the pinned block (copied inside the pass, synced by check_batch)
    const auto h0 = std::chrono::steady_clock::now();
    APEX_TRY(copy_results(c, B.qs.data(), B.nq, res, B.perm.data(), true));
    d2h = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - h0).count();
  } else {
    APEX_CU(cudaEventRecord(c->ev[6], c->stream));
    APEX_TRY(copy_results(c, B.qs.data(), B.nq, res, B.perm.data(), false));
    APEX_CU(cudaEventRecord(c->ev[7], c->stream));
    APEX_CU(cudaEventSynchronize(c->ev[7]));
    cudaEventElapsedTime(&d2h, c->ev[6], c->ev[7]);
  }
  int64_t cand = 0, out = 0, admitted = 0;
  for (int i = 0; i < B.nq; ++i) {
    admitted += (int64_t)c->h_ctl.as<QCtl>()[i].admitted;
    cand += (int64_t)c->h_ctl.as<QCtl>()[i].count;
    out += (int64_t)out_bytes(std::max<int64_t>(B.qs[i].k, 1), B.qs[i].n_constraints);
  }
  B.st.d2h_bytes += out;
  float total = d2h;
  for (int e = 0; e < 5; ++e) total += B.st.ms[e];
  fill_stats(stats, B.st, d2h, total, cand);
  if (stats) stats->admitted = admitted;
  return APEX_OK;
}

int apex_query(apex_ctx* c, const apex_query_spec* qs, int32_t nq, apex_result* res, apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  APEX_TRY(validate_queries(c, qs, nq));
  if (nq > 0 && !res) return set_err(APEX_EINVAL, "null results");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  // group queries by range (each group shares one enumeration schedule)
  std::vector<int> order(nq);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return qs[a].start != qs[b].start ? qs[a].start < qs[b].start : qs[a].end < qs[b].end;
  });
  apex_stats agg;
  std::memset(&agg, 0, sizeof(agg));
  {
    bool view = false, multi_range = false;
    for (int i = 0; i < nq; ++i) {
      const apex_result& r = res[i];
      view = view || (!r.global_index && !r.objective && !r.constraint_values && !r.reaction && !r.digits);
      multi_range = multi_range || qs[i].start != qs[0].start || qs[i].end != qs[0].end;
    }
    if (view && multi_range)
      return set_err(APEX_EINVAL, "result views (null output arrays) need all queries of the call to share one range");
  }
  size_t g0 = 0;
  while (g0 < order.size()) {
    size_t g1 = g0 + 1;
    while (g1 < order.size() && qs[order[g1]].start == qs[order[g0]].start && qs[order[g1]].end == qs[order[g0]].end) ++g1;
    std::vector<apex_query_spec> grp;
    std::vector<int> live;
    for (size_t i = g0; i < g1; ++i) {
      const apex_query_spec& q = qs[order[i]];
      if (q.k > 0 && q.end > q.start) {
        grp.push_back(q);
        live.push_back(order[i]);
      } else {
        apex_result& r = res[order[i]];
        r.n = 0;
        r.scanned = q.end - q.start;
        r.discarded = 0;
        r.candidates = r.admitted = 0;
        r.full_predicate = 0;
      }
    }
    if (!grp.empty()) {
      apex_stats st;
      c->copy_next = true;  // the rows go to the host right away: copy them inside the pass
      const int rq = apex_query_async(c, grp.data(), (int)grp.size(), nullptr);
      c->copy_next = false;
      if (rq != APEX_OK) return rq;
      std::vector<apex_result> tmp(grp.size());
      for (size_t i = 0; i < grp.size(); ++i) tmp[i] = res[live[i]];
      APEX_TRY(apex_query_fetch(c, tmp.data(), &st));
      for (size_t i = 0; i < grp.size(); ++i) res[live[i]] = tmp[i];
      agg.pack_ms += st.pack_ms;
      agg.seed_ms += st.seed_ms;
      agg.scan_ms += st.scan_ms;
      agg.select_ms += st.select_ms;
      agg.finalize_ms += st.finalize_ms;
      agg.d2h_ms += st.d2h_ms;
      agg.total_ms += st.total_ms;
      agg.scan_kernel_ms += st.scan_kernel_ms;
      agg.candidates += st.candidates;
      agg.scan_launches += st.scan_launches;
      agg.kernel_launches += st.kernel_launches;
      agg.retries += st.retries;
      agg.h2d_bytes += st.h2d_bytes;
      agg.d2h_bytes += st.d2h_bytes;
      agg.admitted += st.admitted;
    }
    g0 = g1;
  }
  if (stats) *stats = agg;
  return APEX_OK;
}

int apex_query_local(apex_ctx* c, const apex_query_spec* qs, int32_t nq, apex_entry* out_dev, int64_t* counts,
                     apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  APEX_TRY(validate_queries(c, qs, nq));
  if (nq <= 0) return APEX_OK;
  if (!out_dev || !counts) return set_err(APEX_EINVAL, "null output");
  for (int i = 1; i < nq; ++i)
    if (qs[i].start != qs[0].start || qs[i].end != qs[0].end || qs[i].k != qs[0].k)
      return set_err(APEX_EINVAL, "apex_query_local: all queries must share range and k");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  const int64_t k = qs[0].k;
  if (k == 0 || qs[0].end == qs[0].start) {
    for (int i = 0; i < nq; ++i) counts[i] = 0;
    return APEX_OK;
  }
  APEX_TRY(local_enqueue(c, qs, nq, reinterpret_cast<Entry*>(out_dev), (unsigned long long)k));
  APEX_TRY(local_finish(c, counts, nullptr));
  APEX_CU(cudaStreamSynchronize(c->stream));
  int64_t cand = 0;
  for (int i = 0; i < nq; ++i) cand += (int64_t)c->h_ctl.as<QCtl>()[i].count;
  float total = 0;
  for (int e = 0; e < 5; ++e) total += c->batch.st.ms[e];
  fill_stats(stats, c->batch.st, 0.f, total, cand);
  return APEX_OK;
}

int apex_query_local_async(apex_ctx* c, const apex_query_spec* qs, int32_t nq, apex_entry* out_dev, int64_t stride,
                           apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  APEX_TRY(validate_queries(c, qs, nq));
  if (nq < 1 || !out_dev) return set_err(APEX_EINVAL, "apex_query_local_async: queries and an output buffer required");
  for (int i = 0; i < nq; ++i) {
    if (qs[i].start != qs[0].start || qs[i].end != qs[0].end)
      return set_err(APEX_EINVAL, "apex_query_local_async: all queries must share one index range");
    if (qs[i].k < 1 || qs[i].k > stride) return set_err(APEX_EINVAL, "apex_query_local_async: need 1 <= k <= stride");
  }
  if (qs[0].end == qs[0].start) return set_err(APEX_EINVAL, "apex_query_local_async: empty range");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  APEX_TRY(local_enqueue(c, qs, nq, reinterpret_cast<Entry*>(out_dev), (unsigned long long)stride));
  if (stats) {
    stats->kernel_launches = c->batch.st.launches;
    stats->h2d_bytes = c->batch.st.h2d_bytes;
  }
  return APEX_OK;
}

int apex_query_local_finish(apex_ctx* c, int64_t* counts, int32_t* rerun, apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  int again = 0;
  APEX_TRY(local_finish(c, counts, &again));
  if (rerun) *rerun = again;
  if (stats) {
    int64_t cand = 0;
    for (int i = 0; i < c->batch.nq; ++i) cand += (int64_t)c->h_ctl.as<QCtl>()[i].count;
    float total = 0;
    for (int e = 0; e < 5; ++e) total += c->batch.st.ms[e];
    fill_stats(stats, c->batch.st, 0.f, total, cand);
  }
  return APEX_OK;
}

int apex_merge_finalize_batch(apex_ctx* c, const apex_query_spec* qs, int32_t nq, const apex_entry* entries_dev,
                              int32_t n_src, int64_t stride, uint64_t total_scanned, apex_result* res,
                              apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  if (nq < 0 || n_src < 0 || stride < 0 || (nq > 0 && (!qs || !res)) ||
      (n_src > 0 && stride > 0 && nq > 0 && !entries_dev))
    return set_err(APEX_EINVAL, "bad merge arguments");
  return merge_impl(c, qs, nq, reinterpret_cast<const Entry*>(entries_dev), nullptr, n_src, stride, total_scanned,
                    res, stats);
}

int apex_merge_finalize(apex_ctx* c, const apex_query_spec* q, const apex_entry* entries_dev, int64_t n_entries,
                        uint64_t total_scanned, apex_result* res, apex_stats* stats) {
  if (!q || !res || n_entries < 0 || (n_entries > 0 && !entries_dev)) return set_err(APEX_EINVAL, "bad merge arguments");
  return apex_merge_finalize_batch(c, q, 1, entries_dev, 1, n_entries, total_scanned, res, stats);
}

int apex_set_option(apex_ctx* c, const char* name, int64_t v) {
  APEX_LOCK(c);
  if (!c || !name) return set_err(APEX_EINVAL, "bad option arguments");
  std::string n(name);
  ++c->opt_gen;
  if (n == "cap") c->opt_cap = std::max<int64_t>(v, 1024);
  else if (n == "cb") {
    if (v < 8 || v % 8 || v > 256) return set_err(APEX_EINVAL, "cb must be a multiple of 8 in [8, 256]");
    c->opt_cb = v;
  } else if (n == "rl") c->opt_rl = v;
  else if (n == "samples") c->opt_samples = v;
  else if (n == "chunk_div") c->opt_chunk_div = v;
  else if (n == "force_upload") c->opt_force_upload = v;
  else if (n == "refresh") c->opt_refresh = v;
  else if (n == "corner") c->opt_corner = v;
  else if (n == "pre_rows") c->opt_pre_rows = v;
  else if (n == "corner_mult") c->opt_corner_mult = std::max<int64_t>(1, v);
  else if (n == "vote64") c->opt_vote64 = v;
  else if (n == "dense") c->opt_dense = v;
  else if (n == "sorted") c->opt_sorted = v;
  else if (n == "cpre") c->opt_cpre = v;
  else if (n == "stages") c->opt_stages = v;
  else if (n == "cpre_fused") c->opt_cpre_fused = v;
  else if (n == "lazy_hist") {
    if (v && !c->opt_lazy_hist && c->d_hists.p) APEX_CU(cudaMemset(c->d_hists.p, 0, c->d_hists.bytes));
    c->opt_lazy_hist = v;
  }
  else if (n == "tau_side") c->opt_tau_side = v;
  else if (n == "graph_prio") c->opt_graph_prio = v;
  else if (n == "cpre_prio") {
    c->opt_cpre_prio = v;
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    APEX_CU(cudaStreamSynchronize(c->side2));
    cudaStreamDestroy(c->side2);
    APEX_CU(cudaStreamCreateWithPriority(&c->side2, cudaStreamNonBlocking, v > 0 ? hi : lo));
  }
  else if (n == "fin_part") c->opt_fin_part = v;
  else if (n == "bail") c->opt_bail = std::max<int64_t>(0, v);
  else if (n == "bail_min") c->opt_bail_min = std::max<int64_t>(1, v);
  else if (n == "spin_us") c->opt_spin_us = std::max<int64_t>(0, v);
  else if (n == "cpre_ctas") c->opt_cpre_ctas = std::max<int64_t>(0, v);
  else if (n == "work_ctrs") c->opt_work_ctrs = std::max<int64_t>(1, v);
  else if (n == "rowp") {
    c->opt_rowp = v;
    c->corners_ok = false;  // rebuilt (or dropped) at the next query
  } else if (n == "rowp_bytes") {
    c->opt_rowp_bytes = std::max<int64_t>(0, v);
    c->corners_ok = false;
  }
  else if (n == "fin_bucket") c->opt_fin_bucket = std::max<int64_t>(0, v);
  else if (n == "trace") {
    // records of the admission scan's per-item trace (0: off); debug only
    c->trace_cap = std::max<int64_t>(0, std::min<int64_t>(v, 1ll << 26));
    c->trace_n = 0;
    if (c->trace_cap) {
      APEX_TRY(c->d_trace.ensure((size_t)c->trace_cap * 64));
      APEX_CU(cudaMemset(c->d_trace.p, 0, (size_t)c->trace_cap * 64));
    }
  }
  else if (n == "graph") c->opt_graph = v;
  else if (n == "packed16") c->opt_packed16 = v;
  else if (n == "chunk") c->opt_chunk = std::max<int64_t>(1, v);
  else if (n == "tiles_per_slot") c->opt_tiles_per_slot = std::max<int64_t>(1, v);
  else if (n == "mode") {
    if (v < 0 || v > 3 || v == 1) return set_err(APEX_EINVAL, "mode must be 0, 2 or 3");
    c->opt_mode = v;
  } else if (n == "cb_admit") {
    if (v < 64 || v % 64 || v > 4096) return set_err(APEX_EINVAL, "cb_admit must be a multiple of 64 in [64, 4096]");
    c->opt_cb_admit = v;
  }
  else if (n == "chunk_min") c->opt_chunk_min = std::max<int64_t>(v, 1);
  else if (n == "split_cols" || n == "split_rows") {
    (n == "split_cols" ? c->opt_split_cols : c->opt_split_rows) = std::max<int64_t>(0, v);
    c->batch.plan = nullptr;
    c->batch.plan_rows = nullptr;
    c->batch.pending = false;
    c->plans.clear();
  } else if (n == "heavy_first") {
    c->opt_heavy_first = v;
    c->batch.plan = nullptr;
    c->batch.plan_rows = nullptr;
    c->batch.pending = false;
    c->plans.clear();
  } else if (n == "tile_products") {
    c->opt_tile_products = v;
    c->batch.plan = nullptr;
    c->batch.pending = false;
    c->plans.clear();
  } else if (n == "select_ctas") c->opt_select_ctas = std::max<int64_t>(1, v);
  else return set_err(APEX_EINVAL, "unknown option " + n);
  return APEX_OK;
}

int apex_get_device_info(apex_ctx* c, int32_t* sm, int32_t* ma, int32_t* mi) {
  if (!c) return set_err(APEX_EINVAL, "null context");
  if (sm) *sm = c->sm_count;
  if (ma) *ma = c->cc_major;
  if (mi) *mi = c->cc_minor;
  return APEX_OK;
}

int apex_debug_thresholds(apex_ctx* c, const double* p, const double* b, const double* beta, int64_t n, float* up,
                          float* lo) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (n <= 0) return APEX_OK;
  DBuf dp, db, dbeta, du, dl;
  APEX_TRY(dp.ensure(n * 8));
  APEX_TRY(db.ensure(n * 8));
  APEX_TRY(dbeta.ensure(n * 8));
  APEX_TRY(du.ensure(n * 4));
  APEX_TRY(dl.ensure(n * 4));
  APEX_CU(cudaMemcpy(dp.p, p, n * 8, cudaMemcpyHostToDevice));
  APEX_CU(cudaMemcpy(db.p, b, n * 8, cudaMemcpyHostToDevice));
  APEX_CU(cudaMemcpy(dbeta.p, beta, n * 8, cudaMemcpyHostToDevice));
  thresholds_kernel<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(dp.as<double>(), db.as<double>(),
                                                                        dbeta.as<double>(), (int)n, du.as<float>(),
                                                                        dl.as<float>());
  APEX_CU(cudaGetLastError());
  APEX_CU(cudaStreamSynchronize(c->stream));
  APEX_CU(cudaMemcpy(up, du.p, n * 4, cudaMemcpyDeviceToHost));
  APEX_CU(cudaMemcpy(lo, dl.p, n * 4, cudaMemcpyDeviceToHost));
  for (DBuf* d : {&dp, &db, &dbeta, &du, &dl}) d->release();
  return APEX_OK;
}

int apex_debug_trace(apex_ctx* c, uint64_t* out, int64_t cap, int64_t* n) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  const int64_t m = std::min<int64_t>(cap, c->trace_n);
  if (n) *n = std::max<int64_t>(m, 0);
  if (m <= 0) return APEX_OK;
  APEX_CU(cudaStreamSynchronize(c->stream));
  APEX_CU(cudaMemcpy(out, c->d_trace.p, (size_t)m * 64, cudaMemcpyDeviceToHost));
  return APEX_OK;
}

// ===========================================================================
// Ground-truth evaluation on the device (gt.cuh; evalkit.oracle_topk)
// ===========================================================================

int apex_gt_load(apex_ctx* c, const int64_t* member_ids, int64_t n_pairs, const double* latents, int64_t n_synthons,
                 const apex_gt_task* tasks, int32_t n_tasks) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (!c->lib_loaded) return set_err(APEX_ESTATE, "load the library before the ground-truth oracle");
  if (n_pairs != c->lib_pairs || n_synthons < 1 || n_tasks < 1 || n_tasks > 4096 || !member_ids || !latents || !tasks)
    return set_err(APEX_EINVAL, "bad ground-truth oracle arguments");
  for (int64_t i = 0; i < n_pairs; ++i)
    if (member_ids[i] < 0 || member_ids[i] >= n_synthons) return set_err(APEX_EINVAL, "synthon id out of range");
  APEX_TRY(c->d_gt_members.ensure((size_t)n_pairs * sizeof(long long)));
  APEX_TRY(c->d_gt_latent.ensure((size_t)n_tasks * n_synthons * sizeof(double)));
  APEX_TRY(c->d_gt_tasks.ensure((size_t)n_tasks * sizeof(GtTask)));
  APEX_CU(cudaMemcpy(c->d_gt_members.p, member_ids, (size_t)n_pairs * sizeof(long long), cudaMemcpyHostToDevice));
  APEX_CU(cudaMemcpy(c->d_gt_latent.p, latents, (size_t)n_tasks * n_synthons * sizeof(double), cudaMemcpyHostToDevice));
  c->gt_tasks.assign(n_tasks, GtTask{});
  for (int t = 0; t < n_tasks; ++t) {
    GtTask& T = c->gt_tasks[t];
    T.latent = c->d_gt_latent.as<double>() + (size_t)t * n_synthons;
    T.nl_scale = tasks[t].nonlinear_scale;
    T.nl_alpha = tasks[t].nonlinear_alpha;
    T.pair_scale = tasks[t].pair_scale;
    T.pair_density = tasks[t].pair_density;
    T.salt = tasks[t].salt;
    T.flags = tasks[t].flags;
  }
  APEX_CU(cudaMemcpy(c->d_gt_tasks.p, c->gt_tasks.data(), (size_t)n_tasks * sizeof(GtTask), cudaMemcpyHostToDevice));
  c->gt_synthons = n_synthons;
  c->gt_loaded = true;
  return APEX_OK;
}

int apex_gt_topk(apex_ctx* c, const apex_query_spec* q, apex_result* res, apex_stats* stats) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  if (!c->gt_loaded) return set_err(APEX_ESTATE, "ground-truth oracle not loaded");
  if (!q || !res || !res->global_index || !res->objective || !res->reaction || !res->digits ||
      (q->n_constraints > 0 && !res->constraint_values))
    return set_err(APEX_EINVAL, "bad ground-truth query arguments");
  const int nt = (int)c->gt_tasks.size();
  if (q->objective_task < 0 || q->objective_task >= nt) return set_err(APEX_ETASK, "unknown oracle task");
  if (q->n_constraints < 0 || q->n_constraints > kMaxCons || (q->n_constraints && !q->constraints))
    return set_err(APEX_EINVAL, "bad constraint list");
  for (int m = 0; m < q->n_constraints; ++m)
    if (q->constraints[m].task < 0 || q->constraints[m].task >= nt) return set_err(APEX_ETASK, "unknown oracle task");
  if (q->k < 0) return set_err(APEX_EINVAL, "j must be >= 0");
  if (!(q->start <= q->end && q->end <= c->total)) return set_err(APEX_ERANGE, "index range invalid");
  if (stats) std::memset(stats, 0, sizeof(*stats));
  const uint64_t span = q->end - q->start;
  res->scanned = span;
  res->candidates = res->admitted = 0;
  res->full_predicate = 0;
  res->n = 0;
  res->discarded = 0;
  if (q->k == 0 || span == 0) return APEX_OK;
  const auto t0 = std::chrono::steady_clock::now();
  int64_t max_last = 1;
  for (const auto& R : c->rx) max_last = std::max<int64_t>(max_last, R.size[R.c - 1]);
  Plan* plan = nullptr;
  APEX_TRY(build_plan(c, q->start, q->end, 32, 1, plan, max_last));
  const unsigned long long cap = (unsigned long long)std::max<int64_t>(4 * q->k + 4096, 1 << 22);
  APEX_TRY(c->d_gt_hist.ensure((65536 + 256) * sizeof(unsigned)));
  APEX_TRY(c->d_gt_buf.ensure(cap * sizeof(Entry)));
  APEX_TRY(c->d_gt_misc.ensure(64));
  cudaStream_t s = c->stream;
  GtPass P;
  std::memset(&P, 0, sizeof(P));
  P.rx = c->d_rx.as<DevReaction>();
  P.tiles = plan->d_tiles.as<Tile>();
  P.n_tiles = (unsigned)plan->tiles.size();
  P.members = c->d_gt_members.as<long long>();
  P.tasks = c->d_gt_tasks.as<GtTask>();
  P.obj = q->objective_task;
  P.maximize = q->maximize ? 1 : 0;
  P.n_cons = q->n_constraints;
  for (int m = 0; m < q->n_constraints; ++m) {
    P.cons_task[m] = q->constraints[m].task;
    P.cons_lo[m] = q->constraints[m].lower;
    P.cons_hi[m] = q->constraints[m].upper;
  }
  P.hist = c->d_gt_hist.as<unsigned>();
  P.buf = c->d_gt_buf.as<Entry>();
  P.cap = cap;
  unsigned long long* d_count = reinterpret_cast<unsigned long long*>(c->d_gt_misc.p);
  long long* d_kth = reinterpret_cast<long long*>(c->d_gt_misc.as<unsigned char>() + 16);
  unsigned* d_work = reinterpret_cast<unsigned*>(c->d_gt_misc.as<unsigned char>() + 32);
  P.count = d_count;
  P.work = d_work;
  P.base = 0;
  P.shift = 48;
  P.glimit = q->end;
  const int grid = c->sm_count * 8;
  int64_t launches = 0;
  // narrowing passes: the bin holding the j-th best key, 16 bits at a time
  bool all = false;
  for (int iter = 0;; ++iter) {
    if (iter > 12) return set_err(APEX_ELIMIT, "ground-truth narrowing did not converge");
    P.mode = 0;
    APEX_CU(cudaMemsetAsync(P.hist, 0, (65536 + 256) * sizeof(unsigned), s));
    APEX_CU(cudaMemsetAsync(d_work, 0, sizeof(unsigned), s));
    gt_pass_kernel<<<grid, 256, 0, s>>>(P);
    gt_kth_kernel<<<1, 32, 0, s>>>(P.hist, (unsigned long long)q->k, d_kth);
    launches += 2;
    long long kth[2];
    APEX_CU(cudaMemcpyAsync(kth, d_kth, sizeof(kth), cudaMemcpyDeviceToHost, s));
    APEX_CU(cudaStreamSynchronize(s));
    const long long B = kth[0];
    if (B < 0) {  // fewer than j admitted products: all of them are the answer (first pass: all feasible)
      all = true;
      break;
    }
    if ((unsigned long long)kth[1] <= cap) {  // bound found: collect
      if (!P.tie) {
        P.base = bin_edge((unsigned)B, P.base, P.shift);
        P.shift = 63;  // collect admits key >= base (every key lands in bin 0 or 1)
      } else {
        const unsigned long long glo = P.gbase + ((unsigned long long)(65534 - std::min<long long>(B, 65534)) << P.gshift);
        const unsigned long long ghi = glo + (1ull << P.gshift);
        if (ghi > glo && ghi < P.glimit) P.glimit = ghi;
      }
      break;
    }
    if (!P.tie) {
      const unsigned long long edge = bin_edge((unsigned)B, P.base, P.shift);
      if (B == 65535) {
        unsigned s2 = P.shift;
        while (s2 < 63 && ((~0ull - edge) >> s2) >= 65535ull) ++s2;
        P.base = edge;
        P.shift = s2;
      } else if (P.shift == 0) {
        P.tie = 1;
        P.tie_key = edge;
        P.gbase = q->start;
        P.glimit = q->end;
        unsigned gs = 0;
        while (gs < 63 && (span >> gs) >= 65535ull) ++gs;
        P.gshift = gs;
      } else {
        P.base = edge;
        P.shift = P.shift >= 16 ? P.shift - 16 : 0;
      }
    } else {
      const unsigned long long glo = P.gbase + ((unsigned long long)(65534 - std::min<long long>(B, 65534)) << P.gshift);
      const unsigned long long ghi = glo + (1ull << P.gshift);
      if (ghi > glo && ghi < P.glimit) P.glimit = ghi;
      P.gbase = glo;
      P.gshift = P.gshift >= 16 ? P.gshift - 16 : 0;
    }
  }
  if (all) {  // admit every feasible product at or above the current base (the first pass: base 0, everything)
    P.shift = 63;
  }
  // collect
  P.mode = 2;
  APEX_CU(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  APEX_CU(cudaMemsetAsync(d_work, 0, sizeof(unsigned), s));
  gt_pass_kernel<<<grid, 256, 0, s>>>(P);
  ++launches;
  unsigned long long count = 0;
  APEX_CU(cudaMemcpyAsync(&count, d_count, sizeof(count), cudaMemcpyDeviceToHost, s));
  APEX_CU(cudaStreamSynchronize(s));
  if (count > cap) return set_err(APEX_ELIMIT, "ground-truth candidates exceed the buffer");
  // exact select + order + decode through the merge (candidate buffer as one source)
  apex_query_spec qm;
  std::memset(&qm, 0, sizeof(qm));
  qm.objective_task = 0;
  qm.maximize = 1;
  qm.k = q->k;
  qm.start = q->start;
  qm.end = q->end;
  apex_result r = *res;
  double* cons_keep = r.constraint_values;
  r.constraint_values = nullptr;
  apex_stats mst;
  APEX_TRY(merge_impl(c, &qm, 1, c->d_gt_buf.as<Entry>(), nullptr, 1, (int64_t)count, span, &r, &mst));
  const int n = (int)r.n;
  // the oracle's objective / constraint values of the selected products
  if (n > 0) {
    DBuf dg, dv;
    APEX_TRY(dg.ensure((size_t)n * 8));
    APEX_TRY(dv.ensure((size_t)n * 8 * (1 + q->n_constraints)));
    APEX_CU(cudaMemcpyAsync(dg.p, r.global_index, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    gt_values_kernel<<<(n + 127) / 128, 128, 0, s>>>(P, dg.as<unsigned long long>(), n, c->d_goff.as<unsigned long long>(),
                                                     (int)c->rx.size(), dv.as<double>(), dv.as<double>() + n);
    ++launches;
    APEX_CU(cudaMemcpyAsync(r.objective, dv.p, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    if (q->n_constraints)
      APEX_CU(cudaMemcpyAsync(cons_keep, dv.as<double>() + n, (size_t)n * 8 * q->n_constraints, cudaMemcpyDeviceToHost, s));
    APEX_CU(cudaStreamSynchronize(s));
    dg.release();
    dv.release();
  }
  r.constraint_values = cons_keep;
  r.candidates = (int64_t)count;
  r.discarded = (int64_t)std::min<uint64_t>((uint64_t)q->k, span) - n;
  *res = r;
  if (stats) {
    stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    stats->kernel_launches = launches + mst.kernel_launches;
    stats->candidates = (int64_t)count;
  }
  return APEX_OK;
}

// ===========================================================================
// BatchTrace accounting of the chain-of-batches variant (trace.cuh)
// ===========================================================================

int apex_batch_trace(apex_ctx* c, const apex_query_spec* q, const uint64_t* batch_end, int32_t n_batches,
                     int64_t* new_out, int64_t* carried_out) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, true));
  APEX_TRY(validate_queries(c, q, 1));
  if (n_batches < 0 || (n_batches > 0 && (!batch_end || !new_out || !carried_out)))
    return set_err(APEX_EINVAL, "bad batch-trace arguments");
  if (q->n_constraints > kMaxCons) return set_err(APEX_ELIMIT, "more than 32 constraints in a query");
  for (int m = 0; m < q->n_constraints; ++m)
    if (q->constraints[m].task < 0 || q->constraints[m].task >= c->n_tasks) return set_err(APEX_ETASK, "unknown task index");
  uint64_t prev = q->start;
  for (int i = 0; i < n_batches; ++i) {
    if (batch_end[i] < prev || batch_end[i] > q->end) return set_err(APEX_EINVAL, "batch ends must ascend inside the range");
    prev = batch_end[i];
  }
  const int64_t k = q->k;
  if (k == 0) {
    for (int i = 0; i < n_batches; ++i) new_out[i] = carried_out[i] = 0;
    return APEX_OK;
  }
  const uint64_t kSub = 1ull << 20;  // products evaluated per launch
  const uint64_t cap = kSub + (uint64_t)k;
  uint64_t P_max = 1;
  while (P_max < cap) P_max <<= 1;
  DBuf buf, misc;
  APEX_TRY(buf.ensure((size_t)P_max * sizeof(TEntry)));
  APEX_TRY(misc.ensure(64));
  unsigned long long* d_count = misc.as<unsigned long long>();
  unsigned long long* d_orig = d_count + 1;
  unsigned* d_work = reinterpret_cast<unsigned*>(d_count + 2);
  cudaStream_t s = c->stream;
  TraceEval E;
  std::memset(&E, 0, sizeof(E));
  E.rx = c->d_rx.as<DevReaction>();
  E.values = c->d_values.as<float>();
  E.n_pairs = c->n_pairs;
  E.biases = c->d_biases.as<double>();
  E.obj = q->objective_task;
  E.maximize = q->maximize ? 1 : 0;
  E.n_cons = q->n_constraints;
  for (int m = 0; m < q->n_constraints; ++m) {
    E.cons_task[m] = q->constraints[m].task;
    E.cons_lo[m] = q->constraints[m].lower;
    E.cons_hi[m] = q->constraints[m].upper;
  }
  E.out = buf.as<TEntry>();
  E.count = d_count;
  E.cap = cap;
  E.work = d_work;
  int64_t max_last = 1;
  for (const auto& R : c->rx) max_last = std::max<int64_t>(max_last, R.size[R.c - 1]);
  const size_t small_smem = 4096 * sizeof(TEntry);
  APEX_CU(cudaFuncSetAttribute((const void*)trace_sort_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)small_smem));
  uint64_t carry = 0;
  prev = q->start;
  for (int i = 0; i < n_batches; ++i) {
    const uint64_t a = prev, b = batch_end[i];
    prev = b;
    if (carry) {
      trace_origin_kernel<<<(unsigned)((carry + 255) / 256), 256, 0, s>>>(buf.as<TEntry>(), (unsigned)carry, 0, nullptr);
    }
    for (uint64_t a2 = a; a2 < b; a2 += kSub) {
      const uint64_t b2 = std::min(b, a2 + kSub);
      Plan* plan = nullptr;
      APEX_TRY(build_plan(c, a2, b2, 32, 1, plan, max_last));
      E.tiles = plan->d_tiles.as<Tile>();
      E.n_tiles = (unsigned)plan->tiles.size();
      E.a = a2;
      E.b = b2;
      E.worst = carry == (uint64_t)k ? buf.as<TEntry>() + (k - 1) : nullptr;
      const unsigned long long c0 = carry;
      APEX_CU(cudaMemcpyAsync(d_count, &c0, 8, cudaMemcpyHostToDevice, s));
      APEX_CU(cudaMemsetAsync(d_work, 0, sizeof(unsigned), s));
      trace_eval_kernel<<<c->sm_count * 8, 256, 0, s>>>(E);
      APEX_CU(cudaGetLastError());
      unsigned long long total = 0;
      APEX_CU(cudaMemcpyAsync(&total, d_count, 8, cudaMemcpyDeviceToHost, s));
      APEX_CU(cudaStreamSynchronize(s));
      if (total > cap) return set_err(APEX_ELIMIT, "batch-trace candidate buffer overflow");
      if (total > carry) {  // new candidates: order carry + candidates best-first
        uint64_t P = 1;
        while (P < total) P <<= 1;
        if (P <= 4096) {
          trace_sort_small_kernel<<<1, 1024, small_smem, s>>>(buf.as<TEntry>(), (unsigned)total, (unsigned)P);
        } else {
          trace_pad_kernel<<<(unsigned)((P - total + 255) / 256), 256, 0, s>>>(buf.as<TEntry>(), (unsigned)total, (unsigned)P);
          for (uint64_t size = 2; size <= P; size <<= 1)
            for (uint64_t stride = size >> 1; stride > 0; stride >>= 1)
              trace_sort_step_kernel<<<(unsigned)((P / 2 + 255) / 256), 256, 0, s>>>(buf.as<TEntry>(), (unsigned)P,
                                                                                     (unsigned)size, (unsigned)stride);
        }
        APEX_CU(cudaGetLastError());
      }
      carry = std::min<uint64_t>((uint64_t)k, total);
    }
    unsigned long long n_new = 0;
    if (carry) {
      APEX_CU(cudaMemsetAsync(d_orig, 0, 8, s));
      trace_origin_kernel<<<(unsigned)((carry + 255) / 256), 256, 0, s>>>(buf.as<TEntry>(), (unsigned)carry, 1, d_orig);
      APEX_CU(cudaMemcpyAsync(&n_new, d_orig, 8, cudaMemcpyDeviceToHost, s));
      APEX_CU(cudaStreamSynchronize(s));
    }
    new_out[i] = (int64_t)n_new;
    carried_out[i] = (int64_t)carry - (int64_t)n_new;
  }
  buf.release();
  misc.release();
  return APEX_OK;
}

// ===========================================================================
// K8: the factorizer's hierarchy encoding on the device (k8.cuh)
// ===========================================================================

int apex_encode_hierarchy(apex_ctx* c, const apex_mlp_shape* nets, const double* params, int64_t n_params,
                          const uint8_t* token_bytes, const int64_t* token_off, int64_t n_syn, const uint8_t* salt,
                          int32_t salt_len, int32_t p, double feature_scale, const int64_t* member_ids, int64_t n_pairs,
                          const int64_t* rg_offsets, int32_t n_rg, const int32_t* rg_parent, const int64_t* rx_offsets,
                          int32_t n_rx, int32_t d, int32_t d_u, double* u_out, double* h_s_out, double* h_r_out,
                          double* h_t_out, double* features_out) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (!nets || !params || !token_bytes || !token_off || n_syn < 1 || !member_ids || n_pairs < 0 || !rg_offsets ||
      n_rg < 1 || !rg_parent || !rx_offsets || n_rx < 1 || p < 1 || d < 1 || d_u < 1 || salt_len < 0 || salt_len > 100)
    return set_err(APEX_EINVAL, "bad encode_hierarchy arguments");
  // networks: synthon, rg_phi, rg_rho, rx_phi, rx_rho, value, key; flat params W0, b0, W1, b1, ... per net
  int64_t need = 0;
  std::vector<int64_t> net_off(8, 0);
  for (int k = 0; k < 7; ++k) {
    const apex_mlp_shape& S = nets[k];
    if (S.n_layers < 1 || S.n_layers > 6) return set_err(APEX_EINVAL, "MLP layer count out of range");
    for (int i = 0; i < S.n_layers; ++i) {
      if (S.dims[i] < 1 || S.dims[i + 1] < 1) return set_err(APEX_EINVAL, "bad MLP dims");
      need += (int64_t)S.dims[i] * S.dims[i + 1] + S.dims[i + 1];
    }
    net_off[k + 1] = need;
  }
  if (need != n_params) return set_err(APEX_EINVAL, "parameter count does not match the network shapes");
  const int d_s = nets[0].dims[nets[0].n_layers], d_r = nets[2].dims[nets[2].n_layers], d_t = nets[4].dims[nets[4].n_layers];
  if (nets[0].dims[0] != p || nets[1].dims[0] != d_s || nets[3].dims[0] != d_r || nets[5].dims[0] != d_s ||
      nets[5].dims[nets[5].n_layers] != d_u || nets[6].dims[0] != d_r + d_t ||
      nets[6].dims[nets[6].n_layers] != d * d_u || nets[1].dims[nets[1].n_layers] != nets[2].dims[0] ||
      nets[3].dims[nets[3].n_layers] != nets[4].dims[0])
    return set_err(APEX_EINVAL, "network shapes do not chain (synthon -> deep sets -> value / key -> u)");
  if (rg_offsets[n_rg] != n_pairs || rx_offsets[n_rx] != n_rg) return set_err(APEX_EINVAL, "bad hierarchy offsets");
  for (int64_t i = 0; i < n_pairs; ++i)
    if (member_ids[i] < 0 || member_ids[i] >= n_syn) return set_err(APEX_EINVAL, "member id out of range");
  cudaStream_t st = c->stream;
  DBuf dp, dtok, dtoff, dsalt, dmem, drg, dpar, drx, feat, hs, hr, ht, v, kin, kf, t1, t2;
  auto up = [&](DBuf& b, const void* src, size_t bytes) -> int {
    APEX_TRY(b.ensure(std::max<size_t>(bytes, 8)));
    if (bytes) APEX_CU(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, st));
    return APEX_OK;
  };
  APEX_TRY(up(dp, params, (size_t)n_params * 8));
  APEX_TRY(up(dtok, token_bytes, (size_t)token_off[n_syn]));
  APEX_TRY(up(dtoff, token_off, (size_t)(n_syn + 1) * 8));
  APEX_TRY(up(dsalt, salt, (size_t)salt_len));
  APEX_TRY(up(dmem, member_ids, (size_t)n_pairs * 8));
  APEX_TRY(up(drg, rg_offsets, (size_t)(n_rg + 1) * 8));
  APEX_TRY(up(dpar, rg_parent, (size_t)n_rg * 4));
  APEX_TRY(up(drx, rx_offsets, (size_t)(n_rx + 1) * 8));
  APEX_TRY(feat.ensure((size_t)n_syn * p * 8));
  k8_features_kernel<<<(unsigned)((n_syn + 127) / 128), 128, 0, st>>>(dtok.as<unsigned char>(), dtoff.as<long long>(), n_syn,
                                                                     dsalt.as<unsigned char>(), salt_len, p, feature_scale,
                                                                     feat.as<double>());
  APEX_CU(cudaGetLastError());
  // one MLP (tanh between layers, none after the last) over M rows of X
  auto mlp = [&](int k, const double* X, int ldx, const long long* gather, int64_t M, DBuf& out) -> int {
    const apex_mlp_shape& S = nets[k];
    const double* w = dp.as<double>() + net_off[k];
    const double* x = X;
    int ld = ldx;
    const long long* gth = gather;
    for (int i = 0; i < S.n_layers; ++i) {
      const int K = S.dims[i], N = S.dims[i + 1];
      const bool last = i == S.n_layers - 1;
      DBuf& dst = last ? out : ((i & 1) ? t2 : t1);
      APEX_TRY(dst.ensure((size_t)std::max<int64_t>(M, 1) * N * 8));
      if (M > 0) {
        dim3 grid((unsigned)((N + kGemmTile - 1) / kGemmTile), (unsigned)((M + kGemmTile - 1) / kGemmTile));
        k8_gemm_kernel<<<grid, 256, 0, st>>>(x, ld, gth, M, K, w, w + (int64_t)K * N, N, last ? 0 : 1, dst.as<double>(), N);
        APEX_CU(cudaGetLastError());
      }
      w += (int64_t)K * N + N;
      x = dst.as<double>();
      ld = N;
      gth = nullptr;
    }
    return APEX_OK;
  };
  // h_s = synthon MLP(features)
  APEX_TRY(mlp(0, feat.as<double>(), p, nullptr, n_syn, hs));
  // h_r = DeepSet(h_s[member_ids], rg_offsets); h_t = DeepSet(h_r, rx_offsets)
  DBuf phi_r, pool_r, phi_t, pool_t;
  APEX_TRY(mlp(1, hs.as<double>(), d_s, dmem.as<long long>(), n_pairs, phi_r));
  const int dphr = nets[1].dims[nets[1].n_layers], dpht = nets[3].dims[nets[3].n_layers];
  APEX_TRY(pool_r.ensure((size_t)n_rg * dphr * 8));
  k8_segment_mean_kernel<<<n_rg, 64, 0, st>>>(phi_r.as<double>(), dphr, drg.as<long long>(), pool_r.as<double>());
  APEX_TRY(mlp(2, pool_r.as<double>(), dphr, nullptr, n_rg, hr));
  APEX_TRY(mlp(3, hr.as<double>(), d_r, nullptr, n_rg, phi_t));
  APEX_TRY(pool_t.ensure((size_t)n_rx * dpht * 8));
  k8_segment_mean_kernel<<<n_rx, 64, 0, st>>>(phi_t.as<double>(), dpht, drx.as<long long>(), pool_t.as<double>());
  APEX_TRY(mlp(4, pool_t.as<double>(), dpht, nullptr, n_rx, ht));
  // v = value MLP(h_s); K = key MLP([h_r, h_t[parent]])
  APEX_TRY(mlp(5, hs.as<double>(), d_s, nullptr, n_syn, v));
  APEX_TRY(kin.ensure((size_t)n_rg * (d_r + d_t) * 8));
  k8_key_input_kernel<<<n_rg, 128, 0, st>>>(hr.as<double>(), d_r, ht.as<double>(), d_t, dpar.as<int>(), n_rg, kin.as<double>());
  APEX_TRY(mlp(6, kin.as<double>(), d_r + d_t, nullptr, n_rg, kf));
  // u[p] = v[member[p]] @ K[j]^T
  APEX_TRY(c->d_u_res.ensure((size_t)std::max<int64_t>(n_pairs, 1) * d * 8));
  const size_t ksm = (size_t)d * d_u * 8;
  if (ksm > 200 * 1024) return set_err(APEX_ELIMIT, "key matrix too large for shared memory");
  APEX_CU(cudaFuncSetAttribute((const void*)k8_pairs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm));
  k8_pairs_kernel<<<dim3(n_rg, 8), 256, ksm, st>>>(v.as<double>(), d_u, kf.as<double>(), d, drg.as<long long>(),
                                                   dmem.as<long long>(), c->d_u_res.as<double>());
  APEX_CU(cudaGetLastError());
  c->u_res_pairs = n_pairs;
  c->u_res_d = d;
  auto down = [&](double* dst, const DBuf& b, size_t bytes) -> int {
    if (dst && bytes) APEX_CU(cudaMemcpyAsync(dst, b.p, bytes, cudaMemcpyDeviceToHost, st));
    return APEX_OK;
  };
  APEX_TRY(down(u_out, c->d_u_res, (size_t)n_pairs * d * 8));
  APEX_TRY(down(h_s_out, hs, (size_t)n_syn * d_s * 8));
  APEX_TRY(down(h_r_out, hr, (size_t)n_rg * d_r * 8));
  APEX_TRY(down(h_t_out, ht, (size_t)n_rx * d_t * 8));
  APEX_TRY(down(features_out, feat, (size_t)n_syn * p * 8));
  APEX_CU(cudaStreamSynchronize(st));
  for (DBuf* b : {&dp, &dtok, &dtoff, &dsalt, &dmem, &drg, &dpar, &drx, &feat, &hs, &hr, &ht, &v, &kin, &kf, &t1, &t2,
                  &phi_r, &pool_r, &phi_t, &pool_t})
    b->release();
  return APEX_OK;
}

// K1 from the resident K8 output (no host copy of u): the table becomes resident.
int apex_precompute_resident(apex_ctx* c, const double* head_w, const double* head_b, int32_t n_tasks, float* values_out) {
  APEX_LOCK(c);
  APEX_TRY(check_ctx(c, false));
  if (!c->u_res_pairs || !head_w || !head_b || n_tasks < 1) return set_err(APEX_ESTATE, "no resident pair matrix (run apex_encode_hierarchy)");
  const int64_t n_pairs = c->u_res_pairs;
  const int d = c->u_res_d;
  for (int t = 0; t < n_tasks; ++t)
    if (!std::isfinite(head_b[t])) return set_err(APEX_EINVAL, "non-finite head bias");
  DBuf dw;
  APEX_TRY(dw.ensure((size_t)n_tasks * d * sizeof(double)));
  APEX_TRY(c->d_values.ensure(std::max<size_t>(1, (size_t)n_tasks * n_pairs) * sizeof(float)));
  APEX_TRY(c->d_biases.ensure(n_tasks * sizeof(double)));
  APEX_CU(cudaMemcpyAsync(dw.p, head_w, (size_t)n_tasks * d * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  APEX_CU(cudaMemcpyAsync(c->d_biases.p, head_b, n_tasks * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const bool host_heads = n_tasks == 11 && d == 64 && c->opt_pre_rows == 2;
  int rc = apex_precompute_device(c, c->d_u_res.as<double>(), n_pairs, d, host_heads ? head_w : dw.as<double>(), n_tasks,
                                  c->d_values.as<float>());
  if (rc != APEX_OK) return rc;
  if (values_out && n_pairs > 0)
    APEX_CU(cudaMemcpyAsync(values_out, c->d_values.p, (size_t)n_tasks * n_pairs * sizeof(float), cudaMemcpyDeviceToHost,
                            c->stream));
  APEX_CU(cudaStreamSynchronize(c->stream));
  dw.release();
  c->biases.assign(head_b, head_b + n_tasks);
  c->n_tasks = n_tasks;
  c->n_pairs = n_pairs;
  c->table_loaded = true;
  c->corners_ok = false;
  return APEX_OK;
}

// ===========================================================================
// Multi-GPU context (one process, one host thread, N devices)
// ===========================================================================
// Shards the index range of every query batch into N contiguous g ranges, one
// per device; each device runs its exact local top-k and exports it (padded
// [query][stride] entries) into its own HBM; the merge context on the first
// device waits on the shards' events and runs the exact merge with the
// gather FUSED into its load kernel: merge_load_kernel reads every shard's
// entries through peer pointers over NVLink (no staging copy, no separate
// collective).  Without peer access the entries are staged with
// cudaMemcpyPeerAsync first.  One host sync per batch; a shard whose candidate
// buffer overflowed re-runs exactly and the merge is repeated.
}  // extern "C"

struct apex_multi {
  std::vector<int> dev;               // device of each shard
  std::vector<apex_ctx*> shard;       // local-step context per shard
  apex_ctx* merge = nullptr;          // merge + materialization context (first device)
  std::vector<DBuf> exp;              // per shard: exported entries (on the shard's device)
  std::vector<cudaEvent_t> done;      // per shard: local step + export enqueued
  DBuf d_srcs, d_stage;               // first device: shard pointer array / staged entries
  HBuf h_srcs;
  bool peer = true;
  std::recursive_mutex mu;
};

extern "C" {

static int multi_create(int32_t n_devices, const int32_t* device_ids, apex_multi* m);

int apex_multi_create(int32_t n_devices, const int32_t* device_ids, apex_multi** out) {
  if (!out || n_devices < 1 || !device_ids) return set_err(APEX_EINVAL, "bad multi-device arguments");
  *out = nullptr;
  apex_multi* m = new apex_multi();
  const int rc = multi_create(n_devices, device_ids, m);
  if (rc != APEX_OK) {
    const std::string err = t_err;
    apex_multi_destroy(m);
    t_err = err;
    return rc;
  }
  *out = m;
  return APEX_OK;
}

static int multi_create(int32_t n_devices, const int32_t* device_ids, apex_multi* m) {
  for (int i = 0; i < n_devices; ++i) {
    apex_ctx* c = nullptr;
    APEX_TRY(apex_ctx_create(device_ids[i], nullptr, &c));
    m->shard.push_back(c);
    m->dev.push_back(device_ids[i]);
    m->exp.emplace_back();
    cudaEvent_t e = nullptr;
    APEX_CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m->done.push_back(e);
  }
  APEX_TRY(apex_ctx_create(device_ids[0], nullptr, &m->merge));
  for (int i = 1; i < n_devices; ++i) {
    if (device_ids[i] == device_ids[0]) continue;
    int can = 0;
    APEX_CU(cudaDeviceCanAccessPeer(&can, device_ids[0], device_ids[i]));
    if (!can) {
      m->peer = false;
      continue;
    }
    APEX_CU(cudaSetDevice(device_ids[0]));
    const cudaError_t e = cudaDeviceEnablePeerAccess(device_ids[i], 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return set_err(APEX_ECUDA, std::string("peer access: ") + cudaGetErrorString(e));
  }
  return APEX_OK;
}

void apex_multi_destroy(apex_multi* m) {
  if (!m) return;
  for (size_t i = 0; i < m->shard.size(); ++i) {
    cudaSetDevice(m->dev[i]);
    if (m->shard[i]) cudaStreamSynchronize(m->shard[i]->stream);
    if (i < m->exp.size()) m->exp[i].release();
    if (i < m->done.size() && m->done[i]) cudaEventDestroy(m->done[i]);
  }
  if (m->merge) {
    cudaSetDevice(m->merge->device);
    cudaStreamSynchronize(m->merge->stream);
    m->d_srcs.release();
    m->d_stage.release();
  }
  m->h_srcs.release();
  for (apex_ctx* c : m->shard) apex_ctx_destroy(c);
  if (m->merge) apex_ctx_destroy(m->merge);
  delete m;
}

int apex_multi_load_library(apex_multi* m, const apex_reaction* rx, int32_t n_rx, int64_t n_pairs) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  for (apex_ctx* c : m->shard) APEX_TRY(apex_load_library(c, rx, n_rx, n_pairs));
  return apex_load_library(m->merge, rx, n_rx, n_pairs);
}

int apex_multi_load_table(apex_multi* m, const float* values, const double* biases, int32_t n_tasks, int64_t n_pairs) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  for (apex_ctx* c : m->shard) APEX_TRY(apex_load_table(c, values, biases, n_tasks, n_pairs));
  return apex_load_table(m->merge, values, biases, n_tasks, n_pairs);
}

// K1 once, on the first device; the table then becomes resident on every device.
int apex_multi_load_cache(apex_multi* m, const double* u, int64_t n_pairs, int32_t d, const double* head_w,
                          const double* head_b, int32_t n_tasks, float* values_out) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  std::vector<float> own;
  float* v = values_out;
  if (!v) {
    own.resize((size_t)std::max<int64_t>(n_tasks, 1) * std::max<int64_t>(n_pairs, 1));
    v = own.data();
  }
  APEX_TRY(apex_load_cache(m->merge, u, n_pairs, d, head_w, head_b, n_tasks, v));
  for (apex_ctx* c : m->shard) APEX_TRY(apex_load_table(c, v, head_b, n_tasks, n_pairs));
  return APEX_OK;
}

int apex_multi_set_option(apex_multi* m, const char* name, int64_t value) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  for (apex_ctx* c : m->shard) APEX_TRY(apex_set_option(c, name, value));
  return APEX_OK;
}

int apex_multi_query(apex_multi* m, const apex_query_spec* qs, int32_t nq, apex_result* res, apex_stats* stats) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  std::lock_guard<std::recursive_mutex> lk(m->mu);
  apex_ctx* M = m->merge;
  APEX_TRY(check_ctx(M, true));
  APEX_TRY(validate_queries(M, qs, nq));
  if (nq > 0 && !res) return set_err(APEX_EINVAL, "null results");
  for (int i = 0; i < nq; ++i)
    if (!res[i].global_index || !res[i].objective || !res[i].constraint_values || !res[i].reaction || !res[i].digits)
      return set_err(APEX_EINVAL, "apex_multi_query needs caller-allocated result arrays");
  const auto t0 = std::chrono::steady_clock::now();
  apex_stats agg;
  std::memset(&agg, 0, sizeof(agg));
  std::vector<int> order(nq);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return qs[a].start != qs[b].start ? qs[a].start < qs[b].start : qs[a].end < qs[b].end;
  });
  const int N = (int)m->shard.size();
  size_t g0 = 0;
  while (g0 < order.size()) {
    size_t g1 = g0 + 1;
    while (g1 < order.size() && qs[order[g1]].start == qs[order[g0]].start && qs[order[g1]].end == qs[order[g0]].end) ++g1;
    std::vector<apex_query_spec> grp;
    std::vector<int> live;
    int64_t stride = 1;
    for (size_t i = g0; i < g1; ++i) {
      const apex_query_spec& q = qs[order[i]];
      if (q.k > 0 && q.end > q.start) {
        grp.push_back(q);
        live.push_back(order[i]);
        stride = std::max<int64_t>(stride, q.k);
      } else {
        apex_result& r = res[order[i]];
        r.n = 0;
        r.scanned = q.end - q.start;
        r.discarded = 0;
        r.candidates = r.admitted = 0;
        r.full_predicate = 0;
      }
    }
    g0 = g1;
    if (grp.empty()) continue;
    const int ng = (int)grp.size();
    const uint64_t S = grp[0].start, E = grp[0].end, span = E - S;
    const size_t blk = (size_t)ng * (size_t)stride * sizeof(Entry);
    // local steps: every shard enqueued before any host wait
    std::vector<int> used;
    for (int i = 0; i < N; ++i) {
      const uint64_t a = S + (uint64_t)(((unsigned __int128)span * (unsigned)i) / (unsigned)N);
      const uint64_t b = S + (uint64_t)(((unsigned __int128)span * (unsigned)(i + 1)) / (unsigned)N);
      if (a == b) continue;
      apex_ctx* c = m->shard[i];
      APEX_CU(cudaSetDevice(m->dev[i]));
      APEX_TRY(m->exp[i].ensure(blk));
      std::vector<apex_query_spec> local = grp;
      for (auto& q : local) {
        q.start = a;
        q.end = b;
      }
      APEX_TRY(local_enqueue(c, local.data(), ng, m->exp[i].as<Entry>(), (unsigned long long)stride));
      APEX_CU(cudaEventRecord(m->done[i], c->stream));
      used.push_back(i);
    }
    std::vector<apex_result> rg(ng);
    for (int j = 0; j < ng; ++j) rg[j] = res[live[j]];
    for (int attempt = 0;; ++attempt) {
      APEX_CU(cudaSetDevice(M->device));
      const int ns = (int)used.size();
      for (int i : used) APEX_CU(cudaStreamWaitEvent(M->stream, m->done[i], 0));
      apex_stats st;
      if (m->peer) {
        APEX_TRY(m->h_srcs.ensure(ns * sizeof(void*)));
        APEX_TRY(m->d_srcs.ensure(ns * sizeof(void*)));
        APEX_CU(cudaStreamSynchronize(M->stream));  // the pinned pointer block is reused
        for (int j = 0; j < ns; ++j) m->h_srcs.as<const Entry*>()[j] = m->exp[used[j]].as<Entry>();
        APEX_CU(cudaMemcpyAsync(m->d_srcs.p, m->h_srcs.p, ns * sizeof(void*), cudaMemcpyHostToDevice, M->stream));
        APEX_TRY(merge_impl(M, grp.data(), ng, nullptr, m->d_srcs.as<const Entry*>(), ns, stride, span, rg.data(), &st));
      } else {
        APEX_TRY(m->d_stage.ensure((size_t)ns * blk));
        for (int j = 0; j < ns; ++j)
          APEX_CU(cudaMemcpyPeerAsync(m->d_stage.as<unsigned char>() + (size_t)j * blk, M->device,
                                      m->exp[used[j]].p, m->dev[used[j]], blk, M->stream));
        APEX_TRY(merge_impl(M, grp.data(), ng, m->d_stage.as<Entry>(), nullptr, ns, stride, span, rg.data(), &st));
      }
      agg.select_ms += st.select_ms;
      agg.kernel_launches += st.kernel_launches;
      agg.d2h_bytes += st.d2h_bytes;
      // validate every shard once (overflow => exact re-run + re-export,
      // then one more merge over the now-valid entries)
      if (attempt > 0) break;
      bool again = false;
      for (int i : used) {
        APEX_CU(cudaSetDevice(m->dev[i]));
        int rr = 0;
        APEX_TRY(local_finish(m->shard[i], nullptr, &rr));
        if (rr) APEX_CU(cudaEventRecord(m->done[i], m->shard[i]->stream));
        again = again || rr;
        const RunStats& lst = m->shard[i]->batch.st;
        agg.kernel_launches += lst.launches;
        agg.h2d_bytes += lst.h2d_bytes;
        agg.retries += lst.retries;
        agg.scan_kernel_ms = std::max<double>(agg.scan_kernel_ms, lst.scan_kernel_ms);
        agg.scan_ms = std::max<double>(agg.scan_ms, lst.ms[2]);
        for (int q = 0; q < ng; ++q) agg.candidates += (int64_t)m->shard[i]->h_ctl.as<QCtl>()[q].count;
      }
      if (!again) break;
    }
    for (int j = 0; j < ng; ++j) res[live[j]] = rg[j];
  }
  agg.total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (stats) *stats = agg;
  return APEX_OK;
}

int apex_multi_info(apex_multi* m, int32_t* n_devices, int32_t* peer_access) {
  if (!m) return set_err(APEX_EINVAL, "null multi-device context");
  if (n_devices) *n_devices = (int32_t)m->shard.size();
  if (peer_access) *peer_access = m->peer ? 1 : 0;
  return APEX_OK;
}

}  // extern "C"

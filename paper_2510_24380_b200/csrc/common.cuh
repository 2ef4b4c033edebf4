// common.cuh — shared device helpers for the APEX B200 kernels (sm_100a).
//
// Exactness helpers used by every kernel:
//   * ordered int32 keys over finite fp32 values (threshold bisection);
//   * order-preserving uint64 keys over fp64 scores (selection);
//   * the reference's fp64 accumulation order, ((p + x) + bias) with IEEE
//     round-to-nearest adds that the compiler may not contract or reorder
//     (engine.py:210-222, bias added last at :219).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/apex_b200.h"

namespace apexb200 {

constexpr int kMaxRg = APEX_MAX_RGROUPS;
constexpr int kMaxTests = 24;       // compiled maximum of per-product tests
constexpr int kMaxCons = 32;        // constraints per query (materialization)
constexpr int kQuant = 32;        // quantile steps per sorted column (test choice)
constexpr int kScanWarps = 8;       // warps per enumeration CTA
constexpr int kSelectThreads = 512;
constexpr uint64_t kNoTau = 0ull;   // "no admission threshold yet" (key 0 is never a finite score)
// exported-entry marker of a local result whose candidate buffer overflowed
// (the source re-runs; every merge that sees it reports the gather stale)
constexpr unsigned long long kStaleG = ~0ull - 1ull;

// Reaction descriptor in device memory (positional, csl.py:90-97).
struct DevReaction {
  int32_t c;                      // R-groups
  int32_t _pad;
  int64_t size[kMaxRg];           // synthons per R-group
  int64_t pair_off[kMaxRg];       // table row of digit 0 for each R-group
  uint64_t g_off;                 // reaction_offset
  uint64_t n_rows;                // product of sizes[0..c-2]
  int64_t pcol_off;               // offset of the last R-group in the packed objective column (16-B aligned)
  int64_t row_off;                // first row of this reaction in the row-prefix table (rows of all reactions)
};

// One enumeration tile: rows [row0, row0+nrows) x columns [col0, col0+ncols)
// of one reaction; row = mixed-radix prefix digits, column = last digit.
struct Tile {
  uint64_t row0;
  uint32_t rx;
  uint32_t nrows;
  uint32_t col0;
  uint32_t ncols;
};

// Candidate / exchange entry (== apex_entry): order-preserving key of the
// signed objective and the 64-bit global index.  Best = larger key, then
// smaller g (engine.py:246 ordering (-c, -s, g) restricted to feasible rows).
struct __align__(16) Entry {
  unsigned long long key;
  unsigned long long g;
};

// Per-query control block (device); protocol in capi.cu.
struct QCtl {
  unsigned long long tau_key;     // admission threshold (kNoTau = none)
  unsigned long long count;       // candidates appended by scans (may exceed cap)
  unsigned long long comp_count;  // entries in the compacted array
  unsigned long long sel_count;   // entries selected (<= k)
  unsigned long long bound_key;   // final compaction bound
  unsigned long long min_key;     // select scratch
  unsigned long long hist_base;   // candidate histogram: bin = min((key - base) >> shift, 65535)
  unsigned long long seed_max;    // max key among feasible samples
  unsigned long long admitted;    // products that passed admission (admission-first kernel, stats)
  unsigned int hist_shift;
  unsigned int use_full;          // 1: full-predicate kernel, 0: admission-first kernel
  unsigned int small_done;        // 1: finalize_small_kernel produced sel/sorted (large path skipped)
  unsigned int mat_done;          // 1: finalize_bucket_kernel materialized the rows (materialize_kernel skips)
  unsigned int active;            // participates in the current launch
  unsigned int tile_counter;      // scan work distribution
  unsigned int barrier;           // select grid barrier
  unsigned int out_count;         // select compaction counter
  // Tie mode (a re-run after an overflow whose k-th best key K is exact,
  // capi.cu check_batch): admission is the composite (key, g) bound
  // key > K or (key == K and g < tie_glimit), and the candidate histogram
  // bins the tied products by g (tie_gbase, tie_gshift) instead of keys.
  unsigned long long tie_key;
  unsigned long long tie_gbase;
  unsigned long long tie_glimit;
  unsigned int tie_on;
  unsigned int tie_gshift;
  // Parameters of the next run if this one overflowed (finalize_small_kernel):
  // a narrower key histogram at the k-th best bin, or tie mode at its key.
  unsigned long long nx_tau;
  unsigned long long nx_base;
  unsigned long long nx_gbase;
  unsigned long long nx_glimit;
  unsigned int nx_shift;
  unsigned int nx_tie;            // 1: tie mode at key nx_tau
  unsigned int nx_gshift;
  unsigned int nx_tie_enter;      // 1: first tie run (host sets the g range from the query range)
  unsigned int stale;             // merge: some source exported an overflowed (stale) local result
  unsigned int bail;              // sorted-column kernel gave the query up (pair budget spent): re-run full
  unsigned int fin_bar;           // bucketed finalize: CTAs of the query past the partition
  unsigned int _pad6;
  unsigned long long admit_live;  // pairs the sorted-column kernel has enumerated for the query so far
  unsigned long long bail_tau;    // the admission key when it gave up (a valid lower bound for the re-run)
  unsigned int hist[3][256];      // select histograms (triple-buffered)
};

// Preset of a re-run (one per query, uploaded by check_batch): admission
// threshold, candidate-histogram base/shift and the tie-mode fields above.
struct RunPreset {
  unsigned long long tau;
  unsigned long long base;
  unsigned long long tie_key;
  unsigned long long tie_gbase;
  unsigned long long tie_glimit;
  unsigned int shift;
  unsigned int tie_on;
  unsigned int tie_gshift;
  unsigned int full;              // 1: run the query with the full-predicate kernel (sorted-column bail-out)
};

constexpr int kHistBins = 65536;  // candidate histogram bins

// Candidate histogram bin of a key (relative to the seed threshold, see
// tau_kernel mode 0); the top bin absorbs everything above its lower edge.
__host__ __device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ unsigned hist_bin(unsigned long long key, unsigned long long base, unsigned shift) {
  const unsigned long long rel = (key - base) >> shift;
  return rel > 65535ull ? 65535u : (unsigned)rel;
}
__host__ __device__ __forceinline__ unsigned long long bin_edge(unsigned bin, unsigned long long base, unsigned shift) {
  return base + ((unsigned long long)bin << shift);
}

// Per-query parameters (device, read-only during a launch).
struct ScanQuery {
  const float* packed;            // [n_pairs][ntp] signed test columns (full-predicate kernel)
  const float* obj_col;           // [pcols] signed objective column of every last R-group (admission kernel)
  Entry* buf;                     // candidate buffer (cap entries)
  Entry* sel;                    // selected top-k (k entries, unordered)
  Entry* sorted;                  // best-first (k entries)
  unsigned int* hist;             // [kHistBins] histogram of appended keys (key >> 48)
  unsigned int* coarse;           // [256] histogram of appended keys (key >> 56)
  unsigned int* seed_hist;        // [kHistBins] histogram of feasible sampled keys
  QCtl* ctl;
  unsigned long long cap;         // capacity of buf / comp (entries)
  unsigned long long refresh_shift;  // in-kernel tau refresh every 2^refresh_shift appended candidates
  unsigned long long admit_budget;   // sorted-column kernel: pairs it may enumerate before giving the query up (~0: none)
  long long k;
  int32_t nt;                     // live tests (test 0 = objective admission)
  int32_t ntp;                    // packed row stride (floats, multiple of 4)
  int32_t maximize;
  int32_t obj_task;
  int32_t n_cons;                 // constraints (materialization order)
  int32_t slot;                   // position of the query in the caller's array
  int32_t cset;                   // sorted-column kernel: shared constraint set (pre-pass rows), -1: derived inline
  int32_t cset_off;               // its first test's row block in the pre-pass threshold array
  int32_t test_task[kMaxTests];
  int32_t test_lower[kMaxTests];  // 1: lower-bound test (y = -x), 0: upper (y = x)
  double test_beta[kMaxTests];    // bound (ignored for test 0: derived from tau)
  double test_bias[kMaxTests];
  int32_t cons_task[kMaxCons];
  // materialization outputs (device, capacity k)
  unsigned long long* out_g;
  double* out_obj;
  double* out_cons;               // [k][n_cons]
  int32_t* out_rx;
  int32_t* out_dig;               // [k][kMaxRg]
};

// ---------------------------------------------------------------------------
// fp32 ordered keys: key(-0) == key(+0) == 0, key(FLT_MAX) = 0x7f7fffff.
constexpr int64_t kKeyMax = 0x7f7fffffll;
constexpr int64_t kKeyMin = -0x7f7fffffll;

__device__ __forceinline__ int64_t fkey(float x) {
  int32_t b = __float_as_int(x);
  return b >= 0 ? (int64_t)b : -(int64_t)(b & 0x7fffffff);
}
__device__ __forceinline__ float fromkey(int64_t k) {
  return k >= 0 ? __int_as_float((int32_t)k) : __int_as_float((int32_t)((-k) | 0x80000000ll));
}

// The reference's per-product value for fixed prefix sum p: ((p + x) + b).
__device__ __forceinline__ double fx(double p, float x, double b) {
  return __dadd_rn(__dadd_rn(p, (double)x), b);
}

// fp64 score -> order-preserving key (+-0 canonicalized to +0).
__host__ __device__ __forceinline__ unsigned long long skey(double s) {
  if (s == 0.0) s = 0.0;
  unsigned long long u;
#ifdef __CUDA_ARCH__
  u = (unsigned long long)__double_as_longlong(s);
#else
  __builtin_memcpy(&u, &s, 8);
#endif
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double key_to_score(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double s;
#ifdef __CUDA_ARCH__
  s = __longlong_as_double((long long)u);
#else
  __builtin_memcpy(&s, &u, 8);
#endif
  return s;
}

__device__ __forceinline__ bool entry_better(const Entry& a, const Entry& b) {
  return a.key > b.key || (a.key == b.key && a.g < b.g);
}

// ---------------------------------------------------------------------------
// mbarrier + 1-D bulk async copy (TMA engine, SASS UBLKCP) helpers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed gpu-scope loads of values other CTAs update during a kernel
// (cheaper than volatile, which is system scope)
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t smem_u32_(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// cp.async (LDGSTS): global -> shared copies that complete in the background
// (no register holds the value); cp_async_wait_all() before reading them
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32_(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32_(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32_(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// single-lane atomic add whose result is consumed later: inline PTX so the
// compiler does not turn it into a warp-aggregated atomic, whose shuffle of
// the result waits for the atomic right away (defeating a prefetch)
__device__ __forceinline__ unsigned atom_add_u32(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

}  // namespace apexb200

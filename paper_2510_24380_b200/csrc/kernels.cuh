// kernels.cuh — sm_100a kernels of the APEX enumeration-and-retrieval path.
//
//   K1 precompute_kernel   engine.py:80-92     fp64 head_w @ u^T -> fp32 table (HBM-bound)
//   K2 pack_kernel         engine.py:195-208   per-query signed test columns, [pair][ntp]
//   K3 scan_kernel         engine.py:169-235, 290-307
//                                              fused enumeration + exact constraint /
//                                              admission predicate + candidate append
//   K5 select_kernel       engine.py:288-307 (heap), 385-386 (lexsort)
//                                              exact top-k radix select on (key, g)
//   K6 order kernels       engine.py:246      best-first order (s desc, g asc)
//   K7 materialize_kernel  csl.py:166-184, engine.py:95-101, 238-262
//                                              decode g, objective, constraint values
//
// Included exactly once (by capi.cu): one translation unit, no -rdc.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace apexb200 {

// ---------------------------------------------------------------------------
// Exact per-row thresholds.
//
// For a fixed prefix (row) the reference value of product (row, x) is
// fx(p, x, b) = ((p + x) + b) in fp64 (engine.py:214-219), monotone
// non-decreasing in the fp32 contribution x of the last R-group.  So
// "fx <= beta" holds exactly on a down-set of fp32 values and "fx >= beta" on an
// up-set; we find the boundary exactly (guess, then at most a few ulp steps,
// then bisection over the ordered fp32 keys in the rare degenerate case).
__device__ __noinline__ float thr_upper(double p, double b, double beta) {
  const double gd = __dsub_rn(__dsub_rn(beta, b), p);
  int64_t k;
  if (!(gd < 3.4028234663852886e38)) k = kKeyMax;
  else if (!(gd > -3.4028234663852886e38)) k = kKeyMin;
  else k = fkey(__double2float_rn(gd));
  if (fx(p, fromkey(k), b) <= beta) {
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
      if (k == kKeyMax) return __int_as_float(0x7f800000);
      if (fx(p, fromkey(k + 1), b) <= beta) ++k;
      else return fromkey(k);
    }
    if (fx(p, fromkey(kKeyMax), b) <= beta) return __int_as_float(0x7f800000);
    int64_t lo = k, hi = kKeyMax;  // lo qualifies, hi does not
#pragma unroll 1
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (fx(p, fromkey(mid), b) <= beta) lo = mid; else hi = mid;
    }
    return fromkey(lo);
  } else {
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
      if (k == kKeyMin) return __int_as_float(0x7fffffff);
      --k;
      if (fx(p, fromkey(k), b) <= beta) return fromkey(k);
    }
    if (!(fx(p, fromkey(kKeyMin), b) <= beta)) return __int_as_float(0x7fffffff);
    int64_t lo = kKeyMin, hi = k;  // lo qualifies, hi does not
#pragma unroll 1
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (fx(p, fromkey(mid), b) <= beta) lo = mid; else hi = mid;
    }
    return fromkey(lo);
  }
}

__device__ __noinline__ float thr_lower(double p, double b, double beta) {
  const double gd = __dsub_rn(__dsub_rn(beta, b), p);
  int64_t k;
  if (!(gd < 3.4028234663852886e38)) k = kKeyMax;
  else if (!(gd > -3.4028234663852886e38)) k = kKeyMin;
  else k = fkey(__double2float_rn(gd));
  if (fx(p, fromkey(k), b) >= beta) {
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
      if (k == kKeyMin) return __int_as_float(0xff800000);
      if (fx(p, fromkey(k - 1), b) >= beta) --k;
      else return fromkey(k);
    }
    if (fx(p, fromkey(kKeyMin), b) >= beta) return __int_as_float(0xff800000);
    int64_t lo = kKeyMin, hi = k;  // hi qualifies, lo does not
#pragma unroll 1
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (fx(p, fromkey(mid), b) >= beta) hi = mid; else lo = mid;
    }
    return fromkey(hi);
  } else {
#pragma unroll 1
    for (int it = 0; it < 3; ++it) {
      if (k == kKeyMax) return __int_as_float(0x7fffffff);
      ++k;
      if (fx(p, fromkey(k), b) >= beta) return fromkey(k);
    }
    if (!(fx(p, fromkey(kKeyMax), b) >= beta)) return __int_as_float(0x7fffffff);
    int64_t lo = k, hi = kKeyMax;  // hi qualifies, lo does not
#pragma unroll 1
    while (hi - lo > 1) {
      const int64_t mid = lo + (hi - lo) / 2;
      if (fx(p, fromkey(mid), b) >= beta) hi = mid; else lo = mid;
    }
    return fromkey(hi);
  }
}

// Debug/test entry: thresholds for arrays of (p, b, beta) (used by the GPU
// parity tests of the threshold construction itself).
__global__ void thresholds_kernel(const double* p, const double* b, const double* beta, int n,
                                  float* up, float* lo) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    up[i] = thr_upper(p[i], b[i], beta[i]);
    lo[i] = thr_lower(p[i], b[i], beta[i]);
  }
}

// ---------------------------------------------------------------------------
// K1: values[t][p] = fl32(sum_d head_w[t][d] * u[p][d]), fp64 products and
// accumulation (engine.py:82).  HBM-bound: u is read once (coalesced through
// shared memory), the table written once.  Each CTA stages 128 rows of u
// (128 x d doubles) in smem; thread (row, task-group) computes the dots.
constexpr int kPreRows = 64;
__global__ void __launch_bounds__(256) precompute_kernel(const double* __restrict__ u, int64_t n_pairs, int d,
                                                         const double* __restrict__ head_w, int n_tasks,
                                                         float* __restrict__ values) {
  extern __shared__ double psm[];
  double* w_s = psm;                      // [n_tasks][d]
  double* u_s = psm + n_tasks * d;        // [kPreRows][d+1]
  const int ld = d + 1;
  for (int i = threadIdx.x; i < n_tasks * d; i += blockDim.x) w_s[i] = head_w[i];
  for (int64_t base = (int64_t)blockIdx.x * kPreRows; base < n_pairs; base += (int64_t)gridDim.x * kPreRows) {
    const int rows = (int)(int)(n_pairs - base < kPreRows ? n_pairs - base : kPreRows);
    __syncthreads();
    const double* src = u + base * d;
    for (int i = threadIdx.x; i < rows * d; i += blockDim.x) {
      const int r = i / d, c = i - r * d;
      u_s[r * ld + c] = __ldg(src + i);
    }
    __syncthreads();
    // thread -> (row = tid % 64, task slice = tid / 64 of 4 slices)
    const int r = threadIdx.x & (kPreRows - 1);
    const int slice = threadIdx.x / kPreRows;
    if (r < rows) {
      for (int t = slice; t < n_tasks; t += blockDim.x / kPreRows) {
        double acc = 0.0;
        const double* wr = w_s + t * d;
        const double* ur = u_s + r * ld;
#pragma unroll 8
        for (int c = 0; c < d; ++c) acc = __fma_rn(wr[c], ur[c], acc);
        values[(int64_t)t * n_pairs + base + r] = __double2float_rn(acc);
      }
    }
  }
}


// K1, row-parallel form (n_tasks <= 16, d a multiple of 16): one thread per
// pair row computes every task's dot (16 independent FMA chains), u streamed
// through shared memory in 16-column chunks with the next chunk's loads in
// flight during the current chunk's FMAs (coalesced 8-byte loads, double
// buffered), the heads read as broadcast 16-byte shared loads.  Per (task,
// row) the accumulation order is the same as precompute_kernel's (c = 0..d-1).
constexpr int kPvRows = 128, kPvCols = 16, kPvTasks = 16, kPvLd = kPvCols + 2;
// NT / D > 0: compile-time task count and width (the APEX model: 11 x 64), so
// no lane work is predicated off and every head offset is an immediate
template <int NT, int D>
__global__ void __launch_bounds__(kPvRows) precompute_rows_kernel(const double* __restrict__ u, int64_t n_pairs, int d_rt,
                                                                  const double* __restrict__ head_w, int n_tasks_rt,
                                                                  float* __restrict__ values) {
  const int d = D > 0 ? D : d_rt;
  const int n_tasks = NT > 0 ? NT : n_tasks_rt;
  constexpr int TMAX = NT > 0 ? NT : kPvTasks;
  extern __shared__ __align__(16) double pv[];
  double* w_s = pv;                                   // [n_tasks][d]
  double* u_s = pv + ((n_tasks * d + 1) & ~1);        // [2][kPvRows][kPvLd], 16-B aligned rows
  const int tid = threadIdx.x;
  for (int i = tid; i < n_tasks * d; i += blockDim.x) w_s[i] = head_w[i];
  for (int64_t base = (int64_t)blockIdx.x * kPvRows; base < n_pairs; base += (int64_t)gridDim.x * kPvRows) {
    const int rows = (int)(n_pairs - base < kPvRows ? n_pairs - base : kPvRows);
    double acc[TMAX];
#pragma unroll
    for (int t = 0; t < TMAX; ++t) acc[t] = 0.0;
    double pf[kPvCols];
    // chunk element e = tid + kPvRows * k: row e / kPvCols, column e % kPvCols
#pragma unroll
    for (int k = 0; k < kPvCols; ++k) {
      const int e = tid + kPvRows * k, r = e / kPvCols, col = e % kPvCols;
      pf[k] = r < rows ? __ldg(u + (base + r) * d + col) : 0.0;
    }
    for (int c0 = 0, b = 0; c0 < d; c0 += kPvCols, b ^= 1) {
      double* ub = u_s + b * kPvRows * kPvLd;
      __syncthreads();  // the buffer's previous chunk has been consumed
#pragma unroll
      for (int k = 0; k < kPvCols; ++k) {
        const int e = tid + kPvRows * k, r = e / kPvCols, col = e % kPvCols;
        ub[r * kPvLd + col] = pf[k];
      }
      __syncthreads();
      if (c0 + kPvCols < d) {
#pragma unroll
        for (int k = 0; k < kPvCols; ++k) {
          const int e = tid + kPvRows * k, r = e / kPvCols, col = e % kPvCols;
          pf[k] = r < rows ? __ldg(u + (base + r) * d + c0 + kPvCols + col) : 0.0;
        }
      }
      const double* ur = ub + tid * kPvLd;
#pragma unroll
      for (int cc = 0; cc < kPvCols; cc += 2) {
        const double2 uv = *reinterpret_cast<const double2*>(ur + cc);
#pragma unroll
        for (int t = 0; t < TMAX; ++t) {
          if (NT > 0 || t < n_tasks) {
            const double2 wv = *reinterpret_cast<const double2*>(w_s + t * d + c0 + cc);
            acc[t] = __fma_rn(wv.x, uv.x, acc[t]);
            acc[t] = __fma_rn(wv.y, uv.y, acc[t]);
          }
        }
      }
    }
    if (tid < rows) {
#pragma unroll
      for (int t = 0; t < TMAX; ++t)
        if (NT > 0 || t < n_tasks) values[(int64_t)t * n_pairs + base + tid] = __double2float_rn(acc[t]);
    }
  }
}

// K1, TMA form (compile-time task count x width, the APEX model's 11 x 64):
// HBM-bound by design.  One persistent CTA per SM streams tiles of kBulkRows
// consecutive pair rows of u (kBulkRows x 64 doubles = 64 KB) into a
// kBulkStages-deep shared-memory ring with 2-D TMA tensor copies
// (cp.async.bulk.tensor, four 128-row x 16-column boxes per tile, 128-byte
// swizzle: the 16-byte chunk j of a box row r lands at chunk j ^ (r & 7), so
// the LDS.128 row reads of a warp are bank-conflict free without padding).
// Completion is signalled on a per-stage "full" mbarrier; every warp arrives
// on the stage's "empty" mbarrier when it has read the stage, and warp 0
// refills it after waiting on that barrier alone (no CTA-wide barrier per
// tile: the other warps run ahead on the stages already in flight).  Warp w
// owns rows (w % 4) * 32 + lane of the tile and task group w / 4 (tasks
// [6g, 6g + 6)); the head weights come straight from the kernel-parameter
// constant bank (uniform-register DFMA operands).  Per (task, row) the fp64
// FMA chain runs c = 0..63 from 0.0, the same order as the other forms, then
// rounds to fp32 (engine.py:82).
constexpr int kBulkRows = 128, kBulkStages = 3, kBulkGroups = 2, kBulkThreads = kBulkRows * kBulkGroups;
constexpr int kBulkBoxCols = 16;  // doubles per box row (128 B: the 128-byte swizzle span)
template <int NT, int D>
struct HeadParams {
  double w[NT * D];
};
template <int NT, int D>
constexpr size_t bulk_smem_bytes() {
  return 1024 + (size_t)kBulkStages * kBulkRows * D * sizeof(double) + 2 * kBulkStages * sizeof(uint64_t);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NT, int D, int G>
__device__ __forceinline__ void bulk_dots(const unsigned char* __restrict__ tile, int r, const HeadParams<NT, D>& W,
                                          int64_t n_pairs, int64_t row, float* __restrict__ values) {
  constexpr int TG = (NT + kBulkGroups - 1) / kBulkGroups;
  constexpr int T0 = G * TG, T1 = (T0 + TG < NT) ? T0 + TG : NT;
  double acc[TG];
#pragma unroll
  for (int t = 0; t < TG; ++t) acc[t] = 0.0;
  const int sw = r & 7;
#pragma unroll
  for (int box = 0; box < D / kBulkBoxCols; ++box) {
    const unsigned char* rowp = tile + ((size_t)box * kBulkRows + r) * (kBulkBoxCols * sizeof(double));
#pragma unroll
    for (int j = 0; j < kBulkBoxCols / 2; ++j) {
      const double2 uv = *reinterpret_cast<const double2*>(rowp + ((j ^ sw) << 4));
      const int c = box * kBulkBoxCols + 2 * j;
#pragma unroll
      for (int t = T0; t < T1; ++t) {
        acc[t - T0] = __fma_rn(W.w[t * D + c], uv.x, acc[t - T0]);
        acc[t - T0] = __fma_rn(W.w[t * D + c + 1], uv.y, acc[t - T0]);
      }
    }
  }
#pragma unroll
  for (int t = T0; t < T1; ++t) values[(int64_t)t * n_pairs + row] = __double2float_rn(acc[t - T0]);
}

// tmap: 2-D tensor map of u (dims {D, n_pairs}, box {16, kBulkRows}, 128-byte swizzle), built by capi.cu
template <int NT, int D>
__global__ void __launch_bounds__(kBulkThreads, 1) precompute_bulk_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                          int64_t n_pairs,
                                                                          const __grid_constant__ HeadParams<NT, D> W,
                                                                          float* __restrict__ values) {
  static_assert(kBulkGroups == 2 && D % kBulkBoxCols == 0, "bulk form: two task groups, 16-column boxes");
  constexpr uint32_t kTileBytes = kBulkRows * D * sizeof(double);
  extern __shared__ unsigned char bulk_raw[];
  // the 128-byte swizzle pattern repeats every 1024 bytes: align the ring to that
  unsigned char* ring = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(bulk_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)kBulkStages * kTileBytes);
  uint64_t* empty = full + kBulkStages;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = (warp % (kBulkRows / 32)) * 32 + lane;  // row within the tile
  const int grp = warp / (kBulkRows / 32);              // task group (warp-uniform)
  const int64_t n_tiles = (n_pairs + kBulkRows - 1) / kBulkRows;
  const int64_t grid = gridDim.x;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kBulkStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBulkThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int s) {  // one thread
    mbar_expect_tx(&full[s], kTileBytes);  // out-of-range rows of the last tile are zero-filled and counted
    unsigned char* dst = ring + (size_t)s * kTileBytes;
#pragma unroll
    for (int box = 0; box < D / kBulkBoxCols; ++box)
      tma_load_2d(dst + (size_t)box * kBulkRows * kBulkBoxCols * sizeof(double), &tmap, box * kBulkBoxCols,
                  (int)(tile * kBulkRows), &full[s]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kBulkStages; ++s) {
      const int64_t tile = blockIdx.x + s * grid;
      if (tile < n_tiles) issue(tile, s);
    }
  }
  for (int64_t it = 0;; ++it) {
    const int64_t tile = blockIdx.x + it * grid;
    if (tile >= n_tiles) break;
    const int s = (int)(it % kBulkStages);
    const uint32_t phase = (uint32_t)((it / kBulkStages) & 1);
    mbar_wait(&full[s], phase);
    const int64_t base = tile * kBulkRows;
    const unsigned char* tp = ring + (size_t)s * kTileBytes;
    if (base + r < n_pairs) {
      if (grp == 0) bulk_dots<NT, D, 0>(tp, r, W, n_pairs, base + r, values);
      else bulk_dots<NT, D, 1>(tp, r, W, n_pairs, base + r, values);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    const int64_t next = tile + kBulkStages * grid;
    if (tid == 0 && next < n_tiles) {
      mbar_wait(&empty[s], phase);  // every warp has read stage s
      fence_proxy_async();          // their generic-proxy reads before the async-proxy refill
      issue(next, s);
    }
  }
}

// 64-bit division with a 32-bit fast path (operands below 2^32)
__device__ __forceinline__ void divmod_u64(uint64_t& q, uint64_t& r, uint64_t n, uint64_t d) {
  if ((n >> 32) == 0 && (d >> 32) == 0) {
    const uint32_t n32 = (uint32_t)n, d32 = (uint32_t)d;
    q = n32 / d32;
    r = n32 - (uint32_t)q * d32;
  } else {
    q = n / d;
    r = n - q * d;
  }
}

constexpr int kWorkCtrs = 16;  // sorted-column scan: work counters, one 128-byte line each
constexpr int kWorkWords = 64 + 32 * kWorkCtrs;  // flattened-work counters of the scan launches

// ---------------------------------------------------------------------------
// Control-block init (one CTA per query).  tau0 = preset admission key
// (kNoTau normally; the final threshold of an overflowed run on re-run).
__global__ void init_ctl_kernel(const ScanQuery* __restrict__ qs, const RunPreset* __restrict__ pre,
                                unsigned use_full, unsigned* work, unsigned lazy_zero) {
  const ScanQuery& Q = qs[blockIdx.x];
  QCtl* c = Q.ctl;
  if (lazy_zero) {
    // Histograms zeroed where the last pass left counts (replaces a memset of
    // every bin of every query: 15.8 MB on C2): every fine increment comes
    // with its coarse one, so the fine blocks of the nonzero coarse bins are
    // exactly the dirty ones (the buffer is zeroed once when allocated).
    // gridDim.y CTAs per query share the 768 coarse bins (3 histograms).
    unsigned* const coarse[3] = {Q.coarse, Q.seed_hist + 2 * kHistBins, Q.seed_hist + 2 * kHistBins + 256};
    unsigned* const fine[3] = {Q.hist, Q.seed_hist, Q.seed_hist + kHistBins};
    const unsigned per = (768 + gridDim.y - 1) / gridDim.y, b0 = blockIdx.y * per, b1 = min(768u, b0 + per);
    const unsigned warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = lane_id();
    for (unsigned blk = b0 + warp; blk < b1; blk += nw) {
      const unsigned cv = __ldcg(coarse[blk >> 8] + (blk & 255));
      if (cv) {
        uint4* f = reinterpret_cast<uint4*>(fine[blk >> 8] + (blk & 255) * 256);
        for (unsigned i = lane; i < 64; i += 32) f[i] = make_uint4(0u, 0u, 0u, 0u);
        if (lane == 0) coarse[blk >> 8][blk & 255] = 0u;
      }
    }
    if (blockIdx.y != 0) return;
  }
  // the scan launches' flattened-work counters (replaces a memset node)
  if (work && blockIdx.x == 0 && threadIdx.x < kWorkWords) work[threadIdx.x] = 0u;
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&c->hist[0][0])[i] = 0u;
  // (the candidate / seed histograms are zeroed by one memset per batch)
  if (threadIdx.x == 0) {
    const RunPreset* P = pre ? pre + blockIdx.x : nullptr;
    c->tau_key = P ? P->tau : kNoTau;
    c->hist_base = P ? P->base : 0ull;
    c->hist_shift = P ? P->shift : 48u;
    c->tie_on = P ? P->tie_on : 0u;
    c->tie_key = P ? P->tie_key : 0ull;
    c->tie_gbase = P ? P->tie_gbase : 0ull;
    c->tie_glimit = P ? P->tie_glimit : ~0ull;
    c->tie_gshift = P ? P->tie_gshift : 48u;
    c->nx_tie = 0;
    c->nx_tie_enter = 0;
    c->stale = 0;
    c->use_full = use_full || (P && P->full) ? 1u : 0u;
    c->bail = 0;
    c->fin_bar = 0;
    c->admit_live = 0;
    c->bail_tau = 0;
    c->small_done = 0;
    c->mat_done = 0;
    c->seed_max = 0;
    c->admitted = 0;
    c->count = 0;
    c->comp_count = 0;
    c->sel_count = 0;
    c->bound_key = 0;
    c->min_key = ~0ull;
    c->active = 1;
    c->tile_counter = 0;
    c->barrier = 0;
    c->out_count = 0;
  }
}

// ---------------------------------------------------------------------------
// K2: packed[p][i] = (test i lower ? -v : v)[task_i][p], 0 in padding columns,
// for pair rows [row_lo, row_hi) (the R-groups K3 streams as columns).
__global__ void pack_kernel(const ScanQuery* __restrict__ qs, const float* __restrict__ values, int64_t n_pairs,
                            int64_t row_lo, int64_t row_hi) {
  const ScanQuery& Q = qs[blockIdx.y];
  if (!*(volatile unsigned*)&Q.ctl->use_full) return;
  float* dst = const_cast<float*>(Q.packed);
  const int ntp = Q.ntp;
  const int64_t n = (row_hi - row_lo) * ntp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t qd, rd;
    divmod_u64(qd, rd, (uint64_t)i, (uint64_t)ntp);  // 32-bit path for all realistic tables
    const int64_t p = row_lo + (int64_t)qd;
    const int t = (int)rd;
    float v = 0.0f;
    if (t < Q.nt) {
      v = __ldg(values + (int64_t)Q.test_task[t] * n_pairs + p);
      if (Q.test_lower[t]) v = -v;
      if (v == 0.0f) v = 0.0f;  // never -0: the packed compare reads sign bits
    }
    dst[p * ntp + t] = v;
  }
}

// ---------------------------------------------------------------------------
// Fast exact thresholds: the rounded guess fl32((beta - b) - p) is within one
// fp32 ulp of the boundary unless fp64 absorption is extreme, so two probes
// usually settle it; anything else falls back to the general search above.
__device__ __forceinline__ float next_up(float x) { return fromkey(fkey(x) + 1); }
__device__ __forceinline__ float next_down(float x) { return fromkey(fkey(x) - 1); }

__device__ __forceinline__ float thr_upper_fast(double p, double b, double beta) {
  const double gd = __dsub_rn(__dsub_rn(beta, b), p);
  if (fabs(gd) < 3.0e38) {
    const float x = __double2float_rn(gd);
    if (fx(p, x, b) <= beta) {
      if (!(fx(p, next_up(x), b) <= beta)) return x;
    } else {
      const float xd = next_down(x);
      if (fx(p, xd, b) <= beta) return xd;
    }
  }
  return thr_upper(p, b, beta);
}

__device__ __forceinline__ float thr_lower_fast(double p, double b, double beta) {
  const double gd = __dsub_rn(__dsub_rn(beta, b), p);
  if (fabs(gd) < 3.0e38) {
    const float x = __double2float_rn(gd);
    if (fx(p, x, b) >= beta) {
      if (!(fx(p, next_down(x), b) >= beta)) return x;
    } else {
      const float xu = next_up(x);
      if (fx(p, xu, b) >= beta) return xu;
    }
  }
  return thr_lower(p, b, beta);
}

// K2b: signed objective column of every reaction's last R-group, laid out at
// 16-byte aligned per-reaction offsets (TMA bulk copies need 16-B alignment).
__global__ void pack_obj_kernel(const ScanQuery* __restrict__ qs, const DevReaction* __restrict__ rx,
                                const float* __restrict__ values, int64_t n_pairs) {
  const ScanQuery& Q = qs[blockIdx.z];
  const DevReaction& R = rx[blockIdx.y];
  const int64_t n_last = R.size[R.c - 1];
  const float* v = values + (int64_t)Q.test_task[0] * n_pairs + R.pair_off[R.c - 1];
  float* dst = const_cast<float*>(Q.obj_col) + R.pcol_off;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n_last; j += (int64_t)gridDim.x * blockDim.x) {
    float y = __ldg(v + j);
    if (Q.test_lower[0]) y = -y;
    if (y == 0.0f) y = 0.0f;
    dst[j] = y;
  }
}

// ---------------------------------------------------------------------------
// K3: fused enumeration.
//
// Work unit: one warp takes one Tile (atomic work counter, dynamic balance).
// Lane l owns rows row0 + l + 32*r (r < RL).  For each owned row and each
// test i it computes an exact fp32 threshold thr[r][i] on the packed column
// value y_i, folding the fp64 prefix sum, the bias and the bound (or the
// running admission threshold tau for test 0).  Per product the work is then
// NT fp32 compares (an FSETP predicate chain) against y values broadcast from
// shared memory, where the last R-group's column block was staged by a 1-D
// TMA bulk copy (double-buffered, mbarrier completion).  Every 8 columns the
// warp votes; only if some product passed all tests (feasible AND s >= tau,
// both exact) does it take the slow path: recompute the fp64 score in the
// reference order, append (key, g) with one warp-aggregated atomic, and count
// the key in the per-query histogram that drives tau.
template <int NT>
struct Ntp { static constexpr int value = (NT + 3) / 4 * 4; };

struct ScanLaunch {
  const Tile* tiles;
  unsigned int tile_begin, tile_end;
  const DevReaction* rx;
  const float* values;
  int64_t n_pairs;
  const ScanQuery* queries;
  int cb;                 // columns per smem block (multiple of 8)
  int nq;                 // queries of this launch (<= 64)
  unsigned int* work;     // flattened (tile x query) work counter, zeroed before the launch
  int chunk;              // work items per atomic
  int vote64;             // admission kernel: 64-column pre-vote on/off
  int dense_min;          // admission kernel: admitted products of a row in a tile that flag it dense
  unsigned long long* trace;  // per-item timing records (8 words) or null
  unsigned trace_cap;         // records
  int n_ctr;              // > 1: that many work counters (work + 32 k), counter k hands out items k, k + n_ctr, ...
  unsigned nq_magic;      // ceil(2^32 / nq) when every item index < 2^26 (item_div), else 0
};

// Flattened persistent work distribution: item -> (tile = item / nq,
// query = item % nq), so the queries of a batch advance together over the
// same tiles (shared column data stays hot in L1/L2) and one launch keeps
// every SM busy however many queries there are.  Warps take `chunk` items per
// atomic; items of queries this kernel does not scan (mask) are skipped.
// item / nq by a multiply-high with the launch's reciprocal (nq <= 64; exact
// for item < 2^26, checked on the host, else a division)
__device__ __forceinline__ unsigned item_div(const ScanLaunch& L, unsigned item) {
  return L.nq_magic ? (unsigned)(((unsigned long long)item * L.nq_magic) >> 32) : item / (unsigned)L.nq;
}

struct WorkCursor {
  unsigned cur = 0, lim = 0;
  unsigned nxt = 0;      // lane 0: base of the next chunk, fetched one chunk ahead
  bool primed = false;
  unsigned sk = 0;       // static rounds taken
  unsigned k = 0, tried = 0;  // several counters: the current one, counters found exhausted
  bool tail = false;     // the item just returned is in the last window: nothing claimed ahead
};

// Several work counters (L.n_ctr > 1, each in its own 128-byte line): one
// counter's atomics from every warp of the grid serialise at its L2 slice and
// come back later than a whole item takes (ncu: the warps stalled on the
// prefetched item index); n_ctr counters over interleaved item sets keep the
// heaviest-first order and divide that queue.  A warp starts on counter
// (warp id mod n_ctr) and moves on when it is exhausted.
__device__ __forceinline__ bool next_item_multi(const ScanLaunch& L, WorkCursor& wc, unsigned long long live,
                                                unsigned lane, unsigned& q, unsigned& t) {
  const unsigned total = (L.tile_end - L.tile_begin) * (unsigned)L.nq;
  const unsigned n = (unsigned)L.n_ctr;
  if (!wc.primed) {
    wc.primed = true;
    wc.k = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % n;
    if (lane == 0) wc.nxt = atom_add_u32(L.work + 32 * wc.k, 1u);
  }
  // the last window of items (one per warp of the grid) is claimed just in
  // time: an item claimed ahead by a warp still busy with a heavy item would
  // wait behind it while other warps find the counters empty
  const unsigned long long window = (unsigned long long)gridDim.x * (blockDim.x >> 5);
  for (;;) {
    unsigned local = __shfl_sync(0xffffffffu, wc.nxt, 0);
    if (local == ~0u) {  // not claimed ahead
      if (lane == 0) wc.nxt = atom_add_u32(L.work + 32 * wc.k, 1u);
      local = __shfl_sync(0xffffffffu, wc.nxt, 0);
    }
    const unsigned long long item64 = (unsigned long long)wc.k + (unsigned long long)local * n;
    if (item64 >= total) {
      if (++wc.tried >= n) return false;
      wc.k = wc.k + 1 == n ? 0u : wc.k + 1;
      if (lane == 0) wc.nxt = atom_add_u32(L.work + 32 * wc.k, 1u);
      continue;
    }
    wc.tail = item64 + window >= total;
    if (lane == 0) wc.nxt = wc.tail ? ~0u : atom_add_u32(L.work + 32 * wc.k, 1u);  // one item ahead
    const unsigned item = (unsigned)item64;
    const unsigned tq = item_div(L, item);
    q = item - tq * (unsigned)L.nq;
    t = L.tile_begin + tq;
    if ((live >> q) & 1ull) return true;
  }
}

__device__ __forceinline__ bool next_item(const ScanLaunch& L, WorkCursor& wc, unsigned long long live, unsigned lane,
                                          unsigned& q, unsigned& t) {
  const unsigned total = (L.tile_end - L.tile_begin) * (unsigned)L.nq;
  // every item through the work counter (a static share of the rounds was
  // slower: item costs vary too much, profiles/r2_ab_static_items_rejected.log);
  // k_static stays as the hook for a static prefix
  const unsigned nw = gridDim.x * (blockDim.x >> 5);
  const unsigned wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const unsigned k_static = 0;
  for (;;) {
    unsigned item;
    if (wc.sk < k_static) {
      item = wc.sk * nw + wid;
      ++wc.sk;
    } else {
      if (!wc.primed) {
        wc.primed = true;
        if (lane == 0) wc.nxt = k_static * nw + atom_add_u32(L.work, (unsigned)L.chunk);
      }
      if (wc.cur >= wc.lim) {
        const unsigned base = __shfl_sync(0xffffffffu, wc.nxt, 0);
        if (lane == 0 && base < total) wc.nxt = k_static * nw + atom_add_u32(L.work, (unsigned)L.chunk);  // one chunk ahead
        wc.cur = base;
        wc.lim = base + (unsigned)L.chunk;
      }
      item = wc.cur++;
    }
    if (item >= total) return false;
    const unsigned tq = item_div(L, item);
    q = item - tq * (unsigned)L.nq;
    t = L.tile_begin + tq;
    if ((live >> q) & 1ull) return true;
  }
}

// Warp-aggregated histogram increment (the whole warp calls it, converged):
// lanes with on == true and the same bin add once, by their lowest lane.
// Seed products of one warp mostly share bins (16-bit key prefixes of
// near-equal top values), so this removes most same-address atomics.
__device__ __forceinline__ void hist_add_warp(unsigned int* h, unsigned bin, bool on) {
  const unsigned am = __ballot_sync(0xffffffffu, on);
  if (!on) return;
  const unsigned peers = __match_any_sync(am, bin);
  if ((int)lane_id() == __ffs(peers) - 1) atomicAdd(&h[bin], (unsigned)__popc(peers));
}

// queries of the launch that this kernel form scans
__device__ __forceinline__ unsigned long long live_mask(const ScanLaunch& L, unsigned want_full) {
  // flags written by earlier kernels of the stream: plain loads, one query per lane
  const unsigned lane = lane_id();
  unsigned long long m = 0;
  for (int q0 = 0; q0 < L.nq; q0 += 32) {
    const int q = q0 + (int)lane;
    bool ok = false;
    if (q < L.nq) {
      const QCtl* c = L.queries[q].ctl;
      ok = __ldcg(&c->active) && __ldcg(&c->use_full) == want_full;
    }
    m |= (unsigned long long)__ballot_sync(0xffffffffu, ok) << q0;
  }
  return m;
}

// 256 histogram bins, 8 per lane in blocks from the top: lane l, slot i holds
// bin 255 - 8 l - i (lane 0 the highest block).
__device__ __forceinline__ void load_bins256(const unsigned int* __restrict__ h, unsigned (&v)[8]) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __ldcg(h + (255 - 8 * (int)lane - i));
}

// Highest bin B (scanning from the top) with above + sum_{b >= B} v[b] >= k
// over 256 bins held as load_bins256 does.  Returns B or -1; above += the
// count of the bins above B (or of all); *incl_at = the count at/above B.
// One warp prefix sum over the lanes' block sums finds the block, the lane
// holding it walks its 8 bins (round 1's form scanned 8 slot groups with a
// prefix sum each: ~10x the instructions on this latency-bound chain).
__device__ __forceinline__ int kth_bins256(const unsigned (&v)[8], unsigned long long k, unsigned long long& above,
                                           unsigned long long* incl_at) {
  const unsigned lane = lane_id();
  unsigned long long blk = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) blk += v[i];
  unsigned long long incl = blk;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, off);
    if ((int)lane >= off) incl += o;
  }
  const unsigned m = __ballot_sync(0xffffffffu, above + incl >= k);
  if (!m) {
    above += __shfl_sync(0xffffffffu, incl, 31);
    return -1;
  }
  const int l = __ffs(m) - 1;
  int b = 0;
  unsigned long long run = above + incl - blk, at = 0;  // (meaningful in lane l)
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (b == 0 && run + v[i] >= k) {
      b = 256 - 8 * (int)lane - i;  // bin + 1 (0: not found yet)
      at = run + v[i];
    } else if (b == 0) {
      run += v[i];
    }
  }
  b = __shfl_sync(0xffffffffu, b, l) - 1;
  const unsigned long long run_l = __shfl_sync(0xffffffffu, run, l);
  const unsigned long long at_l = __shfl_sync(0xffffffffu, at, l);
  if (incl_at) *incl_at = at_l;
  above = run_l;
  return b;
}

// Two-level (256 coarse x 256 fine) search by ONE warp of the highest fine
// bin B with sum_{b >= B} fine[b] >= k, where coarse[c] = sum of fine bins
// c*256 .. c*256+255.  Returns B (-1 if the coarse total is below k) and, in
// *count_ge, the number of entries at/above B (or the total).  When the fine
// counts lag the coarse ones (concurrent appends) and do not reach k inside
// the chosen coarse bin, returns that coarse bin's lowest fine bin (still a
// valid bound: the coarse counts above and at it reach k).  Every level's 256
// counts are loaded at once (8 per lane): two dependent L2 round trips.
__device__ int kth_two_level(const unsigned int* __restrict__ fine, const unsigned int* __restrict__ coarse,
                             unsigned long long k, unsigned long long* count_ge) {
  unsigned v[8];
  load_bins256(coarse, v);
  unsigned long long above = 0;
  const int cbin = kth_bins256(v, k, above, nullptr);
  if (cbin < 0) {
    if (count_ge) *count_ge = above;
    return -1;
  }
  load_bins256(fine + (cbin << 8), v);
  unsigned long long at = 0;
  const int fb = kth_bins256(v, k, above, &at);
  if (fb < 0) {
    if (count_ge) *count_ge = above;
    return cbin << 8;
  }
  if (count_ge) *count_ge = at;
  return (cbin << 8) | fb;
}

// kth_two_level's search over preloaded coarse counts (vc, as load_bins256),
// returning also the count of entries in bins strictly above the returned bin
// (*above; the total when -1 is returned).  Used on a complete histogram
// (after the enumeration), where both levels agree.
__device__ int kth_two_level_above(const unsigned int* __restrict__ fine, const unsigned (&vc)[8],
                                   unsigned long long k, unsigned long long* above_out) {
  unsigned v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = vc[i];
  unsigned long long above = 0;
  const int cbin = kth_bins256(v, k, above, nullptr);
  if (cbin < 0) {
    *above_out = above;
    return -1;
  }
  load_bins256(fine + (cbin << 8), v);
  const unsigned long long above_c = above;
  const int fb = kth_bins256(v, k, above, nullptr);
  if (fb < 0) {
    *above_out = above_c;
    return cbin << 8;
  }
  *above_out = above;
  return (cbin << 8) | fb;
}

// Tie mode (QCtl): composite admission of a re-run whose k-th best key K is
// exact — products with key == K pass only below the g limit — and the
// candidate histogram over g for the tied key (better = smaller g = higher
// bin; keys above K and tied products below tie_gbase are all "above").
__device__ __forceinline__ bool tie_reject(const QCtl* ctl, unsigned long long key, unsigned long long g) {
  if (!__ldcg(&ctl->tie_on)) return false;
  const unsigned long long K = __ldcg(&ctl->tie_key);
  return key < K || (key == K && g >= __ldcg(&ctl->tie_glimit));
}
__device__ __forceinline__ unsigned cand_bin(const QCtl* ctl, unsigned long long key, unsigned long long g,
                                             unsigned long long hbase, unsigned hshift) {
  if (__ldcg(&ctl->tie_on)) {
    if (key > __ldcg(&ctl->tie_key)) return 65535u;
    const unsigned long long gb = __ldcg(&ctl->tie_gbase);
    if (g < gb) return 65535u;
    const unsigned long long rel = (g - gb) >> __ldcg(&ctl->tie_gshift);
    return rel >= 65535ull ? 0u : (unsigned)(65534ull - rel);
  }
  return hist_bin(key, hbase, hshift);
}

// In-kernel threshold refresh (one warp): tau = lower edge of the k-th best
// candidate bin, read while other warps keep appending; a stale (smaller)
// count only lowers the bound, so it stays a valid lower bound on the final
// k-th best key.
__device__ __noinline__ void refresh_tau(const ScanQuery& Q) {
  if (__ldcg(&Q.ctl->tie_on)) return;  // tie mode: the bins are g ranges of the tied key, not keys
  const int B = kth_two_level(Q.hist, Q.coarse, (unsigned long long)Q.k, nullptr);
  if (B < 0) return;
  const unsigned long long key = bin_edge((unsigned)B, Q.ctl->hist_base, Q.ctl->hist_shift);
  if (lane_id() == 0) atomicMax(&Q.ctl->tau_key, key);
}

template <int NT, int RL>
__device__ __forceinline__ bool test_cols(const float* __restrict__ ys, int j, const float (&thr)[RL][NT],
                                          bool (&pass)[RL]) {
  constexpr int NTP = Ntp<NT>::value;
  float y[NTP];
  const float4* yp = reinterpret_cast<const float4*>(ys + j * NTP);
#pragma unroll
  for (int q = 0; q < NTP / 4; ++q) {
    const float4 v = yp[q];
    y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
  }
  bool any = false;
#pragma unroll
  for (int r = 0; r < RL; ++r) {
    bool p = y[0] <= thr[r][0];
#pragma unroll
    for (int i = 1; i < NT; ++i) p = p & (y[i] <= thr[r][i]);
    pass[r] = p;
    any = any | p;
  }
  return any;
}

// Packed variant: two tests per instruction.  With t' = nextup(t) (t' = -inf
// for "no x qualifies", +inf for "all"), y <= t  <=>  fl(y - t') < 0, whose
// sign bit is exact (IEEE subtraction never rounds across zero; y is never -0
// after packing).  d = y - t' for a pair of tests is one FADD2 (fp32x2,
// FMA pipe); the pass bits are ANDed with LOP3 (ALU).
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int NT>
struct Np { static constexpr int value = (NT + 1) / 2; };

template <int NT, int RL>
__device__ __forceinline__ unsigned test_cols2(const float* __restrict__ ys, int j,
                                               const unsigned long long (&tp)[RL][Np<NT>::value],
                                               unsigned (&acc)[RL]) {
  constexpr int NTP = Ntp<NT>::value;
  constexpr int NP = Np<NT>::value;
  unsigned long long y[NTP / 2];
  const ulonglong2* yp = reinterpret_cast<const ulonglong2*>(ys + j * NTP);
#pragma unroll
  for (int q = 0; q < NTP / 4; ++q) {
    const ulonglong2 v = yp[q];
    y[2 * q] = v.x;
    y[2 * q + 1] = v.y;
  }
  unsigned any = 0;
#pragma unroll
  for (int r = 0; r < RL; ++r) {
    unsigned a = 0xffffffffu;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const unsigned long long d = fsub2(y[p], tp[r][p]);
      a = a & (unsigned)d & (unsigned)(d >> 32);
    }
    acc[r] = a;
    any = any | a;
  }
  return any;
}

// threshold t (y <= t) -> t' for the packed form
__device__ __forceinline__ float tprime(float t) {
  if (t != t) return __int_as_float(0xff800000);          // none: -inf
  if (t == __int_as_float(0x7f800000)) return t;          // all: +inf
  return next_up(t);
}

template <int NT>
constexpr int scan_min_blocks() { return NT <= 12 ? 3 : 2; }

template <int NT, int RL, int MODE>
__global__ void __launch_bounds__(kScanWarps * 32, scan_min_blocks<NT>()) scan_kernel(const ScanLaunch L) {
  constexpr int NTP = Ntp<NT>::value;
  constexpr int NP = Np<NT>::value;
  extern __shared__ __align__(128) unsigned char sm_raw[];
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  const unsigned long long live = live_mask(L, 1u);
  if (!live) return;
  WorkCursor wc;

  const int cb = L.cb;
  float* sbuf0 = reinterpret_cast<float*>(sm_raw) + (size_t)warp * 2 * cb * NTP;
  float* sbuf1 = sbuf0 + cb * NTP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_raw + (size_t)kScanWarps * 2 * cb * NTP * sizeof(float)) + warp * 2;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phase0 = 0, phase1 = 0;
  unsigned bi = 0;

  // value of padding columns: never passes in either compare form
  const float pad_y = MODE == 1 ? __int_as_float(0x7f800000) : __int_as_float(0x7fffffff);

  unsigned qi, t;
  while (next_item(L, wc, live, lane, qi, t)) {
    const ScanQuery& Q = L.queries[qi];
    QCtl* ctl = Q.ctl;
    Entry* __restrict__ buf = Q.buf;
    unsigned int* __restrict__ hist = Q.hist;
    const unsigned long long cap = Q.cap;
    const int maximize = Q.maximize;
    const float* packed = Q.packed;
    const double b_obj = Q.test_bias[0];
    const int nt = Q.nt;
    const unsigned long long hbase = *(volatile unsigned long long*)&ctl->hist_base;
    const unsigned hshift = *(volatile unsigned*)&ctl->hist_shift;
    const Tile T = L.tiles[t];
    const DevReaction& R = L.rx[T.rx];
    const int c = R.c;
    const int64_t n_last = R.size[c - 1];
    const float* col_src = packed + (size_t)(R.pair_off[c - 1] + T.col0) * NTP;
    const int nblk = (int)((T.ncols + cb - 1) / cb);

    // kick off the first column block before the threshold arithmetic
    if (lane == 0) {
      const uint32_t bytes = (T.ncols < (uint32_t)cb ? T.ncols : (uint32_t)cb) * NTP * 4u;
      fence_proxy_async();
      mbar_expect_tx(&bars[bi], bytes);
      bulk_g2s(bi ? sbuf1 : sbuf0, col_src, bytes, &bars[bi]);
    }

    const unsigned long long tau = ld_relaxed_u64(&ctl->tau_key);
    const double tau_s = key_to_score(tau);
    unsigned long long tau_seen = tau;

    float thr[RL][NT];
    double p_obj[RL];
    unsigned long long gbase[RL];
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const unsigned local = lane + 32u * r;
      const bool valid = local < T.nrows;
      const uint64_t row = T.row0 + (valid ? local : 0u);
      // prefix digits -> table rows of the first c-1 R-groups (registers)
      int64_t pr[kMaxRg - 1];
      {
        uint64_t rem = row;
#pragma unroll
        for (int j = kMaxRg - 2; j >= 1; --j) {
          pr[j] = 0;
          if (j <= c - 2) {
            uint64_t q, d;
            divmod_u64(q, d, rem, (uint64_t)R.size[j]);
            pr[j] = R.pair_off[j] + (int64_t)d;
            rem = q;
          }
        }
        pr[0] = R.pair_off[0] + (int64_t)rem;
      }
      gbase[r] = R.g_off + row * (uint64_t)n_last + T.col0;
#pragma unroll
      for (int i = 0; i < NT; ++i) {
        float th = __int_as_float(0x7f800000);  // +inf: padding test always passes
        if (i < nt) {
          const float* vrow = L.values + (int64_t)Q.test_task[i] * L.n_pairs;
          double p = c > 1 ? (double)__ldg(vrow + pr[0]) : 0.0;  // c == 1: no prefix
#pragma unroll
          for (int j = 1; j < kMaxRg - 1; ++j)
            if (j < c - 1) p = __dadd_rn(p, (double)__ldg(vrow + pr[j]));
          const double b = Q.test_bias[i];
          if (i == 0) {
            p_obj[r] = p;
            if (tau != kNoTau) th = maximize ? -thr_lower_fast(p, b, tau_s) : thr_upper_fast(p, b, -tau_s);
          } else {
            th = Q.test_lower[i] ? -thr_lower_fast(p, b, Q.test_beta[i]) : thr_upper_fast(p, b, Q.test_beta[i]);
          }
        }
        thr[r][i] = th;
      }
      if (!valid) thr[r][0] = __int_as_float(0x7fffffff);  // NaN: never passes
    }
    unsigned long long tp[RL][NP];
    if constexpr (MODE == 1) {
#pragma unroll
      for (int r = 0; r < RL; ++r)
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const float lo = tprime(thr[r][2 * p]);
          const float hi = 2 * p + 1 < NT ? tprime(thr[r][2 * p + 1]) : __int_as_float(0x7f800000);
          tp[r][p] = (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
        }
    }

    for (int blk = 0; blk < nblk; ++blk) {
      const int col_base = blk * cb;
      const int ncol = min(cb, (int)T.ncols - col_base);
      if (blk + 1 < nblk && lane == 0) {
        const unsigned nb = bi ^ 1u;
        const uint32_t bytes = (uint32_t)min(cb, (int)T.ncols - col_base - cb) * NTP * 4u;
        fence_proxy_async();
        mbar_expect_tx(&bars[nb], bytes);
        bulk_g2s(nb ? sbuf1 : sbuf0, col_src + (size_t)(col_base + cb) * NTP, bytes, &bars[nb]);
      }
      // tighten the admission threshold if another warp raised tau
      const unsigned long long tau_now = ld_relaxed_u64(&ctl->tau_key);
      if (tau_now != tau_seen) {
        tau_seen = tau_now;
        const double ts = key_to_score(tau_now);
#pragma unroll
        for (int r = 0; r < RL; ++r)
          if (lane + 32u * r < T.nrows) {
            thr[r][0] = maximize ? -thr_lower_fast(p_obj[r], b_obj, ts) : thr_upper_fast(p_obj[r], b_obj, -ts);
            if constexpr (MODE == 1)
              tp[r][0] = (tp[r][0] & 0xffffffff00000000ull) | __float_as_uint(tprime(thr[r][0]));
          }
      }
      if (bi) { mbar_wait(&bars[1], phase1); phase1 ^= 1u; }
      else    { mbar_wait(&bars[0], phase0); phase0 ^= 1u; }
      float* ys = bi ? sbuf1 : sbuf0;
      const int ngroups = (ncol + 7) >> 3;
      if (ncol & 7) {
        // pad the last group with columns that never pass
        const int pad = (ngroups << 3) - ncol;
        for (int idx = (int)lane; idx < pad * NTP; idx += 32) ys[ncol * NTP + idx] = pad_y;
        __syncwarp();
      }

      for (int gi = 0; gi < ngroups; ++gi) {
        const int j0 = gi << 3;
        bool any = false;
        if constexpr (MODE == 1) {
          unsigned acc[RL];
          unsigned anyw = 0;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) anyw = anyw | test_cols2<NT, RL>(ys, j0 + jj, tp, acc);
          any = (int)anyw < 0;
        } else {
          bool pass[RL];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) any = any | test_cols<NT, RL>(ys, j0 + jj, thr, pass);
        }
        if (__any_sync(0xffffffffu, any)) {
          // slow path: exact fp64 score, warp-aggregated append
          for (int jj = 0; jj < 8; ++jj) {
            bool pass[RL];
            if constexpr (MODE == 1) {
              unsigned acc[RL];
              test_cols2<NT, RL>(ys, j0 + jj, tp, acc);
#pragma unroll
              for (int r = 0; r < RL; ++r) pass[r] = (int)acc[r] < 0;
            } else {
              test_cols<NT, RL>(ys, j0 + jj, thr, pass);
            }
            const float y0 = ys[(j0 + jj) * NTP];
#pragma unroll
            for (int r = 0; r < RL; ++r) {
              Entry e;
              if (pass[r]) {
                const float x = maximize ? -y0 : y0;
                const double val = fx(p_obj[r], x, b_obj);
                e.key = skey(maximize ? val : -val);
                e.g = gbase[r] + (unsigned long long)(col_base + j0 + jj);
                pass[r] = !tie_reject(ctl, e.key, e.g);
              }
              const unsigned m = __ballot_sync(0xffffffffu, pass[r]);
              if (m) {
                const int leader = __ffs(m) - 1;
                unsigned long long base = 0;
                if ((int)lane == leader) base = atomicAdd(&ctl->count, (unsigned long long)__popc(m));
                base = __shfl_sync(0xffffffffu, base, leader);
                if (pass[r]) {
                  const unsigned long long idx = base + __popc(m & ((1u << lane) - 1u));
                  if (idx < cap) buf[idx] = e;
                  const unsigned hb = cand_bin(ctl, e.key, e.g, hbase, hshift);
                  atomicAdd(&hist[hb], 1u);
                  atomicAdd(&Q.coarse[hb >> 8], 1u);
                }
                // every `refresh` candidates, the warp that crosses the mark
                // recomputes tau from the histograms
                if ((base >> Q.refresh_shift) != ((base + __popc(m)) >> Q.refresh_shift)) {
                  __threadfence();
                  refresh_tau(Q);
                }
              }
            }
          }
        }
      }
      __syncwarp();
      bi ^= 1u;
    }
  }
}

// ---------------------------------------------------------------------------
// K3 (admission-first form).  Same tiles, same exact per-row threshold for the
// admission test (s >= tau), but the hot loop streams only the signed
// objective column: per product ONE fp32 compare (an FSETP.OR chain over 8
// columns) and a warp vote.  The constraint predicate is evaluated, exactly in
// fp64 in the reference's order, only for products that pass admission: the
// predicate is a conjunction, so this short-circuit yields the same candidate
// set as evaluating every test on every product.
// min of 16 consecutive fp32 in shared memory (32-bit shared address)
__device__ __forceinline__ float min16_shared(uint32_t addr) {
  float a0, a1, a2, a3, b0, b1, b2, b3, c0, c1, c2, c3, d0, d1, d2, d3;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3) : "r"(addr));
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+16];" : "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3) : "r"(addr));
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+32];" : "=f"(c0), "=f"(c1), "=f"(c2), "=f"(c3) : "r"(addr));
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4+48];" : "=f"(d0), "=f"(d1), "=f"(d2), "=f"(d3) : "r"(addr));
  return fminf(fminf(fminf(fminf(a0, a1), fminf(a2, a3)), fminf(fminf(b0, b1), fminf(b2, b3))),
               fminf(fminf(fminf(c0, c1), fminf(c2, c3)), fminf(fminf(d0, d1), fminf(d2, d3))));
}

// Table rows of the first c-1 R-groups of enumeration row `row` (the last
// R-group varies along the row); mixed-radix digits, least significant last.
__device__ __forceinline__ void decode_prefix(const DevReaction& R, int c, uint64_t row, int64_t (&pr)[kMaxRg - 1]) {
  uint64_t rem = row;
#pragma unroll
  for (int j = kMaxRg - 2; j >= 1; --j) {
    pr[j] = 0;
    if (j <= c - 2) {
      uint64_t q, d;
      divmod_u64(q, d, rem, (uint64_t)R.size[j]);
      pr[j] = R.pair_off[j] + (int64_t)d;
      rem = q;
    }
  }
  pr[0] = c > 1 ? R.pair_off[0] + (int64_t)rem : 0;
}

// Dense-row work item: the rest of one row of a tile whose objective
// threshold admits many columns, with the row's exact thresholds; pushed by
// the warp that found the row dense, finished by whichever warp is free.
struct DenseItem {
  const float* col_src;        // signed objective column at the tile's aligned start
  long long last_pair0;        // table row of the tile's aligned first column
  unsigned long long gbase;    // global index of that column in this row
  double p_obj;                // fp64 objective prefix of the row
  float thr_obj;               // admission threshold (signed objective) when pushed
  int from, ncols;             // columns [from, ncols) of the tile remain
  int q;                       // query of the launch
  unsigned ready;              // 1 once written; reset by the consumer
  unsigned _pad;
  float thrc[kMaxTests];       // constraint thresholds (index 1..nt-1)
};

// One dense row with all 32 lanes across its columns (two per lane), the
// objective and constraint contributions read from L2 with every test's loads
// issued together; candidates appended warp-aggregated.  ts: thresholds
// (ts[i]) and test descriptors (task << 1 | lower, as int bits at
// ts[kMaxTests + i]) in the warp's shared scratch.  Returns admitted products.
__device__ __noinline__ unsigned dense_row(const ScanQuery& Q, const float* __restrict__ values, int64_t n_pairs,
                                           const float* col_src, int64_t last_pair0, unsigned long long gb, double po,
                                           float to, int from, int ncols, const float* ts,
                                           unsigned long long hbase, unsigned hshift) {
  const unsigned lane = lane_id();
  const float pad_y = __int_as_float(0x7fffffff);
  const int nt = Q.nt;
  const int maximize = Q.maximize;
  const double b_obj = Q.test_bias[0];
  QCtl* ctl = Q.ctl;
  unsigned admitted = 0;
  for (int cc = from; cc < ncols; cc += 64) {
    const int col0 = cc + (int)lane, col1 = col0 + 32;
    const bool in0 = col0 < ncols, in1 = col1 < ncols;
    const float y0 = in0 ? __ldcg(col_src + col0) : pad_y;
    const float y1 = in1 ? __ldcg(col_src + col1) : pad_y;
    bool p0 = y0 <= to, p1 = y1 <= to;
    admitted += (p0 ? 1u : 0u) + (p1 ? 1u : 0u);
    if (__any_sync(0xffffffffu, p0 || p1)) {
#pragma unroll 4
      for (int i = 1; i < nt; ++i) {
        const int tl = __float_as_int(ts[kMaxTests + i]);
        const float* vx = values + (int64_t)(tl >> 1) * n_pairs + last_pair0;
        float x0 = in0 ? __ldg(vx + col0) : 0.0f;
        float x1 = in1 ? __ldg(vx + col1) : 0.0f;
        if (tl & 1) {
          x0 = -x0;
          x1 = -x1;
        }
        const float t = ts[i];
        p0 = p0 && x0 <= t;
        p1 = p1 && x1 <= t;
      }
    }
    Entry ee[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h ? p1 : p0)) continue;
      const float y = h ? y1 : y0;
      const float x = maximize ? -y : y;
      const double val = fx(po, x, b_obj);
      ee[h].key = skey(maximize ? val : -val);
      ee[h].g = gb + (unsigned long long)(h ? col1 : col0);
      if (tie_reject(ctl, ee[h].key, ee[h].g)) {
        if (h) p1 = false; else p0 = false;
      }
    }
    const unsigned cnt = (p0 ? 1u : 0u) + (p1 ? 1u : 0u);
    unsigned incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += o;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) continue;
    unsigned long long cbase = 0;
    if (lane == 31) cbase = atomicAdd(&ctl->count, (unsigned long long)tot);
    cbase = __shfl_sync(0xffffffffu, cbase, 31);
    unsigned long long idx = cbase + (incl - cnt);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h ? p1 : p0)) continue;
      const Entry e = ee[h];
      if (idx < Q.cap) Q.buf[idx] = e;
      ++idx;
      const unsigned hb = cand_bin(ctl, e.key, e.g, hbase, hshift);
      atomicAdd(&Q.hist[hb], 1u);
      atomicAdd(&Q.coarse[hb >> 8], 1u);
    }
    if ((cbase >> Q.refresh_shift) != ((cbase + tot) >> Q.refresh_shift)) {
      __threadfence();
      refresh_tau(Q);
    }
  }
  return admitted;
}

constexpr int kBlockDq = 32;  // dense-row queue slots per block (shared memory)

// Claim one queued dense row of the block (lane 0 CAS on the shared head,
// bounded by the tail); returns the slot or ~0u.
__device__ __forceinline__ unsigned claim_dense(unsigned* ctr, unsigned lane) {
  unsigned tk = ~0u;
  if (lane == 0) {
    for (;;) {
      const unsigned h = *(volatile unsigned*)&ctr[0];
      const unsigned tl = *(volatile unsigned*)&ctr[1];
      const unsigned lim = tl < (unsigned)kBlockDq ? tl : (unsigned)kBlockDq;
      if (h >= lim) break;
      if (atomicCAS(&ctr[0], h, h + 1u) == h) {
        tk = h;
        break;
      }
    }
  }
  return __shfl_sync(0xffffffffu, tk, 0);
}

// Run a claimed dense row: wait for its writer, stage its thresholds, scan
// the row with the admission threshold of the query's current tau.
__device__ __noinline__ void run_dense(const ScanLaunch& L, DenseItem* it, float* scratch) {
  const unsigned lane = lane_id();
  if (lane == 0)
    while (*(volatile unsigned*)&it->ready == 0u) {
    }
  __syncwarp();
  __threadfence_block();
  const int q = it->q;
  const ScanQuery& Q = L.queries[q];
  const int nt = Q.nt;
  for (int i = 1 + (int)lane; i < nt; i += 32) {
    scratch[i] = it->thrc[i];
    scratch[kMaxTests + i] = __int_as_float((Q.test_task[i] << 1) | (Q.test_lower[i] ? 1 : 0));
  }
  const float* col_src = it->col_src;
  const long long last_pair0 = it->last_pair0;
  const unsigned long long gb = it->gbase;
  const double po = it->p_obj;
  float to = it->thr_obj;
  const int from = it->from, ncols = it->ncols;
  __syncwarp();
  if (ncols <= from) return;
  // the admission threshold may have risen since the push
  const unsigned long long tau = *(volatile unsigned long long*)&Q.ctl->tau_key;
  if (tau != kNoTau) {
    const double ts = key_to_score(tau);
    to = Q.maximize ? -thr_lower_fast(po, Q.test_bias[0], ts) : thr_upper_fast(po, Q.test_bias[0], -ts);
  }
  const unsigned long long hbase = __ldcg(&Q.ctl->hist_base);
  const unsigned hshift = __ldcg(&Q.ctl->hist_shift);
  const unsigned a = dense_row(Q, L.values, L.n_pairs, col_src, last_pair0, gb, po, to, from, ncols, scratch, hbase,
                               hshift);
  const unsigned as = __reduce_add_sync(0xffffffffu, a);
  if (lane == 0 && as) atomicAdd(&Q.ctl->admitted, (unsigned long long)as);
}

#ifndef APEX_ADMIT_MINB
#define APEX_ADMIT_MINB 2
#endif
template <int RL, bool TRACE>
__global__ void __launch_bounds__(kScanWarps * 32, APEX_ADMIT_MINB) scan_admit_kernel(const ScanLaunch L) {
  extern __shared__ __align__(128) float sm_f[];
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  const unsigned long long live = live_mask(L, 0u);
  if (!live) return;
  WorkCursor wc;

  const int cb = L.cb;
  // shared-memory word offsets of this warp's two column buffers; indexing the
  // extern array (not a generic pointer) keeps the loads plain LDS
  const int off0 = (int)warp * 2 * cb, off1 = off0 + cb;
  const int xo = kScanWarps * 2 * cb + (int)warp * 16 * kMaxTests;  // rare-path scratch: 16 columns x tests
  // admitted-pair list of the rare path: up to 16 columns x 32*RL rows
  unsigned short* pairs = reinterpret_cast<unsigned short*>(sm_f + kScanWarps * 2 * cb + kScanWarps * 16 * kMaxTests) +
                          warp * (512 * RL);
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(sm_f + kScanWarps * 2 * cb + kScanWarps * 16 * kMaxTests +
                                                   kScanWarps * 256 * RL);
  uint64_t* bars = bars_all + warp * 2;
  // block dense-row queue: kBlockDq items, then [head, tail]
  DenseItem* sdq = reinterpret_cast<DenseItem*>(bars_all + kScanWarps * 2);
  unsigned* sdq_ctr = reinterpret_cast<unsigned*>(sdq + kBlockDq);
  // per-row constraint thresholds of the rare path, [r][test][lane] per warp:
  // lane-major (conflict-free for the owner) and readable by any lane of the
  // warp (the pair rounds read the pair's row directly)
  float* sthr = reinterpret_cast<float*>(sdq_ctr + 4) + (size_t)warp * RL * kMaxTests * 32;
  if (threadIdx.x == 0) {
    sdq_ctr[0] = 0u;
    sdq_ctr[1] = 0u;
  }
  for (int i = (int)threadIdx.x; i < kBlockDq; i += (int)blockDim.x) sdq[i].ready = 0u;
  __syncthreads();
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  uint32_t phase0 = 0, phase1 = 0;
  unsigned bi = 0;

  const float* __restrict__ values = L.values;
  const int64_t n_pairs = L.n_pairs;
  const float pad_y = __int_as_float(0x7fffffff);  // NaN: never passes
  constexpr int kTauPoll = 8;                      // column blocks between admission-threshold polls
  int poll = 0;

  // software-pipelined work items: the next item's tile descriptor and its
  // query's admission threshold are loaded while the current item runs
  unsigned qi, t;
  bool have = next_item(L, wc, live, lane, qi, t);
  Tile T_n;
  unsigned long long tau_n = 0;
  if (have) {
    T_n = L.tiles[t];
    tau_n = ld_relaxed_u64(&L.queries[qi].ctl->tau_key);
  }
  for (;;) {
    // queued dense rows first (they are what the tail of the launch waits on)
    if (!have || *(volatile unsigned*)&sdq_ctr[1] > *(volatile unsigned*)&sdq_ctr[0]) {
      for (;;) {
        const unsigned tk = claim_dense(sdq_ctr, lane);
        if (tk == ~0u) break;
        run_dense(L, sdq + tk, sm_f + xo);
      }
    }
    if (!have) break;
    const unsigned q_cur = qi;
    const unsigned t_cur = t;
    const unsigned long long t_start = TRACE ? globaltimer_ns() : 0ull;
    unsigned rare = 0;
    unsigned long long cyc_thr = 0, cyc_stage = 0, cyc_rare = 0, n_cand = 0;
    const Tile T = T_n;
    unsigned admitted = 0;
    unsigned long long tau_pref = tau_n;
    have = next_item(L, wc, live, lane, qi, t);
    if (have) {
      T_n = L.tiles[t];
      tau_n = ld_relaxed_u64(&L.queries[qi].ctl->tau_key);
    }
    const ScanQuery& Q = L.queries[q_cur];
    QCtl* ctl = Q.ctl;
    Entry* __restrict__ buf = Q.buf;
    unsigned int* __restrict__ hist = Q.hist;
    const unsigned long long cap = Q.cap;
    const int maximize = Q.maximize;
    const double b_obj = Q.test_bias[0];
    const float* __restrict__ vobj = values + (int64_t)Q.test_task[0] * n_pairs;
    const int nt = Q.nt;
    const DevReaction& R = L.rx[T.rx];
    const int c = R.c;
    const int64_t n_last = R.size[c - 1];
    // bulk copies need 16-B aligned sources: start the tile at col0 & ~3 and
    // mask the `lead` columns before col0 (partial rows at range cuts)
    const uint32_t lead = T.col0 & 3u;
    const uint32_t ac0 = T.col0 - lead;
    const uint32_t ncols = T.ncols + lead;
    const int64_t last_pair0 = R.pair_off[c - 1] + ac0;
    const float* col_src = Q.obj_col + R.pcol_off + ac0;
    const int nblk = (int)((ncols + cb - 1) / cb);
    if (lane == 0) {
      const uint32_t bytes = ((ncols < (uint32_t)cb ? ncols : (uint32_t)cb) * 4u + 15u) & ~15u;
      fence_proxy_async();
      mbar_expect_tx(&bars[bi], bytes);
      bulk_g2s(sm_f + (bi ? off1 : off0), col_src, bytes, &bars[bi]);
    }
    const unsigned long long tau = tau_pref;
    unsigned long long tau_seen = tau;

    float thr[RL];
    bool thr_ready = false;
    // dense rows (dense_min admitted products so far in this tile): taken out
    // of the column-group vote and finished row-parallel after the tile
    // (below), so a tile whose good rows admit a few columns of every group
    // does not pay the rare path per group
    bool dense[RL];
    int dense_from[RL];
    unsigned adm_row[RL];  // admitted products of the row so far in this tile
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      dense[r] = false;
      dense_from[r] = 0;
      adm_row[r] = 0;
    }
    double p_obj[RL];
    int64_t pr[RL][kMaxRg - 1];
    unsigned long long gbase[RL];
#pragma unroll
    for (int r = 0; r < RL; ++r) {
      const unsigned local = lane + 32u * r;
      const bool valid = local < T.nrows;
      const uint64_t row = T.row0 + (valid ? local : 0u);
      {
        uint64_t rem = row;
#pragma unroll
        for (int j = kMaxRg - 2; j >= 1; --j) {
          pr[r][j] = 0;
          if (j <= c - 2) {
            uint64_t q, d;
            divmod_u64(q, d, rem, (uint64_t)R.size[j]);
            pr[r][j] = R.pair_off[j] + (int64_t)d;
            rem = q;
          }
        }
        pr[r][0] = R.pair_off[0] + (int64_t)rem;
      }
      gbase[r] = R.g_off + row * (uint64_t)n_last + ac0;
      double p = c > 1 ? (double)__ldg(vobj + pr[r][0]) : 0.0;
#pragma unroll
      for (int j = 1; j < kMaxRg - 1; ++j)
        if (j < c - 1) p = __dadd_rn(p, (double)__ldg(vobj + pr[r][j]));
      p_obj[r] = p;
      float th = __int_as_float(0x7f800000);
      if (tau != kNoTau) {
        const double ts = key_to_score(tau);
        th = maximize ? -thr_lower_fast(p, b_obj, ts) : thr_upper_fast(p, b_obj, -ts);
      }
      thr[r] = valid ? th : __int_as_float(0x7fffffff);
    }

    for (int blk = 0; blk < nblk; ++blk) {
      const int col_base = blk * cb;
      const int ncol = min(cb, (int)ncols - col_base);
      if (blk + 1 < nblk && lane == 0) {
        const unsigned nb = bi ^ 1u;
        const uint32_t bytes = ((uint32_t)min(cb, (int)ncols - col_base - cb) * 4u + 15u) & ~15u;
        fence_proxy_async();
        mbar_expect_tx(&bars[nb], bytes);
        bulk_g2s(sm_f + (nb ? off1 : off0), col_src + col_base + cb, bytes, &bars[nb]);
      }
      if (++poll == kTauPoll) {
        poll = 0;
        const unsigned long long tau_now = tau_pref;
        tau_pref = ld_relaxed_u64(&ctl->tau_key);  // consumed at the next poll
        if (tau_now != tau_seen) {
          tau_seen = tau_now;
          const double ts = key_to_score(tau_now);
#pragma unroll
          for (int r = 0; r < RL; ++r)
            if (lane + 32u * r < T.nrows)
              thr[r] = maximize ? -thr_lower_fast(p_obj[r], b_obj, ts) : thr_upper_fast(p_obj[r], b_obj, -ts);
        }
      }
      if (bi) { mbar_wait(&bars[1], phase1); phase1 ^= 1u; }
      else    { mbar_wait(&bars[0], phase0); phase0 ^= 1u; }
      const int yo = bi ? off1 : off0;
      const int ngroups = (ncol + 15) >> 4;
      if ((ncol & 63) || (blk == 0 && lead)) {
        // pad to a multiple of 64 columns with values that never pass
        const int pad = ((ncol + 63) & ~63) - ncol;
        for (int i = (int)lane; i < pad; i += 32) sm_f[yo + ncol + i] = pad_y;
        if (blk == 0 && lane < lead) sm_f[yo + lane] = pad_y;
        __syncwarp();
      }
      float thr_min = dense[0] ? pad_y : thr[0];
#pragma unroll
      for (int r = 1; r < RL; ++r) thr_min = fmaxf(thr_min, dense[r] ? pad_y : thr[r]);
      const uint32_t ybase = smem_u32(sm_f) + (uint32_t)yo * 4u;
      for (int gi = 0; gi < ngroups; ++gi) {
        const int j0 = gi << 4;
        if (L.vote64 && (gi & 3) == 0) {
          // 64 columns per vote: 16 broadcast LDS.128 in flight, four min
          // trees, one compare per lane; skip all four 16-column groups when
          // no lane admits anything
          const uint32_t a0 = ybase + (uint32_t)j0 * 4u;
          const float m64 = fminf(fminf(min16_shared(a0), min16_shared(a0 + 64u)),
                                  fminf(min16_shared(a0 + 128u), min16_shared(a0 + 192u)));
          if (!__any_sync(0xffffffffu, m64 <= thr_min)) {
            gi += 3;
            continue;
          }
        }
        // min over the 16 columns, one compare per lane, one vote per warp
        const float ymin = min16_shared(ybase + (uint32_t)j0 * 4u);
        if (__any_sync(0xffffffffu, ymin <= thr_min)) {
          if (TRACE) ++rare;
          const unsigned long long c_r0 = TRACE ? clock64() : 0ull;
          // rare path.  Admitted products (s >= tau) get the constraint
          // predicate with exact per-row fp32 thresholds (computed once per
          // tile, on first use) against the 16 columns' contributions staged
          // in this warp's scratch; a dense cluster of admitted-but-
          // infeasible products then costs compares, not fp64 chains.
          if (!thr_ready) {
            thr_ready = true;
            const unsigned long long c_t0 = TRACE ? clock64() : 0ull;
#pragma unroll
            for (int r = 0; r < RL; ++r)
              for (int i = 1; i < nt; ++i) {
                const float* v = values + (int64_t)Q.test_task[i] * n_pairs;
                double p = c > 1 ? (double)__ldg(v + pr[r][0]) : 0.0;
                for (int j = 1; j < c - 1; ++j) p = __dadd_rn(p, (double)__ldg(v + pr[r][j]));
                sthr[(r * kMaxTests + i) * 32 + lane] = Q.test_lower[i] ? -thr_lower_fast(p, Q.test_bias[i], Q.test_beta[i])
                                             : thr_upper_fast(p, Q.test_bias[i], Q.test_beta[i]);
              }
            if (TRACE) cyc_thr += clock64() - c_t0;
          }
          const unsigned long long c_s0 = TRACE ? clock64() : 0ull;
          for (int idx = (int)lane; idx < (nt - 1) * 16; idx += 32) {
            const int i = 1 + (idx >> 4), jj = idx & 15;
            const int col = col_base + j0 + jj;
            float x = 0.0f;
            if (col < (int)ncols) x = __ldg(values + (int64_t)Q.test_task[i] * n_pairs + last_pair0 + col);
            sm_f[xo + idx] = Q.test_lower[i] ? -x : x;
          }
          __syncwarp();
          if (TRACE) cyc_stage += clock64() - c_s0;
          // admission masks of this lane's rows over the 16 columns, then the
          // admitted (row, column) pairs are listed in the warp's scratch and
          // the constraint tests run ONE PAIR PER LANE (the row's thresholds
          // fetched by shuffle): a hot row admitted in every column costs the
          // warp one round per 32 admitted products, not 16 lock-step columns
          unsigned am[RL];
#pragma unroll
          for (int r = 0; r < RL; ++r) am[r] = 0u;
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) {
            const float y0 = sm_f[yo + j0 + jj];
#pragma unroll
            for (int r = 0; r < RL; ++r) am[r] |= (!dense[r] && y0 <= thr[r] ? 1u : 0u) << jj;
          }
          {
            bool newly = false;
#pragma unroll
            for (int r = 0; r < RL; ++r)
              if (!dense[r] && (adm_row[r] += __popc(am[r])) >= (unsigned)L.dense_min) {
                dense[r] = true;
                dense_from[r] = col_base + j0 + 16;
                newly = true;
              }
            if (newly) {
              thr_min = dense[0] ? pad_y : thr[0];
#pragma unroll
              for (int r = 1; r < RL; ++r) thr_min = fmaxf(thr_min, dense[r] ? pad_y : thr[r]);
            }
          }
          unsigned cnt = 0;
#pragma unroll
          for (int r = 0; r < RL; ++r) cnt += __popc(am[r]);
          admitted += cnt;
          unsigned incl = cnt;
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
            if ((int)lane >= off) incl += o;
          }
          const unsigned n_adm = __shfl_sync(0xffffffffu, incl, 31);
          {
            unsigned o = incl - cnt;
#pragma unroll
            for (int r = 0; r < RL; ++r) {
              unsigned m = am[r];
              while (m) {
                const unsigned jj = (unsigned)__ffs(m) - 1u;
                m &= m - 1u;
                pairs[o++] = (unsigned short)(((lane + 32u * r) << 4) | jj);
              }
            }
          }
          __syncwarp();
          for (unsigned base = 0; base < n_adm; base += 32) {
            const unsigned pi = base + lane;
            const bool valid = pi < n_adm;
            const unsigned pv = valid ? pairs[pi] : 0u;
            const unsigned row = pv >> 4, jj = pv & 15u, src = row & 31u;
            bool pass = valid;
            for (int i = 1; i < nt; ++i) {
              const float t = sthr[((row >> 5) * kMaxTests + i) * 32 + src];
              pass = pass && (sm_f[xo + ((i - 1) << 4) + jj] <= t);
            }
            double po = __shfl_sync(0xffffffffu, p_obj[0], src);
            unsigned long long gb = __shfl_sync(0xffffffffu, gbase[0], src);
            if (RL == 2) {
              const double po1 = __shfl_sync(0xffffffffu, p_obj[RL - 1], src);
              const unsigned long long gb1 = __shfl_sync(0xffffffffu, gbase[RL - 1], src);
              if (row >= 32u) {
                po = po1;
                gb = gb1;
              }
            }
            Entry e;
            if (pass) {
              const float y0 = sm_f[yo + j0 + jj];
              const float x = maximize ? -y0 : y0;
              const double val = fx(po, x, b_obj);
              e.key = skey(maximize ? val : -val);
              e.g = gb + (unsigned long long)(col_base + j0 + (int)jj);
              pass = !tie_reject(ctl, e.key, e.g);
            }
            const unsigned m = __ballot_sync(0xffffffffu, pass);
            if (TRACE) n_cand += __popc(m);
            if (!m) continue;
            unsigned long long cbase = 0;
            if (lane == 0) cbase = atomicAdd(&ctl->count, (unsigned long long)__popc(m));
            cbase = __shfl_sync(0xffffffffu, cbase, 0);
            if (pass) {
              const unsigned long long idx = cbase + __popc(m & ((1u << lane) - 1u));
              if (idx < cap) buf[idx] = e;
              const unsigned hb = cand_bin(ctl, e.key, e.g, __ldcg(&ctl->hist_base), __ldcg(&ctl->hist_shift));
              atomicAdd(&hist[hb], 1u);
              atomicAdd(&Q.coarse[hb >> 8], 1u);
            }
            if ((cbase >> Q.refresh_shift) != ((cbase + __popc(m)) >> Q.refresh_shift)) {
              __threadfence();
              refresh_tau(Q);
            }
          }
          __syncwarp();
          if (TRACE) cyc_rare += clock64() - c_r0;
        }
      }
      __syncwarp();
      bi ^= 1u;
    }
    // dense rows: the rest of each such row (from the group after the one
    // that flagged it) is pushed to the block's dense-row queue, where any
    // warp of the block takes it at its next item boundary (dense_row: all 32 lanes across the row's columns);
    // the tile itself stays short, so hot tiles do not become stragglers
    {
      unsigned dn = 0;
#pragma unroll
      for (int r = 0; r < RL; ++r) dn += dense[r] ? 1u : 0u;
      if (__any_sync(0xffffffffu, dn != 0u)) {
        unsigned incl = dn;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const unsigned o = __shfl_up_sync(0xffffffffu, incl, off);
          if ((int)lane >= off) incl += o;
        }
        const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(&sdq_ctr[1], tot);
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base + tot <= (unsigned)kBlockDq) {
          unsigned slot = base + incl - dn;
#pragma unroll
          for (int r = 0; r < RL; ++r) {
            if (!dense[r]) continue;
            DenseItem* it = sdq + slot++;
            it->col_src = col_src;
            it->last_pair0 = last_pair0;
            it->gbase = gbase[r];
            it->p_obj = p_obj[r];
            it->thr_obj = thr[r];
            it->from = dense_from[r];
            it->ncols = (int)ncols;
            it->q = (int)q_cur;
            for (int i = 1; i < nt; ++i) it->thrc[i] = sthr[(r * kMaxTests + i) * 32 + lane];
            __threadfence_block();
            *(volatile unsigned*)&it->ready = 1u;
          }
        } else {
          // queue full: empty items for the reserved slots that exist (so no
          // claimer waits forever), then the rows are finished here
          for (unsigned sl = base + lane; sl < (unsigned)kBlockDq && sl < base + tot; sl += 32) {
            DenseItem* it = sdq + sl;
            it->from = 0;
            it->ncols = 0;
            it->q = (int)q_cur;
            __threadfence_block();
            *(volatile unsigned*)&it->ready = 1u;
          }
          float* scratch = sm_f + xo;
          for (int i = 1 + (int)lane; i < nt; i += 32)
            scratch[kMaxTests + i] = __int_as_float((Q.test_task[i] << 1) | (Q.test_lower[i] ? 1 : 0));
#pragma unroll
          for (int r = 0; r < RL; ++r) {
            unsigned dm = __ballot_sync(0xffffffffu, dense[r]);
            while (dm) {
              const int src = __ffs(dm) - 1;
              dm &= dm - 1u;
              for (int i = 1; i < nt; ++i) {
                if (lane == 0) scratch[i] = sthr[(r * kMaxTests + i) * 32 + src];
              }
              const float to = __shfl_sync(0xffffffffu, thr[r], src);
              const double po = __shfl_sync(0xffffffffu, p_obj[r], src);
              const unsigned long long gb = __shfl_sync(0xffffffffu, gbase[r], src);
              const int from = __shfl_sync(0xffffffffu, dense_from[r], src);
              __syncwarp();
              admitted += dense_row(Q, values, n_pairs, col_src, last_pair0, gb, po, to, from, (int)ncols, scratch,
                                    __ldcg(&ctl->hist_base), __ldcg(&ctl->hist_shift));
              __syncwarp();
            }
          }
        }
      }
    }
    {
      const unsigned a = __reduce_add_sync(0xffffffffu, admitted);
      if (a && lane == 0) atomicAdd(&ctl->admitted, (unsigned long long)a);
    }
    if (TRACE && lane == 0) {
      const unsigned rec = (t_cur - L.tile_begin) * (unsigned)L.nq + q_cur;
      if (rec < L.trace_cap) {
        unsigned long long* w = L.trace + 8ull * rec;
        w[4] = cyc_rare;
        w[5] = cyc_thr;
        w[6] = cyc_stage;
        w[7] = n_cand;
        w[0] = t_start;
        w[1] = globaltimer_ns();
        w[2] = (unsigned long long)smid() | ((unsigned long long)(rare < 0xffffffu ? rare : 0xffffffu) << 8) |
               ((unsigned long long)q_cur << 32);
        w[3] = ((unsigned long long)T.rx << 32) | ((unsigned long long)T.ncols << 8) | T.nrows;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3 (sorted-column form, the default admission kernel).  For one row the
// admission test y <= thr is a threshold on the last R-group's value alone,
// so the admitted columns are a prefix (minimize: x ascending, x <= thr) or a
// suffix (maximize: x >= -thr) of that R-group's values sorted once per task
// at table load (build_corners).  A tile of 32 whole rows costs one exact
// fp64 threshold and one galloping search per row; after that, work is spent
// only on admitted (row, column) pairs: exact per-row constraint thresholds
// against the pairs' gathered constraint values, candidates appended exactly
// as in the streaming forms.  The candidate set is identical (feasible and
// s >= tau, both exact), so nothing downstream changes.
struct SortedLaunch {
  const float* packed16;  // [n_pairs][16] pair-major copy of the table (n_tasks <= 16), or null
  const float* sx;        // [task][pcols]: each reaction's last R-group values ascending, at pcol_off
  const uint32_t* scol;   // same layout: column index of each sorted value
  int64_t pcols;
  const float* quant;     // [task][n_rx][kQuant + 1]: evenly spaced values of each sorted column
  int n_rx;
  const float* cthr;      // pre-pass: [cset_off + test - 1][rows_pad] constraint thresholds per row
  const int4* cbest;      // pre-pass: [cset][rows_pad] (best test, its quantile count, range start, count)
  int64_t rows_pad;       // row slots: 32 per row tile of the plan
  const double* rowp;     // [task][rows_total] fp64 prefix sums of every row (bind), or null
  int64_t rows_total;
};


// first index i in [0, n) with !(xs[i] <= t) (n if none); xs ascending
__device__ __forceinline__ int first_gt(const float* __restrict__ xs, int n, float t) {
  int lo = 0, p = 0, step = 1;
  while (p < n && __ldg(xs + p) <= t) {
    lo = p + 1;
    p += step;
    step <<= 1;
  }
  int hi = p < n ? p : n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(xs + mid) <= t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// first index i in [0, n) with !(xs[i] < t) (n if none); xs ascending
__device__ __forceinline__ int first_ge(const float* __restrict__ xs, int n, float t) {
  int lo = 0, p = 0, step = 1;
  while (p < n && __ldg(xs + p) < t) {
    lo = p + 1;
    p += step;
    step <<= 1;
  }
  int hi = p < n ? p : n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(xs + mid) < t) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Approximate passing count (in kQuant+1 quantile steps) of a test on a sorted
// column: upper tests pass x <= t, lower tests pass x >= t.  Used only to pick
// which test's exact range to enumerate.
__device__ __forceinline__ int quant_count(const float* __restrict__ q, bool lower, float t) {
  // the two ends first (independent loads): most tests pass nothing or
  // everything of a row and need no search
  const float q_lo = __ldg(q), q_hi = __ldg(q + kQuant);
  if (!lower) {
    if (!(q_lo <= t)) return 0;
    if (q_hi <= t) return kQuant + 1;
  } else {
    if (!(q_hi >= t)) return 0;
    if (q_lo >= t) return kQuant + 1;
  }
  int lo = 1, hi = kQuant;  // first index failing the monotone predicate, in [1, kQuant]
  if (!lower) {
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(q + mid) <= t) lo = mid + 1; else hi = mid;
    }
    return lo;
  }
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(q + mid) < t) lo = mid + 1; else hi = mid;
  }
  return kQuant + 1 - lo;
}

// quant_count for up to four tests at once (q tables at qbase + task * qstride):
// the ends of every table first, then the binary searches in lockstep, so the
// four dependent-load chains overlap.  th[u] is the signed-value threshold
// (lower tests compare -x <= th, i.e. x >= -th); NaN means nothing passes.
#ifndef APEX_THR_BATCH
#define APEX_THR_BATCH 1
#endif
constexpr int kThrBatch = APEX_THR_BATCH;  // tests whose threshold chains are interleaved
#ifndef APEX_PAIR_BATCH
#define APEX_PAIR_BATCH 1
#endif
// sorted-column pair loop: test gathers issued together (1: one at a time; 4 and
// 8 were slower on C2 — more issue slots and registers for a loop that is not
// latency-bound, profiles/r2_ab_pair_batch_rejected.log)
constexpr int kPairBatch = APEX_PAIR_BATCH;
constexpr unsigned kBailFlush = 4096;  // sorted-column pair budget: per-CTA pairs between flushes
__device__ __forceinline__ void quant_count4(const float* __restrict__ qbase, int64_t qstride,
                                             const int (&task)[kThrBatch], const bool (&lower)[kThrBatch],
                                             const float (&th)[kThrBatch], int (&qc)[kThrBatch]) {
  const float* q[kThrBatch];
  float t[kThrBatch], qlo[kThrBatch], qhi[kThrBatch];
  int lo[kThrBatch], hi[kThrBatch];
#pragma unroll
  for (int u = 0; u < kThrBatch; ++u) {
    q[u] = qbase + (int64_t)task[u] * qstride;
    t[u] = lower[u] ? -th[u] : th[u];
    qlo[u] = __ldg(q[u]);
    qhi[u] = __ldg(q[u] + kQuant);
  }
#pragma unroll
  for (int u = 0; u < kThrBatch; ++u) {
    lo[u] = 1;
    hi[u] = kQuant;
    qc[u] = -1;  // undecided: search
    if (!(th[u] == th[u])) qc[u] = 0;
    else if (!lower[u]) {
      if (!(qlo[u] <= t[u])) qc[u] = 0;
      else if (qhi[u] <= t[u]) qc[u] = kQuant + 1;
    } else {
      if (!(qhi[u] >= t[u])) qc[u] = 0;
      else if (qlo[u] >= t[u]) qc[u] = kQuant + 1;
    }
    if (qc[u] >= 0) lo[u] = hi[u];
  }
#pragma unroll
  for (int step = 0; step < 5; ++step) {  // ceil(log2(kQuant)) halvings of [1, kQuant]
    float x[kThrBatch];
    int mid[kThrBatch];
#pragma unroll
    for (int u = 0; u < kThrBatch; ++u) {
      mid[u] = (lo[u] + hi[u]) >> 1;
      x[u] = lo[u] < hi[u] ? __ldg(q[u] + mid[u]) : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < kThrBatch; ++u) {
      if (lo[u] < hi[u]) {
        const bool go = lower[u] ? (x[u] < t[u]) : (x[u] <= t[u]);
        if (go) lo[u] = mid[u] + 1; else hi[u] = mid[u];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kThrBatch; ++u)
    if (qc[u] < 0) qc[u] = lower[u] ? kQuant + 1 - lo[u] : lo[u];
}

// sorted position of quantile qq: quant[qq] = xs[qpos(qq)] (capi.cu build_corners)
__device__ __forceinline__ int qpos(int qq, int n) { return min(n - 1, (int)(((long long)qq * n) / kQuant)); }

// Exact passing range [start, start + cnt) of a test on a sorted column xs of
// length n: upper tests pass x <= t (a prefix), lower tests x >= t (a suffix).
// qc = the test's quant_count, which brackets the boundary between two
// quantile positions, so only that window is binary-searched.
__device__ __forceinline__ void exact_range(const float* __restrict__ xs, int n, bool lower, float t, int qc,
                                            int& start, int& cnt) {
  if (!lower) {
    // boundary B = first index with xs[B] > t
    int a, b;
    if (qc <= 0) { a = 0; b = 0; }
    else if (qc > kQuant) { a = n; b = n; }
    else { a = qpos(qc - 1, n) + 1; b = qpos(qc, n); }
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (__ldg(xs + mid) <= t) a = mid + 1; else b = mid;
    }
    start = 0;
    cnt = a;
  } else {
    // start = first index with xs[start] >= t; the bracket index is lo = kQuant + 1 - qc
    int a, b;
    if (qc <= 0) { a = n; b = n; }
    else if (qc > kQuant) { a = 0; b = 0; }
    else { const int lo = kQuant + 1 - qc; a = qpos(lo - 1, n) + 1; b = qpos(lo, n); }
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (__ldg(xs + mid) < t) a = mid + 1; else b = mid;
    }
    start = a;
    cnt = n - a;
  }
}

// contribution of task at pair row: from the pair-major copy when present
// (one 64-byte line per pair), else the task-major table
__device__ __forceinline__ float tval(const float* __restrict__ values, const float* __restrict__ p16, int64_t n_pairs,
                                      int task, int64_t pair) {
  return p16 ? __ldg(p16 + pair * 16 + task) : __ldg(values + (int64_t)task * n_pairs + pair);
}

// Constraint pre-pass of the sorted-column kernel.  A constraint set shared
// by several queries of the batch (the objectives of one property preset)
// gives every row the same exact constraint thresholds, quantile counts and
// most selective constraint range whichever query scans it: they are derived
// once per (row tile, set) here — on a stream beside the seed kernels, whose
// time it hides under — and the scan items of those queries read them.
// Two short kernels, so the dependent chains stay one test long: (A) one warp
// per (row tile, test): the exact threshold and its quantile count; (B) one
// warp per (row tile, set): the most selective test and its exact range.
constexpr int kConsPreItems = 384;  // (set, test) pairs per launch of A, sets per launch of B
struct ConsPre {
  const ScanQuery* queries;  // whole batch
  const Tile* tiles;         // row tiles of the plan
  unsigned n_tiles;
  const DevReaction* rx;
  const float* values;
  const float* p16;
  int64_t n_pairs;
  const float* sx;
  const float* quant;
  int64_t pcols;
  int n_rx;
  float* cthr;               // [cset_off + i - 1][rows_pad]
  unsigned char* cqc;        // same layout: quantile counts
  int4* cbest;               // [cset][rows_pad]
  int64_t rows_pad;
  const double* rowp;        // row-prefix table (bind) or null
  int64_t rows_total;
  int n;                     // A: (query, test) pairs; B: sets (leader queries)
  int q[kConsPreItems];      // A: a query of the test's set / B: a query of each set
  unsigned char ti[kConsPreItems];  // A: test index (1..nt-1)
};

// (both pre-pass kernels run a capped, grid-stride grid: a grid of every item
// would take every SM slot first and hold back the seed kernels beside them)
__global__ void __launch_bounds__(256) cons_thr_kernel(const __grid_constant__ ConsPre P) {
  const unsigned lane = lane_id();
  const unsigned items = P.n_tiles * (unsigned)P.n, step = gridDim.x * (blockDim.x >> 5);
  for (unsigned item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < items; item += step) {
  const unsigned t = item / (unsigned)P.n, k = item % (unsigned)P.n;
  const ScanQuery& Q = P.queries[P.q[k]];
  const int i = P.ti[k];
  const Tile T = P.tiles[t];
  const DevReaction& R = P.rx[T.rx];
  const int c = R.c;
  const uint64_t row = T.row0 + (lane < T.nrows ? lane : 0u);
  const int task = Q.test_task[i];
  double p;
  if (P.rowp) {
    p = __ldg(P.rowp + task * P.rows_total + R.row_off + (int64_t)row);
  } else {
    int64_t pr[kMaxRg - 1];
    decode_prefix(R, c, row, pr);
    p = c > 1 ? (double)tval(P.values, P.p16, P.n_pairs, task, pr[0]) : 0.0;
#pragma unroll
    for (int j = 1; j < kMaxRg - 1; ++j)
      if (j < c - 1) p = __dadd_rn(p, (double)tval(P.values, P.p16, P.n_pairs, task, pr[j]));
  }
  const bool lower = Q.test_lower[i] != 0;
  const float th = lower ? -thr_lower_fast(p, Q.test_bias[i], Q.test_beta[i])
                         : thr_upper_fast(p, Q.test_bias[i], Q.test_beta[i]);
  const int qc = th == th ? quant_count(P.quant + ((int64_t)task * P.n_rx + T.rx) * (kQuant + 1), lower,
                                        lower ? -th : th)
                          : 0;
  const int64_t o = (int64_t)(Q.cset_off + i - 1) * P.rows_pad + (int64_t)t * 32 + lane;
  P.cthr[o] = th;
  P.cqc[o] = (unsigned char)qc;
  }
}

__global__ void __launch_bounds__(256) cons_best_kernel(const __grid_constant__ ConsPre P) {
  const unsigned lane = lane_id();
  const unsigned items = P.n_tiles * (unsigned)P.n, step = gridDim.x * (blockDim.x >> 5);
  for (unsigned item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < items; item += step) {
  const unsigned t = item / (unsigned)P.n, si = item % (unsigned)P.n;
  const ScanQuery& Q = P.queries[P.q[si]];
  const Tile T = P.tiles[t];
  const DevReaction& R = P.rx[T.rx];
  const int nt = Q.nt;
  const bool valid = lane < T.nrows;
  const int64_t slot = (int64_t)t * 32 + lane;
  int best = 0, best_q = kQuant + 2;
  for (int i = 1; i < nt; ++i) {  // lowest test index among the smallest counts
    const int qc = P.cqc[(int64_t)(Q.cset_off + i - 1) * P.rows_pad + slot];
    if (qc < best_q) {
      best_q = qc;
      best = i;
    }
  }
  int start = 0, cnt = 0;
  if (valid && best != 0 && best_q > 0) {
    const float th = P.cthr[(int64_t)(Q.cset_off + best - 1) * P.rows_pad + slot];
    const bool lw = Q.test_lower[best] != 0;
    exact_range(P.sx + (int64_t)Q.test_task[best] * P.pcols + R.pcol_off, (int)R.size[R.c - 1], lw, lw ? -th : th,
                best_q, start, cnt);
  }
  P.cbest[(int64_t)Q.cset * P.rows_pad + slot] = make_int4(best, valid ? best_q : kQuant + 2, start, cnt);
  }
}

// The two pre-pass kernels fused: one warp per (row tile, set) derives every
// constraint threshold of the set (all the set's prefix loads issued before
// any threshold, the tests' quantile searches interleaved), keeps the most
// selective test and searches its exact range — one launch and no round trip
// of the quantile counts through memory.
constexpr int kConsFuseBatch = 8;
__global__ void __launch_bounds__(256) cons_fused_kernel(const __grid_constant__ ConsPre P) {
  const unsigned lane = lane_id();
  const unsigned items = P.n_tiles * (unsigned)P.n, step = gridDim.x * (blockDim.x >> 5);
  for (unsigned item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < items; item += step) {
    const unsigned t = item / (unsigned)P.n, si = item % (unsigned)P.n;
    const ScanQuery& Q = P.queries[P.q[si]];
    const Tile T = P.tiles[t];
    const DevReaction& R = P.rx[T.rx];
    const int c = R.c, nt = Q.nt;
    const bool valid = lane < T.nrows;
    const uint64_t row = T.row0 + (valid ? lane : 0u);
    const int64_t slot = (int64_t)t * 32 + lane;
    int64_t pr[kMaxRg - 1];
    if (!P.rowp) decode_prefix(R, c, row, pr);
    const float* qbase = P.quant + (int64_t)T.rx * (kQuant + 1);
    const int64_t qstride = (int64_t)P.n_rx * (kQuant + 1);
    int best = 0, best_q = kQuant + 2;
    float best_th = 0.0f;
    for (int i0 = 1; i0 < nt; i0 += kConsFuseBatch) {
      double p[kConsFuseBatch];
#pragma unroll
      for (int u = 0; u < kConsFuseBatch; ++u) {
        const int i = min(i0 + u, nt - 1);
        const int task = Q.test_task[i];
        if (P.rowp) {
          p[u] = __ldg(P.rowp + task * P.rows_total + R.row_off + (int64_t)row);
        } else {
          double pp = c > 1 ? (double)tval(P.values, P.p16, P.n_pairs, task, pr[0]) : 0.0;
#pragma unroll
          for (int j = 1; j < kMaxRg - 1; ++j)
            if (j < c - 1) pp = __dadd_rn(pp, (double)tval(P.values, P.p16, P.n_pairs, task, pr[j]));
          p[u] = pp;
        }
      }
#pragma unroll
      for (int u = 0; u < kConsFuseBatch; ++u) {
        const int i = i0 + u;
        if (i >= nt) break;
        const bool lower = Q.test_lower[i] != 0;
        const float th = lower ? -thr_lower_fast(p[u], Q.test_bias[i], Q.test_beta[i])
                               : thr_upper_fast(p[u], Q.test_bias[i], Q.test_beta[i]);
        P.cthr[(int64_t)(Q.cset_off + i - 1) * P.rows_pad + slot] = th;
        const int qc = th == th ? quant_count(qbase + Q.test_task[i] * qstride, lower, lower ? -th : th) : 0;
        if (qc < best_q) {  // lowest test index among the smallest counts
          best_q = qc;
          best = i;
          best_th = th;
        }
      }
    }
    int start = 0, cnt = 0;
    if (valid && best != 0 && best_q > 0) {
      const bool lw = Q.test_lower[best] != 0;
      exact_range(P.sx + (int64_t)Q.test_task[best] * P.pcols + R.pcol_off, (int)R.size[R.c - 1], lw,
                  lw ? -best_th : best_th, best_q, start, cnt);
    }
    P.cbest[(int64_t)Q.cset * P.rows_pad + slot] = make_int4(best, valid ? best_q : kQuant + 2, start, cnt);
  }
}

// CTAs per SM of the sorted-column scan (register budget 65536 / (256 x MINB)):
// 3 (80 registers) beat 4 (64 registers, more spills) by 5-8% on C2
// (profiles/r2_ab_sorted_minb.log); 2 (107 registers) was in between
#ifndef APEX_SORTED_MINB
#define APEX_SORTED_MINB 3
#endif
// candidates staged per warp in shared memory before the buffer append
// (0: one append per round with candidates)
#ifndef APEX_CAND_STAGE
#define APEX_CAND_STAGE 1
#endif
#ifndef APEX_CAND_SLOTS
#define APEX_CAND_SLOTS 64
#endif
constexpr int kCandStage = APEX_CAND_SLOTS;
#ifndef APEX_TILE_SMEM
#define APEX_TILE_SMEM 0  // 1: measured neutral (profiles/r2_ab_tile_smem_rejected.log)
#endif
// P16: contributions read from the pair-major copy packed16[pair][16] (one
// 64-byte line per pair holds every task: a row's prefix sums and a pair's
// test values for all tests come from one line each instead of one line per
// task), else from the task-major table values[task][pair].
// ROWP: every row's prefix sums come from the row-prefix table built at bind
// (one coalesced fp64 load per row and task: no mixed-radix decode of the row,
// no gathers of the first R-groups' contributions).
#ifdef APEX_SCAN_TIME
// per-warp start / end times and item counts of the sorted-column scan (debug builds: -DAPEX_SCAN_TIME)
__device__ unsigned long long g_wt[16384][3];
__device__ unsigned g_wt_n, g_wt_done;
#endif
#ifdef APEX_SCAN_PROF
// per-phase cycle totals of the sorted-column scan (debug builds: -DAPEX_SCAN_PROF)
__device__ unsigned long long g_scan_prof[16];
// warp start min/max, end min/max, span sum, warps, max item cycles, max item pairs
__device__ unsigned long long g_scan_t[8] = {~0ull, 0, ~0ull, 0, 0, 0, 0, 0};
__device__ unsigned long long g_scan_hist[64];  // items by log2(cycles) / by log2(admitted pairs + 1)
__device__ unsigned g_scan_done;
#endif
template <bool P16, bool ROWP>
__global__ void __launch_bounds__(kScanWarps * 32, APEX_SORTED_MINB) scan_sorted_kernel(const ScanLaunch L, const SortedLaunch S) {
  extern __shared__ __align__(16) float sm_s[];
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  const unsigned long long live = live_mask(L, 0u);
  if (!live) return;
  float* sthr = sm_s + (size_t)warp * kMaxTests * 32;  // [test][lane]: signed-value thresholds of every test
  int4* scb = reinterpret_cast<int4*>(sm_s + (size_t)kScanWarps * kMaxTests * 32) + warp * 32;  // pre-pass best range
#if APEX_CAND_STAGE
  Entry* stg = reinterpret_cast<Entry*>(reinterpret_cast<int4*>(sm_s + (size_t)kScanWarps * kMaxTests * 32) +
                                        kScanWarps * 32) + warp * kCandStage;  // staged candidates
#endif
  WorkCursor wc;
  const float* __restrict__ values = L.values;
  const float* __restrict__ p16 = S.packed16;
  const int64_t n_pairs = L.n_pairs;
  __shared__ unsigned s_adm[64];  // admitted products per query of the launch (statistics)
  __shared__ unsigned s_live[64];  // enumerated pairs per query not yet flushed to the pair budget
#if APEX_TILE_SMEM
  // the launch's control-block pointers, and each warp's next tile copied in
  // the background (cp.async) while the current item runs: neither is a
  // dependent global load at the top of an item
  __shared__ QCtl* s_ctl[64];
  __shared__ __align__(16) Tile s_tile[kScanWarps];
  for (int q = threadIdx.x; q < L.nq; q += blockDim.x) s_ctl[q] = L.queries[q].ctl;
#endif
  for (int q = threadIdx.x; q < 64; q += blockDim.x) s_adm[q] = s_live[q] = 0;
  __syncthreads();
  auto ld = [&](int task, int64_t pair) -> float {
    return P16 ? __ldg(p16 + pair * 16 + task) : __ldg(values + (int64_t)task * n_pairs + pair);
  };

  unsigned qi, t;
  bool have = (L.n_ctr > 1 ? next_item_multi(L, wc, live, lane, qi, t) : next_item(L, wc, live, lane, qi, t));
  Tile T_n;
  unsigned long long tau_n = 0;
#if APEX_TILE_SMEM
  auto fetch_next = [&]() {
    if (lane < sizeof(Tile) / 8)
      cp_async8(reinterpret_cast<uint64_t*>(&s_tile[warp]) + lane, reinterpret_cast<const uint64_t*>(L.tiles + t) + lane);
    cp_async_commit();
    tau_n = ld_relaxed_u64(&s_ctl[qi]->tau_key);
  };
  if (have) fetch_next();
#else
  if (have) {
    T_n = L.tiles[t];
    tau_n = ld_relaxed_u64(&L.queries[qi].ctl->tau_key);
  }
#endif
#ifdef APEX_SCAN_PROF
  unsigned long long prof[16] = {}, tp = clock64();
  const unsigned long long g_start = globaltimer_ns();
#endif
#ifdef APEX_SCAN_TIME
  const unsigned long long w_start = globaltimer_ns();
  unsigned long long w_items = 0, w_last = w_start;
  unsigned w_rounds = 0, w_crounds = 0, w_refresh = 0, w_cand = 0, w_maxitem_rounds = 0;
  unsigned long long w_maxitem = 0;
#endif
  bool pending = false;  // the next item is fetched after this one (tail window)
  for (;;) {
    if (pending) {
      pending = false;
      have = (L.n_ctr > 1 ? next_item_multi(L, wc, live, lane, qi, t) : next_item(L, wc, live, lane, qi, t));
#if APEX_TILE_SMEM
      if (have) fetch_next();
#else
      if (have) {
        T_n = L.tiles[t];
        tau_n = ld_relaxed_u64(&L.queries[qi].ctl->tau_key);
      }
#endif
    }
    if (!have) break;
#ifdef APEX_SCAN_PROF
    const unsigned long long t_item = clock64();
#endif
#ifdef APEX_SCAN_TIME
    ++w_items;
    w_last = globaltimer_ns();
#endif
    const unsigned q_cur = qi, t_cur = t;
#if APEX_TILE_SMEM
    cp_async_wait_all();
    __syncwarp();
    T_n = s_tile[warp];
    __syncwarp();  // every lane has the tile before the next copy lands
#endif
    const Tile T = T_n;
    const unsigned long long tau = tau_n;
#ifdef APEX_SCAN_PROF
    { const unsigned long long tn = clock64(); prof[14] += tn - tp; tp = tn; }
#endif
    if (wc.tail) {
      pending = true;
    } else {
      have = (L.n_ctr > 1 ? next_item_multi(L, wc, live, lane, qi, t) : next_item(L, wc, live, lane, qi, t));
#ifdef APEX_SCAN_PROF
      if (have && t == 0xffffffffu) prof[9] += 1;
      { const unsigned long long tn = clock64(); prof[15] += tn - tp; tp = tn; }
#endif
#if APEX_TILE_SMEM
      if (have) fetch_next();
#else
      if (have) {
        T_n = L.tiles[t];
        tau_n = ld_relaxed_u64(&L.queries[qi].ctl->tau_key);
      }
#endif
    }
#ifdef APEX_SCAN_PROF
    if (have && t == 0xffffffffu) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[0] += tn - tp; tp = tn; }
#endif
    const ScanQuery& Q = L.queries[q_cur];
#if APEX_TILE_SMEM
    QCtl* ctl = s_ctl[q_cur];
#else
    QCtl* ctl = Q.ctl;
#endif
    const int maximize = Q.maximize;
    const double b_obj = Q.test_bias[0];
    const int nt = Q.nt;
    const DevReaction& R = L.rx[T.rx];
#ifdef APEX_SCAN_PROF
    if (nt == 12345 || maximize == 12345) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[1] += tn - tp; tp = tn; }
#endif
    const int c = R.c;
    const int n_last = (int)R.size[c - 1];
    const int col_lo = (int)T.col0, col_hi = (int)(T.col0 + T.ncols);
    const int64_t last_pair = R.pair_off[c - 1];
#ifdef APEX_SCAN_PROF
    if (n_last == 12345 || last_pair == 12345) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[2] += tn - tp; tp = tn; }
#endif
    // shared constraint set: the pre-pass rows (every constraint threshold,
    // the most selective constraint and its exact range) copied to shared
    // memory in the background (cp.async) while the objective's chain runs
    const int cset = Q.cset;
    if (cset >= 0) {
      const int64_t slot = (int64_t)t_cur * 32 + lane;
      // a test's 32 row thresholds are 128 contiguous bytes: 8 lanes copy
      // one test with 16-byte copies (rows_pad is a multiple of 32)
      const float* cth = S.cthr + (int64_t)(Q.cset_off - 1) * S.rows_pad + (int64_t)t_cur * 32;
      for (int ch = lane + 8; ch < nt * 8; ch += 32)
        cp_async16(sthr + (ch >> 3) * 32 + (ch & 7) * 4, cth + (int64_t)(ch >> 3) * S.rows_pad + (ch & 7) * 4);
      cp_async16(scb + lane, S.cbest + (int64_t)cset * S.rows_pad + slot);
      cp_async_commit();
    }

    const bool valid = lane < T.nrows;
    const uint64_t row = T.row0 + (valid ? lane : 0u);
    int64_t pr[kMaxRg - 1];
    const double* rowp = ROWP ? S.rowp + R.row_off + (int64_t)row : nullptr;
    if (!ROWP) decode_prefix(R, c, row, pr);
    const unsigned long long gbase = R.g_off + row * (uint64_t)n_last;
    // the objective's exact per-row threshold (against tau, +inf without one)
    // and its passing count in quantile steps; only when that is not already
    // small are the constraint thresholds derived to find a more selective test
    double p_obj;
    if (ROWP) {
      p_obj = __ldg(rowp + Q.test_task[0] * S.rows_total);
    } else {
      const int task0 = Q.test_task[0];
      double p = c > 1 ? (double)ld(task0, pr[0]) : 0.0;
#pragma unroll
      for (int j = 1; j < kMaxRg - 1; ++j)
        if (j < c - 1) p = __dadd_rn(p, (double)ld(task0, pr[j]));
      p_obj = p;
    }
#ifdef APEX_SCAN_PROF
    if (__double_as_longlong(p_obj) == 0x123456789ll) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[3] += tn - tp; tp = tn; }
#endif
    float th0 = __int_as_float(0x7f800000);
    if (tau != kNoTau) {
      const double ts = key_to_score(tau);
      th0 = maximize ? -thr_lower_fast(p_obj, b_obj, ts) : thr_upper_fast(p_obj, b_obj, -ts);
    }
    sthr[lane] = th0;
    int best = 0;
    int start = 0, cnt = 0;
    int best_q = 0;
    const float* qbase = S.quant + (int64_t)T.rx * (kQuant + 1);  // + task * n_rx * (kQuant + 1)
    const int64_t qstride = (int64_t)S.n_rx * (kQuant + 1);
    if (valid && th0 == th0) {
      if (th0 == __int_as_float(0x7f800000)) {
        cnt = n_last;  // no threshold: every column passes the objective
        best_q = kQuant + 1;
      } else {
        const float* q = qbase + Q.test_task[0] * qstride;
        best_q = quant_count(q, maximize != 0, maximize ? -th0 : th0);
      }
    }
    bool cons_ready = false;
    // every constraint's exact threshold (and, when choosing, its passing
    // count in quantile steps), kThrBatch tests at a time so their gathers,
    // fp64 threshold math and quantile searches overlap instead of forming
    // one dependent chain per test
    auto constraint_thresholds = [&](bool choose) {
      for (int i0 = 1; i0 < nt; i0 += kThrBatch) {
        double p[kThrBatch];
        int task[kThrBatch];
#pragma unroll
        for (int u = 0; u < kThrBatch; ++u) {
          const int i = min(i0 + u, nt - 1);
          task[u] = Q.test_task[i];
          if (ROWP) {
            p[u] = __ldg(rowp + task[u] * S.rows_total);
          } else {
            double pp = c > 1 ? (double)ld(task[u], pr[0]) : 0.0;
            // fixed trip counts: pr stays in registers (a runtime-indexed pr
            // would live in local memory)
#pragma unroll
            for (int j = 1; j < kMaxRg - 1; ++j)
              if (j < c - 1) pp = __dadd_rn(pp, (double)ld(task[u], pr[j]));
            p[u] = pp;
          }
        }
        float th[kThrBatch];
        bool lower[kThrBatch];
#pragma unroll
        for (int u = 0; u < kThrBatch; ++u) {
          const int i = min(i0 + u, nt - 1);
          lower[u] = Q.test_lower[i] != 0;
          th[u] = lower[u] ? -thr_lower_fast(p[u], Q.test_bias[i], Q.test_beta[i])
                           : thr_upper_fast(p[u], Q.test_bias[i], Q.test_beta[i]);
          if (i0 + u < nt) sthr[(i0 + u) * 32 + lane] = th[u];
        }
        if (choose) {
          int qc[kThrBatch];
          quant_count4(qbase, qstride, task, lower, th, qc);
#pragma unroll
          for (int u = 0; u < kThrBatch; ++u)
            if (i0 + u < nt && qc[u] < best_q) {
              best_q = qc[u];
              best = i0 + u;
            }
        }
      }
      cons_ready = true;
    };
#ifdef APEX_SCAN_PROF
    if (best_q == 123456789) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[4] += tn - tp; tp = tn; }
#endif
    if (cset >= 0) {
      // (the pre-pass rows copied at the top of the item)
      cp_async_wait_all();
      __syncwarp();
      cons_ready = true;
      if (valid && best_q > 2 && nt > 1) {
        const int4 bc = scb[lane];
        if (bc.y < best_q) {
          best = bc.x;
          best_q = bc.y;
          start = bc.z;
          cnt = bc.w;
        }
      }
    } else {
      if (valid && best_q > 2 && nt > 1) constraint_thresholds(true);
      // exact passing range of a constraint that won, searched only inside
      // the quantile bracket its count identifies
      if (valid && best != 0) {
        start = 0;
        cnt = 0;
        if (best_q > 0) {
          const float th = sthr[best * 32 + lane];
          const bool lw = Q.test_lower[best] != 0;
          const int64_t base = (int64_t)Q.test_task[best] * S.pcols + R.pcol_off;
          exact_range(S.sx + base, n_last, lw, lw ? -th : th, best_q, start, cnt);
        }
      }
    }
#ifdef APEX_SCAN_PROF
    if (cnt == 123456789 || best == 77) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[5] += tn - tp; tp = tn; }
#endif
    // the objective's exact range when it is the most selective test
    if (valid && best == 0 && th0 == th0 && th0 != __int_as_float(0x7f800000)) {
      const int64_t base0 = (int64_t)Q.test_task[0] * S.pcols + R.pcol_off;
      exact_range(S.sx + base0, n_last, maximize != 0, maximize ? -th0 : th0, best_q, start, cnt);
    }
#ifdef APEX_SCAN_PROF
    if (cnt == 123456789) prof[9] += 1;
    { const unsigned long long tn = clock64(); prof[6] += tn - tp; tp = tn; }
#endif
    if (cnt > 0 && !cons_ready) constraint_thresholds(false);
    // flatten the warp's admitted (row, sorted position) pairs so every lane
    // has one per round: rows pass only a few columns each in batched passes,
    // and a row-at-a-time walk leaves most lanes idle
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    // pair budget (automatic kernel choice): the pairs this query enumerates
    // are summed per CTA and flushed to its control block every kBailFlush;
    // past the budget the query is given up — its admission key is raised to
    // the maximum, so its remaining items enumerate nothing — and the host
    // re-runs it with the full predicate, which is cheaper for such queries
    if (total > 0 && Q.admit_budget != ~0ull && lane == 0) {
      const unsigned old = atomicAdd(&s_live[q_cur], (unsigned)total);
      if ((unsigned long long)(old + (unsigned)total) >= min((unsigned long long)kBailFlush, Q.admit_budget)) {
        const unsigned v = atomicExch(&s_live[q_cur], 0u);
        if (v && atomicAdd(&ctl->admit_live, (unsigned long long)v) + v > Q.admit_budget &&
            ld_relaxed_u64(&ctl->tau_key) != ~0ull) {
          const unsigned long long prev = atomicExch(&ctl->tau_key, ~0ull);
          if (prev != ~0ull) {
            ctl->bail_tau = prev;
            ctl->bail = 1u;
          }
        }
      }
    }
    // sorted position of flat index j of this lane's row: sbase + j
    const int64_t sbase = (int64_t)Q.test_task[best] * S.pcols + R.pcol_off + start - (incl - cnt);
    __syncwarp();
    unsigned admitted = 0;
    // control fields fixed during the enumeration (set by the control init
    // and the seed), read once per item rather than per candidate
    bool tie_on = false;
    unsigned long long hist_base = 0;
    unsigned hist_shift = 0;
    if (total > 0) {
      tie_on = __ldcg(&ctl->tie_on) != 0;
      hist_base = __ldcg(&ctl->hist_base);
      hist_shift = __ldcg(&ctl->hist_shift);
    }
#ifdef APEX_SCAN_TIME
    w_rounds += (total + 31) / 32;
#endif
#if APEX_CAND_STAGE
    unsigned n_stg = 0;  // warp-uniform
    auto flush_stage = [&]() {
      __syncwarp();
      unsigned long long cb = 0;
      if (lane == 0) cb = atomicAdd(&ctl->count, (unsigned long long)n_stg);
      cb = __shfl_sync(0xffffffffu, cb, 0);
      for (unsigned i = lane; i < n_stg; i += 32)
        if (cb + i < Q.cap) Q.buf[cb + i] = stg[i];
      if ((cb >> Q.refresh_shift) != ((cb + n_stg) >> Q.refresh_shift)) {
        __threadfence();
        refresh_tau(Q);
      }
      n_stg = 0;
      __syncwarp();
    };
#endif
    for (int j0 = 0; j0 < total; j0 += 32) {
      // a query given up (pair budget) stops its items in flight too
      if (((j0 >> 5) & 15) == 15 && Q.admit_budget != ~0ull && ld_relaxed_u64(&ctl->tau_key) == ~0ull) break;
#ifdef APEX_SCAN_PROF
      const unsigned long long r_t0 = clock64();
#endif
      const int jj = j0 + (int)lane;
      const int j = jj < total ? jj : total - 1;
      // owning row: smallest r with incl[r] > j
      int lo = 0, hi = 31;
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int mid = (lo + hi) >> 1;
        if (__shfl_sync(0xffffffffu, incl, mid) > j) hi = mid; else lo = mid + 1;
      }
      const int r = lo;
      const int64_t sb = __shfl_sync(0xffffffffu, sbase, r);
      const double po = __shfl_sync(0xffffffffu, p_obj, r);
      const unsigned long long gb = __shfl_sync(0xffffffffu, gbase, r);
      bool ok = jj < total;
      int col = 0;
      if (ok) {
        col = (int)__ldg(S.scol + sb + j);
        ok = col >= col_lo && col < col_hi;
      }
      // every test on the pair (the chosen one passes by construction):
      // kPairBatch gathers in flight before any compare (they hit one 64-byte
      // line of the pair-major table), no short-circuit
      bool pass = ok;
      float xo = 0.0f;
      for (int i0 = 0; i0 < nt; i0 += kPairBatch) {
        float x[kPairBatch];
#pragma unroll
        for (int u = 0; u < kPairBatch; ++u)
          x[u] = (ok && i0 + u < nt) ? ld(Q.test_task[i0 + u], last_pair + col) : 0.0f;
        if (i0 == 0) xo = x[0];
#pragma unroll
        for (int u = 0; u < kPairBatch; ++u)
          if (i0 + u < nt) pass = pass && ((Q.test_lower[i0 + u] ? -x[u] : x[u]) <= sthr[(i0 + u) * 32 + r]);
      }
      admitted += ok ? 1u : 0u;
      Entry e;
      if (pass) {
        const double val = fx(po, xo, b_obj);
        e.key = skey(maximize ? val : -val);
        e.g = gb + (unsigned long long)col;
        pass = !(tie_on && tie_reject(ctl, e.key, e.g));
      }
      const unsigned mk = __ballot_sync(0xffffffffu, pass);
#ifdef APEX_SCAN_PROF
      if (mk == 0x12345u) prof[9] += 1;
      const unsigned long long r_t1 = clock64();
      prof[11] += r_t1 - r_t0;
      prof[10] += 1;
#endif
      if (!mk) continue;
#ifdef APEX_SCAN_TIME
      ++w_crounds;
      w_cand += __popc(mk);
#endif
#if APEX_CAND_STAGE
      // staged in the warp's shared-memory slots; the buffer append (one
      // atomic round trip) happens once per kCandStage - 31 candidates or at
      // the item's end instead of once per round (the histogram counts them
      // now, so the tau refresh sees them; every staged entry is flushed
      // before the item ends)
      if (pass) {
        stg[n_stg + __popc(mk & ((1u << lane) - 1u))] = e;
        const unsigned hb = tie_on ? cand_bin(ctl, e.key, e.g, hist_base, hist_shift) : hist_bin(e.key, hist_base, hist_shift);
        atomicAdd(&Q.hist[hb], 1u);
        atomicAdd(&Q.coarse[hb >> 8], 1u);
      }
      n_stg += __popc(mk);
      if (n_stg > (unsigned)(kCandStage - 32)) flush_stage();
#ifdef APEX_SCAN_PROF
      if (n_stg == 0x12345u) prof[9] += 1;
      prof[12] += clock64() - r_t1;
      prof[13] += 1;
#endif
#else
      unsigned long long cbase = 0;
      if (lane == 0) cbase = atomicAdd(&ctl->count, (unsigned long long)__popc(mk));
      cbase = __shfl_sync(0xffffffffu, cbase, 0);
      if (pass) {
        const unsigned long long idx = cbase + __popc(mk & ((1u << lane) - 1u));
        if (idx < Q.cap) Q.buf[idx] = e;
        const unsigned hb = tie_on ? cand_bin(ctl, e.key, e.g, hist_base, hist_shift) : hist_bin(e.key, hist_base, hist_shift);
        atomicAdd(&Q.hist[hb], 1u);
        atomicAdd(&Q.coarse[hb >> 8], 1u);
      }
      if ((cbase >> Q.refresh_shift) != ((cbase + __popc(mk)) >> Q.refresh_shift)) {
        __threadfence();
        refresh_tau(Q);
#ifdef APEX_SCAN_TIME
        ++w_refresh;
#endif
      }
#endif
    }
#if APEX_CAND_STAGE
    if (n_stg) flush_stage();
#endif

    __syncwarp();
    const unsigned a = __reduce_add_sync(0xffffffffu, admitted);
    if (a && lane == 0) atomicAdd(&s_adm[q_cur], a);  // per CTA; flushed once at the end
#ifdef APEX_SCAN_PROF
    if (lane == 0) {
      const unsigned long long dur = clock64() - t_item;
      atomicAdd(&g_scan_hist[min(31, 63 - __clzll(dur | 1))], 1ull);
      atomicAdd(&g_scan_hist[32 + min(31, 32 - __clz(total))], 1ull);
      atomicMax(&g_scan_t[6], dur);
      atomicMax(&g_scan_t[7], (unsigned long long)total);
    }
#endif
#ifdef APEX_SCAN_PROF
    prof[8] += 1;
    { const unsigned long long tn = clock64(); prof[7] += tn - tp; tp = tn; }
#endif
  }
#ifdef APEX_SCAN_TIME
  if (lane == 0 && globaltimer_ns() - w_start > 62000)
    printf("SCANLATE warp %u/%u items %llu rounds %u cand_rounds %u cand %u refresh %u span %llu ns last %llu ns\n",
           blockIdx.x, threadIdx.x >> 5, w_items, w_rounds, w_crounds, w_cand, w_refresh, globaltimer_ns() - w_start,
           globaltimer_ns() - w_last);
  if (lane == 0) {
    const unsigned slot = atomicAdd(&g_wt_n, 1u);
    if (slot < 16384) {
      g_wt[slot][0] = w_start;
      g_wt[slot][1] = globaltimer_ns();
      g_wt[slot][2] = w_items | ((globaltimer_ns() - w_last) << 20);
    }
  }
  __threadfence();
#endif
  __syncthreads();
  for (int q = threadIdx.x; q < L.nq; q += blockDim.x)
    if (s_adm[q]) atomicAdd(&L.queries[q].ctl->admitted, (unsigned long long)s_adm[q]);
#ifdef APEX_SCAN_TIME
  if (threadIdx.x == 0 && atomicAdd(&g_wt_done, 1u) == gridDim.x - 1) {
    const unsigned n = min(g_wt_n, 16384u);
    unsigned long long t0 = ~0ull;
    for (unsigned i = 0; i < n; ++i) t0 = min(t0, g_wt[i][0]);
    // end-time histogram in 4 us buckets, items per warp, last-item duration
    unsigned hist[64] = {};
    unsigned long long items = 0, last_sum = 0, last_max = 0, smax = 0;
    for (unsigned i = 0; i < n; ++i) {
      const unsigned long long e = (g_wt[i][1] - t0) / 4000;
      hist[min(63ull, e)]++;
      items += g_wt[i][2] & 0xfffff;
      last_sum += g_wt[i][2] >> 20;
      last_max = max(last_max, g_wt[i][2] >> 20);
      smax = max(smax, g_wt[i][0] - t0);
    }
    printf("SCANWARPS %u warps, items/warp %.2f, last start +%llu ns, last-item mean %llu ns max %llu ns\n", n,
           (double)items / n, smax, last_sum / n, last_max);
    for (int b = 0; b < 64; ++b)
      if (hist[b]) printf("SCANEND %3d-%3d us: %u warps\n", 4 * b, 4 * b + 4, hist[b]);
    g_wt_n = 0;
    g_wt_done = 0;
  }
#endif
#ifdef APEX_SCAN_PROF
  if (lane == 0) {
    const unsigned long long g_end = globaltimer_ns();
    atomicMin(&g_scan_t[0], g_start);
    atomicMax(&g_scan_t[1], g_start);
    atomicMin(&g_scan_t[2], g_end);
    atomicMax(&g_scan_t[3], g_end);
    atomicAdd(&g_scan_t[4], g_end - g_start);
    atomicAdd(&g_scan_t[5], 1ull);
  }
  if (lane == 0)
    for (int i = 0; i < 16; ++i) if (i != 9) atomicAdd(&g_scan_prof[i], prof[i]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&g_scan_done, 1u) == gridDim.x - 1) {
    const unsigned long long n = g_scan_prof[8] ? g_scan_prof[8] : 1;
    printf("SCANPROF items %llu cycles/item: next %llu Q %llu R %llu p_obj %llu thr+quant %llu cset %llu range %llu "
           "pairs %llu\n", g_scan_prof[8], g_scan_prof[0] / n, g_scan_prof[1] / n, g_scan_prof[2] / n,
           g_scan_prof[3] / n, g_scan_prof[4] / n, g_scan_prof[5] / n, g_scan_prof[6] / n, g_scan_prof[7] / n);
    printf("SCANNEXT cycles/item: loop top %llu, next_item %llu, loads %llu\n", g_scan_prof[14] / n, g_scan_prof[15] / n,
           g_scan_prof[0] / n);
    printf("SCANROUNDS %llu rounds, cycles/round: to ballot %llu, append %llu (rounds with candidates %llu)\n",
           g_scan_prof[10], g_scan_prof[11] / (g_scan_prof[10] ? g_scan_prof[10] : 1),
           g_scan_prof[12] / (g_scan_prof[13] ? g_scan_prof[13] : 1), g_scan_prof[13]);
    printf("SCANTIME warps %llu: first start +0, last start +%llu ns, first end +%llu, last end +%llu, mean warp span %llu ns\n",
           g_scan_t[5], g_scan_t[1] - g_scan_t[0], g_scan_t[2] - g_scan_t[0], g_scan_t[3] - g_scan_t[0],
           g_scan_t[4] / (g_scan_t[5] ? g_scan_t[5] : 1));
    printf("SCANITEMS max cycles %llu max pairs %llu\n", g_scan_t[6], g_scan_t[7]);
    for (int i = 0; i < 32; ++i)
      if (g_scan_hist[i] || g_scan_hist[32 + i])
        printf("SCANHIST 2^%d: items by cycles %llu | by pairs (<2^%d) %llu\n", i, g_scan_hist[i], i, g_scan_hist[32 + i]);
    for (int i = 0; i < 64; ++i) g_scan_hist[i] = 0;
    g_scan_t[6] = g_scan_t[7] = 0;
    for (int i = 0; i < 16; ++i) g_scan_prof[i] = 0;
    g_scan_t[0] = g_scan_t[2] = ~0ull;
    g_scan_t[1] = g_scan_t[3] = g_scan_t[4] = g_scan_t[5] = 0;
    g_scan_done = 0;
  }
#endif
}

// ---------------------------------------------------------------------------
// Seed: exact evaluation of S sampled products (without replacement: one per
// equal cell of [start, end), jittered inside the cell).  Feasible samples are
// counted in seed_hist by key >> 48; the k-th best sampled key bin is a valid
// admission threshold because the samples are distinct real products.

struct SampleLaunch {
  const ScanQuery* queries;
  const DevReaction* rx;
  const unsigned long long* g_off;   // [n_rx + 1]
  int n_rx;
  const float* values;
  const float* p16;                  // pair-major copy or null
  int64_t n_pairs;
  unsigned long long start, end, samples;
};

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

__global__ void sample_kernel(const SampleLaunch P, int nq) {
  // grid.y = query: every query evaluates the same sampled products (the
  // decode is repeated per query, it is ALU-only); each test's fp64 sum is
  // formed without short-circuit so all of a sample's loads are in flight
  // together (the kernel is gather-latency bound)
  const ScanQuery& Q = P.queries[blockIdx.y];
  if (!*(volatile unsigned int*)&Q.ctl->active) return;
  (void)nq;
  const unsigned long long span = P.end - P.start, S = P.samples;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned lane = lane_id();
  const int nt = Q.nt;
  unsigned long long mx = 0;
  for (unsigned long long base_i = (unsigned long long)blockIdx.x * blockDim.x; base_i < S; base_i += stride) {
    const unsigned long long i = base_i + threadIdx.x;
    unsigned long long key = 0;
    if (i < S) {
      int64_t pr[kMaxRg];
      const unsigned long long lo = (unsigned long long)(((unsigned __int128)span * i) / S);
      const unsigned long long hi = (unsigned long long)(((unsigned __int128)span * (i + 1)) / S);
      const unsigned long long g = P.start + lo + mix64(i * 0x9e3779b97f4a7c15ull + 17) % (hi - lo);
      int a = 0, b = P.n_rx;
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (P.g_off[mid] <= g) a = mid; else b = mid;
      }
      const DevReaction& R = P.rx[a];
      const int c = R.c;
      uint64_t rem = g - R.g_off;
#pragma unroll
      for (int j = kMaxRg - 1; j >= 0; --j) {
        pr[j] = 0;
        if (j < c) {
          uint64_t q, d;
          divmod_u64(q, d, rem, (uint64_t)R.size[j]);
          pr[j] = R.pair_off[j] + (int64_t)d;
          rem = q;
        }
      }
      bool feasible = true;
      double vobj = 0.0;
      for (int t = 0; t < nt; ++t) {
        const int task = Q.test_task[t];
        double val = (double)tval(P.values, P.p16, P.n_pairs, task, pr[0]);
#pragma unroll
        for (int j = 1; j < kMaxRg; ++j)
          if (j < c) val = __dadd_rn(val, (double)tval(P.values, P.p16, P.n_pairs, task, pr[j]));
        val = __dadd_rn(val, Q.test_bias[t]);
        if (t == 0) vobj = val;
        else feasible = feasible && (Q.test_lower[t] ? (val >= Q.test_beta[t]) : (val <= Q.test_beta[t]));
      }
      if (feasible) key = skey(Q.maximize ? vobj : -vobj);
    }
    hist_add_warp(Q.seed_hist, (unsigned)(key >> 48), key != 0);
    hist_add_warp(Q.seed_hist + 2 * kHistBins, (unsigned)(key >> 56), key != 0);
    mx = max(mx, key);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0 && mx) atomicMax(&Q.ctl->seed_max, mx);
}

// ---------------------------------------------------------------------------
// Seed, part 2: the "corner" of every reaction — all combinations of the
// best-m synthons of each R-group for the query's objective direction (lists
// precomputed per task at table load).  For additive scores the top-k products
// concentrate there, so the k-th best feasible corner product is a tight,
// valid admission threshold.  Counted in seed_hist[kHistBins ..] (disjoint
// from the uniform samples' histogram).
struct CornerLaunch {
  const ScanQuery* queries;
  const DevReaction* rx;
  const float* values;
  const float* p16;                  // pair-major copy or null
  int64_t n_pairs;
  const int32_t* lists;              // [n_tasks][2][slots] digits, best-first (dir 0 = largest, 1 = smallest)
  const int32_t* slot_off;           // [n_rx * kMaxRg] offset of (t, j)'s list within a (task, dir) block
  const int32_t* m;                  // [n_rx * kMaxRg] list length of (t, j)
  const unsigned long long* coff;    // (unused)
  int n_rx;
  int64_t slots;                     // list entries per (task, dir)
  unsigned long long start, end;
  int budget;                        // corner products per reaction
};

// one CTA per (reaction, query): the best-m' x ... x best-m' combinations,
// m' = floor(budget^(1/c)) capped by the list lengths
__global__ void corner_kernel(const CornerLaunch P) {
  const ScanQuery& Q = P.queries[blockIdx.y];
  if (!*(volatile unsigned int*)&Q.ctl->active) return;
  const int t = blockIdx.x;
  const DevReaction& R = P.rx[t];
  const unsigned long long off = R.g_off;
  const unsigned long long rsize = R.n_rows * (unsigned long long)R.size[R.c - 1];
  if (off + rsize <= P.start || off >= P.end) return;
  int mb = P.budget;
  if (R.c == 2) mb = (int)sqrtf((float)P.budget);
  else if (R.c == 3) mb = (int)cbrtf((float)P.budget + 0.5f);
  else if (R.c >= 4) mb = (int)powf((float)P.budget, 1.0f / R.c);
  mb = max(mb, 1);
  // fixed trip counts with guards throughout: the per-R-group arrays stay in
  // registers (runtime-indexed, they would live in local memory)
  int mj[kMaxRg];
  unsigned total = 1;
#pragma unroll
  for (int j = 0; j < kMaxRg; ++j) {
    mj[j] = 1;
    if (j < R.c) {
      mj[j] = min(mb, P.m[t * kMaxRg + j]);
      total *= (unsigned)mj[j];
    }
  }
  const int dir = Q.maximize ? 0 : 1;
  const int32_t* list = P.lists + ((int64_t)Q.test_task[0] * 2 + dir) * P.slots;
  const unsigned lane = lane_id();
  // grid.z CTAs share a reaction's corner (few reactions x queries: C4 has
  // 120 reactions and one query, so one CTA per reaction left SMs idle)
  for (unsigned base_i = blockIdx.z * blockDim.x; base_i < total; base_i += blockDim.x * gridDim.z) {
    const unsigned i = base_i + threadIdx.x;
    unsigned long long key = 0;
    if (i < total) {
      unsigned rem = i;
      int64_t pr[kMaxRg];
      int64_t dig[kMaxRg];
#pragma unroll
      for (int j = kMaxRg - 1; j >= 0; --j) {
        dig[j] = 0;
        pr[j] = 0;
        if (j < R.c) {
          const unsigned idx = rem % (unsigned)mj[j];
          rem /= (unsigned)mj[j];
          dig[j] = list[P.slot_off[t * kMaxRg + j] + idx];
          pr[j] = R.pair_off[j] + dig[j];
        }
      }
      unsigned long long g = 0;
#pragma unroll
      for (int j = 0; j < kMaxRg; ++j)
        if (j < R.c) g = g * (unsigned long long)R.size[j] + (unsigned long long)dig[j];
      g += off;
      if (g >= P.start && g < P.end) {
        bool feasible = true;
        for (int tt = 1; tt < Q.nt && feasible; ++tt) {
          const int task = Q.test_task[tt];
          double val = (double)tval(P.values, P.p16, P.n_pairs, task, pr[0]);
#pragma unroll
          for (int j = 1; j < kMaxRg; ++j)
            if (j < R.c) val = __dadd_rn(val, (double)tval(P.values, P.p16, P.n_pairs, task, pr[j]));
          val = __dadd_rn(val, Q.test_bias[tt]);
          feasible = Q.test_lower[tt] ? (val >= Q.test_beta[tt]) : (val <= Q.test_beta[tt]);
        }
        if (feasible) {
          const int task = Q.test_task[0];
          double val = (double)tval(P.values, P.p16, P.n_pairs, task, pr[0]);
#pragma unroll
          for (int j = 1; j < kMaxRg; ++j)
            if (j < R.c) val = __dadd_rn(val, (double)tval(P.values, P.p16, P.n_pairs, task, pr[j]));
          val = __dadd_rn(val, Q.test_bias[0]);
          key = skey(Q.maximize ? val : -val);
        }
      }
    }
    hist_add_warp(Q.seed_hist + kHistBins, (unsigned)(key >> 48), key != 0);
    hist_add_warp(Q.seed_hist + 2 * kHistBins + 256, (unsigned)(key >> 56), key != 0);
    unsigned long long mx = key;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx) atomicMax(&Q.ctl->seed_max, mx);
  }
}

// tau from key histograms, one warp per query (two-level search).  At least k
// distinct feasible products have key >= the returned bin's lower edge, so it
// is a valid lower bound on the final k-th best key.
//   mode 0: seed — max over the uniform-sample and the corner histograms
//           (separate, so no product is counted twice); the candidate
//           histogram is then re-based on tau with the seeded range [tau,
//           seed_max] spread over ~1/4 of its bins;
//   mode 1: raise tau from the candidate histogram;
//   mode 2: final bound (and the count at/above it) for the select.
constexpr double kSortedFeasibleMax = 65536.0;  // auto choice: estimated feasible products above this -> full predicate
__global__ void tau_kernel(const ScanQuery* __restrict__ qs, int nq, int mode, int auto_kernel = 0,
                           unsigned long long samples = 0, unsigned long long span = 0) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const ScanQuery& Q = qs[q];
  QCtl* ctl = Q.ctl;
  if (!*(volatile unsigned int*)&ctl->active) return;
  const unsigned long long k = (unsigned long long)Q.k;
  const bool lead = lane_id() == 0;
  unsigned long long cnt = 0;
  if (mode == 0) {
    // the two seed histograms (uniform samples, corner) searched together:
    // both coarse levels in flight, then both fine levels
    unsigned v0[8], v1[8];
    load_bins256(Q.seed_hist + 2 * kHistBins, v0);
    load_bins256(Q.seed_hist + 2 * kHistBins + 256, v1);
    unsigned long long a0 = 0, a1 = 0;
    const int c0 = kth_bins256(v0, k, a0, nullptr);
    const int c1 = kth_bins256(v1, k, a1, nullptr);
    if (c0 >= 0) load_bins256(Q.seed_hist + (c0 << 8), v0);
    if (c1 >= 0) load_bins256(Q.seed_hist + kHistBins + (c1 << 8), v1);
    int b0 = -1, b1 = -1;
    if (c0 >= 0) {
      const int f = kth_bins256(v0, k, a0, nullptr);
      b0 = f < 0 ? c0 << 8 : (c0 << 8) | f;
    }
    if (c1 >= 0) {
      const int f = kth_bins256(v1, k, a1, nullptr);
      b1 = f < 0 ? c1 << 8 : (c1 << 8) | f;
    }
    if (lead) {
      unsigned long long key = kNoTau;
      if (b0 >= 0) key = (unsigned long long)b0 << 48;
      if (b1 >= 0) key = max(key, (unsigned long long)b1 << 48);
      if (key > ctl->tau_key) ctl->tau_key = key;
      if (ctl->tau_key != kNoTau) {
        const unsigned long long base = ctl->tau_key;
        const unsigned long long range = ctl->seed_max > base ? ctl->seed_max - base : 0ull;
        unsigned shift = 0;
        while (shift < 48 && (range >> shift) >= 16384ull) ++shift;
        ctl->hist_base = base;
        ctl->hist_shift = shift;
      }
      // automatic kernel choice: without a seeded threshold (fewer than k
      // feasible seed products) the admission test admits nearly everything,
      // so the full-predicate kernel is cheaper
      // (auto 2: the sorted-column kernel enumerates the most selective
      // test per row, so only an unconstrained query without a threshold
      // needs the full predicate)
      if (auto_kernel == 1) ctl->use_full = ctl->tau_key == kNoTau ? 1u : 0u;
      // (auto 2 keeps the full predicate for threshold-less queries whose
      // feasible set is not sparse — the uniform samples found more than
      // 1/512 feasible: there the streaming full predicate beats enumerating
      // broad sorted ranges; sparse ones (e.g. Astex RO3) take the sorted kernel)
      // ... and for threshold-less queries whose feasible set, estimated from
      // the samples, is large in absolute terms: without a threshold the
      // sorted-column kernel appends every feasible product it enumerates
      // (~20 ns each), the full predicate costs ~1 ps per product
      // (C5 over 1e9: 1.1M feasible of 1e9 took 23 ms sorted, 0.9 ms full)
      if (auto_kernel == 2)
        ctl->use_full = (ctl->tau_key == kNoTau &&
                         (Q.nt == 1 || a0 * 512ull > samples ||
                          (samples > 0 && (double)a0 * (double)span / (double)samples > kSortedFeasibleMax)))
                            ? 1u : 0u;
      if (auto_kernel == 3) ctl->use_full = 0u;  // no full-predicate launch in this pass
    }
  } else {
    if (*(volatile unsigned int*)&ctl->tie_on) return;  // tie mode: bins are g ranges (finalize_small_kernel)
    const int B = kth_two_level(Q.hist, Q.coarse, k, &cnt);
    if (lead) {
      if (mode == 1) {
        if (B >= 0) {
          const unsigned long long key = bin_edge((unsigned)B, ctl->hist_base, ctl->hist_shift);
          if (key > ctl->tau_key) ctl->tau_key = key;
        }
        ctl->tile_counter = 0;
      } else {
        ctl->bound_key = B >= 0 ? bin_edge((unsigned)B, ctl->hist_base, ctl->hist_shift) : 0ull;
        ctl->comp_count = cnt;  // candidates with key >= bound
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K5: exact top-k over comp[0, comp_count) by the composite order
// (key desc, g asc): MSB-first radix select over the 128-bit composite
// (key, ~g), 8-bit digits, histograms in smem + global, one grid barrier per
// digit among the CTAs of a query (cooperative launch => co-resident).
__device__ __forceinline__ void query_barrier(unsigned int* ctr, unsigned nb, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned target = gen * nb;
    while (ld_acquire_u32(ctr) < target) __nanosleep(20);
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned digit_of(const Entry& e, int p) {
  return p < 8 ? (unsigned)(e.key >> (56 - 8 * p)) & 0xffu : (unsigned)((~e.g) >> (56 - 8 * (p - 8))) & 0xffu;
}
// top 8p bits of the composite equal the prefix?
__device__ __forceinline__ bool match_prefix(const Entry& e, unsigned long long phi, unsigned long long plo, int p) {
  if (p == 0) return true;
  if (p < 8) return (e.key >> (64 - 8 * p)) == (phi >> (64 - 8 * p));
  if (e.key != phi) return false;
  if (p == 8) return true;
  return ((~e.g) >> (128 - 8 * p)) == (plo >> (128 - 8 * p));
}
// top 8d bits of the composite >= prefix?
__device__ __forceinline__ bool ge_prefix(const Entry& e, unsigned long long phi, unsigned long long plo, int d) {
  if (d <= 8) {
    if (d == 8) return e.key >= phi;
    return (e.key >> (64 - 8 * d)) >= (phi >> (64 - 8 * d));
  }
  if (e.key != phi) return e.key > phi;
  if (d == 16) return (~e.g) >= plo;
  return ((~e.g) >> (128 - 8 * d)) >= (plo >> (128 - 8 * d));
}

__global__ void __launch_bounds__(kSelectThreads) select_kernel(const ScanQuery* __restrict__ qs) {
  const ScanQuery& Q = qs[blockIdx.y];
  QCtl* ctl = Q.ctl;
  if (!*(volatile unsigned int*)&ctl->active || *(volatile unsigned int*)&ctl->small_done) return;
  __shared__ unsigned int sh[256];
  __shared__ unsigned long long s_phi, s_plo, s_need;
  __shared__ int s_depth;
  __shared__ unsigned long long s_min[kSelectThreads / 32];
  const unsigned tid = threadIdx.x, nb = gridDim.x;
  unsigned gen = 0;
  // candidates at/above the final bound (counted by tau_kernel mode 2); the
  // select reads the candidate buffer directly and ignores keys below it
  const unsigned long long n_valid = *(volatile unsigned long long*)&ctl->comp_count;
  const unsigned long long n = min(*(volatile unsigned long long*)&ctl->count, Q.cap);
  const unsigned long long bound = *(volatile unsigned long long*)&ctl->bound_key;
  const unsigned long long k = (unsigned long long)Q.k;
  const Entry* __restrict__ in = Q.buf;
  const unsigned long long start = (unsigned long long)blockIdx.x * blockDim.x + tid;
  const unsigned long long stride = (unsigned long long)nb * blockDim.x;

  const bool take_all = n_valid <= k;
  unsigned long long phi = 0, plo = 0;
  int depth = 0;
  if (!take_all) {
    if (tid == 0) { s_need = k; s_phi = 0; s_plo = 0; s_depth = -1; }
    for (int p = 0; p < 16; ++p) {
      for (unsigned i = tid; i < 256; i += blockDim.x) sh[i] = 0u;
      __syncthreads();
      phi = s_phi; plo = s_plo;
      for (unsigned long long i = start; i < n; i += stride) {
        const Entry e = in[i];
        if (e.key >= bound && match_prefix(e, phi, plo, p)) atomicAdd(&sh[digit_of(e, p)], 1u);
      }
      __syncthreads();
      unsigned int* gh = ctl->hist[p % 3];
      for (unsigned i = tid; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
      if (blockIdx.x == 0)
        for (unsigned i = tid; i < 256; i += blockDim.x) ctl->hist[(p + 1) % 3][i] = 0u;
      query_barrier(&ctl->barrier, nb, gen);
      for (unsigned i = tid; i < 256; i += blockDim.x) sh[i] = __ldcg(&gh[i]);
      __syncthreads();
      if (tid == 0) {
        unsigned long long need = s_need, cum = 0;
        int sel = 0;
        for (int b = 255; b >= 0; --b) {
          if (cum + sh[b] >= need) { sel = b; break; }
          cum += sh[b];
        }
        need -= cum;
        if (p < 8) s_phi = s_phi | ((unsigned long long)sel << (56 - 8 * p));
        else s_plo = s_plo | ((unsigned long long)sel << (56 - 8 * (p - 8)));
        s_need = need;
        if (sh[sel] == need) s_depth = p + 1;
      }
      __syncthreads();
      if (s_depth > 0) break;
    }
    phi = s_phi; plo = s_plo; depth = s_depth;
  }
  // compaction of the selected set + min key
  unsigned long long mn = ~0ull;
  const unsigned lane = tid & 31u;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x + (tid & ~31u); base < n; base += stride) {
    const unsigned long long i = base + lane;
    Entry e;
    bool keep = false;
    if (i < n) {
      e = in[i];
      keep = e.key >= bound && (take_all || ge_prefix(e, phi, plo, depth));
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned pos = 0;
      if ((int)lane == leader) pos = atomicAdd(&ctl->out_count, (unsigned)__popc(m));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (keep) {
        Q.sel[pos + __popc(m & ((1u << lane) - 1u))] = e;
        mn = min(mn, e.key);
      }
    }
  }
  for (int off = 16; off; off >>= 1) mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, off));
  if (lane == 0) s_min[tid >> 5] = mn;
  __syncthreads();
  if (tid == 0) {
    for (unsigned w = 1; w < blockDim.x / 32; ++w) mn = min(mn, s_min[w]);
    if (mn != ~0ull) atomicMin(&ctl->min_key, mn);
  }
  query_barrier(&ctl->barrier, nb, gen);
  if (blockIdx.x == 0 && tid == 0) {
    const unsigned long long cnt = *(volatile unsigned int*)&ctl->out_count;
    ctl->sel_count = cnt;
    if (cnt == k && k > 0) {
      const unsigned long long mk = *(volatile unsigned long long*)&ctl->min_key;
      if (mk > ctl->tau_key) ctl->tau_key = mk;
    }
  }
}

// ---------------------------------------------------------------------------
// Strides s_hi..1 (s_hi < 32) of the bitonic merge of blocks of `size`, in
// registers: lane (i & 31) holds element i, its partner i ^ s is a lane of the
// same warp.  Best-first within segments whose `size` bit is clear.
__device__ __forceinline__ void bitonic_warp_steps(Entry& e, unsigned i, unsigned size, unsigned s_hi) {
  for (unsigned s = s_hi; s > 0; s >>= 1) {
    Entry o;
    o.key = __shfl_xor_sync(0xffffffffu, e.key, s);
    o.g = __shfl_xor_sync(0xffffffffu, e.g, s);
    const bool lower = (i & s) == 0, best_first = (i & size) == 0;
    const bool o_better = entry_better(o, e);
    if (lower == best_first ? o_better : !o_better) e = o;
  }
}

// Best-first bitonic sort of P (a power of two) entries in shared memory by
// the whole block (blockDim a multiple of 32); (key, g) pairs are unique, so
// the order is total.  Strides >= 32 compare-exchange through shared memory
// (one pair per thread, a barrier per stride); the strides below 32 of every
// merge run in registers with warp shuffles, one barrier per merge size.
__device__ void bitonic_best_first(Entry* es, unsigned P) {
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, n_warps = blockDim.x >> 5;
  const unsigned chunks = P >= 32 ? P >> 5 : 0;
  if (chunks == 0) {  // tiny: thread 0 insertion sort
    if (threadIdx.x == 0) {
      for (unsigned i = 1; i < P; ++i) {
        const Entry x = es[i];
        unsigned j = i;
        for (; j > 0 && entry_better(x, es[j - 1]); --j) es[j] = es[j - 1];
        es[j] = x;
      }
    }
    __syncthreads();
    return;
  }
  for (unsigned c = warp; c < chunks; c += n_warps) {
    const unsigned i = (c << 5) | lane;
    Entry e = es[i];
    for (unsigned size = 2; size <= 32; size <<= 1) bitonic_warp_steps(e, i, size, size >> 1);
    es[i] = e;
  }
  __syncthreads();
  for (unsigned size = 64; size <= P; size <<= 1) {
    for (unsigned stride = size >> 1; stride >= 32; stride >>= 1) {
      // one compare-exchange per thread and pair: pair p -> (i, i + stride)
      for (unsigned p = threadIdx.x; p < (P >> 1); p += blockDim.x) {
        const unsigned i = ((p & ~(stride - 1)) << 1) | (p & (stride - 1));
        const unsigned j = i + stride;
        const Entry a = es[i], b = es[j];
        const bool want_a_first = (i & size) == 0;
        const bool b_better = entry_better(b, a);
        if (want_a_first ? b_better : !b_better) {
          es[i] = b;
          es[j] = a;
        }
      }
      __syncthreads();
    }
    for (unsigned c = warp; c < chunks; c += n_warps) {
      const unsigned i = (c << 5) | lane;
      Entry e = es[i];
      bitonic_warp_steps(e, i, size, 16);
      es[i] = e;
    }
    __syncthreads();
  }
}

// K6: best-first order of a large selected set in two launches.  (1) every
// kSortChunk-entry chunk of sel is sorted in shared memory, in place;
// (2) an entry's global rank is its position in its own chunk plus, for each
// other chunk, the number of that chunk's entries better than it (a binary
// search of the sorted chunk) — exact because the order is total — and it is
// scattered straight to sorted[rank].  O(n log n) work instead of the O(n^2)
// of rank counting.  Grids (chunks, queries) / (entry blocks, queries).
constexpr int kSortChunk = 2048;

__global__ void __launch_bounds__(1024) sort_chunks_kernel(const ScanQuery* __restrict__ qs) {
  const ScanQuery& Q = qs[blockIdx.y];
  if (*(volatile unsigned*)&Q.ctl->small_done) return;
  const unsigned long long n = *(volatile unsigned long long*)&Q.ctl->sel_count;
  const unsigned long long c0 = (unsigned long long)blockIdx.x * kSortChunk;
  if (c0 >= n) return;
  const unsigned len = (unsigned)min((unsigned long long)kSortChunk, n - c0);
  __shared__ Entry es[kSortChunk];
  unsigned P = 1;
  while (P < len) P <<= 1;
  for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < len) {
      es[i] = Q.sel[c0 + i];
    } else {
      es[i].key = 0;
      es[i].g = ~0ull;
    }
  }
  __syncthreads();
  bitonic_best_first(es, P);
  for (unsigned i = threadIdx.x; i < len; i += blockDim.x) Q.sel[c0 + i] = es[i];
}

__global__ void __launch_bounds__(256) merge_rank_kernel(const ScanQuery* __restrict__ qs) {
  const ScanQuery& Q = qs[blockIdx.y];
  if (*(volatile unsigned*)&Q.ctl->small_done) return;
  const unsigned long long n = *(volatile unsigned long long*)&Q.ctl->sel_count;
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Entry e = Q.sel[i];
  const unsigned long long own = i / kSortChunk;
  unsigned long long rank = i - own * kSortChunk;
  const unsigned long long n_chunks = (n + kSortChunk - 1) / kSortChunk;
  for (unsigned long long c = 0; c < n_chunks; ++c) {
    if (c == own) continue;
    const Entry* __restrict__ ch = Q.sel + c * kSortChunk;
    unsigned lo = 0, hi = (unsigned)min((unsigned long long)kSortChunk, n - c * kSortChunk);
    while (lo < hi) {
      const unsigned mid = (lo + hi) >> 1;
      if (entry_better(ch[mid], e)) lo = mid + 1; else hi = mid;
    }
    rank += lo;
  }
  Q.sorted[rank] = e;
}

// ---------------------------------------------------------------------------
// K7: materialize best-first rows: decode g (csl.py:166-184), objective in the
// scan's order (block_values, engine.py:210-222), constraint values in
// apex_score's order (engine.py:95-101: acc = 0.0; acc += v_r; + bias).
struct MatLaunch {
  const ScanQuery* queries;
  const DevReaction* rx;
  const unsigned long long* g_off;  // [n_rx + 1]
  int n_rx;
  const float* values;
  const float* p16;                 // pair-major copy or null
  int64_t n_pairs;
  const double* biases;
};

constexpr int kMatBatch = 6;  // tasks whose gathers a materialized row issues together
// goff / rxs: the reactions' g offsets and descriptors (M.g_off / M.rx, or
// shared-memory copies: the row's reaction search and decode then make no
// global round trip)
__device__ __forceinline__ void materialize_row(const MatLaunch& M, const ScanQuery& Q, unsigned long long i,
                                                unsigned long long g, const unsigned long long* goff = nullptr,
                                                const DevReaction* rxs = nullptr) {
  int lo = 0, hi = M.n_rx;
  if (goff) {
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (goff[mid] <= g) lo = mid; else hi = mid;
    }
  } else {
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(M.g_off + mid) <= g) lo = mid; else hi = mid;
    }
  }
  const DevReaction& R = rxs ? rxs[lo] : M.rx[lo];
  const int c = R.c;
  uint64_t rem = g - R.g_off;
  int64_t dig[kMaxRg], pr[kMaxRg];
#pragma unroll
  for (int j = kMaxRg - 1; j >= 0; --j) {
    dig[j] = 0;
    pr[j] = 0;
    if (j < c) {
      uint64_t q, d;
      divmod_u64(q, d, rem, (uint64_t)R.size[j]);
      dig[j] = (int64_t)d;
      pr[j] = R.pair_off[j] + (int64_t)d;
      rem = q;
    }
  }
  // tasks in batches of kMatBatch (t = 0: the objective in the scan's
  // v0 + v1 + ... order, t >= 1: constraint t - 1 in apex_score's
  // acc = 0.0; acc += v_r order, which differs only in the sign of an all-zero
  // sum): every gather of a batch is issued before any sum or store, so a row
  // costs one round trip per batch rather than one per task
  const int n_cons = Q.n_cons;
  for (int t0 = 0; t0 <= n_cons; t0 += kMatBatch) {
    float x[kMatBatch][kMaxRg];
    double bias[kMatBatch];
#pragma unroll
    for (int u = 0; u < kMatBatch; ++u) {
      const int t = t0 + u;
      const int ci = min(max(t - 1, 0), max(n_cons - 1, 0));
      const int task = t == 0 ? Q.obj_task : Q.cons_task[ci];
#pragma unroll
      for (int j = 0; j < kMaxRg; ++j)
        x[u][j] = (t <= n_cons && j < c) ? tval(M.values, M.p16, M.n_pairs, task, pr[j]) : 0.0f;
      bias[u] = t <= n_cons ? __ldg(M.biases + task) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kMatBatch; ++u) {
      const int t = t0 + u;
      if (t > n_cons) break;
      const double v0 = (double)x[u][0];
      double acc = t > 0 ? __dadd_rn(0.0, v0) : v0;
#pragma unroll
      for (int j = 1; j < kMaxRg; ++j)
        if (j < c) acc = __dadd_rn(acc, (double)x[u][j]);
      acc = __dadd_rn(acc, bias[u]);
      if (t == 0) Q.out_obj[i] = acc;
      else Q.out_cons[i * n_cons + t - 1] = acc;
    }
  }
  Q.out_g[i] = g;
  Q.out_rx[i] = lo;
#pragma unroll
  for (int j = 0; j < kMaxRg; ++j) Q.out_dig[i * kMaxRg + j] = (int32_t)dig[j];
}

__global__ void materialize_kernel(const MatLaunch M) {
  // every query (small-set or radix path): rows of sorted[0, sel_count), one
  // thread per row, the whole grid in parallel (a row is a chain of dependent
  // gathers, so rows spread over many SMs rather than one CTA per query)
  const ScanQuery& Q = M.queries[blockIdx.y];
  if (!*(volatile unsigned int*)&Q.ctl->active || *(volatile unsigned int*)&Q.ctl->mat_done) return;
  const unsigned long long n = *(volatile unsigned long long*)&Q.ctl->sel_count;
  const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  materialize_row(M, Q, i, Q.sorted[i].g);
}

// Final bound of a query (one warp, converged): the k-th best candidate
// bin's lower edge and the count at/above it (tie mode: the tied key and every
// admitted product), written to the control block (write = true) together
// with the parameters of the exact re-run if the candidate buffer overflowed.
// Returns the k-th best bin (-1: fewer than k candidates).
__device__ int final_bound(const ScanQuery& Q, bool write, unsigned long long& s_bound, unsigned long long& s_valid) {
  QCtl* ctl = Q.ctl;
  unsigned long long cnt_ge = 0;
  const int B = kth_two_level(Q.hist, Q.coarse, (unsigned long long)Q.k, &cnt_ge);
  if (lane_id() == 0) {
    const bool tie = ctl->tie_on != 0;
    const unsigned long long base = ctl->hist_base;
    const unsigned shift = ctl->hist_shift;
    unsigned long long bound = B >= 0 ? bin_edge((unsigned)B, base, shift) : 0ull;
    if (tie) {  // every admitted product has key >= K; the select orders them exactly
      bound = ctl->tie_key;
      cnt_ge = ctl->count;
    }
    s_bound = bound;
    s_valid = cnt_ge;
    if (write) {
      ctl->bound_key = bound;
      ctl->comp_count = cnt_ge;
    }
    // overflow (count > cap): parameters of the exact re-run (capi.cu
    // check_batch).  Every step either narrows the key bins holding the
    // k-th best by 16 bits, or — once that bin is one exact key K — bins
    // the tied products by g and narrows the admitted g range by 16 bits,
    // so the admitted set shrinks to at most k + one bin.
    if (write && ctl->count > Q.cap && B >= 0) {
      if (!tie) {
        if (B == 65535) {  // the absorbing top bin: re-spread [edge, 2^64) over the bins
          unsigned s2 = shift;
          while (s2 < 63 && ((~0ull - bound) >> s2) >= 65535ull) ++s2;
          ctl->nx_tau = bound;
          ctl->nx_base = bound;
          ctl->nx_shift = s2;
        } else if (shift == 0) {  // bin B is the single key K = bound
          ctl->nx_tau = bound;
          ctl->nx_tie = 1;
          ctl->nx_tie_enter = 1;
        } else {
          ctl->nx_tau = bound;
          ctl->nx_base = bound;
          ctl->nx_shift = shift >= 16 ? shift - 16 : 0u;
        }
      } else {
        const unsigned gs = ctl->tie_gshift;
        const unsigned long long glo = ctl->tie_gbase + ((unsigned long long)(65534 - min(B, 65534)) << gs);
        const unsigned long long ghi = glo + (1ull << gs);
        ctl->nx_tau = ctl->tie_key;
        ctl->nx_tie = 1;
        ctl->nx_gbase = glo;
        ctl->nx_glimit = (ghi > glo && ghi < ctl->tie_glimit) ? ghi : ctl->tie_glimit;
        ctl->nx_gshift = gs >= 16 ? gs - 16 : 0u;
      }
    }
  }
  return B;
}

// Small-candidate-set finalize (one 1024-thread CTA per query): when at most
// kSmallSel candidates are at/above the final bound, load them into shared
// memory, bitonic-sort by (key desc, g asc), keep the first k, and (single-GPU
// path) materialize them — replacing select + sort + materialize.
constexpr int kSmallSel = 8192;

__global__ void __launch_bounds__(1024) finalize_small_kernel(const MatLaunch M, int materialize, int compute_bound) {
  const ScanQuery& Q = M.queries[blockIdx.x];
  QCtl* ctl = Q.ctl;
  if (!*(volatile unsigned int*)&ctl->active) return;
  // final bound first (tau_kernel mode 2, folded in: warp 0): the k-th best
  // candidate bin's lower edge and the count at/above it, for this kernel and
  // for the large path that follows
  __shared__ unsigned long long s_bound, s_valid;
  if (!compute_bound) {  // bound and count preset (multi-GPU merge: every entry is a candidate)
    if (threadIdx.x == 0) {
      s_bound = *(volatile unsigned long long*)&ctl->bound_key;
      s_valid = *(volatile unsigned long long*)&ctl->comp_count;
    }
  } else if (threadIdx.x < 32) {
    final_bound(Q, true, s_bound, s_valid);
  }
  __syncthreads();
  const unsigned long long n_valid = s_valid;
  if (n_valid > (unsigned long long)kSmallSel) return;  // large path
  extern __shared__ __align__(16) unsigned char sm_e[];
  Entry* es = reinterpret_cast<Entry*>(sm_e);
  __shared__ unsigned cnt;
  const unsigned tid = threadIdx.x;
  if (tid == 0) cnt = 0;
  __syncthreads();
  const unsigned long long n = min(*(volatile unsigned long long*)&ctl->count, Q.cap);
  const unsigned long long bound = s_bound;
  const unsigned lane = tid & 31u;
  for (unsigned long long base = tid & ~31u; base < n; base += blockDim.x) {
    const unsigned long long i = base + lane;
    Entry e;
    const bool keep = i < n && (e = Q.buf[i], e.key >= bound);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (!m) continue;
    unsigned pos = 0;
    if (lane == 0) pos = atomicAdd(&cnt, (unsigned)__popc(m));  // one shared atomic per warp round
    pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
    if (keep && pos < (unsigned)kSmallSel) es[pos] = e;
  }
  __syncthreads();
  const unsigned m = min(cnt, (unsigned)kSmallSel);
  unsigned P = 1;
  while (P < m) P <<= 1;
  for (unsigned i = m + tid; i < P; i += blockDim.x) {
    es[i].key = 0;
    es[i].g = ~0ull;
  }
  __syncthreads();
  bitonic_best_first(es, P);
  const unsigned kk = (unsigned long long)Q.k < (unsigned long long)m ? (unsigned)Q.k : m;
  for (unsigned i = tid; i < kk; i += blockDim.x) {
    Q.sel[i] = es[i];
    Q.sorted[i] = es[i];
    if (materialize) materialize_row(M, Q, i, es[i].g);
  }
  if (tid == 0) {
    ctl->sel_count = kk;
    ctl->small_done = 1;
    if (kk == (unsigned long long)Q.k && kk > 0 && es[kk - 1].key > ctl->tau_key) ctl->tau_key = es[kk - 1].key;
  }
}

// Bucketed small finalize (grid: ns CTAs per query).  The candidate
// histogram orders the bins like the entries (a better entry never has a lower
// bin, in tie mode too), so the top-kk ranks split into ns contiguous runs of
// bins: CTA j owns the bins (b_{j+1}, b_j], b_j = the bin of rank j*kk/ns
// (b_0 = the top bin, b_ns = below the k-th best bin B), and its entries take
// the ranks from count(bins > b_j) on.  Each CTA sorts only its own bins'
// entries (bitonic, shared memory) and writes and materializes their rows:
// the one-CTA-per-query sort + separate materialization become one short
// kernel over ns x nq CTAs.  Same outputs as finalize_small_kernel (sel,
// sorted best-first, sel_count, small_done, final tau); CTA 0 writes the bound
// and the overflow re-run parameters.  Every per-thread chain is kept to few
// global round trips (~300-500 cycles each on sm_100, tools/microbench/
// latency.cu): the bound and both rank splits are searched by three warps at
// once, the control fields, g offsets and reaction descriptors are staged by
// the other warps meanwhile, the buffer is read kFinBatch entries per thread
// per round trip, and a materialized row decodes from shared memory.
constexpr int kFinThreads = 512;
constexpr int kFinWarps = kFinThreads / 32;
constexpr int kFinMaxSplit = 64;     // CTAs per query (rank splits)
constexpr int kFinRowsPerCta = 128;  // target ranks per CTA
constexpr int kFinSuffixMin = 16;    // splits from which the suffix-sum search and the partitioned load pay off
#ifndef APEX_FIN_BATCH
#define APEX_FIN_BATCH 8
#endif
constexpr int kFinBatch = APEX_FIN_BATCH;  // buffer entries per thread in flight
constexpr int kFinRx = 256;      // reactions whose descriptors + g offsets are staged in shared memory
__host__ __device__ constexpr size_t fin_bucket_smem() {
  return (size_t)kSmallSel * sizeof(Entry) + (size_t)kFinRx * sizeof(DevReaction) +
         (size_t)(kFinRx + 1) * sizeof(unsigned long long);
}

#ifdef APEX_FIN_DEBUG
#define FIN_T(i) if (threadIdx.x == 0) t_[i] = clock64();
#else
#define FIN_T(i)
#endif
__global__ void __launch_bounds__(kFinThreads) finalize_bucket_kernel(const MatLaunch M, int materialize,
                                                                      Entry* __restrict__ scratch) {
#ifdef APEX_FIN_DEBUG
  unsigned long long t_[8] = {};
#endif
  FIN_T(0)
  const ScanQuery& Q = M.queries[blockIdx.y];
  QCtl* ctl = Q.ctl;
  if (!*(volatile unsigned int*)&ctl->active) return;
  const unsigned ns = gridDim.x, j = blockIdx.x;
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  extern __shared__ __align__(16) unsigned char sm_e[];
  Entry* es = reinterpret_cast<Entry*>(sm_e);
  unsigned* fsuf = reinterpret_cast<unsigned*>(sm_e);  // prologue: per distinct coarse bin, 257 suffix counts
  DevReaction* s_rx = reinterpret_cast<DevReaction*>(sm_e + (size_t)kSmallSel * sizeof(Entry));
  unsigned long long* s_goff = reinterpret_cast<unsigned long long*>(s_rx + kFinRx);
  __shared__ unsigned long long s_bound, s_valid, s_above[kFinMaxSplit], s_n, s_hbase;
  __shared__ int s_bin[kFinMaxSplit], s_B;
  __shared__ unsigned s_hshift, s_tie, cnt;
  __shared__ unsigned s_cis[257];           // inclusive suffix sums of the coarse histogram (+ 0)
  __shared__ short s_cw[kFinMaxSplit], s_cidx[256];
  __shared__ unsigned char s_cflag[256];
  __shared__ short s_clist[kFinMaxSplit];
  __shared__ unsigned s_nd;
  const bool stage_rx = materialize && M.n_rx <= kFinRx;
  // (A) final bound (warp 0; CTA 0 writes it and the re-run parameters), the
  // coarse histogram (warps 1-8), control fields and staging (last warp)
  const bool suffix = ns >= kFinSuffixMin;  // many splits: suffix-sum searches; few: one warp search each
  if (warp == 0) {
    const int B = final_bound(Q, j == 0, s_bound, s_valid);
    if (lane == 0) s_B = B;  // bins below B hold no rank < kk
  } else if (suffix && warp <= 8) {
    const unsigned t = threadIdx.x - 32;
    s_cis[t] = __ldcg(Q.coarse + t);
    s_cflag[t] = 0;
  } else if (!suffix && warp < kFinWarps - 1) {
    if (warp < ns) {
      unsigned v[8];
      load_bins256(Q.coarse, v);
      unsigned long long tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) tot += v[i];
      tot = __reduce_add_sync(0xffffffffu, (unsigned)tot);
      const unsigned long long kk = min((unsigned long long)Q.k, tot);  // kk = min(k, total)
      for (unsigned w = warp; w < ns; w += kFinWarps - 2) {
        const unsigned long long target = (unsigned long long)w * kk / ns + 1;
        unsigned long long above = 0;
        const int b = kk ? kth_two_level_above(Q.hist, v, target, &above) : -1;
        if (lane == 0) {
          s_bin[w] = b;
          s_above[w] = above;
        }
      }
    }
  } else if (warp == kFinWarps - 1) {
    if (lane == 0) {
      s_n = min(*(volatile unsigned long long*)&ctl->count, Q.cap);
      s_hbase = *(volatile unsigned long long*)&ctl->hist_base;
      s_hshift = *(volatile unsigned*)&ctl->hist_shift;
      s_tie = *(volatile unsigned*)&ctl->tie_on;
      cnt = 0;
      s_bin[0] = 65535;
      s_above[0] = 0;
      s_nd = 0;
      s_cis[256] = 0;
    }
    if (stage_rx) {
      const int words = (int)(M.n_rx * (sizeof(DevReaction) / 8));
      const unsigned long long* src = reinterpret_cast<const unsigned long long*>(M.rx);
      unsigned long long* dst = reinterpret_cast<unsigned long long*>(s_rx);
      for (int i = (int)lane; i < words; i += 32) dst[i] = __ldg(src + i);
      for (int i = (int)lane; i <= M.n_rx; i += 32) s_goff[i] = __ldg(M.g_off + i);
    }
  }
  __syncthreads();
  if (suffix) {
    // (B) rank splits (every CTA derives all ns, so all agree on the path):
    // split w is the bin holding rank w*kk/ns, searched in suffix sums of the
    // coarse level, then of the fine blocks of the distinct coarse bins hit
    if (warp == 1) {  // coarse inclusive suffix sums, lane l: bins 8l .. 8l+7
      unsigned v[8], sum = 0;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        v[i] = s_cis[8 * lane + i];
        sum += v[i];
      }
      unsigned suf = sum;  // inclusive suffix over lanes >= this lane
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_down_sync(0xffffffffu, suf, o);
        if ((int)lane + o < 32) suf += y;
      }
      unsigned run = suf - sum;  // bins above this lane's block
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        run += v[i];
        s_cis[8 * lane + i] = run;
      }
    }
    __syncthreads();
    const unsigned long long tot = s_cis[0];
    const unsigned long long kk_all = min((unsigned long long)Q.k, tot);
    if (threadIdx.x >= 1 && threadIdx.x < ns) {
      const unsigned long long r = (unsigned long long)threadIdx.x * kk_all / ns;  // 0-based rank
      int lo = 0, hi = 255;  // largest c with s_cis[c] > r
      if (kk_all == 0 || s_cis[0] <= r) {
        s_cw[threadIdx.x] = -1;
      } else {
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_cis[mid] > r) lo = mid; else hi = mid - 1;
        }
        s_cw[threadIdx.x] = (short)lo;
        s_cflag[lo] = 1;
      }
    }
    __syncthreads();
    if (warp == 0) {  // distinct coarse bins hit -> list
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int cbin = 32 * i + (int)lane;
        const bool f = s_cflag[cbin] != 0;
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) {
          const unsigned d = s_nd + __popc(m & ((1u << lane) - 1u));
          s_clist[d] = (short)cbin;
          s_cidx[cbin] = (short)d;
        }
        __syncwarp();
        if (lane == 0) s_nd += __popc(m);
        __syncwarp();
      }
    }
    __syncthreads();
    for (unsigned d = warp; d < s_nd; d += kFinWarps) {  // fine block of each: inclusive suffix sums
      const int cbin = s_clist[d];
      unsigned* fs = fsuf + d * 257;
      unsigned v[8], sum = 0;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        v[i] = __ldcg(Q.hist + cbin * 256 + 8 * lane + i);
        sum += v[i];
      }
      unsigned suf = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_down_sync(0xffffffffu, suf, o);
        if ((int)lane + o < 32) suf += y;
      }
      unsigned run = suf - sum;
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        run += v[i];
        fs[8 * lane + i] = run;
      }
      if (lane == 0) fs[256] = 0;
    }
    __syncthreads();
    if (threadIdx.x >= 1 && threadIdx.x < ns) {
      const int cbin = s_cw[threadIdx.x];
      if (cbin < 0) {
        s_bin[threadIdx.x] = -1;
        s_above[threadIdx.x] = 0;
      } else {
        const unsigned long long r = (unsigned long long)threadIdx.x * kk_all / ns - s_cis[cbin + 1];
        const unsigned* fs = fsuf + s_cidx[cbin] * 257;
        int lo = 0, hi = 255;  // largest f with fs[f] > r (the fine counts agree with the coarse on a complete histogram)
        if (fs[0] <= r) {
          lo = 0;
        } else {
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (fs[mid] > r) lo = mid; else hi = mid - 1;
          }
        }
        s_bin[threadIdx.x] = cbin * 256 + lo;
        s_above[threadIdx.x] = (unsigned long long)s_cis[cbin + 1] + fs[lo + 1];
      }
    }

  }
  __syncthreads();
  const unsigned long long n_valid = s_valid;
  FIN_T(1)
  // the bucketed path takes every set whose CTAs each hold at most kSmallSel
  // entries (k above kSmallSel included, e.g. C4's k = 10,000); otherwise the
  // large path (select / sort / rank / materialize) follows
  if (n_valid > (unsigned long long)kSmallSel) {
    bool ok = s_tie == 0 && s_B >= 0;
    for (unsigned w = 1; w < ns && ok; ++w) ok = s_bin[w] >= 0;
    for (unsigned w = 0; w < ns && ok; ++w) {
      const unsigned long long hi_ab = s_above[w];
      const unsigned long long lo_ab = w + 1 < ns ? s_above[w + 1] : n_valid;
      ok = lo_ab >= hi_ab && lo_ab - hi_ab <= (unsigned long long)kSmallSel;
    }
    if (!ok) return;
  }
  // this CTA's bins: (lo_excl, hi]
  const int hi = s_bin[j];
  const int lo_excl = j + 1 < ns ? s_bin[j + 1] : (s_B >= 0 ? s_B - 1 : -1);
  const unsigned long long off = s_above[j];
  const unsigned long long kk = min((unsigned long long)Q.k, n_valid);
  if (j == 0 && threadIdx.x == 0) {
    ctl->sel_count = kk;
    ctl->small_done = 1;
    ctl->mat_done = materialize ? 1u : 0u;
  }
  const unsigned long long n = s_n, hbase = s_hbase;
  const unsigned hshift = s_hshift;
  const bool tie = s_tie != 0;
  const int b_low = s_B >= 0 ? s_B : 0;  // bins below hold no rank < kk
  if (scratch) {
    // (C) partition (cooperative launch: the query's CTAs are co-resident):
    // CTA j routes the entries of its 1/ns slice of the buffer to the CTA
    // owning their bin (a region of kSmallSel entries each in scratch), so
    // every entry is read once; then the query's CTAs meet at a barrier
    Entry* reg = scratch + (size_t)(blockIdx.y * ns) * kSmallSel;
    unsigned* rcnt = &ctl->hist[0][0];  // per destination CTA (zeroed by init_ctl; the select never ran)
    const unsigned long long s0 = n * j / ns, s1 = n * (j + 1) / ns;
    for (unsigned long long i = s0 + threadIdx.x; i < s1; i += blockDim.x) {
      const Entry e = Q.buf[i];
      const int b = (int)(tie ? cand_bin(ctl, e.key, e.g, hbase, hshift) : hist_bin(e.key, hbase, hshift));
      if (b < b_low) continue;
      int lo = 0, hi2 = (int)ns - 1;  // owner: largest w with s_bin[w] >= b
      while (lo < hi2) {
        const int mid = (lo + hi2 + 1) >> 1;
        if (s_bin[mid] >= b) lo = mid; else hi2 = mid - 1;
      }
      const unsigned pos = atomicAdd(rcnt + lo, 1u);
      if (pos < (unsigned)kSmallSel) reg[(size_t)lo * kSmallSel + pos] = e;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(&ctl->fin_bar, 1u);
      while (ld_acquire_u32(&ctl->fin_bar) < ns) __nanosleep(64);
    }
    __syncthreads();
    if (hi < 0 || hi <= lo_excl || off >= kk) return;
    const unsigned m0 = min(ld_relaxed_u32(rcnt + j), (unsigned)kSmallSel);
    const Entry* mine = reg + (size_t)j * kSmallSel;
    for (unsigned i = threadIdx.x; i < m0; i += blockDim.x) {  // written by other CTAs: past L1
      const ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2*>(mine + i));
      es[i].key = v.x;
      es[i].g = v.y;
    }
    if (threadIdx.x == 0) cnt = m0;
  } else {
    if (hi < 0 || hi <= lo_excl || off >= kk) return;
    for (unsigned long long base = threadIdx.x & ~31u; base < n; base += (unsigned long long)kFinBatch * blockDim.x) {
      Entry e[kFinBatch];
#pragma unroll
      for (int u = 0; u < kFinBatch; ++u) {
        const unsigned long long i = base + (unsigned long long)u * blockDim.x + lane;
        if (i < n) e[u] = Q.buf[i];
      }
#pragma unroll
      for (int u = 0; u < kFinBatch; ++u) {
        const unsigned long long i = base + (unsigned long long)u * blockDim.x + lane;
        bool keep = false;
        if (i < n) {
          const int b = (int)(tie ? cand_bin(ctl, e[u].key, e[u].g, hbase, hshift) : hist_bin(e[u].key, hbase, hshift));
          keep = b <= hi && b > lo_excl;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (!m) continue;
        unsigned pos = 0;
        if (lane == 0) pos = atomicAdd(&cnt, (unsigned)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < (unsigned)kSmallSel) es[pos] = e[u];
      }
    }
  }
  __syncthreads();
  FIN_T(2)
  const unsigned m = min(cnt, (unsigned)kSmallSel);
  unsigned P = 32;  // at least one warp's worth: sorted by warp shuffles
  while (P < m) P <<= 1;
  for (unsigned i = m + threadIdx.x; i < P; i += blockDim.x) {
    es[i].key = 0;
    es[i].g = ~0ull;
  }
  __syncthreads();
  bitonic_best_first(es, P);
  FIN_T(3)
  const unsigned n_out = (unsigned)min((unsigned long long)m, kk - off);
  for (unsigned i = threadIdx.x; i < n_out; i += blockDim.x) {
    const unsigned long long r = off + i;
    const Entry e = es[i];
    Q.sel[r] = e;
    Q.sorted[r] = e;
    if (materialize) materialize_row(M, Q, r, e.g, stage_rx ? s_goff : nullptr, stage_rx ? s_rx : nullptr);
    if (r == kk - 1 && kk == (unsigned long long)Q.k && e.key > ctl->tau_key) ctl->tau_key = e.key;
  }
#ifdef APEX_FIN_DEBUG
  __syncthreads();
  FIN_T(4)
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x + 1 == gridDim.x || m > 1024))
    printf("FIN q %u cta %u/%u n %llu m %u P %u off %llu cycles: prologue %llu load %llu sort %llu mat %llu\n", blockIdx.y,
           blockIdx.x, gridDim.x, n, m, P, off, t_[1] - t_[0], t_[2] - t_[1], t_[3] - t_[2], t_[4] - t_[3]);
#endif
}

// Control-block headers of every query (the fields before the select
// histograms) gathered into one contiguous block for a single D2H.
__global__ void ctl_export_kernel(const ScanQuery* __restrict__ qs, unsigned char* __restrict__ dst) {
  const QCtl* ctl = qs[blockIdx.x].ctl;
  const unsigned* src = reinterpret_cast<const unsigned*>(ctl);
  unsigned* d = reinterpret_cast<unsigned*>(dst + (size_t)blockIdx.x * ((offsetof(QCtl, hist) + 15) / 16 * 16));
  for (unsigned i = threadIdx.x; i < offsetof(QCtl, hist) / 4; i += blockDim.x) d[i] = __ldcg(src + i);
}

// Multi-GPU: export the local selected set (unordered) to out + slot*stride;
// the slots past the selected count are written as padding (g == ~0), so the
// exported block is complete without a separate memset.
__global__ void export_kernel(const ScanQuery* __restrict__ qs, Entry* __restrict__ out, unsigned long long stride) {
  const ScanQuery& Q = qs[blockIdx.y];
  const unsigned long long n = *(volatile unsigned long long*)&Q.ctl->sel_count;
  // overflowed or given up by the sorted-column kernel: a re-run is pending
  const bool stale = *(volatile unsigned long long*)&Q.ctl->count > Q.cap || *(volatile unsigned*)&Q.ctl->bail;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < stride;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    Entry e;
    if (i < n) {
      e = Q.sel[i];
    } else {
      e.key = ~0ull;
      e.g = ~0ull;
    }
    if (stale && i == 0) e.g = kStaleG;
    out[(unsigned long long)Q.slot * stride + i] = e;
  }
}

// Multi-GPU: load gathered entries (skip padding g == ~0) as the compacted set.
// Multi-GPU: load the gathered entries of query blockIdx.y (skipping padding
// g == ~0) as its candidate set.  Layout: in[(src * nq + q) * stride + i],
// i < stride, for src < n_src (what an all-gather of per-rank [nq][stride]
// buffers produces).
// srcs (optional): one pointer per source rank to its [nq][stride] block —
// on a multi-GPU context these are PEER device pointers, so this kernel is the
// all-gather itself: every entry is loaded over NVLink straight into the
// merge's candidate buffer (no staging copy, no separate collective).
__global__ void merge_load_kernel(const ScanQuery* __restrict__ qs, const Entry* __restrict__ in, int n_src,
                                  int nq, unsigned long long stride, const Entry* const* __restrict__ srcs = nullptr) {
  const int q = blockIdx.y;
  const ScanQuery& Q = qs[q];
  QCtl* ctl = Q.ctl;
  const unsigned lane = lane_id();
  const unsigned long long n = (unsigned long long)n_src * stride;
  const unsigned long long gstride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long base = (unsigned long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += gstride) {
    const unsigned long long i = base + lane;
    Entry e;
    bool keep = false;
    if (i < n) {
      const unsigned long long src = i / stride, j = i - src * stride;
      e = srcs ? srcs[src][(unsigned long long)q * stride + j]
               : in[(src * (unsigned long long)nq + (unsigned long long)q) * stride + j];
      keep = e.g < kStaleG;
      if (e.g == kStaleG) atomicOr(&ctl->stale, 1u);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (m) {
      const int leader = __ffs(m) - 1;
      unsigned long long pos = 0;
      if ((int)lane == leader) {
        pos = atomicAdd(&ctl->count, (unsigned long long)__popc(m));
        atomicAdd(&ctl->comp_count, (unsigned long long)__popc(m));
      }
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (keep) Q.buf[pos + __popc(m & ((1u << lane) - 1u))] = e;
    }
  }
}

}  // namespace apexb200

// multi_scan.cuh — K3, batched full-predicate form for query batches that
// share constraint sets (BASELINE configs[1]: 5 objectives x 4 property
// presets = 20 queries, 13 distinct bounds).
//
// Work item = one tile (<= 32 rows x <= 64 columns of one reaction) for ALL
// queries of the launch (<= 16), instead of one (tile, query) item per query:
//   * per row (lane): the exact fp32 threshold of every DISTINCT constraint
//     test of the launch (a (task, bound, side) shared by several queries is
//     derived once) and every query's admission threshold against its tau;
//   * per column block: the signed column values of those tests and of every
//     query's objective staged once in shared memory (from the pair-major
//     table copy), read back as broadcast LDS.128;
//   * per product: one fp32 compare per distinct test -> a test bitmask; the
//     group feasibility of every distinct constraint set from the mask; one
//     compare per query against its admission threshold; candidates (feasible
//     and s >= tau, both exact, as in every K3 form) appended per query with
//     the same warp-aggregated protocol, histogram and tau refresh.
// Per product the work is |distinct tests| + |queries| compares, not
// sum_q (bounds_q + 1): C2 33 instead of 90.
#pragma once
#include "common.cuh"

namespace apexb200 {

constexpr int kMU = 16;    // distinct constraint tests per launch
constexpr int kMQ = 16;    // queries per launch
constexpr int kMG = 8;     // distinct constraint sets per launch
constexpr int kMCB = 64;   // columns per tile (shared-memory block)
constexpr int kMW = 32;    // staged values per column: tests [0, 16), query objectives [16, 32)

struct MultiLaunch {
  const Tile* tiles;
  unsigned n_tiles;
  unsigned* work;
  const DevReaction* rx;
  const float* p16;          // [n_pairs][16] pair-major table copy
  int64_t n_pairs;
  const ScanQuery* queries;  // batch descriptors (device)
  int nu, nq, ng;
  int u_task[kMU];
  int u_lower[kMU];          // 1: lower bound (compare -x <= -L)
  double u_beta[kMU];
  double u_bias[kMU];
  unsigned g_need[kMG];      // distinct constraint set g: mask over the tests
  unsigned g_queries[kMG];   // the queries (bits) with constraint set g
  int q_idx[kMQ];            // query i of the launch = queries[q_idx[i]]
};

__global__ void __launch_bounds__(kScanWarps * 32, 3) scan_multi_kernel(const MultiLaunch M) {
  extern __shared__ __align__(16) float msm[];
  const unsigned warp = threadIdx.x >> 5, lane = lane_id();
  float* ys = msm + (size_t)warp * kMCB * kMW;  // this warp's staged column block
  const unsigned qmask_all = M.nq >= 32 ? ~0u : ((1u << M.nq) - 1u);
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(M.work, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= M.n_tiles) return;
    const Tile T = M.tiles[t];
    const DevReaction& R = M.rx[T.rx];
    const int c = R.c;
    const int64_t last_pair = R.pair_off[c - 1];
    const int ncols = (int)T.ncols;
    // 1. stage the signed test / objective values of the tile's columns
    __syncwarp();
    for (int idx = lane; idx < ncols * kMW; idx += 32) {
      const int j = idx / kMW, w = idx % kMW;
      float y = __int_as_float(0x7fc00000);  // NaN: an unused slot never passes
      if (w < kMU) {
        if (w < M.nu) {
          const float x = __ldg(M.p16 + (last_pair + T.col0 + j) * 16 + M.u_task[w]);
          y = M.u_lower[w] ? -x : x;
        }
      } else if (w - kMU < M.nq) {
        const ScanQuery& Q = M.queries[M.q_idx[w - kMU]];
        const float x = __ldg(M.p16 + (last_pair + T.col0 + j) * 16 + Q.obj_task);
        y = Q.maximize ? -x : x;  // signed: s >= tau <=> y <= threshold
      }
      ys[j * kMW + w] = y;
    }
    // 2. per-row thresholds (lane = row)
    const bool valid = lane < T.nrows;
    const uint64_t row = T.row0 + (valid ? lane : 0u);
    int64_t pr[kMaxRg - 1];
    decode_prefix(R, c, row, pr);
    auto prefix = [&](int task) -> double {
      double p = c > 1 ? (double)__ldg(M.p16 + pr[0] * 16 + task) : 0.0;
#pragma unroll
      for (int j = 1; j < kMaxRg - 1; ++j)
        if (j < c - 1) p = __dadd_rn(p, (double)__ldg(M.p16 + pr[j] * 16 + task));
      return p;
    };
    const float kNaN = __int_as_float(0x7fc00000);
    float th[kMU];
#pragma unroll
    for (int u = 0; u < kMU; ++u) {
      th[u] = kNaN;
      if (u < M.nu && valid) {
        const double p = prefix(M.u_task[u]);
        th[u] = M.u_lower[u] ? -thr_lower_fast(p, M.u_bias[u], M.u_beta[u])
                             : thr_upper_fast(p, M.u_bias[u], M.u_beta[u]);
      }
    }
    float th0[kMQ];
#pragma unroll
    for (int q = 0; q < kMQ; ++q) {
      th0[q] = kNaN;
      if (q < M.nq && valid) {
        const ScanQuery& Q = M.queries[M.q_idx[q]];
        const unsigned long long tau = ld_relaxed_u64(&Q.ctl->tau_key);
        th0[q] = __int_as_float(0x7f800000);  // no threshold yet: every column passes the admission
        if (tau != kNoTau) {
          const double ts = key_to_score(tau);
          const double p = prefix(Q.obj_task);
          th0[q] = Q.maximize ? -thr_lower_fast(p, Q.test_bias[0], ts) : thr_upper_fast(p, Q.test_bias[0], -ts);
        }
      }
    }
    __syncwarp();
    const unsigned long long gbase = R.g_off + row * (uint64_t)R.size[c - 1] + T.col0;
    // 3. every product of the tile against every test and query
    for (int j = 0; j < ncols; ++j) {
      const float4* yp = reinterpret_cast<const float4*>(ys + j * kMW);
      float y[kMW];
#pragma unroll
      for (int v = 0; v < kMW / 4; ++v) {
        const float4 f = yp[v];
        y[4 * v] = f.x; y[4 * v + 1] = f.y; y[4 * v + 2] = f.z; y[4 * v + 3] = f.w;
      }
      unsigned tm = 0;
#pragma unroll
      for (int u = 0; u < kMU; ++u)
        if (y[u] <= th[u]) tm |= 1u << u;
      unsigned feas = 0;
#pragma unroll
      for (int g = 0; g < kMG; ++g)
        if (g < M.ng && (tm & M.g_need[g]) == M.g_need[g]) feas |= M.g_queries[g];
      unsigned adm = 0;
#pragma unroll
      for (int q = 0; q < kMQ; ++q)
        if (y[kMU + q] <= th0[q]) adm |= 1u << q;
      const unsigned cand = adm & feas & qmask_all;
      unsigned any = __reduce_or_sync(0xffffffffu, cand);
      // rare path: append the candidates of every query with one
      while (any) {
        const int q = __ffs(any) - 1;
        any &= any - 1;
        const ScanQuery& Q = M.queries[M.q_idx[q]];
        QCtl* ctl = Q.ctl;
        bool pass = (cand >> q) & 1u;
        Entry e;
        if (pass) {
          const float x = Q.maximize ? -y[kMU + q] : y[kMU + q];
          const double val = fx(prefix(Q.obj_task), x, Q.test_bias[0]);
          e.key = skey(Q.maximize ? val : -val);
          e.g = gbase + (unsigned long long)j;
          pass = !tie_reject(ctl, e.key, e.g);
        }
        const unsigned mk = __ballot_sync(0xffffffffu, pass);
        if (!mk) continue;
        unsigned long long cbase = 0;
        if (lane == 0) cbase = atomicAdd(&ctl->count, (unsigned long long)__popc(mk));
        cbase = __shfl_sync(0xffffffffu, cbase, 0);
        if (pass) {
          const unsigned long long idx = cbase + __popc(mk & ((1u << lane) - 1u));
          if (idx < Q.cap) Q.buf[idx] = e;
          const unsigned hb = cand_bin(ctl, e.key, e.g, __ldcg(&ctl->hist_base), __ldcg(&ctl->hist_shift));
          atomicAdd(&Q.hist[hb], 1u);
          atomicAdd(&Q.coarse[hb >> 8], 1u);
        }
        if ((cbase >> Q.refresh_shift) != ((cbase + __popc(mk)) >> Q.refresh_shift)) {
          __threadfence();
          refresh_tau(Q);
        }
      }
    }
  }
}

}  // namespace apexb200

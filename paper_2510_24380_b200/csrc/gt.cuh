// gt.cuh — GPU ground-truth evaluation: the exhaustive
// oracle top-j of the reference's evaluation kit on the device, past the
// reference's 1e8-product enumeration guard (evalkit.py:23, 60-64).
//
// Reference: evalkit.oracle_topk (evalkit.py:49-90) over
// props.oracle_block_values (props.py:218-264) — per product and task:
//   base  = ((lat[s0] + lat[s1]) + lat[s2]) ...      (R-group order, fp64)
//   value = base
//   value = value + nonlinear_scale * tanh(nonlinear_alpha * base)   (+nonlinear)
//   value = value + pair_coefficient(s_a, s_b) for a < b, lexicographic (+pairwise)
// with pair_coefficient / _pair_uniform / _splitmix (props.py:162-195) in
// exact uint64 arithmetic; feasible <=> every constraint lo <= v <= hi
// (violation == 0, engine.py:134-144); top-j by (s desc, g asc).
//
// Device protocol (capi.cu apex_gt_topk): histogram passes over the range
// narrow the key bin that holds the j-th best feasible key 16 bits at a
// time (then, for an exact-key tie storm, the g range of that key), until
// the products at or above the bound fit the candidate buffer; one collect
// pass appends them; the ordinary exact merge (select + order + decode)
// returns the best-first global indices.  Everything is exact except the
// tanh, whose CUDA and numpy implementations may differ in the last ulp.
#pragma once
#include "common.cuh"

namespace apexb200 {

constexpr int kGtMaxTasks = 1 + kMaxCons;

struct GtTask {
  const double* latent;   // per synthon id
  double nl_scale, nl_alpha, pair_scale, pair_density;
  unsigned long long salt;
  int32_t flags;          // 1 = +nonlinear, 2 = +pairwise
  int32_t _pad;
};

// One pass over [start, end): which tests and what to do with each feasible key.
struct GtPass {
  const DevReaction* rx;
  const Tile* tiles;
  unsigned n_tiles;
  const long long* members;   // [n_pairs] synthon id of each pair row
  const GtTask* tasks;        // device array
  int obj;                    // task index of the objective
  int maximize;
  int n_cons;
  int cons_task[kMaxCons];
  double cons_lo[kMaxCons], cons_hi[kMaxCons];
  // mode 0: histogram of keys >= base by (key - base) >> shift (65535 absorbs the rest)
  // mode 1: tie: keys > tie_key -> bin 65535; key == tie_key -> g bins (g >= gbase, g < glimit)
  // mode 2: collect entries admitted by the same bound into buf
  int mode;
  int tie;
  unsigned long long base, tie_key, gbase, glimit;
  unsigned shift, gshift;
  unsigned* hist;             // [65536] + coarse [256]
  Entry* buf;
  unsigned long long cap;
  unsigned long long* count;
  unsigned* work;
};

__device__ __forceinline__ unsigned long long gt_splitmix(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// props._pair_uniform: uniform in [0, 1) keyed by the unordered id pair
__device__ __forceinline__ double gt_pair_uniform(unsigned long long a, unsigned long long b, unsigned long long salt) {
  const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
  const unsigned long long h =
      gt_splitmix(gt_splitmix(lo * 0x9E3779B97F4A7C15ull + salt) ^ (hi * 0x94D049BB133111EBull));
  return __dmul_rn((double)(h >> 11), 1.0 / 9007199254740992.0);  // / 2^53 (exact scaling)
}

// props.pair_coefficient
__device__ __forceinline__ double gt_pair_coeff(const GtTask& T, unsigned long long a, unsigned long long b) {
  const double gate = gt_pair_uniform(a, b, T.salt);
  if (!(gate < T.pair_density)) return 0.0;
  const double v = gt_pair_uniform(a, b, T.salt + 0x51EDull);
  return __dmul_rn(T.pair_scale, __dsub_rn(__dmul_rn(2.0, v), 1.0));
}

// props.oracle_block_values for one product (synthon ids s[0..c-1])
__device__ __forceinline__ double gt_value(const GtTask& T, const long long (&s)[kMaxRg], int c) {
  double base = __ldg(T.latent + s[0]);
#pragma unroll
  for (int j = 1; j < kMaxRg; ++j)
    if (j < c) base = __dadd_rn(base, __ldg(T.latent + s[j]));
  double v = base;
  if (T.flags & 1) v = __dadd_rn(v, __dmul_rn(T.nl_scale, tanh(__dmul_rn(T.nl_alpha, base))));
  if (T.flags & 2) {
#pragma unroll
    for (int a = 0; a < kMaxRg; ++a)
#pragma unroll
      for (int b = a + 1; b < kMaxRg; ++b)
        if (b < c) v = __dadd_rn(v, gt_pair_coeff(T, (unsigned long long)s[a], (unsigned long long)s[b]));
  }
  return v;
}

__device__ __forceinline__ unsigned gt_bin(const GtPass& P, unsigned long long key, unsigned long long g, bool& use) {
  use = true;
  if (P.tie) {
    if (key > P.tie_key) return 65535u;
    if (key < P.tie_key || g >= P.glimit) { use = false; return 0u; }
    if (g < P.gbase) return 65535u;
    const unsigned long long rel = (g - P.gbase) >> P.gshift;
    return rel >= 65535ull ? 0u : (unsigned)(65534ull - rel);
  }
  if (key < P.base) { use = false; return 0u; }
  const unsigned long long rel = (key - P.base) >> P.shift;
  return rel > 65535ull ? 65535u : (unsigned)rel;
}

// One warp per tile (atomic work counter); lanes stride the tile's columns.
__global__ void __launch_bounds__(256) gt_pass_kernel(const GtPass P) {
  const unsigned lane = lane_id();
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(P.work, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= P.n_tiles) return;
    const Tile T = P.tiles[t];
    const DevReaction& R = P.rx[T.rx];
    const int c = R.c;
    const int64_t n_last = R.size[c - 1];
    for (unsigned rr = 0; rr < T.nrows; ++rr) {
      const uint64_t row = T.row0 + rr;
      long long sid[kMaxRg];
      {
        uint64_t rem = row;
#pragma unroll
        for (int j = kMaxRg - 2; j >= 0; --j) {
          sid[j] = 0;
          if (j < c - 1) {
            uint64_t q, d;
            divmod_u64(q, d, rem, (uint64_t)R.size[j]);
            sid[j] = __ldg(P.members + R.pair_off[j] + (int64_t)d);
            rem = q;
          }
        }
        sid[kMaxRg - 1] = 0;
      }
      const unsigned long long gbase = R.g_off + row * (uint64_t)n_last;
      for (unsigned cc0 = 0; cc0 < T.ncols; cc0 += 32) {
        const unsigned cc = cc0 + lane;
        bool ok = cc < T.ncols;
        unsigned long long key = 0, g = 0;
        if (ok) {
          const int64_t col = (int64_t)T.col0 + cc;
          long long s[kMaxRg];
#pragma unroll
          for (int j = 0; j < kMaxRg; ++j) s[j] = sid[j];
          // the last R-group's synthon id goes in slot c - 1
#pragma unroll
          for (int j = 0; j < kMaxRg; ++j)
            if (j == c - 1) s[j] = __ldg(P.members + R.pair_off[c - 1] + col);
          g = gbase + (unsigned long long)col;
          for (int m = 0; m < P.n_cons && ok; ++m) {
            const double v = gt_value(P.tasks[P.cons_task[m]], s, c);
            ok = v >= P.cons_lo[m] && v <= P.cons_hi[m];
          }
          if (ok) {
            const double v = gt_value(P.tasks[P.obj], s, c);
            key = skey(P.maximize ? v : -v);
          }
        }
        bool use = false;
        unsigned bin = 0;
        if (ok) bin = gt_bin(P, key, g, use);
        use = use && ok;
        if (P.mode == 2) {
          const unsigned m = __ballot_sync(0xffffffffu, use);
          if (m) {
            unsigned long long pos = 0;
            if (lane == 0) pos = atomicAdd(P.count, (unsigned long long)__popc(m));
            pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
            if (use && pos < P.cap) {
              Entry e;
              e.key = key;
              e.g = g;
              P.buf[pos] = e;
            }
          }
        } else {
          hist_add_warp(P.hist, bin, use);
          hist_add_warp(P.hist + 65536, bin >> 8, use);
        }
      }
    }
  }
}

// K-th best bin of the pass histogram (one warp): bin index and the count at
// or above it; -1 if fewer than k entries.
__global__ void gt_kth_kernel(const unsigned* __restrict__ hist, unsigned long long k, long long* out) {
  unsigned long long cnt = 0;
  const int B = kth_two_level(hist, hist + 65536, k, &cnt);
  if (lane_id() == 0) {
    out[0] = B;
    out[1] = (long long)cnt;
  }
}

// objective and constraint values of the selected products (best-first g)
__global__ void gt_values_kernel(const GtPass P, const unsigned long long* __restrict__ gs, int n,
                                 const unsigned long long* __restrict__ g_off, int n_rx, double* obj, double* cons) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long g = gs[i];
  int lo = 0, hi = n_rx;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (g_off[mid] <= g) lo = mid; else hi = mid;
  }
  const DevReaction& R = P.rx[lo];
  const int c = R.c;
  uint64_t rem = g - R.g_off;
  long long s[kMaxRg];
#pragma unroll
  for (int j = kMaxRg - 1; j >= 0; --j) {
    s[j] = 0;
    if (j < c) {
      uint64_t q, d;
      divmod_u64(q, d, rem, (uint64_t)R.size[j]);
      s[j] = __ldg(P.members + R.pair_off[j] + (int64_t)d);
      rem = q;
    }
  }
  obj[i] = gt_value(P.tasks[P.obj], s, c);
  for (int m = 0; m < P.n_cons; ++m) cons[(size_t)i * P.n_cons + m] = gt_value(P.tasks[P.cons_task[m]], s, c);
}

}  // namespace apexb200

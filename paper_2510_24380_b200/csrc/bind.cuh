// bind.cuh — first-call binding of a (library, table) pair on the device:
// every R-group column of every task sorted once (segmented sort), then the
// per-task sorted last-R-group columns (value, column) and their quantile
// tables used by the sorted-column enumeration kernel, and the best-first
// "corner" digit lists of the threshold seed (capi.cu build_corners).  The
// reference has no counterpart (its per-call check is the O(library)
// fingerprint, engine.py:70-72); this replaces a host sort of the table.
#pragma once
#include "common.cuh"

namespace apexb200 {

constexpr int kBindSmem = 4096;  // segment length sorted in shared memory

// (value, index) -> one 64-bit key, ascending in (value, index)
__device__ __forceinline__ unsigned long long bind_key(float v, unsigned idx) {
  const unsigned u = __float_as_uint(v);
  const unsigned o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | idx;
}
__device__ __forceinline__ float bind_value(unsigned long long k) {
  const unsigned o = (unsigned)(k >> 32);
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

struct BindSeg {
  int64_t pair;     // first pair row of the R-group
  int64_t scratch;  // padded scratch offset (segments longer than kBindSmem), -1 otherwise
  int32_t n;        // synthons in the R-group
  int32_t task;
};

// ascending bitonic sort of P (power of two) keys in `a` (shared or global
// memory) by the whole block
__device__ void bind_bitonic(unsigned long long* a, unsigned P) {
  for (unsigned size = 2; size <= P; size <<= 1)
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      for (unsigned q = threadIdx.x; q < (P >> 1); q += blockDim.x) {
        const unsigned i = ((q & ~(stride - 1)) << 1) | (q & (stride - 1)), j = i + stride;
        const unsigned long long x = a[i], y = a[j];
        const bool up = (i & size) == 0;
        if (up ? (y < x) : (x < y)) {
          a[i] = y;
          a[j] = x;
        }
      }
      __syncthreads();
    }
}

// one CTA per (task, R-group) segment: keys[task][pair .. pair + n) sorted
__global__ void __launch_bounds__(1024) bind_sort_kernel(const BindSeg* __restrict__ segs, const float* __restrict__ values,
                                                         int64_t n_pairs, unsigned long long* __restrict__ keys,
                                                         unsigned long long* __restrict__ scratch) {
  __shared__ unsigned long long sk[kBindSmem];
  const BindSeg S = segs[blockIdx.x];
  const float* v = values + (int64_t)S.task * n_pairs + S.pair;
  unsigned long long* out = keys + (int64_t)S.task * n_pairs + S.pair;
  unsigned P = 1;
  while (P < (unsigned)S.n) P <<= 1;
  unsigned long long* a = S.scratch >= 0 ? scratch + S.scratch : sk;
  for (unsigned i = threadIdx.x; i < P; i += blockDim.x) a[i] = i < (unsigned)S.n ? bind_key(__ldg(v + i), i) : ~0ull;
  __syncthreads();
  bind_bitonic(a, P);
  for (unsigned i = threadIdx.x; i < (unsigned)S.n; i += blockDim.x) out[i] = a[i];
}

struct BindEmit {
  const DevReaction* rx;
  int n_rx;
  int64_t n_pairs;
  const unsigned long long* keys;   // [task][pair] sorted per R-group
  float* sx;                        // [task][pcols]
  uint32_t* scol;
  int64_t pcols;
  float* quant;                     // [task][n_rx][kQuant + 1]
  int32_t* lists;                   // [task][2][slots]
  const int32_t* slot_off;          // [n_rx * kMaxRg]
  const int32_t* m;                 // [n_rx * kMaxRg]
  int64_t slots;
};

// grid (n_rx, n_tasks): the reaction's sorted last column, quantiles and corner lists
__global__ void bind_emit_kernel(const BindEmit E) {
  const int t = blockIdx.x, task = blockIdx.y;
  const DevReaction& R = E.rx[t];
  const unsigned long long* kt = E.keys + (int64_t)task * E.n_pairs;
  const int c = R.c;
  const int64_t n = R.size[c - 1];
  const unsigned long long* kl = kt + R.pair_off[c - 1];
  float* ox = E.sx + (int64_t)task * E.pcols + R.pcol_off;
  uint32_t* oc = E.scol + (int64_t)task * E.pcols + R.pcol_off;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const unsigned long long k = kl[i];
    ox[i] = bind_value(k);
    oc[i] = (uint32_t)k;
  }
  float* oq = E.quant + ((int64_t)task * E.n_rx + t) * (kQuant + 1);
  for (int qq = threadIdx.x; qq <= kQuant; qq += blockDim.x)
    oq[qq] = n > 0 ? bind_value(kl[min(n - 1, (int64_t)qq * n / kQuant)]) : 0.0f;
  for (int j = 0; j < c; ++j) {
    const unsigned long long* kj = kt + R.pair_off[j];
    const int64_t nj = R.size[j];
    const int mj = E.m[t * kMaxRg + j];
    int32_t* up = E.lists + ((int64_t)task * 2 + 0) * E.slots + E.slot_off[t * kMaxRg + j];  // largest first
    int32_t* dn = E.lists + ((int64_t)task * 2 + 1) * E.slots + E.slot_off[t * kMaxRg + j];  // smallest first
    for (int i = threadIdx.x; i < mj; i += blockDim.x) {
      dn[i] = (int32_t)(uint32_t)kj[i];
      up[i] = (int32_t)(uint32_t)kj[nj - 1 - i];
    }
  }
}

// pair-major copy of the table for the sorted-column kernel: packed16[p][t] =
// values[t][p] (t < n_tasks <= 16), 0 in the padding
__global__ void bind_pack16_kernel(const float* __restrict__ values, int64_t n_pairs, int n_tasks,
                                   float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pairs * 16;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i >> 4;
    const int t = (int)(i & 15);
    out[i] = t < n_tasks ? __ldg(values + (int64_t)t * n_pairs + p) : 0.0f;
  }
}

// Row-prefix table (sorted-column and pre-pass kernels): for every row of
// every reaction (a fixed assignment of its first c-1 R-groups) and every
// task, the fp64 prefix sum of those R-groups' contributions in the scan's
// order (v0 + v1 + ..., engine.py:210-222 without the last R-group and the
// bias): rowp[task][row_off + row].  grid.y = reaction, grid-stride rows.
__global__ void bind_rowp_kernel(const DevReaction* __restrict__ rxs, const float* __restrict__ values, int64_t n_pairs,
                                 int n_tasks, int64_t rows_total, double* __restrict__ rowp) {
  const DevReaction R = rxs[blockIdx.y];
  const int c = R.c;
  for (uint64_t row = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; row < R.n_rows;
       row += (uint64_t)gridDim.x * blockDim.x) {
    int64_t pr[kMaxRg - 1];
    decode_prefix(R, c, row, pr);
    for (int task = 0; task < n_tasks; ++task) {
      double p = c > 1 ? (double)__ldg(values + (int64_t)task * n_pairs + pr[0]) : 0.0;
#pragma unroll
      for (int j = 1; j < kMaxRg - 1; ++j)
        if (j < c - 1) p = __dadd_rn(p, (double)__ldg(values + (int64_t)task * n_pairs + pr[j]));
      rowp[task * rows_total + R.row_off + (int64_t)row] = p;
    }
  }
}

}  // namespace apexb200

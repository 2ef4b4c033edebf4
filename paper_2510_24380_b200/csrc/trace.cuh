// trace.cuh — BatchTrace accounting of the chain-of-batches variant on the
// device (reference engine.search_topk_batched,
// engine.py:345-398, BatchTrace :338-342, make_batches :316-335).
//
// The reference keeps, per batch, the k best of (carry ∪ batch) under the
// FULL order — violation c desc, signed objective s desc, global index asc,
// infeasible products included (lexsort((g, -s, -c)), engine.py:385-386) —
// and records how many of the selected came from the batch (new) and how many
// from the carry.  Here the carry lives on the device as composite entries
// (key(c), key(s), g, origin); a batch is evaluated in sub-ranges, products
// that cannot beat the carry's worst entry are skipped, the survivors plus the
// carry are sorted (bitonic, shared memory or global), and the first k become
// the carry.  Exact: c and s are the reference's fp64 values (block_values
// order, bias last; violation's hinge sum in constraint order).
#pragma once
#include "common.cuh"

namespace apexb200 {

struct __align__(16) TEntry {
  unsigned long long kc;  // skey(c): larger = less violation
  unsigned long long ks;  // skey(s)
  unsigned long long g;
  unsigned long long origin;  // 1 = from the current batch
};

__device__ __forceinline__ bool tbetter(const TEntry& a, const TEntry& b) {
  if (a.kc != b.kc) return a.kc > b.kc;
  if (a.ks != b.ks) return a.ks > b.ks;
  return a.g < b.g;
}

struct TraceEval {
  const DevReaction* rx;
  const Tile* tiles;
  unsigned n_tiles;
  unsigned* work;
  const float* values;
  int64_t n_pairs;
  const double* biases;
  int obj, maximize, n_cons;
  int cons_task[kMaxCons];
  double cons_lo[kMaxCons], cons_hi[kMaxCons];
  unsigned long long a, b;     // sub-range of g evaluated by this launch
  const TEntry* worst;         // carry's k-th entry (null: carry not full)
  TEntry* out;                 // appended candidates
  unsigned long long* count;
  unsigned long long cap;
};

// fp64 value of task t for a product (engine.py:210-222: R-group order, bias last)
__device__ __forceinline__ double tr_value(const TraceEval& E, int t, const int64_t (&pr)[kMaxRg], int c) {
  const float* v = E.values + (int64_t)t * E.n_pairs;
  double acc = (double)__ldg(v + pr[0]);
#pragma unroll
  for (int j = 1; j < kMaxRg; ++j)
    if (j < c) acc = __dadd_rn(acc, (double)__ldg(v + pr[j]));
  return __dadd_rn(acc, __ldg(E.biases + t));
}

__global__ void __launch_bounds__(256) trace_eval_kernel(const TraceEval E) {
  const unsigned lane = lane_id();
  TEntry w;
  const bool full = E.worst != nullptr;
  if (full) w = *E.worst;
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(E.work, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= E.n_tiles) return;
    const Tile T = E.tiles[t];
    const DevReaction& R = E.rx[T.rx];
    const int c = R.c;
    const uint64_t n_last = (uint64_t)R.size[c - 1];
    for (unsigned rr = 0; rr < T.nrows; ++rr) {
      const uint64_t row = T.row0 + rr;
      int64_t pr[kMaxRg];
      {
        uint64_t rem = row;
#pragma unroll
        for (int j = kMaxRg - 1; j >= 0; --j) {
          pr[j] = 0;
          if (j < c - 1) {
            uint64_t q, d;
            divmod_u64(q, d, rem, (uint64_t)R.size[j]);
            pr[j] = R.pair_off[j] + (int64_t)d;
            rem = q;
          }
        }
      }
      const unsigned long long gbase = R.g_off + row * n_last;
      for (unsigned cc0 = 0; cc0 < T.ncols; cc0 += 32) {
        const unsigned cc = cc0 + lane;
        const unsigned long long g = gbase + T.col0 + cc;
        bool keep = cc < T.ncols && g >= E.a && g < E.b;
        TEntry e;
        if (keep) {
          int64_t p[kMaxRg];
#pragma unroll
          for (int j = 0; j < kMaxRg; ++j) p[j] = (j == c - 1) ? R.pair_off[c - 1] + (int64_t)(T.col0 + cc) : pr[j];
          double viol = 0.0;  // violation(): c = c - max(0, lo - v); c = c - max(0, v - hi)
          for (int m = 0; m < E.n_cons; ++m) {
            const double v = tr_value(E, E.cons_task[m], p, c);
            viol = __dsub_rn(viol, fmax(0.0, __dsub_rn(E.cons_lo[m], v)));
            viol = __dsub_rn(viol, fmax(0.0, __dsub_rn(v, E.cons_hi[m])));
          }
          const double o = tr_value(E, E.obj, p, c);
          e.kc = skey(viol);
          e.ks = skey(E.maximize ? o : -o);
          e.g = g;
          e.origin = 1;
          keep = !full || tbetter(e, w);
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (!m) continue;
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(E.count, (unsigned long long)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < E.cap) E.out[pos] = e;
      }
    }
  }
}

// Best-first bitonic sort of P (power of two) entries: one CTA in shared memory.
__global__ void __launch_bounds__(1024) trace_sort_small_kernel(TEntry* a, unsigned n, unsigned P) {
  extern __shared__ __align__(16) unsigned char tr_sm[];
  TEntry* es = reinterpret_cast<TEntry*>(tr_sm);
  for (unsigned i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < n) {
      es[i] = a[i];
    } else {
      es[i].kc = 0;
      es[i].ks = 0;
      es[i].g = ~0ull;
      es[i].origin = 0;
    }
  }
  __syncthreads();
  for (unsigned size = 2; size <= P; size <<= 1)
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      for (unsigned q = threadIdx.x; q < (P >> 1); q += blockDim.x) {
        const unsigned i = ((q & ~(stride - 1)) << 1) | (q & (stride - 1)), j = i + stride;
        const TEntry x = es[i], y = es[j];
        const bool first = (i & size) == 0;
        if (first ? tbetter(y, x) : tbetter(x, y)) {
          es[i] = y;
          es[j] = x;
        }
      }
      __syncthreads();
    }
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) a[i] = es[i];
}

// One compare-exchange stage of a best-first bitonic sort in global memory
// (P a power of two; entries past n are padding written by the caller).
__global__ void trace_sort_step_kernel(TEntry* a, unsigned P, unsigned size, unsigned stride) {
  const unsigned q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (P >> 1)) return;
  const unsigned i = ((q & ~(stride - 1)) << 1) | (q & (stride - 1)), j = i + stride;
  const TEntry x = a[i], y = a[j];
  const bool first = (i & size) == 0;
  if (first ? tbetter(y, x) : tbetter(x, y)) {
    a[i] = y;
    a[j] = x;
  }
}

__global__ void trace_pad_kernel(TEntry* a, unsigned n, unsigned P) {
  const unsigned i = n + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  a[i].kc = 0;
  a[i].ks = 0;
  a[i].g = ~0ull;
  a[i].origin = 0;
}

// carry bookkeeping: clear origins at a batch start / count the batch's entries
__global__ void trace_origin_kernel(TEntry* a, unsigned n, int mode, unsigned long long* count) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mode == 0) a[i].origin = 0;
  else if (a[i].origin) atomicAdd(count, 1ull);
}

}  // namespace apexb200

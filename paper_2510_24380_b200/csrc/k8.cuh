// k8.cuh — K8: the factorizer's hierarchy encoding on the device
// (reference factorizer.encode_hierarchy,
// factorizer.py:157-171, 218-233, over nn.MLP, nn.py:44-62, and the synthon
// feature hashing, props.py:43-67).
//
// Pipeline, every stage fp64 like the reference (the table it feeds is
// rounded to fp32 only at K1):
//   features   one thread per synthon: UTF-8 code points of the token, every
//              1/2/3-gram hashed with BLAKE2b-64 of "<salt>:<ngram>" (RFC 7693,
//              digest length 8, no key), bucket = digest % p, count * 0.25;
//   MLPs       tiled fp64 GEMM with the bias and tanh fused in the epilogue
//              (Y = act(X @ W + b)), optional row gather of X (h_s[member_ids]);
//   DeepSets   mean pooling over contiguous segments (np.add.reduceat order:
//              sequential sums), then the rho network;
//   key input  [h_r, h_t[rg_parent]];
//   pairs      u[p] = v[member[p]] @ K[j]^T with K[j] = key MLP row j viewed
//              (d, d_u), one CTA per R-group with K[j] in shared memory.
// The result u stays resident for K1 (no host round trip of the pair
// matrix).  Sums run in a fixed order that differs from numpy's BLAS
// blocking and CUDA's tanh from numpy's in the last ulp, so u agrees with the
// reference to ~1e-15 relative, and the fp32 table to the last bit almost
// everywhere (tests/test_gpu_k8.py states the tolerance).
#pragma once
#include "common.cuh"

namespace apexb200 {

// ---------------------------------------------------------------------------
// BLAKE2b (RFC 7693), one block, unkeyed, digest length 8
__device__ __forceinline__ unsigned long long rotr64(unsigned long long x, int n) { return (x >> n) | (x << (64 - n)); }

__constant__ unsigned long long kBlakeIV[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                               0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                               0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
__constant__ unsigned char kBlakeSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

#define APEX_B2G(a, b, c, d, x, y)   \
  a = a + b + x;                     \
  d = rotr64(d ^ a, 32);             \
  c = c + d;                         \
  b = rotr64(b ^ c, 24);             \
  a = a + b + y;                     \
  d = rotr64(d ^ a, 16);             \
  c = c + d;                         \
  b = rotr64(b ^ c, 63);

// first 8 digest bytes (little-endian) of BLAKE2b-64(msg[0, len)), len <= 128
__device__ unsigned long long blake2b64(const unsigned char* msg, int len) {
  unsigned long long m[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i] = 0;
  for (int i = 0; i < len; ++i) m[i >> 3] |= (unsigned long long)msg[i] << (8 * (i & 7));
  unsigned long long h0 = kBlakeIV[0] ^ 0x01010008ull;  // fanout 1, depth 1, no key, digest length 8
  unsigned long long v[16];
  v[0] = h0;
#pragma unroll
  for (int i = 1; i < 8; ++i) v[i] = kBlakeIV[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) v[8 + i] = kBlakeIV[i];
  v[12] ^= (unsigned long long)len;  // t (bytes compressed), single block
  v[14] = ~v[14];                    // last block
  for (int r = 0; r < 12; ++r) {
    const unsigned char* s = kBlakeSigma[r];
    APEX_B2G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
    APEX_B2G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
    APEX_B2G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
    APEX_B2G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
    APEX_B2G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
    APEX_B2G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
    APEX_B2G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
    APEX_B2G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
  }
  return h0 ^ v[0] ^ v[8];
}
#undef APEX_B2G

// props.synthon_features for every synthon (thread per synthon): features
// [n_syn][p] = 0.25 * count of the token's 1/2/3-gram buckets
__global__ void k8_features_kernel(const unsigned char* __restrict__ bytes, const long long* __restrict__ off,
                                   long long n_syn, const unsigned char* __restrict__ salt, int salt_len, int p,
                                   double scale, double* __restrict__ feat) {
  const long long sidx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (sidx >= n_syn) return;
  const unsigned char* tok = bytes + off[sidx];
  const int nb = (int)(off[sidx + 1] - off[sidx]);
  double* out = feat + sidx * p;
  for (int i = 0; i < p; ++i) out[i] = 0.0;
  // code point starts of the UTF-8 token (n-grams are over code points)
  int starts[65];
  int n_cp = 0;
  for (int i = 0; i < nb && n_cp < 64; ++i)
    if ((tok[i] & 0xC0) != 0x80) starts[n_cp++] = i;
  starts[n_cp] = nb;
  unsigned char msg[128];
  for (int i = 0; i < salt_len; ++i) msg[i] = salt[i];
  for (int n = 1; n <= 3; ++n) {
    for (int i = 0; i + n <= n_cp; ++i) {
      const int b0 = starts[i], b1 = starts[i + n];
      const int len = salt_len + (b1 - b0);
      if (len > 128) continue;  // (tokens are short; the caller rejects longer n-grams)
      for (int k = 0; k < b1 - b0; ++k) msg[salt_len + k] = tok[b0 + k];
      const unsigned long long h = blake2b64(msg, len);
      out[h % (unsigned long long)p] += 1.0;
    }
  }
  for (int i = 0; i < p; ++i) out[i] *= scale;
}

// ---------------------------------------------------------------------------
// Y[M][N] = act(X[rows][K] @ W[K][N] + b) (fp64), X rows optionally gathered
// (row i of the product reads X[gather[i]]).  64 x 64 output tile per CTA,
// 256 threads x (4 x 4) outputs, K in 16-wide shared-memory slabs; each
// output sums k = 0..K-1 in order.
constexpr int kGemmTile = 64, kGemmK = 16;
__global__ void __launch_bounds__(256) k8_gemm_kernel(const double* __restrict__ X, int ldx,
                                                      const long long* __restrict__ gather, long long M, int K,
                                                      const double* __restrict__ W, const double* __restrict__ b,
                                                      int N, int act_tanh, double* __restrict__ Y, int ldy) {
  __shared__ double As[kGemmK][kGemmTile + 1];
  __shared__ double Bs[kGemmK][kGemmTile];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long row0 = (long long)blockIdx.y * kGemmTile;
  const int col0 = blockIdx.x * kGemmTile;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kGemmK) {
    // A slab: 64 rows x 16 k (4 per thread), B slab: 16 k x 64 cols (4 per thread)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = threadIdx.x + 256 * e;
      const int r = idx / kGemmK, kk = idx % kGemmK;
      const long long gr = row0 + r;
      double a = 0.0;
      if (gr < M && k0 + kk < K) {
        const long long src = gather ? gather[gr] : gr;
        a = X[src * ldx + k0 + kk];
      }
      As[kk][r] = a;
      const int kb = idx / kGemmTile, cb = idx % kGemmTile;
      Bs[kb][cb] = (k0 + kb < K && col0 + cb < N) ? W[(long long)(k0 + kb) * N + col0 + cb] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGemmK; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long gr = row0 + ty * 4 + i;
    if (gr >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = col0 + tx * 4 + j;
      if (gc >= N) continue;
      double y = b ? __dadd_rn(acc[i][j], b[gc]) : acc[i][j];
      if (act_tanh) y = tanh(y);
      Y[gr * ldy + gc] = y;
    }
  }
}

// mean over contiguous segments: Y[g][c] = (sum_{i in seg g} X[i][c]) / size
// (np.add.reduceat(...) / sizes: sequential sums in row order)
__global__ void k8_segment_mean_kernel(const double* __restrict__ X, int D, const long long* __restrict__ off,
                                       double* __restrict__ Y) {
  const int g = blockIdx.x;
  const long long a = off[g], e = off[g + 1];
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    double s = 0.0;
    bool first = true;
    for (long long i = a; i < e; ++i) {
      const double x = X[i * D + c];
      s = first ? x : __dadd_rn(s, x);
      first = false;
    }
    Y[(long long)g * D + c] = __ddiv_rn(s, (double)(e - a));
  }
}

// key input [h_r[j], h_t[rg_parent[j]]]
__global__ void k8_key_input_kernel(const double* __restrict__ h_r, int d_r, const double* __restrict__ h_t, int d_t,
                                    const int* __restrict__ parent, int n_rg, double* __restrict__ out) {
  const int j = blockIdx.x;
  if (j >= n_rg) return;
  for (int c = threadIdx.x; c < d_r + d_t; c += blockDim.x)
    out[(long long)j * (d_r + d_t) + c] = c < d_r ? h_r[(long long)j * d_r + c] : h_t[(long long)parent[j] * d_t + c - d_r];
}

// u[p][dd] = sum_e v[member[p]][e] * K[j][dd][e] for the pair rows p of R-group j
__global__ void k8_pairs_kernel(const double* __restrict__ v, int d_u, const double* __restrict__ kflat, int d,
                                const long long* __restrict__ rg_off, const long long* __restrict__ members,
                                double* __restrict__ u) {
  extern __shared__ double Ks[];  // [d][d_u]
  const int j = blockIdx.x;
  const double* K = kflat + (long long)j * d * d_u;
  for (int i = threadIdx.x; i < d * d_u; i += blockDim.x) Ks[i] = K[i];
  __syncthreads();
  const long long a = rg_off[j], e = rg_off[j + 1];
  for (long long idx = a * d + threadIdx.x + (long long)blockIdx.y * blockDim.x; idx < e * d;
       idx += (long long)gridDim.y * blockDim.x) {
    const long long p = idx / d;
    const int dd = (int)(idx - p * d);
    const double* vr = v + members[p] * d_u;
    const double* kr = Ks + dd * d_u;
    double s = 0.0;
    for (int q = 0; q < d_u; ++q) s = __fma_rn(vr[q], kr[q], s);
    u[p * d + dd] = s;
  }
}

}  // namespace apexb200

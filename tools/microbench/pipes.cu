// Microbenchmark: issue rate of the enumeration inner loop variants on sm_100a.
// Measures products/cycle/SM for: (a) FSETP predicate chain, (b) FADD2 + LOP3
// sign-bit chain, with y values broadcast from shared memory and per-row
// thresholds in registers.  Not part of the product; used to pick the design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef NT
#define NT 9
#endif
#define NTP ((NT + 3) / 4 * 4)
#define NCOL 256

template <int RL>
__global__ void k_fsetp(const float* __restrict__ thr_in, int iters, unsigned* out) {
  __shared__ __align__(16) float ys[NCOL * NTP];
  for (int i = threadIdx.x; i < NCOL * NTP; i += blockDim.x) ys[i] = (float)((i * 7919) % 1000) * 0.001f;
  __syncthreads();
  float thr[RL][NT];
#pragma unroll
  for (int r = 0; r < RL; ++r)
#pragma unroll
    for (int i = 0; i < NT; ++i) thr[r][i] = thr_in[(threadIdx.x * RL + r) * NT + i];
  unsigned hits = 0;
  for (int it = 0; it < iters; ++it) {
    for (int j0 = 0; j0 < NCOL; j0 += 8) {
      bool any = false;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const float4* p = reinterpret_cast<const float4*>(ys + (j0 + jj) * NTP);
        float y[NTP];
#pragma unroll
        for (int q = 0; q < NTP / 4; ++q) {
          float4 v = p[q];
          y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          bool pass = true;
#pragma unroll
          for (int i = 0; i < NT; ++i) pass = pass && (y[i] <= thr[r][i]);
          any = any || pass;
        }
      }
      if (__any_sync(0xffffffffu, any)) hits += __popc(__ballot_sync(0xffffffffu, any));
    }
  }
  if (hits == 12345) out[0] = hits;
  out[blockIdx.x * blockDim.x + threadIdx.x] = hits;
}

// FADD2 with sign bits: d = y - t' ; pass iff sign set for all (t' = nextup(t)).
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int RL>
__global__ void k_fadd2(const float* __restrict__ thr_in, int iters, unsigned* out) {
  __shared__ __align__(16) float ys[NCOL * NTP];
  for (int i = threadIdx.x; i < NCOL * NTP; i += blockDim.x) ys[i] = (float)((i * 7919) % 1000) * 0.001f;
  __syncthreads();
  constexpr int NP = (NT + 1) / 2;
  unsigned long long thr[RL][NP];
#pragma unroll
  for (int r = 0; r < RL; ++r)
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      float a = thr_in[(threadIdx.x * RL + r) * NT + 2 * i];
      float b = (2 * i + 1 < NT) ? thr_in[(threadIdx.x * RL + r) * NT + 2 * i + 1] : -__int_as_float(0x7f800000);
      thr[r][i] = (unsigned long long)__float_as_uint(a) | ((unsigned long long)__float_as_uint(b) << 32);
    }
  unsigned hits = 0;
  for (int it = 0; it < iters; ++it) {
    for (int j0 = 0; j0 < NCOL; j0 += 8) {
      unsigned anyw = 0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(ys + (j0 + jj) * NTP);
        unsigned long long y[NTP / 2];
#pragma unroll
        for (int q = 0; q < NTP / 4; ++q) {
          ulonglong2 v = p[q];
          y[2 * q] = v.x; y[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < RL; ++r) {
          unsigned acc = 0xffffffffu;
#pragma unroll
          for (int i = 0; i < NP; ++i) {
            unsigned long long d = fsub2(y[i], thr[r][i]);
            acc &= (unsigned)d & (unsigned)(d >> 32);
          }
          anyw |= acc;
        }
      }
      bool any = (int)anyw < 0;
      if (__any_sync(0xffffffffu, any)) hits += __popc(__ballot_sync(0xffffffffu, any));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = hits;
}

template <typename K>
void run(const char* name, K kern, int rl, const float* thr, unsigned* out, int blocks, int threads, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kern<<<blocks, threads>>>(thr, 2, out);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(thr, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double products = (double)blocks * threads * iters * NCOL * rl;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double pps = products / (ms * 1e-3);
  printf("%-10s NT=%d RL=%d threads=%d blocks=%d: %.3f ms  %.3e products/s  %.2f products/clk/SM (@%d MHz max) err=%s\n",
         name, NT, rl, threads, blocks, ms, pps, pps / (sms * clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* thr; unsigned* out;
  cudaMalloc(&thr, 1 << 24); cudaMalloc(&out, 1 << 24);
  cudaMemset(thr, 0, 1 << 24);
  int iters = 200;
  for (int threads : {256, 512}) {
    int blocks = sms * (2048 / threads);
    run("fsetp", k_fsetp<1>, 1, thr, out, blocks, threads, iters);
    run("fsetp", k_fsetp<2>, 2, thr, out, blocks, threads, iters);
    run("fsetp", k_fsetp<4>, 4, thr, out, blocks, threads, iters / 2);
    run("fadd2", k_fadd2<1>, 1, thr, out, blocks, threads, iters);
    run("fadd2", k_fadd2<2>, 2, thr, out, blocks, threads, iters);
    run("fadd2", k_fadd2<4>, 4, thr, out, blocks, threads, iters / 2);
  }
  printf("SMs=%d\n", sms);
  return 0;
}

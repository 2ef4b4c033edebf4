// Pipe issue rates on sm_100a: warp-instructions per cycle per SM for FSETP
// (predicate chain), FADD, FADD2, LOP3, FMNMX, IADD3, HSETP2.  Independent
// chains, register operands only.  Tuning aid; not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

#define N_IT 4096
#define CH 8

__global__ void k_fsetp(const float* in, int* out) {
  float a[CH], t[CH];
  for (int i = 0; i < CH; ++i) { a[i] = in[threadIdx.x + i]; t[i] = in[threadIdx.x + 32 + i]; }
  int acc = 0;
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      bool p = a[i] <= t[i];
      p = p & (a[(i + 1) % CH] <= t[(i + 3) % CH]);
      p = p & (a[(i + 2) % CH] <= t[(i + 5) % CH]);
      p = p & (a[(i + 3) % CH] <= t[(i + 6) % CH]);
      acc += p;
    }
    a[it & (CH - 1)] += 1.0f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

__global__ void k_fadd2(const unsigned long long* in, int* out) {
  unsigned long long a[CH], t[CH];
  for (int i = 0; i < CH; ++i) { a[i] = in[threadIdx.x + i]; t[i] = in[threadIdx.x + 32 + i]; }
  unsigned acc = 0;
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const unsigned long long d = fsub2(a[i], t[i]);
      const unsigned long long e = fsub2(a[(i + 1) % CH], t[(i + 3) % CH]);
      acc ^= (unsigned)d & (unsigned)(d >> 32) & (unsigned)e;
    }
    a[it & (CH - 1)] += 1;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_fadd(const float* in, int* out) {
  float a[CH], t[CH];
  for (int i = 0; i < CH; ++i) { a[i] = in[threadIdx.x + i]; t[i] = in[threadIdx.x + 32 + i]; }
  float acc = 0;
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      float d = a[i] - t[i];
      float e = a[(i + 1) % CH] - t[(i + 2) % CH];
      float f = a[(i + 2) % CH] - t[(i + 3) % CH];
      float g = a[(i + 3) % CH] - t[(i + 4) % CH];
      acc += d * 0.0f + e * 0.0f + f * 0.0f + g * 0.0f;
      t[i] = d;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (int)acc;
}

__global__ void k_lop3(const unsigned* in, int* out) {
  unsigned a[CH];
  for (int i = 0; i < CH; ++i) a[i] = in[threadIdx.x + i];
  for (int it = 0; it < N_IT; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = (a[i] & a[(i + 1) % CH]) | a[(i + 3) % CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = (a[i] ^ a[(i + 2) % CH]) & a[(i + 5) % CH];
  }
  unsigned acc = 0;
  for (int i = 0; i < CH; ++i) acc ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <typename K, typename T>
void run(const char* name, K kern, const T* in, int* out, double inst_per_iter) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int threads = 256, blocks = sms * 8;
  kern<<<blocks, threads>>>(in, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(in, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_inst = (double)blocks * threads / 32 * N_IT * inst_per_iter;
  double per_clk_sm = warp_inst / (ms * 1e-3) / (sms * (double)clk * 1e3);
  printf("%-8s %.3f ms  %.2f target-warp-inst/clk/SM (@%d MHz)\n", name, ms, per_clk_sm, clk / 1000);
}

int main() {
  void* in; int* out;
  cudaMalloc(&in, 1 << 20); cudaMemset(in, 0, 1 << 20); cudaMalloc(&out, 1 << 24);
  run("fsetp", k_fsetp, (const float*)in, out, CH * 4);
  run("fadd2", k_fadd2, (const unsigned long long*)in, out, CH * 2);
  run("fadd", k_fadd, (const float*)in, out, CH * 4);
  run("lop3", k_lop3, (const unsigned*)in, out, CH * 2);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

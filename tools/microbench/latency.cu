// Microbenchmark: dependent-load latency on sm_100a (pointer chasing, one
// thread) for a working set in L1 / L2 / HBM, and the DADD / 32-bit divide
// dependent-chain latencies.  Calibrates the per-row latency chains of the
// finalize / materialize kernels.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase(const uint32_t* __restrict__ next, int steps, uint32_t start, unsigned long long* out) {
  uint32_t p = start;
  // warm pass
  for (int i = 0; i < steps; ++i) p = next[p];
  const unsigned long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = next[p];
  const unsigned long long t1 = clock64();
  out[0] = (t1 - t0);
  out[1] = p;
}

__global__ void chase_cold(const uint32_t* __restrict__ next, int steps, uint32_t start, unsigned long long* out) {
  uint32_t p = start;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  const unsigned long long t1 = clock64();
  out[0] = (t1 - t0);
  out[1] = p;
}

__global__ void dadd_chain(double x, int n, unsigned long long* out, double* sink) {
  double a = x;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, x);
  const unsigned long long t1 = clock64();
  out[0] = t1 - t0;
  sink[0] = a;
}

__global__ void f2f_chain(float x, int n, unsigned long long* out, double* sink) {
  double a = 0.0;
  float y = x;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = __dadd_rn(a, (double)y);
    y = (float)a;  // dependent: F2F.F64.F32 + DADD + F2F.F32.F64 per step
  }
  const unsigned long long t1 = clock64();
  out[0] = t1 - t0;
  sink[0] = a;
}

__global__ void div_chain(uint32_t x, uint32_t d, int n, unsigned long long* out) {
  uint32_t a = x;
  const unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = a / d + x;
  const unsigned long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = a;
}

int main() {
  unsigned long long* d_out;
  double* d_sink;
  cudaMalloc(&d_out, 64);
  cudaMalloc(&d_sink, 64);
  unsigned long long h[2];
  for (size_t ws : {16u << 10, 256u << 10, 4u << 20, 32u << 20, 512u << 20}) {
    const size_t n = ws / 4;
    std::vector<uint32_t> nx(n);
    // random cycle with stride >= 128 B lines
    const size_t lines = n / 32;
    std::vector<uint32_t> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = (uint32_t)i;
    uint64_t s = 88172645463325252ull;
    for (size_t i = lines - 1; i > 0; --i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      std::swap(perm[i], perm[s % (i + 1)]);
    }
    for (size_t i = 0; i < lines; ++i) nx[perm[i] * 32] = perm[(i + 1) % lines] * 32;
    uint32_t* d;
    cudaMalloc(&d, ws);
    cudaMemcpy(d, nx.data(), ws, cudaMemcpyHostToDevice);
    const int steps = 2000;
    chase<<<1, 1>>>(d, steps, perm[0] * 32, d_out);
    cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    const double warm = (double)h[0] / steps;
    chase_cold<<<1, 1>>>(d, steps, perm[0] * 32, d_out);
    cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
    printf("working set %8zu KB: dependent ld (ld.global, warm) %7.1f cyc   ld.cg %7.1f cyc\n", ws >> 10, warm,
           (double)h[0] / steps);
    cudaFree(d);
  }
  dadd_chain<<<1, 1>>>(1.0, 4096, d_out, d_sink);
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("DADD dependent chain: %.1f cyc/op\n", (double)h[0] / 4096);
  f2f_chain<<<1, 1>>>(1.0f, 4096, d_out, d_sink);
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("F2F.F64.F32 + DADD + F2F.F32.F64 dependent chain: %.1f cyc/step\n", (double)h[0] / 4096);
  div_chain<<<1, 1>>>(123456789u, 977u, 4096, d_out);
  cudaMemcpy(h, d_out, 16, cudaMemcpyDeviceToHost);
  printf("u32 divide + add chain: %.1f cyc/op\n", (double)h[0] / 4096);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}

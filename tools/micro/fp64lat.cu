// FP64 latency probes (cycles per dependent op) on sm_100a: DFMA, DMUL, rsqrt(double), F2F, 64-bit SHFL,
// and the same chain with 8 independent warps per SMSP (throughput check).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double* out, long long* clk, double seed) {
  double v = seed + threadIdx.x * 1e-3;
  float f = (float)seed;
  long long t0, t1;
  const int N = 256;
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = fma(v, 0.999, 1.0);
  t1 = clock64(); if (threadIdx.x == 0) clk[0] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = v * 1.0001;
  t1 = clock64(); if (threadIdx.x == 0) clk[1] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = rsqrt(v + 2.0);
  t1 = clock64(); if (threadIdx.x == 0) clk[2] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.0;
  t1 = clock64(); if (threadIdx.x == 0) clk[3] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) { f = (float)v; v = (double)f + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) clk[4] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.999f, 1.0f);
  t1 = clock64(); if (threadIdx.x == 0) clk[5] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = sqrt(v + 2.0);
  t1 = clock64(); if (threadIdx.x == 0) clk[6] = (t1 - t0);
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = rsqrtf(f + 2.0f);
  t1 = clock64(); if (threadIdx.x == 0) clk[7] = (t1 - t0);
  out[threadIdx.x] = v + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8192 * 8); cudaMalloc(&c, 64 * 8);
  const char* names[] = {"dfma", "dmul", "rsqrt(d)", "shfl64+dadd", "f2f+f2f+dadd", "ffma", "sqrt(d)", "rsqrtf"};
  for (int nt : {32, 256, 1024}) {
    probe<<<1, nt>>>(o, c, 1.0);
    probe<<<1, nt>>>(o, c, 1.0);
    long long h[8]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads=%4d:", nt);
    for (int i = 0; i < 8; ++i) printf(" %s %.1f", names[i], h[i] / 256.0);
    printf("\n");
  }
  return 0;
}

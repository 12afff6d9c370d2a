// Latency probes (cycles per dependent op) on sm_100a: SHFL, FADD, sqrtf, IEEE div, rcp-mul, bar.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(float* out, long long* clk, float seed) {
  float v = seed + threadIdx.x * 1e-3f;
  long long t0, t1;
  const int N = 256;
  // SHFL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1.0f;
  t1 = clock64(); if (threadIdx.x == 0) clk[0] = (t1 - t0);
  // FADD chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = v * 0.999f + 1.0f;
  t1 = clock64(); if (threadIdx.x == 0) clk[1] = (t1 - t0);
  // sqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = sqrtf(v + 2.0f);
  t1 = clock64(); if (threadIdx.x == 0) clk[2] = (t1 - t0);
  // div chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = 3.0f / (v + 1.5f);
  t1 = clock64(); if (threadIdx.x == 0) clk[3] = (t1 - t0);
  // rcp approx chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __fdividef(3.0f, v + 1.5f);
  t1 = clock64(); if (threadIdx.x == 0) clk[4] = (t1 - t0);
  // syncthreads
  __shared__ float s[1024];
  t0 = clock64();
  for (int i = 0; i < N; ++i) { s[threadIdx.x] = v; __syncthreads(); v += s[(threadIdx.x + 1) % blockDim.x]; }
  t1 = clock64(); if (threadIdx.x == 0) clk[5] = (t1 - t0);
  // __frsqrt_rn
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __fsqrt_rn(v + 2.0f);
  t1 = clock64(); if (threadIdx.x == 0) clk[6] = (t1 - t0);
  // shfl idx broadcast chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, i & 31) + 1.0f;
  t1 = clock64(); if (threadIdx.x == 0) clk[7] = (t1 - t0);
  out[threadIdx.x] = v;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 64 * 8);
  const char* names[] = {"shfl_xor+fadd", "ffma", "sqrtf", "ieee div", "fdividef", "bar+sts/lds", "fsqrt_rn", "shfl_idx+fadd"};
  for (int nt : {32, 128, 256}) {
    probe<<<1, nt>>>(o, c, 1.0f);
    probe<<<1, nt>>>(o, c, 1.0f);
    long long h[8]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
    printf("threads=%d:", nt);
    for (int i = 0; i < 8; ++i) printf(" %s=%.1f", names[i], h[i] / 256.0);
    printf("\n");
  }
}

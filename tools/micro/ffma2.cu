// Throughput of FFMA vs FFMA2 (fma.rn.f32x2) per SM: 8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__global__ void k1(float* out, int iters, float s) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], s, 1.0f);
  float t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k2(float* out, int iters, float s) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) a[i] = pk(threadIdx.x + i, i);
  const unsigned long long sv = pk(s, s), one = pk(1.f, 1.f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(sv), "l"(one));
  float t = 0;
  for (int i = 0; i < 8; ++i) { float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i])); t += x + y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000, blocks = 148 * 4, threads = 512;
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (v == 0) k1<<<blocks, threads>>>(out, iters, 0.999f); else k2<<<blocks, threads>>>(out, iters, 0.999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double lanes = (double)blocks * threads * iters * 8 * (v ? 2 : 1);
      if (rep) printf("%s: %.3f ms, %.1f TFLOP/s (FMA=2 flops)\n", v ? "FFMA2" : "FFMA", ms, lanes * 2 / ms / 1e9);
    }
  }
  return 0;
}

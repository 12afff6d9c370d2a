// Latency of 128 independent loads per lane (one warp) with different load flavours.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ float ld(const float* p) {
  float v;
  if (MODE == 0) asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (MODE == 1) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if (MODE == 2) asm volatile("ld.volatile.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
template <int MODE>
__global__ void k(const float* a, long long stride, float* out, long long* cyc) {
  float v[128];
  const int lane = threadIdx.x;
  long long c0 = clock64();
#pragma unroll
  for (int i = 0; i < 128; ++i) v[i] = ld<MODE>(a + (long long)i * stride + lane);
  float s = 0;
#pragma unroll
  for (int i = 0; i < 128; ++i) s += v[i];
  long long c1 = clock64();
  out[lane] = s;
  if (lane == 0) cyc[MODE] = c1 - c0;
}
int main() {
  float* a; cudaMalloc(&a, 64 << 20); cudaMemset(a, 0, 64 << 20);
  float* out; cudaMalloc(&out, 4096);
  long long* cyc; cudaMalloc(&cyc, 64);
  long long h[4];
  for (long long stride : {32LL, 1024LL, 32 * 32 * 33LL}) {
    for (int rep = 0; rep < 2; ++rep) {
      k<0><<<1, 32>>>(a, stride, out, cyc);
      k<1><<<1, 32>>>(a, stride, out, cyc);
      k<2><<<1, 32>>>(a, stride, out, cyc);
      k<3><<<1, 32>>>(a, stride, out, cyc);
      cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    }
    printf("stride %lld floats: relaxed.gpu %lld, cg %lld, volatile %lld, plain %lld cycles\n", stride, h[0], h[1], h[2], h[3]);
  }
  return 0;
}

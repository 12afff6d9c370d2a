// Micro-benchmark: issue rate / latency of the FP32, packed FP32x2 and FP64 FMA pipes and of
// shuffles on one SM (one CTA, `warps` warps), to size the leaf kernel's dependent chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipe_rates.cu -o pipe_rates
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int KIND, int CH>
__global__ void bench(float* out, long long* cyc) {
  float a[CH];
  double d[CH];
  unsigned long long p[CH];
  for (int i = 0; i < CH; ++i) {
    a[i] = threadIdx.x * 1e-3f + i;
    d[i] = a[i];
    float2 f = make_float2(a[i], a[i] + 1);
    p[i] = *reinterpret_cast<unsigned long long*>(&f);
  }
  const float b = 0.999f, c = 1e-4f;
  const unsigned long long bb = 0x3f7fbe773f7fbe77ull, cc = 0x38d1b71738d1b717ull;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (KIND == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b), "f"(c));
      if (KIND == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[i]) : "l"(bb), "l"(cc));
      if (KIND == 2) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[i]) : "d"(0.999), "d"(1e-4));
      if (KIND == 3) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 7)) + c;
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < CH; ++i) s += a[i] + (float)d[i] + __int_as_float((int)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int KIND, int CH>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4 * 1024 * 148);
  cudaMalloc(&cyc, 8 * 148);
  bench<KIND, CH><<<148, 32 * warps>>>(out, cyc);
  bench<KIND, CH><<<148, 32 * warps>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / kIters / CH;  // cycles per instruction per warp (per thread chain)
  printf("%-10s chains/thread %2d warps/SM %2d: %.3f cycles per instr (per warp stream); "
         "warp-instr/clk/SM %.2f\n", name, CH, warps, per, warps / per);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0, 1>("FFMA lat", 1);
  run<1, 1>("FFMA2 lat", 1);
  run<2, 1>("DFMA lat", 1);
  run<3, 1>("SHFL lat", 1);
  for (int w : {4, 8, 16}) {
    run<0, 8>("FFMA", w);
    run<1, 8>("FFMA2", w);
    run<2, 8>("DFMA", w);
    run<3, 8>("SHFL+add", w);
  }
  return 0;
}

// Micro-benchmark: dependent-chain latencies (unrolled, no loop overhead) of FFMA, FFMA2, DFMA,
// SHFL, LDS, STS->LDS round trip through __syncwarp, MUFU sqrt/rcp and the FP64 rsqrt used by the
// leaf kernel (one warp on one SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 chain_lat.cu -o chain_lat
#include <cstdio>
#include <cuda_runtime.h>

#define N 256
__global__ void lat_kernel(float* out, long long* cyc, float b, float c) {
  __shared__ float sh[1024];
  __shared__ double shd[64];
  const int lane = threadIdx.x;
  float a = lane * 1e-3f + 1.0f;
  double d = a;
  unsigned long long p;
  {
    float2 f = make_float2(a, a);
    p = *reinterpret_cast<unsigned long long*>(&f);
  }
  unsigned long long bb = 0x3f7fbe773f7fbe77ull, cc = 0x38d1b71738d1b717ull;
  sh[lane] = a;
  shd[lane] = d;
  __syncwarp();
  long long t[16];
  t[0] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a) : "f"(b), "f"(c));
  t[1] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p) : "l"(bb), "l"(cc));
  t[2] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d) : "d"(0.999), "d"(1e-4));
  t[3] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) a = __shfl_sync(0xffffffffu, a, (lane + 1) & 31);
  t[4] = clock64();
  int idx = lane;
#pragma unroll
  for (int i = 0; i < N; ++i) idx = __float_as_int(sh[idx & 1023]) & 31;  // dependent LDS
  t[5] = clock64();
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {  // STS -> syncwarp -> LDS of another lane's value
    sh[lane] = a;
    __syncwarp();
    a = sh[(lane + 1) & 31] + 1.0f;
    __syncwarp();
  }
  t[6] = clock64();
#pragma unroll
  for (int i = 0; i < N / 4; ++i) a = sqrtf(a) + 1.0f;
  t[7] = clock64();
#pragma unroll
  for (int i = 0; i < N / 4; ++i) a = __frcp_rn(a) + 1.0f;
  t[8] = clock64();
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    const double e = fma(-d, y * y, 1.0);
    d = fma(fma(e, 0.375, 0.5), e * y, y) + 1.0;
  }
  t[9] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("add.f32 %0, %0, %1;" : "+f"(a) : "f"(c));
  t[10] = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) d = __shfl_sync(0xffffffffu, d, (lane + 1) & 31);
  t[11] = clock64();
  out[lane] = a + (float)d + __int_as_float((int)p) + idx;
  if (lane == 0)
    for (int i = 0; i < 11; ++i) cyc[i] = t[i + 1] - t[i];
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4096);
  cudaMalloc(&cyc, 256);
  for (int rep = 0; rep < 2; ++rep) lat_kernel<<<1, 32>>>(out, cyc, 0.999f, 1e-4f);
  cudaDeviceSynchronize();
  long long h[11];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[11] = {"FFMA", "FFMA2", "DFMA", "SHFL.f32", "LDS (dep)", "STS+syncwarp+LDS+FADD (x4 ops)",
                        "sqrtf+FADD", "frcp_rn+FADD", "rsqrt_nr(f64)+DADD", "FADD", "SHFL.f64"};
  const int cnt[11] = {N, N, N, N, N, N / 4, N / 4, N / 4, N / 4, N, N};
  for (int i = 0; i < 11; ++i) printf("%-34s %7.2f cycles per dependent op\n", nm[i], (double)h[i] / cnt[i]);
  return 0;
}

// Micro-benchmark: one 64 x 32 Alg. 4 (MGS) block per warp, lane = column, 4 warps (one per SM
// sub-partition) per CTA, 148 CTAs.  Variants of the step's communication and scalar chain:
//   V0 publish the pivot by lane k+1 after the update (colbuf), q via qbuf;  sqrtf + __frcp_rn
//   V1 = V0 with inv = 1.0f / rkk (IEEE divide, correctly rounded: the same bits as __frcp_rn)
//   V2 pre-update publish + next pivot recomputed in every lane, q in registers; sqrtf + 1/x
//   V3 = V2 with R(k,k), 1/R(k,k) from one FP64 rsqrt
// Prints cycles per step (clock64 around the 32 steps, warp 0 of CTA 0) and checks V1..V3 give
// the same Q bits as V0 (V3 may differ by an ulp: different rounding of 1/R(k,k)).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mgs_warp_bench.cu -o mgs_warp_bench
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra, rb, rc, rd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(ra) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(rc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  float2 d;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d.x), "=f"(d.y) : "l"(rd));
  return d;
}
__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y * y, 1.0);
  return fma(fma(e, 0.375, 0.5), e * y, y);
}

constexpr int BR = 64, LD = 33;

template <int V>
__global__ void __launch_bounds__(128, 1) bench(const float* A, float* Q, float* R, long long* cyc) {
  __shared__ __align__(16) float L[4][BR * LD];  // column-major panel copy [col][row] per warp
  __shared__ __align__(16) float pub[4][2][BR];
  __shared__ __align__(16) float qh[4][2][BR];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* a = A + ((long long)blockIdx.x * 4 + w) * BR * 32;
  float2 x[BR / 2];
#pragma unroll
  for (int i = 0; i < BR / 2; ++i) x[i] = make_float2(a[lane * BR + 2 * i], a[lane * BR + 2 * i + 1]);
  float Rrow[32];
  float* colb = pub[w][0];
  float* qb = qh[w][0];
  float2 v[BR / 2];
  __syncwarp();
  long long t0 = clock64();
  if (V <= 1 || V == 9) {
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < BR / 4; ++i)
        *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
    __syncwarp();
#pragma unroll 1
    for (int k = 0; k < 32; ++k) {
#pragma unroll
      for (int i = 0; i < BR / 4; ++i) {
        const float4 c4 = *reinterpret_cast<const float4*>(colb + 4 * i);
        v[2 * i] = make_float2(c4.x, c4.y);
        v[2 * i + 1] = make_float2(c4.z, c4.w);
      }
      float2 acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) acc[i & 3] = ffma2(v[i], x[i], acc[i & 3]);
      const float tot = ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
      const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, k));
      const bool zero = !(rkk > 0.f) || !isfinite(rkk);
      const float inv = zero ? 0.f : (V == 0 ? __frcp_rn(rkk) : 1.0f / rkk);
      const float rkj = zero ? 0.f : (lane == k ? rkk : tot * inv);
      Rrow[k] = rkj;
      const float q0 = colb[lane] * inv, q1 = colb[lane + 32] * inv;
      if (V == 9) {  // q_k formed in every lane from its copy of the pivot column (same bits)
        L[w][k * LD + lane] = q0;
        L[w][k * LD + lane + 32] = q1;
        const float2 iv = make_float2(inv, inv), nz = make_float2(-0.f, -0.f);
#pragma unroll
        for (int i = 0; i < BR / 2; ++i) v[i] = ffma2(v[i], iv, nz);
        __syncwarp();  // every lane has read colb before lane k + 1 republishes it
      } else {
      __syncwarp();
      qb[lane] = q0;
      qb[lane + 32] = q1;
      L[w][k * LD + lane] = q0;
      L[w][k * LD + lane + 32] = q1;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < BR / 4; ++i) {
        const float4 q4 = *reinterpret_cast<const float4*>(qb + 4 * i);
        v[2 * i] = make_float2(q4.x, q4.y);
        v[2 * i + 1] = make_float2(q4.z, q4.w);
      }
      }
      const float2 nr = make_float2(-rkj, -rkj);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) x[i] = ffma2(v[i], nr, x[i]);
      if (lane == k + 1)
#pragma unroll
        for (int i = 0; i < BR / 4; ++i)
          *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
      __syncwarp();
    }
  } else {
    float* pb0 = pub[w][1];
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < BR / 4; ++i)
        *reinterpret_cast<float4*>(pb0 + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < BR / 4; ++i) {
      const float4 c4 = *reinterpret_cast<const float4*>(pb0 + 4 * i);
      v[2 * i] = make_float2(c4.x, c4.y);
      v[2 * i + 1] = make_float2(c4.z, c4.w);
    }
#pragma unroll 1
    for (int k = 0; k < 32; ++k) {
      float* pb = pub[w][k & 1];
      float* qk = qh[w][k & 1];
      if (lane == k + 1)
#pragma unroll
        for (int i = 0; i < BR / 4; ++i)
          *reinterpret_cast<float4*>(pb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
      float2 acc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) acc[i & 3] = ffma2(v[i], x[i], acc[i & 3]);
      const float tot = ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
      const float n2k = __shfl_sync(0xffffffffu, tot, k);
      const float t1 = __shfl_sync(0xffffffffu, tot, (k + 1) & 31);
      float rkk, inv;
      bool zero;
      if (V == 2) {
        rkk = sqrtf(n2k);
        zero = !(rkk > 0.f) || !isfinite(rkk);
        inv = zero ? 0.f : 1.0f / rkk;
      } else {
        zero = !(n2k > 0.f) || !isfinite(n2k);
        const double nd = (double)n2k;
        const double ri = rsqrt_nr(zero ? 1.0 : nd);
        rkk = zero ? 0.f : (float)(nd * ri);
        inv = zero ? 0.f : (float)ri;
      }
      const float rkj = zero ? 0.f : (lane == k ? rkk : tot * inv);
      const float rk1 = zero ? 0.f : t1 * inv;
      Rrow[k] = rkj;
      const float2 iv = make_float2(inv, inv), nz = make_float2(-0.f, -0.f);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) v[i] = ffma2(v[i], iv, nz);
      if (lane == k)
#pragma unroll
        for (int i = 0; i < BR / 4; ++i)
          *reinterpret_cast<float4*>(qk + 4 * i) = make_float4(v[2 * i].x, v[2 * i].y, v[2 * i + 1].x, v[2 * i + 1].y);
      __syncwarp();
      L[w][k * LD + lane] = qk[lane];
      L[w][k * LD + lane + 32] = qk[lane + 32];
      const float2 n1 = make_float2(-rk1, -rk1), nr = make_float2(-rkj, -rkj);
      float2 xn[BR / 2];
#pragma unroll
      for (int i = 0; i < BR / 4; ++i) {
        const float4 c4 = *reinterpret_cast<const float4*>(pb + 4 * i);
        xn[2 * i] = ffma2(v[2 * i], n1, make_float2(c4.x, c4.y));
        xn[2 * i + 1] = ffma2(v[2 * i + 1], n1, make_float2(c4.z, c4.w));
      }
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) x[i] = ffma2(v[i], nr, x[i]);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) v[i] = xn[i];
    }
  }
  __syncwarp();
  long long t1 = clock64();
  float* q = Q + ((long long)blockIdx.x * 4 + w) * BR * 32;
  for (int j = 0; j < 32; ++j) q[j * BR + lane] = L[w][j * LD + lane], q[j * BR + lane + 32] = L[w][j * LD + lane + 32];
  for (int k = 0; k < 32; ++k) R[((long long)blockIdx.x * 4 + w) * 1024 + k * 32 + lane] = Rrow[k];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// V4/V5: TWO warps per 64 x 32 block (32 rows each, lane = column), warps 2p and 2p+1 (different
// SM sub-partitions; each sub-partition hosts warps of two different blocks).  The dot partials
// meet through shared memory and a 64-thread named barrier.  V4: q via qbuf; V5: q in registers.
template <int V>
__global__ void __launch_bounds__(256, 1) bench2(const float* A, float* Q, float* R, long long* cyc) {
  __shared__ __align__(16) float L[4][BR * LD];
  __shared__ __align__(16) float colb[4][2][32];
  __shared__ __align__(16) float qb[4][2][32];
  __shared__ __align__(16) float red[4][2][2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, pr = w >> 1, half = w & 1;
  const float* a = A + ((long long)blockIdx.x * 4 + pr) * BR * 32;
  float2 x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i)
    x[i] = make_float2(a[lane * BR + half * 32 + 2 * i], a[lane * BR + half * 32 + 2 * i + 1]);
  float Rrow[32];
  float* cb = colb[pr][half];
  float* qq = qb[pr][half];
  float2 v[16];
  __syncwarp();
  long long t0 = clock64();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      *reinterpret_cast<float4*>(cb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
  __syncwarp();
  int buf = 0;
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 c4 = *reinterpret_cast<const float4*>(cb + 4 * i);
      v[2 * i] = make_float2(c4.x, c4.y);
      v[2 * i + 1] = make_float2(c4.z, c4.w);
    }
    float2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i & 3] = ffma2(v[i], x[i], acc[i & 3]);
    const float part = ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) + ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
    float tot = part;
    if (V != 7) {  // V7: ablation without the pair exchange (wrong math, timing only)
      red[pr][buf][half][lane] = part;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + pr) : "memory");
      tot = red[pr][buf][0][lane] + red[pr][buf][1][lane];
      buf ^= 1;
    }
    float rkk, inv;
    if (V == 6) {  // ablation: no sqrt / divide on the chain (wrong math, timing only)
      rkk = __shfl_sync(0xffffffffu, tot, k);
      inv = rkk;
    } else if (V == 8) {  // FP32 rsqrt + one Newton step (approximate 1/R(k,k))
      const float n2 = __shfl_sync(0xffffffffu, tot, k);
      float y = rsqrtf(n2);
      y = y * fmaf(-0.5f * n2, y * y, 1.5f);
      rkk = n2 * y;
      inv = y;
    } else {
      rkk = sqrtf(__shfl_sync(0xffffffffu, tot, k));
      inv = 1.0f / rkk;
    }
    const bool zero = !(rkk > 0.f) || !isfinite(rkk);
    inv = zero ? 0.f : inv;
    const float rkj = zero ? 0.f : (lane == k ? rkk : tot * inv);
    Rrow[k] = rkj;
    const float q0 = cb[lane] * inv;
    L[pr][k * LD + half * 32 + lane] = q0;
    if (V == 4) {
      __syncwarp();
      qq[lane] = q0;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 q4 = *reinterpret_cast<const float4*>(qq + 4 * i);
        v[2 * i] = make_float2(q4.x, q4.y);
        v[2 * i + 1] = make_float2(q4.z, q4.w);
      }
    } else {
      const float2 iv = make_float2(inv, inv), nz = make_float2(-0.f, -0.f);
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = ffma2(v[i], iv, nz);
      __syncwarp();  // every lane has read cb before lane k+1 republishes it
    }
    const float2 nr = make_float2(-rkj, -rkj);
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = ffma2(v[i], nr, x[i]);
    if (lane == k + 1)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(cb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
    __syncwarp();
  }
  long long t1 = clock64();
  __syncthreads();
  float* q = Q + ((long long)blockIdx.x * 4 + pr) * BR * 32;
  for (int j = 0; j < 32; ++j) q[j * BR + half * 32 + lane] = L[pr][j * LD + half * 32 + lane];
  if (half == 0)
    for (int k = 0; k < 32; ++k) R[((long long)blockIdx.x * 4 + pr) * 1024 + k * 32 + lane] = Rrow[k];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int nblk = 148 * 4, ne = nblk * BR * 32;
  float* hA = (float*)malloc(ne * 4);
  srand(1);
  for (int i = 0; i < ne; ++i) hA[i] = (float)rand() / RAND_MAX - 0.5f;
  float *A, *Q, *R;
  long long* cyc;
  cudaMalloc(&A, ne * 4);
  cudaMalloc(&Q, ne * 4);
  cudaMalloc(&R, nblk * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  cudaMemcpy(A, hA, ne * 4, cudaMemcpyHostToDevice);
  float* ref = (float*)malloc(ne * 4);
  float* out = (float*)malloc(ne * 4);
  auto run = [&](auto kern, const char* name, int v) {
    for (int r = 0; r < 3; ++r) kern<<<148, (v >= 4 && v <= 8) ? 256 : 128>>>(A, Q, R, cyc);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(out, Q, ne * 4, cudaMemcpyDeviceToHost);
    if (v == 0) memcpy(ref, out, ne * 4);
    int diff = 0;
    for (int i = 0; i < ne; ++i) diff += out[i] != ref[i];
    printf("%-60s %6.1f cycles/step  (Q entries differing from V0: %d of %d)  %s\n", name, c / 32.0, diff, ne,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(bench<0>, "V0 colbuf publish + qbuf, sqrtf + __frcp_rn", 0);
  run(bench<1>, "V1 = V0 with 1.0f / rkk", 1);
  run(bench<9>, "V9 = V1 with q in registers (every lane scales its pivot copy)", 9);
  run(bench<2>, "V2 pre-update publish + recompute, q in regs, sqrtf + 1/x", 2);
  run(bench<3>, "V3 = V2 with one FP64 rsqrt", 3);
  run(bench2<4>, "V4 two warps per block (row halves), q via qbuf, sqrtf + 1/x", 4);
  run(bench2<5>, "V5 = V4 with q in registers", 5);
  run(bench2<6>, "V6 = V5 without sqrt/divide (ablation, wrong math)", 6);
  run(bench2<7>, "V7 = V5 without the pair exchange (ablation, wrong math)", 7);
  run(bench2<8>, "V8 = V5 with FP32 rsqrt + Newton", 8);
  return 0;
}

// Micro-benchmark: one 64 x 32 Alg. 4 (MGS) block per warp, lane = column, 4 warps per CTA, 148
// CTAs.  U0 = the leaf's current step (normalized pivot q_k broadcast through shared memory);
// U1 = the projection form of the same step: the pivot x_k is broadcast once (unnormalized), one
// lane-local dot gives d_j = x_k' x_j for every lane (lane k: ||x_k||^2), the update is
// x_j -= (d_j / d_k) x_k with x_k already in registers, and every column is normalized once at the
// end (q_j = x_j / R(j,j)); U2 = U1 with c_j = d_j * (1/d_k).  Prints cycles per step and the
// block's orthogonality / residual against an FP64 reference on random and graded blocks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mgs_unnorm.cu -o mgs_unnorm
#include <cmath>
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

constexpr int BR = 64, LD = 68;

template <int V>
__global__ void __launch_bounds__(128, 1) bench(const float* A, float* Q, float* R, long long* cyc) {
  extern __shared__ __align__(16) float dyn[];
  float (*L)[BR * LD] = reinterpret_cast<float (*)[BR * LD]>(dyn);
  float (*pub)[BR] = reinterpret_cast<float (*)[BR]>(dyn + 4 * BR * LD + 4);
  float (*qh)[BR] = reinterpret_cast<float (*)[BR]>(dyn + 4 * BR * LD + 4 + 4 * BR);
  float (*dsh)[32 * 33] = reinterpret_cast<float (*)[32 * 33]>(dyn + 4 * BR * LD + 4 + 8 * BR);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const float* a = A + ((long long)blockIdx.x * 4 + w) * BR * 32;
  float2 x[BR / 2];
#pragma unroll
  for (int i = 0; i < BR / 2; ++i) x[i] = make_float2(a[lane * BR + 2 * i], a[lane * BR + 2 * i + 1]);
  float Rrow[32];
  float* colb = pub[w];
  float* qb = qh[w];
  float2 v[BR / 2];
  __syncwarp();
  long long t0 = clock64();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < BR / 4; ++i)
      *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
  __syncwarp();
  if (V == 0 || V >= 5) {
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
      const float inv = zero ? 0.f : 1.0f / rkk;
      const float rkj = zero ? 0.f : (lane == k ? rkk : tot * inv);
      Rrow[k] = rkj;
      const float q0 = colb[lane] * inv, q1 = colb[lane + 32] * inv;
      __syncwarp();
      qb[lane] = q0;
      qb[lane + 32] = q1;
      if (V == 0) {
        L[w][k * LD + lane] = q0;
        L[w][k * LD + lane + 32] = q1;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < BR / 4; ++i) {
        const float4 q4 = *reinterpret_cast<const float4*>(qb + 4 * i);
        v[2 * i] = make_float2(q4.x, q4.y);
        v[2 * i + 1] = make_float2(q4.z, q4.w);
      }
      const float2 nr = make_float2(-rkj, -rkj);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) x[i] = ffma2(v[i], nr, x[i]);
      if (lane == k + 1)
#pragma unroll
        for (int i = 0; i < BR / 4; ++i)
          *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
      if (V == 5) {
        L[w][k * LD + lane] = q0;
        L[w][k * LD + lane + 32] = q1;
      }
      __syncwarp();
    }
  } else {
    float rjj = 0.f;  // lane j: R(j, j), recorded at step j
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
      const float dk = __shfl_sync(0xffffffffu, tot, k);
      const bool zero = !(dk > 0.f) || !isfinite(dk);
      float c;
      if (V == 1) c = (zero || lane <= k) ? 0.f : tot / dk;
      else if (V == 2 || V == 3) c = (zero || lane <= k) ? 0.f : tot * (1.0f / dk);
      else {
        float rc;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(dk));
        c = (zero || lane <= k) ? 0.f : tot * rc;
      }
      __syncwarp();  // every lane has read colb before lane k + 1 republishes it
      const float2 nc = make_float2(-c, -c);
#pragma unroll
      for (int i = 0; i < BR / 2; ++i) x[i] = ffma2(v[i], nc, x[i]);
      if (lane == k + 1)
#pragma unroll
        for (int i = 0; i < BR / 4; ++i)
          *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
      if (V <= 2) {  // R(k, k) = sqrt(d_k), R(k, j) = d_j / R(k, k) in the step
        const float rkk = sqrtf(dk);
        const float inv = zero ? 0.f : 1.0f / rkk;
        Rrow[k] = zero ? 0.f : (lane == k ? rkk : (lane > k ? tot * inv : 0.f));
        if (lane == k) rjj = zero ? 0.f : rkk;
      } else {  // deferred: record d_j (and d_k in lane k's slot)
        dsh[w][k * 33 + lane] = tot;
      }
      __syncwarp();
    }
    if (V >= 3) {
      // R from the recorded dots: R(k, k) = sqrt(d_k), R(k, j) = d_j / R(k, k) (lane = j)
#pragma unroll 4
      for (int k = 0; k < 32; ++k) {
        const float dk = dsh[w][k * 33 + k];
        const bool zero = !(dk > 0.f) || !isfinite(dk);
        const float rkk = sqrtf(dk);
        const float inv = zero ? 0.f : 1.0f / rkk;
        const float dj = dsh[w][k * 33 + lane];
        Rrow[k] = zero ? 0.f : (lane == k ? rkk : (lane > k ? dj * inv : 0.f));
        if (lane == k) rjj = zero ? 0.f : rkk;
      }
    }
    const float inv = rjj > 0.f ? 1.0f / rjj : 0.f;
#pragma unroll
    for (int i = 0; i < BR / 2; ++i) {
      L[w][lane * LD + 2 * i] = x[i].x * inv;
      L[w][lane * LD + 2 * i + 1] = x[i].y * inv;
    }
  }
  __syncwarp();
  long long t1 = clock64();
  float* q = Q + ((long long)blockIdx.x * 4 + w) * BR * 32;
  if (V == 0 || V >= 5) {
    for (int j = 0; j < 32; ++j) q[j * BR + lane] = L[w][j * LD + lane], q[j * BR + lane + 32] = L[w][j * LD + lane + 32];
  } else {
    for (int i = 0; i < BR; ++i) q[lane * BR + i] = L[w][lane * LD + i];
  }
  for (int k = 0; k < 32; ++k) R[((long long)blockIdx.x * 4 + w) * 1024 + k * 32 + lane] = Rrow[k];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// block b: column-major 64 x 32 at A + b * 2048 (column j at + j * 64)
static void metrics(const float* A, const float* Q, const float* R, int nblk, double* orth, double* res) {
  double om = 0, rm = 0;
  for (int b = 0; b < nblk; ++b) {
    const float* a = A + (long long)b * 2048;
    const float* q = Q + (long long)b * 2048;
    const float* r = R + (long long)b * 1024;  // r[k * 32 + j] = R(k, j)
    double o = 0, na = 0, nr = 0;
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 32; ++j) {
        double s = 0;
        for (int t = 0; t < 64; ++t) s += (double)q[i * 64 + t] * q[j * 64 + t];
        s -= (i == j);
        o += s * s;
      }
    for (int j = 0; j < 32; ++j)
      for (int t = 0; t < 64; ++t) {
        double s = 0;
        for (int k = 0; k <= j; ++k) s += (double)q[k * 64 + t] * r[k * 32 + j];
        const double d = a[j * 64 + t] - s;
        nr += d * d;
        na += (double)a[j * 64 + t] * a[j * 64 + t];
      }
    om = fmax(om, sqrt(o / 32));
    rm = fmax(rm, sqrt(nr / na));
  }
  *orth = om;
  *res = rm;
}

int main() {
  const int nblk = 148 * 4, ne = nblk * BR * 32;
  float* hA = (float*)malloc(ne * 4);
  float *A, *Q, *R;
  long long* cyc;
  cudaMalloc(&A, ne * 4);
  cudaMalloc(&Q, ne * 4);
  cudaMalloc(&R, nblk * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  float* out = (float*)malloc(ne * 4);
  float* rout = (float*)malloc(nblk * 1024 * 4);
  for (int graded = 0; graded < 2; ++graded) {
    srand(1);
    for (int b = 0; b < nblk; ++b)
      for (int j = 0; j < 32; ++j)
        for (int t = 0; t < 64; ++t) {
          // graded: column j scaled by 10^(-4 j / 31) and made nearly dependent on column 0
          float v = (float)rand() / RAND_MAX - 0.5f;
          if (graded) v = v * powf(10.f, -4.f * j / 31.f) + (j ? hA[(long long)b * 2048 + t] : 0.f);
          hA[(long long)b * 2048 + j * 64 + t] = v;
        }
    cudaMemcpy(A, hA, ne * 4, cudaMemcpyHostToDevice);
    auto run = [&](auto kern, const char* name) {
      const int smem = 4 * (4 * BR * LD + 4 + 8 * BR + 4 * 32 * 33);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int r = 0; r < 3; ++r) kern<<<148, 128, smem>>>(A, Q, R, cyc);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(out, Q, ne * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(rout, R, nblk * 1024 * 4, cudaMemcpyDeviceToHost);
      double o, r;
      metrics(hA, out, rout, 64, &o, &r);
      printf("%s %-52s %6.1f cycles/step  orth %.2e  resid %.2e  %s\n", graded ? "graded" : "random", name,
             c / 32.0, o, r, cudaGetErrorString(cudaGetLastError()));
    };
    run(bench<0>, "U0 normalized pivot (leaf's current step)");
    run(bench<1>, "U1 projection form, c = d_j / d_k");
    run(bench<2>, "U2 projection form, c = d_j * (1 / d_k)");
    run(bench<3>, "U3 = U2 with R deferred past the loop");
    run(bench<4>, "U4 = U3 with c = d_j * rcp.approx(d_k)");
    run(bench<5>, "U5 = U0 with the Q column stores after the update");
    run(bench<6>, "U6 = U0 without the Q column stores (timing only)");
  }
  return 0;
}

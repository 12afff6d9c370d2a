// Cycles of the 32x32 FP64 Cholesky chain of the leaf kernel (k_leaf.cu (3a)) run by one warp:
// variant 0 = shuffle broadcast of row k, variant 1 = shared-memory broadcast of row k.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void chol(const double* G, double* out, long long* clk, int pw) {
  __shared__ double Rd[32 * 34];
  const int lane = threadIdx.x & 31;
  double c[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = (i <= lane && lane < pw) ? G[i * 32 + lane] : 0.0;
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = G[lane * 32 + j] * 0.5;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < pw) {
      const double d = __shfl_sync(0xffffffffu, c[k], k);
      const bool ok = d > 0.0 && d <= 1.7976931348623157e308;
      const double ri = ok ? rsqrt(d) : 0.0;
      const double rkj = lane == k ? d * ri : (lane > k ? c[k] * ri : 0.0);
      if (V == 0) {
#pragma unroll
        for (int i = k + 1; i < 32; ++i) c[i] = fma(-__shfl_sync(0xffffffffu, rkj, i), rkj, c[i]);
        Rd[k * 34 + lane] = rkj;
      } else if (V == 2) {
        // pivot path by shuffle (lane k+1's own update), the rest through shared memory, plus the
        // S row of lane (forward substitution) interleaved
        const double rk1 = __shfl_sync(0xffffffffu, rkj, (k + 1) & 31);
        if (k + 1 < 32) c[(k + 1) & 31] = fma(-rk1, rkj, c[(k + 1) & 31]);
        Rd[k * 34 + lane] = rkj;
        __syncwarp();
        const double* rk = Rd + k * 34;
        const double sk = r[k] * ri;
        r[k] = sk;
#pragma unroll
        for (int i = k + 2; i < 32; ++i) c[i] = fma(-rk[i], rkj, c[i]);
#pragma unroll
        for (int j = k + 1; j < 32; ++j) r[j] = fma(-sk, rk[j], r[j]);
      } else {
        Rd[k * 34 + lane] = rkj;
        __syncwarp();
        const double* rk = Rd + k * 34;
#pragma unroll
        for (int i = k + 1; i < 32; ++i) c[i] = fma(-rk[i], rkj, c[i]);
      }
    }
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) clk[V] = t1 - t0;
  for (int i = 0; i < 32; ++i) out[i * 32 + lane] = Rd[i * 34 + lane] + c[i] + r[i];
}
// the rolled, shifted form used by k_leaf.cu (3)
__global__ void chol_rolled(const double* G, double* out, long long* clk, int pw) {
  __shared__ double Rd[32 * 34 + 34];
  __shared__ float Sf[32 * 32];
  const int lane = threadIdx.x & 31;
  double c[32], r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = (i <= lane && lane < pw) ? G[i * 32 + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = G[lane * 32 + j] * 0.5;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int k = 0; k < pw; ++k) {
    const double d = __shfl_sync(0xffffffffu, c[0], k);
    const bool ok = d > 0.0 && d <= 1.7976931348623157e308;
    const double ri = ok ? rsqrt(d) : 0.0;
    const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
    Rd[k * 34 + lane] = rkj;
    const double sk = r[0] * ri;
    Sf[lane * 32 + k] = (float)sk;
    __syncwarp();
    const double* rk = Rd + k * 34 + k + 1;
#pragma unroll
    for (int i = 0; i < 31; ++i) {
      const double v = rk[i];
      c[i] = fma(-v, rkj, c[i + 1]);
      r[i] = fma(-sk, v, r[i + 1]);
    }
    c[31] = 0.0;
    r[31] = 0.0;
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) clk[3] = t1 - t0;
  for (int i = 0; i < 32; ++i) out[i * 32 + lane] = Rd[i * 34 + lane] + Sf[lane * 32 + i];
}
int main() {
  double h[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) h[i * 32 + j] = (i == j ? 40.0 : 0.0) + 1.0 / (1 + i + j);
  double *G, *o; long long* c;
  cudaMalloc(&G, 8192); cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
  cudaMemcpy(G, h, 8192, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    chol<0><<<1, 32>>>(G, o, c, 32);
    chol<1><<<1, 32>>>(G, o, c, 32);
    chol<2><<<1, 32>>>(G, o, c, 32);
    chol_rolled<<<1, 32>>>(G, o, c, 32);
  }
  long long hc[4]; cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost);
  printf("rolled shifted: %lld cycles (%.0f/step)\n", hc[3], hc[3] / 32.0);
  printf("fused chol + S rows, pivot by shuffle: %lld cycles (%.0f/step)\n", hc[2], hc[2] / 32.0);
  printf("chol 32x32 one warp: shfl %lld cycles (%.0f/step), smem %lld cycles (%.0f/step)\n", hc[0],
         hc[0] / 32.0, hc[1], hc[1] / 32.0);
  return 0;
}

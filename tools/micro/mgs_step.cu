// Micro-benchmark: cycle breakdown of one CTA-local MGS step variant (development tool).
#include <cstdio>
#include <cuda_runtime.h>

template <int NT, int RPT>
__global__ void mgs_bench(const float* X, int nrows, int w, float* Qout, long long* clk, int variant) {
  __shared__ float red[2][NT / 32][32];
  __shared__ float rbc[NT / 32][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float x[RPT][32];
  for (int r = 0; r < RPT; ++r)
    for (int j = 0; j < 32; ++j) {
      int i = threadIdx.x + r * NT;
      x[r][j] = (i < nrows && j < w) ? X[i + j * nrows] : 0.f;
    }
  int buf = 0;
  long long t[8];
  for (int k = 0; k < w; ++k) {
    const bool rec = (k == 5 && threadIdx.x == 0);
    if (rec) t[0] = clock64();
    float p[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < RPT; ++r) acc = fmaf(x[r][0], x[r][j], acc);
      p[j] = acc;
    }
    if (rec) t[1] = clock64();
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool upper = (lane & s) != 0;
#pragma unroll
      for (int i = 0; i < s; ++i) {
        const float send = upper ? p[i] : p[i + s];
        const float keep = upper ? p[i + s] : p[i];
        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    if (rec) t[2] = clock64();
    red[buf][warp][lane] = p[0];
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int v = 0; v < NT / 32; ++v) tot += red[buf][v][lane];
    buf ^= 1;
    if (rec) t[3] = clock64();
    const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, 0));
    const float rkj = (lane == 0 ? rkk : tot / rkk);
    float q[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) q[r] = x[r][0] / rkk;
    if (rec) t[4] = clock64();
    if (variant == 0) {
#pragma unroll
      for (int j = 1; j < 32; ++j) {
        const float rj = __shfl_sync(0xffffffffu, rkj, j);
#pragma unroll
        for (int r = 0; r < RPT; ++r) x[r][j - 1] = fmaf(-q[r], rj, x[r][j]);
      }
    } else {
      rbc[warp][lane] = rkj;
      __syncwarp();
#pragma unroll
      for (int j4 = 0; j4 < 32; j4 += 4) {
        const float4 rv = *reinterpret_cast<const float4*>(&rbc[warp][j4]);
        const float rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j4 + u;
          if (j >= 1) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) x[r][j - 1] = fmaf(-q[r], rr[u], x[r][j]);
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) x[r][31] = q[r];  // keep data alive
    if (rec) {
      t[5] = clock64();
      for (int i = 0; i < 6; ++i) clk[i] = t[i];
    }
  }
  for (int r = 0; r < RPT; ++r)
    for (int j = 0; j < 32; ++j) Qout[threadIdx.x + r * NT + j * NT * RPT] = x[r][j];
}

template <int NT, int RPT>
void run(int variant) {
  int nrows = NT * RPT, w = 32;
  float *X, *Q;
  long long* clk;
  cudaMalloc(&X, sizeof(float) * nrows * 32);
  cudaMalloc(&Q, sizeof(float) * nrows * 32);
  cudaMalloc(&clk, sizeof(long long) * 8);
  float* h = new float[nrows * 32];
  for (int i = 0; i < nrows * 32; ++i) h[i] = (float)((i * 7919) % 1000) / 1000.f + (i % 33 == 0);
  cudaMemcpy(X, h, sizeof(float) * nrows * 32, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  mgs_bench<NT, RPT><<<1, NT>>>(X, nrows, w, Q, clk, variant);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) mgs_bench<NT, RPT><<<1, NT>>>(X, nrows, w, Q, clk, variant);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c[8];
  cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  printf("NT=%d RPT=%d var=%d: %.2f us/launch (32 steps) | step k=5 cycles: products %lld transpose %lld bar+red %lld sqrt/div %lld update %lld total %lld\n",
         NT, RPT, variant, ms * 100.f, c[1] - c[0], c[2] - c[1], c[3] - c[2], c[4] - c[3], c[5] - c[4], c[5] - c[0]);
}

int main() {
  for (int v = 0; v < 2; ++v) {
    run<128, 2>(v);
    run<160, 2>(v);
    run<256, 1>(v);
    run<64, 4>(v);
    run<32, 8>(v);
  }
  return 0;
}

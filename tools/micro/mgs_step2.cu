// Micro-benchmark v2: width-switched rotating MGS step (active columns shrink with k).
#include <cstdio>
#include <cuda_runtime.h>

__device__ int g_divmode = 0;
// Lane l ends with the warp sum of v[l % W] (all lanes that share l % W hold the same value).
template <int W>
__device__ __forceinline__ float tr_reduce(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = W / 2; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  float r = v[0];
#pragma unroll
  for (int s = W; s < 32; s <<= 1) r += __shfl_xor_sync(0xffffffffu, r, s);
  return r;
}

template <int NT, int RPT, int W>
__device__ __forceinline__ void step(float (&x)[RPT][32], float* red, int& buf, int nrows, float* qs,
                                     int k) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float p[32];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc = fmaf(x[r][0], x[r][j], acc);
    p[j] = acc;
  }
  const float part = tr_reduce<W>(p);
  red[(buf * (NT / 32) + warp) * 32 + lane] = part;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int v = 0; v < NT / 32; ++v) tot += red[(buf * (NT / 32) + v) * 32 + lane];
  buf ^= 1;
  const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, 0));
  const int dm = g_divmode;
  float rkj, q[RPT];
  if (dm == 0) rkj = ((lane & (W - 1)) == 0) ? rkk : tot / rkk;
  else if (dm == 1) { const float inv = __frcp_rn(rkk); rkj = ((lane & (W - 1)) == 0) ? rkk : tot * inv; }
  else { rkj = rkk; if ((lane & (W - 1)) != 0) { rkj = 0.f; if (tot != 0.f) rkj = tot / rkk; } }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    if (dm == 0) q[r] = x[r][0] / rkk;
    else if (dm == 1) q[r] = x[r][0] * __frcp_rn(rkk);
    else { q[r] = 0.f; if (x[r][0] != 0.f) q[r] = x[r][0] / rkk; }
    const int row = threadIdx.x + r * NT;
    if (row < nrows) qs[row * 33 + k] = q[r];
  }
#pragma unroll
  for (int j = 1; j < W; ++j) {
    const float rj = __shfl_sync(0xffffffffu, rkj, j);
#pragma unroll
    for (int r = 0; r < RPT; ++r) x[r][j - 1] = fmaf(-q[r], rj, x[r][j]);
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) x[r][W - 1] = 0.f;
}

template <int NT, int RPT>
__global__ void __launch_bounds__(NT) mgs_bench(const float* X, int nrows, int w, float* Qout,
                                                long long* clk) {
  __shared__ float red[2 * (NT / 32) * 32];
  extern __shared__ float qs[];
  float x[RPT][32];
  for (int r = 0; r < RPT; ++r)
    for (int j = 0; j < 32; ++j) {
      int i = threadIdx.x + r * NT;
      x[r][j] = (i < nrows && j < w) ? X[i + j * nrows] : 0.f;
    }
  int buf = 0;
  long long t0 = clock64();
  for (int k = 0; k < w; ++k) {
    const int act = w - k;
    if (act > 16) step<NT, RPT, 32>(x, red, buf, nrows, qs, k);
    else if (act > 8) step<NT, RPT, 16>(x, red, buf, nrows, qs, k);
    else if (act > 4) step<NT, RPT, 8>(x, red, buf, nrows, qs, k);
    else if (act > 2) step<NT, RPT, 4>(x, red, buf, nrows, qs, k);
    else if (act > 1) step<NT, RPT, 2>(x, red, buf, nrows, qs, k);
    else step<NT, RPT, 1>(x, red, buf, nrows, qs, k);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) clk[0] = t1 - t0;
  __syncthreads();
  for (int r = 0; r < RPT; ++r)
    for (int j = 0; j < 32; ++j) Qout[threadIdx.x + r * NT + j * NT * RPT] = qs[(threadIdx.x + r * NT) * 33 + j];
}

template <int NT, int RPT>
void run(int tri = 0) {
  int nrows = NT * RPT, w = 32;
  float *X, *Q;
  long long* clk;
  cudaMalloc(&X, sizeof(float) * nrows * 32);
  cudaMalloc(&Q, sizeof(float) * nrows * 32);
  cudaMalloc(&clk, sizeof(long long) * 8);
  float* h = new float[nrows * 32];
  for (int i = 0; i < nrows * 32; ++i) h[i] = (float)((i * 7919) % 1000) / 1000.f + (i % 33 == 0);
  if (tri)  // stack of 32x32 upper triangles (rows a > column j are zero)
    for (int j = 0; j < 32; ++j)
      for (int i = 0; i < nrows; ++i) {
        int a = i % 32;
        if (a > j) h[i + j * nrows] = 0.f;
        if (a == j) h[i + j * nrows] += 2.f;
      }
  cudaMemcpy(X, h, sizeof(float) * nrows * 32, cudaMemcpyHostToDevice);
  int smem = NT * RPT * 33 * 4;
  cudaFuncSetAttribute(mgs_bench<NT, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mgs_bench<NT, RPT><<<1, NT, smem>>>(X, nrows, w, Q, clk);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) mgs_bench<NT, RPT><<<1, NT, smem>>>(X, nrows, w, Q, clk);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  // check orthogonality of Q roughly
  float* q = new float[nrows * 32];
  cudaMemcpy(q, Q, sizeof(float) * nrows * 32, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int a1 = 0; a1 < 32; ++a1)
    for (int b1 = 0; b1 < 32; ++b1) {
      double s = 0;
      for (int i = 0; i < nrows; ++i) s += (double)q[i + a1 * nrows] * q[i + b1 * nrows];
      double e = fabs(s - (a1 == b1));
      if (e > worst) worst = e;
    }
  printf("v2 tri=%d NT=%d RPT=%d rows=%d: %.2f us/launch, 32 steps = %lld cycles (%.0f/step), max|QtQ-I|=%.2e\n",
         tri, NT, RPT, nrows, ms * 100.f, c, c / 32.0, worst);
}

int main() {
  for (int dm = 0; dm < 3; ++dm) {
    cudaMemcpyToSymbol(g_divmode, &dm, sizeof(int));
    printf("divmode %d\n", dm);
    for (int t = 0; t < 2; ++t) {
      run<128, 2>(t);
      run<256, 4>(t);
    }
  }
  return 0;
}

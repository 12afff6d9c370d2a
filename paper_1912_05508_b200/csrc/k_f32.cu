// k_f32.cu -- K2b: FP32 products of the recursion below the tensor-core cutoff (reading R-A1:
// the leaf panelQR is single precision, so Alg. 2 lines 8-9 run in FP32 for
// nodes with w <= cutoff).  Deterministic split-K for R12 = Q1' A2; a row-parallel update.
#include "common.cuh"
#include "kernels.h"

namespace tcqr {

constexpr int kF32Chunk = 32;

// P_s (h x w2, ld h) = sum over rows [r0_s, r1_s) of Q1(r, :)' A2(r, :).  h, w2 <= 64.
__global__ void __launch_bounds__(256) f32_tn_kernel(int m, int h, int w2,
                                                     const float* __restrict__ Q1, long long ldq,
                                                     const float* __restrict__ A2, long long lda,
                                                     float* __restrict__ P, int splits) {
  __shared__ float Qs[kF32Chunk][65];
  __shared__ float As[kF32Chunk][65];
  const int s = blockIdx.x;
  const long long r0 = (long long)s * m / splits, r1 = (long long)(s + 1) * m / splits;
  const int tid = threadIdx.x, ti = tid & 15, tj = tid >> 4;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (long long c0 = r0; c0 < r1; c0 += kF32Chunk) {
    __syncthreads();
    for (int e = tid; e < kF32Chunk * 64; e += 256) {
      const int rr = e & (kF32Chunk - 1), cc = e / kF32Chunk;
      const long long row = c0 + rr;
      const bool rok = row < r1;
      Qs[rr][cc] = (rok && cc < h) ? Q1[row + cc * ldq] : 0.f;
      As[rr][cc] = (rok && cc < w2) ? A2[row + cc * lda] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < kF32Chunk; ++rr) {
      float qv[4], av[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) qv[a] = Qs[rr][ti * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) av[b] = As[rr][tj * 4 + b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(qv[a], av[b], acc[a][b]);
    }
  }
  float* out = P + (long long)s * h * w2;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ti * 4 + a, j = tj * 4 + b;
      if (i < h && j < w2) out[i + (long long)j * h] = acc[a][b];
    }
}

__global__ void f32_reduce_kernel(const float* __restrict__ P, int splits, int hw,
                                  float* __restrict__ T) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < hw; e += gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < splits; ++s) acc += P[(long long)s * hw + e];
    T[e] = acc;
  }
}

cudaError_t f32_tn(int m, int h, int w2, const float* Q1, long long ldq, const float* A2,
                   long long lda, float* T, float* P, long long p_cap, int num_sms,
                   cudaStream_t st) {
  if (h > 64 || w2 > 64) return cudaErrorInvalidValue;
  const int hw = h * w2;
  int splits = (m + 255) / 256;
  if (splits > 2 * num_sms) splits = 2 * num_sms;
  if ((long long)splits * hw > p_cap) splits = (int)(p_cap / hw);
  if (splits < 1) splits = 1;
  if (splits == 1) {
    f32_tn_kernel<<<1, 256, 0, st>>>(m, h, w2, Q1, ldq, A2, lda, T, 1);
    return cudaGetLastError();
  }
  f32_tn_kernel<<<splits, 256, 0, st>>>(m, h, w2, Q1, ldq, A2, lda, P, splits);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  f32_reduce_kernel<<<(hw + 255) / 256, 256, 0, st>>>(P, splits, hw, T);
  return cudaGetLastError();
}

// A2 (m x w2) -= Q1 (m x h) T (h x w2, ld h).  grid (row blocks of 256, column groups of 16).
__global__ void __launch_bounds__(256) f32_nn_kernel(int m, int h, int w2,
                                                     const float* __restrict__ Q1, long long ldq,
                                                     const float* __restrict__ T,
                                                     float* __restrict__ A2, long long lda) {
  __shared__ float Ts[64][16];
  const int j0 = blockIdx.y * 16;
  for (int e = threadIdx.x; e < h * 16; e += 256) {
    const int i = e / 16, jj = e % 16;
    Ts[i][jj] = (j0 + jj < w2) ? T[i + (long long)(j0 + jj) * h] : 0.f;
  }
  __syncthreads();
  const long long row = (long long)blockIdx.x * 256 + threadIdx.x;
  if (row >= m) return;
  float acc[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) acc[jj] = 0.f;
  for (int i = 0; i < h; ++i) {
    const float q = Q1[row + (long long)i * ldq];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) acc[jj] = fmaf(q, Ts[i][jj], acc[jj]);
  }
#pragma unroll
  for (int jj = 0; jj < 16; ++jj)
    if (j0 + jj < w2) {
      float* p = A2 + row + (long long)(j0 + jj) * lda;
      *p = *p - acc[jj];
    }
}

cudaError_t f32_nn_update(int m, int h, int w2, const float* Q1, long long ldq, const float* T,
                          float* A2, long long lda, cudaStream_t st) {
  if (h > 64) return cudaErrorInvalidValue;
  dim3 grid((m + 255) / 256, (w2 + 15) / 16);
  f32_nn_kernel<<<grid, 256, 0, st>>>(m, h, w2, Q1, ldq, T, A2, lda);
  return cudaGetLastError();
}

}  // namespace tcqr

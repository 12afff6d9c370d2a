// k_cgls.cu -- K5/K6/K7: the R-preconditioned CGLS of Alg. 5, corrected per
// DESIGN.md reading R-A10, all vector arithmetic in FP64 (reading R-A13), A read as FP32 data
// (reading R-A14).
//
//   K5  q = A t and v = A' r: FP32 A streamed once per product, FP64 accumulation, deterministic
//       (fixed-order partial sums; one warp per column for A').
//   K6  inv(R)*p and inv(R')*v (Alg. 5 lines 12, 18): R is applied through its explicit inverse
//       M = inv(R), computed once in FP64 (block recursion X12 = -X11 R12 X22) and stored FP64;
//       per iteration t = M p and s = M' v are fully parallel triangular GEMVs (reading R-A13:
//       R is a fixed preconditioner, any consistent application is valid; Alg. 5 itself writes
//       inv(R)).
//   K7  scalar recurrences, stop/restart bookkeeping and the best-iterate copy, on the device, so
//       the host only polls a done flag.
#include "common.cuh"
#include "kernels.h"
#include <algorithm>

#include "cgls_state.h"

namespace tcqr {

// ------------------------------------------------------------------------------------------
// Explicit inverse of an upper-triangular FP32 R, in FP64.
// ------------------------------------------------------------------------------------------
constexpr int kInvBlk = 32;

// One CTA per diagonal block: M_dd = inv(R_dd) by column-wise back substitution in FP64.
__global__ void __launch_bounds__(kInvBlk) trinv_diag_kernel(int n, const float* __restrict__ R,
                                                             long long ldr, double* __restrict__ M,
                                                             long long ldm) {
  __shared__ double Rs[kInvBlk][kInvBlk + 1];
  __shared__ double Xs[kInvBlk][kInvBlk + 1];
  const int d0 = blockIdx.x * kInvBlk;
  const int bs = min(kInvBlk, n - d0);
  for (int e = threadIdx.x; e < kInvBlk * kInvBlk; e += blockDim.x) {
    const int i = e % kInvBlk, j = e / kInvBlk;
    Rs[i][j] = (i < bs && j < bs && i <= j) ? (double)R[(d0 + i) + (long long)(d0 + j) * ldr] : 0.0;
  }
  __syncthreads();
  const int j = threadIdx.x;  // column of the inverse
  if (j < bs) {
    for (int i = kInvBlk - 1; i >= 0; --i) {
      double acc = (i == j) ? 1.0 : 0.0;
      if (i <= j) {
        for (int k = i + 1; k <= j; ++k) acc -= Rs[i][k] * Xs[k][j];
        Xs[i][j] = acc / Rs[i][i];
      } else {
        Xs[i][j] = 0.0;
      }
    }
    for (int i = 0; i <= j; ++i) M[(d0 + i) + (long long)(d0 + j) * ldm] = Xs[i][j];
  }
}

// Batched FP64 GEMM for the inverse recursion: for pair p (rows i0 = p*2b):
//   mode 0: W_p (b1 x b2) = R[i0:i0+b1, i0+b1:i0+b1+b2] * M[i0+b1:.., i0+b1:..]   (R12 * X22)
//   mode 1: M[i0:i0+b1, i0+b1:..] = -M[i0:i0+b1, i0:i0+b1] * W_p                    (-X11 * W)
// 64x64 output tile per CTA, 256 threads x (4x4), K-chunks of 16.
__global__ void __launch_bounds__(256) trinv_pair_gemm_kernel(int n, int b, int mode,
                                                              const float* __restrict__ R,
                                                              long long ldr, double* __restrict__ M,
                                                              long long ldm,
                                                              double* __restrict__ W) {
  __shared__ double As[16][64 + 1];
  __shared__ double Bs[16][64 + 1];
  const int p = blockIdx.z;
  const int i0 = p * 2 * b;
  const int b1 = b;
  const int b2 = min(b, n - (i0 + b));
  if (b2 <= 0) return;
  const int tm = blockIdx.x * 64, tn = blockIdx.y * 64;
  if (tm >= b1 || tn >= b2) return;
  const int K = (mode == 0) ? b2 : b1;
  double* Wp = W + (long long)p * b * b;  // ld = b
  const int tid = threadIdx.x, ti = tid & 15, tj = tid >> 4;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    __syncthreads();
    for (int e = tid; e < 16 * 64; e += 256) {
      const int kk = e / 64, mm = e % 64;  // A element (row tm+mm, k k0+kk)
      const int r = tm + mm, k = k0 + kk;
      double av = 0.0;
      if (r < b1 && k < K) {
        if (mode == 0)
          av = (double)R[(i0 + r) + (long long)(i0 + b1 + k) * ldr];
        else
          av = M[(i0 + r) + (long long)(i0 + k) * ldm];
      }
      As[kk][mm] = av;
      const int c = tn + mm;  // B element (k k0+kk, col tn+mm)
      double bv = 0.0;
      if (c < b2 && k < K) {
        if (mode == 0)
          bv = M[(i0 + b1 + k) + (long long)(i0 + b1 + c) * ldm];
        else
          bv = Wp[k + (long long)c * b];
      }
      Bs[kk][mm] = bv;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], bb[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[kk][ti * 4 + x];
#pragma unroll
      for (int y = 0; y < 4; ++y) bb[y] = Bs[kk][tj * 4 + y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], bb[y], acc[x][y]);
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int r = tm + ti * 4 + x, c = tn + tj * 4 + y;
      if (r < b1 && c < b2) {
        if (mode == 0)
          Wp[r + (long long)c * b] = acc[x][y];
        else
          M[(i0 + r) + (long long)(i0 + b1 + c) * ldm] = -acc[x][y];
      }
    }
}

// Large-tile FP64 pair GEMM (b >= 128): 128 x 128 output tile per CTA, 256 threads with 8 x 8
// register micro-tiles, K-chunks of 16 staged through shared memory with a register prefetch of
// the next chunk; the triangular factor's zero blocks are skipped (mode 0: k < (J+1)*128,
// mode 1: k >= I*128).
template <int MODE>
__global__ void __launch_bounds__(256, 1) trinv_pair_gemm_big(int n, int b,
                                                              const float* __restrict__ R,
                                                              long long ldr,
                                                              double* __restrict__ M,
                                                              long long ldm,
                                                              double* __restrict__ W) {
  constexpr int TB = 128, KB = 8, NLD = KB * TB / 256;
  __shared__ __align__(16) double As[2][KB][TB];
  __shared__ __align__(16) double Bs[2][KB][TB];
  const int p = blockIdx.z;
  const int i0 = p * 2 * b;
  const int b1 = b;
  const int b2 = min(b, n - (i0 + b));
  if (b2 <= 0) return;
  const int tm = blockIdx.x * TB, tn = blockIdx.y * TB;
  if (tm >= b1 || tn >= b2) return;
  double* Wp = W + (long long)p * b * b;  // ld = b
  const int K = (MODE == 0) ? b2 : b1;
  const int kbeg = (MODE == 0) ? 0 : tm;
  const int kend = (MODE == 0) ? min(K, tn + TB) : K;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;  // rows tx*8.., cols ty*8..
  // loader mapping: KB x 128 tile, NLD doubles per thread: kk = e >> 7, mm = e & 127
  auto loadA = [&](int k0, double (&ra)[NLD]) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      const int r = tm + mm, k = k0 + kk;
      double v = 0.0;
      if (r < b1 && k < kend) {
        if (MODE == 0)
          v = (double)__ldg(R + (i0 + r) + (long long)(i0 + b1 + k) * ldr);
        else
          v = M[(i0 + r) + (long long)(i0 + k) * ldm];
      }
      ra[u] = v;
    }
  };
  auto loadB = [&](int k0, double (&rb)[NLD]) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      const int c = tn + mm, k = k0 + kk;
      double v = 0.0;
      if (c < b2 && k < kend) {
        if (MODE == 0)
          v = M[(i0 + b1 + k) + (long long)(i0 + b1 + c) * ldm];
        else
          v = Wp[k + (long long)c * b];
      }
      rb[u] = v;
    }
  };
  double acc[8][8];
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) acc[x][y] = 0.0;
  double ra[NLD], rb[NLD];
  int buf = 0;
  loadA(kbeg, ra);
  loadB(kbeg, rb);
  for (int k0 = kbeg; k0 < kend; k0 += KB) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      As[buf][kk][mm] = ra[u];
      Bs[buf][kk][mm] = rb[u];
    }
    __syncthreads();
    if (k0 + KB < kend) {
      loadA(k0 + KB, ra);
      loadB(k0 + KB, rb);
    }
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      double a[8], bb[8];
#pragma unroll
      for (int x = 0; x < 8; x += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&As[buf][kk][tx * 8 + x]);
        a[x] = v.x;
        a[x + 1] = v.y;
      }
#pragma unroll
      for (int y = 0; y < 8; y += 2) {
        const double2 v = *reinterpret_cast<const double2*>(&Bs[buf][kk][ty * 8 + y]);
        bb[y] = v.x;
        bb[y + 1] = v.y;
      }
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fma(a[x], bb[y], acc[x][y]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int r = tm + tx * 8 + x, c = tn + ty * 8 + y;
      if (r < b1 && c < b2) {
        if (MODE == 0)
          Wp[r + (long long)c * b] = acc[x][y];
        else
          M[(i0 + r) + (long long)(i0 + b1 + c) * ldm] = -acc[x][y];
      }
    }
}

// FP64 tensor-core pair GEMM (b >= 128): the same 128 x 128 tiles, K-ranges and loaders as
// trinv_pair_gemm_big, with the products on DMMA (mma.sync m8n8k4 f64): 8 warps as 4 (M) x 2
// (N), warp tile 32 x 64 = 4 x 8 m8n8 tiles.  Shared rows padded to 136 doubles, so a fragment
// load (4 k-rows x 8 consecutive m) takes the two wavefronts its 256 bytes need.
__device__ __forceinline__ void dmma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) trinv_pair_dmma(int n, int b, const float* __restrict__ R,
                                                          long long ldr, double* __restrict__ M,
                                                          long long ldm, double* __restrict__ W) {
  constexpr int TB = 128, KB = 8, NLD = KB * TB / 256, SP = 136;
  __shared__ __align__(16) double As[2][KB][SP];
  __shared__ __align__(16) double Bs[2][KB][SP];
  const int p = blockIdx.z;
  const int i0 = p * 2 * b;
  const int b1 = b;
  const int b2 = min(b, n - (i0 + b));
  if (b2 <= 0) return;
  // MODE 0's K range grows with the tile column (X22 is upper triangular): take the long tiles
  // first so the short ones fill the tail wave (MODE 1's already come first: K shrinks with tm)
  const int tm = blockIdx.x * TB;
  const int tn = (MODE == 0 ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y) * TB;
  if (tm >= b1 || tn >= b2) return;
  double* Wp = W + (long long)p * b * b;  // ld = b
  const int K = (MODE == 0) ? b2 : b1;
  const int kbeg = (MODE == 0) ? 0 : tm;
  const int kend = (MODE == 0) ? min(K, tn + TB) : K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 64;
  auto loadA = [&](int k0, double (&ra)[NLD]) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      const int r = tm + mm, k = k0 + kk;
      double v = 0.0;
      if (r < b1 && k < kend) {
        if (MODE == 0)
          v = (double)__ldg(R + (i0 + r) + (long long)(i0 + b1 + k) * ldr);
        else
          v = M[(i0 + r) + (long long)(i0 + k) * ldm];
      }
      ra[u] = v;
    }
  };
  auto loadB = [&](int k0, double (&rb)[NLD]) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      const int c = tn + mm, k = k0 + kk;
      double v = 0.0;
      if (c < b2 && k < kend) {
        if (MODE == 0)
          v = M[(i0 + b1 + k) + (long long)(i0 + b1 + c) * ldm];
        else
          v = Wp[k + (long long)c * b];
      }
      rb[u] = v;
    }
  };
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[NLD], rb[NLD];
  int buf = 0;
  loadA(kbeg, ra);
  loadB(kbeg, rb);
  const int fk = lane & 3, fr = lane >> 2;  // fragment k index, row/col within an 8-block
  for (int k0 = kbeg; k0 < kend; k0 += KB) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      As[buf][kk][mm] = ra[u];
      Bs[buf][kk][mm] = rb[u];
    }
    __syncthreads();
    if (k0 + KB < kend) {
      loadA(k0 + KB, ra);
      loadB(k0 + KB, rb);
    }
#pragma unroll
    for (int k4 = 0; k4 < KB; k4 += 4) {
      double af[4], bf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][k4 + fk][wm + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 8; ++j) bf[j] = Bs[buf][k4 + fk][wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_m8n8k4(acc[i][j], af[i], bf[j]);
    }
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = tm + wm + 8 * i + fr, c = tn + wn + 8 * j + 2 * fk + h;
        if (r < b1 && c < b2) {
          if (MODE == 0)
            Wp[r + (long long)c * b] = acc[i][j][h];
          else
            M[(i0 + r) + (long long)(i0 + b1 + c) * ldm] = -acc[i][j][h];
        }
      }
}

cudaError_t trinv_f64(int n, const float* R, long long ldr, double* M, long long ldm, double* W,
                      int num_sms, cudaStream_t st) {
  (void)num_sms;
  cudaError_t e = cudaMemsetAsync(M, 0, sizeof(double) * (size_t)ldm * n, st);
  if (e != cudaSuccess) return e;
  const int nblk = (n + kInvBlk - 1) / kInvBlk;
  trinv_diag_kernel<<<nblk, kInvBlk, 0, st>>>(n, R, ldr, M, ldm);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  for (int b = kInvBlk; b < n; b *= 2) {
    const int pairs = (n + 2 * b - 1) / (2 * b);
    if (b >= 128) {
      dim3 grid((b + 127) / 128, (b + 127) / 128, pairs);
      trinv_pair_dmma<0><<<grid, 256, 0, st>>>(n, b, R, ldr, M, ldm, W);
      trinv_pair_dmma<1><<<grid, 256, 0, st>>>(n, b, R, ldr, M, ldm, W);
    } else {
      dim3 grid((b + 63) / 64, (b + 63) / 64, pairs);
      trinv_pair_gemm_kernel<<<grid, 256, 0, st>>>(n, b, 0, R, ldr, M, ldm, W);
      trinv_pair_gemm_kernel<<<grid, 256, 0, st>>>(n, b, 1, R, ldr, M, ldm, W);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------------------------------
// Dense FP32 GEMVs with FP64 accumulation (K5)
// ------------------------------------------------------------------------------------------
constexpr int kGvRows = 256;  // rows per CTA (one per thread)
constexpr int kGvCols = 512;  // columns per CTA chunk (partials: m x n/512 doubles)

// part[cb][i] = sum_{j in chunk cb} A[i, j] v[j]    (grid: row blocks x column chunks); eight
// column loads in flight per thread, four FP64 accumulators (fixed order)
__global__ void __launch_bounds__(kGvRows) gemv_n_part_kernel(int m, int n,
                                                              const float* __restrict__ A,
                                                              long long lda,
                                                              const double* __restrict__ v,
                                                              double* __restrict__ part,
                                                              const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double vs[kGvCols];
  const int cb = blockIdx.y;
  const int j0 = cb * kGvCols;
  const int nc = min(kGvCols, n - j0);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) vs[j] = v[j0 + j];
  __syncthreads();
  const long long i = (long long)blockIdx.x * kGvRows + threadIdx.x;
  if (i >= m) return;
  const float* a = A + i + (long long)j0 * lda;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int j = 0;
  for (; j + 8 <= nc; j += 8) {
    float av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldg(a + (long long)(j + u) * lda);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u & 3] = fma((double)av[u], vs[j + u], acc[u & 3]);
  }
  for (; j < nc; ++j) acc[0] = fma((double)a[(long long)j * lda], vs[j], acc[0]);
  part[(long long)cb * m + i] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// y[i] = sum_cb part[cb][i] (fixed order); optional: dpart[block] = sum of y^2 over the block,
// and y2[i] = base[i] - y[i] (residual form).
__global__ void __launch_bounds__(256) gemv_n_reduce_kernel(int m, int nchunks,
                                                            const double* __restrict__ part,
                                                            double* __restrict__ y,
                                                            double* __restrict__ dpart,
                                                            const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double red[8];
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  double acc = 0.0;
  if (i < m) {
    for (int c = 0; c < nchunks; ++c) acc += part[(long long)c * m + i];
    y[i] = acc;
  }
  if (dpart) {
    double sq = warp_sum_d(acc * acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      dpart[blockIdx.x] = t;
    }
  }
}

// y[j] = sum_i A[i, j] v[i], column-blocked: a CTA takes 64 columns (8 per warp) of one row split;
// v is staged in shared memory 1024 rows at a time and each of its values feeds the warp's 8
// columns from registers (one warp per column re-read v from L2 once per column: 2x the bytes of
// A).  Lanes read A down the columns in 16-byte pieces; FP64 accumulation; per-split partials
// part[s * n + j] summed in split order by gemv_t_reduce_kernel (deterministic).
// CGLS form (q != null): the staged values are r - alpha q (alpha = gamma / delta, Alg. 5 line 17
// fused into the A' r pass), written to r_out by the CTAs of column block 0.
constexpr int kGtCols = 64;
constexpr int kGtChunk = 1024;

__global__ void __launch_bounds__(256) gemv_t_part_kernel(int m, int n, const float* __restrict__ A,
                                                          long long lda, const double* __restrict__ v,
                                                          const double* __restrict__ q,
                                                          const CgState* __restrict__ st,
                                                          double* __restrict__ v_out, int rps,
                                                          double* __restrict__ part,
                                                          const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ __align__(16) double vs[kGtChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * kGtCols + warp * 8;
  const long long r_begin = (long long)blockIdx.y * rps;
  const long long r_end = min((long long)m, r_begin + rps);
  const double alpha = q ? st->gamma / st->delta : 0.0;
  const bool vec = ((lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.0;
  for (long long c = r_begin; c < r_end; c += kGtChunk) {
    const int cn = (int)min((long long)kGtChunk, r_end - c);
    __syncthreads();
    for (int i = threadIdx.x; i < cn; i += 256) {
      double x = v[c + i];
      if (q) {
        x = fma(-alpha, q[c + i], x);
        if (blockIdx.x == 0) v_out[c + i] = x;
      }
      vs[i] = x;
    }
    __syncthreads();
    if (vec && cn == kGtChunk && j0 + 8 <= n) {
      // the warp's 8 columns all exist: unpredicated loads (a predicate per load measured 1.4x
      // slower in the persistent variant of this kernel)
      const float* a0 = A + (long long)j0 * lda + c;
#pragma unroll 2
      for (int i = lane * 4; i < kGtChunk; i += 128) {
        const double2 v01 = *reinterpret_cast<const double2*>(vs + i);
        const double2 v23 = *reinterpret_cast<const double2*>(vs + i + 2);
        float4 a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(a0 + (long long)u * lda + i));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc[u] = fma((double)a[u].x, v01.x, acc[u]);
          acc[u] = fma((double)a[u].y, v01.y, acc[u]);
          acc[u] = fma((double)a[u].z, v23.x, acc[u]);
          acc[u] = fma((double)a[u].w, v23.y, acc[u]);
        }
      }
    } else {
      for (int i = lane; i < cn; i += 32) {
        const double x = vs[i];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (j0 + u < n) acc[u] = fma((double)A[(long long)(j0 + u) * lda + c + i], x, acc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double sum = warp_sum_d(acc[u]);
    if (lane == 0 && j0 + u < n) part[(long long)blockIdx.y * n + j0 + u] = sum;
  }
}

__global__ void gemv_t_reduce_kernel(int n, int splits, const double* __restrict__ part,
                                     double* __restrict__ y, const int* __restrict__ done) {
  if (done && *done) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = part[j];
  for (int s = 1; s < splits; ++s) acc += part[(long long)s * n + j];
  y[j] = acc;
}

// Row splits of the A' v kernel: whole 1024-row chunks, enough CTAs for about 14 per SM (many
// short CTAs balance across the SMs: at configs[3] 16 splits of 2048 rows take 205 us per pass,
// 4 splits 223 us -- the 3-CTA-per-SM residency left a tail wave; tools/micro/gemv_bench.cu).
static void gemv_t_plan(int m, int n, int* splits, int* rps) {
  const int cblocks = (n + kGtCols - 1) / kGtCols;
  int s = (14 * 148 + cblocks - 1) / cblocks;
  const int chunks = (m + kGtChunk - 1) / kGtChunk;
  s = std::max(1, std::min(s, chunks));
  const int cps = (chunks + s - 1) / s;
  *rps = cps * kGtChunk;
  *splits = (m + *rps - 1) / *rps;
}

int cg_gemv_t_part_count(int m, int n) {
  int s, rps;
  gemv_t_plan(m, n, &s, &rps);
  return s * n;
}

cudaError_t gemv_f32_n(int m, int n, const float* A, long long lda, const double* v, double* y,
                       double* part, long long part_cap, cudaStream_t st) {
  const int nch = (n + kGvCols - 1) / kGvCols;
  if ((long long)nch * m > part_cap) return cudaErrorInvalidValue;
  dim3 g1((m + kGvRows - 1) / kGvRows, nch);
  gemv_n_part_kernel<<<g1, kGvRows, 0, st>>>(m, n, A, lda, v, part, nullptr);
  gemv_n_reduce_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, nch, part, y, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t gemv_f32_t(int m, int n, const float* A, long long lda, const double* v, double* y,
                       double* part, cudaStream_t st) {
  int splits, rps;
  gemv_t_plan(m, n, &splits, &rps);
  gemv_t_part_kernel<<<dim3((n + kGtCols - 1) / kGtCols, splits), 256, 0, st>>>(
      m, n, A, lda, v, nullptr, nullptr, nullptr, rps, part, nullptr);
  gemv_t_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, splits, part, y, nullptr);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// Triangular (upper) FP64 GEMVs with the explicit inverse M (K6)
// ------------------------------------------------------------------------------------------
constexpr int kTriBlk = 256;

// part[cb][i] = sum_{j in chunk cb, j >= i} M[i, j] p[j], only for chunks cb >= row block.
template <typename TM>
__global__ void __launch_bounds__(kTriBlk) tri_n_part_kernel(int n, const TM* __restrict__ M,
                                                             long long ldm,
                                                             const double* __restrict__ p,
                                                             double* __restrict__ part,
                                                             const int* __restrict__ done) {
  if (done && *done) return;
  // compact grid over the upper block triangle only (no CTAs that exit at once): block p ->
  // (rb, cb), cb >= rb, row-major over the triangle
  const int nch = (n + kTriBlk - 1) / kTriBlk;
  int rb = 0, rest = blockIdx.x;
  while (rest >= nch - rb) {
    rest -= nch - rb;
    ++rb;
  }
  const int cb = rb + rest;
  __shared__ double ps[kTriBlk];
  const int j0 = cb * kTriBlk;
  const int nc = min(kTriBlk, n - j0);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) ps[j] = p[j0 + j];
  __syncthreads();
  const int i = rb * kTriBlk + threadIdx.x;
  if (i >= n) return;
  const TM* mm = M + i + (long long)j0 * ldm;
  // 8 loads in flight per thread (with 2 the kernel ran at 3.5 TB/s)
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  int j = 0;
  for (; j + 8 <= nc; j += 8) {
    TM mv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) mv[u] = __ldg(mm + (long long)(j + u) * ldm);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u & 3] = fma((double)mv[u], ps[j + u], acc[u & 3]);
  }
  for (; j < nc; ++j) acc[0] = fma((double)mm[(long long)j * ldm], ps[j], acc[0]);
  part[(long long)cb * n + i] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// The FP32 M with 16-byte row quads (n, ldm multiples of 4, M 16-byte aligned): the same blocks
// and partials, thread = (row quad q, column slice cs): rows 4q..4q+3 of the block over the
// slice's 64 columns, one 16-byte load per column (8 in flight: 128 bytes per thread, where one
// 4-byte row per thread kept too few bytes in flight for HBM), the four slices added in order
// through shared memory.
__global__ void __launch_bounds__(kTriBlk) tri_n_part_f32v_kernel(int n, const float* __restrict__ M,
                                                                  long long ldm,
                                                                  const double* __restrict__ p,
                                                                  double* __restrict__ part,
                                                                  const int* __restrict__ done) {
  if (done && *done) return;
  const int nch = (n + kTriBlk - 1) / kTriBlk;
  int rb = 0, rest = blockIdx.x;
  while (rest >= nch - rb) {
    rest -= nch - rb;
    ++rb;
  }
  const int cb = rb + rest;
  __shared__ double ps[kTriBlk];
  __shared__ double sl[3][kTriBlk];
  const int j0 = cb * kTriBlk;
  const int nc = min(kTriBlk, n - j0);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) ps[j] = p[j0 + j];
  __syncthreads();
  const int q = threadIdx.x & 63, cs = threadIdx.x >> 6;
  const int i0 = rb * kTriBlk + 4 * q;  // n % 4 == 0: the quad is entirely in or out
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int js = cs * 64, je = min(nc, js + 64);
  if (i0 < n) {
    const float* mm = M + i0 + (long long)j0 * ldm;
    int j = js;
    for (; j + 8 <= je; j += 8) {
      float4 mv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        mv[u] = __ldg(reinterpret_cast<const float4*>(mm + (long long)(j + u) * ldm));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double pj = ps[j + u];
        acc[0] = fma((double)mv[u].x, pj, acc[0]);
        acc[1] = fma((double)mv[u].y, pj, acc[1]);
        acc[2] = fma((double)mv[u].z, pj, acc[2]);
        acc[3] = fma((double)mv[u].w, pj, acc[3]);
      }
    }
    for (; j < je; ++j) {
      const float4 mv = __ldg(reinterpret_cast<const float4*>(mm + (long long)j * ldm));
      const double pj = ps[j];
      acc[0] = fma((double)mv.x, pj, acc[0]);
      acc[1] = fma((double)mv.y, pj, acc[1]);
      acc[2] = fma((double)mv.z, pj, acc[2]);
      acc[3] = fma((double)mv.w, pj, acc[3]);
    }
  }
  if (cs > 0)
#pragma unroll
    for (int r = 0; r < 4; ++r) sl[cs - 1][4 * q + r] = acc[r];
  __syncthreads();
  if (cs == 0 && i0 < n)
#pragma unroll
    for (int r = 0; r < 4; ++r)
      part[(long long)cb * n + i0 + r] = ((acc[r] + sl[0][4 * q + r]) + sl[1][4 * q + r]) + sl[2][4 * q + r];
}

__global__ void tri_n_reduce_kernel(int n, int nch, const double* __restrict__ part,
                                    double* __restrict__ t, const int* __restrict__ done) {
  if (done && *done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc = 0.0;
  for (int c = i / kTriBlk; c < nch; ++c) acc += part[(long long)c * n + i];
  t[i] = acc;
}

// s[j] = sum_{i <= j} M[i, j] v[i]: one warp per column.
__global__ void __launch_bounds__(256) tri_t_kernel(int n, const double* __restrict__ M,
                                                    long long ldm, const double* __restrict__ v,
                                                    double* __restrict__ s,
                                                    const int* __restrict__ done) {
  if (done && *done) return;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double* mm = M + (long long)j * ldm;
  double a0 = 0.0, a1 = 0.0;
  int i = 0;
  // rows [0, j]: 16-byte loads, four in flight per lane (256 rows per warp step) when M's
  // columns are 16-byte aligned
  if ((ldm & 1) == 0 && (reinterpret_cast<uintptr_t>(M) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    const int j256 = ((j + 1) / 256) * 256;
    for (; i < j256; i += 256) {
      double2 mv[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mv[u] = __ldg(reinterpret_cast<const double2*>(mm + i + 64 * u + 2 * lane));
        vv[u] = *reinterpret_cast<const double2*>(v + i + 64 * u + 2 * lane);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(mv[u].x, vv[u].x, a0);
        a1 = fma(mv[u].y, vv[u].y, a1);
      }
    }
  }
  for (i += lane; i <= j; i += 32) a0 = fma(mm[i], v[i], a0);
  const double r = warp_sum_d(a0 + a1);
  if (lane == 0) s[j] = r;
}

// The same with M stored in FP32 (the CGLS preconditioner, reading R-A13): 16-byte loads of four
// rows, two in flight per lane (256 rows per warp step).
__global__ void __launch_bounds__(256) tri_t_f32_kernel(int n, const float* __restrict__ M,
                                                        long long ldm, const double* __restrict__ v,
                                                        double* __restrict__ s,
                                                        const int* __restrict__ done) {
  if (done && *done) return;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const float* mm = M + (long long)j * ldm;
  double a0 = 0.0, a1 = 0.0;
  int i = 0;
  if ((ldm & 3) == 0 && (reinterpret_cast<uintptr_t>(M) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(v) & 15) == 0) {
    const int j256 = ((j + 1) / 256) * 256;
    for (; i < j256; i += 256) {
      float4 mv[2];
      double2 vv[4];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        mv[u] = __ldg(reinterpret_cast<const float4*>(mm + i + 128 * u + 4 * lane));
        vv[2 * u] = *reinterpret_cast<const double2*>(v + i + 128 * u + 4 * lane);
        vv[2 * u + 1] = *reinterpret_cast<const double2*>(v + i + 128 * u + 4 * lane + 2);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        a0 = fma((double)mv[u].x, vv[2 * u].x, a0);
        a1 = fma((double)mv[u].y, vv[2 * u].y, a1);
        a0 = fma((double)mv[u].z, vv[2 * u + 1].x, a0);
        a1 = fma((double)mv[u].w, vv[2 * u + 1].y, a1);
      }
    }
  }
  for (i += lane; i <= j; i += 32) a0 = fma((double)mm[i], v[i], a0);
  const double r = warp_sum_d(a0 + a1);
  if (lane == 0) s[j] = r;
}

// s = M' v with the FP32 upper-triangular M (zero below the diagonal), column-blocked like
// gemv_t_part_kernel: CTA (column block of 64, row chunk c of 1024) -- chunks entirely below the
// block's last column's diagonal only) -- v staged in shared memory, each value feeding the warp's
// 8 columns; part[c * n + j] summed over c in order by tri_t_reduce_kernel.  (One warp per column
// re-read v from L2 once per column: twice the bytes of M.)
constexpr int kTtChunk = 1024;
__global__ void __launch_bounds__(256) tri_t_part_f32_kernel(int n, const float* __restrict__ M,
                                                             long long ldm,
                                                             const double* __restrict__ v,
                                                             double* __restrict__ part,
                                                             const int* __restrict__ done) {
  if (done && *done) return;
  const int jb = blockIdx.x * kGtCols;
  const long long c0 = (long long)blockIdx.y * kTtChunk;
  if (c0 > jb + kGtCols - 1 || jb >= n) return;  // no row <= any of the block's columns
  __shared__ __align__(16) double vs[kTtChunk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = jb + warp * 8;
  const int cn = (int)min((long long)kTtChunk, (long long)n - c0);
  for (int i = threadIdx.x; i < cn; i += 256) vs[i] = v[c0 + i];
  __syncthreads();
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.0;
  const bool vec = ((ldm & 3) == 0) && ((reinterpret_cast<uintptr_t>(M) & 15) == 0) &&
                   cn == kTtChunk;
  if (vec) {
#pragma unroll 2
    for (int i = lane * 4; i < kTtChunk; i += 128) {
      const double2 v01 = *reinterpret_cast<const double2*>(vs + i);
      const double2 v23 = *reinterpret_cast<const double2*>(vs + i + 2);
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        a[u] = (j0 + u < n && c0 + i <= j0 + u)
                   ? __ldg(reinterpret_cast<const float4*>(M + (long long)(j0 + u) * ldm + c0 + i))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[u] = fma((double)a[u].x, v01.x, acc[u]);
        acc[u] = fma((double)a[u].y, v01.y, acc[u]);
        acc[u] = fma((double)a[u].z, v23.x, acc[u]);
        acc[u] = fma((double)a[u].w, v23.y, acc[u]);
      }
    }
  } else {
    for (int i = lane; i < cn; i += 32) {
      const double x = vs[i];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < n && c0 + i <= j0 + u)
          acc[u] = fma((double)M[(long long)(j0 + u) * ldm + c0 + i], x, acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const double sum = warp_sum_d(acc[u]);
    if (lane == 0 && j0 + u < n) part[(long long)blockIdx.y * n + j0 + u] = sum;
  }
}

// s[j] = sum over the chunks c <= j / 1024 of part[c * n + j] (fixed order)
__global__ void tri_t_reduce_kernel(int n, const double* __restrict__ part, double* __restrict__ s,
                                    const int* __restrict__ done) {
  if (done && *done) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int jb = (j / kGtCols) * kGtCols + kGtCols - 1;  // the last column of j's block
  double acc = part[j];
  for (int c = 1; (long long)c * kTtChunk <= jb && c * kTtChunk < n; ++c) acc += part[(long long)c * n + j];
  s[j] = acc;
}

// M32 = fl32(M) on the upper triangle (zero below): the FP32 copy of the CGLS preconditioner.
__global__ void m_to_f32_kernel(int n, const double* __restrict__ M, long long ldm,
                                float* __restrict__ M32) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)n * n) return;
  const int i = (int)(e % n), j = (int)(e / n);
  M32[e] = i <= j ? (float)M[i + (long long)j * ldm] : 0.f;
}

// ------------------------------------------------------------------------------------------
// CGLS scalar / vector kernels (K7)
// ------------------------------------------------------------------------------------------
// Deterministic single-CTA sum of parts -> *out (FP64).
__global__ void __launch_bounds__(1024) sum_parts_kernel(int np, const double* __restrict__ parts,
                                                         double* __restrict__ out,
                                                         const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += parts[i];
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

// alpha = gamma / delta; x += alpha t (n); r -= alpha q (m).   (Alg. 5 lines 15-17, R-A10)
__global__ void cg_update_xr_kernel(int m, int n, CgState* __restrict__ st,
                                    double* __restrict__ x, const double* __restrict__ t,
                                    double* __restrict__ r, const double* __restrict__ q) {
  if (st->done) return;
  const double alpha = st->gamma / st->delta;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = fma(alpha, t[i], x[i]);
  if (i < m) r[i] = fma(-alpha, q[i], r[i]);
}

// Pass set-up after s = R^-T A' r has been formed: gamma, s0, p = s, x = 0, best tracking.
__global__ void __launch_bounds__(1024) cg_init_kernel(int n, CgState* __restrict__ st,
                                                       const double* __restrict__ s,
                                                       double* __restrict__ p,
                                                       double* __restrict__ x,
                                                       double* __restrict__ xbest) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = fma(s[i], s[i], acc);
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < 32; ++w) g += red[w];
    st->gamma = g;
    st->s0 = sqrt(g);
    if (st->sref <= 0.0) st->sref = st->s0;
    st->best = st->s0;
    st->since = 0;
    st->k = 0;
    st->reason = -1;
    st->done = (g == 0.0) ? 1 : 0;
    if (g == 0.0) st->reason = 3;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    p[i] = s[i];
    x[i] = 0.0;
    xbest[i] = 0.0;
  }
}

// After s = R^-T A' r: gamma' = ||s||^2, history, best iterate, stop tests (R-A11), beta, p.
__global__ void __launch_bounds__(1024) cg_finish_kernel(int n, CgState* __restrict__ st,
                                                         const double* __restrict__ s,
                                                         double* __restrict__ p,
                                                         double* __restrict__ x,
                                                         double* __restrict__ xbest,
                                                         double* __restrict__ hist) {
  if (st->done) return;
  __shared__ double red[32];
  __shared__ int action;  // 0 continue, 1 stop keep x, 2 stop use xbest
  __shared__ int newbest;
  __shared__ double beta_sh;
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = fma(s[i], s[i], acc);
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double g = 0.0;
    for (int w = 0; w < 32; ++w) g += red[w];
    const double ns = sqrt(g);
    const int k = ++st->k;
    if (hist && k <= st->hist_cap) hist[k - 1] = ns / st->s0;
    newbest = 0;
    if (ns < st->best) {
      st->best = ns;
      st->since = 0;
      newbest = 1;
    } else {
      st->since += 1;
    }
    action = 0;
    if (ns / st->s0 <= st->tol) {
      action = 1;
      st->reason = 0;
    } else if (st->best < st->floor * st->sref && st->since >= st->window) {
      action = 2;
      st->reason = 1;
    } else if (k >= st->maxit) {
      action = 2;
      st->reason = 2;
    }
    if (action) st->done = 1;
    const double beta = g / st->gamma;
    beta_sh = beta;
    if (!action) st->gamma = g;
  }
  __syncthreads();
  if (newbest || action == 2) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (newbest) xbest[i] = x[i];
      else x[i] = xbest[i];  // action == 2 and this iterate is not the best
    }
  }
  if (action == 0) {
    const double beta = beta_sh;
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = fma(beta, p[i], s[i]);
  }
}

// r = b - q (restart residual); used with q = A x.
__global__ void residual_kernel(int m, const double* __restrict__ b, const double* __restrict__ q,
                                double* __restrict__ r) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) r[i] = b[i] - q[i];
}

__global__ void axpy_kernel(int n, double a, const double* __restrict__ xx,
                            double* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fma(a, xx[i], y[i]);
}

// ------------------------------------------------------------------------------------------
// Host launchers used by the driver (tcqr.cu)
// ------------------------------------------------------------------------------------------
int cg_gemv_n_chunks(int n) { return (n + kGvCols - 1) / kGvCols; }
int cg_tri_chunks(int n) { return (n + kTriBlk - 1) / kTriBlk; }

cudaError_t cg_launch_tri_n(int n, const double* M, long long ldm, const double* p, double* t,
                            double* part, const int* done, cudaStream_t st) {
  const int nch = cg_tri_chunks(n);
  tri_n_part_kernel<double><<<nch * (nch + 1) / 2, kTriBlk, 0, st>>>(n, M, ldm, p, part, done);
  tri_n_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, nch, part, t, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_tri_n(int n, const float* M, long long ldm, const double* p, double* t,
                            double* part, const int* done, cudaStream_t st) {
  const int nch = cg_tri_chunks(n);
  static int v4 = -1;  // env TCQR_TRI_N_V4=0: one row per thread
  if (v4 < 0) {
    const char* e = getenv("TCQR_TRI_N_V4");
    v4 = (e && e[0] == '0') ? 0 : 1;
  }
  if (v4 && n % 4 == 0 && ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(M) & 15) == 0)
    tri_n_part_f32v_kernel<<<nch * (nch + 1) / 2, kTriBlk, 0, st>>>(n, M, ldm, p, part, done);
  else
    tri_n_part_kernel<float><<<nch * (nch + 1) / 2, kTriBlk, 0, st>>>(n, M, ldm, p, part, done);
  tri_n_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, nch, part, t, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_tri_t(int n, const double* M, long long ldm, const double* v, double* s,
                            const int* done, cudaStream_t st) {
  tri_t_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, M, ldm, v, s, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_tri_t(int n, const float* M, long long ldm, const double* v, double* s,
                            double* part, const int* done, cudaStream_t st) {
  const dim3 g((n + kGtCols - 1) / kGtCols, (n + kTtChunk - 1) / kTtChunk);
  tri_t_part_f32_kernel<<<g, 256, 0, st>>>(n, M, ldm, v, part, done);
  tri_t_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, part, s, done);
  return cudaGetLastError();
}

int cg_tri_t_part_count(int n) { return ((n + kTtChunk - 1) / kTtChunk) * n; }

cudaError_t cg_launch_m_to_f32(int n, const double* M, long long ldm, float* M32, cudaStream_t st) {
  const long long nn = (long long)n * n;
  m_to_f32_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(n, M, ldm, M32);
  return cudaGetLastError();
}

cudaError_t cg_launch_update_x(int n, CgState* s, double* x, const double* t, cudaStream_t st) {
  cg_update_xr_kernel<<<(n + 255) / 256, 256, 0, st>>>(0, n, s, x, t, nullptr, nullptr);
  return cudaGetLastError();
}

// q = A t with delta partials (dpart sized (m+255)/256).
cudaError_t cg_launch_a_n(int m, int n, const float* A, long long lda, const double* t, double* q,
                          double* part, double* dpart, const int* done, cudaStream_t st) {
  const int nch = (n + kGvCols - 1) / kGvCols;
  dim3 g1((m + kGvRows - 1) / kGvRows, nch);
  gemv_n_part_kernel<<<g1, kGvRows, 0, st>>>(m, n, A, lda, t, part, done);
  gemv_n_reduce_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, nch, part, q, dpart, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_a_t(int m, int n, const float* A, long long lda, const double* r, double* v,
                          double* part, const int* done, cudaStream_t st, const double* q,
                          const CgState* cst, double* r_out) {
  int splits, rps;
  gemv_t_plan(m, n, &splits, &rps);
  gemv_t_part_kernel<<<dim3((n + kGtCols - 1) / kGtCols, splits), 256, 0, st>>>(
      m, n, A, lda, r, q, cst, r_out, rps, part, done);
  gemv_t_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, splits, part, v, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_sum_parts(int np, const double* parts, double* out, const int* done,
                                cudaStream_t st) {
  sum_parts_kernel<<<1, 1024, 0, st>>>(np, parts, out, done);
  return cudaGetLastError();
}

cudaError_t cg_launch_update_xr(int m, int n, CgState* s, double* x, const double* t, double* r,
                                const double* q, cudaStream_t st) {
  const int mx = m > n ? m : n;
  cg_update_xr_kernel<<<(mx + 255) / 256, 256, 0, st>>>(m, n, s, x, t, r, q);
  return cudaGetLastError();
}

cudaError_t cg_launch_init(int n, CgState* s, const double* sv, double* p, double* x,
                           double* xbest, cudaStream_t st) {
  cg_init_kernel<<<1, 1024, 0, st>>>(n, s, sv, p, x, xbest);
  return cudaGetLastError();
}

cudaError_t cg_launch_finish(int n, CgState* s, const double* sv, double* p, double* x,
                             double* xbest, double* hist, cudaStream_t st) {
  cg_finish_kernel<<<1, 1024, 0, st>>>(n, s, sv, p, x, xbest, hist);
  return cudaGetLastError();
}

cudaError_t cg_launch_residual(int m, const double* b, const double* q, double* r,
                               cudaStream_t st) {
  residual_kernel<<<(m + 255) / 256, 256, 0, st>>>(m, b, q, r);
  return cudaGetLastError();
}

cudaError_t cg_launch_axpy(int n, double a, const double* x, double* y, cudaStream_t st) {
  axpy_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, a, x, y);
  return cudaGetLastError();
}

}  // namespace tcqr

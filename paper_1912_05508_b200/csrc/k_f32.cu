// k_f32.cu -- K2b: FP32 products of the recursion below the tensor-core cutoff (reading R-A1:
// the leaf panelQR is single precision, so Alg. 2 lines 8-9 run in FP32 for
// nodes with w <= cutoff).  Deterministic split-K for R12 = Q1' A2; a row-parallel update.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcqr {

constexpr int kTnRows = 64;   // rows per shared-memory chunk
constexpr int kTnPad = 68;    // row stride (floats) of the staged tiles, 16-byte aligned
#ifndef TCQR_PROJ_OCC
#define TCQR_PROJ_OCC 2
#endif
#ifndef TCQR_PROJ_SLICE
#define TCQR_PROJ_SLICE 16
#endif
// streaming projection: CTAs per SM and the update's column slice (registers: two CTAs per SM
// need <= 128 per thread)
constexpr int kProjOcc = TCQR_PROJ_OCC, kProjSlice = TCQR_PROJ_SLICE;
constexpr int kResSmemMax = 220 * 1024;  // dynamic shared memory cap of the resident projection

// P_s (h x w2, ld h) = sum over rows [r0_s, r1_s) of Q1(r, :)' A2(r, :).  h, w2 <= 64.
// 256 threads = 4 row groups x (8 x 8 threads) each owning an 8 x 8 output micro-tile.
__global__ void __launch_bounds__(256) f32_tn_kernel(int m, int h, int w2,
                                                     const float* __restrict__ Q1, long long ldq,
                                                     const float* __restrict__ A2, long long lda,
                                                     float* __restrict__ P, int splits) {
  __shared__ __align__(16) float Qs[kTnRows][kTnPad];
  __shared__ __align__(16) float As[kTnRows][kTnPad];
  const int s = blockIdx.x;
  const long long r0 = (long long)s * m / splits, r1 = (long long)(s + 1) * m / splits;
  const int tid = threadIdx.x, grp = tid >> 6, t = tid & 63, ti = t & 7, tj = t >> 3;
  float acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;
  // software-pipelined: the next chunk's 32 loads per thread are in flight while the current
  // chunk (staged in shared memory) is multiplied
  float qv_[16], av_[16];
  auto fetch = [&](long long c0) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 256;
      const int rr = e & (kTnRows - 1), cc = e / kTnRows;
      const long long row = c0 + rr;
      const bool rok = row < r1;
      qv_[u] = (rok && cc < h) ? __ldg(Q1 + row + cc * ldq) : 0.f;
      av_[u] = (rok && cc < w2) ? __ldg(A2 + row + cc * lda) : 0.f;
    }
  };
  if (r0 < r1) fetch(r0);
  for (long long c0 = r0; c0 < r1; c0 += kTnRows) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = tid + u * 256;
      const int rr = e & (kTnRows - 1), cc = e / kTnRows;
      Qs[rr][cc] = qv_[u];
      As[rr][cc] = av_[u];
    }
    __syncthreads();
    if (c0 + kTnRows < r1) fetch(c0 + kTnRows);
#pragma unroll 4
    for (int rr = grp; rr < kTnRows; rr += 4) {
      const float4 q0 = *reinterpret_cast<const float4*>(&Qs[rr][ti * 8]);
      const float4 q1 = *reinterpret_cast<const float4*>(&Qs[rr][ti * 8 + 4]);
      const float4 a0 = *reinterpret_cast<const float4*>(&As[rr][tj * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[rr][tj * 8 + 4]);
      const float qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      const float2 av2[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w),
                             make_float2(a1.x, a1.y), make_float2(a1.z, a1.w)};
#pragma unroll
      for (int a = 0; a < 8; ++a) {  // FFMA2: the same fmaf sequence per entry
        const float2 qa = make_float2(qv[a], qv[a]);
#pragma unroll
        for (int b2 = 0; b2 < 4; ++b2) {
          const float2 c = ffma2(qa, av2[b2], make_float2(acc[a][2 * b2], acc[a][2 * b2 + 1]));
          acc[a][2 * b2] = c.x;
          acc[a][2 * b2 + 1] = c.y;
        }
      }
    }
  }
  // combine the 4 row groups in a fixed order (deterministic)
  __syncthreads();
  float* red = &Qs[0][0];  // 64 x 64 floats fit in Qs (64 x 68)
  for (int g = 0; g < 4; ++g) {
    if (grp == g) {
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          float* p = red + (ti * 8 + a) * kTnPad + tj * 8 + b;
          *p = (g == 0) ? acc[a][b] : *p + acc[a][b];
        }
    }
    __syncthreads();
  }
  float* out = P + (long long)s * h * w2;
  for (int e = tid; e < h * w2; e += 256) {
    const int i = e % h, j = e / h;
    out[i + (long long)j * h] = red[i * kTnPad + j];
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
  if (splits > num_sms) splits = num_sms;
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

// A2 (m x w2) -= Q1 (m x h) T (h x w2, ld h).  One thread per row, all w2 <= 64 columns.
template <int W2>
__global__ void __launch_bounds__(128) f32_nn_kernel(int m, int h, int w2,
                                                     const float* __restrict__ Q1, long long ldq,
                                                     const float* __restrict__ T,
                                                     float* __restrict__ A2, long long lda) {
  __shared__ __align__(16) float Ts[64][W2];
  for (int e = threadIdx.x; e < h * W2; e += blockDim.x) {
    const int i = e / W2, j = e % W2;
    Ts[i][j] = (j < w2) ? T[i + (long long)j * h] : 0.f;
  }
  __syncthreads();
  const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= m) return;
  float acc[W2];
#pragma unroll
  for (int j = 0; j < W2; ++j) acc[j] = 0.f;
  for (int i0 = 0; i0 < h; i0 += 8) {
    float qb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) qb[u] = (i0 + u < h) ? __ldg(Q1 + row + (long long)(i0 + u) * ldq) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u < h) {
        const float2 qu = make_float2(qb[u], qb[u]);
#pragma unroll
        for (int j = 0; j < W2; j += 4) {  // FFMA2: the same fmaf sequence per entry
          const float4 tv = *reinterpret_cast<const float4*>(&Ts[i0 + u][j]);
          const float2 c01 = ffma2(qu, make_float2(tv.x, tv.y), make_float2(acc[j], acc[j + 1]));
          const float2 c23 = ffma2(qu, make_float2(tv.z, tv.w), make_float2(acc[j + 2], acc[j + 3]));
          acc[j] = c01.x;
          acc[j + 1] = c01.y;
          acc[j + 2] = c23.x;
          acc[j + 3] = c23.y;
        }
      }
    }
  }
  float cold[W2];
#pragma unroll
  for (int j = 0; j < W2; ++j) cold[j] = (j < w2) ? A2[row + (long long)j * lda] : 0.f;
#pragma unroll
  for (int j = 0; j < W2; ++j)
    if (j < w2) A2[row + (long long)j * lda] = cold[j] - acc[j];
}

// The same for 32 < w2 <= 64 with two threads per row (64 rows per CTA, thread g = threadIdx.x / 64
// takes columns [32 g, 32 g + 32)): the one-thread-per-row version held 64 accumulators and 64
// old values (255 registers with spills, one CTA per SM).  The two threads of a row read the same
// Q1 values (the second read hits L1).
__global__ void __launch_bounds__(128) f32_nn2_kernel(int m, int h, int w2,
                                                      const float* __restrict__ Q1, long long ldq,
                                                      const float* __restrict__ T,
                                                      float* __restrict__ A2, long long lda) {
  __shared__ __align__(16) float Ts[64][64];
  for (int e = threadIdx.x; e < h * 64; e += blockDim.x) {
    const int i = e / 64, j = e % 64;
    Ts[i][j] = (j < w2) ? T[i + (long long)j * h] : 0.f;
  }
  __syncthreads();
  const int g = threadIdx.x >> 6;
  const long long row = (long long)blockIdx.x * 64 + (threadIdx.x & 63);
  if (row >= m) return;
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = 0.f;
  for (int i0 = 0; i0 < h; i0 += 8) {
    float qb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) qb[u] = (i0 + u < h) ? __ldg(Q1 + row + (long long)(i0 + u) * ldq) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (i0 + u < h) {
        const float2 qu = make_float2(qb[u], qb[u]);
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 tv = *reinterpret_cast<const float4*>(&Ts[i0 + u][32 * g + j]);
          const float2 c01 = ffma2(qu, make_float2(tv.x, tv.y), make_float2(acc[j], acc[j + 1]));
          const float2 c23 = ffma2(qu, make_float2(tv.z, tv.w), make_float2(acc[j + 2], acc[j + 3]));
          acc[j] = c01.x;
          acc[j + 1] = c01.y;
          acc[j + 2] = c23.x;
          acc[j + 3] = c23.y;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int jj = 32 * g + j;
    if (jj < w2) A2[row + (long long)jj * lda] -= acc[j];
  }
}

cudaError_t f32_nn_update(int m, int h, int w2, const float* Q1, long long ldq, const float* T,
                          float* A2, long long lda, cudaStream_t st) {
  if (h > 64 || w2 > 64) return cudaErrorInvalidValue;
  if (w2 <= 32)
    f32_nn_kernel<32><<<(m + 127) / 128, 128, 0, st>>>(m, h, w2, Q1, ldq, T, A2, lda);
  else
    f32_nn2_kernel<<<(m + 63) / 64, 128, 0, st>>>(m, h, w2, Q1, ldq, T, A2, lda);
  return cudaGetLastError();
}


// ------------------------------------------------------------------------------------------
// Fused projection (one cooperative launch): R12 = Q1' A2 (deterministic), R block <- R12,
// A2 -= Q1 R12.  CTA b owns rows [b m / G, (b+1) m / G).
//   phase 1  partial P_b = Q1_b' A2_b (same micro-tiles as f32_tn_kernel)
//   barrier
//   phase 2  CTA b sums its slice of the h*w2 entries over all G partials in a fixed order
//   barrier
//   phase 3  A2_b -= Q1_b R12 (R12 staged in shared memory)
// ------------------------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long gtimer_f() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
unsigned long long* g_proj_dbg = nullptr;

// Phase 2 of the fused projection: CTA b sums its slice of the h*w2 entries over all G partials
// in a fixed order (8 partial-groups x 32 entries per pass, all loads of a thread in flight, then
// a fixed-order combine in shared memory `part` [8][32]); writes T and the R block.
__device__ __forceinline__ void proj_phase2(const float* P, float* T, float* Rblk, long long ldr,
                                            int h, int hw, int G, int b, float* part) {
  const int tid = threadIdx.x;
  const int e0 = (int)((long long)b * hw / G), e1 = (int)((long long)(b + 1) * hw / G);
  const int el = tid & 31, pg = tid >> 5;
  const int gper = (G + 7) / 8, g0 = pg * gper, g1 = min(G, g0 + gper);
  for (int eb = e0; eb < e1; eb += 32) {
    const int e = eb + el;
    float s = 0.f;
    if (e < e1) {
      // up to 24 partials per thread: all loads in flight, then the fixed-order sum
      int g = g0;
      for (; g + 24 <= g1; g += 24) {
        float v[24];
#pragma unroll
        for (int u = 0; u < 24; ++u) v[u] = __ldcg(P + (long long)(g + u) * hw + e);
#pragma unroll
        for (int u = 0; u < 24; ++u) s += v[u];
      }
      if (g < g1) {
        float v[24];
#pragma unroll
        for (int u = 0; u < 24; ++u) v[u] = g + u < g1 ? __ldcg(P + (long long)(g + u) * hw + e) : 0.f;
#pragma unroll
        for (int u = 0; u < 24; ++u)
          if (g + u < g1) s += v[u];
      }
    }
    __syncthreads();
    part[pg * 32 + el] = s;
    __syncthreads();
    if (pg == 0 && e < e1) {
      float tot = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) tot += part[q * 32 + el];
      T[e] = tot;
      const int i = e % h, j = e / h;
      Rblk[i + (long long)j * ldr] = tot;
    }
  }
}

template <int TD>  // TD = 32 or 64: h, w2 <= TD
__global__ void __launch_bounds__(256, kProjOcc) f32_project_kernel(int m, int h, int w2,
                                                             const float* __restrict__ Q1,
                                                             long long ldq, float* A2,
                                                             long long lda, float* Rblk,
                                                             long long ldr, float* P, float* T,
                                                             int* bar, unsigned long long* dbg) {
#define PDBG(i) if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[i] = gtimer_f();
  constexpr int MT = TD / 8;  // micro-tile edge
  PDBG(0);
  __shared__ __align__(16) float Qs[kTnRows][kTnPad];
  __shared__ __align__(16) float As[kTnRows][kTnPad];
  const int G = gridDim.x, b = blockIdx.x;
  const long long r0 = (long long)b * m / G, r1 = (long long)(b + 1) * m / G;
  const int tid = threadIdx.x, grp = tid >> 6, t = tid & 63, ti = t & 7, tj = t >> 3;
  const int hw = h * w2;
  // ---- phase 1: P_b = Q1_b' A2_b ----
  {
    float acc[MT][MT];
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int c = 0; c < MT; ++c) acc[a][c] = 0.f;
    constexpr int NL = kTnRows * TD / 256;  // loads per thread per matrix per chunk
    // the next chunk's loads are issued before the current chunk's products (register double
    // buffering): one HBM round trip per chunk overlaps the compute instead of following it
    float qv_[NL], av_[NL];
    auto load_chunk = [&](long long c0) {
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        const int rr = e & (kTnRows - 1), cc = e / kTnRows;
        const long long row = c0 + rr;
        const bool rok = row < r1;
        qv_[u] = (rok && cc < h) ? __ldg(Q1 + row + cc * ldq) : 0.f;
        av_[u] = (rok && cc < w2) ? A2[row + cc * lda] : 0.f;
      }
    };
    if (r0 < r1) load_chunk(r0);
    for (long long c0 = r0; c0 < r1; c0 += kTnRows) {
      __syncthreads();
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        const int rr = e & (kTnRows - 1), cc = e / kTnRows;
        Qs[rr][cc] = qv_[u];
        As[rr][cc] = av_[u];
      }
      __syncthreads();
      if (c0 + kTnRows < r1) load_chunk(c0 + kTnRows);
#pragma unroll 4
      for (int rr = grp; rr < kTnRows; rr += 4) {
        float qv[MT], av[MT];
#pragma unroll
        for (int v4 = 0; v4 < MT; v4 += 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(&Qs[rr][ti * MT + v4]);
          const float4 a4 = *reinterpret_cast<const float4*>(&As[rr][tj * MT + v4]);
          qv[v4] = q4.x; qv[v4 + 1] = q4.y; qv[v4 + 2] = q4.z; qv[v4 + 3] = q4.w;
          av[v4] = a4.x; av[v4 + 1] = a4.y; av[v4 + 2] = a4.z; av[v4 + 3] = a4.w;
        }
#pragma unroll
        for (int a = 0; a < MT; ++a) {  // FFMA2: the same fmaf sequence per entry
          const float2 qa = make_float2(qv[a], qv[a]);
#pragma unroll
          for (int c = 0; c < MT; c += 2) {
            const float2 r = ffma2(qa, make_float2(av[c], av[c + 1]),
                                   make_float2(acc[a][c], acc[a][c + 1]));
            acc[a][c] = r.x;
            acc[a][c + 1] = r.y;
          }
        }
      }
    }
    __syncthreads();
    float* red = &Qs[0][0];
    for (int g = 0; g < 4; ++g) {
      if (grp == g) {
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int c = 0; c < MT; ++c) {
            float* p = red + (ti * MT + a) * kTnPad + tj * MT + c;
            *p = (g == 0) ? acc[a][c] : *p + acc[a][c];
          }
      }
      __syncthreads();
    }
    float* out = P + (long long)b * hw;
    for (int e = tid; e < hw; e += 256) {
      const int i = e % h, j = e / h;
      out[e] = red[i * kTnPad + j];
    }
  }
  PDBG(1);
  grid_barrier(bar, G);
  PDBG(2);
  proj_phase2(P, T, Rblk, ldr, h, hw, G, b, &As[0][0]);
  PDBG(3);
  grid_barrier(bar, G);
  PDBG(4);
  // ---- phase 3: A2_b -= Q1_b T  (all loads of a row issued before any store) ----
  {
    float* Ts = &Qs[0][0];  // [h][TD]
    {
      // coalesced read of T (h x w2, column-major) with all loads of a thread in flight; the
      // transpose into Ts [h][TD] happens in shared memory
      constexpr int NL = TD * TD / 256;
      float tv[NL];
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        tv[u] = e < hw ? __ldcg(T + e) : 0.f;
      }
      for (int e = tid; e < h * TD; e += 256) Ts[e] = 0.f;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        if (e < hw) Ts[(e % h) * TD + e / h] = tv[u];
      }
    }
    __syncthreads();
    for (long long row = r0 + tid; row < r1; row += 256) {
      // the whole Q1 row first (h <= TD loads in flight), then each 32-column half of A2
      float qrow[TD];
#pragma unroll
      for (int i = 0; i < TD; ++i) qrow[i] = (i < h) ? __ldg(Q1 + row + (long long)i * ldq) : 0.f;
#pragma unroll 1
      for (int jh = 0; jh < TD; jh += kProjSlice) {  // column slices keep registers bounded
        float cold[kProjSlice];
#pragma unroll
        for (int j = 0; j < kProjSlice; ++j) cold[j] = (jh + j < w2) ? A2[row + (long long)(jh + j) * lda] : 0.f;
        float acc[kProjSlice];
#pragma unroll
        for (int j = 0; j < kProjSlice; ++j) acc[j] = 0.f;
#pragma unroll
        for (int i = 0; i < TD; ++i) {
          if (i < h) {
            const float2 qi = make_float2(qrow[i], qrow[i]);
#pragma unroll
            for (int j = 0; j < kProjSlice; j += 4) {  // FFMA2: the same fmaf sequence per entry
              const float4 tv = *reinterpret_cast<const float4*>(&Ts[i * TD + jh + j]);
              const float2 c01 = ffma2(qi, make_float2(tv.x, tv.y), make_float2(acc[j], acc[j + 1]));
              const float2 c23 = ffma2(qi, make_float2(tv.z, tv.w),
                                       make_float2(acc[j + 2], acc[j + 3]));
              acc[j] = c01.x;
              acc[j + 1] = c01.y;
              acc[j + 2] = c23.x;
              acc[j + 3] = c23.y;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kProjSlice; ++j)
          if (jh + j < w2) A2[row + (long long)(jh + j) * lda] = cold[j] - acc[j];
      }
    }
  }
  PDBG(5);
#undef PDBG
}


// ------------------------------------------------------------------------------------------
// Resident fused projection: CTA b owns rows [b RB, (b+1) RB) (RB a multiple of 4) and keeps its
// rows of Q1 and A2 in shared memory from one cp.async round trip to the update, so Q1 and A2
// are read from HBM once and A2 written once.  Same three phases and the same fixed
// accumulation orders per entry as f32_project_kernel (rows in increasing order inside a
// thread, row groups combined 0..3, partials 0..G-1, T columns l = 0..h-1).
// Shared layout: column c of Q1 / A2 at c*RBp + skew(c), skew = ((c / MT) & 7) * 4 floats, so the
// eight micro-tile column groups of a warp hit distinct banks with 16-byte row-quad loads.
// ------------------------------------------------------------------------------------------
template <int TD>
__device__ __forceinline__ int res_col(int c, int RBp) {
  return c * RBp + ((c / (TD / 8)) & 7) * 4;
}

template <int TD>
__host__ __device__ constexpr int res_smem_floats(int RBp) {
  return 2 * (TD * RBp + 32) + TD * (TD + 1) + TD * TD;
}

template <int TD>
__global__ void __launch_bounds__(256, 1) f32_project_res_kernel(
    int m, int h, int w2, int RB, int RBp, const float* __restrict__ Q1, long long ldq, float* A2,
    long long lda, float* Rblk, long long ldr, float* P, float* T, int* bar, int vec,
    unsigned long long* dbg) {
#define PDBG(i) if (dbg && blockIdx.x == 0 && threadIdx.x == 0) dbg[i] = gtimer_f();
  constexpr int MT = TD / 8;
  PDBG(0);
  extern __shared__ __align__(16) float dsm[];
  float* Qs = dsm;
  float* As = Qs + TD * RBp + 32;
  float* red = As + TD * RBp + 32;  // [TD][TD + 1] row-group combine
  float* Ts = red + TD * (TD + 1);  // [h][TD] R12 for the update; phase-2 scratch before that
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const long long r0 = (long long)b * RB;
  const int nrows = (int)min((long long)RB, (long long)m - r0);
  const int nq = RB / 4, hw = h * w2;
  // ---- load: Q1_b, A2_b -> shared (rows >= nrows and columns >= h / w2 are zero) ----
  if (vec) {
    for (int e = tid; e < (h + w2) * nq; e += 256) {
      const int c = e / nq, q = e - c * nq;
      const bool isq = c < h;
      const int cc = isq ? c : c - h;
      const float* col = isq ? Q1 + r0 + (long long)cc * ldq : A2 + r0 + (long long)cc * lda;
      const int valid = max(0, min(4, nrows - 4 * q));
      const float* src = valid > 0 ? col + 4 * q : col;
      const unsigned dst = static_cast<unsigned>(
          __cvta_generic_to_shared((isq ? Qs : As) + res_col<TD>(cc, RBp) + 4 * q));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                   "r"(valid * 4) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  } else {
    for (int e = tid; e < (h + w2) * RB; e += 256) {
      const int c = e / RB, r = e - c * RB;
      const bool isq = c < h;
      const int cc = isq ? c : c - h;
      const float v = r < nrows ? (isq ? Q1[r0 + r + (long long)cc * ldq]
                                       : A2[r0 + r + (long long)cc * lda])
                                : 0.f;
      (isq ? Qs : As)[res_col<TD>(cc, RBp) + r] = v;
    }
  }
  for (int e = tid; e < (TD - h) * RB; e += 256) Qs[res_col<TD>(h + e / RB, RBp) + e % RB] = 0.f;
  for (int e = tid; e < (TD - w2) * RB; e += 256) As[res_col<TD>(w2 + e / RB, RBp) + e % RB] = 0.f;
  if (vec) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  PDBG(6);
  // ---- phase 1: P_b = Q1_b' A2_b; 4 row groups x (8 x 8 threads) with MT x MT micro-tiles ----
  {
    const int grp = tid >> 6, t = tid & 63, ti = t & 7, tj = t >> 3;
    const float* qb = Qs + res_col<TD>(ti * MT, RBp);  // column ti*MT + a at qb + a*RBp
    const float* ab = As + res_col<TD>(tj * MT, RBp);
    float acc[MT][MT];
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int c = 0; c < MT; ++c) acc[a][c] = 0.f;
    for (int q = grp; q < nq; q += 4) {
      float4 qv[MT], av[MT];
#pragma unroll
      for (int a = 0; a < MT; ++a) qv[a] = *reinterpret_cast<const float4*>(qb + a * RBp + 4 * q);
#pragma unroll
      for (int c = 0; c < MT; ++c) av[c] = *reinterpret_cast<const float4*>(ab + c * RBp + 4 * q);
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int c = 0; c < MT; ++c) {
          acc[a][c] = fmaf(qv[a].x, av[c].x, acc[a][c]);
          acc[a][c] = fmaf(qv[a].y, av[c].y, acc[a][c]);
          acc[a][c] = fmaf(qv[a].z, av[c].z, acc[a][c]);
          acc[a][c] = fmaf(qv[a].w, av[c].w, acc[a][c]);
        }
    }
    PDBG(7);
    for (int g = 0; g < 4; ++g) {
      if (grp == g) {
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int c = 0; c < MT; ++c) {
            float* p = red + (tj * MT + c) * (TD + 1) + ti * MT + a;  // [j][i]: P reads below
                                                                       // are conflict-free
            *p = (g == 0) ? acc[a][c] : *p + acc[a][c];
          }
      }
      __syncthreads();
    }
    float* out = P + (long long)b * hw;
    for (int e = tid; e < hw; e += 256) {
      const int i = e % h, j = e / h;
      out[e] = red[j * (TD + 1) + i];
    }
  }
  PDBG(1);
  grid_barrier(bar, G);
  PDBG(2);
  proj_phase2(P, T, Rblk, ldr, h, hw, G, b, Ts);
  PDBG(3);
  grid_barrier(bar, G);
  PDBG(4);
  // ---- phase 3: A2_b -= Q1_b T from shared memory; task = (row quad, TD/4-column group) ----
  {
    {
      // coalesced read of T (h x w2, column-major) with all loads of a thread in flight; the
      // transpose into Ts [h][TD] happens in shared memory
      constexpr int NL = TD * TD / 256;
      float tv[NL];
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        tv[u] = e < hw ? __ldcg(T + e) : 0.f;
      }
      for (int e = tid; e < h * TD; e += 256) Ts[e] = 0.f;
      __syncthreads();
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int e = tid + u * 256;
        if (e < hw) Ts[(e % h) * TD + e / h] = tv[u];
      }
    }
    __syncthreads();
    PDBG(8);
    constexpr int CW = TD / 4;
    for (int task = tid; task < nq * 4; task += 256) {
      const int q = task % nq, cg = task / nq;
      if (4 * q >= nrows || cg * CW >= w2) continue;
      float acc[4][CW];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int j = 0; j < CW; ++j) acc[r][j] = 0.f;
      for (int l = 0; l < h; ++l) {
        const float4 qv = *reinterpret_cast<const float4*>(Qs + res_col<TD>(l, RBp) + 4 * q);
        const float* tr = Ts + l * TD + cg * CW;
#pragma unroll
        for (int j = 0; j < CW; j += 4) {
          const float4 tv = *reinterpret_cast<const float4*>(tr + j);
          const float tj4[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc[0][j + u] = fmaf(qv.x, tj4[u], acc[0][j + u]);
            acc[1][j + u] = fmaf(qv.y, tj4[u], acc[1][j + u]);
            acc[2][j + u] = fmaf(qv.z, tj4[u], acc[2][j + u]);
            acc[3][j + u] = fmaf(qv.w, tj4[u], acc[3][j + u]);
          }
        }
      }
      const bool full = vec && 4 * q + 4 <= nrows;
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int col = cg * CW + j;
        if (col < w2) {
          const float4 a4 = *reinterpret_cast<const float4*>(As + res_col<TD>(col, RBp) + 4 * q);
          const float4 o = make_float4(a4.x - acc[0][j], a4.y - acc[1][j], a4.z - acc[2][j],
                                       a4.w - acc[3][j]);
          float* dst = A2 + r0 + 4 * q + (long long)col * lda;
          if (full) {
            *reinterpret_cast<float4*>(dst) = o;
          } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
            for (int r = 0; r < 4 && 4 * q + r < nrows; ++r) dst[r] = ov[r];
          }
        }
      }
    }
  }
  PDBG(5);
#undef PDBG
}

template <int TD>
static int f32_project_capacity(int num_sms) {
  static int per_sm = -1;
  if (per_sm < 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f32_project_kernel<TD>, 256, 0) !=
          cudaSuccess)
    per_sm = 0;
  return per_sm * num_sms;
}

template <int TD>
static int f32_project_res_capacity(int num_sms, int smem) {
  static int set = 0;
  if (!set) {
    cudaFuncSetAttribute(f32_project_res_kernel<TD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kResSmemMax);
    set = 1;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f32_project_res_kernel<TD>, 256,
                                                    smem) != cudaSuccess)
    per_sm = 0;
  return per_sm * num_sms;
}

static cudaLaunchConfig_t coop_cfg(int G, int smem, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// One cooperative launch; cudaErrorNotSupported when it cannot be made co-resident.  The
// resident variant (one CTA per SM, rows kept in shared memory) is used whenever a CTA's rows
// fit; otherwise the streaming variant re-reads Q1 and A2 in the update.
cudaError_t f32_project(int m, int h, int w2, const float* Q1, long long ldq, float* A2,
                        long long lda, float* Rblk, long long ldr, float* T, float* P,
                        long long p_cap, int* bar, int num_sms, cudaStream_t st) {
  if (h > 64 || w2 > 64) return cudaErrorNotSupported;
  const bool small = (h <= 32 && w2 <= 32);
  const int TD = small ? 32 : 64;
  cudaLaunchAttribute attr[1];
  {
    int G = std::min(num_sms, std::max(1, m / 64));
    int RB = ((m + G - 1) / G + 3) / 4 * 4;
    G = (m + RB - 1) / RB;
    const int RBp = (RB + 31) / 32 * 32;
    const int smem = (int)sizeof(float) * (small ? res_smem_floats<32>(RBp) : res_smem_floats<64>(RBp));
    const int cap = smem > kResSmemMax ? 0
                    : small ? f32_project_res_capacity<32>(num_sms, smem)
                            : f32_project_res_capacity<64>(num_sms, smem);
    if (smem <= kResSmemMax && G <= cap && (long long)G * h * w2 <= p_cap) {
      const int vec = ((reinterpret_cast<uintptr_t>(Q1) | reinterpret_cast<uintptr_t>(A2)) % 16 == 0) &&
                      ldq % 4 == 0 && lda % 4 == 0;
      cudaLaunchConfig_t cfg = coop_cfg(G, smem, st, attr);
      return small ? cudaLaunchKernelEx(&cfg, f32_project_res_kernel<32>, m, h, w2, RB, RBp, Q1,
                                        ldq, A2, lda, Rblk, ldr, P, T, bar, vec, g_proj_dbg)
                   : cudaLaunchKernelEx(&cfg, f32_project_res_kernel<64>, m, h, w2, RB, RBp, Q1,
                                        ldq, A2, lda, Rblk, ldr, P, T, bar, vec, g_proj_dbg);
    }
  }
  (void)TD;
  int G = (m + 255) / 256;
  const int cap = small ? f32_project_capacity<32>(num_sms) : f32_project_capacity<64>(num_sms);
  if (G > cap) G = cap;
  if ((long long)G * h * w2 > p_cap) G = (int)(p_cap / ((long long)h * w2));
  if (G < 1) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = coop_cfg(G, 0, st, attr);
  return small ? cudaLaunchKernelEx(&cfg, f32_project_kernel<32>, m, h, w2, Q1, ldq, A2, lda,
                                    Rblk, ldr, P, T, bar, g_proj_dbg)
               : cudaLaunchKernelEx(&cfg, f32_project_kernel<64>, m, h, w2, Q1, ldq, A2, lda,
                                    Rblk, ldr, P, T, bar, g_proj_dbg);
}

}  // namespace tcqr

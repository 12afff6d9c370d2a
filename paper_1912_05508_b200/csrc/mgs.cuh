// mgs.cuh -- the Alg. 4 MGS step shared by the CAQR panel kernels
// (k_panel.cu) and the fused leaf kernel (k_leaf.cu).  Device code only.
#pragma once
#include "common.cuh"

namespace tcqr {

// Lane l ends with the warp sum of v[l % W] (all lanes sharing l % W hold the same value).
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

// One MGS step with reduction width W (>= active columns).  Columns >= W are zero.
template <int NT, int RPT, int W>
__device__ __forceinline__ void mgs_step(float (&x)[RPT][32], int nrows, int w, int k,
                                         float* const (&qp)[RPT], int qstride, float* Rdst,
                                         long long rs, long long cs, bool check, int* status,
                                         int col0, float* red, int& buf,
                                         bool write_lower = true, bool idle = false,
                                         int bar_cnt = NT) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // idle (warp-uniform): every row of this warp is zero and stays zero in this step; the warp
  // only contributes a zero partial (x + 0 = x: the sums are unchanged) and meets the barrier
  float part = 0.f;
  if (!idle) {
    float p[32];
#pragma unroll
    for (int j = 0; j < W; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int r = 0; r < RPT; ++r) acc = fmaf(x[r][0], x[r][j], acc);
      p[j] = acc;
    }
    part = tr_reduce<W>(p);  // lane j: warp sum of a_k' a_{k+(j%W)}
  }
  red[(buf * NW + warp) * 32 + lane] = part;
  // named barrier 1 over the bar_cnt participating threads (all NT unless the caller grows the
  // participating warp set step by step, as the pipelined root does)
  asm volatile("bar.sync 1, %0;" ::"r"(bar_cnt) : "memory");
  if (idle) {
    buf ^= 1;
    return;
  }
  float tot = 0.f;
#pragma unroll
  for (int v = 0; v < NW; ++v) tot += red[(buf * NW + v) * 32 + lane];
  buf ^= 1;
  const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, 0));
  const bool zero = !(rkk > 0.f) || !isfinite(rkk);
  if (check && zero && threadIdx.x == 0 && status) atomicMin(status, col0 + k + 1);
  const int jl = lane & (W - 1);
  // Q(:,k)/R(k,k) and the R(k,j) quotients use one correctly rounded reciprocal: the IEEE
  // divide's FCHK slow path fires on zero dividends (half of every stacked-triangle level) and
  // made those steps 1.6x slower (tools/micro/mgs_step2.cu).  <= 1 extra rounding.
  const float inv = zero ? 0.f : __frcp_rn(rkk);
  const float rkj = zero ? 0.f : (jl == 0 ? rkk : tot * inv);
  if (warp == 0) {  // R(k, j) at Rdst[k*rs + j*cs]
    if (lane < w - k && lane < W) Rdst[k * rs + (long long)(k + lane) * cs] = rkj;
    if (write_lower && lane < k) Rdst[k * rs + (long long)lane * cs] = 0.f;
  }
  float q[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    q[r] = x[r][0] * inv;
    const int row = threadIdx.x + r * NT;
    if (row < nrows && qp[r]) qp[r][k * qstride] = q[r];  // null sink: the row is not stored
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

// Alg. 4 on the rows held in x (thread t owns rows t + r*NT): Q columns -> qs, R rows -> Rdst.
// One step k with the reduction width chosen from the active column count.
template <int NT, int RPT>
__device__ __forceinline__ void mgs_step_any(float (&x)[RPT][32], int nrows, int w, int k,
                                             float* const (&qp)[RPT], int qstride, float* Rdst,
                                             long long rs, long long cs, bool check, int* status,
                                             int col0, float* red, int& buf,
                                             bool idle = false, int bar_cnt = NT) {
  const int act = w - k;
  if (act > 16)
    mgs_step<NT, RPT, 32>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
  else if (act > 8)
    mgs_step<NT, RPT, 16>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
  else if (act > 4)
    mgs_step<NT, RPT, 8>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
  else if (act > 2)
    mgs_step<NT, RPT, 4>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
  else if (act > 1)
    mgs_step<NT, RPT, 2>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
  else
    mgs_step<NT, RPT, 1>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, true, idle, bar_cnt);
}

}  // namespace tcqr

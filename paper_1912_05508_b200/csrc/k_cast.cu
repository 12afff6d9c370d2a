// k_cast.cu -- K1: FP16 range guard and cast (reading R-A4), the R12
// finalize step (unscale, write R, scaled FP16 copy for K4), input validation and small copies.
//
// The paper is silent on FP16 range (PAPER.md:127-141 only notes FP16's "significantly
// constrained range"); reading R-A4 guards it with a per-column power-of-two scale
// s_j = 2^-floor(log2 max_i |X_ij|), exact to apply and undo.
#include <cooperative_groups.h>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace tcqr {

// streaming (evict-first) loads and stores of the cast (env TCQR_L2_EF=0: plain): see g_l2_ef in
// k_gemm_tc.cu -- the casts stream GBs beside the leaves and must not evict the leaf's code
__constant__ int g_cast_ef = 1;


constexpr int kCastThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, red[i]);
  return r;
}

// One CTA per column: pass 1 max|x| (and non-finite detection), pass 2 scaled RNE cast.
__global__ void __launch_bounds__(kCastThreads) cast_scale_kernel(
    int m, const float* __restrict__ X, long long ldx, __half* __restrict__ Xh, long long ldh,
    float* __restrict__ inv_s, int scaling, int* status, int col_base) {
  __shared__ float red[32];
  const int j = blockIdx.x;
  const float* x = X + (long long)j * ldx;
  __half* xh = Xh + (long long)j * ldh;
  const bool vec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                   ((ldh & 3) == 0) && ((reinterpret_cast<uintptr_t>(Xh) & 7) == 0);
  const int m4 = vec ? (m & ~3) : 0;
  float mx = 0.f;
  bool bad = false;
#pragma unroll 8
  for (int i = threadIdx.x * 4; i < m4; i += kCastThreads * 4) {  // 8 loads in flight
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  for (int i = m4 + threadIdx.x; i < m; i += kCastThreads) {
    const float v = x[i];
    mx = fmaxf(mx, fabsf(v));
    bad |= !isfinite(v);
  }
  if (bad && status) atomicMin(status, col_base + j + 1);
  float s = 1.f;
  if (scaling) {
    mx = block_max(mx, red);
    s = pow2_scale_for(mx);
  }
  if (threadIdx.x == 0 && inv_s) inv_s[j] = 1.f / s;
#pragma unroll 8
  for (int i = threadIdx.x * 4; i < m4; i += kCastThreads * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + i);
    __half2 lo = __floats2half2_rn(v.x * s, v.y * s);
    __half2 hi = __floats2half2_rn(v.z * s, v.w * s);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(xh + i) = pk;
  }
  for (int i = m4 + threadIdx.x; i < m; i += kCastThreads) xh[i] = __float2half_rn(x[i] * s);
}

// Pass 1 of the parallel cast: per-(row chunk, column) max |x| folded into cmax[j] with an
// integer atomicMax on the float bits (max is order-independent: deterministic).
__global__ void __launch_bounds__(256) colmax_kernel(int m, const float* __restrict__ X,
                                                     long long ldx, unsigned int* cmax,
                                                     int* status, int col_base, int rows_per) {
  __shared__ float red[32];
  const int j = blockIdx.y;
  const long long r0 = (long long)blockIdx.x * rows_per;
  const long long r1 = min((long long)m, r0 + rows_per);
  const float* x = X + (long long)j * ldx;
  float mx = 0.f;
  bool bad = false;
  const bool vec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) && ((r0 & 3) == 0);
  long long i = r0;
  if (vec) {
    for (long long q = r0 + threadIdx.x * 4; q + 3 < r1; q += 256 * 4) {
      const float4 v = *reinterpret_cast<const float4*>(x + q);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    i = r0 + ((r1 - r0) & ~3LL);
  }
  for (long long q = i + threadIdx.x; q < r1; q += 256) {
    const float v = x[q];
    mx = fmaxf(mx, fabsf(v));
    bad |= !isfinite(v);
  }
  if (bad && status) atomicMin(status, col_base + j + 1);
  mx = block_max(mx, red);
  if (threadIdx.x == 0 && mx > 0.f) atomicMax(cmax + j, __float_as_uint(mx));
}

// Pass 2: scaled RNE cast of a (row chunk, column) tile; inv_s written by chunk 0.
__global__ void __launch_bounds__(256) cast_pass2_kernel(int m, const float* __restrict__ X,
                                                         long long ldx, __half* __restrict__ Xh,
                                                         long long ldh,
                                                         const unsigned int* __restrict__ cmax,
                                                         float* __restrict__ inv_s, int scaling,
                                                         int rows_per) {
  const int j = blockIdx.y;
  const long long r0 = (long long)blockIdx.x * rows_per;
  const long long r1 = min((long long)m, r0 + rows_per);
  const float s = scaling ? pow2_scale_for(__uint_as_float(cmax[j])) : 1.f;
  if (blockIdx.x == 0 && threadIdx.x == 0 && inv_s) inv_s[j] = 1.f / s;
  const float* x = X + (long long)j * ldx;
  __half* xh = Xh + (long long)j * ldh;
  const bool vec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                   ((ldh & 3) == 0) && ((reinterpret_cast<uintptr_t>(Xh) & 7) == 0) &&
                   ((r0 & 3) == 0);
  long long i = r0;
  if (vec) {
    for (long long q = r0 + threadIdx.x * 4; q + 3 < r1; q += 256 * 4) {
      const float4 v = *reinterpret_cast<const float4*>(x + q);
      __half2 lo = __floats2half2_rn(v.x * s, v.y * s);
      __half2 hi = __floats2half2_rn(v.z * s, v.w * s);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      if (g_cast_ef)
        __stcs(reinterpret_cast<uint2*>(xh + q), pk);
      else
        *reinterpret_cast<uint2*>(xh + q) = pk;
    }
    i = r0 + ((r1 - r0) & ~3LL);
  }
  for (long long q = i + threadIdx.x; q < r1; q += 256) xh[q] = __float2half_rn(x[q] * s);
}

// Few columns x many rows, fused: one thread-block cluster per column, CTA r of the cluster owns
// rows [r * RPC, (r + 1) * RPC) with its 4 * V rows per thread held in registers.  Pass 1 (max |x|
// and non-finite detection) reads HBM once; the per-CTA maxima meet through distributed shared
// memory (max is order-independent: the same s as the two-kernel path, bit for bit); pass 2 casts
// from the registers.  One launch and one read of X instead of memset + colmax + cast_pass2.
template <int V>
__global__ void __launch_bounds__(256) cast_cluster_kernel(int m, const float* X, long long ldx,
                                                           __half* __restrict__ Xh,
                                                           long long ldh, float* __restrict__ inv_s,
                                                           int scaling, int* status, int col_base,
                                                           const float* __restrict__ src,
                                                           long long lds) {
  namespace cg = cooperative_groups;
  constexpr int RPC = 256 * 4 * V;  // rows per CTA
  __shared__ float red[32];
  __shared__ float cmv[8];  // cmv[r] = max |x| over CTA r's rows, pushed by CTA r
  cg::cluster_group cluster = cg::this_cluster();
  const int j = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const long long r0 = (long long)rank * RPC;
  // copy-cast (src non-null): the column is read from the factorization's input and its FP32
  // copy written to X on the way (the first touch of these columns: no separate copy pass)
  const float* x = src ? src + (long long)j * lds : X + (long long)j * ldx;
  float* xc = src ? const_cast<float*>(X) + (long long)j * ldx : nullptr;
  // every CTA of the cluster must be running before any CTA touches a peer's shared memory: a
  // relaxed arrive now, the matching wait just before the distributed stores (it overlaps the
  // HBM loads below)
  if (scaling) cluster.barrier_arrive();
  float4 v[V];
  float mx = 0.f;
  bool bad = false;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long q = r0 + 4LL * (threadIdx.x + 256 * u);
    if (q + 3 < m) {
      v[u] = g_cast_ef ? __ldcs(reinterpret_cast<const float4*>(x + q))
                       : *reinterpret_cast<const float4*>(x + q);
    } else {
      v[u].x = q < m ? x[q] : 0.f;
      v[u].y = q + 1 < m ? x[q + 1] : 0.f;
      v[u].z = q + 2 < m ? x[q + 2] : 0.f;
      v[u].w = q + 3 < m ? x[q + 3] : 0.f;
    }
  }
  if (xc) {
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const long long q = r0 + 4LL * (threadIdx.x + 256 * u);
      if (q + 3 < m) {
        if (g_cast_ef)
          __stcs(reinterpret_cast<float4*>(xc + q), v[u]);
        else
          *reinterpret_cast<float4*>(xc + q) = v[u];
      } else {
        if (q < m) xc[q] = v[u].x;
        if (q + 1 < m) xc[q + 1] = v[u].y;
        if (q + 2 < m) xc[q + 2] = v[u].z;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < V; ++u) {
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[u].x), fabsf(v[u].y)), fmaxf(fabsf(v[u].z), fabsf(v[u].w))));
    bad |= !(isfinite(v[u].x) && isfinite(v[u].y) && isfinite(v[u].z) && isfinite(v[u].w));
  }
  if (bad && status) atomicMin(status, col_base + j + 1);
  float s = 1.f;
  if (scaling) {
    mx = block_max(mx, red);
    const int nblk = (int)cluster.num_blocks();
    // push this CTA's max into every peer's slot (all peers are running: the entry arrive /
    // this wait); after the cluster barrier (release / acquire) each CTA reads only its own
    // shared memory, so no further barrier keeps peers alive
    cluster.barrier_wait();
    if ((int)threadIdx.x < nblk) *cluster.map_shared_rank(&cmv[rank], (int)threadIdx.x) = mx;
    cluster.sync();
    float g = 0.f;
    for (int r = 0; r < nblk; ++r) g = fmaxf(g, cmv[r]);
    s = pow2_scale_for(g);
  }
  if (rank == 0 && threadIdx.x == 0 && inv_s) inv_s[j] = 1.f / s;
  __half* xh = Xh + (long long)j * ldh;
#pragma unroll
  for (int u = 0; u < V; ++u) {
    const long long q = r0 + 4LL * (threadIdx.x + 256 * u);
    if (q + 3 < m) {
      __half2 lo = __floats2half2_rn(v[u].x * s, v[u].y * s);
      __half2 hi = __floats2half2_rn(v[u].z * s, v[u].w * s);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      if (g_cast_ef)
        __stcs(reinterpret_cast<uint2*>(xh + q), pk);
      else
        *reinterpret_cast<uint2*>(xh + q) = pk;
    } else {
      if (q < m) xh[q] = __float2half_rn(v[u].x * s);
      if (q + 1 < m) xh[q + 1] = __float2half_rn(v[u].y * s);
      if (q + 2 < m) xh[q + 2] = __float2half_rn(v[u].z * s);
    }
  }
}

template <int V>
static cudaError_t launch_cast_cluster(int m, int w, const float* X, long long ldx, __half* Xh,
                                       long long ldh, float* inv_s, int scaling, int* status,
                                       int col_base, int nchunks, cudaStream_t st,
                                       const float* src, long long lds) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nchunks, w);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nchunks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, cast_cluster_kernel<V>, m, X, ldx, Xh, ldh, inv_s, scaling, status,
                            col_base, src, lds);
}

cudaError_t cast_scale(int m, int w, const float* X, long long ldx, __half* Xh, long long ldh,
                       float* inv_s, int scaling, int* status, int col_base, unsigned int* cmax,
                       cudaStream_t st, const float* src, long long lds) {
  if (m <= 0 || w <= 0) return cudaSuccess;
  if (src == X && lds == ldx) src = nullptr;  // in place: nothing to copy
  // Range guard with m <= 65536 (every config's local height): the cluster kernel at any width
  // (one HBM read; at config 3 it beat the per-column two-pass kernel for w >= 1024 as well:
  // K1 3.81 -> 3.57 ms per factor, profiles/r01_bench_cfg3_v14_*).  Otherwise few columns x many
  // rows: split rows (2-D grid, pass 1 = column max via atomicMax); many columns: one CTA per
  // column (two passes over the column).
  static int use_cluster = -1;  // env TCQR_CAST_CLUSTER=0: the paths below
  if (use_cluster < 0) {
    const char* ev = getenv("TCQR_CAST_CLUSTER");
    use_cluster = ev ? atoi(ev) : 1;
  }
  const bool vec = ((ldx & 3) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0) &&
                   ((ldh & 3) == 0) && ((reinterpret_cast<uintptr_t>(Xh) & 7) == 0) &&
                   (!src || (((lds & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)));
  static bool ef_done = false;
  if (!ef_done) {
    ef_done = true;
    const char* e = getenv("TCQR_L2_EF");
    const int v = (e ? atoi(e) : 1) & 1;
    if (v != 1) cudaMemcpyToSymbol(g_cast_ef, &v, sizeof(int));
  }
  if (use_cluster && vec && (scaling || status) && m <= 8 * 8192) {
    // 8192-row CTAs (8 float4 loads in flight per thread) by default: at config 3 K1 3.03 ->
    // 2.76 ms against 4096-row CTAs (profiles/r01_bench_cfg3_v19_*); env TCQR_CAST_V8=0 for those
    static int v8 = -1;
    if (v8 < 0) {
      const char* ev = getenv("TCQR_CAST_V8");
      v8 = ev ? atoi(ev) : 1;
    }
    if (m <= 8 * 4096 && !v8) return launch_cast_cluster<4>(m, w, X, ldx, Xh, ldh, inv_s, scaling, status,
                                                     col_base, (m + 4095) / 4096, st, src, lds);
    return launch_cast_cluster<8>(m, w, X, ldx, Xh, ldh, inv_s, scaling, status, col_base,
                                  (m + 8191) / 8192, st, src, lds);
  }
  if (src) {  // the other casts read X: copy first
    const cudaError_t e = cudaMemcpy2DAsync(const_cast<float*>(X), sizeof(float) * ldx, src,
                                            sizeof(float) * lds, sizeof(float) * m, w,
                                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  static int col_min = -1;  // per-column kernel from this width on (env TCQR_CAST_COL_MIN)
  if (col_min < 0) {
    const char* e = getenv("TCQR_CAST_COL_MIN");
    col_min = e ? atoi(e) : 1024;
  }
  if (w >= col_min || (!scaling && !status) || !cmax) {
    if (!scaling && !status) {
      const int rows_per = 8192;
      dim3 g((m + rows_per - 1) / rows_per, w);
      cast_pass2_kernel<<<g, 256, 0, st>>>(m, X, ldx, Xh, ldh, nullptr, inv_s, 0, rows_per);
      return cudaGetLastError();
    }
    cast_scale_kernel<<<w, kCastThreads, 0, st>>>(m, X, ldx, Xh, ldh, inv_s, scaling, status,
                                                   col_base);
    return cudaGetLastError();
  }
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(unsigned int) * w, st);
  if (e != cudaSuccess) return e;
  const int rows_per = 8192;
  dim3 g((m + rows_per - 1) / rows_per, w);
  colmax_kernel<<<g, 256, 0, st>>>(m, X, ldx, cmax, status, col_base, rows_per);
  cast_pass2_kernel<<<g, 256, 0, st>>>(m, X, ldx, Xh, ldh, cmax, inv_s, scaling, rows_per);
  return cudaGetLastError();
}

// One CTA per column j of R12: R block <- T (already unscaled), s'_j from the column max, R12h.
__global__ void __launch_bounds__(kCastThreads) r12_finalize_kernel(
    int h, const float* __restrict__ T, long long ldt, float* __restrict__ Rblk, long long ldr,
    __half* __restrict__ R12h, long long ldh2, float* __restrict__ inv_s2, int scaling) {
  __shared__ float red[32];
  const int j = blockIdx.x;
  const float* t = T + (long long)j * ldt;
  float* r = Rblk + (long long)j * ldr;
  float mx = 0.f;
  for (int i = threadIdx.x; i < h; i += kCastThreads) {
    const float v = t[i];
    if (r != t) r[i] = v;
    mx = fmaxf(mx, fabsf(v));
  }
  float s = 1.f;
  if (scaling) {
    mx = block_max(mx, red);
    s = pow2_scale_for(mx);
  }
  if (threadIdx.x == 0) inv_s2[j] = 1.f / s;
  if (R12h) {
    __half* o = R12h + (long long)j * ldh2;
    for (int i = threadIdx.x; i < h; i += kCastThreads) o[i] = __float2half_rn(t[i] * s);
  }
}

// Split-K reduction fused with the finalize: column j of R12 = (sum_s P[s](:, j)) * col_mult[j]
// (partials summed in the fixed order s = 0..splits-1), written to the R block, then the column
// scale s' and the scaled FP16 copy as in r12_finalize_kernel.
// Split-K finalize, one CTA (kFinThreads) per column j: R12(i, j) = col_mult(j) * sum_s P_s(i, j)
// in a fixed order (deterministic).  Thread t sums entry i = t mod hb over the split group
// g = t / hb (splits g, g + G, ..., 16 loads in flight), then the G group sums are added in group
// order through shared memory.  With G > 1 the short deep-level columns (h = 128, 64 splits) keep
// 512 threads busy instead of 128 threads with 64 dependent L2 rounds (10 us -> see DESIGN).
constexpr int kFinThreads = 512;

__global__ void __launch_bounds__(kFinThreads) r12_splitk_finalize_kernel(
    int h, const float* __restrict__ P, int splits, long long pstride, long long ldp,
    const float* __restrict__ col_mult, float* __restrict__ Rblk, long long ldr,
    __half* __restrict__ R12h, long long ldh2, float* __restrict__ inv_s2, int scaling) {
  __shared__ float red[32];
  __shared__ float gs[kFinThreads];
  const int j = blockIdx.x;
  const float cm = col_mult ? col_mult[j] : 1.f;
  float* r = Rblk + (long long)j * ldr;
  float mx = 0.f;
  // hb = entries per pass (a power of two >= 32 dividing kFinThreads), G = split groups
  int hb = 32;
  while (hb < h && hb < kFinThreads) hb <<= 1;
  const int G = kFinThreads / hb;
  const int ii = threadIdx.x % hb, g = threadIdx.x / hb;
  for (int i0 = 0; i0 < h; i0 += hb) {
    const int i = i0 + ii;
    float acc = 0.f;
    if (i < h) {
      const float* p = P + i + (long long)j * ldp;
      int s0 = g;
      for (; s0 + 15 * G < splits; s0 += 16 * G) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcg(p + (long long)(s0 + u * G) * pstride);
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
      }
      for (; s0 < splits; s0 += G) acc += __ldcg(p + (long long)s0 * pstride);
    }
    if (G > 1) {
      gs[threadIdx.x] = acc;
      __syncthreads();
      if (g == 0) {
#pragma unroll 1
        for (int q = 1; q < G; ++q) acc += gs[q * hb + ii];
      }
      __syncthreads();
    }
    if (g == 0 && i < h) {
      const float v = acc * cm;
      r[i] = v;
      mx = fmaxf(mx, fabsf(v));
    }
  }
  float sc = 1.f;
  if (scaling) {
    mx = block_max(mx, red);
    sc = pow2_scale_for(mx);
  }
  if (threadIdx.x == 0) inv_s2[j] = 1.f / sc;
  if (R12h) {
    __syncthreads();  // r[] written by group 0 (global memory, same CTA)
    __half* o = R12h + (long long)j * ldh2;
    for (int i = threadIdx.x; i < h; i += kFinThreads) o[i] = __float2half_rn(__ldcg(r + i) * sc);
  }
}

// NEXT-4 (error-compensated FP16 split; the paper's related-work pointer on
// tensor-core precision): the low half of the FP16 split of X diag(s),
// Xl = fl16(X diag(s) - Xh) with Xh = fl16(X diag(s)) already written.  X diag(s) is exact (s is a
// power of two) and so is its difference with Xh in FP32, so Xl carries the next 11 bits (FP16
// subnormals below 2^-14: absolute error <= 2^-25 against a column max in [1, 2)).  inv_s null:
// s = 1.  One CTA per (row chunk, column); 4 elements per thread step.
__global__ void __launch_bounds__(256) cast_lo_kernel(int m, const float* __restrict__ X,
                                                      long long ldx,
                                                      const __half* __restrict__ Xh,
                                                      long long ldh, const float* __restrict__ inv_s,
                                                      __half* __restrict__ Xl, long long ldl,
                                                      int rows_per) {
  const int j = blockIdx.y;
  const long long r0 = (long long)blockIdx.x * rows_per;
  const long long r1 = min((long long)m, r0 + rows_per);
  const float s = inv_s ? 1.f / inv_s[j] : 1.f;
  const float* x = X + (long long)j * ldx;
  const __half* xh = Xh + (long long)j * ldh;
  __half* xl = Xl + (long long)j * ldl;
  for (long long q = r0 + threadIdx.x; q < r1; q += 256) {
    const float v = x[q] * s;
    xl[q] = __float2half_rn(v - __half2float(xh[q]));
  }
}

cudaError_t cast_lo(int m, int w, const float* X, long long ldx, const __half* Xh, long long ldh,
                    const float* inv_s, __half* Xl, long long ldl, cudaStream_t st) {
  if (m <= 0 || w <= 0) return cudaSuccess;
  const int rows_per = 8192;
  dim3 grid((m + rows_per - 1) / rows_per, w);
  cast_lo_kernel<<<grid, 256, 0, st>>>(m, X, ldx, Xh, ldh, inv_s, Xl, ldl, rows_per);
  return cudaGetLastError();
}

// dst[i] += a[i] + b[i] (NEXT-4: the three split products of R12 summed before the finalize;
// the small corrections are added together first).
__global__ void add3_kernel(long long n, float* __restrict__ dst, const float* __restrict__ a,
                            const float* __restrict__ b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = dst[i] + (a[i] + b[i]);
}

cudaError_t add3(long long n, float* dst, const float* a, const float* b, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  long long g = (n + 255) / 256;
  if (g > 4096) g = 4096;
  add3_kernel<<<(int)g, 256, 0, st>>>(n, dst, a, b);
  return cudaGetLastError();
}

cudaError_t r12_splitk_finalize(int h, int w2, const float* P, int splits, long long pstride,
                                long long ldp, const float* col_mult, float* Rblk, long long ldr,
                                __half* R12h, long long ldh2, float* inv_s2, int scaling,
                                cudaStream_t st) {
  if (h <= 0 || w2 <= 0) return cudaSuccess;
  r12_splitk_finalize_kernel<<<w2, kFinThreads, 0, st>>>(h, P, splits, pstride, ldp, col_mult,
                                                          Rblk, ldr, R12h, ldh2, inv_s2, scaling);
  return cudaGetLastError();
}

cudaError_t r12_finalize(int h, int w2, const float* T, long long ldt, float* Rblk, long long ldr,
                         __half* R12h, long long ldh2, float* inv_s2, int scaling,
                         cudaStream_t st) {
  if (h <= 0 || w2 <= 0) return cudaSuccess;
  r12_finalize_kernel<<<w2, kCastThreads, 0, st>>>(h, T, ldt, Rblk, ldr, R12h, ldh2, inv_s2,
                                                    scaling);
  return cudaGetLastError();
}

__global__ void copy_validate_kernel(int m, const float* __restrict__ A, long long lda,
                                     float* __restrict__ Q, long long ldq, int* status, int col0) {
  const int j = blockIdx.y;
  const float* a = A + (long long)j * lda;
  float* q = Q + (long long)j * ldq;
  bool bad = false;
  const bool inplace = q == a;
  int i0 = 0;
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(q)) & 15) == 0) {
    // 16-byte path: four independent float4 loads in flight per thread (the scalar loop ran at
    // ~3.1 TB/s of the 6.5 measured copy bandwidth at config 3)
    const int m4 = m >> 2, stride = gridDim.x * blockDim.x;
    const float4* a4 = reinterpret_cast<const float4*>(a);
    float4* q4 = reinterpret_cast<float4*>(q);
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < m4; i += 4 * stride) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(a4 + i + u * stride);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        bad |= !isfinite(v[u].x) || !isfinite(v[u].y) || !isfinite(v[u].z) || !isfinite(v[u].w);
        if (!inplace) q4[i + u * stride] = v[u];
      }
    }
    for (; i < m4; i += stride) {
      const float4 v = __ldcs(a4 + i);
      bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
      if (!inplace) q4[i] = v;
    }
    i0 = m4 << 2;
  }
  for (int i = i0 + blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const float v = a[i];
    bad |= !isfinite(v);
    if (!inplace) q[i] = v;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicMin(status, col0 + j + 1);
}

cudaError_t copy_validate(int m, int n, const float* A, long long lda, float* Q, long long ldq,
                          int* status, cudaStream_t st, int col0) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  int gx = (m + 4095) / 4096;  // ~4 float4 per thread
  if (gx > 64) gx = 64;
  dim3 grid(gx, n);
  copy_validate_kernel<<<grid, 256, 0, st>>>(m, A, lda, Q, ldq, status, col0);
  return cudaGetLastError();
}

__global__ void copy_block_kernel(int h, int w, const float* __restrict__ S, long long lds,
                                  float* __restrict__ D, long long ldd) {
  const long long total = (long long)h * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % h), j = (int)(e / h);
    D[i + j * ldd] = S[i + j * lds];
  }
}

cudaError_t copy_block(int h, int w, const float* S, long long lds, float* D, long long ldd,
                       cudaStream_t st) {
  if (h <= 0 || w <= 0) return cudaSuccess;
  long long total = (long long)h * w;
  int grid = (int)((total + 255) / 256);
  if (grid > 1184) grid = 1184;
  copy_block_kernel<<<grid, 256, 0, st>>>(h, w, S, lds, D, ldd);
  return cudaGetLastError();
}

__global__ void zero_lower_kernel(int n, float* R, long long ldr) {
  const int j = blockIdx.x;
  for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) R[i + (long long)j * ldr] = 0.f;
}

cudaError_t zero_lower(int n, float* R, long long ldr, cudaStream_t st) {
  if (n <= 1) return cudaSuccess;
  zero_lower_kernel<<<n, 256, 0, st>>>(n, R, ldr);
  return cudaGetLastError();
}

// C = A * B for upper-triangular n x n FP32 A, B (column-major, leading dims lda/ldb/ldc): the
// re-orthogonalized R = R2 * R1 (NEXT-1).  64 x 64 tiles, 4 x 4 per thread,
// only upper tiles; the k range of tile (I, J) is [I*64, (J+1)*64) (zeros elsewhere).
__global__ void __launch_bounds__(256) trmm_upper_kernel(int n, const float* __restrict__ A,
                                                         long long lda, const float* __restrict__ B,
                                                         long long ldb, float* __restrict__ C,
                                                         long long ldc) {
  __shared__ float As[16][65];
  __shared__ float Bs[16][65];
  const int tI = blockIdx.x, tJ = blockIdx.y;
  const int tid = threadIdx.x, ti = tid & 15, tj = tid >> 4;
  const int i0 = tI * 64, j0 = tJ * 64;
  if (tI > tJ) {
    for (int e = tid; e < 64 * 64; e += 256) {
      const int r = i0 + (e & 63), c = j0 + (e >> 6);
      if (r < n && c < n) C[r + (long long)c * ldc] = 0.f;
    }
    return;
  }
  float acc[4][4] = {};
  const int k_end = min(n, j0 + 64);
  for (int k0 = i0; k0 < k_end; k0 += 16) {
    __syncthreads();
    for (int e = tid; e < 16 * 64; e += 256) {
      const int kk = e >> 6, mm = e & 63;
      const int k = k0 + kk;
      As[kk][mm] = (i0 + mm < n && k < k_end) ? A[(i0 + mm) + (long long)k * lda] : 0.f;
      Bs[kk][mm] = (j0 + mm < n && k < k_end) ? B[k + (long long)(j0 + mm) * ldb] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = As[kk][ti * 4 + x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = Bs[kk][tj * 4 + y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(a[x], b[y], acc[x][y]);
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int r = i0 + ti * 4 + x, c = j0 + tj * 4 + y;
      if (r < n && c < n) C[r + (long long)c * ldc] = acc[x][y];
    }
}

// 128 x 128 tiles, 8 x 8 register micro-tiles, register-prefetched double-buffered K-chunks.
__global__ void __launch_bounds__(256, 1) trmm_upper_big(int n, const float* __restrict__ A,
                                                         long long lda, const float* __restrict__ B,
                                                         long long ldb, float* __restrict__ C,
                                                         long long ldc) {
  constexpr int TB = 128, KB = 16, NLD = KB * TB / 256;
  __shared__ __align__(16) float As[2][KB][TB];
  __shared__ __align__(16) float Bs[2][KB][TB];
  const int tI = blockIdx.x, tJ = blockIdx.y;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = tI * TB, j0 = tJ * TB;
  if (tI > tJ) {
    for (int e = tid; e < TB * TB; e += 256) {
      const int r = i0 + (e & (TB - 1)), c = j0 + e / TB;
      if (r < n && c < n) C[r + (long long)c * ldc] = 0.f;
    }
    return;
  }
  const int kbeg = i0, kend = min(n, j0 + TB);
  auto load = [&](int k0, float (&ra)[NLD], float (&rb)[NLD]) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      const int k = k0 + kk;
      ra[u] = (i0 + mm < n && k < kend) ? __ldg(A + (i0 + mm) + (long long)k * lda) : 0.f;
      rb[u] = (j0 + mm < n && k < kend) ? __ldg(B + k + (long long)(j0 + mm) * ldb) : 0.f;
    }
  };
  float2 acc[8][4];  // acc[x][y2] = columns (2 y2, 2 y2 + 1) of row x: FFMA2, the same fmaf per entry
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = make_float2(0.f, 0.f);
  float ra[NLD], rb[NLD];
  int buf = 0;
  load(kbeg, ra, rb);
  for (int k0 = kbeg; k0 < kend; k0 += KB) {
#pragma unroll
    for (int u = 0; u < NLD; ++u) {
      const int e = tid + u * 256, kk = e >> 7, mm = e & 127;
      As[buf][kk][mm] = ra[u];
      Bs[buf][kk][mm] = rb[u];
    }
    __syncthreads();
    if (k0 + KB < kend) load(k0 + KB, ra, rb);
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tx * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][tx * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][ty * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][ty * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float2 bb[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w),
                            make_float2(b1.x, b1.y), make_float2(b1.z, b1.w)};
#pragma unroll
      for (int x = 0; x < 8; ++x) {
        const float2 ax = make_float2(a[x], a[x]);
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = ffma2(ax, bb[y], acc[x][y]);
      }
    }
    buf ^= 1;
  }
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < 8; ++y) {
      const int r = i0 + tx * 8 + x, c = j0 + ty * 8 + y;
      if (r < n && c < n) C[r + (long long)c * ldc] = (y & 1) ? acc[x][y >> 1].y : acc[x][y >> 1].x;
    }
}

// X <- I - X (n x n, column-major): NEXT-1's R2 turned into the small correction I - R2 of
// R2 R1 = R1 - (I - R2) R1 (the tensor-core form of the product, tcqr.cu reorth_product_tc).
__global__ void eye_minus_kernel(int n, float* __restrict__ X, long long ldx) {
  const long long total = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % n), j = (int)(e / n);
    float* p = X + i + (long long)j * ldx;
    *p = (i == j ? 1.f : 0.f) - *p;
  }
}

cudaError_t eye_minus(int n, float* X, long long ldx, cudaStream_t st) {
  const long long total = (long long)n * n;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  eye_minus_kernel<<<std::max(grid, 1), 256, 0, st>>>(n, X, ldx);
  return cudaGetLastError();
}

cudaError_t trmm_upper(int n, const float* A, long long lda, const float* B, long long ldb,
                       float* C, long long ldc, cudaStream_t st) {
  if (n >= 512) {
    const int t = (n + 127) / 128;
    trmm_upper_big<<<dim3(t, t), 256, 0, st>>>(n, A, lda, B, ldb, C, ldc);
  } else {
    const int t = (n + 63) / 64;
    trmm_upper_kernel<<<dim3(t, t), 256, 0, st>>>(n, A, lda, B, ldb, C, ldc);
  }
  return cudaGetLastError();
}

}  // namespace tcqr

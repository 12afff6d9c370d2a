// k_panels.cu -- K2S: the Eq. (6) CAQR panel for panels too tall for the
// pipelined / whole-leaf kernels (m > 32768 rows: config 5 at one GPU, the 4194304 x 128
// orthogonalization of NEXT-3), in ONE cooperative launch with the rows streamed from L2 / HBM.
//
//   (1) Alg. 4 (MGS) on 64-row blocks, ONE WARP per block (two rows per lane,
//       warp-shuffle reductions, no CTA barrier on the 32-step chain): every warp of the grid
//       walks its blocks b = warp_id, warp_id + W, ...; Q_b is written back in place (FP32), R_b
//       to a scratch stack, and the warp accumulates the stack's Gram G_w += R_b' R_b in FP64.
//       64 = 4^3 rows keeps the planted pin exact (reading R-A6); any blocking gives the same
//       factors in exact arithmetic (Eq. (6)).
//   (2)-(3) the stack [R_1; ...; R_nblk] factored through its Gram (reading R-A28): the warp Grams
//       are summed per CTA in warp order, then across CTAs in a fixed order (grid barriers), every
//       CTA factors R = chol(G) redundantly (warp 0, FP64) together with R^-1 (forward
//       substitution of the identity rows).
//   (4) Q_b <- Q_b S_b with S_b = R_b R^-1 (FP64 products, rounded to FP32), FP32 Q and its FP16
//       shadow written.
// Two grid barriers per panel; deterministic (fixed block ownership and summation order).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace tcqr {

namespace {

constexpr int kSNT = 256;          // threads per CTA
constexpr int kSW = kSNT / 32;     // warps per CTA
constexpr int kBR = 64;            // rows per CAQR block (one warp, two rows per lane)

struct PanelSArgs {
  float* X;  // panel column j at X + j * ldx, m rows
  long long ldx;
  __half* Xh;  // FP16 shadow of the final Q (nullable), ld ldh
  long long ldh;
  float* R;  // the panel's R (pw x pw) at R[i + j * ldr]
  long long ldr;
  int m, pw, nblk;
  float* Rbs;     // nblk x 1024: R_b row-major
  double* gpart;  // gridDim x 1024
  double* gsum;   // 1024
  unsigned* bar;  // grid barrier counter (monotonic arrivals)
  unsigned bar_base;  // arrivals before this launch (the host counts them)
  int* status;
  int col0;
};

struct SmemS {
  double Gw[kSW][1024];    // per-warp Gram (upper triangle used), then scratch
  double Rd[32 * 34 + 34]; // R (FP64, row-major, ld 34)
  double Ri[32 * 32];      // R^-1 (FP64, row-major)
  float Rw[kSW][32 * 33];  // per-warp R_b / S_b (row-major, ld 33)
  unsigned barseq;
};

__device__ __forceinline__ void grid_bar(const PanelSArgs& a, SmemS& s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = a.bar_base + (++s.barseq) * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    } while (v < target);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ int blk_row(int b, int m, int nblk) {
  return (int)((long long)b * m / nblk);
}

// Lane l ends with the warp sum of v[l % W].
template <int W>
__device__ __forceinline__ float wsum_tr(float (&v)[32]) {
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

// One warp-level MGS step k (Alg. 4 lines 3-7) with reduction width W >= active columns:
// x[r][j] holds column k + j of row (lane + 32 r); R(k, k + j) -> Rw[k * 33 + k + j]; q -> qcol.
template <int W>
__device__ __forceinline__ void mgs_wstep(float (&x)[2][32], int w, int k, float* Rw,
                                          float* const (&qrow)[2], long long ldx) {
  const int lane = threadIdx.x & 31;
  float p[32];
#pragma unroll
  for (int j = 0; j < W; ++j) p[j] = fmaf(x[0][0], x[0][j], x[1][0] * x[1][j]);
  const float tot = wsum_tr<W>(p);  // lane l: a_k' a_{k + l % W}
  const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, 0));
  // a locally zero column (R-A8): q = 0, r = 0; only the global (stack) factorization may fail
  const bool zero = !(rkk > 0.f) || !isfinite(rkk);
  const float inv = zero ? 0.f : __frcp_rn(rkk);
  const int jl = lane & (W - 1);
  const float rkj = zero ? 0.f : (jl == 0 ? rkk : tot * inv);
  if (lane < W && lane < w - k) Rw[k * 33 + k + lane] = rkj;
  float q[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    q[r] = x[r][0] * inv;
    if (qrow[r]) qrow[r][(long long)k * ldx] = q[r];
  }
#pragma unroll
  for (int j = 1; j < W; ++j) {
    const float rj = __shfl_sync(0xffffffffu, rkj, j);
#pragma unroll
    for (int r = 0; r < 2; ++r) x[r][j - 1] = fmaf(-q[r], rj, x[r][j]);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) x[r][W - 1] = 0.f;
}

__device__ __forceinline__ void mgs_wstep_any(float (&x)[2][32], int w, int k, float* Rw,
                                              float* const (&qrow)[2], long long ldx) {
  const int act = w - k;
  if (act > 16)
    mgs_wstep<32>(x, w, k, Rw, qrow, ldx);
  else if (act > 8)
    mgs_wstep<16>(x, w, k, Rw, qrow, ldx);
  else if (act > 4)
    mgs_wstep<8>(x, w, k, Rw, qrow, ldx);
  else if (act > 2)
    mgs_wstep<4>(x, w, k, Rw, qrow, ldx);
  else if (act > 1)
    mgs_wstep<2>(x, w, k, Rw, qrow, ldx);
  else
    mgs_wstep<1>(x, w, k, Rw, qrow, ldx);
}

__global__ void __launch_bounds__(kSNT, 1) panels_kernel(const __grid_constant__ PanelSArgs a) {
  extern __shared__ __align__(16) unsigned char pans_smem[];
  SmemS& s = *reinterpret_cast<SmemS*>(pans_smem);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int pw = a.pw;
  const int gw = blockIdx.x * kSW + warp, nw = gridDim.x * kSW;
  if (t == 0) s.barseq = 0;
  float* Rw = s.Rw[warp];
  // ---- (1) per-warp block MGS, R_b to the stack, Gram accumulated in FP64 ----
  double g[32];  // lane j: G_w(i, j), i <= j
#pragma unroll
  for (int i = 0; i < 32; ++i) g[i] = 0.0;
  // the block's rows are loaded one block ahead: the next block's loads are issued right after
  // this block's MGS and overlap its R_b store and Gram update
  float x[2][32];
  auto load_block = [&](int b) {
    const int r0 = blk_row(b, a.m, a.nblk), nr = blk_row(b + 1, a.m, a.nblk) - r0;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = lane + 32 * r;
      const bool ok = row < nr;
      const float* src = a.X + r0 + (ok ? row : 0);
#pragma unroll
      for (int j = 0; j < 32; ++j) x[r][j] = (ok && j < pw) ? __ldcg(src + (long long)j * a.ldx) : 0.f;
    }
  };
  if (gw < a.nblk) load_block(gw);
  for (int b = gw; b < a.nblk; b += nw) {
    const int r0 = blk_row(b, a.m, a.nblk), nr = blk_row(b + 1, a.m, a.nblk) - r0;
    float* qrow[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) qrow[r] = (lane + 32 * r) < nr ? a.X + r0 + lane + 32 * r : nullptr;
    for (int e = lane; e < 32 * 33; e += 32) Rw[e] = 0.f;
    __syncwarp();
    for (int k = 0; k < pw; ++k) mgs_wstep_any(x, pw, k, Rw, qrow, a.ldx);
    __syncwarp();
    if (b + nw < a.nblk) load_block(b + nw);
    // R_b to the stack (row-major 32 x 32) and G_w += R_b' R_b (lane j = column j)
    float* dst = a.Rbs + (long long)b * 1024;
#pragma unroll 4
    for (int i = 0; i < 32; ++i) dst[i * 32 + lane] = Rw[i * 33 + lane];
    // widen R_b to FP64 once (the warp's Gw slot is free until the end of the block loop)
    double* rd = s.Gw[warp];
#pragma unroll 4
    for (int i = 0; i < 32; ++i) rd[i * 32 + lane] = (double)Rw[i * 33 + lane];
    __syncwarp();
#pragma unroll 1
    for (int l = 0; l < pw; ++l) {
      const double rlj = rd[l * 32 + lane];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i >= l) g[i] = fma(rd[l * 32 + i], rlj, g[i]);
    }
    __syncwarp();
  }
  // CTA sum of the warp Grams in warp order -> this CTA's partial
#pragma unroll
  for (int i = 0; i < 32; ++i) s.Gw[warp][i * 32 + lane] = (i <= lane) ? g[i] : 0.0;
  __syncthreads();
  for (int e = t; e < 1024; e += kSNT) {
    double v = s.Gw[0][e];
#pragma unroll
    for (int w = 1; w < kSW; ++w) v += s.Gw[w][e];
    a.gpart[(long long)blockIdx.x * 1024 + e] = v;
  }
  grid_bar(a, s);
  // fixed-order cross-CTA sum: entry e (lane) of chunk c = blockIdx.x, ...; warp w sums CTAs
  // w, w + 8, ... in increasing order, then the 8 warp sums in warp order
  for (int c = blockIdx.x; c < 32; c += gridDim.x) {
    const int e = c * 32 + lane;
    double v = 0.0;
    for (int p = warp; p < (int)gridDim.x; p += kSW) v += __ldcg(a.gpart + (long long)p * 1024 + e);
    s.Gw[warp][e] = v;
    __syncthreads();
    if (warp == 0) {
      double tsum = s.Gw[0][e];
#pragma unroll
      for (int w = 1; w < kSW; ++w) tsum += s.Gw[w][e];
      a.gsum[e] = tsum;
    }
    __syncthreads();
  }
  grid_bar(a, s);
  // ---- (3) R = chol(G) and R^-1 (rows of the identity under forward substitution), warp 0 ----
  if (warp == 0) {
    double c[32], r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = (i <= lane && lane < pw) ? __ldcg(a.gsum + i * 32 + lane) : 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = (j == lane && lane < pw) ? 1.0 : 0.0;
    double d = __shfl_sync(0xffffffffu, c[0], 0);
    bool ok = d > 0.0 && d <= 1.7976931348623157e308;
    double ri = rsqrt_nr(ok ? d : 1.0);
#pragma unroll 1
    for (int k = 0; k < pw; ++k) {
      ri = ok ? ri : 0.0;
      const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
      s.Rd[k * 34 + lane] = rkj;
      if (!ok && lane == 0 && blockIdx.x == 0 && a.status) atomicMin(a.status, a.col0 + k + 1);
      const double sk = r[0] * ri;
      s.Ri[lane * 32 + k] = sk;  // R^-1(lane, k)
      __syncwarp();
      const double* rk = s.Rd + k * 34 + k + 1;
      const double v0 = rk[0];
      c[0] = fma(-v0, rkj, c[1]);
      r[0] = fma(-sk, v0, r[1]);
      d = __shfl_sync(0xffffffffu, c[0], (k + 1) & 31);
      ok = d > 0.0 && d <= 1.7976931348623157e308;
      ri = rsqrt_nr(ok ? d : 1.0);
#pragma unroll
      for (int i = 1; i < 31; ++i) {
        const double v = rk[i];
        c[i] = fma(-v, rkj, c[i + 1]);
        r[i] = fma(-sk, v, r[i + 1]);
      }
      c[31] = 0.0;
      r[31] = 0.0;
    }
#pragma unroll 1
    for (int j = pw; j < 32; ++j) s.Ri[lane * 32 + j] = 0.0;
  }
  __syncthreads();
  if (blockIdx.x == 0) {  // the panel's R block (upper triangle; the lower one stays zero)
    for (int e = t; e < pw * pw; e += kSNT) {
      const int i = e % pw, j = e / pw;
      if (i <= j) a.R[i + (long long)j * a.ldr] = (float)s.Rd[i * 34 + j];
    }
  }
  // ---- (4) Q_b <- Q_b S_b, S_b = R_b R^-1 ----
  for (int b = gw; b < a.nblk; b += nw) {
    const int r0 = blk_row(b, a.m, a.nblk), nr = blk_row(b + 1, a.m, a.nblk) - r0;
    {
      // lane i: row i of S_b = sum_l R_b(i, l) R^-1(l, :) (R_b upper: l >= i)
      const float4* rb = reinterpret_cast<const float4*>(a.Rbs + (long long)b * 1024 + lane * 32);
      float rrow[32];
#pragma unroll
      for (int q4 = 0; q4 < 8; ++q4) {
        const float4 v = __ldcg(rb + q4);
        rrow[4 * q4] = v.x;
        rrow[4 * q4 + 1] = v.y;
        rrow[4 * q4 + 2] = v.z;
        rrow[4 * q4 + 3] = v.w;
      }
      double sr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) sr[j] = 0.0;
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        if (l < pw) {
          const double ril = (double)rrow[l];
          const double* rinv = s.Ri + l * 32;
#pragma unroll
          for (int j = 0; j < 32; ++j) sr[j] = fma(ril, rinv[j], sr[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) Rw[lane * 33 + j] = (float)sr[j];
    }
    __syncwarp();
    float qa[2][32];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = lane + 32 * r;
      const float* src = a.X + r0 + (row < nr ? row : 0);
#pragma unroll
      for (int l = 0; l < 32; ++l) qa[r][l] = (l < pw && row < nr) ? __ldcg(src + (long long)l * a.ldx) : 0.f;
    }
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {
      const int row = lane + 32 * r;
      if (row < nr) {
        float* src = a.X + r0 + row;
        float q[32], y[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) q[l] = r == 0 ? qa[0][l] : qa[1][l];
#pragma unroll
        for (int j = 0; j < 32; ++j) y[j] = 0.f;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          if (l < pw) {
#pragma unroll
            for (int j = 0; j < 32; ++j) y[j] = fmaf(q[l], Rw[l * 33 + j], y[j]);
          }
        }
        __half* dh = a.Xh ? a.Xh + r0 + row : nullptr;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < pw) {
            src[(long long)j * a.ldx] = y[j];
            if (dh) dh[(long long)j * a.ldh] = __float2half_rn(y[j]);
          }
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace

size_t panels_scratch_floats(int m) { return (size_t)((m + kBR - 1) / kBR) * 1024; }

cudaError_t panel_stream(int m, int pw, float* X, long long ldx, __half* Xh, long long ldh,
                         float* R, long long ldr, int col0, int* status, float* Rbs,
                         size_t rbs_floats, void* scratch, size_t scratch_bytes, unsigned* bar,
                         unsigned* bar_seq, int num_sms, cudaStream_t st) {
  if (pw < 1 || pw > 32 || m < 2 * kBR) return cudaErrorNotSupported;
  const int nblk = (m + kBR - 1) / kBR;
  if ((size_t)nblk * 1024 > rbs_floats) return cudaErrorNotSupported;
  static int per_sm = -1;
  const int smem = (int)sizeof(SmemS);
  if (per_sm < 0) {
    cudaFuncSetAttribute(panels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panels_kernel, kSNT, smem) !=
        cudaSuccess)
      per_sm = 0;
  }
  int grid = per_sm * num_sms;
  const int need = (nblk + kSW - 1) / kSW;
  if (grid > need) grid = need;
  if (grid < 1) return cudaErrorNotSupported;
  if (scratch_bytes < sizeof(double) * ((size_t)grid * 1024 + 1024)) return cudaErrorNotSupported;
  PanelSArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.Xh = Xh;
  a.ldh = ldh;
  a.R = R;
  a.ldr = ldr;
  a.m = m;
  a.pw = pw;
  a.nblk = nblk;
  a.Rbs = Rbs;
  a.gpart = static_cast<double*>(scratch);
  a.gsum = a.gpart + (size_t)grid * 1024;
  a.bar = bar;
  a.bar_base = *bar_seq;
  a.status = status;
  a.col0 = col0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, panels_kernel, a);
  if (e == cudaSuccess) *bar_seq += 2u * (unsigned)grid;
  return e;
}

}  // namespace tcqr

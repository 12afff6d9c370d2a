// k_leaf.cu -- K2L: a whole leaf of Alg. 2 (w <= 128 columns, every node below the tensor-core
// cutoff) in ONE cooperative launch, one CTA per 256-row block, the block's rows of all the leaf's
// columns resident in shared memory from the first panel to the last.
//
// The leaf is the same recursion as Alg. 2: split h = 32 ceil(w/64) (R-A2),
// FP32 products below the cutoff (R-A1), 32-column CAQR panels (Eq. (6)).  The
// host flattens it into a short program of ops that the kernel runs in order:
//
//   PANEL(c0, pw)   Eq. (6) on columns [c0, c0+pw):
//     (1) every CTA runs Alg. 4 (MGS) on its 256 x pw block -- the paper's
//         256 x 32 submatrix with one row per thread -- Q_b in place in shared
//         memory, R_b (pw x pw) in shared memory;
//     (2)-(3) the stack [R_1; ...; R_nb] is factored through its Gram matrix in FP64:
//         G = sum_b R_b' R_b (each product exact in FP64, fixed-order sums), R = chol(G), and the
//         stack's Q slice of block b is S_b = R_b R^-1 (forward substitution, IEEE division).
//         This is a QR of the stacked R's (G = R'R, diag(R) > 0 -- the unique R of Eq. (6) step
//         (3)); reading R-B1 in DESIGN.md: the paper factors the stack with the same MGS kernel,
//         here the FP64 Gram route takes the 32-step dependency chain out of FP32 block
//         reductions (R is more accurate than the FP32 MGS R for kappa < ~1e7);
//     (4) Q_b <- Q_b S_b in shared memory.
//   PROJ(c0, h, w2) Alg. 2 lines 8-9 in FP32 below the cutoff: R12 = Q1' A2 (per-CTA partial over
//     its rows, fixed-order sum over the CTAs), R block <- R12, A2 -= Q1 R12.
//
// Cross-CTA steps (the Gram / R12 sums) go through L2 between grid barriers; every CTA computes
// the 32 x 32 Cholesky redundantly (same inputs, same code: bit-identical R everywhere), so a
// panel costs two grid barriers.  At the end each CTA writes its rows of the final Q (FP32 and the
// FP16 shadow the tensor-core GEMMs above read) and CTA 0 has written the leaf's R blocks.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "mgs.cuh"

namespace tcqr {

namespace {

constexpr int kNT = 256;      // threads per CTA; thread t owns row t of the block
constexpr int kRows = 256;    // rows per CTA (max)
constexpr int kCols = 128;    // leaf width (max)
constexpr int kLd = 132;      // shared row stride in floats: 16-byte rows, 4 floats of skew
constexpr int kMaxOps = 16;
constexpr int kNW = kNT / 32;

struct LeafOp {
  int kind;  // 0 panel (c0, h = width), 1 projection (c0, h, w2)
  int c0, h, w2;
};

struct LeafArgs {
  float* X;  // column c of the leaf at X + c * ldx (rows 0..m-1)
  long long ldx;
  __half* Xh;  // FP16 shadow of the final Q (nullable), ld ldh
  long long ldh;
  float* R;  // R(c0 + i, c0 + j) of the leaf at R[i + j * ldr]
  long long ldr;
  int m, wl, nb, nops;
  LeafOp ops[kMaxOps];
  double* gpart;  // nb x 1024 Gram partials
  double* gsum;   // 1024
  float* ppart;   // nb x 4096 projection partials
  float* r12;     // 4096
  unsigned* bar;  // grid barrier arrival counter (zeroed before the factorization's first leaf)
  unsigned bar_base;  // barriers completed before this launch (the host counts them)
  int* status;
  int col0;       // global column of the leaf's column 0 (breakdown codes)
  unsigned long long* dbg;  // optional phase timestamps of CTA 0 (globaltimer ns), 128 slots
  int mgs_rpt;    // rows per thread of the block MGS (2: 128 threads (default), 1: 256 threads)
};

struct Smem {
  float L[kRows * kLd];  // the block's rows of the leaf, row-major
  float Rb[32 * 32];     // R_b of the current panel, row-major
  float Sf[32 * 32];     // S_b (FP32), row-major [l][j]
  double Rd[32 * 34 + 34];  // the panel's R in FP64, row-major (ld 34; one row of slack)
  double Rbd[32 * 32];   // R_b widened to FP64, row-major
  float T[4096];         // R12 (row-major [i][w2p]) / projection group partials
  float red[2 * kNW * 32];
  float wsum[kNW * 32];  // per-warp partial sums of the cross-CTA reductions
  unsigned barseq;       // grid barriers passed by this CTA in this launch (thread 0)
};

// Grid barrier on a monotonic arrival counter: barrier i of this launch completes when the
// counter reaches (bar_base + i) * nb.  Fire-and-forget release arrival, relaxed polling, one
// acquire load at the end (the CTA barriers carry the ordering to the other threads).
__device__ __forceinline__ void leaf_barrier(const LeafArgs& a, Smem& s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (a.bar_base + (++s.barseq)) * (unsigned)a.nb;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
    } while (v < target);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ void leaf_ts(const LeafArgs& a, int& slot) {
  if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && slot < 128) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[slot] = v;
  }
  ++slot;
}

__device__ __forceinline__ int leaf_row(int b, int m, int nb) {
  return (int)((long long)b * m / nb);
}

// Fixed-order cross-CTA sum: out[e] = sum_{b=0..nb-1} part[b * pstride + e] for the entries
// e in [0, E) that belong to this CTA (chunks of 32 consecutive entries, chunk c on CTA c % nb).
// Lane = entry, warp w sums the partials b = w, w + 8, ... in increasing order, then the 8 warp
// sums are added in warp order.  Deterministic; reads bypass L1 (written by other CTAs).
template <typename T>
__device__ __forceinline__ void cross_sum(const T* part, long long pstride, int E, int nb,
                                          T* out, T* wsum, float* Rblk, long long ldr, int h,
                                          int w2, int w2p, int c0, bool to_r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunks = (E + 31) / 32;
  for (int c = blockIdx.x; c < nchunks; c += nb) {
    const int e = c * 32 + lane;
    T s = 0;
    if (e < E) {
      T v[4];
      int b = warp;
      for (; b + 3 * kNW < nb; b += 4 * kNW) {
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(part + (long long)(b + u * kNW) * pstride + e);
#pragma unroll
        for (int u = 0; u < 4; ++u) s += v[u];
      }
      for (; b < nb; b += kNW) s += __ldcg(part + (long long)b * pstride + e);
    }
    wsum[warp * 32 + lane] = s;
    __syncthreads();
    if (warp == 0 && e < E) {
      T t = wsum[lane];
#pragma unroll
      for (int u = 1; u < kNW; ++u) t += wsum[u * 32 + lane];
      out[e] = t;
      if (to_r) {  // projection: R(c0 + i, c0 + h + j) = R12(i, j)
        const int i = e / w2p, j = e % w2p;
        if (i < h && j < w2) Rblk[(c0 + i) + (long long)(c0 + h + j) * ldr] = (float)t;
      }
    }
    __syncthreads();
  }
}

// Alg. 4 on the block's rows of columns [c0, c0 + pw): thread t < kNT / RPT holds rows
// t + r kNT / RPT; Q_b in place in shared memory, R_b row-major into s.Rb.
template <int RPT>
__device__ __forceinline__ void mgs_block(Smem& s, int nrows, int c0, int pw) {
  constexpr int NT = kNT / RPT;
  const int t = threadIdx.x;
  if (t >= NT) return;
  float x[RPT][32];
  float* qp[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int row = t + r * NT;
    const float* src = s.L + row * kLd + c0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(src + 4 * q);
      x[r][4 * q] = v.x;
      x[r][4 * q + 1] = v.y;
      x[r][4 * q + 2] = v.z;
      x[r][4 * q + 3] = v.w;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j >= pw) x[r][j] = 0.f;
    qp[r] = row < nrows ? s.L + row * kLd + c0 : nullptr;
  }
  int buf = 0;
  for (int k = 0; k < pw; ++k)
    mgs_step_any<NT, RPT>(x, nrows, pw, k, qp, 1, s.Rb, 32, 1, false, nullptr, 0, s.red, buf);
}

// Columns [32, kCols) of block row r (zero-filled past the block and past the leaf): 4-byte
// cp.async down each column (a warp covers 32 consecutive rows), waited for by the first PROJ.
__device__ __forceinline__ void leaf_issue_rest(const LeafArgs& a, Smem& s, int nrows, int r) {
  const int row0 = leaf_row(blockIdx.x, a.m, a.nb);
  const float* src = a.X + row0 + min(r, nrows - 1);
  float* dst = s.L + r * kLd;
  const uint32_t sz = r < nrows ? 4u : 0u;  // 0: zero fill
#pragma unroll 8
  for (int j = 32; j < kCols; ++j) {
    if (j < a.wl) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst + j)),
                   "l"(src + (long long)j * a.ldx), "r"(sz)
                   : "memory");
    } else {
      dst[j] = 0.f;
    }
  }
}

// Row r of the block's final Q columns [c0, c0 + pw) to global (FP32 and the FP16 shadow).
__device__ __forceinline__ void leaf_store_row(const LeafArgs& a, const Smem& s, int r, int c0,
                                               int pw) {
  const int row0 = leaf_row(blockIdx.x, a.m, a.nb);
  const float* srcr = s.L + r * kLd + c0;
  float* dst = a.X + row0 + r + (long long)c0 * a.ldx;
  __half* dh = a.Xh ? a.Xh + row0 + r + (long long)c0 * a.ldh : nullptr;
#pragma unroll 8
  for (int j = 0; j < 32; ++j) {
    if (j < pw) {
      const float v = srcr[j];
      __stcg(dst + (long long)j * a.ldx, v);
      if (dh) dh[(long long)j * a.ldh] = __float2half_rn(v);
    }
  }
}

// ---- PANEL ------------------------------------------------------------------------------------
__device__ __noinline__ void leaf_panel(const LeafArgs& a, Smem& s, int nrows, int c0, int pw,
                                        int& slot, bool first, int st_c0, int st_pw, bool defer) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // first panel with the 128-thread MGS: the idle upper half issues the async loads of the leaf's
  // later columns (two rows per thread) beside the MGS instead of before it
  if (first && a.mgs_rpt == 2 && t >= kNT / 2) {
    leaf_issue_rest(a, s, nrows, t - kNT / 2);
    leaf_issue_rest(a, s, nrows, t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  // (1) Alg. 4 on the block: RPT rows per thread over the first kNT / RPT threads (rows >= nrows
  // are zero and store nothing)
  if (a.mgs_rpt == 2) {
    mgs_block<2>(s, nrows, c0, pw);
  } else {
    mgs_block<1>(s, nrows, c0, pw);
  }
  __syncthreads();
  leaf_ts(a, slot);
  // (2) this block's Gram G_b = R_b' R_b (upper triangle), FP64.  R_b is widened to FP64 once
  // (the FP32 -> FP64 conversions run at 1/8 of the FMA rate: widening inside the product loop
  // cost ~1 us per panel)
  for (int e = t; e < 1024; e += kNT) s.Rbd[e] = (double)s.Rb[e];
  __syncthreads();
  for (int e = t; e < 1024; e += kNT) {
    const int i = e >> 5, j = e & 31;
    double g = 0.0;
    if (i <= j && j < pw) {
      for (int l = 0; l <= i; ++l) g = fma(s.Rbd[l * 32 + i], s.Rbd[l * 32 + j], g);
    }
    a.gpart[(long long)blockIdx.x * 1024 + e] = g;
  }
  leaf_barrier(a, s);
  leaf_ts(a, slot);
  cross_sum<double>(a.gpart, 1024, 1024, a.nb, a.gsum, reinterpret_cast<double*>(s.T), nullptr, 0,
                    0, 0, 1, 0, false);
  leaf_ts(a, slot);
  leaf_barrier(a, s);
  leaf_ts(a, slot);
  if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: Cholesky start
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[100] = v;
  }
  // (3) R = chol(G) and S_b = R_b R^-1 in warp 0, one ROLLED pass over k (the fully unrolled
  // 32-step chain was ~100 KB of straight-line code run once per panel: instruction-fetch bound).
  // Lane j holds column j of the trailing Gram, c[i] = W(k+i, j) (shifted down one slot per step,
  // so the pivot is always c[0]), and row j of S_b under forward substitution, r[i] = the running
  // value of column k+i.  Step k: the pivot G(k,k) from lane k by shuffle, one FP64 reciprocal
  // square root (1/R(k,k), <= 1 ulp: R(k,j) = W(k,j) / R(k,k) and the S_b quotients become
  // products; FP64 values within an ulp round to the same FP32 R and Q, exact inputs stay exact
  // -- the planted pin), row k of R broadcast through shared memory.
  if (warp == 0) {
    double c[32], r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = (i <= lane && lane < pw) ? __ldcg(a.gsum + i * 32 + lane) : 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = (lane < pw && j < pw) ? s.Rbd[lane * 32 + j] : 0.0;
    if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: Cholesky inputs loaded
      unsigned long long v;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v) : "d"(c[31]), "d"(r[31]));
      a.dbg[101] = v;
    }
    // software-pipelined: the pivot of step k+1 (lane k+1's first update -> shuffle -> rsqrt) is
    // issued at the top of step k's trailing updates; branch-free so it all schedules together
    double d = __shfl_sync(0xffffffffu, c[0], 0);
    bool ok = d > 0.0 && d <= 1.7976931348623157e308;
    double ri = rsqrt_nr(ok ? d : 1.0);
#pragma unroll 1
    for (int k = 0; k < pw; ++k) {
      ri = ok ? ri : 0.0;
      const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
      s.Rd[k * 34 + lane] = rkj;
      if (!ok && lane == 0 && blockIdx.x == 0 && a.status) atomicMin(a.status, a.col0 + c0 + k + 1);
      const double sk = r[0] * ri;
      s.Sf[lane * 32 + k] = (float)sk;
      __syncwarp();
      const double* rk = s.Rd + k * 34 + k + 1;  // R(k, k+1+i); entries past column 31 are unused
      const double v0 = rk[0];
      c[0] = fma(-v0, rkj, c[1]);
      r[0] = fma(-sk, v0, r[1]);
      d = __shfl_sync(0xffffffffu, c[0], (k + 1) & 31);  // next pivot (unused after the last step)
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
    for (int j = pw; j < 32; ++j) s.Sf[lane * 32 + j] = 0.f;
  } else if (st_pw > 0 && warp != 4) {
    // the previous panel's deferred Q stores (those columns are final) beside the one-warp
    // Cholesky chain, on the six warps that do not share its scheduler (warp 4 does)
    const int idx = (warp < 4 ? warp - 1 : warp - 2) * 32 + lane;
    if (idx < nrows) leaf_store_row(a, s, idx, st_c0, st_pw);
    if (idx + 192 < nrows) leaf_store_row(a, s, idx + 192, st_c0, st_pw);
  }
  __syncthreads();
  if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: Cholesky + S end
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[102] = v;
  }
  leaf_ts(a, slot);
  if (blockIdx.x == 0) {  // the panel's R block (upper triangle; the lower one stays zero)
    for (int e = t; e < pw * pw; e += kNT) {
      const int i = e % pw, j = e / pw;
      if (i <= j) a.R[(c0 + i) + (long long)(c0 + j) * a.ldr] = (float)s.Rd[i * 34 + j];
    }
  }
  // (4) Q_b <- Q_b S_b (S_b upper triangular: the zero terms add exactly nothing).  Rolled over
  // groups of four l: Q_b(t, l..l+3) is one conflict-free 16-byte shared load (the scalar load per
  // l hit 8 banks per warp), then four unrolled rank-1 steps in the same l order as before.  Rows
  // l >= pw of S_b are zero (lanes >= pw above), so the padded tail adds exact zeros.
  if (t < nrows) {
    float* row = s.L + t * kLd + c0;
    float y[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) y[j] = 0.f;
#pragma unroll 1
    for (int l4 = 0; l4 < pw; l4 += 4) {
      const float4 q4 = *reinterpret_cast<const float4*>(row + l4);
      const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float ql = qv[u];
        const float4* sr = reinterpret_cast<const float4*>(s.Sf + (l4 + u) * 32);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 v = sr[j4];
          y[4 * j4] = fmaf(ql, v.x, y[4 * j4]);
          y[4 * j4 + 1] = fmaf(ql, v.y, y[4 * j4 + 1]);
          y[4 * j4 + 2] = fmaf(ql, v.z, y[4 * j4 + 2]);
          y[4 * j4 + 3] = fmaf(ql, v.w, y[4 * j4 + 3]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < pw) row[j] = y[j];
  }
  __syncthreads();
  if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: apply end (before the Q stores)
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[104] = v;
  }
  // these pw columns of Q are final (later ops only read them): stream them out (FP32 and the
  // FP16 shadow), coalesced down each column -- now, or (defer) by the idle upper half of the CTA
  // beside the next panel's MGS
  if (!defer && t < nrows) leaf_store_row(a, s, t, c0, pw);
  leaf_ts(a, slot);
}

// ---- PROJ: R12 = Q1' A2, R block <- R12, A2 -= Q1 R12 (FP32) ------------------------------------
// H = h (32 or 64), W2P = w2 rounded up to 32 (the columns past the leaf are zero in shared memory
// and stay zero).
template <int H, int W2P>
__device__ __noinline__ void leaf_proj(const LeafArgs& a, Smem& s, int nrows, int c0, int w2,
                                       int& slot) {
  constexpr int TJ = W2P / 4, TILES = (H / 4) * TJ, G = kNT / TILES;
  const int t = threadIdx.x;
  asm volatile("cp.async.wait_all;" ::: "memory");  // the leaf's later columns (loaded async)
  __syncthreads();
  const int tile = t % TILES, grp = t / TILES;
  const int ti = tile / TJ, tj = tile % TJ;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  {
    const float* q1 = s.L + c0 + 4 * ti;
    const float* a2 = s.L + c0 + H + 4 * tj;
#pragma unroll 4
    for (int r = grp; r < nrows; r += G) {
      const float4 qv = *reinterpret_cast<const float4*>(q1 + r * kLd);
      const float4 av = *reinterpret_cast<const float4*>(a2 + r * kLd);
      const float qq[4] = {qv.x, qv.y, qv.z, qv.w}, aa[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(qq[i], aa[j], acc[i][j]);
    }
  }
  float* pp = a.ppart + (long long)blockIdx.x * 4096;
  if (G == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(pp + (4 * ti + i) * W2P + 4 * tj) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  } else {
    // row groups: combine in group order through shared memory
#pragma unroll
    for (int i = 0; i < 4; ++i)
      *reinterpret_cast<float4*>(s.T + grp * (H * W2P) + (4 * ti + i) * W2P + 4 * tj) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    __syncthreads();
    for (int e = t; e < H * W2P; e += kNT) {
      float v = s.T[e];
#pragma unroll
      for (int g = 1; g < G; ++g) v += s.T[g * (H * W2P) + e];
      pp[e] = v;
    }
  }
  leaf_ts(a, slot);
  leaf_barrier(a, s);
  leaf_ts(a, slot);
  cross_sum<float>(a.ppart, 4096, H * W2P, a.nb, a.r12, s.wsum, a.R, a.ldr, H, w2, W2P, c0,
                   true);
  leaf_ts(a, slot);
  leaf_barrier(a, s);
  leaf_ts(a, slot);
  for (int e = t; e < H * W2P; e += kNT) s.T[e] = __ldcg(a.r12 + e);
  __syncthreads();
  // A2 -= Q1 R12: thread = rows (t % 128, t % 128 + 128), columns [jh * W2P/2, (jh+1) * W2P/2)
  constexpr int JC = W2P / 2;
  const int r0 = t % 128, jh = t / 128;
  float u[2][JC];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int j = 0; j < JC; ++j) u[rr][j] = 0.f;
  const float* qa = s.L + r0 * kLd + c0;
  const float* qb = s.L + (r0 + 128) * kLd + c0;
#pragma unroll 2
  for (int i4 = 0; i4 < H; i4 += 4) {
    const float4 va = *reinterpret_cast<const float4*>(qa + i4);
    const float4 vb = *reinterpret_cast<const float4*>(qb + i4);
    const float qx[2][4] = {{va.x, va.y, va.z, va.w}, {vb.x, vb.y, vb.z, vb.w}};
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const float4* tr = reinterpret_cast<const float4*>(s.T + (i4 + ii) * W2P + jh * JC);
#pragma unroll
      for (int j4 = 0; j4 < JC / 4; ++j4) {
        const float4 v = tr[j4];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          u[rr][4 * j4] = fmaf(qx[rr][ii], v.x, u[rr][4 * j4]);
          u[rr][4 * j4 + 1] = fmaf(qx[rr][ii], v.y, u[rr][4 * j4 + 1]);
          u[rr][4 * j4 + 2] = fmaf(qx[rr][ii], v.z, u[rr][4 * j4 + 2]);
          u[rr][4 * j4 + 3] = fmaf(qx[rr][ii], v.w, u[rr][4 * j4 + 3]);
        }
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < 2; ++rr) {
    const int r = r0 + rr * 128;
    if (r < nrows) {
      float* dst = s.L + r * kLd + c0 + H + jh * JC;
#pragma unroll
      for (int j4 = 0; j4 < JC / 4; ++j4) {
        float4 v = *reinterpret_cast<float4*>(dst + 4 * j4);
        v.x -= u[rr][4 * j4];
        v.y -= u[rr][4 * j4 + 1];
        v.z -= u[rr][4 * j4 + 2];
        v.w -= u[rr][4 * j4 + 3];
        *reinterpret_cast<float4*>(dst + 4 * j4) = v;
      }
    }
  }
  __syncthreads();
  leaf_ts(a, slot);
}

__global__ void __launch_bounds__(kNT, 1) leaf_kernel(const __grid_constant__ LeafArgs a) {
  extern __shared__ __align__(16) unsigned char leaf_smem[];
  Smem& s = *reinterpret_cast<Smem*>(leaf_smem);
  const int t = threadIdx.x;
  const int row0 = leaf_row(blockIdx.x, a.m, a.nb);
  const int nrows = leaf_row(blockIdx.x + 1, a.m, a.nb) - row0;
  int slot = 0;
  if (t == 0) s.barseq = 0;
  leaf_ts(a, slot);
  // load the block's rows of the leaf; columns past the leaf and rows past the block are zero.
  // Columns [0, 32) (the first panel) now, 16-byte loads down the columns (a warp = 2 row quads x
  // 16 columns, so the transposing shared stores hit 32 distinct banks: row stride 132 = 4 mod 32
  // banks); columns [32, 128) with cp.async (thread = row, zero-filled past the block), waited for
  // by the first projection.
  const bool vec = ((row0 | nrows) & 3) == 0 && (a.ldx & 3) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.X) & 15) == 0;
  const int lane = t & 31, warp = t >> 5;
  if (vec) {
    float4 v[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int q = 2 * (warp + 8 * (it >> 1)) + (lane >> 4), j = 16 * (it & 1) + (lane & 15);
      v[it] = (4 * q < nrows && j < a.wl)
                  ? __ldg(reinterpret_cast<const float4*>(a.X + row0 + 4 * q + (long long)j * a.ldx))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int q = 2 * (warp + 8 * (it >> 1)) + (lane >> 4), j = 16 * (it & 1) + (lane & 15);
      float* d = s.L + 4 * q * kLd + j;
      d[0] = v[it].x;
      d[kLd] = v[it].y;
      d[2 * kLd] = v[it].z;
      d[3 * kLd] = v[it].w;
    }
  } else {
    const float* src = a.X + row0 + t;
    float* dst = s.L + t * kLd;
    const bool ok = t < nrows;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) dst[j] = (ok && j < a.wl) ? src[(long long)j * a.ldx] : 0.f;
  }
  if (a.mgs_rpt != 2 || a.ops[0].kind != 0) {  // otherwise issued beside the first MGS
    leaf_issue_rest(a, s, nrows, t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __syncthreads();
  leaf_ts(a, slot);
  int last_panel = 0;
  for (int o = 0; o < a.nops; ++o)
    if (a.ops[o].kind == 0) last_panel = o;
  int st_c0 = 0, st_pw = 0;  // a panel's Q columns whose stores wait for the next panel's MGS
  for (int o = 0; o < a.nops; ++o) {
    const LeafOp op = a.ops[o];
    if (op.kind == 0) {
      const bool defer = a.mgs_rpt == 2 && o != last_panel;
      leaf_panel(a, s, nrows, op.c0, op.h, slot, o == 0, st_c0, st_pw, defer);
      st_c0 = op.c0;
      st_pw = defer ? op.h : 0;
    } else if (op.h == 64) {
      if (op.w2 > 32)
        leaf_proj<64, 64>(a, s, nrows, op.c0, op.w2, slot);
      else
        leaf_proj<64, 32>(a, s, nrows, op.c0, op.w2, slot);
    } else {
      leaf_proj<32, 32>(a, s, nrows, op.c0, op.w2, slot);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  leaf_ts(a, slot);
}

int leaf_split(int w) { return 32 * ((w + 63) / 64); }

void leaf_plan(int c0, int w, LeafArgs& a) {
  if (w <= 32) {
    a.ops[a.nops++] = LeafOp{0, c0, w, 0};
    return;
  }
  const int h = leaf_split(w), w2 = w - h;
  leaf_plan(c0, h, a);
  a.ops[a.nops++] = LeafOp{1, c0, h, w2};
  leaf_plan(c0 + h, w2, a);
}

}  // namespace

unsigned long long* g_leaf_dbg = nullptr;

size_t leaf_scratch_bytes() {
  return sizeof(double) * (148 * 1024 + 1024) + sizeof(float) * (148 * 4096 + 4096) + 1024;
}

cudaError_t leaf_fused(int m, int wl, float* X, long long ldx, __half* Xh, long long ldh, float* R,
                       long long ldr, int col0, int* status, void* scratch, size_t scratch_bytes,
                       unsigned* bar, unsigned* bar_seq, int num_sms, cudaStream_t st) {
  if (wl < 1 || wl > kCols || m < wl) return cudaErrorNotSupported;
  const int nb = (m + kRows - 1) / kRows;
  static int per_sm = -1;
  const int smem = (int)sizeof(Smem);
  if (per_sm < 0) {
    cudaFuncSetAttribute(leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, leaf_kernel, kNT, smem) !=
        cudaSuccess)
      per_sm = 0;
  }
  if (nb > per_sm * num_sms || nb > 148) return cudaErrorNotSupported;
  if (scratch_bytes < leaf_scratch_bytes()) return cudaErrorNotSupported;
  LeafArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.Xh = Xh;
  a.ldh = ldh;
  a.R = R;
  a.ldr = ldr;
  a.m = m;
  a.wl = wl;
  a.nb = nb;
  a.nops = 0;
  leaf_plan(0, wl, a);
  char* p = static_cast<char*>(scratch);
  a.gpart = reinterpret_cast<double*>(p);
  a.gsum = a.gpart + 148 * 1024;
  a.ppart = reinterpret_cast<float*>(a.gsum + 1024);
  a.r12 = a.ppart + 148 * 4096;
  a.bar = bar;
  a.bar_base = *bar_seq;
  a.status = status;
  a.col0 = col0;
  a.dbg = g_leaf_dbg;
  {
    static int rpt = -1;
    if (rpt < 0) {
      const char* e = getenv("TCQR_LEAF_MGS_RPT");
      rpt = (e && atoi(e) == 1) ? 1 : 2;  // 128 threads x 2 rows measured faster (14.3 vs 17.2 us)
    }
    a.mgs_rpt = rpt;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, leaf_kernel, a);
  if (e == cudaSuccess) *bar_seq += 2u * (unsigned)a.nops;  // two grid barriers per op
  return e;
}

}  // namespace tcqr

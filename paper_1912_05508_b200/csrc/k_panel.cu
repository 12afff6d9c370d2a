// k_panel.cu -- K2: the communication-avoiding MGS panel (Eq. (6), Alg. 4).
//
// Primary path: panel_fused_kernel (below) runs the whole Eq. (6) tree in ONE cooperative launch.
// Fallback (tree wider than the co-resident grid): one launch of panel_mgs_kernel per level plus
// panel_apply_kernel.  In both, CTA b owns row block b (br rows; the last block absorbs a
// remainder shorter than w rows, reading R-A6), keeps it in registers (two rows per thread, the
// paper's "each thread ... a single row" design) and runs Alg. 4 on it:
//     for k: R(k,k) = ||q_k||; q_k /= R(k,k); R(k,k+1:) = q_k' Q(:,k+1:); Q(:,k+1:) -= q_k R(k,k+1:)
// The norm and the w-k dot products of step k are ONE block reduction: each thread forms its
// partial products, a 31-shuffle transpose-reduce leaves lane j with the warp sum of product j,
// and a double-buffered shared array combines the warps in a fixed order (deterministic).
// R(k,j) = (a_k' a_j) / R(k,k) equals q_k' a_j up to rounding order.
// The stacked R's are factored by the same step (step 3); step 4 ("batched SGEMM" in the paper,
// PAPER.md:453-455) multiplies each local Q by its slice of the stack's Q.
#include "common.cuh"
#include "kernels.h"
#include "mgs.cuh"

namespace tcqr {


int panel_num_blocks(int rows, int br, int w) {
  int nb = (rows + br - 1) / br;
  if (nb < 1) nb = 1;
  const int last = rows - (nb - 1) * br;
  if (nb > 1 && last < w) --nb;
  return nb;
}

// (panel_mgs_kernel is defined below, after the rotating MGS step it shares.)

// X_b <- X_b * T_b with T_b = S[b*w:(b+1)*w, 0:w] (lds): Eq. (6) step 4.  A CTA takes 128 rows
// with two threads per row, each forming 16 of the (up to 32) output columns by FFMA2 (the same
// fmaf sequence per entry: l in increasing order); the row's 32 inputs are read by both threads
// (the second read hits L1).  Register-lean (three CTAs per SM) so that enough loads are in
// flight to stream the panel at HBM rate -- the one-thread-per-row version held 64 values per
// thread (167 registers, one CTA per SM) and ran at 1.1 TB/s.  T_b staged in shared memory per
// block the CTA's rows touch (br is a multiple of 32, CTAs may straddle two blocks).
__global__ void __launch_bounds__(256, 3) panel_apply_kernel(int rows, int w, float* __restrict__ X,
                                                             long long ldx, int br, int nb,
                                                             const float* __restrict__ S,
                                                             long long lds) {
  __shared__ __align__(16) float T[32][36];
  const int half = threadIdx.x >> 7;
  const int i = blockIdx.x * 128 + (threadIdx.x & 127);
  const int row_first = blockIdx.x * 128;
  int b_first = row_first / br;
  if (b_first > nb - 1) b_first = nb - 1;
  int row_last = row_first + 127;
  if (row_last > rows - 1) row_last = rows - 1;
  int b_last = row_last / br;
  if (b_last > nb - 1) b_last = nb - 1;
  const bool ok = i < rows;
  int bi = ok ? i / br : 0;
  if (bi > nb - 1) bi = nb - 1;
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (ok && j < w) ? X[(long long)i + (long long)j * ldx] : 0.f;
  float2 y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) y[j] = make_float2(0.f, 0.f);
  for (int b = b_first; b <= b_last; ++b) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int l = e & 31, j = e >> 5;
      T[l][j] = (l < w && j < w) ? S[(long long)(b * w + l) + (long long)j * lds] : 0.f;
    }
    __syncthreads();
    if (ok && bi == b) {
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        const float2 xl = make_float2(x[l], x[l]);
        const float4* t4 = reinterpret_cast<const float4*>(&T[l][16 * half]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 t = t4[q];
          y[2 * q] = ffma2(xl, make_float2(t.x, t.y), y[2 * q]);
          y[2 * q + 1] = ffma2(xl, make_float2(t.z, t.w), y[2 * q + 1]);
        }
      }
    }
  }
  if (ok) {
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) {
      const int j = 16 * half + 2 * j2;
      if (j < w) X[(long long)i + (long long)j * ldx] = y[j2].x;
      if (j + 1 < w) X[(long long)i + (long long)(j + 1) * ldx] = y[j2].y;
    }
  }
}

cudaError_t panel_apply(int rows, int w, float* X, long long ldx, int br, int nb, const float* S,
                        long long lds, cudaStream_t st) {
  const int grid = (rows + 127) / 128;
  panel_apply_kernel<<<grid, 256, 0, st>>>(rows, w, X, ldx, br, nb, S, lds);
  return cudaGetLastError();
}


// ==========================================================================================
// Fused single-launch CAQR panel (Eq. (6) steps 1-5 in ONE cooperative kernel).
//
// CTA b runs Alg. 4 on row block b (step 1) with a rotating register window: at step k the pivot
// column is always x[.][0] and the trailing update writes column j into slot j-1, so the loop
// body has no data-dependent register indexing and stays small for the instruction cache (the
// fully unrolled v1 kernel spent 55% of its cycles in no_instructions stalls; ncu,
// profiles/r01_ncu_panel_mgs_v1_details.csv).  The reduction width follows the active column
// count.  The stacked R's (step 2) are factored (step 3) by the LAST child CTA to finish each
// tree node (atomic arrival counter), level by level, so no CTA waits for another until the root
// is done.  Then every CTA forms its composite transform T_b = S1[b] S2[parent(b)] ... (step 4)
// from the stack-Q slices and writes its final Q rows (FP32 and the FP16 shadow used by the
// tensor-core GEMMs above), step 5.  Co-residency of all CTAs is guaranteed by the cooperative
// launch.  Two shapes: 128 threads x 2 rows (256-row blocks, fan-in 8) and 256 threads x 4 rows
// (1024-row blocks, fan-in 32: two tree levels up to m = 32768).
// ==========================================================================================
constexpr int kMaxLevels = 8;

struct FusedPanelArgs {
  float* X;
  long long ldx;
  __half* Xh;  // may be null
  long long ldh;
  int m, w, br, nb, F, L;       // L = tree levels above the row blocks (0 if nb == 1)
  int nodes[kMaxLevels + 1];    // nodes[l] = nodes at level l (nodes[0] = nb, nodes[L] = 1)
  float* Rbuf[kMaxLevels + 1];  // R of every node at level l: nodes[l] * w * w floats
  float* Qst[kMaxLevels + 1];   // stack-Q slices for the children of level-l nodes (l >= 1)
  int* cnt[kMaxLevels + 1];     // arrival counters of level-l nodes (l >= 1)
  int* done;                    // [0] root done flag, [1] exit counter
  float* Rout;                  // final R (w x w, ldr)
  long long ldr;
  int root_is_global;           // 1: a zero/non-finite norm at the root is a breakdown
  int* status;
  int col0;
  unsigned long long* dbg;      // optional phase timestamps (globaltimer), 64 slots
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG_T(slot)                                          \
  do {                                                       \
    if (a.dbg && threadIdx.x == 0) a.dbg[(slot)] = gtimer(); \
  } while (0)

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// Where the Q columns of an MGS go: shared [row][33] (row blocks) or a global stack-Q slice
// layout (children blocks of w x w, column-major): row s -> child s / w, row s % w.
struct QSink {
  float* sm;       // shared rows x 33, or null
  float* g;        // global slices base, or null
  int w;
  // element (row, k) lives at base(row) + k * stride
  __device__ __forceinline__ float* base(int row) const {
    return sm ? sm + row * 33 : g + (long long)(row / w) * w * w + (row % w);
  }
  __device__ __forceinline__ int stride() const { return sm ? 1 : w; }
};


template <int NT, int RPT>
__device__ __forceinline__ void mgs_rotating(float (&x)[RPT][32], int nrows, int w,
                                             const QSink& qs, float* Rdst, long long rs,
                                             long long cs, bool check, int* status, int col0,
                                             float* red, unsigned long long* dbg = nullptr,
                                             bool write_lower = true) {
  float* qp[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int row = threadIdx.x + r * NT;
    qp[r] = qs.base(row < nrows ? row : 0);
  }
  const int qstride = qs.stride();
  int buf = 0;
  for (int k = 0; k < w; ++k) {
    if (dbg && threadIdx.x == 0) dbg[k] = gtimer();
    const int act = w - k;
    if (act > 16)
      mgs_step<NT, RPT, 32>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
    else if (act > 8)
      mgs_step<NT, RPT, 16>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
    else if (act > 4)
      mgs_step<NT, RPT, 8>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
    else if (act > 2)
      mgs_step<NT, RPT, 4>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
    else if (act > 1)
      mgs_step<NT, RPT, 2>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
    else
      mgs_step<NT, RPT, 1>(x, nrows, w, k, qp, qstride, Rdst, rs, cs, check, status, col0, red, buf, write_lower);
  }
}

template <int NT, int RPT>
struct FusedShape {
  static constexpr int CAP = NT * RPT;
  static constexpr int SMEM = (int)sizeof(float) * (CAP * 33 + 3 * 32 * 36 + 2 * (NT / 32) * 32) + 16;
};

// Balanced row blocks: block b covers [b*m/nb, (b+1)*m/nb), every block <= br rows (Eq. (6) is
// exact for any blocking; reading R-A6 folds remainders, this spreads them).
__device__ __forceinline__ int blk_row(int b, int m, int nb) {
  return (int)((long long)b * m / nb);
}

template <int NT, int RPT>
__global__ void __launch_bounds__(NT, 1) panel_fused_kernel(FusedPanelArgs a) {
  using Sh = FusedShape<NT, RPT>;
  extern __shared__ float fsm[];
  float* qA = fsm;                                     // Q of the current MGS [CAP][33]
  float* T = fsm + ((Sh::CAP * 33 + 3) & ~3);          // [32][36] (16-byte aligned rows)
  float* T2 = T + 32 * 36;                             // [32][36]
  float* Sst = T2 + 32 * 36;                           // [32][36] staged stack-Q slice
  float* red = Sst + 32 * 36;                          // [2][NT/32][32]
  __shared__ int s_last;
  const int b = blockIdx.x, w = a.w;
  const int row0 = blk_row(b, a.m, a.nb);
  const int nrows = blk_row(b + 1, a.m, a.nb) - row0;

  // ---- step 1: Alg. 4 on this row block; steps 2-3: the last child to arrive factors each
  // tree node (single MGS call site so the step body is instantiated once) ----
  if (b == 0) DBG_T(0);
  float x[RPT][32];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = threadIdx.x + r * NT;
    const bool ok = i < nrows;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      x[r][j] = (ok && j < w) ? a.X[(long long)(row0 + i) + (long long)j * a.ldx] : 0.f;
  }
  const bool single = (a.L == 0);
  int node = b, level = 0, rows_now = nrows, first = 0;
  bool root = single, spilled = false;
  while (true) {
    const bool top = (level == a.L);
    // node R's are stored ROW-major (stack rows become contiguous 128-byte loads); the final R
    // is column-major with leading dimension ldr.
    float* Rn = top ? a.Rout : a.Rbuf[level] + (long long)node * w * w;
    if (b == 0 && level == 0) DBG_T(1);
    mgs_rotating<NT, RPT>(x, rows_now, w, QSink{qA, nullptr, w}, Rn, top ? 1 : w,
                          top ? a.ldr : 1, top && a.root_is_global, a.status, a.col0, red,
                          a.dbg ? (level == 0 ? (b == 0 ? a.dbg + 32 : nullptr) : a.dbg + 64)
                                : nullptr);
    __syncthreads();
    if (level == 0) {
      if (b == 0) DBG_T(2);
      if (single) break;
    } else {
      // stack Q -> per-child w x w slices (column-major) of Qst[level]
      float* Qd = a.Qst[level] + (long long)first * w * w;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int sr = threadIdx.x + r * NT;
        if (sr < rows_now) {
          const int ci = sr / w, aa = sr - ci * w;
          float* dst = Qd + (long long)ci * w * w + aa;
          for (int j = 0; j < w; ++j) dst[(long long)j * w] = qA[sr * 33 + j];
        }
      }
      DBG_T(10 + 4 * level);
      if (top) {
        root = true;
        break;
      }
    }
    // arrive at the parent; continue only if this CTA completed it
    __threadfence();
    __syncthreads();
    const int parent = node / a.F;
    first = parent * a.F;
    const int nchild = min(a.F, a.nodes[level] - first);
    if (threadIdx.x == 0) s_last = (atomicAdd(a.cnt[level + 1] + parent, 1) == nchild - 1);
    __syncthreads();
    if (!s_last) break;
    __threadfence();
    if (level == 0) {
      // this CTA climbs the tree: park its local Q_b in X (re-read by step 4) so shared memory
      // is free for the stack levels; the other CTAs keep Q_b in shared memory.
      spilled = true;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = threadIdx.x + r * NT;
        if (i < nrows)
          for (int j = 0; j < w; ++j) a.X[(long long)(row0 + i) + (long long)j * a.ldx] = qA[i * 33 + j];
      }
    }
    ++level;
    node = parent;
    DBG_T(8 + 4 * level);
    rows_now = nchild * w;
    // stack row sr = child sr / w, row sr % w of its row-major R: w contiguous floats
    const float* Rc = a.Rbuf[level - 1] + (long long)first * w * w;
    const bool vec = (w == 32);
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int sr = threadIdx.x + r * NT;
      const bool ok = sr < rows_now;
      const float* src = Rc + (long long)(ok ? sr : 0) * w;
      if (vec) {
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4) {
          const float4 v = ok ? __ldcg(reinterpret_cast<const float4*>(src + j4))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          x[r][j4] = v.x;
          x[r][j4 + 1] = v.y;
          x[r][j4 + 2] = v.z;
          x[r][j4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[r][j] = (ok && j < w) ? __ldcg(src + j) : 0.f;
      }
    }
    DBG_T(9 + 4 * level);
  }
  if (root && !single) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release(a.done, 1);
  }

  // ---- step 4: T_b = S1[b] S2[b/F] ... ; Q_b <- Q_b T_b ----
  if (!single) {
    if (threadIdx.x == 0) {
      while (ld_relaxed(a.done) == 0) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
    if (b == 0) DBG_T(3);
    int idx = b;
    for (int e = threadIdx.x; e < 32 * 32; e += NT) {
      const int i = e & 31, j = e >> 5;
      T[i * 36 + j] = (i < w && j < w) ? __ldcg(a.Qst[1] + (long long)idx * w * w + i + j * w) : 0.f;
    }
    for (int l = 2; l <= a.L; ++l) {
      idx /= a.F;
      const float* S = a.Qst[l] + (long long)idx * w * w;
      for (int e = threadIdx.x; e < 32 * 32; e += NT) {
        const int i = e & 31, j = e >> 5;
        Sst[i * 36 + j] = (i < w && j < w) ? __ldcg(S + i + j * w) : 0.f;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 32; e += NT) {
        const int i = e & 31, j = e >> 5;
        float acc = 0.f;
#pragma unroll 8
        for (int t = 0; t < 32; ++t) acc = fmaf(T[i * 36 + t], Sst[t * 36 + j], acc);
        T2[i * 36 + j] = acc;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * 32; e += NT) T[(e & 31) * 36 + (e >> 5)] = T2[(e & 31) * 36 + (e >> 5)];
    }
    __syncthreads();
  }
  if (b == 0) DBG_T(4);
  // ---- step 5: final Q rows (FP32 + FP16 shadow) ----
#pragma unroll 1
  for (int r = 0; r < RPT; ++r) {
    const int i = threadIdx.x + r * NT;
    if (i >= nrows) continue;
    const long long gi = (long long)(row0 + i);
    float y[32];
    if (single) {
#pragma unroll
      for (int j = 0; j < 32; ++j) y[j] = qA[i * 33 + j];
    } else {
      float xr[32];
      if (spilled) {
#pragma unroll
        for (int j = 0; j < 32; ++j) xr[j] = (j < w) ? a.X[gi + (long long)j * a.ldx] : 0.f;
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) xr[j] = qA[i * 33 + j];
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) y[j] = 0.f;
#pragma unroll
      for (int l_ = 0; l_ < 32; ++l_) {
        const float ql = xr[l_];
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4) {
          const float4 tv = *reinterpret_cast<const float4*>(T + l_ * 36 + j4);
          y[j4] = fmaf(ql, tv.x, y[j4]);
          y[j4 + 1] = fmaf(ql, tv.y, y[j4 + 1]);
          y[j4 + 2] = fmaf(ql, tv.z, y[j4 + 2]);
          y[j4 + 3] = fmaf(ql, tv.w, y[j4 + 3]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < w) {
        a.X[gi + (long long)j * a.ldx] = y[j];
        if (a.Xh) a.Xh[gi + (long long)j * a.ldh] = __float2half_rn(y[j]);
      }
    }
  }
  if (b == 0) DBG_T(5);
  // ---- reset the arrival state for the next panel (last CTA out) ----
  if (!single) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(a.done + 1, 1) == a.nb - 1) {
        for (int l = 1; l <= a.L; ++l)
          for (int g = 0; g < a.nodes[l]; ++g) a.cnt[l][g] = 0;
        a.done[1] = 0;
        __threadfence();
        st_release(a.done, 0);
      }
    }
  }
}

// One CAQR level as its own launch (used when the fused tree does not fit the co-resident grid):
// MGS on every row block of X; local Q in place; R_b -> stack rows [b*w, (b+1)*w) of S or Rout.
// Blocks follow the fold rule of reading R-A6 (panel_num_blocks).
constexpr int kLvlNT = 128, kLvlRPT = 4;
__global__ void __launch_bounds__(kLvlNT) panel_mgs_kernel(
    int rows, int w, float* __restrict__ X, long long ldx, int br, int nb, float* __restrict__ S,
    long long lds, float* __restrict__ Rout, long long ldr, int top, int* status, int col0) {
  extern __shared__ float fsm[];
  float* qs = fsm;
  float* red = qs + kLvlNT * kLvlRPT * 33;
  const int b = blockIdx.x;
  const int row0 = b * br;
  const int nrows = (b == nb - 1) ? rows - row0 : br;
  float x[kLvlRPT][32];
#pragma unroll
  for (int r = 0; r < kLvlRPT; ++r) {
    const int i = threadIdx.x + r * kLvlNT;
    const bool ok = i < nrows;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      x[r][j] = (ok && j < w) ? X[(long long)(row0 + i) + (long long)j * ldx] : 0.f;
  }
  float* Rdst = (nb == 1) ? Rout : S + (long long)b * w;
  const long long ldR = (nb == 1) ? ldr : lds;
  mgs_rotating<kLvlNT, kLvlRPT>(x, nrows, w, QSink{qs, nullptr, w}, Rdst, 1, ldR, top != 0,
                                status, col0, red);
  __syncthreads();
  for (int r = 0; r < kLvlRPT; ++r) {
    const int i = threadIdx.x + r * kLvlNT;
    if (i < nrows)
      for (int j = 0; j < w; ++j) X[(long long)(row0 + i) + (long long)j * ldx] = qs[i * 33 + j];
  }
}

cudaError_t panel_mgs_level(int rows, int w, float* X, long long ldx, int br, int nb, float* S,
                            long long lds, float* Rout, long long ldr, int top, int* status,
                            int col0, cudaStream_t st) {
  constexpr int cap = kLvlNT * kLvlRPT;
  if (nb > 1 && br + w - 1 > cap) return cudaErrorInvalidValue;
  if (nb == 1 && rows > cap) return cudaErrorInvalidValue;
  const int smem = (int)sizeof(float) * (cap * 33 + 2 * (kLvlNT / 32) * 32);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(panel_mgs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  panel_mgs_kernel<<<nb, kLvlNT, smem, st>>>(rows, w, X, ldx, br, nb, S, lds, Rout, ldr, top,
                                             status, col0);
  return cudaGetLastError();
}

unsigned long long* g_panel_dbg = nullptr;

// ==========================================================================================
// Pipelined single-level panel (nb <= F row blocks, one root): the stacked node is a stack of
// upper triangles, so the root's MGS step k only touches rows (b, i <= k), which child b produced
// at ITS step k (R_b(k, k:)).  The root therefore runs one step behind the children instead of
// after them.  Likewise the final Q column j of block b is Q_b * S_b(:, j), and S_b(:, j) (rows of
// the root's Q column j) is final after root step j: the children apply it column by column
// while the root is still running.  Every R / S value doubles as its own ready flag: the
// scratch is NaN-initialized, producers store plain values, consumers poll until non-NaN and
// reset the slot to NaN after use (no fences on the critical path).
// ==========================================================================================
struct PipeArgs {
  float* X;
  long long ldx;
  __half* Xh;  // may be null
  long long ldh;
  int m, w, nb;
  float* Rb;   // nb row-major w x w child R's (NaN between uses)
  float* S;    // nb column-major w x w slices of the root Q (NaN between uses)
  float* Rout;
  long long ldr;
  int root_is_global;
  int* status;
  int col0;
  unsigned long long* dbg;  // optional timestamps: child 0 [0..1], apply columns [32+j], root [64+k]
};

__device__ __forceinline__ float ld_relaxed_f(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

// same load without a memory clobber, so consecutive polls are issued back to back
__device__ __forceinline__ float ld_relaxed_nc(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// Hand-off sentinel of the pipelined panel: the all-ones bit pattern (a negative quiet NaN) that
// the workspace memset (0xff bytes) and the consumers' resets write.  Arithmetic never produces
// it -- the GPU's NaN results are the canonical 0x7fffffff and every published value is an
// arithmetic result -- so a NaN in the data (non-finite input) cannot be mistaken for "not yet
// written" and stall the pipeline.
__device__ __forceinline__ bool pending(float v) { return __float_as_uint(v) == 0xffffffffu; }

template <int NT, int RPT>
__global__ void __launch_bounds__(NT, 1) panel_pipe_kernel(PipeArgs a) {
  extern __shared__ float fsm[];
  float* qA = fsm;                                      // child: Q_b [CAP][33]
  float* sj = fsm + ((NT * RPT * 33 + 3) & ~3);         // child: [2][32] current S column
  float* red = sj + 64;                                 // [2][NT/32][32]
  const int w = a.w, b = blockIdx.x;
  const float qnan = __uint_as_float(0xffffffffu);  // the hand-off sentinel
  if (b < a.nb) {
    // ----------------------------- child: row block b -----------------------------------------
    if (a.dbg && b == 0 && threadIdx.x == 0) a.dbg[0] = gtimer();
    const int row0 = blk_row(b, a.m, a.nb);
    const int nrows = blk_row(b + 1, a.m, a.nb) - row0;
    float x[RPT][32];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = threadIdx.x + r * NT;
      const bool ok = i < nrows;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        x[r][j] = (ok && j < w) ? a.X[(long long)(row0 + i) + (long long)j * a.ldx] : 0.f;
    }
    // only the slots the root consumes are written (no zero lower triangle): a stale value in a
    // never-consumed slot could alias a polled slot of a later panel with another width
    
    mgs_rotating<NT, RPT>(x, nrows, w, QSink{qA, nullptr, w}, a.Rb + (long long)b * w * w, w, 1,
                          false, a.status, a.col0, red,
                          nullptr, false);
    __syncthreads();
    
    if (a.dbg && b == 0 && threadIdx.x == 0) a.dbg[1] = gtimer();
    // ---- apply: X_b(:, c) = Q_b S(:, c) (S = the root's Q slice of this block, upper
    // triangular), column groups of 8 as the root publishes them.  Q_b's rows stay in registers
    // (x is dead after the MGS) and S(l, c) = 0 for l > c, so each output is a full 32-term dot
    // product in the order l = 0..31 (the zero terms add exactly nothing). ----
    float qr[RPT][32];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = threadIdx.x + r * NT;
#pragma unroll
      for (int l = 0; l < 32; ++l) qr[r][l] = (i < nrows && l < w) ? qA[i * 33 + l] : 0.f;
    }
    __syncthreads();                 // qA is free from here on
    float* Ss = qA;                  // S block, column-major [32][32]
    // S element (l, c) of block b at S[(c*w + l)*32 + b]: the root writes one 128-byte line per
    // step and stack row, the children read with a 128-byte lane stride
    float* Sb = a.S + b;
    const int si = threadIdx.x;      // warp 0 lane l = row l of S
    for (int c0 = 0; c0 < w; c0 += 8) {
      if (si < 32) {
        // the group's columns: all loads in flight, then re-poll what the root has not written
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u;
          v[u] = (c < w && si <= c) ? ld_relaxed_nc(Sb + (c * w + si) * 32) : 0.f;
        }
        bool ready = true;
#pragma unroll
        for (int u = 0; u < 8; ++u) ready &= !pending(v[u]);
        while (!ready) {
          __nanosleep(20);
          ready = true;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (pending(v[u])) v[u] = ld_relaxed_nc(Sb + ((c0 + u) * w + si) * 32);
            ready &= !pending(v[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u;
          Ss[c * 32 + si] = v[u];
          if (c < w && si <= c) Sb[(c * w + si) * 32] = qnan;  // consumed: reset for the next panel
        }
      }
      __syncthreads();
      if (a.dbg && b == 0 && threadIdx.x == 0) a.dbg[32 + min(c0 + 7, w - 1)] = gtimer();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u;
        if (c < w) {
          const float4* sc = reinterpret_cast<const float4*>(Ss + c * 32);
          float y[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) y[r] = 0.f;
#pragma unroll
          for (int l4 = 0; l4 < 8; ++l4) {
            const float4 sv = sc[l4];
            const float s4[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
#pragma unroll
              for (int r = 0; r < RPT; ++r) y[r] = fmaf(qr[r][l4 * 4 + e], s4[e], y[r]);
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int i = threadIdx.x + r * NT;
            if (i < nrows) {
              a.X[(long long)(row0 + i) + (long long)c * a.ldx] = y[r];
              if (a.Xh) a.Xh[(long long)(row0 + i) + (long long)c * a.ldh] = __float2half_rn(y[r]);
            }
          }
        }
      }
    }
  } else {
    // ----------------------------- root: the stack of child R's -------------------------------
    // Stack row (b, i) lives in warp i/4, lane b, register slot i%4.  Warp w's rows are all zero
    // before step 4w, so it stays out of the steps until then: it polls its four rows in the
    // meantime (off the step chain), joins the step barrier at step 4w-1 (idle: a zero partial)
    // and computes from step 4w on.  The barrier count grows with the joined warps.  Row
    // i = 4w + r is placed for the window of step 4w: x[r][c] = R_b(i, 4w + c), zero for c < r --
    // steps 4w..i-1 see a zero leading column in it, which is exactly MGS on a row that starts at
    // column i.  Until step i its Q sink is null (S slots are written only when consumed).
    static_assert(NT == 256 && RPT == 4, "root mapping: 8 warps x 4 rows cover 32 stack rows");
    constexpr int NW = NT / 32;
    const int srows = a.nb * w;
    const int wid = threadIdx.x >> 5;
    const int tb = threadIdx.x & 31;          // child block of this thread's rows
    const int i0 = wid * 4;                   // first in-block row index (warp-uniform)
    const bool tvalid = tb < a.nb;
    const int nwa = min(NW, (w + 3) / 4);     // warps that hold rows
    // partial slots of warps that have not joined read as zero
    __shared__ int s_step;                    // last step whose barrier warp 0 has passed
    for (int e = threadIdx.x; e < 2 * NW * 32; e += NT) red[e] = 0.f;
    if (threadIdx.x == 0) s_step = -1;
    __syncthreads();
    // Warp 0's rows (rows 0..3 of every block) gate the first step: all warps fetch them together
    // (coalesced, one 128-byte row per load instruction, polled until no NaN is left) into
    // shared memory [block][129] (row r at r*32 + column).
    float* st0 = fsm;
    float* Rsm = fsm + 32 * 129;  // the panel's R, column-major 32 x 32 (R(k,j) at k + 32 j)
    {
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int t = wid + NW * u, r = t & 3, bb = t >> 2;
        const bool ok = bb < a.nb && r < w && tb >= r && tb < w;
        v[u] = ok ? ld_relaxed_nc(a.Rb + (long long)bb * w * w + (long long)r * w + tb) : 0.f;
      }
      while (true) {
        bool ready = true;
#pragma unroll
        for (int u = 0; u < 16; ++u) ready &= !pending(v[u]);
        if (__all_sync(0xffffffffu, ready)) break;
        __nanosleep(20);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int t = wid + NW * u, r = t & 3, bb = t >> 2;
          if (pending(v[u])) v[u] = ld_relaxed_nc(a.Rb + (long long)bb * w * w + (long long)r * w + tb);
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int t = wid + NW * u, r = t & 3, bb = t >> 2;
        if (bb < a.nb) st0[bb * 129 + r * 32 + tb] = v[u];
      }
    }
    __syncthreads();
    if (wid < nwa) {
      const float* rb = a.Rb + (long long)tb * w * w;
      float x[RPT][32];
      float* qp[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) qp[r] = nullptr;
      if (wid == 0) {
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int c = 0; c < 32; ++c) x[r][c] = (tvalid && c >= r) ? st0[tb * 129 + r * 32 + c] : 0.f;
      } else {
      // wait (one load per lane per round) until the last element of this warp's last row is
      // written -- the child writes the rows in order -- then fetch the four rows with 16-byte
      // loads from column i0 (x[r][c] = R_b(i0 + r, i0 + c); the lower part c < r is never
      // written and is zeroed), re-polling elements still NaN.  16-byte loads: the load count,
      // not the latency, bounds this fetch (~28 cycles per load instruction and warp).
      {
        const int il = min(i0 + RPT, w) - 1;
        const float* sent = rb + (long long)il * w + (w - 1);
        if (tvalid)
          while (pending(ld_relaxed_nc(sent))) __nanosleep(256);
        __syncwarp();
      }
      const bool vec = (w & 3) == 0;
      auto fetch = [&]() {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int i = i0 + r;
          const float* src = rb + (long long)i * w + i0;
          const bool ok = tvalid && i < w;
          if (vec) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
              if (ok && 4 * q < w - i0)
                asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "l"(src + 4 * q));
              x[r][4 * q] = v.x;
              x[r][4 * q + 1] = v.y;
              x[r][4 * q + 2] = v.z;
              x[r][4 * q + 3] = v.w;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) x[r][c] = (ok && c < w - i0) ? ld_relaxed_nc(src + c) : 0.f;
          }
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c < r) x[r][c] = 0.f;  // below the diagonal: never written
        }
      };
      fetch();
      while (true) {
        bool ready = true;
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int c = 0; c < 32; ++c) ready &= !pending(x[r][c]);
        if (__all_sync(0xffffffffu, ready)) break;
        __nanosleep(200);
        fetch();
      }
      }
      const int kfirst = wid == 0 ? 0 : i0 - 1;
      int buf = kfirst & 1;
      // a joining warp may only arrive at the step barrier once the previous step's barrier has
      // completed (a named barrier must not see arrivals of two generations with different counts)
      if (wid > 0) {
        if (tb == 0)
          while (atomicAdd(&s_step, 0) < kfirst - 1) __nanosleep(20);  // flag: shared atomics
        __syncwarp();
      }
      for (int k = kfirst; k < w; ++k) {
        if (a.dbg && threadIdx.x == 0) a.dbg[64 + k] = gtimer();
        if (tvalid && k >= i0 && k < i0 + RPT) {
          float* const qrow = a.S + k * 32 + tb;  // (block tb, row k, col j) at + j*w*32
          switch (k & 3) {  // uniform: k - i0 = k % 4
            case 0: qp[0] = qrow; break;
            case 1: qp[1] = qrow; break;
            case 2: qp[2] = qrow; break;
            default: qp[3] = qrow; break;
          }
        }
        const int cnt = 32 * min(nwa, (k + 1) / 4 + 1);  // warps joined at step k
        mgs_step_any<NT, RPT>(x, NT * RPT, w, k, qp, 32 * w, Rsm, 1, 32,
                              a.root_is_global != 0, a.status, a.col0, red, buf, k < i0, cnt);
        if (threadIdx.x == 0) atomicExch(&s_step, k);  // barrier k passed
      }
    }
    __syncthreads();
    // the panel's R (built in shared memory: the per-step row stores would be 32 scattered
    // global stores each) -> Rout, column by column
    for (int e = threadIdx.x; e < w * w; e += NT) {
      const int i = e % w, j = e / w;
      a.Rout[i + (long long)j * a.ldr] = Rsm[i + 32 * j];
    }
    // every stack row has been consumed: reset the slots to NaN for the next panel in bulk (off
    // the per-step critical path; the children are still applying the last columns)
    const long long tot = (long long)srows * w;
    if ((w & 3) == 0) {
      float4* p4 = reinterpret_cast<float4*>(a.Rb);
      const float4 n4 = make_float4(qnan, qnan, qnan, qnan);
      for (long long i = threadIdx.x; i < tot / 4; i += NT) p4[i] = n4;
    } else {
      for (long long i = threadIdx.x; i < tot; i += NT) a.Rb[i] = qnan;
    }
  }
}

template <int NT, int RPT>
static int pipe_capacity(int num_sms) {
  static int per_sm = -1;
  if (per_sm < 0) {
    const int smem = (int)sizeof(float) * (((NT * RPT * 33 + 3) & ~3) + 64 + 2 * (NT / 32) * 32);
    cudaFuncSetAttribute(panel_pipe_kernel<NT, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panel_pipe_kernel<NT, RPT>, NT,
                                                      smem) != cudaSuccess)
      per_sm = 0;
  }
  return per_sm * num_sms;
}

// m rows in nb = ceil(m / 1024) <= 1024 / w blocks + one root CTA; Rb, S: NaN-initialized scratch
// of 32 * 32 * 32 floats each.  cudaErrorNotSupported when the shape does not qualify.
cudaError_t panel_pipe(int m, int w, float* X, long long ldx, __half* Xh, long long ldh, int br,
                       float* Rout, long long ldr, int root_is_global, int* status, int col0,
                       float* Rb, float* S, int num_sms, cudaStream_t st) {
  if (w < 1 || w > 32 || br != 1024) return cudaErrorNotSupported;
  const int nb = (m + br - 1) / br;
  if (nb < 2 || nb * w > 1024 || nb > 32) return cudaErrorNotSupported;
  if (nb + 1 > pipe_capacity<256, 4>(num_sms)) return cudaErrorNotSupported;
  PipeArgs a{X, ldx, Xh, ldh, m, w, nb, Rb, S, Rout, ldr, root_is_global, status, col0,
             g_panel_dbg};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nb + 1);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = (int)sizeof(float) * (((256 * 4 * 33 + 3) & ~3) + 64 + 2 * 8 * 32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, panel_pipe_kernel<256, 4>, a);
}


template <int NT, int RPT>
static int fused_capacity(int num_sms) {
  static int per_sm = -1;
  if (per_sm < 0) {
    const int smem = FusedShape<NT, RPT>::SMEM;
    cudaFuncSetAttribute(panel_fused_kernel<NT, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, panel_fused_kernel<NT, RPT>, NT,
                                                      smem) != cudaSuccess)
      per_sm = 0;
  }
  return per_sm * num_sms;
}

int fused_panel_capacity(int num_sms) { return fused_capacity<256, 4>(num_sms); }
int fused_panel_smem_bytes() { return FusedShape<256, 4>::SMEM; }
int fused_panel_max_rows() { return 1024; }

// Plan the tree and launch.  br <= 256 uses the 128 x 2 shape, else the 256 x 4 shape (br <=
// 1024).  ws: float scratch (node R's and stack-Q slices), iws: zeroed int scratch (counters,
// flags) that the kernel leaves zeroed.  cudaErrorNotSupported if the tree does not fit the
// co-resident grid (the caller then uses the multi-launch path).
cudaError_t panel_fused(int m, int w, float* X, long long ldx, __half* Xh, long long ldh, int br,
                        float* Rout, long long ldr, int root_is_global, int* status, int col0,
                        float* ws, long long ws_cap, int* iws, long long iws_cap, int num_sms,
                        cudaStream_t st) {
  const bool big = br > 256;
  if (w < 1 || w > 32 || br > 1024) return cudaErrorNotSupported;
  FusedPanelArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.Xh = Xh;
  a.ldh = ldh;
  a.m = m;
  a.w = w;
  a.br = br;
  a.nb = (m + br - 1) / br;
  if (a.nb < 1) a.nb = 1;
  const int cap = big ? fused_capacity<256, 4>(num_sms) : fused_capacity<128, 2>(num_sms);
  if (a.nb > cap) return cudaErrorNotSupported;
  a.F = br / w;
  if (a.F < 2) return cudaErrorNotSupported;
  a.nodes[0] = a.nb;
  int L = 0;
  while (a.nodes[L] > 1) {
    if (L + 1 > kMaxLevels) return cudaErrorNotSupported;
    a.nodes[L + 1] = (a.nodes[L] + a.F - 1) / a.F;
    ++L;
  }
  a.L = L;
  long long off = 0, ioff = 0;
  const long long ww = (long long)w * w;
  for (int l = 0; l <= L; ++l) {
    a.Rbuf[l] = ws + off;
    off += a.nodes[l] * ww;
    if (l >= 1) {
      a.Qst[l] = ws + off;
      off += a.nodes[l - 1] * ww;
      a.cnt[l] = iws + ioff;
      ioff += a.nodes[l];
    }
  }
  a.done = iws + ioff;
  ioff += 2;
  if (off > ws_cap || ioff > iws_cap) return cudaErrorNotSupported;
  a.Rout = Rout;
  a.ldr = ldr;
  a.root_is_global = root_is_global;
  a.status = status;
  a.col0 = col0;
  a.dbg = g_panel_dbg;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nb);
  cfg.blockDim = dim3(big ? 256 : 128);
  cfg.dynamicSmemBytes = big ? FusedShape<256, 4>::SMEM : FusedShape<128, 2>::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = (a.L > 0) ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return big ? cudaLaunchKernelEx(&cfg, panel_fused_kernel<256, 4>, a)
             : cudaLaunchKernelEx(&cfg, panel_fused_kernel<128, 2>, a);
}

}  // namespace tcqr

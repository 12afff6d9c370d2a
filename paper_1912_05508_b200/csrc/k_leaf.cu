// k_leaf.cu -- K2L: a whole leaf of Alg. 2 (w <= 128 columns, every node below the tensor-core
// cutoff) in ONE cooperative launch, one CTA per 256-row block, the block's rows of all the leaf's
// columns resident in shared memory from the first panel to the last.
//
// The leaf is the same recursion as Alg. 2: split h = 32 ceil(w/64) (R-A2),
// FP32 products below the cutoff (R-A1), 32-column CAQR panels (Eq. (6)).  The
// host flattens it into a short program of ops that the kernel runs in order:
//
//   PANEL(c0, pw)   Eq. (6) on columns [c0, c0+pw):
//     (1) Alg. 4 (MGS) on every 64 x pw block of the CTA's rows -- four blocks
//         per CTA, one warp each (the paper's 256 x 32 submatrices, cut to 64
//         rows so a block's reductions stay inside one warp: lane j holds column j of the block,
//         the pivot column and the normalized q_k are broadcast through shared memory, every
//         norm and dot is a lane-local FFMA2 chain; no CTA barrier per MGS step).  Q_b in place
//         in shared memory, R_b (pw x pw, FP64) in shared memory;
//     (2)-(3) the stack [R_1; ...; R_nb] is factored through its Gram matrix in FP64:
//         G = sum_b R_b' R_b (each product exact in FP64, fixed-order sums), R = chol(G) (one
//         warp, redundantly in every CTA), and the stack's Q slice of block b is S_b = R_b R^-1
//         (forward substitution, one warp per block, after the Cholesky).  This is a QR of the
//         stacked R's (G = R'R, diag(R) > 0 -- the unique R of Eq. (6) step (3)); reading R-B1 in
//         the paper factors the stack with the same MGS kernel, here the FP64 Gram
//         route takes the 32-step dependency chain out of FP32 block reductions;
//     (4) Q_b <- Q_b S_b in shared memory (S_b upper triangular: only its nonzero terms).
//   PROJ(c0, h, w2) Alg. 2 lines 8-9 in FP32 below the cutoff: R12 = Q1' A2 (per-CTA partial over
//     its rows, fixed-order sum over the CTAs), R block <- R12, A2 -= Q1 R12.
//
// Cross-CTA steps (the Gram / R12 sums) go through L2 as tagged words, without grid barriers:
// every CTA stores its partial as 64-bit words {payload, tag} (tag = the reduction's sequence
// number in the factorization), the owner CTA of each 32-entry chunk polls the nb partials of its
// entries until their tags match, sums them in a fixed order and stores the tagged sum, and every
// CTA polls the sums it needs.  Each value is its own ready flag (an 8-byte store is single-copy
// atomic), so a reduction costs two L2 round trips instead of two grid barriers plus a pass; the
// words are zeroed once per factorization (tags start at 1).  Every CTA computes the 32 x 32
// Cholesky redundantly (same inputs, same code: bit-identical R everywhere).  At the end each CTA writes its rows of the final Q (FP32 and the
// FP16 shadow the tensor-core GEMMs above read) and CTA 0 has written the leaf's R blocks.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace tcqr {

namespace {

constexpr int kNT = 256;      // threads per CTA
constexpr int kRows = 256;    // rows per CTA (max)
constexpr int kCols = 128;    // leaf width (max)
constexpr int kLd = 132;      // shared row stride in floats: 16-byte rows, 4 floats of skew
constexpr int kMaxOps = 16;
constexpr int kNW = kNT / 32;
constexpr int kBR = 64;       // rows per MGS block (4^3: powers of 4 keep the planted pin exact)
constexpr int kMW = kRows / kBR;  // MGS blocks (= warps) per CTA: one per SM sub-partition
constexpr int kLdR = 33;      // ld of the blocks' R_b (FP64) in shared memory
constexpr int kLdS = 36;      // ld of the blocks' S_b (FP32; 16-byte rows: four columns per load)

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
  unsigned long long* tg;  // tagged words (leaf_tag_words(), zeroed before the first leaf)
  unsigned tag0;           // reductions of the earlier launches (the host counts them)
  int* status;    // breakdown status (null: local leaf of a rank, zero norms allowed, R-A8)
  int col0;       // global column of the leaf's column 0 (breakdown codes)
  unsigned long long* dbg;  // optional phase timestamps of CTA 0 (globaltimer ns), 128 slots
  unsigned long long* trace;  // optional per-launch trace: [0] count, then CTA 0 (start, end) pairs
};

struct Smem {
  float L[kRows * kLd];        // the block's rows of the leaf, row-major
  double Rbd[kMW][32 * kLdR];  // R_b of each MGS block of the current panel, row-major (FP64)
  union {
    float T[4096];             // PROJ: R12 (row-major [i][w2p]) / group partials; Gram wsum
    float Sf[kMW][32 * kLdS];  // PANEL: S_b of each block (FP32), row-major [l][j]
    double Gp[kMW][528];       // PANEL: each block's Gram R_b' R_b, packed upper triangle
  } u;
  double Rd[32 * 34 + 34];     // the panel's R in FP64, row-major (ld 34; one row of slack)
  double rowb[kMW][2][64];     // Cholesky: row k of R twice over, per chain warp (step parity)
  float colbuf[kMW][kBR];      // MGS: the pivot column of each block
  double Gs[528];              // PANEL: the stack's Gram (packed upper triangle), from the owners
  float wsum[kNW * 32];        // per-warp partial sums of the cross-CTA reductions (FP32)
  double wsumd[kNW * 32];      //   (FP64)
};

// tagged-word layout (u64 words): [0] abort word; Gram partials nb x 528 entries x 2 words (low,
// high half of the FP64 value); Gram sums 528 x 2; projection partials nb x 4096; sums 4096
constexpr long long kTgGP = 8;
constexpr long long kTgGS = kTgGP + 148LL * 528 * 2;
constexpr long long kTgPP = kTgGS + 528 * 2;
constexpr long long kTgPS = kTgPP + 148LL * 4096;
constexpr long long kTgWords = kTgPS + 4096;

// Tagged words: {payload (low 32 bits), tag (high 32 bits)}, stored and polled at GPU scope (L2).
__device__ __forceinline__ void st_tag(unsigned long long* p, unsigned payload, unsigned tag) {
  const unsigned long long v = ((unsigned long long)tag << 32) | payload;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tag(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_tag2(unsigned long long* p, unsigned lo, unsigned hi,
                                        unsigned tag) {
  const unsigned long long v0 = ((unsigned long long)tag << 32) | lo;
  const unsigned long long v1 = ((unsigned long long)tag << 32) | hi;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v0), "l"(v1) : "memory");
}
__device__ __forceinline__ void ld_tag2(const unsigned long long* p, unsigned long long& v0,
                                        unsigned long long& v1) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "l"(p) : "memory");
}
// Watchdog of the polls: a value still missing after 2 s (a co-residency failure) raises the
// abort word, which releases every other waiter of the launch, and the launch reports
// TCQR_ERR_CUDA through the status word, so a bug fails the call instead of hanging the device.
__device__ __noinline__ bool poll_watchdog(const LeafArgs& a, unsigned long long& t0) {
  if (ld_tag(a.tg) != 0ull) return true;
  unsigned long long now;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
  if (t0 == 0) {
    t0 = now;
  } else if (now - t0 > 2000000000ull) {
    st_tag(a.tg, 1u, 1u);
    if (a.status) atomicMin(a.status, -1001);
    return true;
  }
  return false;
}
// Load the words p[i] (null: none) until every one carries `tag`; each round re-issues the loads
// of all the words still missing together (one L2 round trip per round).
// Pairs (p[2i], p[2i] + 1) loaded with one 16-byte load; each half still carries its own tag.
template <int N>
__device__ __forceinline__ void poll_pairs(const LeafArgs& a, unsigned long long (&v)[2 * N],
                                           const unsigned long long* const (&p)[N],
                                           unsigned tag) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    v[2 * i] = v[2 * i + 1] = 0ull;
    if (p[i]) ld_tag2(p[i], v[2 * i], v[2 * i + 1]);
  }
  unsigned long long t0 = 0;
  for (unsigned it = 1;; ++it) {
    bool done = true;
#pragma unroll
    for (int i = 0; i < N; ++i)
      done &= !p[i] || ((unsigned)(v[2 * i] >> 32) == tag && (unsigned)(v[2 * i + 1] >> 32) == tag);
    if (done) return;
    __nanosleep(64);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (p[i] && ((unsigned)(v[2 * i] >> 32) != tag || (unsigned)(v[2 * i + 1] >> 32) != tag))
        ld_tag2(p[i], v[2 * i], v[2 * i + 1]);
    if ((it & 255) == 0 && poll_watchdog(a, t0)) return;
  }
}
template <int N>
__device__ __forceinline__ void poll_words(const LeafArgs& a, unsigned long long (&v)[N],
                                           const unsigned long long* const (&p)[N],
                                           unsigned tag) {
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = p[i] ? ld_tag(p[i]) : 0ull;
  unsigned long long t0 = 0;
  for (unsigned it = 1;; ++it) {
    bool done = true;
#pragma unroll
    for (int i = 0; i < N; ++i) done &= !p[i] || (unsigned)(v[i] >> 32) == tag;
    if (done) return;
    __nanosleep(64);  // back off: a storm of polls would slow the stores it waits for
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (p[i] && (unsigned)(v[i] >> 32) != tag) v[i] = ld_tag(p[i]);
    if ((it & 255) == 0 && poll_watchdog(a, t0)) return;
  }
}
template <typename T>
struct TagWords;
template <>
struct TagWords<float> {
  static constexpr int W = 1;
  __device__ static void put(unsigned long long* p, float v, unsigned tag) {
    st_tag(p, __float_as_uint(v), tag);
  }
  __device__ static float get(const unsigned long long* v) { return __uint_as_float((unsigned)v[0]); }
};
template <>
struct TagWords<double> {
  static constexpr int W = 2;
  __device__ static void put(unsigned long long* p, double v, unsigned tag) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    st_tag2(p, (unsigned)b, (unsigned)(b >> 32), tag);  // one 16-byte store (each half tagged)
  }
  __device__ static double get(const unsigned long long* v) {
    return __longlong_as_double((long long)(((v[1] & 0xffffffffull) << 32) | (v[0] & 0xffffffffull)));
  }
};

__device__ __forceinline__ void leaf_ts(const LeafArgs& a, int& slot) {
  if (a.dbg && blockIdx.x == 0 && threadIdx.x == 0 && slot < 128) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[slot] = v;
  }
  ++slot;
}

// CTA b's rows start at leaf_row(b): balanced in row quads (16-byte loads), the last CTA ragged
__device__ __forceinline__ int leaf_row(int b, int m, int nb) {
  const long long mq = (m + 3) / 4;
  return (int)min((long long)m, 4 * ((long long)b * mq / nb));
}

// Fixed-order cross-CTA sum of tagged partials: out[e] = sum_{b=0..nb-1} part[b][e] for the
// entries e in [0, E) owned by this CTA (chunks of 32 consecutive entries, chunk c on CTA c % nb).
// Lane = entry (coalesced loads of one partial row per warp), warp w sums the partials b = w,
// w + 8, ... in increasing order (up to 16 partials in flight, polled until their tags match, with
// a short back-off between rounds), then the 8 warp sums are added in warp order and stored
// tagged.  Deterministic.  (Measured, tools/micro/xcta_reduce.cu: 2.9 us for 528 FP64 entries on
// 128 CTAs against 4.6 us for barrier + sum + barrier.)  Projection sums also go to the R block.
template <typename T>
__device__ __forceinline__ void tagged_sum(const LeafArgs& a, const unsigned long long* part,
                                           long long pstride, int E, unsigned tag,
                                           unsigned long long* out, T* wsum, int h, int w2,
                                           int w2p, int c0, bool to_r) {
  constexpr int W = TagWords<T>::W, NBT = 16, N = NBT * W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunks = (E + 31) / 32;
  for (int c = blockIdx.x; c < nchunks; c += a.nb) {
    const int e = c * 32 + lane;
    T s = 0;
    if (e < E) {
      for (int b0 = warp; b0 < a.nb; b0 += NBT * kNW) {
        unsigned long long v[N];
        if constexpr (W == 2) {
          const unsigned long long* p[NBT];
#pragma unroll
          for (int u = 0; u < NBT; ++u) {
            const int b = b0 + u * kNW;
            p[u] = b < a.nb ? part + b * pstride + e * W : nullptr;
          }
          poll_pairs<NBT>(a, v, p, tag);
        } else {
          const unsigned long long* p[N];
#pragma unroll
          for (int u = 0; u < NBT; ++u) {
            const int b = b0 + u * kNW;
            p[u] = b < a.nb ? part + b * pstride + e : nullptr;
          }
          poll_words<N>(a, v, p, tag);
        }
#pragma unroll
        for (int u = 0; u < NBT; ++u)
          if (b0 + u * kNW < a.nb) s += TagWords<T>::get(v + u * W);
      }
    }
    wsum[warp * 32 + lane] = s;
    __syncthreads();
    if (warp == 0 && e < E) {
      T t = wsum[lane];
#pragma unroll
      for (int u = 1; u < kNW; ++u) t += wsum[u * 32 + lane];
      TagWords<T>::put(out + e * W, t, tag);
      if (to_r) {  // projection: R(c0 + i, c0 + h + j) = R12(i, j)
        const int i = e / w2p, j = e % w2p;
        if (i < h && j < w2) a.R[(c0 + i) + (long long)(c0 + h + j) * a.ldr] = (float)t;
      }
    }
    __syncthreads();
  }
}

// Every CTA: dst[e] = the tagged sums out[e], e in [0, E) (up to 16 entries per thread in flight)
template <typename T>
__device__ __forceinline__ void tagged_gather(const LeafArgs& a, const unsigned long long* out,
                                              int E, unsigned tag, T* dst) {
  constexpr int W = TagWords<T>::W, U = 16 / W, N = U * W;
  for (int e0 = threadIdx.x; e0 < E; e0 += U * kNT) {
    unsigned long long v[N];
    if constexpr (W == 2) {
      const unsigned long long* p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) p[u] = e0 + u * kNT < E ? out + (e0 + u * kNT) * W : nullptr;
      poll_pairs<U>(a, v, p, tag);
    } else {
      const unsigned long long* p[N];
#pragma unroll
      for (int u = 0; u < U; ++u) p[u] = e0 + u * kNT < E ? out + e0 + u * kNT : nullptr;
      poll_words<N>(a, v, p, tag);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * kNT < E) dst[e0 + u * kNT] = TagWords<T>::get(v + u * W);
  }
  __syncthreads();
}

// Alg. 4 on MGS block `blk` = rows [64 blk, 64 blk + 64) of the CTA, columns
// [c0, c0 + pw), by one warp.  Lane j holds column j of the block (rows in FP32 pairs, FFMA2).
// Step k: the pivot column x_k (published in colbuf by lane k) is broadcast to every lane; lane j
// forms a_k' a_j over the block's 64 rows (lane k: the norm^2); R(k, k) = sqrt, one correctly
// rounded reciprocal (reading R-B2); R(k, j) = (a_k' a_j) / R(k, k) (R-A7); q_k = x_k / R(k, k)
// (line 6) is formed by every lane from its copy of x_k (lane r writes rows r, r + 32 to L as the
// block's final Q column k); lines 7-8 update every lane's column by FFMA2.  A locally
// zero norm gives q = 0, r = 0 (R-A8; only the stack's Cholesky reports breakdowns).  Afterwards
// the warp forms the block's Gram R_b' R_b (FP64, packed upper triangle) for the stack.
__device__ __forceinline__ void mgs_warp(Smem& s, int blk, int c0, int pw) {
  const int lane = threadIdx.x & 31;
  const int r0 = blk * kBR;
  float* colb = s.colbuf[blk];
  double* Rb = s.Rbd[blk];
  float2 x[kBR / 2];  // x[i] = rows (r0 + 2i, r0 + 2i + 1) of column c0 + lane
#pragma unroll
  for (int i = 0; i < kBR / 2; ++i)
    x[i] = make_float2(s.L[(r0 + 2 * i) * kLd + c0 + lane], s.L[(r0 + 2 * i + 1) * kLd + c0 + lane]);
#pragma unroll 4
  for (int k = 0; k < 32; ++k) Rb[k * kLdR + lane] = 0.0;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < kBR / 4; ++i)
      *reinterpret_cast<float4*>(colb + 4 * i) = make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x,
                                                             x[2 * i + 1].y);
  }
  __syncwarp();
#pragma unroll 1
  for (int k = 0; k < pw; ++k) {
    float2 v[kBR / 2];
#pragma unroll
    for (int i = 0; i < kBR / 4; ++i) {
      const float4 c4 = *reinterpret_cast<const float4*>(colb + 4 * i);
      v[2 * i] = make_float2(c4.x, c4.y);
      v[2 * i + 1] = make_float2(c4.z, c4.w);
    }
    float2 acc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < kBR / 2; ++i) acc[i & 3] = ffma2(v[i], x[i], acc[i & 3]);
    const float tot = ((acc[0].x + acc[0].y) + (acc[1].x + acc[1].y)) +
                      ((acc[2].x + acc[2].y) + (acc[3].x + acc[3].y));
    const float rkk = sqrtf(__shfl_sync(0xffffffffu, tot, k));
    const bool zero = !(rkk > 0.f) || !isfinite(rkk);
    const float inv = zero ? 0.f : 1.0f / rkk;  // correctly rounded: the bits of __frcp_rn
    const float rkj = zero ? 0.f : (lane == k ? rkk : tot * inv);
    if (lane >= k && lane < pw) Rb[k * kLdR + lane] = (double)rkj;
    const float q0 = colb[lane] * inv, q1 = colb[lane + 32] * inv;
    s.L[(r0 + lane) * kLd + c0 + k] = q0;
    s.L[(r0 + lane + 32) * kLd + c0 + k] = q1;
    // q_k in every lane's registers: its copy of the pivot column times 1/R(k,k) (x * inv + -0 is
    // x * inv exactly: the same bits as q0 / q1), no shared-memory round trip on the chain
    // (tools/micro/mgs_warp_bench.cu V9: 815 -> 794 cycles per step)
    const float2 iv = make_float2(inv, inv), nz = make_float2(-0.f, -0.f);
#pragma unroll
    for (int i = 0; i < kBR / 2; ++i) v[i] = ffma2(v[i], iv, nz);
    __syncwarp();  // every lane has read colb before lane k + 1 republishes it below
    const float2 nr = make_float2(-rkj, -rkj);
#pragma unroll
    for (int i = 0; i < kBR / 2; ++i) x[i] = ffma2(v[i], nr, x[i]);  // x_j - q_k R(k, j)
    if (lane == k + 1) {
#pragma unroll
      for (int i = 0; i < kBR / 4; ++i)
        *reinterpret_cast<float4*>(colb + 4 * i) =
            make_float4(x[2 * i].x, x[2 * i].y, x[2 * i + 1].x, x[2 * i + 1].y);
    }
    __syncwarp();
  }
}

// The block's Gram G_b(i, j) = sum_{l <= i} R_b(l, i) R_b(l, j), i <= j (lane j: column j of R_b in
// registers, R_b(l, i) broadcast), packed upper triangle into u.Gp[blk]; rows i of parity `half`
// (two warps per block after the MGS: warps b and b + 4, the same entries and order as one warp)
__device__ __forceinline__ void block_gram(Smem& s, int blk, int half, int step) {
  const int lane = threadIdx.x & 31;
  const double* Rb = s.Rbd[blk];
  double rj[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) rj[l] = Rb[l * kLdR + lane];
  double* gp = s.u.Gp[blk];
#pragma unroll
  for (int i = half; i < 32; i += step) {
    double g = 0.0;
#pragma unroll
    for (int l = 0; l <= i; ++l) g = fma(Rb[l * kLdR + i], rj[l], g);
    if (i <= lane) gp[lane * (lane + 1) / 2 + i] = g;
  }
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

struct CholCtx {
  const LeafArgs& a;
  Smem& s;
  float* Sf;
  int warp, lane, c0;
};
// Steps [k0, k1) of the panel's Cholesky + S_b chain (see (3) in leaf_panel); T = live terms of the
// trailing triangle for every step of the phase (31 - k0).  Slots c[T..], r[T..] go stale: from
// step k0 on they stand for rows / columns past 31.
template <int T>
__device__ __forceinline__ void chol_phase(const CholCtx& x, int k0, int k1, double (&c)[32],
                                           double (&r)[32], double& d, bool& ok, double& ri) {
  const int lane = x.lane;
#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    ri = ok ? ri : 0.0;
    const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
    const double dn = fma(-rkj, rkj, c[1]);  // lane k+1: W(k+1,k+1) - R(k,k+1)^2
    d = __shfl_sync(0xffffffffu, dn, (k + 1) & 31);  // next pivot (unused after the last step)
    double* rowk = x.s.rowb[x.warp][k & 1];
    rowk[lane] = rkj;  // twice: rowk[k + 1 + i] is R(k, k+1+i), and 0 past column 31
    rowk[lane + 32] = rkj;
    if (x.warp == 0) {
      x.s.Rd[k * 34 + lane] = rkj;
      if (!ok && lane == 0 && blockIdx.x == 0 && x.a.status)
        atomicMin(x.a.status, x.a.col0 + x.c0 + k + 1);
    }
    const double sk = r[0] * ri;  // S_b(lane, k)
    x.Sf[lane * kLdS + k] = (float)sk;
    ok = d > 0.0 && d <= 1.7976931348623157e308;
    ri = rsqrt_nr(ok ? d : 1.0);
    __syncwarp();
    // R(k, k+1+i); slots past column 31 read R(k, 0..k-1) = 0 from the second copy
    const double* rk = rowk + k + 1;
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const double v = rk[i];
      c[i] = fma(-v, rkj, c[i + 1]);
      r[i] = fma(-sk, v, r[i + 1]);
    }
  }
}

// ---- PANEL ------------------------------------------------------------------------------------
__device__ __noinline__ void leaf_panel(const LeafArgs& a, Smem& s, int nrows, int c0, int pw,
                                        int& slot, bool first, int st_c0, int st_pw, bool defer,
                                        unsigned tag) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // first panel: the upper half (warps 4-7, idle during the MGS) issues the async loads of the
  // leaf's later columns (two rows per thread) beside the MGS instead of before it
  if (first && t >= kNT / 2) {
    leaf_issue_rest(a, s, nrows, t - kNT / 2);
    leaf_issue_rest(a, s, nrows, t);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // (1) Alg. 4 on the CTA's four 64-row blocks, one warp each (rows >= nrows are zero), and each
  // block's Gram R_b' R_b; blocks entirely past the CTA's rows (CTAs of 64 or 128 rows) only clear
  // their R_b and Gram (an all-zero block would take the divide's special-value path every step)
  if (warp < kMW) {
    if (warp * kBR < nrows) {
      mgs_warp(s, warp, c0, pw);
    } else {
#pragma unroll 4
      for (int k = 0; k < 32; ++k) s.Rbd[warp][k * kLdR + lane] = 0.0;
    }
    // zero R_b (blocks past the rows): zero Gram.  First panel: the upper warps are still issuing
    // the leaf's later columns, so each MGS warp takes its whole Gram before the barrier
    if (first) {
      __syncwarp();
      block_gram(s, warp, 0, 1);
    }
  }
  __syncthreads();
  if (!first) {  // later panels: warps b and b + 4 split block b's Gram
    block_gram(s, warp & (kMW - 1), warp / kMW, 2);
    __syncthreads();
  }
  leaf_ts(a, slot);
  // (2) the CTA's part of the stack's Gram: G = (G_0 + G_1) + (G_2 + G_3) (FP64, fixed order;
  // packed upper triangle, zero past the panel), stored tagged; the owners sum the nb partials
  // (fixed order) and every CTA gathers the sum
  for (int e = t; e < 528; e += kNT) {
    int j = (int)((sqrtf(8.f * e + 1.f) - 1.f) * 0.5f);  // e = j (j + 1) / 2 + i, i <= j
    if (j * (j + 1) / 2 > e) --j;
    if ((j + 1) * (j + 2) / 2 <= e) ++j;
    const double g = j < pw ? (s.u.Gp[0][e] + s.u.Gp[1][e]) + (s.u.Gp[2][e] + s.u.Gp[3][e]) : 0.0;
    TagWords<double>::put(a.tg + kTgGP + ((long long)blockIdx.x * 528 + e) * 2, g, tag);
  }
  leaf_ts(a, slot);
  if (a.dbg && t == 0) {  // debug: the latest CTA's publish time of this op
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    atomicMax(a.dbg + 120 + min(7u, tag - a.tag0 - 1u), v);
  }
  tagged_sum<double>(a, a.tg + kTgGP, 528 * 2, 528, tag, a.tg + kTgGS, s.wsumd, 0, 0, 1, 0, false);
  leaf_ts(a, slot);
  tagged_gather<double>(a, a.tg + kTgGS, 528, tag, s.Gs);
  leaf_ts(a, slot);
  if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: Cholesky start
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[100] = v;
  }
  // (3) R = chol(G) and S_b = R_b R^-1, in warps 0-3 (one per SM sub-partition): warp b runs the
  // Cholesky redundantly (same inputs, same code: the same R bits in every warp and CTA) with the
  // forward substitution of ITS block's R_b fused in.  Rolled passes over k (a fully unrolled
  // 32-step chain is instruction-fetch bound) in four phases of eight steps whose inner loops
  // cover only the live part of the trailing triangle (31, 23, 15, 7 terms).  Lane j holds column
  // j of the trailing Gram, c[i] = W(k+i, j) (shifted down one slot per step, so the pivot is
  // always c[0]), and row j of S_b, r[i] = the running value of column k+i.  Step k: the pivot
  // G(k,k) by shuffle, one FP64 reciprocal square root ri = 1/R(k,k) (<= 1 ulp; R(k,j) = W(k,j) ri
  // and the substitution's quotients become products; FP64 values within an ulp round to the
  // same FP32 R and Q, exact inputs stay exact -- the planted pin), row k of R broadcast through
  // the warp's row buffer.  The pivot of step k+1 comes from lane k+1's own values (its update of
  // W(k+1,k+1) with its own R(k,k+1)), so shuffle -> rsqrt starts before the row is in shared
  // memory.
  if (warp < kMW) {
    const double* Rb = s.Rbd[warp];
    float* Sf = s.u.Sf[warp];
    double c[32], r[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) c[i] = (i <= lane && lane < pw) ? s.Gs[lane * (lane + 1) / 2 + i] : 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) r[j] = (lane < pw && j < pw) ? Rb[lane * kLdR + j] : 0.0;
    double d = __shfl_sync(0xffffffffu, c[0], 0);
    bool ok = d > 0.0 && d <= 1.7976931348623157e308;
    double ri = rsqrt_nr(ok ? d : 1.0);
    CholCtx cc{a, s, Sf, warp, lane, c0};
    chol_phase<31>(cc, 0, min(pw, 8), c, r, d, ok, ri);
    chol_phase<23>(cc, 8, min(pw, 16), c, r, d, ok, ri);
    chol_phase<15>(cc, 16, min(pw, 24), c, r, d, ok, ri);
    chol_phase<7>(cc, 24, pw, c, r, d, ok, ri);
#pragma unroll 1
    for (int j = pw; j < 32; ++j) Sf[lane * kLdS + j] = 0.f;
  } else if (st_pw > 0) {
    // the previous panel's deferred Q stores (those columns are final) on the four warps that run
    // no chain
    const int idx = (warp - kMW) * 32 + lane;
#pragma unroll 1
    for (int rr = idx; rr < nrows; rr += 128) leaf_store_row(a, s, rr, st_c0, st_pw);
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
  // (4) Q_b <- Q_b S_b: thread t = row t (block t / 64).  S_b is upper triangular, so column j
  // takes the terms l <= j only, summed in increasing l from zero (the same value as the full
  // product: the skipped terms are exact zeros); one 16-byte load feeds two FFMA2 on column pairs
  // (the quad's extra terms S(l, j < l) are exact zeros too).  Rows l >= pw of S_b are zero.
  if (t < nrows) {
    float* row = s.L + t * kLd + c0;
    const float* Sf = s.u.Sf[t / kBR];
    float q[32];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 q4 = *reinterpret_cast<const float4*>(row + 4 * i);
      q[4 * i] = q4.x;
      q[4 * i + 1] = q4.y;
      q[4 * i + 2] = q4.z;
      q[4 * i + 3] = q4.w;
    }
    float2 y[16];
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) y[j2] = make_float2(0.f, 0.f);
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      const float2 ql = make_float2(q[l], q[l]);
#pragma unroll
      for (int j4 = l / 4; j4 < 8; ++j4) {  // from the quad holding column l (S_b(l, j < l) = 0)
        const float4 s4 = *reinterpret_cast<const float4*>(Sf + l * kLdS + 4 * j4);
        y[2 * j4] = ffma2(ql, make_float2(s4.x, s4.y), y[2 * j4]);
        y[2 * j4 + 1] = ffma2(ql, make_float2(s4.z, s4.w), y[2 * j4 + 1]);
      }
    }
#pragma unroll
    for (int j2 = 0; j2 < 16; ++j2) {
      if (2 * j2 < pw) row[2 * j2] = y[j2].x;
      if (2 * j2 + 1 < pw) row[2 * j2 + 1] = y[j2].y;
    }
  }
  __syncthreads();
  if (a.dbg && blockIdx.x == 0 && t == 0) {  // debug: apply end (before the Q stores)
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    a.dbg[104] = v;
  }
  // these pw columns of Q are final (later ops only read them): stream them out (FP32 and the
  // FP16 shadow), coalesced down each column -- now, or (defer) by the warps that idle beside the
  // next panel's Cholesky
  if (!defer && t < nrows) leaf_store_row(a, s, t, c0, pw);
  leaf_ts(a, slot);
}

// column of entry c (0..7) of column tile tj in the projection's partial R12 (see leaf_proj)
template <int W2P>
__device__ __forceinline__ int tile_col(int tj, int c) {
  if constexpr (W2P == 64)
    return (c < 4 ? 4 * tj : 32 + 4 * tj) + (c & 3);
  else
    return 8 * tj + c;
}

// ---- PROJ: R12 = Q1' A2, R block <- R12, A2 -= Q1 R12 (FP32) ------------------------------------
// H = h (32 or 64), W2P = w2 rounded up to 32 (the columns past the leaf are zero in shared memory
// and stay zero).
template <int H, int W2P>
__device__ __noinline__ void leaf_proj(const LeafArgs& a, Smem& s, int nrows, int c0, int w2,
                                       int& slot, unsigned tag) {
  // partial R12 = Q1' A2 over the CTA's rows: 8 x 8 output tiles, G = 256 / tiles threads per tile
  // (adjacent lanes), thread g of a tile takes the rows g, g + G, ... (two 16-byte loads of Q1 and
  // two of A2 per row feed 32 FFMA2: FMA-bound, where 4 x 4 tiles were shared-memory bound); the
  // G partial tiles are added by a transposing xor-shuffle reduction (each level halves the values a
  // lane keeps, fixed order), after which lane g holds entries [g 64/G, (g+1) 64/G) of the tile
  constexpr int TJ = W2P / 8, TILES = (H / 8) * TJ, G = kNT / TILES, KEEP = 64 / G;
  static_assert(G >= 2 && G <= 32 && (G & (G - 1)) == 0, "tile groups");
  const int t = threadIdx.x;
  asm volatile("cp.async.wait_all;" ::: "memory");  // the leaf's later columns (loaded async)
  __syncthreads();
  const int tile = t / G, grp = t % G;
  const int ti = tile / TJ, tj = tile % TJ;
  float2 acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  {
    const float* q1 = s.L + c0 + 8 * ti;
    // the tile's 8 A2 columns: 8 tj .. 8 tj + 7, or for 8 column tiles (W2P = 64: 4 row groups per
    // tile, so a quarter-warp holds 2 tiles x 4 rows) the quads 4 tj and 32 + 4 tj, which keeps
    // the quarter-warp's 16-byte loads on distinct banks (8 tj would put tiles tj and tj + 4 on
    // the same banks: a 2-way conflict on half the loads)
    const int ca0 = tile_col<W2P>(tj, 0), ca4 = tile_col<W2P>(tj, 4);
    const float* a2 = s.L + c0 + H;
#pragma unroll 2
    for (int r = grp; r < nrows; r += G) {
      const float4 q0 = *reinterpret_cast<const float4*>(q1 + r * kLd);
      const float4 q4 = *reinterpret_cast<const float4*>(q1 + r * kLd + 4);
      const float4 a0 = *reinterpret_cast<const float4*>(a2 + r * kLd + ca0);
      const float4 a4 = *reinterpret_cast<const float4*>(a2 + r * kLd + ca4);
      const float qq[8] = {q0.x, q0.y, q0.z, q0.w, q4.x, q4.y, q4.z, q4.w};
      const float2 av[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w),
                            make_float2(a4.x, a4.y), make_float2(a4.z, a4.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 qi = make_float2(qq[i], qq[i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(qi, av[j], acc[i][j]);
      }
    }
  }
  float v[64];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[8 * i + 2 * j] = acc[i][j].x;
      v[8 * i + 2 * j + 1] = acc[i][j].y;
    }
#pragma unroll
  for (int o = G / 2, hs = 32; o >= 1; o /= 2, hs /= 2) {
    const bool up = (grp & o) != 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      if (k < hs) {
        const float send = up ? v[k] : v[k + hs];
        const float keep = up ? v[k + hs] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
  unsigned long long* pp = a.tg + kTgPP + (long long)blockIdx.x * 4096;
#pragma unroll
  for (int k = 0; k < KEEP; ++k) {
    const int idx = grp * KEEP + k;
    TagWords<float>::put(pp + (8 * ti + idx / 8) * W2P + tile_col<W2P>(tj, idx % 8), v[k], tag);
  }
  leaf_ts(a, slot);
  tagged_sum<float>(a, a.tg + kTgPP, 4096, H * W2P, tag, a.tg + kTgPS, s.wsum, H, w2, W2P, c0,
                    true);
  leaf_ts(a, slot);
  tagged_gather<float>(a, a.tg + kTgPS, H * W2P, tag, s.u.T);
  leaf_ts(a, slot);
  if (nrows <= 128) {
    // A2 -= Q1 R12 for CTAs of <= 128 rows: thread = row t % 128, columns [jq * W2P/4, ...)
    constexpr int JQ = W2P / 4;
    const int r = t % 128, jq = t / 128 * 2;  // two column quarters per thread: jq, jq + 1
    if (r < nrows) {
      float u[2 * JQ];
#pragma unroll
      for (int j = 0; j < 2 * JQ; ++j) u[j] = 0.f;
      const float* qa = s.L + r * kLd + c0;
#pragma unroll 2
      for (int i4 = 0; i4 < H; i4 += 4) {
        const float4 va = *reinterpret_cast<const float4*>(qa + i4);
        const float qx[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const float4* tr = reinterpret_cast<const float4*>(s.u.T + (i4 + ii) * W2P + jq * JQ);
          const float2 qi = make_float2(qx[ii], qx[ii]);
#pragma unroll
          for (int j4 = 0; j4 < JQ / 2; ++j4) {
            const float4 v = tr[j4];
            const float2 c01 = ffma2(qi, make_float2(v.x, v.y), make_float2(u[4 * j4], u[4 * j4 + 1]));
            const float2 c23 = ffma2(qi, make_float2(v.z, v.w),
                                     make_float2(u[4 * j4 + 2], u[4 * j4 + 3]));
            u[4 * j4] = c01.x;
            u[4 * j4 + 1] = c01.y;
            u[4 * j4 + 2] = c23.x;
            u[4 * j4 + 3] = c23.y;
          }
        }
      }
      float* dst = s.L + r * kLd + c0 + H + jq * JQ;
#pragma unroll
      for (int j4 = 0; j4 < JQ / 2; ++j4) {
        float4 v = *reinterpret_cast<float4*>(dst + 4 * j4);
        v.x -= u[4 * j4];
        v.y -= u[4 * j4 + 1];
        v.z -= u[4 * j4 + 2];
        v.w -= u[4 * j4 + 3];
        *reinterpret_cast<float4*>(dst + 4 * j4) = v;
      }
    }
    __syncthreads();
    leaf_ts(a, slot);
    return;
  }
  // A2 -= Q1 R12: thread = rows rq + 64 rr (rr = 0..3; a warp's lanes take consecutive rows, so
  // the 16-byte loads of Q1 are conflict-free), columns [jq W2P/4, (jq+1) W2P/4): four rows share
  // every (broadcast) load of R12, so the FFMA2 issue dominates; terms summed in increasing i
  constexpr int JC = W2P / 4;
  const int rq = t % 64, jq = t / 64;
  float2 u[4][JC / 2];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int j = 0; j < JC / 2; ++j) u[rr][j] = make_float2(0.f, 0.f);
#pragma unroll 1
  for (int i4 = 0; i4 < H; i4 += 4) {
    float qx[4][4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      const float4 q = *reinterpret_cast<const float4*>(s.L + (rq + 64 * rr) * kLd + c0 + i4);
      qx[rr][0] = q.x;
      qx[rr][1] = q.y;
      qx[rr][2] = q.z;
      qx[rr][3] = q.w;
    }
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const float4* tr = reinterpret_cast<const float4*>(s.u.T + (i4 + ii) * W2P + jq * JC);
#pragma unroll
      for (int j4 = 0; j4 < JC / 4; ++j4) {
        const float4 v = tr[j4];
        const float2 v01 = make_float2(v.x, v.y), v23 = make_float2(v.z, v.w);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const float2 qi = make_float2(qx[rr][ii], qx[rr][ii]);
          u[rr][2 * j4] = ffma2(qi, v01, u[rr][2 * j4]);
          u[rr][2 * j4 + 1] = ffma2(qi, v23, u[rr][2 * j4 + 1]);
        }
      }
    }
  }
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) {
    const int r = rq + 64 * rr;
    if (r < nrows) {
      float* dst = s.L + r * kLd + c0 + H + jq * JC;
#pragma unroll
      for (int j4 = 0; j4 < JC / 4; ++j4) {
        float4 v = *reinterpret_cast<float4*>(dst + 4 * j4);
        v.x -= u[rr][2 * j4].x;
        v.y -= u[rr][2 * j4].y;
        v.z -= u[rr][2 * j4 + 1].x;
        v.w -= u[rr][2 * j4 + 1].y;
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
  leaf_ts(a, slot);
  unsigned long long t_start = 0;
  if (a.trace && blockIdx.x == 0 && t == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_start));
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
  if (a.ops[0].kind != 0) {  // otherwise issued beside the first MGS
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
    const unsigned tag = a.tag0 + 1u + (unsigned)o;  // one reduction per op
    if (op.kind == 0) {
      const bool defer = o != last_panel;
      leaf_panel(a, s, nrows, op.c0, op.h, slot, o == 0, st_c0, st_pw, defer, tag);
      st_c0 = op.c0;
      st_pw = defer ? op.h : 0;
    } else if (op.h == 64) {
      if (op.w2 > 32)
        leaf_proj<64, 64>(a, s, nrows, op.c0, op.w2, slot, tag);
      else
        leaf_proj<64, 32>(a, s, nrows, op.c0, op.w2, slot, tag);
    } else {
      leaf_proj<32, 32>(a, s, nrows, op.c0, op.w2, slot, tag);
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  leaf_ts(a, slot);
  if (a.trace && blockIdx.x == 0 && t == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_end));
    const unsigned long long i = atomicAdd(a.trace, 1ull);
    if (i < 4095) {
      a.trace[1 + 2 * i] = t_start;
      a.trace[2 + 2 * i] = t_end;
    }
  }
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

// X (m x w, ldx) <- X S, S (w x w, lds) a dense FP32 block, w <= 128, in place; the FP16 shadow
// of the result into Xh when non-null.  CTA = 64 rows: the rows and S are staged in shared memory
// (the CTA reads all its rows before writing any), thread (warp g, lane) accumulates rows
// 8g..8g+7 x columns lane + 32u in the fixed l order (deterministic).
constexpr int kApRows = 64;
__global__ void __launch_bounds__(256) apply_right_kernel(int m, int w, float* X, long long ldx,
                                                          const float* S, long long lds,
                                                          __half* Xh, long long ldh) {
  extern __shared__ __align__(16) float ap_smem[];
  float* Ss = ap_smem;                    // [w][128] row l, column j
  float* Xs = ap_smem + 128 * 128;        // [kApRows][w + 1]
  const int t = threadIdx.x, lane = t & 31, g = t >> 5;
  const long long row0 = (long long)blockIdx.x * kApRows;
  const int rows = (int)(m - row0 < kApRows ? m - row0 : kApRows);
  const int ldxs = w + 1;
  for (int e = t; e < w * w; e += 256) {
    const int l = e % w, j = e / w;  // coalesced down the columns of S
    Ss[l * 128 + j] = S[l + (long long)j * lds];
  }
  for (int e = t; e < kApRows * w; e += 256) {
    const int r = e % kApRows, l = e / kApRows;
    Xs[r * ldxs + l] = r < rows ? X[row0 + r + (long long)l * ldx] : 0.f;
  }
  __syncthreads();
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[i][u] = 0.f;
  for (int l = 0; l < w; ++l) {
    float sv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sv[u] = Ss[l * 128 + lane + 32 * u];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float xv = Xs[(8 * g + i) * ldxs + l];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[i][u] = fmaf(xv, sv[u], acc[i][u]);
    }
  }
  __syncthreads();
  // transpose through shared memory for column-coalesced stores
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (lane + 32 * u < w) Xs[(8 * g + i) * ldxs + lane + 32 * u] = acc[i][u];
  __syncthreads();
  for (int e = t; e < kApRows * w; e += 256) {
    const int r = e % kApRows, j = e / kApRows;
    if (r < rows) {
      const float v = Xs[r * ldxs + j];
      X[row0 + r + (long long)j * ldx] = v;
      if (Xh) Xh[row0 + r + (long long)j * ldh] = __float2half_rn(v);
    }
  }
}

}  // namespace

cudaError_t apply_right(int m, int w, float* X, long long ldx, const float* S, long long lds,
                        __half* Xh, long long ldh, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  if (w < 1 || w > 128) return cudaErrorInvalidValue;
  const int smem = (int)sizeof(float) * (128 * 128 + kApRows * (128 + 1));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(apply_right_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  apply_right_kernel<<<(m + kApRows - 1) / kApRows, 256, smem, st>>>(m, w, X, ldx, S, lds, Xh,
                                                                      ldh);
  return cudaGetLastError();
}

namespace {

// Replicated leaf across ranks (tcqr.cu leaf_replicated): the rank's m x w rows packed into an
// mpad x w column-major block (zero rows past m) for the allgather, and its rows of the factored
// full panel unpacked back into X with the FP16 shadow (Xh nullable).
__global__ void pack_rows_kernel(int m, int w, const float* __restrict__ X, long long ldx, int mpad,
                                 float* __restrict__ dst) {
  const long long total = (long long)mpad * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % mpad), j = (int)(e / mpad);
    dst[e] = i < m ? X[i + (long long)j * ldx] : 0.f;
  }
}
__global__ void unpack_rows_kernel(int m, int w, const float* __restrict__ src, long long lds,
                                   float* __restrict__ X, long long ldx, __half* __restrict__ Xh,
                                   long long ldh) {
  const long long total = (long long)m * w;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % m), j = (int)(e / m);
    const float v = src[i + (long long)j * lds];
    X[i + (long long)j * ldx] = v;
    if (Xh) Xh[i + (long long)j * ldh] = __float2half_rn(v);
  }
}

}  // namespace

cudaError_t pack_rows(int m, int w, const float* X, long long ldx, int mpad, float* dst,
                      cudaStream_t st) {
  const long long total = (long long)mpad * w;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  pack_rows_kernel<<<std::max(grid, 1), 256, 0, st>>>(m, w, X, ldx, mpad, dst);
  return cudaGetLastError();
}
cudaError_t unpack_rows(int m, int w, const float* src, long long lds, float* X, long long ldx,
                        __half* Xh, long long ldh, cudaStream_t st) {
  const long long total = (long long)m * w;
  const int grid = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  unpack_rows_kernel<<<std::max(grid, 1), 256, 0, st>>>(m, w, src, lds, X, ldx, Xh, ldh);
  return cudaGetLastError();
}

unsigned long long* g_leaf_dbg = nullptr;
unsigned long long* g_leaf_trace = nullptr;
unsigned long long* g_leaf_dbg_multi = nullptr;
unsigned g_leaf_dbg_idx = 0;

size_t leaf_tag_words() { return (size_t)kTgWords; }

cudaError_t leaf_fused(int m, int wl, float* X, long long ldx, __half* Xh, long long ldh, float* R,
                       long long ldr, int col0, int* status, unsigned long long* tg,
                       unsigned* tag_seq, int num_sms, cudaStream_t st) {
  if (wl < 1 || wl > kCols || m < wl) return cudaErrorNotSupported;
  // rows per CTA: the fewest 64-row MGS blocks per CTA that still fit the rows in one CTA per SM
  // of the budget (the MGS and Cholesky chains take the same time for 1 to 4 blocks, the
  // projections and the Q_b S_b apply scale with the CTA's rows)
  // (64-row MGS blocks and power-of-two CTA heights: a block never straddles two CTAs, and the
  // planted pin's blocks stay Hadamard-exact)
  const int rows_cta = m <= num_sms * 64 ? 64 : (m <= num_sms * 128 ? 128 : kRows);
  const int nb = (m + rows_cta - 1) / rows_cta;
  static int per_sm = -1;
  const int smem = (int)sizeof(Smem);
  if (per_sm < 0) {
    cudaFuncSetAttribute(leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, leaf_kernel, kNT, smem) !=
        cudaSuccess)
      per_sm = 0;
  }
  if (nb > per_sm * num_sms || nb > 148) return cudaErrorNotSupported;
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
  a.tg = tg;
  a.tag0 = tag_seq[0];
  a.status = status;
  a.col0 = col0;
  a.dbg = g_leaf_dbg_multi ? g_leaf_dbg_multi + 128 * (g_leaf_dbg_idx++ & 127) : g_leaf_dbg;
  a.trace = g_leaf_trace;
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
  if (e == cudaSuccess) tag_seq[0] += (unsigned)a.nops;  // one reduction per op
  return e;
}

}  // namespace tcqr

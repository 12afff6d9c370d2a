// k_gemm_tc.cu -- K3 / K4: FP16-input, FP32-accumulate tcgen05 GEMMs of Alg. 2 lines 8-9.
//
//   K3 (MODE_TN):  R12 = Q1' * A2          (Alg. 2 line 8)
//       D (h x w2) = A' B, A = fl16(Q1) (m x h), B = fl16(A2 diag(s)) (m x w2): both operands are
//       K-major (the contraction index m is contiguous in the column-major buffers).  Split-K over
//       m is deterministic: each split writes its own FP32 partial, reduced in a fixed order.
//   K4 (MODE_NN):  A2 <- A2 - Q1 * R12     (Alg. 2 line 9 argument)
//       D (m x w2) = A B, A = fl16(Q1) is MN-major (m contiguous), B = fl16(R12 diag(s')) is
//       K-major; the epilogue reads the FP32 A2 tile and writes A2 - D diag(1/s').
//
// Design (sm_100a): persistent warp-specialized CTA, 192 threads:
//   warp 0      TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, mbarrier complete_tx)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (128 x BN x 16 per instruction)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> coalesced column-major stores
// Two TMEM accumulators (2 x BN columns) let the epilogue of tile i overlap the MMAs of tile i+1.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace tcqr {

template <int BN, int MODE, int NBUF = 0>
struct TcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // NN keeps four 128 x 32 FP32 C chunks (16 KB each) for the TMA epilogue; its K = h is short,
  // so fewer mainloop stages suffice
  // NBUF = 0: direct-load epilogue; 2 / 4: TMA epilogue with that many 16 KB C-chunk buffers (4
  // buffers prefetch three chunks ahead for short-K updates at the cost of one mainloop stage; 2
  // keep the full mainloop depth for long K, where the epilogue hides behind the next tile)
  // NBUF = 2 is the short-K update (K = h <= 1024, BN = 128): two mainloop stages, 97 KB of
  // shared memory and 256 TMEM columns, so TWO CTAs share an SM and one CTA's C loads overlap the
  // other's epilogue (the deep levels are HBM-bound on the C read-modify-write)
  static constexpr int CBUF = NBUF * 16384;
  static constexpr int ST = (NBUF == 2) ? 2 : (NBUF == 4) ? ((BN == 128) ? 4 : 3) : ((BN == 128) ? 6 : 4);
  static constexpr int OCC = (NBUF == 2 && BN == 128) ? 2 : 1;  // CTAs per SM
  static constexpr uint32_t TMEM_COLS = 2 * BN;
  static constexpr int SMEM = ST * STAGE + CBUF + 1024 /*align*/ + 256 /*barriers*/;
};

// Work unit w -> (tile row mb, tile column nb, split s).  Tile rows are taken in groups of 16:
// inside a group the row index runs fastest and the column index next, so the tiles in flight at
// once share 16 row blocks of A and a few column blocks of B through L2 (the plain row-fastest
// order streams a different A row block per CTA for every column block: 4x the HBM traffic of
// the top-level update).
__device__ __forceinline__ void tile_of(int w, int tiles_m, int tiles_n, int& mb, int& nb, int& s) {
  constexpr int GM = 16;
  const int per = tiles_m * tiles_n;
  s = w / per;
  const int t = w - s * per;
  const int g = t / (GM * tiles_n);
  const int gm = min(GM, tiles_m - g * GM);
  const int l = t - g * GM * tiles_n;
  mb = g * GM + l % gm;
  nb = l / gm;
}

__constant__ int nn_pre_all = 1;
// L2 policy of the streamed operands and C tiles: evict_first for what one launch reads once (an
// operand whose other dimension fits one tile, the C tiles of the update), so the streams between
// two leaves do not push the whole-leaf kernel's 190 KB of code (and the next leaf's columns) out
// of L2 (measured: a leaf whose code comes from HBM runs 10-20 us longer,
// tools/leaf_phases_insitu.py); operands re-read across tiles keep evict_normal (their L2 reuse).
// The first kKeepCols columns of an update -- the right subtree's first leaf, read next -- keep
// evict_normal.  Bits of the per-launch ef argument:
constexpr int kEfA = 1, kEfB = 2, kEfC = 4;
// host mask (env TCQR_L2_EF): 1 the K1 casts (k_cast.cu), 2 the C tiles, 4 read-once operands,
// 8 every operand.  Default 5 (config 3, interleaved benches: 0 -> 44.50 ms, 5 -> 44.02, 7 -> 44.12,
// 6 -> 44.09; 15 -> +1.2 ms of gaps: the wide levels' operands need their L2 reuse)
constexpr int kL2EfDefault = 5;
constexpr int kKeepCols = 128;
// direct-epilogue C accesses: streaming (evict-first) loads, stores past the kept columns
__device__ __forceinline__ float c_load(int ef, const float* p) { return (ef & kEfC) ? __ldcs(p) : *p; }
__device__ __forceinline__ void c_store(float* p, float v, int col, int ef) {
  if ((ef & kEfC) && col >= kKeepCols)
    __stcs(p, v);
  else
    *p = v;
}

template <int BN, int MODE, int NBUF>
__global__ void __launch_bounds__(192, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, int M, int N, int K, int splits,
                   float* __restrict__ C, long long ldc, long long split_stride,
                   const float* __restrict__ col_mult, int ef) {
  using Cfg = TcCfg<BN, MODE, NBUF>;
  constexpr bool TMAC = NBUF > 0;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, ST = Cfg::ST, STAGE = Cfg::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* cbuf = reinterpret_cast<float*>(smem + ST * STAGE);  // NN: [4][32 cols][128 rows]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE + Cfg::CBUF);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint64_t* cfull = tempty + 2;  // NN: C chunk loaded (4)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cfull + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int nkb = (K + BK - 1) / BK;
  const int total = tiles_m * tiles_n * splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&cfull[i], 1);
    if (TMAC) tma_prefetch_desc(&tmC);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer ----------------
      const uint64_t pol_a = l2_policy(ef & kEfA), pol_b = l2_policy(ef & kEfB);
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x) {
        int mb, nb, s;
        tile_of(w, tiles_m, tiles_n, mb, nb, s);
        const int kb0 = (int)((long long)s * nkb / splits), kb1 = (int)((long long)(s + 1) * nkb / splits);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], STAGE);
          uint8_t* sa = smem + stage * STAGE;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (MODE == kModeTN) {
            tma_load_2d_hint(sa, &tmA, &full[stage], kb * BK, mb * BM, pol_a);
          } else {
            tma_load_2d_hint(sa, &tmA, &full[stage], mb * BM, kb * BK, pol_a);
            tma_load_2d_hint(sa + 8192, &tmA, &full[stage], mb * BM + 64, kb * BK, pol_a);
          }
          tma_load_2d_hint(sb, &tmB, &full[stage], kb * BK, nb * BN, pol_b);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = make_idesc_f16(128, BN, MODE == kModeNN ? 1 : 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = blockIdx.x; w < total; w += gridDim.x, ++it) {
        const int s = w / (tiles_m * tiles_n);
        const int kb0 = (int)((long long)s * nkb / splits), kb1 = (int)((long long)(s + 1) * nkb / splits);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t base_a = smem_u32(smem + stage * STAGE);
          const uint32_t base_b = base_a + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            uint64_t da;
            if (MODE == kModeTN)
              da = make_sw128_desc(base_a + kk * 32, 16, 1024);
            else
              da = make_sw128_desc(base_a + kk * 2048, 8192, 1024);
            const uint64_t db = make_sw128_desc(base_b + kk * 32, 16, 1024);
            mma_f16_ss(tacc, da, db, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (TMAC) {
    // ---------------- NN epilogue through TMA (warps 2..5) ----------------
    // 128 x 32 FP32 chunks of C: TMA-loaded up to three chunks ahead into four shared buffers,
    // updated in place (C - D diag(col_mult)), TMA-stored back.  One elected thread issues the
    // copies; the buffers are [col][row] (row fastest), so thread (row) accesses are conflict-free.
    const int q = warp & 3;
    const int rt = q * 32 + lane;  // row within the tile (= TMEM lane)
    const bool issuer = (warp == 2 && lane == 0);
    const uint64_t pol_ef = l2_policy(ef & kEfC), pol_n = l2_policy(0);
    uint32_t cph = 0;
    int it = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++it) {
      int mb, nb, s_unused;
      tile_of(w, tiles_m, tiles_n, mb, nb, s_unused);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int ncol = min(BN, N - nb * BN), nch = (ncol + 31) / 32;
      // PRE chunks of C in flight: every buffer is refilled as soon as its chunk's store has read
      // it (env TCQR_NN_PRE_ALL=0: NBUF - 1 ahead, the buffer of chunk c - 1 refilled for c + 3)
      const int pre = nn_pre_all ? NBUF : NBUF - 1;
      if (issuer) {
        bulk_wait_read<0>();  // the previous tile's stores have read their buffers
        for (int c = 0; c < pre && c < nch; ++c) {
          mbar_arrive_expect_tx(&cfull[c], 16384);
          tma_load_2d_hint(cbuf + c * 4096, &tmC, &cfull[c], mb * BM, nb * BN + 32 * c, pol_ef);
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        const int buf = c % (NBUF > 0 ? NBUF : 1);
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + 32 * c, r);
        mbar_wait(&cfull[buf], (cph >> buf) & 1);
        cph ^= 1u << buf;
        tmem_ld_wait();
        float* cb = cbuf + buf * 4096;
        const int col0 = nb * BN + 32 * c;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = col0 + j;
          const float mlt = col_mult ? (col < N ? __ldg(col_mult + col) : 0.f) : 1.f;
          cb[j * 128 + rt] = cb[j * 128 + rt] - __uint_as_float(r[j]) * mlt;
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the TMA store
        named_bar_sync(1, 128);
        if (issuer) {
          tma_store_2d_hint(&tmC, cb, mb * BM, col0, col0 >= kKeepCols ? pol_ef : pol_n);
          bulk_commit();
          if (c + pre < nch) {
            // the buffer of chunk c + pre was last used by chunk c + pre - NBUF (c or c - 1),
            // whose store must have read it
            const int nbuf = (c + pre) % NBUF;
            if (pre == NBUF)
              bulk_wait_read<0>();
            else
              bulk_wait_read<1>();
            mbar_arrive_expect_tx(&cfull[nbuf], 16384);
            tma_load_2d_hint(cbuf + nbuf * 4096, &tmC, &cfull[nbuf], mb * BM, nb * BN + 32 * (c + pre),
                             pol_ef);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (issuer) bulk_wait<0>();
  } else {  // ---------------- epilogue warps 2..5 ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int it = 0;
    for (int w = blockIdx.x; w < total; w += gridDim.x, ++it) {
      int mb, nb, s;
      tile_of(w, tiles_m, tiles_n, mb, nb, s);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row = mb * BM + q * 32 + lane;
      const bool rok = row < M;
      // NN: the first chunk of the FP32 C tile is loaded BEFORE waiting for the accumulator
      // (overlaps the mainloop); later chunks are prefetched one chunk ahead.
      float cv[32];
      if (MODE == kModeNN) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = nb * BN + j;
          cv[j] = (rok && col < N) ? c_load(ef, C + row + (long long)col * ldc) : 0.f;
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c, r);
        const int col0 = nb * BN + c;
        if (MODE == kModeTN) {
          tmem_ld_wait();
          if (rok) {
            float* out = C + (splits > 1 ? (long long)s * split_stride : 0LL) + row;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < N) {
                float v = __uint_as_float(r[j]);
                if (splits == 1 && col_mult) v *= __ldg(col_mult + col);
                out[(long long)col * ldc] = v;
              }
            }
          }
        } else {
          float cn[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = col0 + 32 + j;
            cn[j] = (rok && c + 32 < BN && col < N) ? c_load(ef, C + row + (long long)col * ldc) : 0.f;
          }
          tmem_ld_wait();
          if (rok) {
            float* out = C + row;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < N) {
                const float mlt = col_mult ? __ldg(col_mult + col) : 1.f;
                c_store(out + (long long)col * ldc, cv[j] - __uint_as_float(r[j]) * mlt, col, ef);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) cv[j] = cn[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<Cfg::TMEM_COLS>(tmem_base);
  }
}

// ------------------------------------------------------------------------------------------
// K3 on CTA pairs (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 256 tile of
// R12 = A' B.  Each CTA stages its own 128 rows of A (M = h) and its own 128 columns of B
// (N = w2) per K-block, both CTAs' TMA loads complete on the leader's full barrier, and the
// leader issues one 256 x 256 x 16 tcgen05.mma per K step that reads both CTAs' shared
// operands (halving the shared-memory operand traffic per SM of the 1-CTA 128 x 256 tile).  Each
// CTA's TMEM holds its 128 accumulator rows; the commits multicast to both CTAs' barriers.
// Deterministic split-K exactly as the 1-CTA kernel (own partial per split, fixed-order sum).
// ------------------------------------------------------------------------------------------
struct Tc2Cfg {
  static constexpr int BM = 128, BN = 256, BK = 64;  // per CTA: 128 A rows, 128 B columns
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;    // 32 KB
  static constexpr int ST = 6;
  static constexpr uint32_t TMEM_COLS = 2 * BN;      // two 256-column accumulators
  static constexpr int SMEM = ST * STAGE + 1024 + 256;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the leader CTA's copy of a shared-memory object (shared::cluster address, rank bit cleared)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  return smem_u32(p) & 0xFEFFFFFFu;
}

template <int MODE>
__global__ void __launch_bounds__(192, 1) __cluster_dims__(2, 1, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmB, int M, int N, int K, int splits,
                       float* __restrict__ C, long long ldc, long long split_stride,
                       const float* __restrict__ col_mult, int ef) {
  using Cfg = Tc2Cfg;
  constexpr int BK = Cfg::BK, ST = Cfg::ST, STAGE = Cfg::STAGE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int tiles_m = (M + 255) / 256, tiles_n = (N + 255) / 256;
  const int nkb = (K + BK - 1) / BK;
  const int total = tiles_m * tiles_n * splits;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // four epilogue warps in each CTA of the pair
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialized, TMEM allocated
  __syncthreads();     // (also a CTA barrier: compute-sanitizer's racecheck orders the tcgen05.alloc
                       // write of tmem_slot before the reads below only through a CTA barrier)
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs) ----------------
      const uint64_t pol_a = l2_policy(ef & kEfA), pol_b = l2_policy(ef & kEfB);
      int stage = 0;
      uint32_t phase = 0;
      for (int w = pair; w < total; w += npairs) {
        int mb, nb, s;
        tile_of(w, tiles_m, tiles_n, mb, nb, s);
        const int kb0 = (int)((long long)s * nkb / splits), kb1 = (int)((long long)(s + 1) * nkb / splits);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * STAGE);  // both CTAs' bytes
          uint8_t* sa = smem + stage * STAGE;
          uint8_t* sb = sa + Cfg::A_BYTES;
          const uint32_t bar = leader_addr(&full[stage]);
          if (MODE == kModeTN) {
            asm volatile(
                "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(sa)),
                "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(bar), "r"(kb * BK),
                "r"(mb * 256 + (int)rank * 128)
                , "l"(pol_a)
                : "memory");
          } else {  // A = Q1 MN-major: two 64 (M) x 64 (K) boxes of this CTA's 128 rows
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              asm volatile(
                  "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                  " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(sa + hh * 8192)),
                  "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(bar),
                  "r"(mb * 256 + (int)rank * 128 + hh * 64), "r"(kb * BK)
                  , "l"(pol_a)
                : "memory");
          }
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
              " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(sb)),
              "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(bar), "r"(kb * BK),
              "r"(nb * 256 + (int)rank * 128)
              , "l"(pol_b)
              : "memory");
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only) ----------------
      constexpr uint32_t idesc = make_idesc_f16(256, 256, MODE == kModeNN ? 1 : 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int w = pair; w < total; w += npairs, ++it) {
        const int s = w / (tiles_m * tiles_n);
        const int kb0 = (int)((long long)s * nkb / splits), kb1 = (int)((long long)(s + 1) * nkb / splits);
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * Cfg::BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t base_a = smem_u32(smem + stage * STAGE);
          const uint32_t base_b = base_a + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = (MODE == kModeTN) ? make_sw128_desc(base_a + kk * 32, 16, 1024)
                                                  : make_sw128_desc(base_a + kk * 2048, 8192, 1024);
            const uint64_t db = make_sw128_desc(base_b + kk * 32, 16, 1024);
            const uint32_t accum = (kb > kb0 || kk > 0) ? 1u : 0u;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "setp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
                "}\n" ::"r"(tacc),
                "l"(da), "l"(db), "r"(idesc), "r"(accum)
                : "memory");
          }
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
              " [%0], %1;" ::"r"(smem_u32(&empty[stage])),
              "h"((unsigned short)3)
              : "memory");
          if (++stage == ST) {
            stage = 0;
            phase ^= 1;
          }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(smem_u32(&tfull[acc])),
            "h"((unsigned short)3)
            : "memory");
      }
    }
  } else {  // ---------------- epilogue warps 2..5 (both CTAs): own 128 rows ----------------
    const int q = warp & 3;
    int it = 0;
    for (int w = pair; w < total; w += npairs, ++it) {
      int mb, nb, s;
      tile_of(w, tiles_m, tiles_n, mb, nb, s);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row = mb * 256 + (int)rank * 128 + q * 32 + lane;
      const bool rok = row < M;
      // NN: the first FP32 C chunk is loaded before waiting for the accumulator, later chunks
      // one ahead (as the 1-CTA kernel)
      float cv[32];
      if (MODE == kModeNN) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = nb * Cfg::BN + j;
          cv[j] = (rok && col < N) ? c_load(ef, C + row + (long long)col * ldc) : 0.f;
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * Cfg::BN;
#pragma unroll 1
      for (int c = 0; c < Cfg::BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c, r);
        const int col0 = nb * Cfg::BN + c;
        if (MODE == kModeTN) {
          tmem_ld_wait();
          if (rok) {
            float* out = C + (splits > 1 ? (long long)s * split_stride : 0LL) + row;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < N) {
                float v = __uint_as_float(r[j]);
                if (splits == 1 && col_mult) v *= __ldg(col_mult + col);
                out[(long long)col * ldc] = v;
              }
            }
          }
        } else {
          float cn[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int col = col0 + 32 + j;
            cn[j] = (rok && c + 32 < Cfg::BN && col < N) ? c_load(ef, C + row + (long long)col * ldc) : 0.f;
          }
          tmem_ld_wait();
          if (rok) {
            float* out = C + row;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < N) {
                const float mlt = col_mult ? __ldg(col_mult + col) : 1.f;
                c_store(out + (long long)col * ldc, cv[j] - __uint_as_float(r[j]) * mlt, col, ef);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) cv[j] = cn[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(&tempty[acc]))
                     : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(Cfg::TMEM_COLS)
                 : "memory");
  }
}

// Deterministic split-K reduction: C[i + j*ldc] = (sum_s P[s][i + j*ldp]) * col_mult[j].
// 8 threads per output element (each sums a contiguous range of splits with all loads in
// flight), combined in a fixed order through shared memory.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ P, int splits,
                                                            long long pstride, int ldp, int M,
                                                            int N, float* __restrict__ C,
                                                            long long ldc,
                                                            const float* __restrict__ col_mult) {
  __shared__ float part[8][33];
  const long long total = (long long)M * N;
  const int el = threadIdx.x & 31, sg = threadIdx.x >> 5;  // 32 elements x 8 split groups
  const int per = (splits + 7) / 8, s0 = sg * per, s1 = min(splits, s0 + per);
  for (long long eb = (long long)blockIdx.x * 32; eb < total; eb += (long long)gridDim.x * 32) {
    const long long e = eb + el;
    float acc = 0.f;
    if (e < total) {
      const int i = (int)(e % M), j = (int)(e / M);
      const float* p = P + i + (long long)j * ldp;
      int s = s0;
      for (; s + 8 <= s1; s += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (long long)(s + u) * pstride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
      }
      for (; s < s1; ++s) acc += __ldcg(p + (long long)s * pstride);
    }
    __syncthreads();
    part[sg][el] = acc;
    __syncthreads();
    if (sg == 0 && e < total) {
      float t = 0.f;
#pragma unroll
      for (int g = 0; g < 8; ++g) t += part[g][el];
      const int i = (int)(e % M), j = (int)(e / M);
      if (col_mult) t *= col_mult[j];
      C[i + (long long)j * ldc] = t;
    }
  }
}

// ------------------------------------------------------------------------------------------
// Host side
// ------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// 2-D FP16 map: inner (contiguous) extent, outer extent, leading dimension (elements).
static bool make_map_f16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D FP32 map (no swizzle) for the NN epilogue's C chunks: 128 rows x 32 columns.
static bool make_map_f32(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                         uint64_t ld, uint32_t box_inner, uint32_t box_outer) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int l2_ef_mask() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TCQR_L2_EF");
    v = e ? atoi(e) : kL2EfDefault;
  }
  return v;
}
// per-launch ef bits: an operand is read once when the output's other dimension is one tile
static int launch_ef(int mode, int M, int N, int tile_m, int tile_n) {
  const int g = l2_ef_mask();
  int ef = (g & 2) ? kEfC : 0;
  const bool all = (g & 8) != 0, once = (g & 4) != 0;
  if (all || (once && N <= tile_n)) ef |= kEfA;
  if (mode == kModeTN && (all || (once && M <= tile_m))) ef |= kEfB;
  return ef;
}

template <int BN, int MODE, int NBUF = 0>
static cudaError_t launch_tc(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& cm,
                             int M, int N, int K, int splits, float* C, long long ldc,
                             long long sstride, const float* mult, int num_sms, cudaStream_t st) {
  using Cfg = TcCfg<BN, MODE, NBUF>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm_kernel<BN, MODE, NBUF>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = ((M + 127) / 128) * ((N + BN - 1) / BN) * splits;
  const int slots = Cfg::OCC * num_sms;
  const int grid = tiles < slots ? tiles : slots;
  tc_gemm_kernel<BN, MODE, NBUF><<<grid, 192, Cfg::SMEM, st>>>(a, b, cm, M, N, K, splits, C, ldc,
                                                               sstride, mult,
                                                               launch_ef(MODE, M, N, 128, BN));
  return cudaGetLastError();
}

// CTA-pair launches: one cluster pair per 256 x 256 tile (and split for TN).
template <int MODE>
static cudaError_t launch_tc2(const CUtensorMap& ma, const CUtensorMap& mb, int M, int N, int K,
                              int splits, float* C, long long ldc, long long sstride,
                              const float* mult, int num_sms, cudaStream_t st) {
  using Cfg = Tc2Cfg;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_gemm2_kernel<MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int units = ((M + 255) / 256) * ((N + 255) / 256) * splits;
  const int npairs = std::min(units, num_sms / 2);
  tc_gemm2_kernel<MODE><<<2 * npairs, 192, Cfg::SMEM, st>>>(ma, mb, M, N, K, splits, C, ldc,
                                                             sstride, mult,
                                                             launch_ef(MODE, M, N, 256, 256));
  return cudaGetLastError();
}

static cudaError_t launch_tc2_tn(const __half* A1h, long long lda1, const __half* A2h,
                                 long long lda2, int m, int h, int w2, int splits, float* C,
                                 long long ldc, long long sstride, const float* mult, int num_sms,
                                 cudaStream_t st) {
  CUtensorMap ma, mb;
  if (!make_map_f16(&ma, A1h, m, h, lda1, 64, 128)) return cudaErrorInvalidValue;
  if (!make_map_f16(&mb, A2h, m, w2, lda2, 64, 128)) return cudaErrorInvalidValue;
  return launch_tc2<kModeTN>(ma, mb, h, w2, m, splits, C, ldc, sstride, mult, num_sms, st);
}

static int kTc2NnMinK = 2049;  // NN on CTA pairs from this K = h on (env TCQR_TC2_NN_MINK)

static bool use_tc2() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("TCQR_TC2");
    on = (e && e[0] == '0') ? 0 : 1;
    const char* k = getenv("TCQR_TC2_NN_MINK");
    if (k) kTc2NnMinK = atoi(k);
  }
  return on == 1;
}

// fewest K-blocks (of 64 rows) per split-K slice of the TN product (env TCQR_TN_MINKB)
static int tn_min_kb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TCQR_TN_MINKB");
    v = e ? atoi(e) : 8;
    if (v < 1) v = 1;
  }
  return v;
}

// D (h x w2) = A1h' A2h ; writes C (ldc) directly (splits == 1, scaled by col_mult) or the
// partials P (splits > 1; P has room for splits * ldp * w2 floats) followed by the reduction.
cudaError_t tc_gemm_tn(int m, int h, int w2, const __half* A1h, long long lda1, const __half* A2h,
                       long long lda2, float* C, long long ldc, const float* col_mult, float* P,
                       long long p_cap, int num_sms, cudaStream_t st, const R12Finalize* fin) {
  if (m <= 0 || h <= 0 || w2 <= 0) return cudaSuccess;
  const int nkb = (m + 63) / 64;
  if (use_tc2() && h >= 256 && w2 >= 256) {
    // CTA pairs: 256 x 256 tiles, split-K over the pairs
    const int tiles2 = ((h + 255) / 256) * ((w2 + 255) / 256);
    int splits = 1;
    const int np = num_sms / 2;
    if (tiles2 < np) {
      splits = np / tiles2;
      if (splits > nkb / tn_min_kb()) splits = nkb / tn_min_kb();
      if (splits < 1) splits = 1;
      const long long per = (long long)h * w2;
      if (P == nullptr || per * splits > p_cap) splits = P ? (int)(p_cap / per) : 1;
      if (splits < 1) splits = 1;
    }
    cudaError_t e;
    if (splits == 1) {
      e = launch_tc2_tn(A1h, lda1, A2h, lda2, m, h, w2, 1, C, ldc, 0, col_mult, num_sms, st);
      if (e != cudaSuccess || !fin) return e;
      return r12_finalize(h, w2, C, ldc, fin->Rblk, fin->ldr, fin->R12h, fin->ldh2, fin->inv_s2,
                          fin->scaling, st);
    }
    const long long sstride = (long long)h * w2;
    e = launch_tc2_tn(A1h, lda1, A2h, lda2, m, h, w2, splits, P, h, sstride, nullptr, num_sms, st);
    if (e != cudaSuccess) return e;
    if (fin)
      return r12_splitk_finalize(h, w2, P, splits, sstride, h, col_mult, fin->Rblk, fin->ldr,
                                 fin->R12h, fin->ldh2, fin->inv_s2, fin->scaling, st);
    const long long total = (long long)h * w2;
    int grid = (int)((total + 31) / 32);
    if (grid > 8 * num_sms) grid = 8 * num_sms;
    splitk_reduce_kernel<<<grid, 256, 0, st>>>(P, splits, sstride, h, h, w2, C, ldc, col_mult);
    return cudaGetLastError();
  }
  CUtensorMap ma, mb;
  const int BN = (w2 > 128) ? 256 : 128;
  if (!make_map_f16(&ma, A1h, m, h, lda1, 64, 128)) return cudaErrorInvalidValue;
  if (!make_map_f16(&mb, A2h, m, w2, lda2, 64, BN)) return cudaErrorInvalidValue;
  const int tiles = ((h + 127) / 128) * ((w2 + BN - 1) / BN);
  int splits = 1;
  if (tiles < num_sms) {
    splits = num_sms / tiles;
    // keep >= 8 K-blocks per split: the partials (and their reduction) cost HBM traffic and a
    // split that only fills the pipeline is latency, not throughput
    if (splits > nkb / tn_min_kb()) splits = nkb / tn_min_kb();
    if (splits < 1) splits = 1;
    const long long per = (long long)h * w2;
    if (P == nullptr || per * splits > p_cap) splits = P ? (int)(p_cap / per) : 1;
    if (splits < 1) splits = 1;
  }
  cudaError_t e;
  if (splits == 1) {
    e = (BN == 256)
            ? launch_tc<256, kModeTN>(ma, mb, ma, h, w2, m, 1, C, ldc, 0, col_mult, num_sms, st)
            : launch_tc<128, kModeTN>(ma, mb, ma, h, w2, m, 1, C, ldc, 0, col_mult, num_sms, st);
    if (e != cudaSuccess || !fin) return e;
    return r12_finalize(h, w2, C, ldc, fin->Rblk, fin->ldr, fin->R12h, fin->ldh2, fin->inv_s2,
                        fin->scaling, st);
  }
  const long long sstride = (long long)h * w2;
  e = (BN == 256) ? launch_tc<256, kModeTN>(ma, mb, ma, h, w2, m, splits, P, h, sstride,
                                            nullptr, num_sms, st)
                  : launch_tc<128, kModeTN>(ma, mb, ma, h, w2, m, splits, P, h, sstride,
                                            nullptr, num_sms, st);
  if (e != cudaSuccess) return e;
  if (fin)
    return r12_splitk_finalize(h, w2, P, splits, sstride, h, col_mult, fin->Rblk, fin->ldr,
                               fin->R12h, fin->ldh2, fin->inv_s2, fin->scaling, st);
  const long long total = (long long)h * w2;
  int grid = (int)((total + 31) / 32);
  if (grid > 8 * num_sms) grid = 8 * num_sms;
  splitk_reduce_kernel<<<grid, 256, 0, st>>>(P, splits, sstride, h, h, w2, C, ldc, col_mult);
  return cudaGetLastError();
}

// K = h up to which the update runs as the two-CTAs-per-SM short-K variant (env TCQR_NN_SHORTK)
static int nn_short_k() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TCQR_NN_SHORTK");
    v = e ? atoi(e) : 1024;  // config 3: 1024 -> w = 2048 gaps 221 -> 204 us (2048: w = 4096 worse)
  }
  return v;
}

// C (m x w2) -= (Qh Bh) diag(col_mult);  Qh m x h (ldq), Bh h x w2 (ldb).
cudaError_t tc_gemm_nn_update(int m, int h, int w2, const __half* Qh, long long ldq,
                              const __half* Bh, long long ldb, float* C, long long ldc,
                              const float* col_mult, int num_sms, cudaStream_t st) {
  if (m <= 0 || h <= 0 || w2 <= 0) return cudaSuccess;
  static int pre_all = -1;
  if (pre_all < 0) {
    const char* e = getenv("TCQR_NN_PRE_ALL");
    pre_all = e ? atoi(e) : 1;
    if (pre_all != 1) cudaMemcpyToSymbol(nn_pre_all, &pre_all, sizeof(int));
  }
  CUtensorMap ma, mb;
  if (!make_map_f16(&ma, Qh, m, h, ldq, 64, 64)) return cudaErrorInvalidValue;
  if (use_tc2() && h >= kTc2NnMinK && w2 >= 256) {
    // long K: CTA pairs with 256 x 256 tiles (each CTA stages 128 columns of B)
    if (!make_map_f16(&mb, Bh, h, w2, ldb, 64, 128)) return cudaErrorInvalidValue;
    return launch_tc2<kModeNN>(ma, mb, m, w2, h, 1, C, ldc, 0, col_mult, num_sms, st);
  }
  const int BN = (w2 > 128) ? 256 : 128;
  if (!make_map_f16(&mb, Bh, h, w2, ldb, 64, BN)) return cudaErrorInvalidValue;
  // TMA epilogue (C chunks through shared memory, four buffers) for short K = h, where the
  // update is epilogue-bound, when C's columns are 16-byte aligned; the direct-load epilogue with
  // the deeper mainloop for long K (measured: the 2-buffer TMA variant is 6% slower at h = 8192)
  CUtensorMap mc;
  const bool tmac = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0) &&
                    make_map_f32(&mc, C, m, w2, ldc, 128, 32);
  if (tmac && h <= nn_short_k()) {
    CUtensorMap mb1;
    if (!make_map_f16(&mb1, Bh, h, w2, ldb, 64, 128)) return cudaErrorInvalidValue;
    return launch_tc<128, kModeNN, 2>(ma, mb1, mc, m, w2, h, 1, C, ldc, 0, col_mult, num_sms, st);
  }
  if (tmac && h <= 2048)
    return (BN == 256) ? launch_tc<256, kModeNN, 4>(ma, mb, mc, m, w2, h, 1, C, ldc, 0, col_mult,
                                                    num_sms, st)
                       : launch_tc<128, kModeNN, 4>(ma, mb, mc, m, w2, h, 1, C, ldc, 0, col_mult,
                                                    num_sms, st);
  return (BN == 256) ? launch_tc<256, kModeNN>(ma, mb, ma, m, w2, h, 1, C, ldc, 0, col_mult, num_sms,
                                               st)
                     : launch_tc<128, kModeNN>(ma, mb, ma, m, w2, h, 1, C, ldc, 0, col_mult, num_sms,
                                               st);
}

}  // namespace tcqr

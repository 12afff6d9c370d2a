// k_panel.cu -- K2: the communication-avoiding MGS panel (Eq. (6), Alg. 4).
//
// One CAQR level = one launch of panel_mgs_kernel: CTA b owns row block b (br rows; the last
// block absorbs a remainder shorter than w rows, reading R-A6), keeps it in registers (one or two
// rows per thread, as the paper's "256 threads ... a single row" design) and
// runs Alg. 4 on it:
//     for k: R(k,k) = ||q_k||; q_k /= R(k,k); R(k,k+1:) = q_k' Q(:,k+1:); Q(:,k+1:) -= q_k R(k,k+1:)
// The norm and the w-k dot products of step k are ONE block reduction: each thread forms its
// partial products, a 31-shuffle transpose-reduce leaves lane j with the warp sum of product j,
// and a double-buffered shared array combines the warps in a fixed order (deterministic).
// R(k,j) = (a_k' a_j) / R(k,k) equals q_k' a_j up to rounding order.
// The stacked R's are factored by the same kernel (step 3); panel_apply_kernel is step 4
// ("batched SGEMM" in the paper).
#include "common.cuh"
#include "kernels.h"

namespace tcqr {

constexpr int kPanelThreads = 256;
constexpr int kPanelWarps = kPanelThreads / 32;
constexpr int kPanelRPT = 2;  // rows per thread -> up to 512 rows per block (br <= 480 + w)

int panel_num_blocks(int rows, int br, int w) {
  int nb = (rows + br - 1) / br;
  if (nb < 1) nb = 1;
  const int last = rows - (nb - 1) * br;
  if (nb > 1 && last < w) --nb;
  return nb;
}

// Transpose-reduce: on exit v[0] in lane l holds sum over the warp of the input v[l].
__device__ __forceinline__ float transpose_reduce32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const float send = upper ? v[i] : v[i + s];
      const float keep = upper ? v[i + s] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

__global__ void __launch_bounds__(kPanelThreads) panel_mgs_kernel(
    int rows, int w, float* __restrict__ X, long long ldx, int br, int nb, float* __restrict__ S,
    long long lds, float* __restrict__ Rout, long long ldr, int top, int* status, int col0) {
  __shared__ float red[2][kPanelWarps][32];
  const int b = blockIdx.x;
  const int row0 = b * br;
  const int nrows = (b == nb - 1) ? rows - row0 : br;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  float x[kPanelRPT][32];
#pragma unroll
  for (int r = 0; r < kPanelRPT; ++r) {
    const int i = tid + r * kPanelThreads;
    const bool ok = i < nrows;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      x[r][j] = (ok && j < w) ? X[(long long)(row0 + i) + (long long)j * ldx] : 0.f;
  }
  float* Rdst = (nb == 1) ? Rout : S + (long long)b * w;
  const long long ldR = (nb == 1) ? ldr : lds;

  int buf = 0;
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    if (k < w) {
      float p[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float acc = 0.f;
        if (j >= k) {
#pragma unroll
          for (int r = 0; r < kPanelRPT; ++r) acc = fmaf(x[r][k], x[r][j], acc);
        }
        p[j] = acc;
      }
      const float part = transpose_reduce32(p);  // lane j: warp sum of a_k' a_j
      red[buf][warp][lane] = part;
      __syncthreads();
      float tot = 0.f;
#pragma unroll
      for (int v = 0; v < kPanelWarps; ++v) tot += red[buf][v][lane];
      buf ^= 1;
      const float nrm2 = __shfl_sync(0xffffffffu, tot, k);
      const float rkk = sqrtf(nrm2);
      const bool zero = !(rkk > 0.f) || !isfinite(rkk);
      if (top && zero && tid == 0 && status) atomicMin(status, col0 + k + 1);
      float rkj = zero ? 0.f : tot / rkk;  // lane j > k: R(k, j)
      if (lane == k) rkj = zero ? 0.f : rkk;
      if (lane < k) rkj = 0.f;
      if (warp == 0 && lane < w) Rdst[k + (long long)lane * ldR] = rkj;
      float qk[kPanelRPT];
#pragma unroll
      for (int r = 0; r < kPanelRPT; ++r) {
        qk[r] = zero ? 0.f : x[r][k] / rkk;
        x[r][k] = qk[r];
      }
#pragma unroll
      for (int j = k + 1; j < 32; ++j) {
        const float rj = __shfl_sync(0xffffffffu, rkj, j);
#pragma unroll
        for (int r = 0; r < kPanelRPT; ++r) x[r][j] = fmaf(-qk[r], rj, x[r][j]);
      }
    } else if (warp == 0 && k < 32 && lane < w) {
      // unreachable rows of R beyond w are not stored
    }
  }
  // Zero the strictly-lower part of this R block (rows k > j) so the stack is a proper R.
  if (warp == 0) {
    for (int k = 1; k < w; ++k)
      if (lane < k) Rdst[k + (long long)lane * ldR] = 0.f;
  }
#pragma unroll
  for (int r = 0; r < kPanelRPT; ++r) {
    const int i = tid + r * kPanelThreads;
    if (i < nrows) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < w) X[(long long)(row0 + i) + (long long)j * ldx] = x[r][j];
    }
  }
}

cudaError_t panel_mgs_level(int rows, int w, float* X, long long ldx, int br, int nb, float* S,
                            long long lds, float* Rout, long long ldr, int top, int* status,
                            int col0, cudaStream_t st) {
  panel_mgs_kernel<<<nb, kPanelThreads, 0, st>>>(rows, w, X, ldx, br, nb, S, lds, Rout, ldr, top,
                                                 status, col0);
  return cudaGetLastError();
}

// X_b <- X_b * T_b with T_b = S[b*w:(b+1)*w, 0:w] (lds).  grid.x = row chunks of 256 rows.
__global__ void __launch_bounds__(256) panel_apply_kernel(int rows, int w, float* __restrict__ X,
                                                          long long ldx, int br, int nb,
                                                          const float* __restrict__ S,
                                                          long long lds) {
  __shared__ float T[32][33];
  const int i = blockIdx.x * 256 + threadIdx.x;
  // block index of the first row of this CTA (CTAs never straddle: chunks are 256 rows and br is
  // a multiple of 32 but not necessarily of 256 -> compute per row below, T loaded per block).
  const int row_first = blockIdx.x * 256;
  int b_first = row_first / br;
  if (b_first > nb - 1) b_first = nb - 1;
  int row_last = row_first + 255;
  if (row_last > rows - 1) row_last = rows - 1;
  int b_last = row_last / br;
  if (b_last > nb - 1) b_last = nb - 1;
  float x[32];
  const bool ok = i < rows;
  int bi = ok ? i / br : 0;
  if (bi > nb - 1) bi = nb - 1;
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (ok && j < w) ? X[(long long)i + (long long)j * ldx] : 0.f;
  float y[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) y[j] = 0.f;
  for (int b = b_first; b <= b_last; ++b) {
    __syncthreads();
    for (int e = threadIdx.x; e < w * w; e += 256) {
      const int l = e % w, j = e / w;
      T[l][j] = S[(long long)(b * w + l) + (long long)j * lds];
    }
    __syncthreads();
    if (ok && bi == b) {
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        if (l < w) {
          const float xl = x[l];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < w) y[j] = fmaf(xl, T[l][j], y[j]);
        }
      }
    }
  }
  if (ok) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < w) X[(long long)i + (long long)j * ldx] = y[j];
  }
}

cudaError_t panel_apply(int rows, int w, float* X, long long ldx, int br, int nb, const float* S,
                        long long lds, cudaStream_t st) {
  const int grid = (rows + 255) / 256;
  panel_apply_kernel<<<grid, 256, 0, st>>>(rows, w, X, ldx, br, nb, S, lds);
  return cudaGetLastError();
}

}  // namespace tcqr

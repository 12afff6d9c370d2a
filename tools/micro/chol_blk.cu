// Blocked (8 x 8) right-looking form of the leaf's 32 x 32 FP64 Cholesky + S_b = R_b R^-1 on one
// warp (lane j = column j of the trailing Gram / row j of S_b), against the current rolled fused
// chain (chol2.cu B): within a block of 8 steps only the block's own rows are updated per step;
// the rank-8 update of the rows below (and of S_b's later columns) runs once per block as a burst
// of independent DFMAs.  Registers are shifted down by 8 after every block (loop-invariant code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 chol_blk.cu -o bin/chol_blk
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y * y, 1.0);
  return fma(fma(e, 0.375, 0.5), e * y, y);
}

// reference: the current fused rolled chain (chol2.cu B), all 32 steps, T = 31
__device__ void chain_ref(int lane, double (&c)[32], double (&r)[32], double* rowbuf, double* Rd,
                          float* Sf) {
  double d = __shfl_sync(0xffffffffu, c[0], 0);
  bool ok = d > 0.0;
  double ri = rsqrt_nr(ok ? d : 1.0);
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    ri = ok ? ri : 0.0;
    const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
    const double dn = fma(-rkj, rkj, c[1]);
    d = __shfl_sync(0xffffffffu, dn, (k + 1) & 31);
    double* rowk = rowbuf + (k & 1) * 64;
    rowk[lane] = rkj;
    rowk[lane + 32] = rkj;
    Rd[k * 34 + lane] = rkj;
    const double sk = r[0] * ri;
    Sf[lane * 34 + k] = (float)sk;
    ok = d > 0.0;
    ri = rsqrt_nr(ok ? d : 1.0);
    __syncwarp();
    const double* rk = rowk + k + 1;
#pragma unroll
    for (int i = 0; i < 31; ++i) {
      const double v = rk[i];
      c[i] = fma(-v, rkj, c[i + 1]);
      r[i] = fma(-sk, v, r[i + 1]);
    }
  }
}

// blocked: c[i] = W(8K + i, j) (block-relative), r[i] = running S_b(lane, 8K + i)
template <int TB>  // live rows below the block (24, 16, 8, 0)
__device__ __forceinline__ void blk(int K, int lane, double (&c)[32], double (&r)[32], double* Rd,
                                    float* Sf) {
  double rk8[8];  // this lane's R(8K + s, j) for the block's steps s (j = lane)
  double sk8[8];  // this lane's S_b(lane, 8K + s)
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int k = 8 * K + s;
    const double d = __shfl_sync(0xffffffffu, c[s], k & 31);  // W(k, k), up to date
    const bool ok = d > 0.0;
    const double ri = ok ? rsqrt_nr(d) : 0.0;
    const double rkj = lane == k ? d * ri : (lane > k ? c[s] * ri : 0.0);
    rk8[s] = rkj;
    Rd[k * 34 + lane] = rkj;
    const double sk = r[s] * ri;
    sk8[s] = sk;
    Sf[lane * 34 + k] = (float)sk;
    __syncwarp();
    // the block's own later rows (and S_b's later columns of the block)
#pragma unroll
    for (int t = s + 1; t < 8; ++t) {
      const double v = Rd[k * 34 + 8 * K + t];  // R(k, 8K + t)
      c[t] = fma(-v, rkj, c[t]);
      r[t] = fma(-sk, v, r[t]);
    }
  }
  // rank-8 burst: rows (columns of S_b) below the block
#pragma unroll
  for (int i = 0; i < TB; ++i) {
    double cv = c[8 + i], rv = r[8 + i];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const double v = Rd[(8 * K + s) * 34 + 8 * K + 8 + i];
      cv = fma(-v, rk8[s], cv);
      rv = fma(-sk8[s], v, rv);
    }
    c[i] = cv;  // shifted down by 8
    r[i] = rv;
  }
}

template <int V>
__global__ void chol(const double* G, const double* Rb, double* outR, float* outS, long long* clk) {
  __shared__ double Rd[32 * 34 + 34];
  __shared__ double rowbuf[128];
  __shared__ float Sf[32 * 34];
  const int lane = threadIdx.x & 31;
  double c[32], r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = (i <= lane) ? G[i * 32 + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = Rb[lane * 32 + j];
  for (int e = lane; e < 32 * 34 + 34; e += 32) Rd[e] = 0.0;
  __syncwarp();
  long long t0 = clock64();
  if (V == 0) {
    chain_ref(lane, c, r, rowbuf, Rd, Sf);
  } else {
    blk<24>(0, lane, c, r, Rd, Sf);
    blk<16>(1, lane, c, r, Rd, Sf);
    blk<8>(2, lane, c, r, Rd, Sf);
    blk<0>(3, lane, c, r, Rd, Sf);
  }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) clk[V] = t1 - t0;
  for (int i = 0; i < 32; ++i) {
    outR[i * 32 + lane] = Rd[i * 34 + lane];
    outS[i * 32 + lane] = Sf[lane * 34 + i];
  }
}

int main() {
  double hG[1024], hRb[1024];
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) hRb[i * 32 + j] = j >= i ? ((i * 7 + j * 13) % 17 - 8) / 8.0 + (i == j ? 3.0 : 0.0) : 0.0;
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) {
      double s = 0;
      for (int l = 0; l < 32; ++l) s += hRb[l * 32 + i] * hRb[l * 32 + j];
      hG[i * 32 + j] = s + (i == j ? 1.0 : 0.0);
    }
  double *G, *Rb, *oR;
  float* oS;
  long long* c;
  cudaMalloc(&G, 8192); cudaMalloc(&Rb, 8192); cudaMalloc(&oR, 8192); cudaMalloc(&oS, 4096); cudaMalloc(&c, 64);
  cudaMemcpy(G, hG, 8192, cudaMemcpyHostToDevice);
  cudaMemcpy(Rb, hRb, 8192, cudaMemcpyHostToDevice);
  double refR[1024], R[1024];
  float refS[1024], S[1024];
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      if (v == 0) chol<0><<<1, 32>>>(G, Rb, oR, oS, c);
      else chol<1><<<1, 32>>>(G, Rb, oR, oS, c);
    }
    cudaDeviceSynchronize();
    long long hc[2];
    cudaMemcpy(hc, c, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(R, oR, 8192, cudaMemcpyDeviceToHost);
    cudaMemcpy(S, oS, 4096, cudaMemcpyDeviceToHost);
    if (v == 0) memcpy(refR, R, 8192), memcpy(refS, S, 4096);
    int dr = 0, ds = 0;
    double mr = 0;
    for (int i = 0; i < 1024; ++i) {
      dr += R[i] != refR[i], ds += S[i] != refS[i];
      const double e = R[i] - refR[i];
      if ((e < 0 ? -e : e) > mr) mr = e < 0 ? -e : e;
    }
    printf("%s: %lld cycles (%.0f per step); R diffs %d (max %.2e), S diffs %d  %s\n",
           v == 0 ? "fused rolled (current)" : "blocked 8x8", hc[v], hc[v] / 32.0, dr, mr, ds,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

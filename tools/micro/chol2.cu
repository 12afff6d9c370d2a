// Cycles of the leaf's 32 x 32 FP64 Cholesky (k_leaf.cu (3)) on one warp:
//   A  the current rolled, shifted chain with the block's S_b substitution fused in (31 + 31 DFMA
//      per step);
//   B  A with triangular trip counts (four phases of eight steps: 31, 23, 15, 7 terms);
//   C  the Cholesky alone with triangular trip counts;
//   D  the S_b = R_b R^-1 substitution alone as a post-pass (R rows and 1/R(k,k) in shared memory,
//      lane = row of S_b, fully unrolled) -- run by four warps at once in the leaf.
// Checks B..D reproduce A's R and S bits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 chol2.cu -o chol2
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_nr(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double e = fma(-d, y * y, 1.0);
  return fma(fma(e, 0.375, 0.5), e * y, y);
}

template <int T>
__device__ __forceinline__ void chol_steps(int k0, int k1, int lane, double (&c)[32], double (&r)[32],
                                           double& d, bool& ok, double& ri, double* Rd, double* rowbuf,
                                           float* Sf, double* ris, bool withS) {
#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    ri = ok ? ri : 0.0;
    const double rkj = lane == k ? d * ri : (lane > k ? c[0] * ri : 0.0);
    const double dn = fma(-rkj, rkj, c[1]);
    d = __shfl_sync(0xffffffffu, dn, (k + 1) & 31);
    double* rowk = rowbuf + (k & 1) * 64;
    rowk[lane] = rkj;
    rowk[lane + 32] = rkj;
    Rd[k * 34 + lane] = rkj;
    if (lane == 0) ris[k] = ri;
    double sk = 0.0;
    if (withS) {
      sk = r[0] * ri;
      Sf[lane * 34 + k] = (float)sk;
    }
    ok = d > 0.0 && d <= 1.7976931348623157e308;
    ri = rsqrt_nr(ok ? d : 1.0);
    __syncwarp();
    const double* rk = rowk + k + 1;
#pragma unroll
    for (int i = 0; i < T; ++i) {
      const double v = rk[i];
      c[i] = fma(-v, rkj, c[i + 1]);
      if (withS) r[i] = fma(-sk, v, r[i + 1]);
    }

  }
}

template <int V>
__global__ void chol(const double* G, const double* Rb, double* outR, float* outS, long long* clk) {
  __shared__ double Rd[32 * 34 + 34];
  __shared__ double rowbuf[128];
  __shared__ double ris[32];
  __shared__ float Sf[4][32 * 34];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double c[32], r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) c[i] = (i <= lane) ? G[i * 32 + lane] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = Rb[lane * 32 + j];
  __syncthreads();
  long long t0 = clock64();
  if (V <= 2) {
    if (warp == 0) {
      double d = __shfl_sync(0xffffffffu, c[0], 0);
      bool ok = d > 0.0;
      double ri = rsqrt_nr(ok ? d : 1.0);
      if (V == 0) {
        chol_steps<31>(0, 32, lane, c, r, d, ok, ri, Rd, rowbuf, Sf[0], ris, true);
      } else {
        const bool ws = V == 1;
        chol_steps<31>(0, 8, lane, c, r, d, ok, ri, Rd, rowbuf, Sf[0], ris, ws);
        chol_steps<23>(8, 16, lane, c, r, d, ok, ri, Rd, rowbuf, Sf[0], ris, ws);
        chol_steps<15>(16, 24, lane, c, r, d, ok, ri, Rd, rowbuf, Sf[0], ris, ws);
        chol_steps<7>(24, 32, lane, c, r, d, ok, ri, Rd, rowbuf, Sf[0], ris, ws);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (V == 2 || V == 3) {
    // D: S(lane, k) = (R_b(lane, k) - sum_{l<k} S(lane, l) R(l, k)) / R(k, k), right-looking in l
    if (warp < 4) {
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double sk = r[k] * ris[k];
        Sf[warp][lane * 34 + k] = (float)sk;
#pragma unroll
        for (int j = k + 1; j < 32; ++j) r[j] = fma(-sk, Rd[k * 34 + j], r[j]);
      }
    }
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    clk[2 * V] = t1 - t0;
    clk[2 * V + 1] = t2 - t1;
  }
  if (warp == 0)
    for (int i = 0; i < 32; ++i) {
      outR[i * 32 + lane] = Rd[i * 34 + lane];
      outS[i * 32 + lane] = Sf[0][lane * 34 + i];
    }
}

// E: the Cholesky split over four warps (warp w owns trailing rows [8w, 8w + 8), lane j = column
// j, absolute row indices: no register shifting), one named barrier per step; the owner warp of
// row k publishes R(k, :) (double-buffered) and 1/R(k,k); then the S_b substitution post-pass.
__global__ void chol_coop(const double* G, const double* Rb, double* outR, float* outS, long long* clk) {
  __shared__ double Rd[32 * 34 + 34];
  __shared__ double rowbuf[2][32];
  __shared__ double ris[32];
  __shared__ float Sf[4][32 * 34];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double cw[8];
#pragma unroll
  for (int ii = 0; ii < 8; ++ii) {
    const int r = 8 * warp + ii;
    cw[ii] = (r <= lane) ? G[r * 32 + lane] : 0.0;
  }
  double r[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = Rb[lane * 32 + j];
  __syncthreads();
  long long t0 = clock64();
  bool okall = true;
#pragma unroll 1
  for (int k = 0; k < 32; ++k) {
    const int o = k >> 3;
    if (warp == o) {
      double dv = 0.0;
#pragma unroll
      for (int ii = 0; ii < 8; ++ii) if (ii == (k & 7)) dv = cw[ii];
      const double d = __shfl_sync(0xffffffffu, dv, k);
      const bool ok = d > 0.0 && d <= 1.7976931348623157e308;
      okall &= ok;
      const double ri = ok ? rsqrt_nr(d) : 0.0;
      const double rkj = lane == k ? d * ri : (lane > k ? dv * ri : 0.0);
      rowbuf[k & 1][lane] = rkj;
      Rd[k * 34 + lane] = rkj;
      if (lane == 0) ris[k] = ri;
    }
    asm volatile("bar.sync 2, 128;" ::: "memory");
    const double rk = rowbuf[k & 1][lane];
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) {
      const int rr = 8 * warp + ii;
      if (rr > k) cw[ii] = fma(-rowbuf[k & 1][rr], rk, cw[ii]);
    }
  }
  asm volatile("bar.sync 2, 128;" ::: "memory");
  long long t1 = clock64();
  // S_b post-pass (as D): S(lane, k) = (R_b(lane, k) - sum_{l<k} S(lane, l) R(l, k)) / R(k, k)
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const double sk = r[k] * ris[k];
    Sf[warp][lane * 34 + k] = (float)sk;
#pragma unroll
    for (int j = k + 1; j < 32; ++j) r[j] = fma(-sk, Rd[k * 34 + j], r[j]);
  }
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    clk[6] = t1 - t0;
    clk[7] = t2 - t1;
  }
  if (warp == 0)
    for (int i = 0; i < 32; ++i) {
      outR[i * 32 + lane] = Rd[i * 34 + lane];
      outS[i * 32 + lane] = Sf[0][lane * 34 + i];
    }
  (void)okall;
}

int main() {
  double hG[1024], hRb[1024];
  // G = R_b' R_b + diag for a random upper-triangular R_b
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
  cudaMalloc(&G, 8192); cudaMalloc(&Rb, 8192); cudaMalloc(&oR, 8192); cudaMalloc(&oS, 4096); cudaMalloc(&c, 128);
  cudaMemcpy(G, hG, 8192, cudaMemcpyHostToDevice);
  cudaMemcpy(Rb, hRb, 8192, cudaMemcpyHostToDevice);
  double refR[1024], R[1024];
  float refS[1024], S[1024];
  const char* names[4] = {"A rolled fused (current)", "B rolled fused, triangular trips",
                          "C Cholesky only, triangular trips + D post-pass S", "E four-warp Cholesky + D post-pass S"};
  for (int v = 0; v < 4; ++v) {
    for (int rep = 0; rep < 3; ++rep) {
      if (v == 0) chol<0><<<1, 128>>>(G, Rb, oR, oS, c);
      if (v == 1) chol<1><<<1, 128>>>(G, Rb, oR, oS, c);
      if (v == 2) chol<2><<<1, 128>>>(G, Rb, oR, oS, c);
      if (v == 3) chol_coop<<<1, 128>>>(G, Rb, oR, oS, c);
    }
    cudaDeviceSynchronize();
    long long hc[8];
    cudaMemcpy(hc, c, 64, cudaMemcpyDeviceToHost);
    cudaMemcpy(R, oR, 8192, cudaMemcpyDeviceToHost);
    cudaMemcpy(S, oS, 4096, cudaMemcpyDeviceToHost);
    if (v == 0) memcpy(refR, R, 8192), memcpy(refS, S, 4096);
    int dr = 0, ds = 0;
    for (int i = 0; i < 1024; ++i) dr += R[i] != refR[i], ds += S[i] != refS[i];
    printf("%-52s chain %lld cycles (%.0f/step), post-pass %lld cycles; R diffs %d, S diffs %d  %s\n", names[v],
           hc[2 * v], hc[2 * v] / 32.0, hc[2 * v + 1], dr, ds, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

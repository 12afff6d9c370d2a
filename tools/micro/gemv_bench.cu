// GEMV variants of the CGLS iteration (K5) on the configs[3] shape, 32768 x 8192 FP32 column-major
// A, FP64 vectors and accumulation (CUDA events, 20 reps, warm):
//   N0  q = A t, thread per row, eight 4-byte column loads in flight (k_cgls.cu gemv_n_part)
//   N1  four consecutive rows per thread, 16-byte loads, eight columns in flight
//   T0  v = A' r, 64 columns per CTA, r staged in shared memory 1024 rows at a time (gemv_t_part)
//   T1  v = A' r, 64 columns per CTA (8 per warp), r read by each lane from L1/L2 (no staging, no
//       CTA barriers), two row groups of 128 in flight per lane
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 gemv_bench.cu -o gemv_bench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 32768, N = 8192;

__global__ void __launch_bounds__(256) n0(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, double* __restrict__ part) {
  __shared__ double vs[512];
  const int cb = blockIdx.y, j0 = cb * 512, nc = min(512, n - j0);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) vs[j] = v[j0 + j];
  __syncthreads();
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  if (i >= m) return;
  const float* a = A + i + (long long)j0 * lda;
  double acc[4] = {0, 0, 0, 0};
  for (int j = 0; j + 8 <= nc; j += 8) {
    float av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldg(a + (long long)(j + u) * lda);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u & 3] = fma((double)av[u], vs[j + u], acc[u & 3]);
  }
  part[(long long)cb * m + i] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

template <int CH>
__global__ void __launch_bounds__(256) n1(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, double* __restrict__ part) {
  __shared__ double vs[CH];
  const int cb = blockIdx.y, j0 = cb * CH, nc = min(CH, n - j0);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) vs[j] = v[j0 + j];
  __syncthreads();
  const long long i = ((long long)blockIdx.x * 256 + threadIdx.x) * 4;
  if (i >= m) return;
  const float* a = A + i + (long long)j0 * lda;
  double acc[4][2] = {};
  for (int j = 0; j + 8 <= nc; j += 8) {
    float4 av[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) av[u] = __ldg(reinterpret_cast<const float4*>(a + (long long)(j + u) * lda));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double x = vs[j + u];
      acc[0][u & 1] = fma((double)av[u].x, x, acc[0][u & 1]);
      acc[1][u & 1] = fma((double)av[u].y, x, acc[1][u & 1]);
      acc[2][u & 1] = fma((double)av[u].z, x, acc[2][u & 1]);
      acc[3][u & 1] = fma((double)av[u].w, x, acc[3][u & 1]);
    }
  }
  double* p = part + (long long)cb * m + i;
  p[0] = acc[0][0] + acc[0][1];
  p[1] = acc[1][0] + acc[1][1];
  p[2] = acc[2][0] + acc[2][1];
  p[3] = acc[3][0] + acc[3][1];
}

__global__ void __launch_bounds__(256) t0(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, int rps, double* __restrict__ part) {
  __shared__ __align__(16) double vs[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * 64 + warp * 8;
  const long long r_begin = (long long)blockIdx.y * rps, r_end = min((long long)m, r_begin + rps);
  double acc[8] = {};
  for (long long c = r_begin; c < r_end; c += 1024) {
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += 256) vs[i] = v[c + i];
    __syncthreads();
#pragma unroll 2
    for (int i = lane * 4; i < 1024; i += 128) {
      const double2 v01 = *reinterpret_cast<const double2*>(vs + i);
      const double2 v23 = *reinterpret_cast<const double2*>(vs + i + 2);
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A + (long long)(j0 + u) * lda + c + i));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[u] = fma((double)a[u].x, v01.x, acc[u]);
        acc[u] = fma((double)a[u].y, v01.y, acc[u]);
        acc[u] = fma((double)a[u].z, v23.x, acc[u]);
        acc[u] = fma((double)a[u].w, v23.y, acc[u]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double s = acc[u];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[(long long)blockIdx.y * n + j0 + u] = s;
  }
}

template <int UN>
__global__ void __launch_bounds__(256) t1(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, int rps, double* __restrict__ part) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * 64 + warp * 8;
  const long long r_begin = (long long)blockIdx.y * rps, r_end = min((long long)m, r_begin + rps);
  double acc[8] = {};
#pragma unroll UN
  for (long long i = r_begin + lane * 4; i < r_end; i += 128) {
    const double2 v01 = __ldg(reinterpret_cast<const double2*>(v + i));
    const double2 v23 = __ldg(reinterpret_cast<const double2*>(v + i + 2));
    float4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A + (long long)(j0 + u) * lda + i));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] = fma((double)a[u].x, v01.x, acc[u]);
      acc[u] = fma((double)a[u].y, v01.y, acc[u]);
      acc[u] = fma((double)a[u].z, v23.x, acc[u]);
      acc[u] = fma((double)a[u].w, v23.y, acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double s = acc[u];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) part[(long long)blockIdx.y * n + j0 + u] = s;
  }
}

// T4: CTA = 8 columns x a row split; warp w takes rows [c + 128 w, c + 128 w + 128) of every
// 1024-row chunk (each column read in 4 KB runs per CTA iteration), r read per lane from L2,
// warp sums combined in warp order through shared memory
template <int UN>
__global__ void __launch_bounds__(256) t4(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, int rps, double* __restrict__ part) {
  __shared__ double ws[8][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * 8;
  const long long r_begin = (long long)blockIdx.y * rps, r_end = min((long long)m, r_begin + rps);
  double acc[8] = {};
#pragma unroll UN
  for (long long i = r_begin + warp * 128 + lane * 4; i < r_end; i += 1024) {
    const double2 v01 = __ldg(reinterpret_cast<const double2*>(v + i));
    const double2 v23 = __ldg(reinterpret_cast<const double2*>(v + i + 2));
    float4 a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A + (long long)(j0 + u) * lda + i));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] = fma((double)a[u].x, v01.x, acc[u]);
      acc[u] = fma((double)a[u].y, v01.y, acc[u]);
      acc[u] = fma((double)a[u].z, v23.x, acc[u]);
      acc[u] = fma((double)a[u].w, v23.y, acc[u]);
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    double s = acc[u];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) ws[warp][u] = s;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    double s = ws[0][threadIdx.x];
    for (int w = 1; w < 8; ++w) s += ws[w][threadIdx.x];
    part[(long long)blockIdx.y * n + j0 + threadIdx.x] = s;
  }
}

// T5: persistent, balanced: grid = CTAs of the resident wave; item = (64-column block, 1024-row
// chunk) in column-block-major order, each CTA a contiguous item range (<= 2 column blocks), r
// staged per chunk, per-(CTA, column block) partials
__global__ void __launch_bounds__(256) t5(int m, int n, const float* __restrict__ A, long long lda,
                                          const double* __restrict__ v, int nitems, double* __restrict__ part) {
  __shared__ __align__(16) double vs[1024];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (m + 1023) / 1024;
  const int i0 = (int)((long long)blockIdx.x * nitems / gridDim.x);
  const int i1 = (int)((long long)(blockIdx.x + 1) * nitems / gridDim.x);
  double acc[8] = {};
  int cur_cb = i0 < i1 ? i0 / nch : -1, slot = 0;
  for (int it = i0; it < i1; ++it) {
    const int cb = it / nch, ch = it % nch;
    if (cb != cur_cb) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        double s = acc[u];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) part[((long long)blockIdx.x * 2 + slot) * n + cur_cb * 64 + warp * 8 + u] = s;
        acc[u] = 0.0;
      }
      cur_cb = cb;
      slot = 1;
    }
    const long long c = (long long)ch * 1024;
    __syncthreads();
    for (int i = threadIdx.x; i < 1024; i += 256) vs[i] = v[c + i];
    __syncthreads();
    const int j0 = cb * 64 + warp * 8;
#pragma unroll 2
    for (int i = lane * 4; i < 1024; i += 128) {
      const double2 v01 = *reinterpret_cast<const double2*>(vs + i);
      const double2 v23 = *reinterpret_cast<const double2*>(vs + i + 2);
      float4 a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = __ldg(reinterpret_cast<const float4*>(A + (long long)(j0 + u) * lda + c + i));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc[u] = fma((double)a[u].x, v01.x, acc[u]);
        acc[u] = fma((double)a[u].y, v01.y, acc[u]);
        acc[u] = fma((double)a[u].z, v23.x, acc[u]);
        acc[u] = fma((double)a[u].w, v23.y, acc[u]);
      }
    }
  }
  if (cur_cb >= 0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double s = acc[u];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) part[((long long)blockIdx.x * 2 + slot) * n + cur_cb * 64 + warp * 8 + u] = s;
    }
  }
}

int main() {
  float* A;
  double *v, *part;
  cudaMalloc(&A, (size_t)M * N * 4);
  cudaMalloc(&v, (size_t)M * 8);
  cudaMalloc(&part, (size_t)1200 * N * 8);
  cudaMemset(A, 0, (size_t)M * N * 4);
  cudaMemset(v, 0, (size_t)M * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 4.0 * M * N;
  auto time = [&](const char* name, auto launch) {
    for (int r = 0; r < 3; ++r) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-60s %8.1f us  %7.1f GB/s  %s\n", name, ms * 1e3 / 20, bytes / (ms * 1e-3 / 20) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  };
  time("N0 thread per row, 8 x 4-byte loads", [&] { n0<<<dim3(M / 256, N / 512), 256>>>(M, N, A, M, v, part); });
  time("N1 4 rows per thread, 16-byte loads, 512-col chunks", [&] { n1<512><<<dim3(M / 1024, N / 512), 256>>>(M, N, A, M, v, part); });
  time("N1 4 rows per thread, 16-byte loads, 256-col chunks", [&] { n1<256><<<dim3(M / 1024, N / 256), 256>>>(M, N, A, M, v, part); });
  time("N1 4 rows per thread, 16-byte loads, 1024-col chunks", [&] { n1<1024><<<dim3(M / 1024, N / 1024), 256>>>(M, N, A, M, v, part); });
  for (int per : {2, 3, 4}) {
    const int grid = 148 * per, nitems = (N / 64) * (M / 1024);
    char name[96];
    snprintf(name, sizeof name, "T5 persistent balanced, %d CTAs per SM", per);
    time(name, [&] { t5<<<grid, 256>>>(M, N, A, M, v, nitems, part); });
  }
  for (int s : {16}) {
    const int rps = M / s;
    char name[96];
    snprintf(name, sizeof name, "T4 8 cols per CTA, warps on row slices, %d splits, unroll 2", s);
    time(name, [&] { t4<2><<<dim3(N / 8, s), 256>>>(M, N, A, M, v, rps, part); });
    snprintf(name, sizeof name, "T4 8 cols per CTA, warps on row slices, %d splits, unroll 4", s);
    time(name, [&] { t4<4><<<dim3(N / 8, s), 256>>>(M, N, A, M, v, rps, part); });
  }
  for (int s : {16, 32}) {
    const int rps = M / s;
    char name[96];
    snprintf(name, sizeof name, "T0 staged r, %d row splits (many CTAs)", s);
    time(name, [&] { t0<<<dim3(N / 64, s), 256>>>(M, N, A, M, v, rps, part); });
  }
  for (int s : {4}) {
    const int rps = (M + s - 1) / s / 1024 * 1024 + (((M + s - 1) / s) % 1024 ? 1024 : 0);
    char name[96];
    snprintf(name, sizeof name, "T0 staged r, %d row splits", s);
    time(name, [&] { t0<<<dim3(N / 64, (M + rps - 1) / rps), 256>>>(M, N, A, M, v, rps, part); });
    snprintf(name, sizeof name, "T1 direct r, %d row splits, unroll 2", s);
    time(name, [&] { t1<2><<<dim3(N / 64, (M + rps - 1) / rps), 256>>>(M, N, A, M, v, rps, part); });
    snprintf(name, sizeof name, "T1 direct r, %d row splits, unroll 4", s);
    time(name, [&] { t1<4><<<dim3(N / 64, (M + rps - 1) / rps), 256>>>(M, N, A, M, v, rps, part); });
  }
  return 0;
}

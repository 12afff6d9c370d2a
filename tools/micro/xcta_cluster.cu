// Cross-CTA all-reduce of E = 528 FP64 partials on 128 CTAs through clusters of 8 (tools/micro):
// partials reduced inside each cluster through distributed shared memory (CTA r of a cluster sums
// the entries e = r mod 8 over its 8 peers), the 16 cluster partials published as tagged words in
// parity slots, every CTA polls and sums all 16 in fixed order.  Compared with xcta_reduce.cu
// variant 1 (owners, 2.9 us).  Watchdog: an abort word ends every poll.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 xcta_cluster.cu -o bin/xcta_cluster
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
typedef unsigned long long u64;
constexpr int NT = 256, NB = 128, REPS = 200, E = 528;

__device__ __forceinline__ void st_rel(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_rel(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(NT, 1) red_cluster(u64* part, volatile int* abort_flag, float* out,
                                                     unsigned long long* ns, int* stuck_it) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double mine[2][544];
  __shared__ float dst[1024];
  __shared__ int bad;
  const int t = threadIdx.x;
  const int rank = (int)cl.block_rank(), cid = blockIdx.x / 8, ncl = gridDim.x / 8;
  if (t == 0) bad = 0;
  __syncthreads();
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  float acc = 0.f;
  for (int it = 1; it <= REPS; ++it) {
    const unsigned tag = (unsigned)it;
    double* m = mine[it & 1];
    for (int e = t; e < E; e += NT) m[e] = (double)(e + blockIdx.x);
    cl.sync();
    for (int e = rank + 8 * t; e < E; e += 8 * NT) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) s += cl.map_shared_rank(m, r)[e];
      const u64 b = (u64)__double_as_longlong(s);
      u64* p = part + ((long long)((it & 1) * 16 + cid) * E + e) * 2;
      st_rel(p, ((u64)tag << 32) | (unsigned)b);
      st_rel(p + 1, ((u64)tag << 32) | (unsigned)(b >> 32));
    }
    for (int e = t; e < E; e += NT) {
      u64 v[32];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const u64* p = part + ((long long)((it & 1) * 16 + c) * E + e) * 2;
        v[2 * c] = c < ncl ? ld_rel(p) : 0ull;
        v[2 * c + 1] = c < ncl ? ld_rel(p + 1) : 0ull;
      }
      for (long long spin = 0;; ++spin) {
        bool done = true;
#pragma unroll
        for (int i = 0; i < 32; ++i) done &= (i / 2 >= ncl) || (unsigned)(v[i] >> 32) == tag;
        if (done || *abort_flag) break;
        if (spin > 200000) {
          *abort_flag = 1;
          *stuck_it = it;
          break;
        }
        __nanosleep(64);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const u64* p = part + ((long long)((it & 1) * 16 + c) * E + e) * 2;
          if (c < ncl && (unsigned)(v[2 * c] >> 32) != tag) v[2 * c] = ld_rel(p);
          if (c < ncl && (unsigned)(v[2 * c + 1] >> 32) != tag) v[2 * c + 1] = ld_rel(p + 1);
        }
      }
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < ncl)
          s += __longlong_as_double(
              (long long)(((v[2 * c + 1] & 0xffffffffull) << 32) | (v[2 * c] & 0xffffffffull)));
      dst[e] = (float)s;
    }
    __syncthreads();
    acc += dst[(t * 7 + it) % E];
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  cl.sync();
  out[blockIdx.x * NT + t] = acc;
  if (blockIdx.x == 0 && t == 0) *ns = t1 - t0;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  u64* part;
  int *abort_flag, *stuck;
  float* out;
  unsigned long long* ns;
  cudaMalloc(&part, (size_t)32 * E * 2 * 8);
  cudaMalloc(&abort_flag, 4);
  cudaMalloc(&stuck, 4);
  cudaMalloc(&out, NB * NT * 4);
  cudaMalloc(&ns, 8);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(NB);
  cfg.blockDim = dim3(NT);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 8;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = -1;
  cudaOccupancyMaxActiveClusters(&ncl, red_cluster, &cfg);
  printf("max active clusters of 8: %d\n", ncl);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(part, 0, (size_t)32 * E * 2 * 8);
    cudaMemset(abort_flag, 0, 4);
    cudaMemset(stuck, 0, 4);
    cudaError_t e = cudaLaunchKernelEx(&cfg, red_cluster, part, (volatile int*)abort_flag, out, ns, stuck);
    cudaError_t e2 = cudaDeviceSynchronize();
    int ab = 0, st = 0;
    unsigned long long h = 0;
    cudaMemcpy(&ab, abort_flag, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&st, stuck, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
    printf("rep %d: %s / %s, abort %d (iteration %d), %.2f us per reduction\n", rep,
           cudaGetErrorString(e), cudaGetErrorString(e2), ab, st, h / 1000.0 / REPS);
  }
  return 0;
}

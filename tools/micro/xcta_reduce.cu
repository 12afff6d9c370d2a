// Cost of one cross-CTA all-reduce of E partials (the leaf kernel's Gram / R12 sums) on 128
// co-resident CTAs of 256 threads, per strategy (globaltimer in CTA 0 over 200 reductions):
//   0  grid barrier, owners (lane = entry, chunks of 32) sum with plain L2 loads, grid barrier,
//      everyone loads the sums (round 1 of the leaf kernel)
//   1  tagged words: owners (lane = entry) poll the tagged partials, store tagged sums, everyone
//      polls the sums
//   2  tagged, owners spread over all CTAs (g threads per entry + shuffle tree)
//   3  = 2 with a 64 ns back-off between polls
//   4  grid barrier, spread owners with plain loads, tagged sums polled by everyone
//   5  two grid barriers only (no data)
//   6  per-CTA flags: each CTA stores its partial, then a release flag; owners poll the nb flags
//      (one word each), load, store tagged sums
// E = 528 FP64 (2 tagged words each) or 1024 FP32.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 xcta_reduce.cu -o xcta_reduce
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 256, NB = 128, REPS = 200;
typedef unsigned long long u64;

__device__ __forceinline__ void st_rel(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_rel(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_bar(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while ((int)(v - target) < 0);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
  }
  __syncthreads();
}
template <int N>
__device__ __forceinline__ void poll(u64 (&v)[N], const u64* const (&p)[N], unsigned tag, bool backoff) {
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = p[i] ? ld_rel(p[i]) : 0ull;
  for (;;) {
    bool done = true;
#pragma unroll
    for (int i = 0; i < N; ++i) done &= !p[i] || (unsigned)(v[i] >> 32) == tag;
    if (done) return;
    if (backoff) __nanosleep(64);
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (p[i] && (unsigned)(v[i] >> 32) != tag) v[i] = ld_rel(p[i]);
  }
}

// W = words per entry (payload 32 bits each)
template <int V, int W, int SKEW = 0, int ONEB = 0, int BO = 0>
__global__ void __launch_bounds__(NT, 1) red(int E, u64* part, u64* sums, unsigned* bar, unsigned* flags,
                                              float* out, unsigned long long* ns) {
  __shared__ float dst[1024];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned nbar = 0;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  float acc = 0.f;
  for (int it = 1; it <= REPS; ++it) {
    const unsigned tag = (unsigned)it;
    // publish the partial
    if (SKEW) {
      unsigned long long a0, a1;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(a0));
      do { asm volatile("mov.u64 %0, %globaltimer;" : "=l"(a1)); } while (a1 - a0 < (blockIdx.x % 8) * 150ull);
    }
    for (int e = t; e < E; e += NT)
#pragma unroll
      for (int q = 0; q < W; ++q)
        st_rel(part + ((long long)blockIdx.x * E + e) * W + q, ((u64)tag << 32) | (unsigned)(e + q + blockIdx.x));
    if (V == 5) {
      grid_bar(bar, ++nbar * NB);
      grid_bar(bar, ++nbar * NB);
      continue;
    }
    if (V == 0 || V == 4) grid_bar(bar, ++nbar * NB);
    if (V == 6) {
      __syncthreads();
      if (t == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(tag) : "memory");
      }
    }
    if (V == 0 || V == 1) {
      const int nch = (E + 31) / 32;
      for (int c = blockIdx.x; c < nch; c += NB) {
        const int e = c * 32 + lane;
        float s = 0.f;
        if (e < E) {
          constexpr int NBT = ONEB ? 16 : 8;
          for (int b0 = warp; b0 < NB; b0 += 8 * NBT) {
            const u64* p[NBT * W];
            u64 v[NBT * W];
#pragma unroll
            for (int u = 0; u < NBT; ++u)
#pragma unroll
              for (int q = 0; q < W; ++q) p[u * W + q] = part + ((long long)(b0 + 8 * u) * E + e) * W + q;
            if (V == 1) {
              poll<NBT * W>(v, p, tag, BO);
            } else {
#pragma unroll
              for (int i = 0; i < NBT * W; ++i) v[i] = __ldcg(p[i]);
            }
#pragma unroll
            for (int i = 0; i < NBT * W; ++i) s += (float)(unsigned)v[i];
          }
        }
        __shared__ float ws[8][32];
        ws[warp][lane] = s;
        __syncthreads();
        if (warp == 0 && e < E) {
          float tt = 0.f;
          for (int u = 0; u < 8; ++u) tt += ws[u][lane];
#pragma unroll
          for (int q = 0; q < W; ++q) st_rel(sums + e * W + q, ((u64)tag << 32) | (unsigned)tt);
        }
        __syncthreads();
      }
    } else {
      int epc = 8;
      while (epc < 256 && epc * NB < E) epc *= 2;
      const int g = NT / epc, j = t % g;
      if (V == 6 && (int)blockIdx.x * epc < E) {
        if (t < NB) {
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + t) : "memory");
          } while (v != tag);
        }
        __syncthreads();
      }
      for (int base = blockIdx.x * epc; base < E; base += NB * epc) {
        const int e = base + t / g;
        float s = 0.f;
        if (e < E) {
          for (int b0 = j; b0 < NB; b0 += 8 * g) {
            const u64* p[8 * W];
            u64 v[8 * W];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int q = 0; q < W; ++q)
                p[u * W + q] = b0 + u * g < NB ? part + ((long long)(b0 + u * g) * E + e) * W + q : nullptr;
            if (V == 4 || V == 6) {
#pragma unroll
              for (int i = 0; i < 8 * W; ++i) v[i] = p[i] ? __ldcg(p[i]) : 0ull;
            } else {
              poll<8 * W>(v, p, tag, V == 3);
            }
#pragma unroll
            for (int i = 0; i < 8 * W; ++i) s += (float)(unsigned)v[i];
          }
        }
        for (int o = g / 2; o >= 1; o /= 2) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (j == 0 && e < E)
#pragma unroll
          for (int q = 0; q < W; ++q) st_rel(sums + e * W + q, ((u64)tag << 32) | (unsigned)s);
      }
    }
    // everyone: the sums
    if (V == 0) {
      grid_bar(bar, ++nbar * NB);
      for (int e = t; e < E; e += NT) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < W; ++q) s += (float)(unsigned)__ldcg(sums + e * W + q);
        dst[e] = s;
      }
    } else {
      for (int e0 = t; e0 < E; e0 += 4 * NT) {
        const u64* p[4 * W];
        u64 v[4 * W];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < W; ++q) p[u * W + q] = e0 + u * NT < E ? sums + (e0 + u * NT) * W + q : nullptr;
        poll<4 * W>(v, p, tag, V == 3 || BO);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (e0 + u * NT < E) dst[e0 + u * NT] = (float)(unsigned)v[u * W];
      }
    }
    __syncthreads();
    acc += dst[(t * 7 + it) % E];
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  out[blockIdx.x * NT + t] = acc;
  if (blockIdx.x == 0 && t == 0) *ns = t1 - t0;
}

// 7: clusters of 8: partials reduced inside the cluster through distributed shared memory (each
//    CTA sums a 1/8 slice of the entries over its 8 peers), the 16 cluster partials published
//    tagged, every CTA polls and sums all 16 (fixed order).  FP64 as 2 tagged words.
#include <cooperative_groups.h>
__global__ void __launch_bounds__(NT, 1) __cluster_dims__(8, 1, 1)
    red_cluster(int E, u64* part, float* out, unsigned long long* ns) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double mine[2][544];
  __shared__ float dst[1024];
  const int t = threadIdx.x;
  const int rank = (int)cl.block_rank(), cid = blockIdx.x / 8, ncl = gridDim.x / 8;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  float acc = 0.f;
  for (int it = 1; it <= REPS; ++it) {
    const unsigned tag = (unsigned)it;
    double* m = mine[it & 1];
    for (int e = t; e < E; e += NT) m[e] = (double)(e + blockIdx.x);
    cl.sync();  // every peer's partial in its shared memory (double-buffered by parity: the
                // previous use of this buffer ended before the previous cluster barrier)
    for (int e = rank + 8 * t; e < E; e += 8 * NT) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) s += cl.map_shared_rank(m, r)[e];
      const unsigned long long b = (unsigned long long)__double_as_longlong(s);
      u64* p = part + ((long long)((it & 1) * 16 + cid) * E + e) * 2;  // parity slots
      st_rel(p, ((u64)tag << 32) | (unsigned)b);
      st_rel(p + 1, ((u64)tag << 32) | (unsigned)(b >> 32));
    }
    for (int e = t; e < E; e += NT) {
      const u64* p[32];
      u64 v[32];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        p[2 * c] = c < ncl ? part + ((long long)((it & 1) * 16 + c) * E + e) * 2 : nullptr;
        p[2 * c + 1] = c < ncl ? p[2 * c] + 1 : nullptr;
      }
      poll<32>(v, p, tag, true);
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < ncl) s += __longlong_as_double((long long)(((v[2 * c + 1] & 0xffffffffull) << 32) | (v[2 * c] & 0xffffffffull)));
      dst[e] = (float)s;
    }
    __syncthreads();
    acc += dst[(t * 7 + it) % E];
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
  out[blockIdx.x * NT + t] = acc;
  if (blockIdx.x == 0 && t == 0) *ns = t1 - t0;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  u64 *part, *sums;
  unsigned *bar, *flags;
  float* out;
  unsigned long long* ns;
  cudaMalloc(&part, (size_t)NB * 1024 * 2 * 8);
  cudaMalloc(&sums, 1024 * 2 * 8);
  cudaMalloc(&bar, 4);
  cudaMalloc(&flags, NB * 4);
  cudaMalloc(&out, NB * NT * 4);
  cudaMalloc(&ns, 8);
  const char* names[7] = {"0 barrier + owner sum + barrier", "1 tagged, lane=entry owners",
                          "2 tagged, spread owners", "3 = 2 + 64 ns back-off",
                          "4 barrier + spread owners + tagged gather", "5 two barriers only",
                          "6 per-CTA release flags + spread owners + tagged gather"};
  auto run = [&](auto kern, int v, int E, const char* what) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(part, 0, (size_t)NB * 1024 * 2 * 8);
      cudaMemset(sums, 0, 1024 * 2 * 8);
      cudaMemset(bar, 0, 4);
      cudaMemset(flags, 0, NB * 4);
      kern<<<NB, NT>>>(E, part, sums, bar, flags, out, ns);
      cudaDeviceSynchronize();
    }
    unsigned long long h;
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
    printf("%-58s %s: %6.2f us per reduction  %s\n", names[v], what, h / 1000.0 / REPS,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(red<0, 2>, 0, 528, "E=528 FP64");
  run(red<1, 2>, 1, 528, "E=528 FP64");
  run(red<1, 2, 0, 1>, 1, 528, "E=528 FP64 one batch");
  run(red<1, 2, 0, 1, 1>, 1, 528, "E=528 FP64 one batch + back-off");
  run(red<0, 2, 1>, 0, 528, "E=528 FP64 skewed");
  run(red<1, 2, 1>, 1, 528, "E=528 FP64 skewed");
  run(red<1, 2, 1, 1>, 1, 528, "E=528 FP64 skewed one batch");
  run(red<1, 2, 1, 1, 1>, 1, 528, "E=528 FP64 skewed one batch + back-off");
  run(red<5, 2, 1>, 5, 528, "E=528 FP64 skewed");
  run(red<0, 1>, 0, 1024, "E=1024 FP32");
  run(red<1, 1>, 1, 1024, "E=1024 FP32");
  run(red<1, 1, 0, 1>, 1, 1024, "E=1024 FP32 one batch");
  run(red<0, 1, 1>, 0, 1024, "E=1024 FP32 skewed");
  run(red<1, 1, 1, 1>, 1, 1024, "E=1024 FP32 skewed one batch");
  run(red<1, 1, 1, 1, 1>, 1, 1024, "E=1024 FP32 skewed one batch + back-off");
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(part, 0, (size_t)NB * 1024 * 2 * 8);
    red_cluster<<<NB, NT>>>(528, part, out, ns);
    cudaDeviceSynchronize();
  }
  {
    unsigned long long h;
    cudaMemcpy(&h, ns, 8, cudaMemcpyDeviceToHost);
    printf("%-58s %s: %6.2f us per reduction  %s\n", "7 cluster-8 DSMEM + all poll 16 cluster partials",
           "E=528 FP64", h / 1000.0 / REPS, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

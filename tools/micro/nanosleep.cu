// Actual duration of __nanosleep(t) on one warp (cycles per call, averaged over 100 calls).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(long long* out, int t, int n) {
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) __nanosleep(t);
  long long c1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (c1 - c0) / n;
}
int main() {
  long long* d; cudaMalloc(&d, 1024 * 8);
  long long h[8];
  for (int t : {0, 20, 32, 100, 256, 1000, 4000}) {
    for (int threads : {32, 256}) {
      k<<<1, threads>>>(d, t, 100);
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      printf("nanosleep(%d) threads=%d: %lld cycles/call\n", t, threads, h[0]);
    }
  }
  return 0;
}

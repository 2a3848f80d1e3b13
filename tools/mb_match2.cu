// match_any throughput vs number of distinct values in the warp (sm_100a)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void thr(unsigned* out, int iters, int ndist) {
  unsigned v[8], acc = 0;
  for (int k = 0; k < 8; ++k) v[k] = ((threadIdx.x & 31) % ndist) * 977u + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { unsigned p = __match_any_sync(0xffffffffu, v[k] + (unsigned)i * 131u); acc += p; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned)((t1 - t0) / (iters * 8));
  out[1 + (threadIdx.x) % 1024] = acc;
}
int main() {
  unsigned* d; cudaMalloc(&d, 8192); unsigned h[2];
  for (int nd : {1, 2, 4, 8, 16, 32}) {
    thr<<<1, 32 * 32>>>(d, 500, nd); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("32 warps/SM, %2d distinct values: %u cyc per match per warp (%.1f per SM)\n", nd, h[0], h[0] / 32.0);
  }
  return 0;
}

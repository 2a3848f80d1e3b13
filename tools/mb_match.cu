// microbenchmark: __match_any_sync latency and throughput on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(unsigned* out, int iters, unsigned seed) {
  unsigned v = (threadIdx.x * 2654435761u + seed) & 255u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    unsigned p = __match_any_sync(0xffffffffu, v);
    v = (v + p) & 255u;  // dependent chain
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (unsigned)((t1 - t0) / iters); }
  out[1 + threadIdx.x] = v;
}
__global__ void thr(unsigned* out, int iters, unsigned seed) {
  unsigned v[8], acc = 0;
  for (int k = 0; k < 8; ++k) v[k] = ((threadIdx.x + k * 7) * 2654435761u + seed) & 255u;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { unsigned p = __match_any_sync(0xffffffffu, v[k] + i); acc += p; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (unsigned)((t1 - t0) / (iters * 8));
  out[1 + (blockIdx.x * blockDim.x + threadIdx.x) % 1024] = acc;
}
__global__ void shfl_lat(unsigned* out, int iters) {
  unsigned v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (unsigned)((t1 - t0) / iters);
  out[1 + threadIdx.x] = v;
}
int main() {
  unsigned* d; cudaMalloc(&d, 8192); unsigned h[2];
  lat<<<1, 32>>>(d, 10000, 1); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); printf("match_any latency (1 warp): %u cyc\n", h[0]);
  shfl_lat<<<1, 32>>>(d, 10000); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); printf("shfl latency: %u cyc\n", h[0]);
  for (int w : {1, 4, 8, 16, 32}) {
    thr<<<1, 32 * w>>>(d, 2000, 3); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("match_any issue interval, %d warps / SM (8 independent per warp): %u cyc per match per warp\n", w, h[0]);
  }
  return 0;
}

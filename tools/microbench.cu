// Micro-benchmarks that bound the design of the point kernels (not product
// code): cost of 1.3M random global atomics on 32400 counters, with and
// without return, and of a pure streaming read of 1M xyz records.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench.cu -o /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_red(const uint32_t* tile, int n, uint32_t* cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + tile[i], 1u);
}
__global__ void k_atom_store(const uint32_t* tile, int n, uint32_t* cnt, unsigned long long* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t p = atomicAdd(cnt + tile[i], 1u);
    out[p % n] = i;
  }
}
__global__ void k_atom_only(const uint32_t* tile, int n, uint32_t* cnt, int K, uint32_t* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t p = atomicAdd(cnt + tile[i] * K + (i % K), 1u);
    if (p == 0xFFFFFFFFu) sink[0] = 1;
  }
}
__global__ void k_red_k(const uint32_t* tile, int n, uint32_t* cnt, int K) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + tile[i] * K + (i % K), 1u);
}
__global__ void k_read(const float* xyz, int n, float* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = xyz[3 * i] + xyz[3 * i + 1] * xyz[3 * i + 2];
    if (v == 12345.f) sink[0] = v;
  }
}
__global__ void k_read4(const float4* xyz, int n4, float* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) {
    float4 v = xyz[i];
    if (v.x + v.y + v.z + v.w == 12345.f) sink[0] = 1;
  }
}
__global__ void k_gather32(const float4* rec, const uint32_t* idx, int n, float* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t j = idx[i];
    float4 a = rec[2 * j], b = rec[2 * j + 1];
    if (a.x + b.y == 12345.f) sink[0] = 1;
  }
}
__global__ void k_gather_aos(const float* xyz, const float* op, const float4* f, const uint32_t* idx, int n, float* sink) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    uint32_t j = idx[i];
    float s = xyz[3 * j] + xyz[3 * j + 1] + xyz[3 * j + 2] + op[j];
    float4 v = f[j];
    if (s + v.x + v.w == 12345.f) sink[0] = 1;
  }
}
__global__ void flush(float* b, size_t n, float v) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = v;
}

int main() {
  const int n = 1300000, T = 32400, NP = 1 << 20;
  uint32_t* h = new uint32_t[n];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % T; }
  uint32_t *tile, *cnt, *idx;
  unsigned long long* out;
  float *xyz, *sink, *fl, *op;
  float4 *rec, *f;
  cudaMalloc(&tile, n * 4); cudaMalloc(&cnt, (size_t)n * 4 * 2); cudaMalloc(&out, n * 8);
  cudaMalloc(&xyz, NP * 12); cudaMalloc(&sink, 64); cudaMalloc(&op, NP * 4); cudaMalloc(&f, NP * 16);
  cudaMalloc(&rec, NP * 32); cudaMalloc(&idx, n * 4);
  size_t nfl = 64ull << 20; cudaMalloc(&fl, nfl * 4);
  cudaMemcpy(tile, h, n * 4, cudaMemcpyHostToDevice);
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % NP; }
  cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(xyz, 0, NP * 12); cudaMemset(rec, 0, NP * 32); cudaMemset(op, 0, NP * 4); cudaMemset(f, 0, NP * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto time = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      flush<<<1184, 256>>>(fl, nfl, (float)r);
      cudaMemset(cnt, 0, T * 4 * 16);
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (r) best = ms < best ? ms : best;
    }
    printf("%-40s %8.2f us  (%s)\n", name, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  int g = (n + 255) / 256;
  time("RED 1.3M random on 32400 ctrs", [&] { k_red<<<g, 256>>>(tile, n, cnt); });
  time("ATOM+STG 1.3M random", [&] { k_atom_store<<<g, 256>>>(tile, n, cnt, out); });
  for (int K : {1, 4, 16}) {
    char nm[64];
    snprintf(nm, 64, "ATOM(ret) 1.3M on %d ctrs", T * K);
    time(nm, [&] { k_atom_only<<<g, 256>>>(tile, n, cnt, K, (uint32_t*)sink); });
    snprintf(nm, 64, "RED 1.3M on %d ctrs", T * K);
    time(nm, [&] { k_red_k<<<g, 256>>>(tile, n, cnt, K); });
  }
  time("read xyz AoS 1M (12 MB)", [&] { k_read<<<(NP + 255) / 256, 256>>>(xyz, NP, sink); });
  time("read 12 MB float4", [&] { k_read4<<<(NP * 3 / 4 + 255) / 256, 256>>>((float4*)xyz, NP * 3 / 4, sink); });
  time("gather 1.3M x 32B records", [&] { k_gather32<<<g, 256>>>(rec, idx, n, sink); });
  time("gather 1.3M x (xyz,o,f) AoS", [&] { k_gather_aos<<<g, 256>>>(xyz, op, f, idx, n, sink); });
  time("empty kernel", [&] { k_read<<<1, 32>>>(xyz, 0, sink); });
  return 0;
}

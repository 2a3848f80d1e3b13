// spatial_order.cuh — one-time spatial (Morton) ordering of a static cloud.
//
// Not a step of the rasterizer: a preprocessing the caller may apply once to
// a static point cloud (the pre-extracted global cloud of P:94-95 /
// P:146-153, or the shared cloud of a training view batch) so that points
// close in space are close in memory.  The rasterizer's result is defined on
// whatever order the caller passes (the tie-break is the index in that
// order, R8); on a spatially ordered cloud the per-(point, tile)
// slot atomics of a warp hit a handful of tiles (warp-aggregated), the tile
// buckets are written in runs, and the blends' record gathers and gradient
// atomics stay in L2.
//
// perm = stable sort of the points by the 30-bit Morton code of their
// position quantised to a 1024^3 grid over the cloud's bounding box
// (non-finite points last), by the device-wide LSD radix kernels of
// single_sort.cuh (4 passes of 8-bit digits).
#pragma once
#include "single_sort.cuh"

namespace inpc {

// monotone map float -> uint32 (total order of finite floats)
__device__ __forceinline__ uint32_t float_order_key(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float float_from_order_key(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

// box[0..2] = ordered min, box[3..5] = ordered max (init 0xFFFFFFFF / 0)
__global__ void __launch_bounds__(256) k_aabb(const float* __restrict__ xyz, int64_t N, uint32_t* box) {
  uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const float p[3] = {__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2)};
    if (!(isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]))) continue;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint32_t k = float_order_key(p[a]);
      lo[a] = min(lo[a], k);
      hi[a] = max(hi[a], k);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
    hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(box + a, lo[a]);
      atomicMax(box + 3 + a, hi[a]);
    }
  }
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}

__global__ void __launch_bounds__(256) k_morton_keys(const float* __restrict__ xyz, int64_t N,
                                                     const uint32_t* __restrict__ box,
                                                     unsigned long long* __restrict__ keys,
                                                     uint32_t* __restrict__ vals) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const float p[3] = {__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2)};
  uint32_t code = 0xFFFFFFFFu;  // non-finite: last
  if (isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2])) {
    code = 0u;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float lo = float_from_order_key(box[a]), hi = float_from_order_key(box[3 + a]);
      const float ext = hi - lo;
      const float t = ext > 0.0f ? (p[a] - lo) / ext : 0.0f;
      const uint32_t q = (uint32_t)min(max((int)(t * 1024.0f), 0), 1023);
      code |= spread10(q) << a;
    }
  }
  keys[i] = code;
  vals[i] = (uint32_t)i;
}

}  // namespace inpc

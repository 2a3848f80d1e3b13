// single_sort.cuh — NEXT f4: the original INPC ordering as an A/B baseline
// (PAPER.md P:100): four fragment copies per point, one 64-bit key
// (pixel index << 32 | depth bits) per copy, one device-wide stable LSD radix
// sort (8-bit digits, ceil(53/8) = 7 passes at 1080p), per-pixel ranges.
//
// Stability and the input order (point index, block corner) make every
// pixel's list equal to its (depth, index) order: the same per-pixel order the
// tiled path reaches (tests compare both with the oracle's O7).
#pragma once
#include "kernels.cuh"

namespace inpc {

constexpr int kRxItems = 16;                 // elements per lane per radix tile
constexpr int kRxTile = 32 * kRxItems;       // one warp per tile
constexpr int kRxWarps = 4;                  // warps (tiles) per CTA

// Emit the 4 fragment copies of every point at fixed slots 4 i + corner;
// copies outside the image (or of culled points) get the all-ones key and
// sort last.  Counts the real copies.
__global__ void __launch_bounds__(256) k_emit_pixel_frags(DevCfg g, const PointRec* __restrict__ rec,
                                                          int64_t N, unsigned long long* __restrict__ keys,
                                                          uint32_t* __restrict__ vals,
                                                          unsigned long long* __restrict__ n_valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t cnt = 0;
  if (i < N) {
    const float4 A = __ldg(&rec[i].a);
    Foot f;
    const bool ok = rec_foot<0>(g, A, 0.0f, f);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int px = f.x0 + (c & 1), py = f.y0 + (c >> 1);
      unsigned long long k = ~0ull;
      if (ok && px >= f.xlo && px <= f.xhi && py >= f.ylo && py <= f.yhi) {
        k = ((unsigned long long)(uint32_t)(py * g.W + px) << 32) | __float_as_uint(A.z);
        ++cnt;
      }
      keys[4 * i + c] = k;
      vals[4 * i + c] = (uint32_t)i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_valid, (unsigned long long)cnt);
}

// Per-tile digit histograms, stored digit-major: hist[d * tiles + tile].
__global__ void __launch_bounds__(kRxWarps * 32) k_rx_hist(const unsigned long long* __restrict__ keys,
                                                           int64_t n, int shift, int tiles,
                                                           uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[kRxWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kRxWarps + warp;
  for (int d = lane; d < 256; d += 32) cnt[warp][d] = 0u;
  __syncwarp();
  if (tile < tiles) {
    const int64_t base = (int64_t)tile * kRxTile;
#pragma unroll 4
    for (int r = 0; r < kRxItems; ++r) {
      const int64_t e = base + r * 32 + lane;
      if (e < n) atomicAdd(&cnt[warp][(uint32_t)(keys[e] >> shift) & 255u], 1u);
    }
    __syncwarp();
    for (int d = lane; d < 256; d += 32) hist[(size_t)d * tiles + tile] = cnt[warp][d];
  }
}

// Stable scatter: rounds of 32 consecutive elements in order; lanes with the
// same digit rank themselves (warp_peers ballots); the warp's running
// per-digit cursor starts at the scanned offset of (digit, tile).
__global__ void __launch_bounds__(kRxWarps * 32) k_rx_scatter(
    const unsigned long long* __restrict__ kin, const uint32_t* __restrict__ vin, int64_t n, int shift,
    int tiles, const uint32_t* __restrict__ offs, unsigned long long* __restrict__ kout,
    uint32_t* __restrict__ vout) {
  __shared__ uint32_t cur[kRxWarps][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x * kRxWarps + warp;
  if (tile >= tiles) return;
  for (int d = lane; d < 256; d += 32) cur[warp][d] = offs[(size_t)d * tiles + tile];
  __syncwarp();
  const int64_t base = (int64_t)tile * kRxTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < kRxItems; ++r) {
    const int64_t e = base + r * 32 + lane;
    const bool valid = e < n;
    unsigned long long k = 0;
    uint32_t v = 0, d = 0u;
    if (valid) {
      k = kin[e];
      v = vin[e];
      d = (uint32_t)(k >> shift) & 255u;
    }
    const unsigned peers = warp_peers<8>(d, valid);
    if (valid) {
      const uint32_t pos = cur[warp][d] + __popc(peers & lt);
      kout[pos] = k;
      vout[pos] = v;
    }
    __syncwarp();
    if (valid && (peers & lt) == 0) cur[warp][d] += __popc(peers);  // the lowest peer advances
    __syncwarp();
  }
}

// Generic exclusive scan of n u32 (decoupled look-back, one pass); state
// and ctl are zero on entry and left zero on exit.
__global__ void __launch_bounds__(kScanThreads) k_scan_u32(int64_t n, uint32_t* __restrict__ data,
                                                           unsigned long long* state, ScanCtl* ctl) {
  __shared__ uint32_t warp_tot[kScanThreads / 32];
  __shared__ uint32_t s_prefix, s_bid;
  if (threadIdx.x == 0) s_bid = atomicAdd(&ctl->ticket, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const int64_t i0 = (int64_t)bid * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    c[k] = i0 + k < n ? data[i0 + k] : 0u;
    sum += c[k];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < kScanThreads / 32 ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = w;
  }
  __syncthreads();
  const uint32_t excl = (wid ? warp_tot[wid - 1] : 0u) + x - sum;
  const uint32_t agg = warp_tot[kScanThreads / 32 - 1];
  if (threadIdx.x == 0) {
    volatile unsigned long long* vs = state;
    if (bid == 0) {
      vs[0] = (2ull << 32) | agg;
      s_prefix = 0;
    } else {
      vs[bid] = (1ull << 32) | agg;
      uint32_t prefix = 0;
      int b = (int)bid - 1;
      while (true) {
        unsigned long long v = vs[b];
        uint32_t flag = (uint32_t)(v >> 32);
        if (flag == 0) continue;
        prefix += (uint32_t)v;
        if (flag == 2) break;
        --b;
      }
      __threadfence();
      vs[bid] = (2ull << 32) | (prefix + agg);
      s_prefix = prefix;
    }
  }
  __syncthreads();
  uint32_t off = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (i0 + k < n) data[i0 + k] = off;
    off += c[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_bid = atomicAdd(&ctl->done, 1u);
  }
  __syncthreads();
  if (s_bid == gridDim.x - 1) {
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) state[b] = 0ull;
    if (threadIdx.x == 0) {
      ctl->ticket = 0u;
      ctl->done = 0u;
    }
  }
}

// pixel_ranges[p] = first sorted position with pixel >= p, p in [0, P].
__global__ void __launch_bounds__(256) k_pixel_ranges(const unsigned long long* __restrict__ keys, int64_t n,
                                                      int64_t P, uint32_t* __restrict__ ranges) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t p = i < n ? min((int64_t)(keys[i] >> 32), P) : P;
  const int64_t q = i > 0 ? min((int64_t)(keys[i - 1] >> 32), P) : -1;
  for (int64_t t = q + 1; t <= p; ++t) ranges[t] = (uint32_t)i;
}

}  // namespace inpc

// kernels.cuh — the sm_100a kernels of the rasterizer hot path (H1-H8).
//
//   k_project_count  H1+H2: project, footprint, count entries per 8x8 tile
//   k_scan_tiles     H3:    decoupled look-back exclusive scan of the tile
//                           counts -> tile ranges, F_t; list of big tiles
//   k_scatter        H5:    write (depth key << 32 | point index) into the
//                           tile buckets (bucket order arbitrary)
//   k_sort_big       H4+H6 for tiles over the warp-sort cap: SMEM chunk
//                           sort + merge passes (cooperative, grid sync)
//   k_blend_fwd      H4+H6 for the other tiles (warp bitonic sort of the
//                           unique 64-bit keys) fused with H7: one warp per
//                           8x8 tile, per-pixel fragment bitmasks, front-to-
//                           back blend (Eq. 1), alpha clamp, early termination
//   k_blend_bwd      H8:    one warp per tile, reverse-order backward
//                           (Eq. 2 corrected), SMEM pre-reduction per point
//
// The two-stage sort of the paper (depth sort of the points, then
// a stable sort of the tile copies by tile key) is replaced by a bucket
// scatter + per-tile sort of the unique (depth, index) key: the same per-tile
// lists bit for bit at a fraction of the sort traffic.
#pragma once
#include <cooperative_groups.h>

#include "raster_math.cuh"

namespace inpc {

#ifndef INPC_WPB
#define INPC_WPB 4
#endif
constexpr int kWarpsPerBlock = INPC_WPB;  // blend kernels: one warp per tile, WPB warps per CTA
constexpr int kWarpSortCap = 256;    // tiles above this go through k_sort_big
constexpr int kBigChunk = 2048;      // chunk of k_sort_big's SMEM sort (16 KB of keys)
constexpr int kBigThreads = 512;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;        // tiles per scan thread
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kPointThreads = 256;
constexpr int kPPT = 4;              // points per thread in the point kernels

// ---------------------------------------------------------------- H1 + H2
// Per-point record written once by the projection kernel and gathered by
// every later stage (one 32-byte sector per point instead of xyz + o + f
// scattered over three arrays):
//   bilinear: u, v, z_c, o, f0..f3 (features packed when C == 4, else 0)
//   Gaussian: u, v, z_c, o, conic a, b, c, radius r
// z_c = 0 marks a point without footprint (culled or off image).
struct __align__(16) PointRec {
  float4 a;  // u, v, z_c, o
  float4 b;  // features | conic + radius
};

// NEXT f1: evaluate the point's SH features (feat = coefficients [N, C, 9])
// into the packed record (C == 4) or the per-view feature buffer feat_out.
__device__ __forceinline__ void sh_point_features(const DevCam& cam, const DevCfg& g,
                                                  const float* __restrict__ sh, int64_t i, float X,
                                                  float Y, float Z, bool packed, float4& F,
                                                  float* __restrict__ feat_out) {
  float B[9];
  sh_dir_basis(cam, X, Y, Z, B);
  const float* shi = sh + (size_t)i * g.C * 9;
  if (packed) {
    // 36 coefficients = 9 aligned float4 (144 B per point)
    float q[36];
    const float4* s4 = reinterpret_cast<const float4*>(shi);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const float4 v = __ldg(s4 + k);
      q[4 * k] = v.x; q[4 * k + 1] = v.y; q[4 * k + 2] = v.z; q[4 * k + 3] = v.w;
    }
    float f[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      f[c] = 0.0f;
#pragma unroll
      for (int k = 0; k < 9; ++k) f[c] += q[c * 9 + k] * B[k];
    }
    F = make_float4(f[0], f[1], f[2], f[3]);
  } else {
    for (int c = 0; c < g.C; ++c) feat_out[(size_t)i * g.C + c] = sh_feature(shi, c, B);
  }
}

// NEXT f1 backward: dL/dcoeff[c][k] += dL/df_c Y_k(d)  (g_sh [N, C, 9]).
// A block handles kShPts points: their basis values and dL/df are staged in
// SMEM and the kShPts*C*9 contiguous coefficient gradients are
// read-modify-written with consecutive threads on consecutive floats
// (C = 4: float4, 9 per point; divisions by constants).  Points whose dL/df
// is zero (not visible) are not touched.
constexpr int kShPts = 64;
template <int CT>
__global__ void __launch_bounds__(256) k_sh_grad(DevCam cam, DevCfg g, const float* __restrict__ xyz,
                                                 int64_t N, const float* __restrict__ g_f,
                                                 float* __restrict__ g_sh) {
  __shared__ float sB[kShPts][9];
  __shared__ float sG[kShPts * 64];
  const int64_t p0 = (int64_t)blockIdx.x * kShPts;
  const int np = (int)min((int64_t)kShPts, N - p0);
  const int C = CT ? CT : g.C;
  if (threadIdx.x < np) {
    const int64_t i = p0 + threadIdx.x;
    sh_dir_basis(cam, __ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2), sB[threadIdx.x]);
  }
  for (int j = threadIdx.x; j < np * C; j += blockDim.x) sG[j] = __ldg(g_f + p0 * C + j);
  __syncthreads();
  if (CT == 4) {
    float4* out4 = reinterpret_cast<float4*>(g_sh + p0 * 36);  // 144 B per point: 16-B aligned
    for (int j4 = threadIdx.x; j4 < np * 9; j4 += blockDim.x) {
      const int p = j4 / 9, r0 = 4 * (j4 - p * 9);
      float gf[4], bk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = r0 + q, c = r / 9, k = r - c * 9;
        gf[q] = sG[p * 4 + c];
        bk[q] = sB[p][k];
      }
      if (gf[0] == 0.0f && gf[1] == 0.0f && gf[2] == 0.0f && gf[3] == 0.0f) continue;
      float4 v = out4[j4];
      v.x += gf[0] * bk[0];
      v.y += gf[1] * bk[1];
      v.z += gf[2] * bk[2];
      v.w += gf[3] * bk[3];
      out4[j4] = v;
    }
  } else {
    const int per_pt = C * 9;
    float* out = g_sh + p0 * per_pt;
    for (int j = threadIdx.x; j < np * per_pt; j += blockDim.x) {
      const int p = j / per_pt, r = j - p * per_pt, c = r / 9, k = r - c * 9;
      const float gf = sG[p * C + c];
      if (gf != 0.0f) out[j] += gf * sB[p][k];
    }
  }
}

// ---------------------------------------------------------------- chunk culling
// A static cloud in spatial order is cut into chunks of kChunkPoints
// consecutive points with a bounding box each (k_chunk_bounds, once).  The
// binning kernels of a view then skip the chunks whose box cannot produce a
// footprint in the view's frame -- behind the near plane, or projecting
// wholly outside the image or the screen band (sort-first sharding, SURVEY
// §8(e)).  One CTA of the projection / scatter kernels covers exactly one
// chunk.  Conservative: a box crossing the near plane is kept; the projected
// hull of the 8 corners bounds every interior point (perspective keeps
// convexity in front of the camera), widened by 2 px for the 2x2 footprint
// and fp32 rounding.
constexpr int kChunkPoints = kPointThreads * kPPT;  // 1024

__global__ void __launch_bounds__(kPointThreads) k_chunk_bounds(const float* __restrict__ xyz, int64_t N,
                                                                float* __restrict__ box) {
  const int64_t i0 = (int64_t)blockIdx.x * kChunkPoints + threadIdx.x;
  float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    const int64_t i = i0 + k * kPointThreads;
    if (i >= N) break;
    const float p[3] = {__ldg(xyz + 3 * i), __ldg(xyz + 3 * i + 1), __ldg(xyz + 3 * i + 2)};
    if (!(isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]))) continue;  // never has a footprint
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = fminf(lo[a], p[a]);
      hi[a] = fmaxf(hi[a], p[a]);
    }
  }
  __shared__ float red[6][kPointThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
    if (lane == 0) {
      red[a][w] = lo[a];
      red[3 + a][w] = hi[a];
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    float v = red[threadIdx.x][0];
    for (int q = 1; q < kPointThreads / 32; ++q)
      v = threadIdx.x < 3 ? fminf(v, red[threadIdx.x][q]) : fmaxf(v, red[threadIdx.x][q]);
    box[(size_t)blockIdx.x * 6 + threadIdx.x] = v;
  }
}

// true when chunk `b`'s box can hold a point with a footprint in the view's
// frame / band (warp-uniform: lanes 0-7 project the 8 corners, lane 0's
// reductions are broadcast)
__device__ __forceinline__ bool chunk_live(const DevCam& cam, const DevCfg& g, const float* __restrict__ box,
                                           int64_t b) {
  const int lane = threadIdx.x & 31;
  const float* bx = box + (size_t)b * 6;
  const float x0 = __ldg(bx), y0 = __ldg(bx + 1), z0 = __ldg(bx + 2);
  const float x1 = __ldg(bx + 3), y1 = __ldg(bx + 4), z1 = __ldg(bx + 5);
  if (!(x0 <= x1 && y0 <= y1 && z0 <= z1)) return false;  // no finite point: no footprint
  const bool act = lane < 8;
  const float X = (lane & 1) ? x1 : x0, Y = (lane & 2) ? y1 : y0, Z = (lane & 4) ? z1 : z0;
  const float xc = cam.R[0] * X + cam.R[1] * Y + cam.R[2] * Z + cam.t[0];
  const float yc = cam.R[3] * X + cam.R[4] * Y + cam.R[5] * Z + cam.t[1];
  const float zc = cam.R[6] * X + cam.R[7] * Y + cam.R[8] * Z + cam.t[2];
  auto allmax = [&](float v) {
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return __shfl_sync(0xffffffffu, v, 0);
  };
  auto allmin = [&](float v) {
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return __shfl_sync(0xffffffffu, v, 0);
  };
  // z_c is affine in the point: its extremes over the box are at corners
  if (allmax(act ? zc : -INFINITY) < cam.z_near * 0.999f) return false;  // all behind the near plane
  if (!(allmin(act ? zc : INFINITY) > cam.z_near * 1.001f)) return true;  // crosses it: keep
  const float u = cam.fx * (xc / zc) + cam.cx, v = cam.fy * (yc / zc) + cam.cy;
  const float umin = allmin(act ? u : INFINITY), umax = allmax(act ? u : -INFINITY);
  const float vmin = allmin(act ? v : INFINITY), vmax = allmax(act ? v : -INFINITY);
  if (!(isfinite(umin) && isfinite(umax) && isfinite(vmin) && isfinite(vmax))) return true;
  // a point's 2x2 block covers pixels floor(u - 1/2) + {0, 1}: within [umin - 1/2, umax + 1/2]
  const float row_lo = (float)(g.ty0 * kTile), row_hi = (float)min(g.ty1 * kTile, g.H);
  if (umax + 2.5f < 0.0f || umin - 2.5f >= (float)g.W) return false;
  if (vmax + 2.5f < row_lo || vmin - 2.5f >= row_hi) return false;
  return true;
}

// kPPT points per thread, the position / opacity loads of all of them issued
// before any compute so enough bytes are in flight to cover HBM latency.
// Bilinear with a scatter record (the unfused path of large clouds): the
// record, the slots and the packed features are touched only for points with
// a footprint (culled points cost their 16 input bytes and an 8-byte zero
// scatter record), and the per-(point, tile) slot atomics are aggregated over
// the lanes of a warp that hit the same tile (__match_any_sync per block
// corner, one atomicAdd per distinct tile) when a warp's 32 consecutive
// points fall into a handful of tiles (a spatially ordered cloud).
template <int MODE, bool SH>
__global__ void __launch_bounds__(kPointThreads, 4) k_project_count(
    DevCam cam, DevCfg g, const float* __restrict__ xyz, const float* __restrict__ opacity,
    const float* __restrict__ feat, bool pack, int64_t N, PointRec* __restrict__ rec,
    uint32_t* __restrict__ tile_count, uint4* __restrict__ slots, uint32_t* __restrict__ dbg_key,
    uint32_t* __restrict__ dbg_tiles, float* __restrict__ feat_out, uint2* __restrict__ scat,
    const float* __restrict__ chunk_box, uint8_t* __restrict__ chunk_alive) {
  // CTA b covers points [b kChunkPoints, (b + 1) kChunkPoints): one chunk
  const int64_t stride = kPointThreads;
  const int64_t i0 = (int64_t)blockIdx.x * kChunkPoints + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  // bilinear + scatter record: visible-only writes, warp-aggregated slots
  const bool agg = MODE == 0 && scat != nullptr && tile_count != nullptr;
  if (agg && chunk_box) {  // the whole chunk is skipped when its box cannot reach the frame / band
    const bool live = chunk_live(cam, g, chunk_box, blockIdx.x);
    if (threadIdx.x == 0) chunk_alive[blockIdx.x] = live ? 1 : 0;
    if (!live) return;
  }
  float X[kPPT], Y[kPPT], Z[kPPT], O[kPPT];
  float4 Fv[kPPT];
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    Fv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < N) {
      X[k] = __ldg(xyz + 3 * i);
      Y[k] = __ldg(xyz + 3 * i + 1);
      Z[k] = __ldg(xyz + 3 * i + 2);
      O[k] = __ldg(opacity + i);
      if (MODE == 0 && pack && !SH && !agg) Fv[k] = __ldg(reinterpret_cast<const float4*>(feat) + i);
    }
  }
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    if (agg) {
      if (!__any_sync(0xffffffffu, i < N)) break;  // warp-uniform: the slot collectives need every lane
    } else if (i >= N) {
      break;
    }
    const bool inr = i < N;
    Proj p;
    Foot f;
    float ca = 0.f, cb = 0.f, cc = 0.f, r = 0.f;
    bool vis = false, ok = false;
    if (inr) {
      vis = project_point(cam, X[k], Y[k], Z[k], p);
      if (vis) {
        if (MODE == 0) ok = foot_bilinear(g, p.u, p.v, f);
        else ok = gauss_conic(cam, g, p, ca, cb, cc, r) && gauss_rect(g, p.u, p.v, r, f);
      }
    }
    if (agg && ok && pack && !SH) Fv[k] = __ldg(reinterpret_cast<const float4*>(feat) + i);
    if (SH && ok) sh_point_features(cam, g, feat, i, X[k], Y[k], Z[k], MODE == 0 && pack, Fv[k], feat_out);
    if (inr && dbg_key) {
      dbg_key[i] = vis ? __float_as_uint(p.zc) : 0xFFFFFFFFu;
      dbg_tiles[i] = ok ? (uint32_t)((f.xhi / kTile - f.xlo / kTile + 1) *
                                     (f.yhi / kTile - f.ylo / kTile + 1))
                        : 0u;
    }
    if (agg) {
      // footprint tiles of the 2x2 block (corner c = 2 dy + dx), band-clipped
      uint32_t tile[4];
      uint32_t tb = 0u;
      if (ok) {
        const int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
        const int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
        uint32_t vm = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int tx = tx_lo + (c & 1), ty = ty_lo + (c >> 1);
          const bool in = tx <= tx_hi && ty <= ty_hi;
          tile[c] = in ? (uint32_t)(ty * g.tiles_x + tx) : 0xFFFFFFFFu;
          vm |= (in ? 1u : 0u) << c;
        }
        tb = (uint32_t)(ty_lo * g.tiles_x + tx_lo) | (vm << 28);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) tile[c] = 0xFFFFFFFFu;
      }
      // all four corners' atomics in flight before any result is used.
      // (__match_any_sync costs ~2 cycles per distinct value per SM; a
      // guard that skipped it for warps with many distinct tiles measured
      // slower on the spatially ordered cfg 4 / cfg 5 clouds: 441 -> 777 us)
      unsigned peers[4];
      uint32_t base[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        peers[c] = __match_any_sync(0xffffffffu, tile[c]);
        base[c] = 0u;
        if (tile[c] != 0xFFFFFFFFu && lane == __ffs(peers[c]) - 1)
          base[c] = atomicAdd(tile_count + tile[c], (uint32_t)__popc(peers[c]));
      }
      if (ok) {
        if (g.flags & kFlagRec16) {  // compact record, features stay in feat
          reinterpret_cast<float4*>(rec)[i] = make_float4(p.u, p.v, p.zc, O[k]);
        } else {
          PointRec pr;
          pr.a = make_float4(p.u, p.v, p.zc, O[k]);
          pr.b = pack ? Fv[k] : make_float4(0.f, 0.f, 0.f, 0.f);
          rec[i] = pr;
        }
      }
      uint32_t sl[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t b = __shfl_sync(0xffffffffu, base[c], __ffs(peers[c]) - 1);
        sl[c] = tile[c] != 0xFFFFFFFFu ? b + (uint32_t)__popc(peers[c] & lt) : 0xFFFFFFFFu;
      }
      if (ok) slots[i] = make_uint4(sl[0], sl[1], sl[2], sl[3]);
      if (inr) scat[i] = ok ? make_uint2(__float_as_uint(p.zc), tb) : make_uint2(0u, 0u);
      continue;
    }
    PointRec pr;
    pr.a = make_float4(p.u, p.v, ok ? p.zc : 0.0f, O[k]);
    if (MODE == 0) pr.b = pack ? Fv[k] : make_float4(0.f, 0.f, 0.f, 0.f);
    else pr.b = make_float4(ca, cb, cc, r);
    rec[i] = pr;
    if (!ok || !tile_count) continue;  // tile_count null: records only (f4 baseline)
    int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
    int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
    if (MODE == 0) {
      uint32_t sl[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int tx = tx_lo + (c & 1), ty = ty_lo + (c >> 1);
        sl[c] = (tx <= tx_hi && ty <= ty_hi) ? atomicAdd(tile_count + (size_t)ty * g.tiles_x + tx, 1u)
                                             : 0xFFFFFFFFu;
      }
      slots[i] = make_uint4(sl[0], sl[1], sl[2], sl[3]);
    } else {
      for (int ty = ty_lo; ty <= ty_hi; ++ty)
        for (int tx = tx_lo; tx <= tx_hi; ++tx) atomicAdd(tile_count + (size_t)ty * g.tiles_x + tx, 1u);
    }
  }
}

// Footprint rectangle of a point from its record (same ops as at projection).
template <int MODE>
__device__ __forceinline__ bool rec_foot(const DevCfg& g, float4 a, float radius, Foot& f) {
  if (!(a.z > 0.0f)) return false;
  if (MODE == 0) return foot_bilinear(g, a.x, a.y, f);
  return gauss_rect(g, a.x, a.y, radius, f);
}

// ---------------------------------------------------------------- H3
// Scalars shared between the kernels of one view (device memory, zeroed
// before k_scan_tiles).
struct ViewScalars {
  uint32_t Ft;       // total tile entries
  uint32_t num_big;  // tiles with more than kWarpSortCap entries (reset by k_sort_big / k_sort_mid)
  uint32_t max_big;  // largest of them
  uint32_t pad;      // big-tile chunk dispenser (k_sort_big), zero between calls
  uint32_t num_huge;  // unfused path: tiles over kMidMax entries (k_sort_big's list; reset by it)
  uint32_t max_huge;  // largest of them
  uint32_t num_l2, num_l3;  // k_sort_mid_merge: tiles of 1025..2048 / 2049..8192 entries (reset by their consumers)
  uint32_t pad7;
  uint32_t pad4, pad5, pad6;
};

// Scan bookkeeping, zero on entry and left zero on exit (the last CTA to
// finish cleans up), so no memset is needed between calls.
struct ScanCtl {
  uint32_t ticket;  // CTA order of the look-back
  uint32_t done;    // CTAs finished
};

// Decoupled look-back scan (one pass over the counts): each CTA scans
// kScanTile counts, publishes its aggregate, and adds the prefix found by
// walking back over its predecessors' published values.  Two prefixes in one
// pass: entries (tile ranges) and big tiles (> kWarpSortCap entries), so the
// big-tile list is in raster order with no atomics, and so is the optional
// blend order (big tiles first, the others after them in reverse raster
// order: neighbouring warps blend neighbouring tiles).
// state[b] = flag << 62 | big << 32 | entries, flag 1 = aggregate, 2 = inclusive prefix.
// The counts are zeroed as they are consumed (ready for the next call).
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(
    int T, uint32_t* __restrict__ count, uint32_t* __restrict__ ranges,
    uint32_t* __restrict__ cursor, uint32_t* __restrict__ big_tiles,
    unsigned long long* state, ScanCtl* ctl, ViewScalars* sc, uint32_t* __restrict__ huge_tiles,
    uint32_t huge_min, uint32_t* __restrict__ order) {
  __shared__ uint32_t warp_tot[kScanThreads / 32], warp_big[kScanThreads / 32];
  __shared__ uint32_t s_prefix, s_bprefix, s_bid;
  if (threadIdx.x == 0) s_bid = atomicAdd(&ctl->ticket, 1u);
  __syncthreads();
  const uint32_t bid = s_bid;
  const int i0 = bid * kScanTile + threadIdx.x * kScanItems;
  uint32_t c[kScanItems];
  uint32_t sum = 0, nb = 0, mx = 0;
  if (i0 + kScanItems <= T) {
    uint4* p = reinterpret_cast<uint4*>(count + i0);
    const uint4 a = p[0], b = p[1];
    p[0] = make_uint4(0u, 0u, 0u, 0u);
    p[1] = make_uint4(0u, 0u, 0u, 0u);
    c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
    c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      c[k] = (i0 + k < T) ? count[i0 + k] : 0u;
      if (i0 + k < T) count[i0 + k] = 0u;
    }
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    sum += c[k];
    nb += c[k] > (uint32_t)kWarpSortCap ? 1u : 0u;
  }
  // block exclusive scans of the per-thread sums (entries, big tiles)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = sum, xb = nb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    const uint32_t yb = __shfl_up_sync(0xffffffffu, xb, o);
    if (lane >= o) {
      x += y;
      xb += yb;
    }
  }
  if (lane == 31) {
    warp_tot[wid] = x;
    warp_big[wid] = xb;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < kScanThreads / 32 ? warp_tot[lane] : 0u;
    uint32_t wb = lane < kScanThreads / 32 ? warp_big[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      const uint32_t yb = __shfl_up_sync(0xffffffffu, wb, o);
      if (lane >= o) {
        w += y;
        wb += yb;
      }
    }
    if (lane < kScanThreads / 32) {
      warp_tot[lane] = w;
      warp_big[lane] = wb;
    }
  }
  __syncthreads();
  const uint32_t excl = (wid ? warp_tot[wid - 1] : 0u) + x - sum;
  const uint32_t bexcl = (wid ? warp_big[wid - 1] : 0u) + xb - nb;
  const uint32_t agg = warp_tot[kScanThreads / 32 - 1];
  const uint32_t bagg = warp_big[kScanThreads / 32 - 1];
  if (wid == 0) {
    volatile unsigned long long* vs = state;
    const unsigned long long mine = ((unsigned long long)bagg << 32) | agg;
    if (bid == 0) {
      if (lane == 0) {
        vs[0] = (2ull << 62) | mine;
        s_prefix = 0;
        s_bprefix = 0;
      }
    } else {
      if (lane == 0) vs[bid] = (1ull << 62) | mine;
      // warp-parallel look-back: 32 predecessors per round (one L2 round trip
      // instead of one per predecessor)
      uint32_t prefix = 0, bprefix = 0;
      int b = (int)bid - 1;
      while (true) {
        const int idx = b - lane;
        const unsigned long long v = idx >= 0 ? vs[idx] : (2ull << 62);
        const uint32_t flag = (uint32_t)(v >> 62);
        const unsigned inc = __ballot_sync(0xffffffffu, flag == 2u);
        const unsigned zero = __ballot_sync(0xffffffffu, flag == 0u);
        const int first = inc ? __ffs(inc) - 1 : 32;  // nearest inclusive prefix
        const unsigned upto = first == 32 ? 0xffffffffu : ((2u << first) - 1u);
        if (zero & upto) continue;  // a predecessor before it has not published yet
        const bool take = ((1u << lane) & upto) != 0u;
        prefix += __reduce_add_sync(0xffffffffu, take ? (uint32_t)v : 0u);
        bprefix += __reduce_add_sync(0xffffffffu, take ? (uint32_t)(v >> 32) & 0x3FFFFFFFu : 0u);
        if (first < 32) break;
        b -= 32;
      }
      if (lane == 0) {
        __threadfence();
        vs[bid] = (2ull << 62) | ((unsigned long long)(bprefix + bagg) << 32) | (prefix + agg);
        s_prefix = prefix;
        s_bprefix = bprefix;
      }
    }
  }
  __syncthreads();
  uint32_t off = s_prefix + excl, bpos = s_bprefix + bexcl, mxh = 0u;
  const unsigned lt = (1u << lane) - 1u;
  // huge list (rare): one atomic per warp for all its items
  unsigned hm[kScanItems];
  uint32_t nhuge = 0u;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const bool huge = huge_tiles && i0 + k < T && c[k] > (uint32_t)kWarpSortCap && c[k] > huge_min;
    hm[k] = __ballot_sync(0xffffffffu, huge);
    nhuge += __popc(hm[k]);
  }
  uint32_t hb = 0u;
  if (lane == 0 && nhuge) hb = atomicAdd(&sc->num_huge, nhuge);
  hb = __shfl_sync(0xffffffffu, hb, 0);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int t = i0 + k;
    if (t < T) {
      ranges[t] = off;
      cursor[t] = off;
      if (c[k] > (uint32_t)kWarpSortCap) {
        big_tiles[bpos] = (uint32_t)t;
        if (order) order[bpos] = (uint32_t)t;
        mx = max(mx, c[k]);
        ++bpos;
      } else if (order) {
        order[T - 1 - ((uint32_t)t - bpos)] = (uint32_t)t;  // t - bpos small tiles precede t
      }
    }
    if ((hm[k] >> lane) & 1u) {
      huge_tiles[hb + __popc(hm[k] & lt)] = t;
      mxh = max(mxh, c[k]);
    }
    hb += __popc(hm[k]);
    off += c[k];
  }
  if (mx) atomicMax(&sc->max_big, mx);
  if (mxh) atomicMax(&sc->max_huge, mxh);
  if (i0 < T && i0 + kScanItems >= T) {  // the thread owning the last tile
    ranges[T] = off;
    sc->Ft = off;
    sc->num_big = bpos;  // all big tiles (the list's consumers reset it)
  }
  // the last CTA to finish leaves the look-back state zero for the next call
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

// ---------------------------------------------------------------- H5
template <int MODE>
__global__ void __launch_bounds__(kPointThreads) k_scatter(
    DevCfg g, const PointRec* __restrict__ rec, int64_t N, uint32_t* __restrict__ cursor,
    unsigned long long* __restrict__ entries, uint64_t cap, uint32_t* __restrict__ overflow) {
  const int64_t stride = (int64_t)gridDim.x * kPointThreads;
  const int64_t i0 = (int64_t)blockIdx.x * kPointThreads + threadIdx.x;
  float4 A[kPPT];
  float Rd[kPPT];
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    Rd[k] = 0.0f;
    if (i < N) {
      A[k] = __ldg(&rec[i].a);
      if (MODE == 1) Rd[k] = __ldg(&rec[i].b.w);
    }
  }
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    if (i >= N) break;
    Foot f;
    if (!rec_foot<MODE>(g, A[k], Rd[k], f)) continue;
    unsigned long long kv = ((unsigned long long)__float_as_uint(A[k].z) << 32) | (uint32_t)i;
    int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
    int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
    for (int ty = ty_lo; ty <= ty_hi; ++ty)
      for (int tx = tx_lo; tx <= tx_hi; ++tx) {
        uint32_t pos = atomicAdd(cursor + (size_t)ty * g.tiles_x + tx, 1u);
        if (pos < cap) entries[pos] = kv;
        else atomicOr(overflow, 1u);
      }
  }
}

// Bilinear H5 without atomics: entry k of point i goes to
// ranges[tile_k] + slot_k, the slot taken in k_project_count.
__global__ void __launch_bounds__(kPointThreads) k_scatter_slots(
    DevCfg g, const PointRec* __restrict__ rec, const uint4* __restrict__ slots, int64_t N,
    const uint32_t* __restrict__ ranges, unsigned long long* __restrict__ entries,
    const uint2* __restrict__ scat, const uint8_t* __restrict__ chunk_alive) {
  const int64_t stride = kPointThreads;  // CTA b: chunk b, as in k_project_count
  const int64_t i0 = (int64_t)blockIdx.x * kChunkPoints + threadIdx.x;
  if (chunk_alive && !chunk_alive[blockIdx.x]) return;
  if (scat) {  // 8 bytes per point (+ 16 per visible point) instead of the 32-byte record
    uint2 q[kPPT];
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
      int64_t i = i0 + k * stride;
      q[k] = i < N ? __ldg(scat + i) : make_uint2(0u, 0u);
    }
#pragma unroll
    for (int k = 0; k < kPPT; ++k) {
      int64_t i = i0 + k * stride;
      if (!q[k].x) continue;
      const uint4 s4 = __ldg(slots + i);
      const uint32_t sl[4] = {s4.x, s4.y, s4.z, s4.w};
      const unsigned long long kv = ((unsigned long long)q[k].x << 32) | (uint32_t)i;
      const uint32_t t0 = q[k].y & 0x0FFFFFFFu;
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if ((q[k].y >> (28 + c)) & 1u)
          entries[__ldg(ranges + t0 + (uint32_t)(c & 1) + (uint32_t)(c >> 1) * g.tiles_x) + sl[c]] = kv;
    }
    return;
  }
  float4 A[kPPT];
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    if (i < N) A[k] = __ldg(&rec[i].a);
  }
#pragma unroll
  for (int k = 0; k < kPPT; ++k) {
    int64_t i = i0 + k * stride;
    if (i >= N) break;
    Foot f;
    if (!rec_foot<0>(g, A[k], 0.0f, f)) continue;
    const uint4 s4 = __ldg(slots + i);
    const uint32_t sl[4] = {s4.x, s4.y, s4.z, s4.w};
    const unsigned long long kv = ((unsigned long long)__float_as_uint(A[k].z) << 32) | (uint32_t)i;
    const int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
    const int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int tx = tx_lo + (c & 1), ty = ty_lo + (c >> 1);
      if (tx <= tx_hi && ty <= ty_hi)
        entries[__ldg(ranges + (size_t)ty * g.tiles_x + tx) + sl[c]] = kv;
    }
  }
}

// ---------------------------------------------------------------- sort helpers
// Lanes of the warp whose BITS-bit digit equals this lane's, among the lanes
// with `valid` set (meaningful for valid lanes only): BITS + 1 ballots.
// Replaces __match_any_sync, whose throughput on sm_100a is about one
// instruction per 64 cycles per SM when the 32 values are distinct
// (tools/mb_match.cu: 2048 cycles per match per warp at 32 warps / SM).
template <int BITS>
__device__ __forceinline__ unsigned warp_peers(uint32_t d, bool valid) {
  unsigned peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
  for (int j = 0; j < BITS; ++j) {
    const bool bit = (d >> j) & 1u;
    const unsigned b = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? b : ~b;
  }
  return peers;
}

// 8-byte async global->shared copy (LDGSTS): a tile's keys are all in
// flight at once instead of one load latency per loop iteration.
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all8() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// In-place ascending bitonic sort of np (power of two) 64-bit keys in SMEM by
// the whole block.
__device__ __forceinline__ void block_bitonic(unsigned long long* s, int np) {
  for (int k = 2; k <= np; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
        int i = 2 * t - (t & (j - 1));  // i has bit j clear
        int ixj = i + j;
        unsigned long long a = s[i], b = s[ixj];
        bool up = (i & k) == 0;
        if ((a > b) == up) {
          s[i] = b;
          s[ixj] = a;
        }
      }
      __syncthreads();
    }
}

// Compare-exchange steps j = JMAX .. 1 (JMAX <= 32) of bitonic level k on
// the 64-element segment held by a warp in registers: element i = seg + 32 r
// + lane in v[r]; the direction uses the global index i.  Fully unrolled.
template <int JMAX, typename KT>
__device__ __forceinline__ void seg_bitonic_low(KT (&v)[2], int seg, int k, int lane) {
#pragma unroll
  for (int j = JMAX; j > 0; j >>= 1) {
    if (j == 32) {
      const bool up = ((seg + lane) & k) == 0;  // bit 5 clear for r = 0
      const KT a = v[0], b = v[1];
      const bool sw = (a > b) == up;
      v[0] = sw ? b : a;
      v[1] = sw ? a : b;
    } else {
      const bool lower = (lane & j) == 0;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const KT o = __shfl_xor_sync(0xffffffffu, v[r], j);
        const bool up = ((seg + r * 32 + lane) & k) == 0;
        v[r] = (lower == up) ? (o < v[r] ? o : v[r]) : (o > v[r] ? o : v[r]);
      }
    }
  }
}

// Block-wide ascending bitonic sort of np (power of two, >= 64) keys in
// SMEM with most steps in registers: every step with partner distance < 64
// runs on 64-key warp segments with shuffles, only the steps with distance
// >= 64 go through SMEM with block barriers (10 of 55 barriers at np = 1024).
template <typename KT>
__device__ __forceinline__ void block_bitonic_fast(KT* s, int np) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // levels k <= 64 entirely in registers
  for (int seg = wid * 64; seg < np; seg += nw * 64) {
    KT v[2] = {s[seg + lane], s[seg + 32 + lane]};
    seg_bitonic_low<1>(v, seg, 2, lane);
    seg_bitonic_low<2>(v, seg, 4, lane);
    seg_bitonic_low<4>(v, seg, 8, lane);
    seg_bitonic_low<8>(v, seg, 16, lane);
    seg_bitonic_low<16>(v, seg, 32, lane);
    seg_bitonic_low<32>(v, seg, 64, lane);
    s[seg + lane] = v[0];
    s[seg + 32 + lane] = v[1];
  }
  __syncthreads();
  for (int k = 128; k <= np; k <<= 1) {
    for (int j = k >> 1; j >= 64; j >>= 1) {
      for (int t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
        const int i = 2 * t - (t & (j - 1));
        const int ixj = i + j;
        const KT a = s[i], b = s[ixj];
        const bool up = (i & k) == 0;
        if ((a > b) == up) {
          s[i] = b;
          s[ixj] = a;
        }
      }
      __syncthreads();
    }
    for (int seg = wid * 64; seg < np; seg += nw * 64) {
      KT v[2] = {s[seg + lane], s[seg + 32 + lane]};
      seg_bitonic_low<32>(v, seg, k, lane);
      s[seg + lane] = v[0];
      s[seg + 32 + lane] = v[1];
    }
    __syncthreads();
  }
}

// Register bitonic sort of 32*K 64-bit keys held by a warp, element
// i = 32 r + lane in v[r]: partners at distance j < 32 are exchanged with
// shuffles, larger distances are register swaps.  Ascending.
template <int K>
__device__ __forceinline__ void reg_bitonic(unsigned long long (&v)[K], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if ((r & jr) == 0) {
            const int r2 = r | jr;
            const bool up = ((r * 32) & k) == 0;
            const unsigned long long a = v[r], b = v[r2];
            const bool sw = (a > b) == up;
            v[r] = sw ? b : a;
            v[r2] = sw ? a : b;
          }
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          const bool keep_min = lower == up;
          v[r] = keep_min ? (o < v[r] ? o : v[r]) : (o > v[r] ? o : v[r]);
        }
      }
    }
  }
}

template <int K>
__device__ __forceinline__ void warp_sort_k(unsigned long long* keys,
                                            const unsigned long long* __restrict__ src, int n,
                                            int lane) {
  unsigned long long v[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = r * 32 + lane;
    v[r] = i < n ? src[i] : ~0ull;
  }
  reg_bitonic<K>(v, lane);
#pragma unroll
  for (int r = 0; r < K; ++r) keys[r * 32 + lane] = v[r];
  __syncwarp();
}

// 32-bit register bitonic (same network as reg_bitonic, half the shuffles
// and compares of the 64-bit keys).
template <int K>
__device__ __forceinline__ void reg_bitonic32(uint32_t (&v)[K], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * K; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int jr = j >> 5;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if ((r & jr) == 0) {
            const int r2 = r | jr;
            const bool up = ((r * 32) & k) == 0;
            const uint32_t a = v[r], b = v[r2];
            const bool sw = (a > b) == up;
            v[r] = sw ? b : a;
            v[r2] = sw ? a : b;
          }
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, v[r], j);
          const bool up = ((r * 32 + lane) & k) == 0;
          v[r] = (lower == up) ? min(o, v[r]) : max(o, v[r]);
        }
      }
    }
  }
}

// Tile-list sort through 32-bit keys: (depth bits - tile minimum) shifted to
// 24 bits, then the 8-bit list slot.  That order equals the (depth, index)
// order unless two entries share a truncated depth; the result is checked
// for order on the full 64-bit keys and, if any adjacent pair is out of
// order, re-sorted with the 64-bit network (exactly the same result).
template <int K>
__device__ __forceinline__ void warp_sort_k32(unsigned long long* keys,
                                              const unsigned long long* __restrict__ src, int n,
                                              int lane) {
  unsigned long long f[K];
  uint32_t dmin = 0xFFFFFFFFu, dmax = 0u;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = r * 32 + lane;
    f[r] = i < n ? src[i] : ~0ull;
    if (i < n) {
      const uint32_t d = (uint32_t)(f[r] >> 32);
      dmin = min(dmin, d);
      dmax = max(dmax, d);
      keys[i] = f[r];
    }
  }
  dmin = __reduce_min_sync(0xffffffffu, dmin);
  dmax = __reduce_max_sync(0xffffffffu, dmax);
  const uint32_t range = dmax - dmin;
  const int shift = max(0, (32 - __clz(range)) - 24);
  uint32_t v[K];
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = r * 32 + lane;
    v[r] = i < n ? ((((uint32_t)(f[r] >> 32) - dmin) >> shift) << 8) | (uint32_t)i : 0xFFFFFFFFu;
  }
  reg_bitonic32<K>(v, lane);
  __syncwarp();
  bool bad = false;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const int i = r * 32 + lane;
    f[r] = i < n ? keys[v[r] & 255u] : ~0ull;
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {  // element i + 1 is lane + 1 of row r, or lane 0 of row r + 1
    unsigned long long nx = __shfl_down_sync(0xffffffffu, f[r], 1);
    const unsigned long long nr = __shfl_sync(0xffffffffu, f[r + 1 < K ? r + 1 : r], 0);
    if (lane == 31) nx = nr;
    const int i = r * 32 + lane;
    if (i + 1 < n && f[r] > nx) bad = true;
  }
  if (__any_sync(0xffffffffu, bad)) reg_bitonic<K>(f, lane);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < K; ++r) keys[r * 32 + lane] = f[r];
  __syncwarp();
}

// Warp-level sort of n <= kWarpSortCap unique 64-bit (depth key, index)
// keys read from src into keys[0..n) (SMEM), all in registers.
__device__ __forceinline__ void warp_sort(unsigned long long* keys,
                                          const unsigned long long* __restrict__ src, int n,
                                          int lane) {
  if (n <= 32) warp_sort_k32<1>(keys, src, n, lane);
  else if (n <= 64) warp_sort_k32<2>(keys, src, n, lane);
  else if (n <= 128) warp_sort_k32<4>(keys, src, n, lane);
  else warp_sort_k32<8>(keys, src, n, lane);
}

__device__ __forceinline__ uint32_t upper_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const unsigned long long* a, uint32_t n,
                                                    unsigned long long x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// H4+H6 for big tiles (more than kWarpSortCap entries): (0) block 0 builds
// the element / chunk prefixes of the big-tile list, (1) chunks of kBigChunk
// keys are sorted in SMEM, (2) runs are merged pairwise (rank by binary
// search; keys are unique), (3) the point indices go to sorted_idx.  Grid-
// synchronised between phases; returns at once if no tile is big.  Any
// block size <= kBigThreads; s holds kBigChunk keys.
#ifdef INPC_PHASE_TIMES  // diagnostics: %globaltimer at the phase boundaries of k_bin_bilinear
__device__ unsigned long long g_bin_ts[8];
#define BIN_TS(k)                                                                      \
  do {                                                                                 \
    if (threadIdx.x == 0) {                                                            \
      unsigned long long t_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                           \
      if (blockIdx.x == 0 && (k) < 4) g_bin_ts[k] = t_;                                \
      if ((k) >= 4) atomicMax(&g_bin_ts[k], t_);                                       \
    }                                                                                  \
  } while (0)
#else
#define BIN_TS(k) do { } while (0)
#endif

constexpr int kRadixItems = 8;
constexpr int kRadixMinN = 2048;  // smaller chunks: the bitonic network is cheaper than the passes
constexpr bool kUseRadix = true;  // chunks > kRadixMinN: radix (cfg 4: 1.15 ms vs 1.48 ms with 32-bit bitonic chunks)
constexpr int kRadixMaxRun = 64;
#ifndef INPC_SORT_BIG_MINB
#define INPC_SORT_BIG_MINB 2  // k_sort_big CTAs per SM (32 registers)
#endif
#ifndef INPC_BUCKET_MIN_N
#define INPC_BUCKET_MIN_N 1024  // smaller chunks: the 32-bit bitonic network is cheaper (cfg 5)
#endif
constexpr int kBucketMinN = INPC_BUCKET_MIN_N;  // k_sort_big chunks above this: bucket sort first
constexpr int kRadixStride = 257;  // hist row stride (digit-major scan reads are conflict-free)
constexpr int kRadixSmemU32 = 32 * kRadixStride + 32 + 4;
__device__ __forceinline__ bool block_radix_depth(unsigned long long* s, int n, uint32_t* sm);
template <int BITS>
__device__ __forceinline__ bool block_bucket_sort(unsigned long long* s, int n, uint32_t* sm);
__device__ __forceinline__ bool block_sort32_depth(const unsigned long long* s, int n, int np, uint32_t* u,
                                                   uint32_t* misc);

template <int CHUNK>
__device__ __forceinline__ void big_sort_body(
    cooperative_groups::grid_group& grid, unsigned long long* s, uint32_t* carry,
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ big_tiles, uint32_t* list_count,
    uint32_t* list_max, uint32_t* big_elem, uint32_t* big_chunk, ViewScalars* sc, unsigned long long* entries,
    unsigned long long* tmp, uint32_t* __restrict__ sorted_idx, uint32_t* radix_smem = nullptr,
    uint32_t min_n = (uint32_t)kWarpSortCap) {
  // tiles of the big-tile list with at most min_n entries were sorted by
  // k_sort_mid: they get no chunks here
  const uint32_t nb = *(volatile uint32_t*)list_count;
  if (nb == 0) return;
  if (blockIdx.x == 0) {
    // exclusive prefixes over the big-tile list (its order is arbitrary; it
    // only decides which CTA works on what): chunks of every big tile, and
    // elements of the tiles that need merging (more than one chunk)
    uint32_t* wsum = reinterpret_cast<uint32_t*>(s);  // [2][32] warp totals
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) carry[0] = carry[1] = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nb; b0 += blockDim.x) {
      const uint32_t j = b0 + threadIdx.x;
      uint32_t sz = 0, ch = 0;
      if (j < nb) {
        const uint32_t t = big_tiles[j];
        const uint32_t n = ranges[t + 1] - ranges[t];
        ch = n > min_n ? (n + CHUNK - 1) / CHUNK : 0u;
        sz = ch > 1 ? n : 0u;
      }
      uint32_t xs = sz, xc = ch;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ys = __shfl_up_sync(0xffffffffu, xs, o), yc = __shfl_up_sync(0xffffffffu, xc, o);
        if (lane >= o) { xs += ys; xc += yc; }
      }
      if (lane == 31) { wsum[wid] = xs; wsum[32 + wid] = xc; }
      __syncthreads();
      uint32_t ps = carry[0], pc = carry[1];
      for (int w = 0; w < wid; ++w) { ps += wsum[w]; pc += wsum[32 + w]; }
      if (j < nb) {
        big_elem[j] = ps + xs - sz;
        big_chunk[j] = pc + xc - ch;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 0; w < nw; ++w) { carry[0] += wsum[w]; carry[1] += wsum[32 + w]; }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      big_elem[nb] = carry[0];
      big_chunk[nb] = carry[1];
    }
    __syncthreads();
  }
  grid.sync();
  BIN_TS(4);
  const uint32_t total_chunks = big_chunk[nb], total = big_elem[nb], maxn = *list_max;
  if (total_chunks == 0u) {  // every listed tile was sorted by k_sort_mid (grid-uniform)
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // all CTAs read the count before the sync above
      *list_count = 0u;
      *list_max = 0u;
      sc->pad = 0u;
    }
    return;
  }
  // chunks handed out dynamically (sizes vary by tile): carry[0] is this CTA's next chunk
  // (thread 0 draws the chunk and finds its tile: carry = {chunk, list slot})
  if (threadIdx.x == 0) {
    carry[0] = atomicAdd(&sc->pad, 1u);
    carry[1] = carry[0] < total_chunks ? upper_bound_u32(big_chunk, nb, carry[0]) - 1 : 0u;
  }
  __syncthreads();
  for (uint32_t gch = carry[0]; gch < total_chunks;) {
    const uint32_t j = carry[1];
    const uint32_t t = big_tiles[j];
    const uint32_t c = gch - big_chunk[j];
    const uint32_t tn = ranges[t + 1] - ranges[t];
    const uint32_t begin = ranges[t] + c * CHUNK;
    const uint32_t n = min((uint32_t)CHUNK, ranges[t + 1] - begin);
    int np = 64;  // sort network of the next power of two, not the full chunk
    while (np < (int)n) np <<= 1;
    bool sorted = false, perm = false;
    uint32_t* u = radix_smem;                                  // 32-bit keys / permutation
    uint32_t* misc = radix_smem ? radix_smem + 32 * kRadixStride + 32 : nullptr;
    if (radix_smem && n > (uint32_t)kBucketMinN) {
      for (int k = threadIdx.x; k < (int)n; k += blockDim.x) cp_async8(&s[k], entries + begin + k);
      cp_async_wait_all8();
      __syncthreads();
      // about 4 buckets per key
      sorted = n > 2048u ? block_bucket_sort<14>(s, (int)n, radix_smem) : block_bucket_sort<13>(s, (int)n, radix_smem);
      if (!sorted && kUseRadix && n > (uint32_t)kRadixMinN) sorted = block_radix_depth(s, (int)n, radix_smem);
    } else if (radix_smem) {
      for (int k = threadIdx.x; k < (int)n; k += blockDim.x) cp_async8(&s[k], entries + begin + k);
      cp_async_wait_all8();
      __syncthreads();
      sorted = perm = block_sort32_depth(s, (int)n, np, u, misc);
    }
    if (!sorted) {
      if (radix_smem) {
        for (int k = (int)n + threadIdx.x; k < np; k += blockDim.x) s[k] = ~0ull;
      } else {
        for (int k = threadIdx.x; k < np; k += blockDim.x) s[k] = k < (int)n ? entries[begin + k] : ~0ull;
      }
      __syncthreads();
      block_bitonic_fast(s, np);
    }
    const uint32_t pm = (uint32_t)np - 1u;
    if (tn <= (uint32_t)CHUNK) {  // one chunk = the whole tile: final order
      for (int k = threadIdx.x; k < (int)n; k += blockDim.x)
        sorted_idx[begin + k] = (uint32_t)s[perm ? (u[k] & pm) : k];
    } else {
      for (int k = threadIdx.x; k < (int)n; k += blockDim.x) entries[begin + k] = s[perm ? (u[k] & pm) : k];
    }
    if (threadIdx.x == 0) {
      carry[0] = atomicAdd(&sc->pad, 1u);
      carry[1] = carry[0] < total_chunks ? upper_bound_u32(big_chunk, nb, carry[0]) - 1 : 0u;
    }
    __syncthreads();
    gch = carry[0];
  }
  BIN_TS(5);
  if (total > 0) {  // tiles over one chunk: pairwise merges of the sorted runs
    grid.sync();
    unsigned long long* src = entries;
    unsigned long long* dst = tmp;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t L = CHUNK; L < maxn; L <<= 1) {
      for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
        uint32_t j = upper_bound_u32(big_elem, nb, e) - 1;
        while (j + 1 < nb && big_elem[j + 1] == big_elem[j]) ++j;  // skip single-chunk tiles
        uint32_t t = big_tiles[j];
        uint32_t begin = ranges[t], n = ranges[t + 1] - begin;
        uint32_t pos = e - big_elem[j];
        uint32_t r = pos / L, run0 = r * L, p0 = (r ^ 1u) * L;
        unsigned long long key = src[begin + pos];
        uint32_t out = pos;
        if (p0 < n) {
          uint32_t p1 = min(p0 + L, n);
          uint32_t rank = lower_bound_u64(src + begin + p0, p1 - p0, key);
          out = min(run0, p0) + (pos - run0) + rank;
        }
        dst[begin + out] = key;
      }
      grid.sync();
      unsigned long long* sw = src;
      src = dst;
      dst = sw;
    }
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      uint32_t j = upper_bound_u32(big_elem, nb, e) - 1;
      while (j + 1 < nb && big_elem[j + 1] == big_elem[j]) ++j;
      uint32_t begin = ranges[big_tiles[j]];
      uint32_t pos = e - big_elem[j];
      sorted_idx[begin + pos] = (uint32_t)src[begin + pos];
    }
  }
  grid.sync();  // everybody has read the big-tile counters: zero them for the next call
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *list_count = 0u;
    *list_max = 0u;
    sc->pad = 0u;
  }
}

// CTA bucket sort of n <= 8192 unique 64-bit keys (depth bits << 32 | point
// index) in SMEM, 1024 threads: one counting pass on the 14 most significant
// depth bits that vary in the chunk (16384 buckets, two 16-bit counters per
// SMEM word; SMEM atomics, so the order inside a bucket is arbitrary), then
// every bucket is insertion-sorted on the full key by one thread (measured
// on cfg 4, chunks of 2-7k keys: 12 bits 1.38 ms, 13 bits 0.76 ms, against
// 1.14 ms for three radix passes -- the insertion chains of the largest
// buckets set the time).  The keys are unique, so no stability is needed.
// One pass instead of three radix passes.  Returns false, s holding the same
// keys in some order, when the depths do not vary or a bucket holds more than
// kBucketMax keys: the caller then runs the radix sort.
constexpr int kBigChunkLarge = 8192;
constexpr int kBigThreadsLarge = 1024;
constexpr int kBucketBits = 14;
constexpr int kBuckets = 1 << kBucketBits;
constexpr int kBucketMax = 64;
static_assert(kBuckets / 2 + 36 <= kRadixSmemU32, "bucket sort scratch");
static_assert(kBigChunkLarge < 65536, "16-bit bucket counters");

template <int BITS>
__device__ __forceinline__ bool block_bucket_sort(unsigned long long* s, int n, uint32_t* sm) {
  // pos: bucket b's 16-bit counter / offset / cursor is half (b & 1) of word b >> 1
  uint32_t* pos = sm;                      // [kBuckets / 2]
  uint32_t* misc = sm + kBuckets / 2;      // [0] OR, [1] AND, [2] fail flag, [4..35] warp sums
  auto half = [](uint32_t word, uint32_t b) { return (b & 1u) ? word >> 16 : word & 0xFFFFu; };
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int kItems = kBigChunkLarge / kBigThreadsLarge;
  constexpr int kPer = (1 << BITS) / kBigThreadsLarge;  // buckets per thread in the scan
  uint32_t o = 0u, a = 0xFFFFFFFFu;
  for (int i = tid; i < n; i += kBigThreadsLarge) {
    const uint32_t d = (uint32_t)(s[i] >> 32);
    o |= d;
    a &= d;
  }
  static_assert(BITS >= 11 && BITS <= kBucketBits, "bucket bits");
  constexpr int bits = BITS, nbk = 1 << BITS, per = nbk / kBigThreadsLarge;
  for (int b = tid; b < nbk / 2; b += kBigThreadsLarge) pos[b] = 0u;
  if (tid == 0) {
    misc[0] = 0u;
    misc[1] = 0xFFFFFFFFu;
    misc[2] = 0u;
  }
  __syncthreads();
  o = __reduce_or_sync(0xffffffffu, o);
  a = __reduce_and_sync(0xffffffffu, a);
  if (lane == 0) {
    atomicOr(&misc[0], o);
    atomicAnd(&misc[1], a);
  }
  __syncthreads();
  const uint32_t vary = misc[0] ^ misc[1];
  if (vary == 0u) return false;  // one depth: index order only (radix run fix-up / bitonic)
  const int hi = 31 - __clz(vary);
  const int sh = hi >= bits - 1 ? hi - (bits - 1) : 0;  // bits above hi are equal
  auto digit = [&](unsigned long long k) { return (uint32_t)(k >> (32 + sh)) & (uint32_t)(nbk - 1); };
  unsigned long long kv[kItems];  // the chunk's keys, held across the count and the scatter
#pragma unroll
  for (int r = 0; r < kItems; ++r) {
    const int i = r * kBigThreadsLarge + tid;
    kv[r] = i < n ? s[i] : 0ull;
    if (i < n) {
      const uint32_t d = digit(kv[r]);
      atomicAdd(&pos[d >> 1], (d & 1u) ? 0x10000u : 1u);
    }
  }
  __syncthreads();
  {  // exclusive scan of the counts: thread t owns buckets per t .. per t + per - 1
    uint32_t c[kPer], sum = 0u;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t b = per * tid + k;
      c[k] = k < per ? half(pos[b >> 1], b) : 0u;
      sum += c[k];
    }
    uint32_t x = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) misc[4 + w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t v = misc[4 + lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
        if (lane >= off) v += y;
      }
      misc[4 + lane] = v;
    }
    __syncthreads();
    uint32_t run = (w ? misc[4 + w - 1] : 0u) + x - sum;
#pragma unroll
    for (int k = 0; k < kPer; k += 2) {  // per even: whole words per thread
      if (k < per) pos[(per * tid + k) >> 1] = run | ((run + c[k]) << 16);
      run += c[k] + c[k + 1];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; ++r)
    if (r * kBigThreadsLarge + tid < n) {
      const uint32_t d = digit(kv[r]);
      s[half(atomicAdd(&pos[d >> 1], (d & 1u) ? 0x10000u : 1u), d)] = kv[r];
    }
  __syncthreads();
  // pos[b] is now the end of bucket b, pos[b - 1] its start
  bool bad = false;
  for (int b = tid; b < nbk; b += kBigThreadsLarge) {
    const int lo = b ? (int)half(pos[(b - 1) >> 1], b - 1) : 0, hi2 = (int)half(pos[b >> 1], b);
    if (hi2 - lo > kBucketMax) {
      bad = true;
      continue;
    }
    for (int k = lo + 1; k < hi2; ++k) {
      const unsigned long long v = s[k];
      int j = k - 1;
      while (j >= lo && s[j] > v) {
        s[j + 1] = s[j];
        --j;
      }
      s[j + 1] = v;
    }
  }
  if (bad) misc[2] = 1u;
  __syncthreads();
  return misc[2] == 0u;
}

// CTA radix sort of n <= 1024 * kRadixItems 64-bit keys (depth bits << 32 |
// point index) in SMEM, for k_sort_big (1024 threads).  LSD passes of 8-bit
// digits over the depth bits that vary in this chunk only (a tile's depths
// share exponent and leading mantissa bits: 3 passes on cfg 4), each pass
// stable: warp w owns elements [32 E w, 32 E (w+1)) in rounds of 32, lanes
// with the same digit rank themselves (warp_peers ballots), per-(digit,
// warp) counts are scanned digit-major.  The keys of a pass sit in
// registers, so the scatter goes back into s in place.  Stability keeps equal
// depths in input order; runs of equal depth are then put in index order by
// one thread each (insertion sort).  Returns false (s unchanged in content,
// order undefined) when a run is longer than kRadixMaxRun: the caller then
// sorts the chunk with the 64-bit bitonic network.

__device__ __forceinline__ bool block_radix_depth(unsigned long long* s, int n, uint32_t* sm) {
  uint32_t* hist = sm;                       // [32 warps][kRadixStride]
  uint32_t* wsum = sm + 32 * kRadixStride;   // [32]
  uint32_t* misc = wsum + 32;                // [0] OR, [1] AND, [2] long-run flag
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int E = (n + 1023) >> 10;
  const int wbase = w * 32 * E;
  unsigned long long kv[kRadixItems];
  uint32_t o = 0u, a = 0xFFFFFFFFu;
#pragma unroll
  for (int r = 0; r < kRadixItems; ++r) {
    const int i = wbase + r * 32 + lane;
    kv[r] = 0ull;
    if (r < E && i < n) {
      kv[r] = s[i];
      const uint32_t d = (uint32_t)(kv[r] >> 32);
      o |= d;
      a &= d;
    }
  }
  if (threadIdx.x == 0) {
    misc[0] = 0u;
    misc[1] = 0xFFFFFFFFu;
    misc[2] = 0u;
  }
  __syncthreads();
  o = __reduce_or_sync(0xffffffffu, o);
  a = __reduce_and_sync(0xffffffffu, a);
  if (lane == 0) {
    atomicOr(&misc[0], o);
    atomicAnd(&misc[1], a);
  }
  __syncthreads();
  const uint32_t vary = misc[0] ^ misc[1];
  if (vary) {
    const int lo = __ffs(vary) - 1, hi = 31 - __clz(vary);
    for (int sh = lo; sh <= hi; sh += 8) {
      uint32_t rank[kRadixItems];
      for (int d = lane; d < 256; d += 32) hist[w * kRadixStride + d] = 0u;
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        if (r >= E) break;
        const int i = wbase + r * 32 + lane;
        const bool valid = i < n;
        const uint32_t d = (uint32_t)(kv[r] >> (32 + sh)) & 255u;
        const unsigned peers = warp_peers<8>(d, valid);
        const int leader = __ffs(peers) - 1;
        uint32_t cnt = 0;  // the leader advances the warp's counter of d; SMEM atomics keep rounds in order
        if (valid && lane == leader) cnt = atomicAdd(&hist[w * kRadixStride + d], (uint32_t)__popc(peers));
        cnt = __shfl_sync(0xffffffffu, cnt, leader);
        rank[r] = cnt + __popc(peers & lt);
      }
      __syncthreads();
      {  // exclusive scan of the counts in (digit, warp) order: thread t = 4 d + q owns warps 8q..8q+7
        const int d = threadIdx.x >> 2, q = threadIdx.x & 3;
        uint32_t c[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          c[k] = hist[(8 * q + k) * kRadixStride + d];
          sum += c[k];
        }
        uint32_t x = sum;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
          if (lane >= off) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
          uint32_t v = wsum[lane];
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, v, off);
            if (lane >= off) v += y;
          }
          wsum[lane] = v;
        }
        __syncthreads();
        uint32_t run = (w ? wsum[w - 1] : 0u) + x - sum;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          hist[(8 * q + k) * kRadixStride + d] = run;
          run += c[k];
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        if (r >= E) break;
        const int i = wbase + r * 32 + lane;
        if (i < n) s[hist[w * kRadixStride + ((uint32_t)(kv[r] >> (32 + sh)) & 255u)] + rank[r]] = kv[r];
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kRadixItems; ++r) {
        if (r >= E) break;
        const int i = wbase + r * 32 + lane;
        if (i < n) kv[r] = s[i];
      }
    }
  }
  // equal depths: index order within each run (runs are short; long ones fall back)
  for (int p = threadIdx.x; p + 1 < n; p += blockDim.x) {
    const uint32_t dp = (uint32_t)(s[p] >> 32);
    if ((uint32_t)(s[p + 1] >> 32) != dp || (p > 0 && (uint32_t)(s[p - 1] >> 32) == dp)) continue;
    int end = p + 2;
    while (end < n && (uint32_t)(s[end] >> 32) == dp && end - p <= kRadixMaxRun) ++end;
    if (end - p > kRadixMaxRun) {
      misc[2] = 1u;
      continue;
    }
    for (int k = p + 1; k < end; ++k) {
      const unsigned long long v = s[k];
      int j = k - 1;
      while (j >= p && s[j] > v) {
        s[j + 1] = s[j];
        --j;
      }
      s[j + 1] = v;
    }
  }
  __syncthreads();
  return misc[2] == 0u;
}

// Chunk sort through 32-bit keys for k_sort_big: u[k] = (depth bits - chunk
// minimum) shifted into 32 - log2(np) bits, then the slot k.  The sorted u
// is a permutation of s (s itself is not moved).  Equal truncated depths may
// leave neighbours out of (depth, index) order: up to four odd-even
// transposition passes over u, comparing the full keys s[slot], repair that;
// returns false if the chunk is still unsorted (the caller then runs the
// 64-bit network on s).
__device__ __forceinline__ bool block_sort32_depth(const unsigned long long* s, int n, int np, uint32_t* u,
                                                   uint32_t* misc) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const uint32_t d = (uint32_t)(s[k] >> 32);
    lo = min(lo, d);
    hi = max(hi, d);
  }
  if (threadIdx.x == 0) {
    misc[0] = 0xFFFFFFFFu;
    misc[1] = 0u;
  }
  __syncthreads();
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) {
    atomicMin(&misc[0], lo);
    atomicMax(&misc[1], hi);
  }
  __syncthreads();
  const uint32_t dmin = misc[0], range = misc[1] - dmin;
  const int sb = __ffs(np) - 1;
  const uint32_t mask = (uint32_t)np - 1u;
  const int shift = max(0, (32 - __clz(range)) - (32 - sb));
  for (int k = threadIdx.x; k < np; k += blockDim.x)
    u[k] = k < n ? ((((uint32_t)(s[k] >> 32) - dmin) >> shift) << sb) | (uint32_t)k : 0xFFFFFFFFu;
  __syncthreads();
  block_bitonic_fast<uint32_t>(u, np);
  for (int pass = 0; pass < 4; ++pass) {
    int sw = 0;
    for (int ph = 0; ph < 2; ++ph) {
      for (int k = 2 * threadIdx.x + ph; k + 1 < n; k += 2 * blockDim.x) {
        const uint32_t a = u[k], b = u[k + 1];
        if ((a >> sb) == (b >> sb) && s[a & mask] > s[b & mask]) {
          u[k] = b;
          u[k + 1] = a;
          sw = 1;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(sw)) return true;
  }
  return false;
}

// Stand-alone big-tile sort: 1024 threads, chunks of kBigChunkLarge keys in
// 64 KB of dynamic SMEM (+ the radix counters), so tiles up to 8192 entries
// (cfg 4: 7750 tiles of 2-7k entries) sort in one chunk without merge passes;
// chunks are sorted by block_radix_depth (bitonic fallback on long ties).
__global__ void __launch_bounds__(kBigThreadsLarge, INPC_SORT_BIG_MINB) k_sort_big(
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ big_tiles,
    uint32_t* big_elem, uint32_t* big_chunk, ViewScalars* sc,
    unsigned long long* entries, unsigned long long* tmp, uint32_t* __restrict__ sorted_idx, uint32_t min_n,
    const uint32_t* __restrict__ huge_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t carry[2];
  unsigned long long* s = reinterpret_cast<unsigned long long*>(smem_raw);
  uint32_t* rs = reinterpret_cast<uint32_t*>(s + kBigChunkLarge);
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  // huge list (tiles over kMidMax, the rest went through k_sort_mid) or, with
  // min_n == kWarpSortCap (A/B without k_sort_mid), the whole big-tile list
  const bool huge = min_n > (uint32_t)kWarpSortCap;
  big_sort_body<kBigChunkLarge>(grid, s, carry, ranges, huge ? huge_tiles : big_tiles,
                                huge ? &sc->num_huge : &sc->num_big, huge ? &sc->max_huge : &sc->max_big,
                                big_elem, big_chunk, sc, entries, tmp, sorted_idx, rs, min_n);
}

// ---------------------------------------------------------------- H4+H6 mid tiles
// Tiles of kWarpSortCap + 1 .. kMidMax entries -- the common big tile of the
// dense clouds (cfg 5: ~800 entries) -- without the chunk
// machinery of k_sort_big: one CTA of kMidThreads per tile, the tile's
// unique 64-bit keys in SMEM, ordered through 32-bit keys
//   k32 = ((depth bits - tile minimum) >> shift) << slot bits | slot,
// the depth part quantised to the kDepthBits most significant varying bits,
// by a stable LSD radix sort of 4-bit digits over those bits only.
// Ranking without a serial counter chain: the keys are taken in rounds of 32
// (round R = keys [32R, 32R + 32) of the current order); in a round each
// lane finds the lanes with its digit by 4 + 1 ballots (warp_peers), the
// lowest of them stores the round's count in cnt[digit][R] and every lane
// keeps its rank inside the round; one exclusive scan of cnt in (digit,
// round) order then gives every (digit, round) its output base -- stable,
// and every round independent of the others (the __match_any_sync /
// per-warp-counter variants measured 2-3x slower: MATCH.ANY costs ~2 SM
// cycles per distinct value, and a leader's load-add-store chain per round
// serialises the rounds).  Equal quantised depths stay in slot order; one
// thread per such run then insertion-sorts it on the full (depth, index)
// key, so the result is the (depth, index) order bit for bit.  A run longer
// than kMaxRun (many equal depths) falls back to the 64-bit bitonic network.
#ifdef INPC_PHASE_TIMES  // diagnostics: clock64 cycles per phase of the mid-tile CTA sort (thread 0)
__device__ unsigned long long g_mid_cyc[8];
#define MID_T(k)                            \
  do {                                      \
    if (prof && threadIdx.x == 0) {         \
      const long long t_ = clock64();       \
      prof[k] += (unsigned long long)(t_ - tp_); \
      tp_ = t_;                             \
    }                                       \
  } while (0)
#else
#define MID_T(k) do { } while (0)
#endif

template <int NT, int MAXN>
struct MidSort {
  static constexpr int kWarps = NT / 32;
  static constexpr int kItems = MAXN / NT;         // keys (rounds) per thread
  static constexpr int kRounds = MAXN / 32;        // rounds of 32 keys
  static constexpr int kSlotBits = MAXN == 2048 ? 11 : MAXN == 4096 ? 12 : 13;
  static constexpr int kDepthBits = 20;            // quantised depth bits in the key
  static constexpr int kDigitBits = 4;
  static constexpr int kDigits = 1 << kDigitBits;
  static constexpr int kCnt = kDigits * kRounds;   // [digit][round]
  static constexpr int kCntPerThread = kCnt / NT;
  static constexpr int kMaxRun = 64;
  static_assert(MAXN == (1 << kSlotBits) && kDepthBits + kSlotBits <= 32, "key layout");
  static_assert(kCnt % NT == 0 && kCntPerThread % 4 == 0, "counter layout");
  struct Smem {
    unsigned long long s[MAXN];  // full keys, slot order (bitonic fallback: sorted in place)
    uint32_t k32[MAXN];          // scatter buffer, finally the sorted 32-bit keys
    __align__(16) uint32_t cnt[kCnt];
    uint32_t wsum[kWarps];
    uint32_t red[2][kWarps];
  };
};
constexpr int kMidThreads = 128;
constexpr int kMidMax = 2048;
constexpr int kMergeMax = 8192;
#ifndef INPC_MID_NT1
#define INPC_MID_NT1 64
#endif
#ifndef INPC_MID_NT2
#define INPC_MID_NT2 128
#endif
constexpr int kMidNT1 = INPC_MID_NT1;  // merge-sort threads per tile of <= 1024 entries
constexpr int kMidNT2 = INPC_MID_NT2;  // ... of <= 2048 entries  // k_sort_mid_merge's largest tiles; k_sort_big takes the rest
using MidCfg = MidSort<kMidThreads, kMidMax>;

// Sort the n keys of S.s (slot order); returns true with S.k32 holding the
// sorted 32-bit keys (slot = k32 & (MAXN - 1)), false with S.s itself sorted
// (bitonic fallback).  Block-uniform result.
template <int NT, int MAXN>
__device__ __forceinline__ bool block_radix32(typename MidSort<NT, MAXN>::Smem& S, int n,
                                              unsigned long long* prof = nullptr) {
  using M = MidSort<NT, MAXN>;
#ifdef INPC_PHASE_TIMES
  long long tp_ = clock64();
#endif
  (void)prof;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  for (int k = tid; k < n; k += NT) {
    const uint32_t d = (uint32_t)(S.s[k] >> 32);
    lo = min(lo, d);
    hi = max(hi, d);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lane == 0) {
    S.red[0][w] = lo;
    S.red[1][w] = hi;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < M::kWarps; ++q) {
    lo = min(lo, S.red[0][q]);
    hi = max(hi, S.red[1][q]);
  }
  const uint32_t range = hi - lo;
  const int vbits = range ? 32 - __clz(range) : 0;
  const int shift = vbits > M::kDepthBits ? vbits - M::kDepthBits : 0;
  const int npass = (vbits - shift + M::kDigitBits - 1) / M::kDigitBits;
  MID_T(2);
  // warp w owns rounds R = w * E + r (keys 32 R + lane), r < E
  const int nr = (n + 31) >> 5;
  const int E = (nr + M::kWarps - 1) / M::kWarps;
  uint32_t kv[M::kItems], rk[M::kItems];
#pragma unroll
  for (int r = 0; r < M::kItems; ++r) {
    const int i = (w * E + r) * 32 + lane;
    kv[r] = (r < E && i < n) ? ((((uint32_t)(S.s[i] >> 32) - lo) >> shift) << M::kSlotBits) | (uint32_t)i : 0u;
  }
  if (npass == 0) {  // one depth: slot order, fixed below
#pragma unroll
    for (int r = 0; r < M::kItems; ++r) {
      const int i = (w * E + r) * 32 + lane;
      if (r < E && i < n) S.k32[i] = kv[r];
    }
  }
  constexpr int Q = M::kCntPerThread / 4;
  for (int p = 0; p < npass; ++p) {
    const int sh = M::kSlotBits + M::kDigitBits * p;
#pragma unroll
    for (int q = 0; q < Q; ++q) reinterpret_cast<uint4*>(S.cnt)[tid * Q + q] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < M::kItems; ++r) {
      if (r >= E) break;
      const int R = w * E + r;
      const bool valid = R * 32 + lane < n;
      const uint32_t d = (kv[r] >> sh) & (uint32_t)(M::kDigits - 1);
      const unsigned peers = warp_peers<M::kDigitBits>(d, valid);
      if (valid && (peers & lt) == 0u) S.cnt[d * M::kRounds + R] = (uint32_t)__popc(peers);
      rk[r] = (uint32_t)__popc(peers & lt);
    }
    __syncthreads();
    {  // exclusive scan of the counters in (digit, round) order
      uint32_t c[M::kCntPerThread], sum = 0u;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const uint4 v = reinterpret_cast<const uint4*>(S.cnt)[tid * Q + q];
        c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int q = 0; q < M::kCntPerThread; ++q) sum += c[q];
      uint32_t x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) S.wsum[w] = x;
      __syncthreads();
      uint32_t run = x - sum;
#pragma unroll
      for (int q = 0; q < M::kWarps; ++q) run += q < w ? S.wsum[q] : 0u;
#pragma unroll
      for (int q = 0; q < M::kCntPerThread; ++q) {
        const uint32_t cq = c[q];
        c[q] = run;
        run += cq;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)
        reinterpret_cast<uint4*>(S.cnt)[tid * Q + q] = make_uint4(c[4 * q], c[4 * q + 1], c[4 * q + 2], c[4 * q + 3]);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < M::kItems; ++r) {
      if (r >= E) break;
      const int R = w * E + r;
      if (R * 32 + lane < n)
        S.k32[S.cnt[((kv[r] >> sh) & (uint32_t)(M::kDigits - 1)) * M::kRounds + R] + rk[r]] = kv[r];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < M::kItems; ++r) {
      if (r >= E) break;
      const int i = (w * E + r) * 32 + lane;
      if (i < n) kv[r] = S.k32[i];
    }
  }
  __syncthreads();
  MID_T(3);
  // runs of equal quantised depth: (depth, index) order on the full keys
  constexpr uint32_t smask = (uint32_t)MAXN - 1u;
  bool bad = false;
  for (int p = tid; p + 1 < n; p += NT) {
    const uint32_t a = S.k32[p] >> M::kSlotBits;
    if ((S.k32[p + 1] >> M::kSlotBits) != a || (p > 0 && (S.k32[p - 1] >> M::kSlotBits) == a)) continue;
    int end = p + 2;
    while (end < n && (S.k32[end] >> M::kSlotBits) == a && end - p <= M::kMaxRun) ++end;
    if (end - p > M::kMaxRun) {
      bad = true;
      continue;
    }
    for (int k = p + 1; k < end; ++k) {
      const uint32_t v = S.k32[k];
      const unsigned long long fv = S.s[v & smask];
      int j = k - 1;
      while (j >= p && S.s[S.k32[j] & smask] > fv) {
        S.k32[j + 1] = S.k32[j];
        --j;
      }
      S.k32[j + 1] = v;
    }
  }
  if (__syncthreads_or(bad)) {
    int np = 64;
    while (np < n) np <<= 1;
    for (int k = n + tid; k < np; k += NT) S.s[k] = ~0ull;
    __syncthreads();
    block_bitonic_fast(S.s, np);
    MID_T(4);
    return false;
  }
  MID_T(4);
  return true;
}

// The mid tiles (kWarpSortCap < n <= kMidMax; larger ones are left to
// k_sort_big), one CTA per tile (block_radix32), grid-stride over the
// big-tile list.  Its last CTA zeroes the list count for the next call.
// (A one-warp-per-tile variant with the same ranking measured 16.6 vs
// 13.4 ms per cfg 5 step: fewer tiles in flight did not pay for the
// barriers saved.)
__global__ void __launch_bounds__(kMidThreads) k_sort_mid(const uint32_t* __restrict__ ranges,
                                                              const uint32_t* __restrict__ big_tiles,
                                                              ViewScalars* __restrict__ sc,
                                                              const unsigned long long* __restrict__ entries,
                                                              uint32_t* __restrict__ sorted_idx,
                                                              uint32_t* __restrict__ done) {
  __shared__ MidCfg::Smem S;
  __shared__ uint32_t s_last;
  const uint32_t nb = sc->num_big;
#ifdef INPC_PHASE_TIMES
  unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tp_ = clock64();
#else
  unsigned long long* prof = nullptr;
#endif
  for (uint32_t j = blockIdx.x; j < nb; j += gridDim.x) {
    const uint32_t t = big_tiles[j];
    const uint32_t begin = ranges[t], n = ranges[t + 1] - begin;
    if (n > (uint32_t)kMidMax) continue;  // block-uniform
    MID_T(0);
    for (int k = threadIdx.x; k < (int)n; k += kMidThreads) cp_async8(&S.s[k], entries + begin + k);
    cp_async_wait_all8();
    __syncthreads();
    MID_T(1);
#ifdef INPC_PHASE_TIMES
    const bool ok = block_radix32<kMidThreads, kMidMax>(S, (int)n, prof);
    tp_ = clock64();
#else
    const bool ok = block_radix32<kMidThreads, kMidMax>(S, (int)n);
#endif
    if (ok) {
      for (int k = threadIdx.x; k < (int)n; k += kMidThreads)
        sorted_idx[begin + k] = (uint32_t)S.s[S.k32[k] & (uint32_t)(kMidMax - 1)];
    } else {
      for (int k = threadIdx.x; k < (int)n; k += kMidThreads) sorted_idx[begin + k] = (uint32_t)S.s[k];
    }
    __syncthreads();
    MID_T(5);
    if (prof && threadIdx.x == 0) prof[6] += 1;
  }
#ifdef INPC_PHASE_TIMES
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_mid_cyc[k], prof[k]);
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {  // every CTA has read the list count
    *done = 0u;
    sc->num_big = 0u;
    sc->max_big = 0u;
  }
}

// ---------------------------------------------------------------- H4+H6 (mid tiles, merge sort)
// NT threads per tile of LO < n <= MAXN entries, grid-stride over the
// big-tile list.  The tile's keys become unique 32-bit keys (depth - tile
// minimum, quantised to 32 - SB bits) << SB | list slot; each thread sorts a
// run of q = (padded n) / NT keys in registers (sorting network, no
// shuffles), then log2(NT) merge passes through SMEM ping-pong buffers:
// thread t writes outputs [t q, (t + 1) q) of every pass, starting from a
// merge-path co-rank search, so an output costs a handful of instructions
// instead of a network stage or a radix pass per key.  Quantisation ties are
// put in (depth, index) order on the full keys (short runs: insertion; long
// runs: 64-bit bitonic of the whole tile in the same SMEM).  Same lists, bit
// for bit, as every other sort path (R7/R8).  NT > 32 spreads one tile's
// serial merge chain over more threads (a warp per 2k-entry tile is bound by
// the latency of its ~400 dependent merge steps).
template <int NT, int MAXN>
struct MidMerge {
  static constexpr int kSlotBits = MAXN == 1024 ? 10 : MAXN == 2048 ? 11 : MAXN == 4096 ? 12 : 13;
  static constexpr int kQMax = MAXN / NT + 1;     // keys per thread (odd: conflict-free thread strides)
  static constexpr int kBuf = NT * kQMax;         // padded tile length
  static constexpr size_t kSmem = 2 * (size_t)kBuf * 4;  // two ping-pong buffers (dynamic SMEM)
  static constexpr int kMaxRun = 64;
  static_assert(MAXN == (1 << kSlotBits), "slot bits");
  static_assert(kQMax <= 17 && 2 * kBuf * 4 >= MAXN * 8, "run length / 64-bit fallback room");
};

template <int NT>
__device__ __forceinline__ void mm_sync() {
  if (NT == 32) __syncwarp();
  else __syncthreads();
}

// Sorting network on Q keys in registers (compile-time indices): ascending.
template <int Q>
__device__ __forceinline__ void lane_sort(uint32_t (&v)[Q]) {
#pragma unroll
  for (int k = 2; k <= Q; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const uint32_t a = v[i], b = v[l];
          if ((i & k) == 0) {
            v[i] = min(a, b);
            v[l] = max(a, b);
          } else {
            v[i] = max(a, b);
            v[l] = min(a, b);
          }
        }
      }
}

// Run `run` (keys [run q, run q + q), from the quantised depths in db) sorted
// in a Q-register network (Q >= q, the extra registers hold the pad key),
// its q smallest stored to dst.
template <int Q>
__device__ __forceinline__ void mm_run(const uint32_t* db, uint32_t* dst, int run, int q, int n, uint32_t dmin,
                                       int shift, int sb) {
  uint32_t v[Q];
  const int s = run * q;
#pragma unroll
  for (int t = 0; t < Q; ++t) {
    const int i = s + t;
    v[t] = (t < q && i < n) ? (((db[i] - dmin) >> shift) << sb) | (uint32_t)i : 0xFFFFFFFFu;
  }
  lane_sort<Q>(v);
#pragma unroll
  for (int t = 0; t < Q; ++t)
    if (t < q) dst[s + t] = v[t];
}

// Ascending bitonic sort of np (power of two) 64-bit keys in SMEM by NT threads.
template <int NT>
__device__ __forceinline__ void mm_bitonic64(unsigned long long* s, int np, int tid) {
  for (int k = 2; k <= np; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = tid; t < (np >> 1); t += NT) {
        const int i = 2 * t - (t & (j - 1));
        const int ixj = i + j;
        const unsigned long long a = s[i], b = s[ixj];
        const bool up = (i & k) == 0;
        if ((a > b) == up) {
          s[i] = b;
          s[ixj] = a;
        }
      }
      mm_sync<NT>();
    }
}

template <int NT, int MAXN>
__global__ void __launch_bounds__(NT) k_sort_mid_merge(
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ list_in, uint32_t* count_in,
    uint32_t* reset_also, const unsigned long long* __restrict__ entries, uint32_t* __restrict__ sorted_idx,
    uint32_t* __restrict__ list_out, uint32_t* count_out, uint32_t* __restrict__ done) {
  using M = MidMerge<NT, MAXN>;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) uint32_t buf[];  // 2 * kBuf
  __shared__ uint32_t red[2][NW];
  __shared__ uint32_t s_last;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  uint32_t* buf0 = buf;
  uint32_t* buf1 = buf + M::kBuf;
  constexpr int SB = M::kSlotBits;
  constexpr uint32_t smask = (uint32_t)MAXN - 1u;
  const uint32_t nb = *count_in;
  for (uint32_t j = blockIdx.x; j < nb; j += gridDim.x) {
    const uint32_t t = list_in[j];
    const uint32_t begin = ranges[t], n = ranges[t + 1] - begin;
    if (n > (uint32_t)MAXN) {  // block-uniform: the next size class's list
      if (list_out && tid == 0) list_out[atomicAdd(count_out, 1u)] = t;
      continue;
    }
    const unsigned long long* src = entries + begin;
    // depth bits to buf1, tile minimum / maximum
    uint32_t dlo = 0xFFFFFFFFu, dhi = 0u;
    for (uint32_t i = tid; i < n; i += NT) {
      const uint32_t d = (uint32_t)(__ldg(src + i) >> 32);
      buf1[i] = d;
      dlo = min(dlo, d);
      dhi = max(dhi, d);
    }
    dlo = __reduce_min_sync(0xffffffffu, dlo);
    dhi = __reduce_max_sync(0xffffffffu, dhi);
    if (NW > 1) {
      if (lane == 0) {
        red[0][w] = dlo;
        red[1][w] = dhi;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        dlo = min(dlo, red[0][k]);
        dhi = max(dhi, red[1][k]);
      }
    } else {
      __syncwarp();
    }
    const uint32_t range = dhi - dlo;
    const int vbits = range ? 32 - __clz(range) : 0;
    const int shift = vbits > 32 - SB ? vbits - (32 - SB) : 0;
    // per-thread runs of q keys (q odd: the thread strides of every pass hit
    // distinct banks) sorted in registers, written to buf0
    const int q = (((int)n + NT - 1) / NT) | 1;
    if (q <= 8) mm_run<8>(buf1, buf0, tid, q, (int)n, dlo, shift, SB);
    else if (q <= 16) mm_run<16>(buf1, buf0, tid, q, (int)n, dlo, shift, SB);
    else mm_run<32>(buf1, buf0, tid, q, (int)n, dlo, shift, SB);
    mm_sync<NT>();
    // merge passes: runs of L -> 2L; thread t writes outputs [t q, t q + q)
    const int np = NT * q;
    uint32_t* srcb = buf0;
    uint32_t* dstb = buf1;
    for (int L = q, ps = 1; L < np; L <<= 1, ++ps) {
      const int o0 = tid * q;
      const int P = (tid >> ps) * (2 * L);  // o0 / 2L with 2L = q 2^ps: no integer division
      const int d = o0 - P;
      int lo = d > L ? d - L : 0, hi = d < L ? d : L;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (srcb[P + mid] <= srcb[P + L + d - mid - 1]) lo = mid + 1;
        else hi = mid;
      }
      int ia = lo, ib = d - lo;
      uint32_t a = ia < L ? srcb[P + ia] : 0xFFFFFFFFu;
      uint32_t b = ib < L ? srcb[P + L + ib] : 0xFFFFFFFFu;
      // branch-free: one select of the taken side, one load of its successor
      uint32_t* dp = dstb + o0;
#pragma unroll 4
      for (int k = 0; k < q; ++k) {
        const bool ta = a <= b;
        dp[k] = ta ? a : b;
        ia += ta;
        ib += !ta;
        const int nx = ta ? ia : L + ib;
        const uint32_t v = (ta ? ia : ib) < L ? srcb[P + nx] : 0xFFFFFFFFu;
        a = ta ? v : a;
        b = ta ? b : v;
      }
      mm_sync<NT>();
      uint32_t* tmp = srcb;
      srcb = dstb;
      dstb = tmp;
    }
    // equal quantised depths: (depth, index) order on the full keys
    bool tie_bad = false;
    for (uint32_t p = tid; p + 1 < n; p += NT) {
      const uint32_t ka = srcb[p], kb = srcb[p + 1];
      if ((ka >> SB) == (kb >> SB) && __ldg(src + (ka & smask)) > __ldg(src + (kb & smask))) tie_bad = true;
    }
    const bool any_bad = NT == 32 ? __any_sync(0xffffffffu, tie_bad) : __syncthreads_or(tie_bad);
    if (any_bad) {
      bool too_long = false;
      for (uint32_t p = tid; p + 1 < n; p += NT) {
        const uint32_t a0 = srcb[p] >> SB;
        if ((srcb[p + 1] >> SB) != a0 || (p > 0 && (srcb[p - 1] >> SB) == a0)) continue;
        uint32_t end = p + 2;
        while (end < n && (srcb[end] >> SB) == a0 && end - p <= (uint32_t)M::kMaxRun) ++end;
        if (end - p > (uint32_t)M::kMaxRun) {
          too_long = true;
          continue;
        }
        for (uint32_t k = p + 1; k < end; ++k) {  // insertion sort of the run on the full keys
          const uint32_t v = srcb[k];
          const unsigned long long fv = __ldg(src + (v & smask));
          int jj = (int)k - 1;
          while (jj >= (int)p && __ldg(src + (srcb[jj] & smask)) > fv) {
            srcb[jj + 1] = srcb[jj];
            --jj;
          }
          srcb[jj + 1] = v;
        }
      }
      if (NT == 32) __syncwarp();
      const bool any_long = NT == 32 ? __any_sync(0xffffffffu, too_long) : __syncthreads_or(too_long);
      if (any_long) {  // long tie runs: 64-bit bitonic of the tile
        unsigned long long* s64 = reinterpret_cast<unsigned long long*>(buf);
        int np2 = 32;
        while (np2 < (int)n) np2 <<= 1;
        for (int i = tid; i < np2; i += NT) s64[i] = i < (int)n ? __ldg(src + i) : ~0ull;
        mm_sync<NT>();
        mm_bitonic64<NT>(s64, np2, tid);
        for (uint32_t i = tid; i < n; i += NT) sorted_idx[begin + i] = (uint32_t)s64[i];
        mm_sync<NT>();
        continue;
      }
    }
    const uint32_t* src32 = reinterpret_cast<const uint32_t*>(src);  // low word = point index
    for (uint32_t i = tid; i < n; i += NT) sorted_idx[begin + i] = __ldg(src32 + 2 * (srcb[i] & smask));
    mm_sync<NT>();
  }
  // the last CTA clears its input list's count for the next call
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    *done = 0u;
    *count_in = 0u;
    if (reset_also) *reset_also = 0u;
  }
}

// ---------------------------------------------------------------- H1..H6 fused (bilinear)
// One cooperative launch for the whole binning of a bilinear view: every
// thread keeps KP points' depth key, tile block and entry slots in
// registers across the grid barriers, so the slots never go to memory and
// the records are not read back.
//   phase 1  H1+H2: project, record, atomic slot per (point, tile)
//   phase 2  H3:    scan of the tile counts (per-CTA block scan + prefix of
//                   the CTA aggregates), counts zeroed for the next call
//   phase 3  H5:    scatter of the 64-bit keys to ranges[tile] + slot
//   phase 4  H4/H6: tiles over the warp-sort cap (big_sort_body)
constexpr int kBinThreads = 512;

template <int KP>
constexpr size_t bin_smem_bytes() {
  return (size_t)KP * 4 * kBinThreads * 4 > (size_t)kBigChunk * 8 ? (size_t)KP * 4 * kBinThreads * 4
                                                                   : (size_t)kBigChunk * 8;
}

template <int KP, bool SH>
__global__ void __launch_bounds__(kBinThreads, 2) k_bin_bilinear(
    DevCam cam, DevCfg g, const float* __restrict__ xyz, const float* __restrict__ opacity,
    const float* __restrict__ feat, bool pack, int64_t N, int T, PointRec* __restrict__ rec,
    uint32_t* counts, uint32_t* ranges, uint32_t* agg, uint32_t* big_tiles, uint32_t* big_elem,
    uint32_t* big_chunk, ViewScalars* sc, unsigned long long* entries, unsigned long long* tmp,
    uint32_t* sorted_idx, uint32_t* __restrict__ dbg_key, uint32_t* __restrict__ dbg_tiles,
    float* __restrict__ feat_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // dynamic SMEM (bin_smem_bytes<KP>()): the per-point tile slots of phases
  // 1-3 ([k][corner][thread], conflict-free), then phase 4's sort chunk
  extern __shared__ __align__(16) unsigned char bin_smem[];
  unsigned long long* s = reinterpret_cast<unsigned long long*>(bin_smem);
  uint32_t* s_sl = reinterpret_cast<uint32_t*>(bin_smem);
  __shared__ uint32_t carry[2];
  __shared__ uint32_t wt[kBinThreads / 32];
  const int64_t nthr = (int64_t)gridDim.x * kBinThreads;
  const int64_t tid = (int64_t)blockIdx.x * kBinThreads + threadIdx.x;
  BIN_TS(0);
  // ---- phase 1
  // per point in registers: depth key and tile base | corner mask << 28
  // (T < 2^28); the slots wait in SMEM.  Software pipeline (issue is in
  // order): the inputs of point k + 1 are loaded while point k is projected,
  // and the slots returned by point k's atomics are stored to SMEM two points
  // later, so that no instruction waits on an atomic's round trip.
  constexpr int kDefer = 2;
  uint32_t key[KP], tb[KP];
  uint32_t psl[kDefer][4];
  float nX = 0.f, nY = 0.f, nZ = 0.f, nO = 0.f;
  float4 nF = make_float4(0.f, 0.f, 0.f, 0.f);
  auto load_in = [&](int64_t i) {
    if (i < N) {
      nX = __ldg(xyz + 3 * i);
      nY = __ldg(xyz + 3 * i + 1);
      nZ = __ldg(xyz + 3 * i + 2);
      nO = __ldg(opacity + i);
      if (!SH && pack) nF = __ldg(reinterpret_cast<const float4*>(feat) + i);
    }
  };
  auto store_slots = [&](int k) {
    const uint32_t vm = tb[k] >> 28;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if ((vm >> c) & 1u) s_sl[(k * 4 + c) * kBinThreads + threadIdx.x] = psl[k % kDefer][c];
  };
  load_in(tid);
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const int64_t i = tid + k * nthr;
    key[k] = 0u;
    tb[k] = 0u;
    const float X = nX, Y = nY, Z = nZ, O = nO;
    const float4 Fv = nF;
    if (k + 1 < KP) load_in(i + nthr);
    if (i < N) {
      Proj p;
      Foot f;
      const bool vis = project_point(cam, X, Y, Z, p);
      const bool ok = vis && foot_bilinear(g, p.u, p.v, f);
      PointRec pr;
      pr.a = make_float4(p.u, p.v, ok ? p.zc : 0.0f, O);
      pr.b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (SH) {
        if (ok) sh_point_features(cam, g, feat, i, X, Y, Z, pack, pr.b, feat_out);
      } else if (pack) {
        pr.b = Fv;
      }
      rec[i] = pr;
      if (dbg_key) {
        dbg_key[i] = vis ? __float_as_uint(p.zc) : 0xFFFFFFFFu;
        dbg_tiles[i] = ok ? (uint32_t)((f.xhi / kTile - f.xlo / kTile + 1) * (f.yhi / kTile - f.ylo / kTile + 1)) : 0u;
      }
      if (k >= kDefer) store_slots(k - kDefer);
      if (ok) {
        const int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
        const int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
        key[k] = __float_as_uint(p.zc);
        uint32_t vm = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int tx = tx_lo + (c & 1), ty = ty_lo + (c >> 1);
          if (tx <= tx_hi && ty <= ty_hi) {
            psl[k % kDefer][c] = atomicAdd(counts + (size_t)ty * g.tiles_x + tx, 1u);
            vm |= 1u << c;
          }
        }
        tb[k] = (uint32_t)(ty_lo * g.tiles_x + tx_lo) | (vm << 28);
      }
    } else if (k >= kDefer) {
      store_slots(k - kDefer);
    }
  }
#pragma unroll
  for (int k = KP - kDefer; k < KP; ++k)
    if (k >= 0) store_slots(k);
  grid.sync();
  BIN_TS(1);
  // ---- phase 2: CTA b scans tiles [b*per, (b+1)*per)
  const int per = (T + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(T, t0 + per);
  const int items = (per + kBinThreads - 1) / kBinThreads;  // consecutive tiles per thread
  const int my0 = t0 + threadIdx.x * items;
  uint32_t sum = 0;
  for (int q = 0; q < items; ++q) {
    const int t = my0 + q;
    if (t < t1) sum += counts[t];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wt[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < kBinThreads / 32 ? wt[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kBinThreads / 32) wt[lane] = w;
  }
  __syncthreads();
  const uint32_t excl = (wid ? wt[wid - 1] : 0u) + x - sum;
  if (threadIdx.x == 0) agg[blockIdx.x] = wt[kBinThreads / 32 - 1];
  grid.sync();
  // prefix of the preceding CTAs' aggregates
  uint32_t pre = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += kBinThreads) pre += agg[b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  __syncthreads();
  if (lane == 0) wt[wid] = pre;
  __syncthreads();
  uint32_t cta_pre = 0;
#pragma unroll
  for (int w = 0; w < kBinThreads / 32; ++w) cta_pre += wt[w];
  uint32_t off = cta_pre + excl, mx = 0;
  for (int q = 0; q < items; ++q) {
    const int t = my0 + q;
    if (t >= t1) break;
    const uint32_t c = counts[t];
    counts[t] = 0u;  // ready for the next call
    ranges[t] = off;
    if (c > (uint32_t)kWarpSortCap) {
      big_tiles[atomicAdd(&sc->num_big, 1u)] = t;
      mx = max(mx, c);
    }
    off += c;
  }
  if (mx) atomicMax(&sc->max_big, mx);
  grid.sync();
  BIN_TS(2);
  if (blockIdx.x == 0) {  // grand total = F_t
    uint32_t tot = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kBinThreads) tot += agg[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) wt[wid] = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kBinThreads / 32; ++w) t += wt[w];
      ranges[T] = t;
      sc->Ft = t;
    }
  }
  // ---- phase 3: scatter
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (!key[k]) continue;
    const int64_t i = tid + k * nthr;
    const unsigned long long kv = ((unsigned long long)key[k] << 32) | (uint32_t)i;
    const uint32_t t0 = tb[k] & 0x0FFFFFFFu;
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if ((tb[k] >> (28 + c)) & 1u) {
        const uint32_t t = t0 + (uint32_t)(c & 1) + (uint32_t)(c >> 1) * g.tiles_x;
        entries[ranges[t] + s_sl[(k * 4 + c) * kBinThreads + threadIdx.x]] = kv;
      }
  }
  grid.sync();
  BIN_TS(3);
  // ---- phase 4: big tiles
  big_sort_body<kBigChunk>(grid, s, carry, ranges, big_tiles, &sc->num_big, &sc->max_big, big_elem, big_chunk,
                           sc, entries, tmp,
                           sorted_idx);
  BIN_TS(7);
}

// ---------------------------------------------------------------- H7 / H8 per-warp staging
// One chunk of 32 tile-list entries staged in SMEM (SoA, slot = lane) plus
// the per-pixel fragment masks of the chunk: bit e of mask[p] is set when
// entry e has a (possible) fragment at tile pixel p = 8*row + col.
//   bilinear: block origin (x0, y0) and, per block corner k = 2 dy + dx,
//             the weight w_k (pinned fp32, R1/R3)
//   Gaussian: u, v and the conic; the pixel lane evaluates q and w (R17)
// One chunk's point records (and unpacked C = 4 features), copied into SMEM
// with cp.async one chunk ahead of their use: the gathers of chunk k + 1 are
// in flight while chunk k's pixels are composited, at no register cost.
template <int NS>
struct RecBufT {
  float4 A[NS], B[NS], F[NS];
};
using RecBuf = RecBufT<32>;

template <int CMAX>
struct ChunkSmem {
  union {
    struct {
      int xy[32];               // bilinear block origin, x0 | y0 << 16
      int cbase[32];            // bilinear corner base: corner = cb + 2 ly + lx at tile pixel (lx, ly)
      float ac[32][4];          // bilinear alpha = min(o w, alpha_max) per block corner
    };
    struct {
      float u[32], v[32], ca[32], cb[32], cc[32];  // Gaussian
    };
  };
  float o[32], z[32];
  float f[32][CMAX];
  uint32_t mask[64];
  uint32_t idx[32];
};

template <int CMAX, bool PF = false>
struct FwdSmem {
  unsigned long long keys[kWarpSortCap];
  ChunkSmem<CMAX> ch;
  RecBuf rb;
};
// without the record prefetch the SMEM footprint stays small (a larger L1
// carveout: measured 508 vs 731 us on cfg 4)
template <int CMAX>
struct FwdSmem<CMAX, false> {
  unsigned long long keys[kWarpSortCap];
  ChunkSmem<CMAX> ch;
  RecBufT<1> rb;  // unused
};

// Backward per-warp SMEM.  The pixel's upstream gradient G is staged per
// tile (Gs), so a fragment only needs two scalars: ta = T_k alpha_k
// (dL/df_k = ta G) and go = dL/do contribution.  Bilinear: every fragment of
// an entry in the tile is one of its 2x2 block corners, so each fragment
// owns a slot [entry][corner] and the entry lane sums its <= 4 corners with
// no SMEM atomics (float atomicAdd on SMEM is a CAS loop on this part).
// Gaussian: the pixel lane adds ta G and go to the entry with SMEM atomics.
template <int MODE, int CMAX>
struct BwdSmem {
  static constexpr bool kSlots = MODE == 0;
  // bilinear: 8 floats per entry (4 corners x {T alpha, dL/do}) + pad, rows
  // 8-byte aligned for one 64-bit store per fragment; Gaussian: odd stride
  static constexpr int kStride = kSlots ? 10 : CMAX + 2;
  ChunkSmem<CMAX> ch;
  float gw[32][4];   // bilinear dalpha/do per corner: w, or 0 where clamped
  float rc[32][4];   // bilinear 1 / (1 - alpha) per corner (approximate: the recovery adds a Newton step)
  float Gs[64][CMAX];
  __align__(8) float acc[32][kStride];
  RecBuf rb;
};

// 1/x to ~1 ulp (MUFU.RCP; x in [0.01, 1] here): the backward's T recovery
// corrects it with one Newton step of the residual
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The global loads of one tile-list entry, issued a chunk ahead of their
// use (software pipelining: the warp works on chunk k while chunk k+1's
// record gathers are in flight).
struct EntryRegs {
  float4 A, B, F;  // record halves; F = features when they are not packed
  uint32_t idx;
};

template <int CMAX>
__device__ __forceinline__ EntryRegs load_entry(const DevCfg& g, const PointRec* __restrict__ rec,
                                                const float* __restrict__ feat, bool packed,
                                                uint32_t idx) {
  EntryRegs r;
  r.idx = idx;
  if (g.flags & kFlagRec16) {
    r.A = __ldg(reinterpret_cast<const float4*>(rec) + idx);
    r.B = make_float4(0.f, 0.f, 0.f, 0.f);
  } else {
    r.A = __ldg(&rec[idx].a);
    r.B = __ldg(&rec[idx].b);
  }
  if (CMAX == 4 && !packed && g.C == 4) r.F = __ldg(reinterpret_cast<const float4*>(feat) + idx);
  return r;
}

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Issue the copies of entry `idx`'s record into slot `lane` (valid lanes only).
template <int CMAX, typename RB>
__device__ __forceinline__ void prefetch_entry(RB& rb, const DevCfg& g, const PointRec* __restrict__ rec,
                                               const float* __restrict__ feat, bool packed, uint32_t idx,
                                               bool valid, int lane) {
  if (valid) {
    if (g.flags & kFlagRec16) {
      cp_async16(&rb.A[lane], reinterpret_cast<const float4*>(rec) + idx);
    } else {
      cp_async16(&rb.A[lane], &rec[idx].a);
      cp_async16(&rb.B[lane], &rec[idx].b);
    }
    if (CMAX == 4 && !packed && g.C == 4) cp_async16(&rb.F[lane], reinterpret_cast<const float4*>(feat) + idx);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <typename RB>
__device__ __forceinline__ EntryRegs entry_from_buf(const RB& rb, uint32_t idx, int lane) {
  EntryRegs r;
  r.idx = idx;
  r.A = rb.A[lane];
  r.B = rb.B[lane];
  r.F = rb.F[lane];
  return r;
}

// Stage a loaded entry in slot `lane` and mark its pixels of the tile
// (origin tx0, ty0) in the chunk masks.
template <int MODE, int CMAX, bool BWD>
__device__ __forceinline__ void stage_entry(ChunkSmem<CMAX>& cs, int lane, const DevCfg& g,
                                            const EntryRegs& r, const float* __restrict__ feat,
                                            bool packed, int tx0, int ty0, float* gw_out = nullptr,
                                            float* rc_out = nullptr) {
  const float4 A = r.A, B = r.B;
  const uint32_t idx = r.idx;
  Foot f;
  bool ok = rec_foot<MODE>(g, A, B.w, f);
  cs.idx[lane] = idx;
  cs.o[lane] = A.w;
  cs.z[lane] = A.z;
  if (MODE == 0) {
    cs.xy[lane] = (f.x0 & 0xFFFF) | (f.y0 << 16);
    cs.cbase[lane] = -(2 * (f.y0 - ty0) + (f.x0 - tx0));
    const float fa1 = __fsub_rn(1.0f, f.fa), fb1 = __fsub_rn(1.0f, f.fb);
    const float w[4] = {__fmul_rn(fa1, fb1), __fmul_rn(f.fa, fb1), __fmul_rn(fa1, f.fb),
                        __fmul_rn(f.fa, f.fb)};
    float al[4], gw[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float ow = __fmul_rn(A.w, w[c]);
      al[c] = fminf(ow, g.amax);
      gw[c] = ow < g.amax ? w[c] : 0.0f;
    }
    *reinterpret_cast<float4*>(&cs.ac[lane][0]) = make_float4(al[0], al[1], al[2], al[3]);
    if (BWD) {
      *reinterpret_cast<float4*>(gw_out) = make_float4(gw[0], gw[1], gw[2], gw[3]);
      *reinterpret_cast<float4*>(rc_out) =
          make_float4(rcp_approx(__fsub_rn(1.0f, al[0])), rcp_approx(__fsub_rn(1.0f, al[1])),
                      rcp_approx(__fsub_rn(1.0f, al[2])), rcp_approx(__fsub_rn(1.0f, al[3])));
    }
  } else {
    cs.u[lane] = A.x;
    cs.v[lane] = A.y;
    cs.ca[lane] = B.x;
    cs.cb[lane] = B.y;
    cs.cc[lane] = B.z;
  }
  if (CMAX == 4 && packed) {
    *reinterpret_cast<float4*>(&cs.f[lane][0]) = B;
  } else if (CMAX == 4 && g.C == 4) {
    *reinterpret_cast<float4*>(&cs.f[lane][0]) = r.F;
  } else {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)  // channels >= C are zero so vector reads stay finite
      cs.f[lane][c] = c < g.C ? __ldg(feat + (size_t)idx * g.C + c) : 0.0f;
  }
  if (!ok) return;
  // footprint rectangle clipped to the tile, tile-local coordinates
  const int xl = max(f.xlo, tx0) - tx0, xh = min(f.xhi, tx0 + kTile - 1) - tx0;
  const int yl = max(f.ylo, ty0) - ty0, yh = min(f.yhi, ty0 + kTile - 1) - ty0;
  if (MODE == 0) {  // the 2x2 block: four predicated marks, no loops
    const int bx = f.x0 - tx0, by = f.y0 - ty0;
    // SKIP_ZERO_ALPHA_GRAD (A/B of the original INPC behaviour): the
    // backward leaves alpha = 0 fragments out of its masks
    const bool skipz = BWD && (g.flags & kFlagSkipZero);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int xx = bx + (k & 1), yy = by + (k >> 1);
      if (xx >= xl && xx <= xh && yy >= yl && yy <= yh && !(skipz && cs.ac[lane][k] == 0.0f))
        atomicOr(&cs.mask[yy * kTile + xx], 1u << lane);
    }
  } else {
    for (int yy = yl; yy <= yh; ++yy)
      for (int xx = xl; xx <= xh; ++xx) atomicOr(&cs.mask[yy * kTile + xx], 1u << lane);
  }
}

// Fragment of staged entry e at pixel (px, py): alpha (R4, R5), dalpha/do
// (0 where the clamp is active) and the bilinear block corner.  Bilinear:
// every pixel of the rectangle is a fragment.  Gaussian: q <= 9 (R17).
template <int MODE, int CMAX>
__device__ __forceinline__ bool entry_alpha(const ChunkSmem<CMAX>& cs, const DevCfg& g, int e,
                                            int px, int py, int pc, float& alpha, float& gw,
                                            int& corner) {
  if (MODE == 0) {
    corner = cs.cbase[e] + pc;  // pc = 2 ly + lx of the pixel in its tile
    alpha = cs.ac[e][corner];
    gw = 0.0f;  // forward only: the backward reads its packed corner data
    return true;
  } else {
    corner = 0;
    const float q = gauss_q(cs.ca[e], cs.cb[e], cs.cc[e], cs.u[e], cs.v[e], px, py);
    if (!(q <= 9.0f)) return false;
    const float w = expf(__fmul_rn(-0.5f, q));
    const float ow = __fmul_rn(cs.o[e], w);
    alpha = fminf(ow, g.amax);
    gw = ow < g.amax ? w : 0.0f;
    return true;
  }
}

// Background of pixel (px, py) from the environment map env [He, We, C].
template <int CMAX>
__device__ __forceinline__ void env_lookup(const DevCam& cam, const DevCfg& g,
                                           const float* __restrict__ env, int px, int py, float* b) {
  int id[4];
  float w[4];
  env_weights(cam, g, px, py, id, w);
  if (CMAX == 4 && g.C == 4) {
    float4 t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = __ldg(reinterpret_cast<const float4*>(env) + id[q]);
    b[0] = (w[0] * t[0].x + w[1] * t[1].x) + (w[2] * t[2].x + w[3] * t[3].x);
    b[1] = (w[0] * t[0].y + w[1] * t[1].y) + (w[2] * t[2].y + w[3] * t[3].y);
    b[2] = (w[0] * t[0].z + w[1] * t[1].z) + (w[2] * t[2].z + w[3] * t[3].z);
    b[3] = (w[0] * t[0].w + w[1] * t[1].w) + (w[2] * t[2].w + w[3] * t[3].w);
  } else {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      b[c] = c < g.C ? (w[0] * __ldg(env + (size_t)id[0] * g.C + c) + w[1] * __ldg(env + (size_t)id[1] * g.C + c)) +
                           (w[2] * __ldg(env + (size_t)id[2] * g.C + c) + w[3] * __ldg(env + (size_t)id[3] * g.C + c))
                     : 0.0f;
  }
}

struct BlendOut {
  float* F;           // [H,W,C]
  float* A;           // [H,W] or null
  float* D;           // [H,W] or null
  int32_t* nfrag;     // or null
  int32_t* ncontrib;  // or null
  float* T_final;     // saved [H,W]
  uint32_t* last;     // saved [H,W]: list position + 1 of the last composited fragment
  const uint32_t* order;  // tile visiting order (big tiles first) or null: band order
};

template <int CMAX>
struct PixFwd {
  float T, D;
  float F[CMAX];
  uint32_t last;
  int nfrag, ncontrib;
  bool done;
};

// Composite the fragments of one pixel in this chunk (bits of m, ascending =
// list order), Eq. 1 with alpha clamp (R5) and early termination (R6).
template <int MODE, int CMAX, bool COUNT>
__device__ __forceinline__ void blend_pixel(const ChunkSmem<CMAX>& cs, const DevCfg& g,
                                            uint32_t m, int px, int py, int pc, uint32_t base,
                                            PixFwd<CMAX>& s) {
  const bool count = COUNT;
  if (s.done && !count) return;
  while (m) {
    const int e = __ffs(m) - 1;
    m &= m - 1;
    float alpha, gw;
    int corner;
    if (!entry_alpha<MODE, CMAX>(cs, g, e, px, py, pc, alpha, gw, corner)) continue;
    if (COUNT) s.nfrag++;
    if (s.done) continue;
    const float Tn = __fmul_rn(s.T, __fsub_rn(1.0f, alpha));
    if (Tn < g.tmin) {
      s.done = true;
      if (!count) return;
      continue;
    }
    const float wgt = alpha * s.T;
    if (CMAX == 4) {
      const float4 fv = *reinterpret_cast<const float4*>(&cs.f[e][0]);
      s.F[0] += wgt * fv.x;
      s.F[1] += wgt * fv.y;
      s.F[2] += wgt * fv.z;
      s.F[3] += wgt * fv.w;
    } else {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < g.C) s.F[c] += wgt * cs.f[e][c];
    }
    s.D += wgt * cs.z[e];
    s.T = Tn;
    s.last = base + e + 1;
    if (COUNT) s.ncontrib++;
  }
}

template <int CMAX>
__device__ __forceinline__ void write_pixel(const DevCam& cam, const DevCfg& g, const BlendOut& out,
                                            const float* __restrict__ bg, int px, int py,
                                            PixFwd<CMAX>& s) {
  const size_t pix = (size_t)py * g.W + px;
  if (bg && (g.flags & kFlagEnv)) {  // NEXT f2: environment-map background
    float b[CMAX];
    env_lookup<CMAX>(cam, g, bg, px, py, b);
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) s.F[c] += s.T * b[c];
  } else if (bg) {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) s.F[c] += s.T * __ldg(bg + pix * g.C + c);
  }
  if (CMAX == 4 && g.C == 4) {
    reinterpret_cast<float4*>(out.F)[pix] = make_float4(s.F[0], s.F[1], s.F[2], s.F[3]);
  } else {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) out.F[pix * g.C + c] = s.F[c];
  }
  if (out.A) out.A[pix] = 1.0f - s.T;
  if (out.D) out.D[pix] = s.D;
  out.T_final[pix] = s.T;
  out.last[pix] = s.last;
  if (out.nfrag) out.nfrag[pix] = s.nfrag;      // set only in COUNT mode
  if (out.ncontrib) out.ncontrib[pix] = s.ncontrib;
}

// ---------------------------------------------------------------- H4/H6 (small tiles) + H7
// One warp per 8x8 tile; lane l owns pixels (l & 7, l >> 3) and (l & 7, 4 + (l >> 3)).
// PF: records of the next chunk copied into SMEM (cp.async) while this one is
// composited, for tiles whose list fits the warp sort.  Chosen by the host
// from the cloud density (measured: cfg 3 fwd 261 -> 244 us, cfg 5 16.3 ->
// 14.6 ms per 64 views, cfg 2 neutral; cfg 4 (~1000 points per tile, long
// lists ended by early termination) 514 -> 780 us, so dense clouds run
// without).
template <int MODE, int CMAX, bool COUNT, int WPB = kWarpsPerBlock, bool PF = false>
#ifndef INPC_FWD_MINB
#define INPC_FWD_MINB (32 / INPC_WPB)  // 64 registers (measured optimum: 76 at 1 CTA, 48 + spills at 40 warps are slower)
#endif
#ifndef INPC_BWD_WARPS_PER_SM
#define INPC_BWD_WARPS_PER_SM 28
#endif
__global__ void __launch_bounds__(WPB * 32, INPC_FWD_MINB) k_blend_fwd(
    DevCam cam, DevCfg g, int band_tiles, const PointRec* __restrict__ rec,
    const float* __restrict__ feat, bool packed, const float* __restrict__ bg,
    const uint32_t* __restrict__ ranges, const unsigned long long* __restrict__ entries,
    uint32_t* __restrict__ sorted_idx, BlendOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FwdSmem<CMAX, PF>& S = reinterpret_cast<FwdSmem<CMAX, PF>*>(smem_raw)[warp];
  const int tl = blockIdx.x * WPB + warp;
  if (tl >= band_tiles) return;  // warp-uniform; no block barriers below
  const int tile = out.order ? (int)out.order[tl] : g.ty0 * g.tiles_x + tl;
  const int tx0 = (tile % g.tiles_x) * kTile, ty0 = (tile / g.tiles_x) * kTile;
  const int px = tx0 + (lane & 7), pyA = ty0 + (lane >> 3), pyB = pyA + 4;
  const int pcA = 2 * (lane >> 3) + (lane & 7);  // 2 ly + lx of pixel A (B: + 8)
  const bool inA = px < g.W && pyA < g.H, inB = px < g.W && pyB < g.H;
  const uint32_t begin = ranges[tile], n = ranges[tile + 1] - begin;
  const bool small = n <= (uint32_t)kWarpSortCap;
  if (small && n > 0) {
    warp_sort(S.keys, entries + begin, (int)n, lane);
    for (uint32_t k = lane; k < n; k += 32) sorted_idx[begin + k] = (uint32_t)S.keys[k];
  }
  const bool count = COUNT;  // debug counts (n_frag, n_contrib): no early exit
  PixFwd<CMAX> a, b;
  a.T = b.T = 1.0f;
  a.D = b.D = 0.0f;
#pragma unroll
  for (int c = 0; c < CMAX; ++c) a.F[c] = b.F[c] = 0.0f;
  a.last = b.last = 0;
  a.nfrag = b.nfrag = a.ncontrib = b.ncontrib = 0;
  a.done = !inA;
  b.done = !inB;
  ChunkSmem<CMAX>& cs = S.ch;
  auto idx_at = [&](uint32_t e) -> uint32_t {
    return e < n ? (small ? (uint32_t)S.keys[e] : __ldg(sorted_idx + begin + e)) : 0u;
  };
  constexpr bool pf = PF;
  // list indices one chunk ahead of the records (a big tile's indices come
  // from global memory: the record gathers never wait on them)
  uint32_t idx = idx_at(lane), idx_nx = idx_at(lane + 32);
  if (pf) prefetch_entry<CMAX>(S.rb, g, rec, feat, packed, idx, lane < n, lane);
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t e = base + lane;
    cs.mask[lane] = 0u;
    cs.mask[lane + 32] = 0u;
    if (pf) cp_async_wait_all();
    __syncwarp();
    if (e < n) {
      const EntryRegs r = pf ? entry_from_buf(S.rb, idx, lane) : load_entry<CMAX>(g, rec, feat, packed, idx);
      stage_entry<MODE, CMAX, false>(cs, lane, g, r, feat, packed, tx0, ty0);
    }
    __syncwarp();
    if (base + 32 < n) {  // the next chunk's records fly while this one is composited
      if (pf) prefetch_entry<CMAX>(S.rb, g, rec, feat, packed, idx_nx, e + 32 < n, lane);
      idx = idx_nx;
      idx_nx = idx_at(e + 64);
    }
    blend_pixel<MODE, CMAX, COUNT>(cs, g, cs.mask[lane], px, pyA, pcA, base, a);
    blend_pixel<MODE, CMAX, COUNT>(cs, g, cs.mask[lane + 32], px, pyB, pcA + 8, base, b);
    __syncwarp();
    if (!count && __all_sync(0xffffffffu, a.done && b.done)) break;
  }
  if (inA) write_pixel<CMAX>(cam, g, out, bg, px, pyA, a);
  if (inB) write_pixel<CMAX>(cam, g, out, bg, px, pyB, b);
  if (PF) cp_async_wait_all();  // an early exit may leave the next chunk's copies in flight
}

// ---------------------------------------------------------------- H8
struct BwdIn {
  const float* gF;       // [H,W,C]
  const float* gA;       // [H,W] or null
  const float* gD;       // [H,W] or null
  const float* T_final;  // saved
  const uint32_t* last;  // saved
  float* g_feat;         // [N,C] +=
  float* g_op;           // [N] +=
  // deterministic mode (INPC_FLAG_DETERMINISTIC_GRADS): per-entry sums go to
  // det_f [F_t][C] / det_o [F_t] at the entry's list position (no atomics);
  // k_det_reduce adds them per point in a fixed order
  float* det_f;
  float* det_o;
  const uint32_t* order;  // tile visiting order or null (as the forward's)
};

template <int CMAX>
struct PixBwd {
  float T, GA, GD, S, SD, P;  // S = G . R (R: everything behind, normalised), SD likewise for depth;
                              // default build: S holds the unnormalised Q (bwd_pixel), SD / P unused
  float G[CMAX];
  uint32_t last;
};

template <int MODE, int CMAX>
__device__ __forceinline__ void load_pixel_bwd(const DevCam& cam, const DevCfg& g, const BwdIn& in,
                                               const float* __restrict__ bg, bool inside, int px,
                                               int py, float* Gs, PixBwd<CMAX>& s) {
  s.T = 1.0f;
  s.GA = s.GD = s.S = s.SD = 0.0f;
  s.P = 1.0f;
  s.last = 0;
#pragma unroll
  for (int c = 0; c < CMAX; ++c) s.G[c] = 0.0f;
  if (inside) {
    const size_t pix = (size_t)py * g.W + px;
    s.last = in.last[pix];
    s.T = in.T_final[pix];
    if (in.gA) s.GA = in.gA[pix];
    if (in.gD) s.GD = in.gD[pix];
    const bool env = bg && (g.flags & kFlagEnv);
    if (CMAX == 4 && g.C == 4) {
      float4 v = __ldg(reinterpret_cast<const float4*>(in.gF) + pix);
      s.G[0] = v.x; s.G[1] = v.y; s.G[2] = v.z; s.G[3] = v.w;
      if (bg && !env) {  // S starts as G . bg: the background is behind every fragment
        float4 r = __ldg(reinterpret_cast<const float4*>(bg) + pix);
        s.S = (v.x * r.x + v.y * r.y) + (v.z * r.z + v.w * r.w);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < g.C) {
          s.G[c] = in.gF[pix * g.C + c];
          if (bg && !env) s.S += s.G[c] * bg[pix * g.C + c];
        }
    }
    if (env) {  // NEXT f2: the environment lookup is the background
      float b[CMAX];
      env_lookup<CMAX>(cam, g, bg, px, py, b);
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < g.C) s.S += s.G[c] * b[c];
    }
  }
#ifndef INPC_BWD_NORMALISED
  // unnormalised accumulator of everything behind the current fragment:
  // Q = T_final (G . bg - G_A), grown by T_k alpha_k (G . f_k + G_D z_k)
  s.S = s.T * (s.S - s.GA);
#endif
#pragma unroll
  for (int c = 0; c < CMAX; ++c) Gs[c] = s.G[c];
}

// Reverse-order backward of one pixel over this chunk's fragments (bits of
// m, descending = reverse list order):
//   T_k = T_{k+1} / (1 - alpha_k)
//   dL/dalpha_k = T_k [G.f_k - S_k + G_D (z_k - SD_k) + G_A P_k]   (Eq. 2 corrected, R12)
//   dL/df_k = T_k alpha_k G ;  dL/do += w_k dL/dalpha_k (0 where clamped)
//   S <- alpha G.f_k + (1 - alpha) S, SD likewise with z, P <- (1 - alpha) P
// where S = G . R carries the composited colour behind fragment k (R starts
// as the background).  alpha = 0 fragments are processed (R13).
template <int MODE, int CMAX>
__device__ __forceinline__ void bwd_pixel(BwdSmem<MODE, CMAX>& S, const DevCfg& g, uint32_t m,
                                          int px, int py, int pc, PixBwd<CMAX>& s) {
  using SM = BwdSmem<MODE, CMAX>;
  const ChunkSmem<CMAX>& cs = S.ch;
  while (m) {
    const int e = 31 - __clz(m);
    m &= ~(1u << e);
    float alpha, gw, one_m, rcp, z;
    int corner = 0;
    if (MODE == 0) {
      corner = cs.cbase[e] + pc;
      alpha = cs.ac[e][corner];
      gw = S.gw[e][corner];
      rcp = S.rc[e][corner];
      z = cs.z[e];
      one_m = __fsub_rn(1.0f, alpha);
    } else {
      if (!entry_alpha<MODE, CMAX>(cs, g, e, px, py, pc, alpha, gw, corner)) continue;
      one_m = __fsub_rn(1.0f, alpha);
      rcp = __frcp_rn(one_m);
      z = cs.z[e];
      if ((g.flags & kFlagSkipZero) && alpha == 0.0f) continue;
    }
    // T_k = T_{k+1} / (1 - alpha_k) from the staged reciprocal plus one
    // Newton correction of the residual (as accurate as the IEEE division on
    // 0 <= alpha < 1, without its special-case branch).  The recovery error
    // grows with the list length; the plain 2-ulp fast division fails the
    // 1e-3 gate on 40k-fragment pixels.
    const float q0 = s.T * rcp;
    const float Tk = fmaf(fmaf(-q0, one_m, s.T), rcp, q0);
    float gf = 0.0f;
    if (CMAX == 4) {
      const float4 fv = *reinterpret_cast<const float4*>(&cs.f[e][0]);
      gf = (s.G[0] * fv.x + s.G[1] * fv.y) + (s.G[2] * fv.z + s.G[3] * fv.w);
    } else {
#pragma unroll
      for (int c = 0; c < CMAX; ++c) gf += s.G[c] * cs.f[e][c];
    }
#ifdef INPC_BWD_NORMALISED
    const float dA = Tk * ((gf - s.S) + s.GD * (z - s.SD) + s.GA * s.P);
#else
    // Eq. 2 with the behind-terms unnormalised: T_k S_k = B_k / (1 - alpha_k),
    // T_k SD_k = BD_k / (1 - alpha_k), T_k P_k = T_final / (1 - alpha_k), so
    // dL/dalpha_k = T_k (G.f_k + G_D z_k) - Q_k / (1 - alpha_k) with
    // Q_k = B_k + G_D BD_k - G_A T_final (one running sum instead of three)
    const float h = fmaf(s.GD, z, gf);
    const float dA = fmaf(-s.S, rcp, Tk * h);
#endif
    const float ta = Tk * alpha;
    const float go = gw * dA;  // dalpha/do = w, or 0 where the clamp is active
    if (SM::kSlots) {
      *reinterpret_cast<float2*>(&S.acc[e][2 * corner]) = make_float2(ta, go);
    } else {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < g.C) atomicAdd(&S.acc[e][c], ta * s.G[c]);
      atomicAdd(&S.acc[e][CMAX], go);
    }
#ifdef INPC_BWD_NORMALISED
    s.S = alpha * gf + one_m * s.S;
    s.SD = alpha * z + one_m * s.SD;
    s.P *= one_m;
#else
    s.S = fmaf(ta, h, s.S);
#endif
    s.T = Tk;
  }
}

__device__ __forceinline__ uint32_t below_mask(uint32_t last, uint32_t base) {
  // bits e with base + e < last
  if (last <= base) return 0u;
  uint32_t k = last - base;
  return k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
}

// 7 CTAs of 4 warps per SM (<= 73 registers): measured 82 vs 93 us at 6 CTAs on cfg 2
template <int MODE, int CMAX, int WPB = kWarpsPerBlock>
__global__ void __launch_bounds__(WPB * 32, CMAX <= 4 ? INPC_BWD_WARPS_PER_SM / WPB : 1) k_blend_bwd(
    DevCam cam, DevCfg g, int band_tiles, const PointRec* __restrict__ rec,
    const float* __restrict__ feat, bool packed, const float* __restrict__ bg,
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ sorted_idx, BwdIn in) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  using SM = BwdSmem<MODE, CMAX>;
  SM& S = reinterpret_cast<SM*>(smem_raw)[warp];
  const int tl = blockIdx.x * WPB + warp;
  if (tl >= band_tiles) return;
  const int tile = in.order ? (int)in.order[tl] : g.ty0 * g.tiles_x + tl;
  const int tx0 = (tile % g.tiles_x) * kTile, ty0 = (tile / g.tiles_x) * kTile;
  const int px = tx0 + (lane & 7), pyA = ty0 + (lane >> 3), pyB = pyA + 4;
  const int pcA = 2 * (lane >> 3) + (lane & 7);  // 2 ly + lx of pixel A (B: + 8)
  const bool inA = px < g.W && pyA < g.H, inB = px < g.W && pyB < g.H;
  const uint32_t begin = ranges[tile];
  PixBwd<CMAX> a, b;
  load_pixel_bwd<MODE, CMAX>(cam, g, in, bg, inA, px, pyA, &S.Gs[lane][0], a);
  load_pixel_bwd<MODE, CMAX>(cam, g, in, bg, inB, px, pyB, &S.Gs[lane + 32][0], b);
  uint32_t tmax = max(a.last, b.last);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
  if (tmax == 0) return;
  ChunkSmem<CMAX>& cs = S.ch;
  const int chunk0 = (int)((tmax - 1) >> 5);
  // software pipeline over the chunks (reverse order): the records of the
  // next chunk are copied into SMEM (cp.async) while this one is processed,
  // and the list indices are loaded one chunk further ahead
  uint32_t idx = chunk0 * 32 + lane < tmax ? __ldg(sorted_idx + begin + chunk0 * 32 + lane) : 0u;
  prefetch_entry<CMAX>(S.rb, g, rec, feat, packed, idx, chunk0 * 32 + lane < tmax, lane);
  uint32_t idx_next = chunk0 > 0 ? __ldg(sorted_idx + begin + chunk0 * 32 - 32 + lane) : 0u;
  for (int chunk = chunk0; chunk >= 0; --chunk) {
    const uint32_t base = (uint32_t)chunk * 32;
    const uint32_t e = base + lane;
    cs.mask[lane] = 0u;
    cs.mask[lane + 32] = 0u;
#pragma unroll
    for (int c = 0; c < SM::kStride; ++c) S.acc[lane][c] = 0.0f;
    cp_async_wait_all();
    __syncwarp();
    if (e < tmax)
      stage_entry<MODE, CMAX, true>(cs, lane, g, entry_from_buf(S.rb, idx, lane), feat, packed, tx0, ty0,
                                    &S.gw[lane][0], &S.rc[lane][0]);
    __syncwarp();
    const uint32_t idx_pf = idx_next;  // chunk - 1 (every entry below tmax)
    if (chunk > 0) {
      prefetch_entry<CMAX>(S.rb, g, rec, feat, packed, idx_pf, true, lane);
      if (chunk > 1) idx_next = __ldg(sorted_idx + begin + base - 64 + lane);
    }
    bwd_pixel<MODE, CMAX>(S, g, cs.mask[lane] & below_mask(a.last, base), px, pyA, pcA, a);
    bwd_pixel<MODE, CMAX>(S, g, cs.mask[lane + 32] & below_mask(b.last, base), px, pyB, pcA + 8, b);
    __syncwarp();
    if (e < tmax) {  // entries without a contribution (all sums zero) send nothing
      float gsum[CMAX + 1];
#pragma unroll
      for (int c = 0; c <= CMAX; ++c) gsum[c] = 0.0f;
      if (SM::kSlots) {
        // corner k of the block is tile pixel (x0 + (k & 1), y0 + (k >> 1))
        const int xy = cs.xy[lane];
        const int lx = (int)(short)(xy & 0xFFFF) - tx0, ly = (xy >> 16) - ty0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int cx = lx + (k & 1), cy = ly + (k >> 1);
          if (cx < 0 || cx >= kTile || cy < 0 || cy >= kTile) continue;
          const float2 sl = *reinterpret_cast<const float2*>(&S.acc[lane][2 * k]);
          const float* Gp = &S.Gs[cy * kTile + cx][0];
#pragma unroll
          for (int c = 0; c < CMAX; ++c) gsum[c] += sl.x * Gp[c];
          gsum[CMAX] += sl.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c <= CMAX; ++c) gsum[c] = S.acc[lane][c];
      }
      bool nz = false;
#pragma unroll
      for (int c = 0; c <= CMAX; ++c) nz |= gsum[c] != 0.0f;
      if (in.det_o) {  // deterministic mode: this entry's sums at its list position
        const size_t pos = (size_t)begin + e;
        if (CMAX == 4 && g.C == 4) {
          reinterpret_cast<float4*>(in.det_f)[pos] = make_float4(gsum[0], gsum[1], gsum[2], gsum[3]);
        } else {
#pragma unroll
          for (int c = 0; c < CMAX; ++c)
            if (c < g.C) in.det_f[pos * g.C + c] = gsum[c];
        }
        in.det_o[pos] = gsum[CMAX];
      } else if (nz) {
        if (CMAX == 4 && g.C == 4) {
          atomicAdd(reinterpret_cast<float4*>(in.g_feat) + idx,
                    make_float4(gsum[0], gsum[1], gsum[2], gsum[3]));
        } else {
#pragma unroll
          for (int c = 0; c < CMAX; ++c)
            if (c < g.C) atomicAdd(in.g_feat + (size_t)idx * g.C + c, gsum[c]);
        }
        atomicAdd(in.g_op + idx, gsum[CMAX]);
      }
    }
    __syncwarp();
    idx = idx_pf;
  }
}

// ---------------------------------------------------------------- deterministic gradients
// INPC_FLAG_DETERMINISTIC_GRADS: the backward writes each entry's sums at its
// list position; the (point, position) pairs are then stably radix-sorted by
// point (single_sort.cuh's LSD kernels), so a point's entries follow in
// ascending list position (tile-major), and k_det_reduce adds them to the
// point's gradient in that fixed order -- no float atomics, the same bits on
// every run.
__global__ void __launch_bounds__(256) k_det_keys(const uint32_t* __restrict__ sorted_idx, int64_t n,
                                                  unsigned long long* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  keys[k] = sorted_idx[k];
  vals[k] = (uint32_t)k;
}

__global__ void __launch_bounds__(256) k_det_reduce(const unsigned long long* __restrict__ keys,
                                                    const uint32_t* __restrict__ pos, int64_t n, int C,
                                                    const float* __restrict__ det_f, const float* __restrict__ det_o,
                                                    float* __restrict__ g_feat, float* __restrict__ g_op) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t idx = (uint32_t)keys[k];
  if (k > 0 && (uint32_t)keys[k - 1] == idx) return;  // the first entry of the point's run sums the run
  float so = 0.0f;
  float sf[64];
  for (int c = 0; c < C; ++c) sf[c] = 0.0f;
  for (int64_t j = k; j < n && (uint32_t)keys[j] == idx; ++j) {
    const size_t p = pos[j];
    for (int c = 0; c < C; ++c) sf[c] += det_f[p * C + c];
    so += det_o[p];
  }
  for (int c = 0; c < C; ++c) g_feat[(size_t)idx * C + c] += sf[c];
  g_op[idx] += so;
}

}  // namespace inpc

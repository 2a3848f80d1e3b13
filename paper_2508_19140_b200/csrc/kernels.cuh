// kernels.cuh — the sm_100a kernels of the rasterizer hot path (H1-H8).
//
//   k_project_count  H1+H2: project, footprint, count entries per 8x8 tile
//   k_scan_tiles     H3:    exclusive scan of tile counts -> tile ranges, F_t;
//                           list of tiles too large for the in-SMEM sort
//   k_scatter        H5:    write (depth key << 32 | point index) into the
//                           tile buckets (bucket order arbitrary)
//   k_sort_big       H4+H6 for tiles over the SMEM cap: chunk sort + merge
//                           passes (cooperative, grid-synchronised)
//   k_blend_fwd      H4+H6 for the other tiles (bitonic sort of the unique
//                           64-bit keys in SMEM) fused with H7: front-to-back
//                           blend, Eq. 1, alpha clamp, early termination
//   k_blend_bwd      H8:    reverse-order backward, Eq. 2 corrected
//
// The two-stage sort of the paper (depth sort of the points, then
// a stable sort of the tile copies by tile key) is replaced by a bucket
// scatter + per-tile sort of the unique (depth, index) key: same per-tile
// lists bit for bit, a fraction of the sort traffic.
#pragma once
#include <cooperative_groups.h>

#include "raster_math.cuh"

namespace inpc {

constexpr int kBlendThreads = 64;    // one thread per pixel of an 8x8 tile
constexpr int kSmemSortCap = 1024;   // tiles above this go through k_sort_big
constexpr int kBigChunk = 2048;      // chunk of k_sort_big's SMEM sort
constexpr int kBigThreads = 512;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;

// ---------------------------------------------------------------- H1 + H2
template <int MODE>
__global__ void __launch_bounds__(256) k_project_count(DevCam cam, DevCfg g, const float* __restrict__ xyz,
                                                       int64_t N, uint32_t* __restrict__ tile_count,
                                                       uint32_t* __restrict__ dbg_key,
                                                       uint32_t* __restrict__ dbg_tiles) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  Proj p;
  Foot f;
  bool vis = false, ok = false;
  {
    float X = __ldg(xyz + 3 * i), Y = __ldg(xyz + 3 * i + 1), Z = __ldg(xyz + 3 * i + 2);
    vis = project_point(cam, X, Y, Z, p);
    if (vis) ok = MODE == 0 ? foot_bilinear(g, p, f) : foot_gauss(cam, g, p, f);
  }
  if (dbg_key) {
    dbg_key[i] = vis ? __float_as_uint(p.zc) : 0xFFFFFFFFu;
    dbg_tiles[i] = ok ? (uint32_t)((f.xhi / kTile - f.xlo / kTile + 1) * (f.yhi / kTile - f.ylo / kTile + 1))
                      : 0u;
  }
  if (!ok) return;
  int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
  int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
  for (int ty = ty_lo; ty <= ty_hi; ++ty)
    for (int tx = tx_lo; tx <= tx_hi; ++tx) atomicAdd(tile_count + (size_t)ty * g.tiles_x + tx, 1u);
}

// ---------------------------------------------------------------- H3
// Block-wide exclusive scan of one value per thread (kScanThreads threads).
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t* warp_tot, uint32_t& total) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < (kScanThreads / 32) ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_tot[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  uint32_t base = wid ? warp_tot[wid - 1] : 0u;
  total = warp_tot[kScanThreads / 32 - 1];
  __syncthreads();
  return base + x - v;
}

// Scalars shared between kernels of one view (device memory).
struct ViewScalars {
  uint32_t Ft;        // total tile entries
  uint32_t num_big;   // tiles with more than kSmemSortCap entries
  uint32_t max_big;   // largest of them
  uint32_t pad;
};

__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(
    int T, const uint32_t* __restrict__ count, uint32_t* __restrict__ ranges,
    uint32_t* __restrict__ cursor, uint32_t* __restrict__ big_tiles, uint32_t* __restrict__ big_elem,
    uint32_t* __restrict__ big_chunk, ViewScalars* sc) {
  __shared__ uint32_t wt[32];
  uint32_t carry = 0, carry_big = 0, carry_be = 0, carry_bc = 0, maxbig = 0;
  for (int base = 0; base < T; base += kScanThreads * kScanItems) {
    int i0 = base + threadIdx.x * kScanItems;
    uint32_t c[kScanItems];
    uint32_t s = 0, nb = 0, be = 0, bc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      c[k] = (i0 + k < T) ? count[i0 + k] : 0u;
      s += c[k];
      if (c[k] > (uint32_t)kSmemSortCap) {
        nb++;
        be += c[k];
        bc += (c[k] + kBigChunk - 1) / kBigChunk;
        maxbig = max(maxbig, c[k]);
      }
    }
    uint32_t tot, tot_nb, tot_be, tot_bc;
    uint32_t off = block_exscan(s, wt, tot) + carry;
    uint32_t off_nb = block_exscan(nb, wt, tot_nb) + carry_big;
    uint32_t off_be = block_exscan(be, wt, tot_be) + carry_be;
    uint32_t off_bc = block_exscan(bc, wt, tot_bc) + carry_bc;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      if (i0 + k < T) {
        ranges[i0 + k] = off;
        cursor[i0 + k] = off;
        if (c[k] > (uint32_t)kSmemSortCap) {
          big_tiles[off_nb] = i0 + k;
          big_elem[off_nb] = off_be;
          big_chunk[off_nb] = off_bc;
          off_nb++;
          off_be += c[k];
          off_bc += (c[k] + kBigChunk - 1) / kBigChunk;
        }
      }
      off += c[k];
    }
    carry += tot;
    carry_big += tot_nb;
    carry_be += tot_be;
    carry_bc += tot_bc;
  }
  // max over threads
  for (int o = 16; o > 0; o >>= 1) maxbig = max(maxbig, __shfl_xor_sync(0xffffffffu, maxbig, o));
  __shared__ uint32_t smax;
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicMax(&smax, maxbig);
  __syncthreads();
  if (threadIdx.x == 0) {
    ranges[T] = carry;
    big_elem[carry_big] = carry_be;
    big_chunk[carry_big] = carry_bc;
    sc->Ft = carry;
    sc->num_big = carry_big;
    sc->max_big = smax;
  }
}

// ---------------------------------------------------------------- H5
template <int MODE>
__global__ void __launch_bounds__(256) k_scatter(DevCam cam, DevCfg g, const float* __restrict__ xyz,
                                                 int64_t N, uint32_t* __restrict__ cursor,
                                                 unsigned long long* __restrict__ entries,
                                                 uint64_t cap, uint32_t* __restrict__ overflow) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  Proj p;
  Foot f;
  if (!point_foot<MODE>(cam, g, xyz, i, p, f)) return;
  unsigned long long kv = ((unsigned long long)__float_as_uint(p.zc) << 32) | (uint32_t)i;
  int ty_lo = max(f.ylo / kTile, g.ty0), ty_hi = min(f.yhi / kTile, g.ty1 - 1);
  int tx_lo = f.xlo / kTile, tx_hi = f.xhi / kTile;
  for (int ty = ty_lo; ty <= ty_hi; ++ty)
    for (int tx = tx_lo; tx <= tx_hi; ++tx) {
      uint32_t pos = atomicAdd(cursor + (size_t)ty * g.tiles_x + tx, 1u);
      if (pos < cap) entries[pos] = kv;
      else atomicOr(overflow, 1u);
    }
}

// ---------------------------------------------------------------- sort helpers
// In-place ascending bitonic sort of np (power of two) 64-bit keys in SMEM.
__device__ __forceinline__ void smem_bitonic(unsigned long long* s, int np) {
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

// H4+H6 for big tiles: (1) sort chunks of kBigChunk keys in SMEM, (2) merge
// runs pairwise (rank by binary search; keys are unique), grid-synchronised,
// (3) write the point indices to sorted_idx.  Exits at once if no tile is big.
__global__ void __launch_bounds__(kBigThreads) k_sort_big(
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ big_tiles,
    const uint32_t* __restrict__ big_elem, const uint32_t* __restrict__ big_chunk,
    const ViewScalars* sc, unsigned long long* entries, unsigned long long* tmp,
    uint32_t* __restrict__ sorted_idx) {
  namespace cg = cooperative_groups;
  const uint32_t nb = sc->num_big;
  if (nb == 0) return;
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long s[kBigChunk];
  const uint32_t total_chunks = big_chunk[nb], total = big_elem[nb], maxn = sc->max_big;
  for (uint32_t gch = blockIdx.x; gch < total_chunks; gch += gridDim.x) {
    uint32_t j = upper_bound_u32(big_chunk, nb, gch) - 1;
    uint32_t t = big_tiles[j];
    uint32_t c = gch - big_chunk[j];
    uint32_t begin = ranges[t] + c * kBigChunk;
    uint32_t n = min((uint32_t)kBigChunk, ranges[t + 1] - begin);
    for (int k = threadIdx.x; k < kBigChunk; k += blockDim.x) s[k] = k < (int)n ? entries[begin + k] : ~0ull;
    __syncthreads();
    smem_bitonic(s, kBigChunk);
    for (int k = threadIdx.x; k < (int)n; k += blockDim.x) entries[begin + k] = s[k];
    __syncthreads();
  }
  grid.sync();
  unsigned long long* src = entries;
  unsigned long long* dst = tmp;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t L = kBigChunk; L < maxn; L <<= 1) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      uint32_t j = upper_bound_u32(big_elem, nb, e) - 1;
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
    uint32_t begin = ranges[big_tiles[j]];
    uint32_t pos = e - big_elem[j];
    sorted_idx[begin + pos] = (uint32_t)src[begin + pos];
  }
}

// ---------------------------------------------------------------- H7 / H8 shared staging
// One chunk (kBlendThreads entries) of a tile list staged in SMEM, SoA.
template <int CMAX>
struct ChunkSmem {
  int xlo[kBlendThreads], xhi[kBlendThreads], ylo[kBlendThreads], yhi[kBlendThreads];
  float pa[kBlendThreads], pb[kBlendThreads];   // bilinear fa, fb | Gaussian u, v
  float ca[kBlendThreads], cb[kBlendThreads], cc[kBlendThreads];
  float o[kBlendThreads], z[kBlendThreads];
  float f[kBlendThreads][CMAX];
};

template <int MODE, int CMAX>
__device__ __forceinline__ void stage_entry(ChunkSmem<CMAX>& cs, int slot, const DevCam& cam,
                                            const DevCfg& g, const float* __restrict__ xyz,
                                            const float* __restrict__ feat,
                                            const float* __restrict__ opacity, uint32_t idx) {
  Proj p;
  Foot f;
  bool ok = point_foot<MODE>(cam, g, xyz, idx, p, f);
  // a listed point always has a footprint; guard anyway (empty rectangle)
  if (!ok) {
    f.xlo = 1;
    f.xhi = 0;
    f.ylo = 1;
    f.yhi = 0;
  }
  cs.xlo[slot] = f.xlo;
  cs.xhi[slot] = f.xhi;
  cs.ylo[slot] = f.ylo;
  cs.yhi[slot] = f.yhi;
  if (MODE == 0) {
    cs.pa[slot] = f.fa;
    cs.pb[slot] = f.fb;
    cs.ca[slot] = __int_as_float(f.x0);
    cs.cb[slot] = __int_as_float(f.y0);
  } else {
    cs.pa[slot] = p.u;
    cs.pb[slot] = p.v;
    cs.ca[slot] = f.ca;
    cs.cb[slot] = f.cb;
    cs.cc[slot] = f.cc;
  }
  cs.o[slot] = __ldg(opacity + idx);
  cs.z[slot] = p.zc;
  if (CMAX == 4 && g.C == 4) {
    float4 v = __ldg(reinterpret_cast<const float4*>(feat) + idx);
    cs.f[slot][0] = v.x;
    cs.f[slot][1] = v.y;
    cs.f[slot][2] = v.z;
    cs.f[slot][3] = v.w;
  } else {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) cs.f[slot][c] = __ldg(feat + (size_t)idx * g.C + c);
  }
}

// Weight of the staged entry e at pixel (px, py); false if not a fragment.
template <int MODE, int CMAX>
__device__ __forceinline__ bool entry_weight(const ChunkSmem<CMAX>& cs, int e, int px, int py,
                                             float& w) {
  if (px < cs.xlo[e] || px > cs.xhi[e] || py < cs.ylo[e] || py > cs.yhi[e]) return false;
  if (MODE == 0) {
    int dx = px - __float_as_int(cs.ca[e]), dy = py - __float_as_int(cs.cb[e]);
    float wx = dx ? cs.pa[e] : __fsub_rn(1.0f, cs.pa[e]);
    float wy = dy ? cs.pb[e] : __fsub_rn(1.0f, cs.pb[e]);
    w = __fmul_rn(wx, wy);
    return true;
  } else {
    float q = gauss_q(cs.ca[e], cs.cb[e], cs.cc[e], cs.pa[e], cs.pb[e], px, py);
    if (!(q <= 9.0f)) return false;
    w = expf(__fmul_rn(-0.5f, q));
    return true;
  }
}

struct BlendOut {
  float* F;          // [H,W,C]
  float* A;          // [H,W] or null
  float* D;          // [H,W] or null
  int32_t* nfrag;    // or null
  int32_t* ncontrib; // or null
  float* T_final;    // saved [H,W]
  uint32_t* last;    // saved [H,W]: list position + 1 of the last composited fragment
};

// ---------------------------------------------------------------- H4/H6 (small tiles) + H7
template <int MODE, int CMAX>
__global__ void __launch_bounds__(kBlendThreads) k_blend_fwd(
    DevCam cam, DevCfg g, const float* __restrict__ xyz, const float* __restrict__ feat,
    const float* __restrict__ opacity, const float* __restrict__ bg,
    const uint32_t* __restrict__ ranges, const unsigned long long* __restrict__ entries,
    uint32_t* __restrict__ sorted_idx, BlendOut out) {
  __shared__ unsigned long long skey[kSmemSortCap];
  __shared__ ChunkSmem<CMAX> cs;
  const int tile = g.ty0 * g.tiles_x + blockIdx.x;
  const int tx = tile % g.tiles_x, ty = tile / g.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 7), py = ty * kTile + (threadIdx.x >> 3);
  const bool inside = px < g.W && py < g.H;
  const uint32_t begin = ranges[tile], n = ranges[tile + 1] - begin;
  const bool small = n <= (uint32_t)kSmemSortCap;
  if (small && n > 0) {
    int np = 64;
    while (np < (int)n) np <<= 1;
    for (int k = threadIdx.x; k < np; k += kBlendThreads) skey[k] = k < (int)n ? entries[begin + k] : ~0ull;
    __syncthreads();
    smem_bitonic(skey, np);
    for (int k = threadIdx.x; k < (int)n; k += kBlendThreads) sorted_idx[begin + k] = (uint32_t)skey[k];
  }
  const bool count_frags = out.nfrag != nullptr;
  float T = 1.0f, Dv = 0.0f;
  float Fv[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) Fv[c] = 0.0f;
  uint32_t last = 0;
  int nfrag = 0, ncontrib = 0;
  bool done = !inside;
  for (uint32_t base = 0; base < n; base += kBlendThreads) {
    uint32_t j = base + threadIdx.x;
    __syncthreads();  // previous chunk fully consumed
    if (j < n) {
      uint32_t idx = small ? (uint32_t)skey[j] : sorted_idx[begin + j];
      stage_entry<MODE, CMAX>(cs, threadIdx.x, cam, g, xyz, feat, opacity, idx);
    }
    __syncthreads();
    const int m = min((uint32_t)kBlendThreads, n - base);
    if (inside && (!done || count_frags)) {
      for (int e = 0; e < m; ++e) {
        float w;
        if (!entry_weight<MODE, CMAX>(cs, e, px, py, w)) continue;
        nfrag++;
        if (done) continue;
        float alpha = fminf(__fmul_rn(cs.o[e], w), g.amax);
        float Tn = __fmul_rn(T, __fsub_rn(1.0f, alpha));
        if (Tn < g.tmin) {
          done = true;
          continue;
        }
        float wgt = alpha * T;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < g.C) Fv[c] += wgt * cs.f[e][c];
        Dv += wgt * cs.z[e];
        T = Tn;
        last = base + e + 1;
        ncontrib++;
      }
    }
    if (!count_frags && __syncthreads_and(done)) break;
  }
  if (!inside) return;
  const size_t pix = (size_t)py * g.W + px;
  if (bg) {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) Fv[c] += T * __ldg(bg + pix * g.C + c);
  }
  if (CMAX == 4 && g.C == 4) {
    reinterpret_cast<float4*>(out.F)[pix] = make_float4(Fv[0], Fv[1], Fv[2], Fv[3]);
  } else {
#pragma unroll
    for (int c = 0; c < CMAX; ++c)
      if (c < g.C) out.F[pix * g.C + c] = Fv[c];
  }
  if (out.A) out.A[pix] = 1.0f - T;
  if (out.D) out.D[pix] = Dv;
  out.T_final[pix] = T;
  out.last[pix] = last;
  if (out.nfrag) out.nfrag[pix] = nfrag;
  if (out.ncontrib) out.ncontrib[pix] = ncontrib;
}

// ---------------------------------------------------------------- H8
struct BwdIn {
  const float* gF;      // [H,W,C]
  const float* gA;      // [H,W] or null
  const float* gD;      // [H,W] or null
  const float* T_final; // saved
  const uint32_t* last; // saved
  float* g_feat;        // [N,C] +=
  float* g_op;          // [N] +=
};

template <int MODE, int CMAX>
__global__ void __launch_bounds__(kBlendThreads) k_blend_bwd(
    DevCam cam, DevCfg g, const float* __restrict__ xyz, const float* __restrict__ feat,
    const float* __restrict__ opacity, const float* __restrict__ bg,
    const uint32_t* __restrict__ ranges, const uint32_t* __restrict__ sorted_idx, BwdIn in) {
  __shared__ ChunkSmem<CMAX> cs;
  __shared__ float acc_f[kBlendThreads][CMAX];
  __shared__ float acc_o[kBlendThreads];
  __shared__ int touched[kBlendThreads];
  __shared__ uint32_t smax;
  const int tile = g.ty0 * g.tiles_x + blockIdx.x;
  const int tx = tile % g.tiles_x, ty = tile / g.tiles_x;
  const int px = tx * kTile + (threadIdx.x & 7), py = ty * kTile + (threadIdx.x >> 3);
  const bool inside = px < g.W && py < g.H;
  const uint32_t begin = ranges[tile];
  const size_t pix = (size_t)py * g.W + px;
  uint32_t last = 0;
  float T = 1.0f, GA = 0.0f, GD = 0.0f, RD = 0.0f, P = 1.0f;
  float G[CMAX], R[CMAX];
#pragma unroll
  for (int c = 0; c < CMAX; ++c) {
    G[c] = 0.0f;
    R[c] = 0.0f;
  }
  if (inside) {
    last = in.last[pix];
    T = in.T_final[pix];
    if (in.gA) GA = in.gA[pix];
    if (in.gD) GD = in.gD[pix];
    if (CMAX == 4 && g.C == 4) {
      float4 v = __ldg(reinterpret_cast<const float4*>(in.gF) + pix);
      G[0] = v.x; G[1] = v.y; G[2] = v.z; G[3] = v.w;
      if (bg) {
        float4 b = __ldg(reinterpret_cast<const float4*>(bg) + pix);
        R[0] = b.x; R[1] = b.y; R[2] = b.z; R[3] = b.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CMAX; ++c)
        if (c < g.C) {
          G[c] = in.gF[pix * g.C + c];
          if (bg) R[c] = bg[pix * g.C + c];
        }
    }
  }
  if (threadIdx.x == 0) smax = 0;
  __syncthreads();
  if (last) atomicMax(&smax, last);
  __syncthreads();
  const uint32_t tmax = smax;
  if (tmax == 0) return;
  for (int chunk = (int)((tmax - 1) / kBlendThreads); chunk >= 0; --chunk) {
    const uint32_t base = (uint32_t)chunk * kBlendThreads;
    const uint32_t j = base + threadIdx.x;
    uint32_t idx = 0;
    if (j < tmax) {
      idx = sorted_idx[begin + j];
      stage_entry<MODE, CMAX>(cs, threadIdx.x, cam, g, xyz, feat, opacity, idx);
#pragma unroll
      for (int c = 0; c < CMAX; ++c) acc_f[threadIdx.x][c] = 0.0f;
      acc_o[threadIdx.x] = 0.0f;
      touched[threadIdx.x] = 0;
    }
    __syncthreads();
    if (last > base) {
      const int e_hi = (int)min((uint32_t)kBlendThreads, last - base) - 1;
      for (int e = e_hi; e >= 0; --e) {
        float w;
        if (!entry_weight<MODE, CMAX>(cs, e, px, py, w)) continue;
        const float ow = __fmul_rn(cs.o[e], w);
        const float alpha = fminf(ow, g.amax);
        if ((g.flags & kFlagSkipZero) && alpha == 0.0f) continue;
        const float one_m = __fsub_rn(1.0f, alpha);
        const float Tk = __fdiv_rn(T, one_m);
        float dA = 0.0f;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < g.C) dA += G[c] * (cs.f[e][c] - R[c]);
        dA += GD * (cs.z[e] - RD) + GA * P;
        dA *= Tk;
        const float ta = Tk * alpha;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < g.C) atomicAdd(&acc_f[e][c], ta * G[c]);
        if (ow < g.amax) atomicAdd(&acc_o[e], w * dA);
        touched[e] = 1;
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < g.C) R[c] = alpha * cs.f[e][c] + one_m * R[c];
        RD = alpha * cs.z[e] + one_m * RD;
        P *= one_m;
        T = Tk;
      }
    }
    __syncthreads();
    if (j < tmax && touched[threadIdx.x]) {
      if (CMAX == 4 && g.C == 4) {
        atomicAdd(reinterpret_cast<float4*>(in.g_feat) + idx,
                  make_float4(acc_f[threadIdx.x][0], acc_f[threadIdx.x][1], acc_f[threadIdx.x][2],
                              acc_f[threadIdx.x][3]));
      } else {
#pragma unroll
        for (int c = 0; c < CMAX; ++c)
          if (c < g.C) atomicAdd(in.g_feat + (size_t)idx * g.C + c, acc_f[threadIdx.x][c]);
      }
      atomicAdd(in.g_op + idx, acc_o[threadIdx.x]);
    }
    __syncthreads();
  }
}

}  // namespace inpc

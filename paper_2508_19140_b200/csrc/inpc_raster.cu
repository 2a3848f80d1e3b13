// inpc_raster.cu — C ABI of the B200-native INPC rasterizer (include/inpc_raster.h).
//
// Host side: argument validation, the ctx's scratch arena and saved state,
// and the stream-ordered launch sequence of the kernels in kernels.cuh.
// Paper passages per step are cited in kernels.cuh and DESIGN.md §1.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only; ranges are free unless a profiler injects NVTX

#include "inpc_raster.h"
#include "kernels.cuh"
#include "single_sort.cuh"
#include "spatial_order.cuh"

using namespace inpc;

namespace {

thread_local std::string g_last_error;

// Optional caller allocator (inpc_ctx_set_allocator), made current for the
// duration of an API call by AllocScope.
struct Allocator {
  inpc_alloc_fn alloc = nullptr;
  inpc_free_fn free = nullptr;
  void* user = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
};
thread_local const Allocator* g_alloc = nullptr;

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

enum Stage : int {
  kStMemset = 0,
  kStProject,
  kStScan,
  kStScatter,
  kStSortBig,
  kStBlendFwd,
  kStBlendBwd,
  kStBin,
  kStShGrad,
  kStSingleSort,
  kStSortMid,
  kNumStages
};
const char* kStageNames[kNumStages] = {"memset",    "project_count", "scan_tiles", "scatter",
                                       "sort_big",  "blend_fwd",     "blend_bwd",  "bin_fused",
                                       "sh_grad",   "single_sort",   "sort_mid"};

// Per-view scratch of the binning (stream ordered).  Two sets, so that two
// views can be in flight on the context's two internal streams.
struct Scratch {
  Buf scat;  // unfused bilinear binning: depth key + tile block | corner mask per point
  Buf zeroed, cursor, big_tiles, huge_tiles, big_elem, big_chunk, entries, tmp, overflow, slots, agg, g_eval;
  Buf chunk_alive, mid_l2, mid_l3;  // k_sort_mid_merge size-class lists
};

struct ViewState {
  Buf ranges, sorted_idx, T_final, last, dbg_key, dbg_tiles, scalars, rec, feat_eval, order;
  uint64_t idx_cap = 0;
  bool has_order = false;  // the forward blended in `order` (big tiles first); the backward follows it
};

struct EventPair {
  cudaEvent_t a, b;
  int stage;
};

}  // namespace

struct inpc_ctx {
  int device = 0;
  int num_sms = 148;
  int big_grid = 0;
  int mid_grid = 0;       // k_sort_mid: resident CTAs (grid-stride over the big-tile list)
  bool no_mid_sort = false; // env INPC_NO_MID_SORT=1: every big tile through k_sort_big (A/B)
  bool mid_cta = false;     // env INPC_MID_SORT=cta: mid tiles through the CTA radix k_sort_mid (A/B)
  // tiles of 2049..8192 entries by the 512-thread merge sort instead of
  // k_sort_big (cfg 4: 1.755 -> 1.69 ms) for dense clouds (N >= 512 T), where
  // such tiles are likely; not for sparser ones, where the extra 70 KB-SMEM
  // launch per view costs (cfg 5: 1.9 ms per 64-view step with an empty list:
  // it cannot co-reside with the other view stream's blends).  Either way every
  // tile is sorted; env INPC_MERGE8K=0 / 1 forces the choice (A/B).
  int merge8k_env = -1;
  int midw_grid[3] = {0, 0, 0}; // k_sort_mid_merge (<= 1024, <= 2048, <= 8192 entries): resident CTAs
  // chunk bounds of a static cloud (inpc_ctx_set_chunks): used by forwards over that cloud
  const float* chunk_box = nullptr;
  const float* chunk_xyz = nullptr;
  int64_t chunk_N = 0;
  // scratch: two sets (views alternate between the two internal streams)
  static constexpr int kMaxViewStreams = 8;
  Scratch scr[kMaxViewStreams];
  cudaStream_t vstream[kMaxViewStreams] = {};  // internal non-blocking streams for multi-view calls
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxViewStreams] = {};
  int view_streams = 8;                        // env INPC_VIEW_STREAMS (1 = one stream, A/B)
  Buf det_f, det_o;  // deterministic gradients: per-entry sums at list positions
  Buf f4_rec, f4_keys, f4_vals, f4_keys2, f4_vals2, f4_hist, f4_scan, f4_misc;  // NEXT f4 baseline
  int bin_grid[3] = {0, 0, 0};  // cooperative grid of k_bin_bilinear<2,4,8>
  bool no_fused_bin = false;     // env INPC_NO_FUSED_BIN=1: separate binning kernels
  bool rec16_pref = true;        // env INPC_REC16=0: 32-byte records with packed features (A/B)
  int tile_order_mode = 1;       // env INPC_TILE_ORDER: 0 raster order; 1 big first for one-view calls; 2 / 3: also even / all views of batches (A/B)
  bool rec16 = false;            // saved state: the forward wrote 16-byte records
  uint64_t entry_cap = 0;
  std::vector<ViewState> views;
  // saved-state signature
  bool have_state = false;
  int32_t V = 0, H = 0, W = 0, C = 0, mode = 0, ty0 = 0, ty1 = 0;
  int64_t N = 0;
  unsigned flags = 0;
  float sigma = 0, dil = 0, amax = 0, tmin = 0;
  // profiling
  bool profiling = false;
  std::vector<EventPair> pending;
  std::vector<cudaEvent_t> pool;
  double stage_ms[kNumStages] = {};
  int64_t stage_launches[kNumStages] = {};
  int64_t pending_launches[kNumStages] = {};  // kernel launches behind the pending event pairs
  cudaStream_t last_stream = nullptr;
  uint32_t* host_scalars = nullptr;  // pinned
  Allocator allocator;               // caller allocator (or cudaMalloc when unset)
};



namespace {

int fail_cuda(cudaError_t e, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  g_last_error = buf;
  return INPC_CUDA;
}

#define CK(expr)                                   \
  do {                                             \
    cudaError_t e_ = (expr);                       \
    if (e_ != cudaSuccess) return fail_cuda(e_, #expr); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Grow-only buffer.  Growing synchronises the stream first (the old buffer
// may still be in use by enqueued work).
int ensure(Buf& b, size_t bytes, cudaStream_t s, bool* fresh = nullptr) {
  if (fresh) *fresh = false;
  if (bytes <= b.bytes && b.p) return INPC_OK;
  if (fresh) *fresh = true;
  size_t nb = bytes < 256 ? 256 : bytes + bytes / 4;
  if (b.p) {
    cudaStreamSynchronize(s);
    if (g_alloc && g_alloc->free) g_alloc->free(b.p, b.bytes, g_alloc->device, (void*)s, g_alloc->user);
    else cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
  }
  if (g_alloc && g_alloc->alloc) {
    b.p = g_alloc->alloc(nb, g_alloc->device, (void*)s, g_alloc->user);
    if (!b.p) {
      g_last_error = "caller allocator returned NULL";
      return INPC_OOM;
    }
  } else if (cudaMalloc(&b.p, nb) != cudaSuccess) {
    cudaGetLastError();
    g_last_error = "cudaMalloc failed";
    return INPC_OOM;
  }
  b.bytes = nb;
  return INPC_OK;
}

void free_buf(Buf& b) {
  if (b.p) {
    if (g_alloc && g_alloc->free) g_alloc->free(b.p, b.bytes, g_alloc->device, nullptr, g_alloc->user);
    else cudaFree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
}

struct AllocScope {
  const Allocator* prev;
  explicit AllocScope(inpc_ctx* c) : prev(g_alloc) { g_alloc = c->allocator.alloc ? &c->allocator : nullptr; }
  ~AllocScope() { g_alloc = prev; }
};

void release_all(inpc_ctx* c) {
  for (Scratch& x : c->scr)
    for (Buf* b : {&x.mid_l2, &x.mid_l3, &x.chunk_alive, &x.scat, &x.zeroed, &x.cursor, &x.big_tiles, &x.huge_tiles, &x.big_elem,
                   &x.big_chunk, &x.entries, &x.slots, &x.agg, &x.g_eval, &x.tmp, &x.overflow})
      free_buf(*b);
  for (Buf* b : {&c->det_f, &c->det_o, &c->f4_rec, &c->f4_keys, &c->f4_vals, &c->f4_keys2, &c->f4_vals2, &c->f4_hist, &c->f4_scan,
                 &c->f4_misc})
    free_buf(*b);
  for (auto& v : c->views)
    for (Buf* b : {&v.ranges, &v.sorted_idx, &v.T_final, &v.last, &v.dbg_key, &v.dbg_tiles, &v.scalars,
                   &v.rec, &v.feat_eval})
      free_buf(*b);
  c->views.clear();
  c->have_state = false;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaEvent_t get_event(inpc_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// NVTX range for the lifetime of a scope (API calls, views, stages)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct StageTimer {
  inpc_ctx* c;
  cudaStream_t s;
  EventPair ep{};
  bool on;
  NvtxRange nv;
  StageTimer(inpc_ctx* ctx, cudaStream_t st, int stage, int launches)
      : c(ctx), s(st), on(ctx->profiling), nv(kStageNames[stage]) {
    c->stage_launches[stage] += launches;
    if (!on) return;
    c->pending_launches[stage] += launches;
    ep.a = get_event(c);
    ep.b = get_event(c);
    ep.stage = stage;
    cudaEventRecord(ep.a, s);
  }
  ~StageTimer() {
    if (!on) return;
    cudaEventRecord(ep.b, s);
    c->pending.push_back(ep);
  }
};

int validate_cfg(const inpc_raster_cfg* cfg, const inpc_camera* cams, int32_t V) {
  if (!cfg || !cams || V <= 0) return INPC_INVALID_ARG;
  if (cfg->H <= 0 || cfg->W <= 0 || cfg->H > 32768 || cfg->W > 32768) return INPC_INVALID_ARG;
  if (cfg->C <= 0) return INPC_INVALID_ARG;
  if (cfg->C > 64) return INPC_UNSUPPORTED;
  if (cfg->splat_mode != INPC_SPLAT_BILINEAR && cfg->splat_mode != INPC_SPLAT_GAUSSIAN)
    return INPC_INVALID_ARG;
  if (!(cfg->alpha_max > 0.0f && cfg->alpha_max < 1.0f)) return INPC_INVALID_ARG;
  if (!(cfg->t_min >= 0.0f && cfg->t_min < 1.0f)) return INPC_INVALID_ARG;
  if (cfg->splat_mode == INPC_SPLAT_GAUSSIAN) {
    if (!(cfg->dilation >= 0.0f) || !isfinite(cfg->dilation)) return INPC_INVALID_ARG;
    if ((cfg->flags & INPC_FLAG_SIGMA_IS_PIXELS) && !(cfg->sigma > 0.0f)) return INPC_INVALID_ARG;
  }
  if ((cfg->flags & INPC_FLAG_ENV_BACKGROUND) && (cfg->env_h <= 0 || cfg->env_w <= 0))
    return INPC_INVALID_ARG;
  int tiles_y = (cfg->H + kTile - 1) / kTile;
  if (!(cfg->tile_y_begin == 0 && cfg->tile_y_end == 0)) {
    if (cfg->tile_y_begin < 0 || cfg->tile_y_end > tiles_y || cfg->tile_y_begin >= cfg->tile_y_end)
      return INPC_INVALID_ARG;
  }
  for (int v = 0; v < V; ++v) {
    const inpc_camera& c = cams[v];
    if (!(c.fx > 0.0f && c.fy > 0.0f && c.z_near > 0.0f) || !isfinite(c.fx) || !isfinite(c.fy) ||
        !isfinite(c.cx) || !isfinite(c.cy) || !isfinite(c.z_near))
      return INPC_INVALID_ARG;
  }
  return INPC_OK;
}

void make_dev(const inpc_raster_cfg* cfg, const inpc_camera& cam, DevCam& dc, DevCfg& g) {
  memcpy(dc.R, cam.R, sizeof dc.R);
  memcpy(dc.t, cam.t, sizeof dc.t);
  dc.fx = cam.fx;
  dc.fy = cam.fy;
  dc.cx = cam.cx;
  dc.cy = cam.cy;
  dc.z_near = cam.z_near;
  for (int k = 0; k < 3; ++k)  // camera centre -R^T t
    dc.cw[k] = (float)-((double)cam.R[k] * cam.t[0] + (double)cam.R[3 + k] * cam.t[1] +
                        (double)cam.R[6 + k] * cam.t[2]);
  g.H = cfg->H;
  g.W = cfg->W;
  g.C = cfg->C;
  g.mode = cfg->splat_mode;
  g.sigma = cfg->sigma;
  g.dil = cfg->dilation;
  g.amax = cfg->alpha_max;
  g.tmin = cfg->t_min;
  g.tiles_x = (cfg->W + kTile - 1) / kTile;
  g.tiles_y = (cfg->H + kTile - 1) / kTile;
  bool band = !(cfg->tile_y_begin == 0 && cfg->tile_y_end == 0);
  g.ty0 = band ? cfg->tile_y_begin : 0;
  g.ty1 = band ? cfg->tile_y_end : g.tiles_y;
  g.flags = 0;
  if (cfg->flags & INPC_FLAG_SIGMA_IS_PIXELS) g.flags |= kFlagSigmaPx;
  if (cfg->flags & INPC_FLAG_SKIP_ZERO_ALPHA_GRAD) g.flags |= kFlagSkipZero;
  if (cfg->flags & INPC_FLAG_SH_FEATURES) g.flags |= kFlagSH;
  if (cfg->flags & INPC_FLAG_ENV_BACKGROUND) g.flags |= kFlagEnv;
  g.env_h = cfg->env_h;
  g.env_w = cfg->env_w;
}

// Upper bound of the tiles one Gaussian footprint can touch in a view (R15-
// R17), or 0 when none can be given (the caller then reads F_t back).
// The 3-sigma radius satisfies r^2 <= 9 (a + c) (lambda_max <= trace) with
// a = s^2 jx^2 (1 + xz^2) + dil, s jx <= s fx / z_near = px (z > z_near), and
// a footprint that meets the image has |fx xz| <= mx + r (mx = the larger
// distance of cx to the image edges), so r^2 <= A + B r + K r^2 with
//   A = 9 (px^2 (1 + mx^2/fx^2) + py^2 (1 + my^2/fy^2) + 2 dil),
//   B = 18 (px^2 mx / fx^2 + py^2 my / fy^2),  K = 9 (px^2/fx^2 + py^2/fy^2),
// finite when K < 1 (s well below z_near / 3: the paper's auto sigma gives
// K ~ 1e-4).  SIGMA_IS_PIXELS: r = 3 sqrt(sigma^2 + dil) exactly.  A span of
// 2r pixels covers at most floor(2r / 8) + 2 tile columns.
uint64_t gauss_tiles_bound(const inpc_raster_cfg* cfg, const inpc_camera& cam, int band_rows, int tiles_x) {
  double r;
  const double dil = cfg->dilation;
  if (cfg->flags & INPC_FLAG_SIGMA_IS_PIXELS) {
    r = 3.0 * sqrt((double)cfg->sigma * cfg->sigma + dil);
  } else {
    const double fx = cam.fx, fy = cam.fy;
    const double sg = cfg->sigma > 0.0f ? (double)cfg->sigma : 5.0 * cam.z_near / (fx > fy ? fx : fy);
    const double px = sg * fx / cam.z_near, py = sg * fy / cam.z_near;
    const double mx = fmax(fabs((double)cam.cx), fabs((double)cfg->W - cam.cx));
    const double my = fmax(fabs((double)cam.cy), fabs((double)cfg->H - cam.cy));
    const double K = 9.0 * (px * px / (fx * fx) + py * py / (fy * fy));
    if (!(K < 0.5)) return 0;
    const double A = 9.0 * (px * px * (1.0 + mx * mx / (fx * fx)) + py * py * (1.0 + my * my / (fy * fy)) + 2.0 * dil);
    const double B = 18.0 * (px * px * mx / (fx * fx) + py * py * my / (fy * fy));
    r = (B + sqrt(B * B + 4.0 * (1.0 - K) * A)) / (2.0 * (1.0 - K));
  }
  if (!isfinite(r)) return 0;
  r = r * 1.01 + 1.0;  // fp32 rounding of the kernel's covariance, conic and radius
  const double span = floor(2.0 * r / kTile) + 2.0;
  const uint64_t tx = (uint64_t)fmin(span, (double)tiles_x), ty = (uint64_t)fmin(span, (double)band_rows);
  return tx * ty;
}

int cmax_for(int C) { return C <= 4 ? 4 : C <= 8 ? 8 : C <= 16 ? 16 : C <= 32 ? 32 : 64; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <int MODE, int CMAX, bool COUNT, int WPB, bool PF>
void launch_blend_fwd_w(int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                        const PointRec* rec, const float* feat, bool packed, const float* bg,
                        const uint32_t* ranges, const unsigned long long* entries,
                        uint32_t* sorted_idx, const BlendOut& o) {
  const size_t smem = WPB * sizeof(FwdSmem<CMAX, PF>);
  static bool once = (set_smem(k_blend_fwd<MODE, CMAX, COUNT, WPB, PF>, smem), true);
  (void)once;
  const int grid = (band_tiles + WPB - 1) / WPB;
  k_blend_fwd<MODE, CMAX, COUNT, WPB, PF><<<grid, WPB * 32, smem, s>>>(
      dc, g, band_tiles, rec, feat, packed, bg, ranges, entries, sorted_idx, o);
}

int env_wpb(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : kWarpsPerBlock;
}

// record prefetch in the forward (PF) below this many input points per tile
constexpr int64_t kFwdPrefetchMaxDensity = 512;

template <int MODE, int CMAX, bool COUNT>
void launch_blend_fwd_t(int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                        const PointRec* rec, const float* feat, bool packed, const float* bg,
                        const uint32_t* ranges, const unsigned long long* entries,
                        uint32_t* sorted_idx, const BlendOut& o, bool pf) {
#ifdef INPC_FAST_BUILD
  static const int w = env_wpb("INPC_WPB_FWD");
  if (w == 1) return launch_blend_fwd_w<MODE, CMAX, COUNT, 1, false>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries, sorted_idx, o);
  if (w == 2) return launch_blend_fwd_w<MODE, CMAX, COUNT, 2, false>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries, sorted_idx, o);
#endif
  if (CMAX == 4 && pf)
    launch_blend_fwd_w<MODE, CMAX, COUNT, kWarpsPerBlock, CMAX == 4>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries, sorted_idx, o);
  else
    launch_blend_fwd_w<MODE, CMAX, COUNT, kWarpsPerBlock, false>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries, sorted_idx, o);
}

template <int MODE, int CMAX>
void launch_blend_fwd(int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                      const PointRec* rec, const float* feat, bool packed, const float* bg,
                      const uint32_t* ranges, const unsigned long long* entries,
                      uint32_t* sorted_idx, const BlendOut& o, bool pf) {
  // the debug counts (n_frag, n_contrib) need every fragment visited
  if (o.nfrag || o.ncontrib)
    launch_blend_fwd_t<MODE, CMAX, true>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries,
                                         sorted_idx, o, pf);
  else
    launch_blend_fwd_t<MODE, CMAX, false>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, entries,
                                          sorted_idx, o, pf);
}

template <int MODE, int CMAX, int WPB>
void launch_blend_bwd_w(int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                        const PointRec* rec, const float* feat, bool packed, const float* bg,
                        const uint32_t* ranges, const uint32_t* sorted_idx, const BwdIn& in) {
  const size_t smem = WPB * sizeof(BwdSmem<MODE, CMAX>);
  static bool once = (set_smem(k_blend_bwd<MODE, CMAX, WPB>, smem), true);
  (void)once;
  const int grid = (band_tiles + WPB - 1) / WPB;
  k_blend_bwd<MODE, CMAX, WPB><<<grid, WPB * 32, smem, s>>>(dc, g, band_tiles, rec, feat, packed,
                                                            bg, ranges, sorted_idx, in);
}

template <int MODE, int CMAX>
void launch_blend_bwd(int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                      const PointRec* rec, const float* feat, bool packed, const float* bg,
                      const uint32_t* ranges, const uint32_t* sorted_idx, const BwdIn& in) {
#ifdef INPC_FAST_BUILD
  static const int w = env_wpb("INPC_WPB_BWD");
  if (w == 1) return launch_blend_bwd_w<MODE, CMAX, 1>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, sorted_idx, in);
  if (w == 2) return launch_blend_bwd_w<MODE, CMAX, 2>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, sorted_idx, in);
#endif
  launch_blend_bwd_w<MODE, CMAX, kWarpsPerBlock>(band_tiles, s, dc, g, rec, feat, packed, bg, ranges, sorted_idx, in);
}

template <int MODE>
void dispatch_blend_fwd(int cmax, int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                        const PointRec* xyz, const float* feat, bool op, const float* bg,
                        const uint32_t* ranges, const unsigned long long* entries,
                        uint32_t* sorted_idx, const BlendOut& o, bool pf) {
  switch (cmax) {
    case 4: launch_blend_fwd<MODE, 4>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
#ifndef INPC_FAST_BUILD  // diagnostics build: C <= 4 kernels only
    case 8: launch_blend_fwd<MODE, 8>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
    case 16: launch_blend_fwd<MODE, 16>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
    case 32: launch_blend_fwd<MODE, 32>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
    default: launch_blend_fwd<MODE, 64>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
#else
    default: launch_blend_fwd<MODE, 4>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, entries, sorted_idx, o, pf); break;
#endif
  }
}

template <int MODE>
void dispatch_blend_bwd(int cmax, int band_tiles, cudaStream_t s, const DevCam& dc, const DevCfg& g,
                        const PointRec* xyz, const float* feat, bool op, const float* bg,
                        const uint32_t* ranges, const uint32_t* sorted_idx, const BwdIn& in) {
  switch (cmax) {
    case 4: launch_blend_bwd<MODE, 4>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
#ifndef INPC_FAST_BUILD  // diagnostics build: C <= 4 kernels only
    case 8: launch_blend_bwd<MODE, 8>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
    case 16: launch_blend_bwd<MODE, 16>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
    case 32: launch_blend_bwd<MODE, 32>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
    default: launch_blend_bwd<MODE, 64>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
#else
    default: launch_blend_bwd<MODE, 4>(band_tiles, s, dc, g, xyz, feat, op, bg, ranges, sorted_idx, in); break;
#endif
  }
}

}  // namespace

// Stable LSD radix sort of n (key, value) pairs by the low `bits` key bits
// on stream s, in the ctx's f4 buffers (keys must already be in f4_keys,
// values in f4_vals); returns the buffers holding the sorted pairs.
int radix_pairs(inpc_ctx* c, int64_t n, int bits, cudaStream_t s, unsigned long long** keys_out,
                uint32_t** vals_out) {
  const int tiles = (int)((n + kRxTile - 1) / kRxTile);
  const int64_t hist_n = (int64_t)256 * tiles;
  const int scan_blocks = (int)((hist_n + kScanTile - 1) / kScanTile);
  bool fresh = false;
  int st;
  if ((st = ensure(c->f4_keys2, (size_t)(n > 0 ? n : 1) * 8, s))) return st;
  if ((st = ensure(c->f4_vals2, (size_t)(n > 0 ? n : 1) * 4, s))) return st;
  if ((st = ensure(c->f4_hist, (size_t)(hist_n > 0 ? hist_n : 1) * 4, s))) return st;
  if ((st = ensure(c->f4_scan, (size_t)scan_blocks * 8 + sizeof(ScanCtl) + 16, s, &fresh))) return st;
  if (fresh) CK(cudaMemsetAsync(c->f4_scan.p, 0, c->f4_scan.bytes, s));
  unsigned long long* state = (unsigned long long*)c->f4_scan.p;
  ScanCtl* ctl = (ScanCtl*)(state + scan_blocks);
  unsigned long long* ka = (unsigned long long*)c->f4_keys.p;
  unsigned long long* kb = (unsigned long long*)c->f4_keys2.p;
  uint32_t* va = (uint32_t*)c->f4_vals.p;
  uint32_t* vb = (uint32_t*)c->f4_vals2.p;
  const int rblocks = (tiles + kRxWarps - 1) / kRxWarps;
  for (int q = 0; n > 0 && q * 8 < bits; ++q) {
    k_rx_hist<<<rblocks, kRxWarps * 32, 0, s>>>(ka, n, 8 * q, tiles, (uint32_t*)c->f4_hist.p);
    k_scan_u32<<<scan_blocks, kScanThreads, 0, s>>>(hist_n, (uint32_t*)c->f4_hist.p, state, ctl);
    k_rx_scatter<<<rblocks, kRxWarps * 32, 0, s>>>(ka, va, n, 8 * q, tiles, (const uint32_t*)c->f4_hist.p, kb, vb);
    unsigned long long* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  CK(cudaGetLastError());
  *keys_out = ka;
  *vals_out = va;
  return INPC_OK;
}

extern "C" {

const char* inpc_version(void) { return "inpc_raster 0.1 sm_100a"; }

const char* inpc_status_string(int status) {
  switch (status) {
    case INPC_OK: return "ok";
    case INPC_INVALID_ARG: return "invalid argument";
    case INPC_UNSUPPORTED: return "unsupported configuration";
    case INPC_KEY_OVERFLOW: return "tile/entry count exceeds 32-bit indices";
    case INPC_OOM: return "device allocation failed";
    case INPC_CUDA: return g_last_error.empty() ? "CUDA error" : g_last_error.c_str();
    case INPC_NO_STATE: return "backward without a matching forward on this context";
    default: return "unknown status";
  }
}

const char* inpc_stage_name(int32_t stage) {
  return (stage >= 0 && stage < kNumStages) ? kStageNames[stage] : nullptr;
}

int inpc_ctx_create(inpc_ctx** out, int device) {
  if (!out) return INPC_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    g_last_error = "no such CUDA device";
    return INPC_CUDA;
  }
  DeviceGuard dg(device);
  inpc_ctx* c = new inpc_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  int per_sm = 0;
  const int big_smem = kBigChunkLarge * 8 + kRadixSmemU32 * 4;
  cudaFuncSetAttribute(k_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, big_smem);
  cudaFuncSetAttribute(k_sort_big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sort_big, kBigThreadsLarge, big_smem);
  c->big_grid = c->num_sms * (per_sm > 0 ? per_sm : 1);
  {
    // k_sort_big is launched for every unfused view and mostly finds its list
    // empty: a cooperative grid of every resident CTA must wait for whole SMs
    // while the other view streams' kernels run (cfg 5: 37.4 ms per step with
    // 296 CTAs, 36.3 with 32, 36.2 with 16).  32 CTAs still sort the rare huge
    // tiles (dense clouds send their 2049-8192-entry tiles to the merge sort).
    // env INPC_BIG_GRID: CTAs, 0 = every resident CTA (A/B)
    const char* e = getenv("INPC_BIG_GRID");
    const int want = e ? atoi(e) : 32;
    if (want > 0 && want < c->big_grid) c->big_grid = want;
  }
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sort_mid, kMidThreads, 0);
  c->mid_grid = c->num_sms * (per_sm > 0 ? per_sm : 1);
  {
    const char* e = getenv("INPC_NO_MID_SORT");
    c->no_mid_sort = e && e[0] == '1';
    const char* m = getenv("INPC_MID_SORT");
    c->mid_cta = m && !strcmp(m, "cta");
    int o1 = 0, o2 = 0, o3 = 0;
    cudaFuncSetAttribute(k_sort_mid_merge<512, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)MidMerge<512, 8192>::kSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_sort_mid_merge<kMidNT1, 1024>, kMidNT1, MidMerge<kMidNT1, 1024>::kSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_sort_mid_merge<kMidNT2, 2048>, kMidNT2, MidMerge<kMidNT2, 2048>::kSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o3, k_sort_mid_merge<512, 8192>, 512, MidMerge<512, 8192>::kSmem);
    c->midw_grid[2] = c->num_sms * (o3 > 0 ? o3 : 1);
    c->midw_grid[0] = c->num_sms * (o1 > 0 ? o1 : 1);
    c->midw_grid[1] = c->num_sms * (o2 > 0 ? o2 : 1);
  }
  {
    int o2 = 0, o4 = 0, o8 = 0;
    cudaFuncSetAttribute(k_bin_bilinear<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bin_smem_bytes<2>());
    cudaFuncSetAttribute(k_bin_bilinear<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bin_smem_bytes<4>());
    cudaFuncSetAttribute(k_bin_bilinear<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bin_smem_bytes<8>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_bin_bilinear<2, false>, kBinThreads, bin_smem_bytes<2>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o4, k_bin_bilinear<4, false>, kBinThreads, bin_smem_bytes<4>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o8, k_bin_bilinear<8, false>, kBinThreads, bin_smem_bytes<8>());
    c->bin_grid[0] = c->num_sms * o2;
    c->bin_grid[1] = c->num_sms * o4;
    c->bin_grid[2] = c->num_sms * o8;
  }
  {
    const char* e = getenv("INPC_NO_FUSED_BIN");
    c->no_fused_bin = e && e[0] == '1';
    const char* m8 = getenv("INPC_MERGE8K");
    c->merge8k_env = m8 ? (m8[0] == '1' ? 1 : 0) : -1;
    const char* to = getenv("INPC_TILE_ORDER");
    c->tile_order_mode = to ? atoi(to) : 1;
    const char* r = getenv("INPC_REC16");
    c->rec16_pref = !(r && r[0] == '0');
  }
  {
    const char* e = getenv("INPC_VIEW_STREAMS");
    c->view_streams = e ? atoi(e) : 8;  // cfg 5 step: 2 / 4 / 6 / 8 streams 36.8 / 36.3 / 36.16 / 36.09 ms (round-2 end)
    if (c->view_streams < 1) c->view_streams = 1;
    if (c->view_streams > inpc_ctx::kMaxViewStreams) c->view_streams = inpc_ctx::kMaxViewStreams;
  }
  for (int k = 0; k < inpc_ctx::kMaxViewStreams; ++k) {
    cudaStreamCreateWithFlags(&c->vstream[k], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&c->ev_join[k], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  if (cudaMallocHost(&c->host_scalars, 64) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return INPC_OOM;
  }
  *out = c;
  return INPC_OK;
}

int inpc_ctx_destroy(inpc_ctx* c) {
  if (!c) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  cudaDeviceSynchronize();
  {
    AllocScope as(c);
    release_all(c);
  }
  for (auto& e : c->pending) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  for (int k = 0; k < inpc_ctx::kMaxViewStreams; ++k) {
    if (c->vstream[k]) cudaStreamDestroy(c->vstream[k]);
    if (c->ev_join[k]) cudaEventDestroy(c->ev_join[k]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->host_scalars) cudaFreeHost(c->host_scalars);
  delete c;
  return INPC_OK;
}

int inpc_ctx_set_allocator(inpc_ctx* c, inpc_alloc_fn alloc, inpc_free_fn free_fn, void* user) {
  if (!c || (!alloc) != (!free_fn)) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  cudaDeviceSynchronize();
  {
    AllocScope as(c);  // the arena goes back to whoever allocated it
    release_all(c);
  }
  c->allocator.alloc = alloc;
  c->allocator.free = free_fn;
  c->allocator.user = user;
  c->allocator.device = c->device;
  return INPC_OK;
}

int inpc_ctx_set_profiling(inpc_ctx* c, int enable) {
  if (!c) return INPC_INVALID_ARG;
  c->profiling = enable != 0;
  return INPC_OK;
}

int inpc_ctx_stage_times(inpc_ctx* c, float* ms_out, int64_t* launches_out, int32_t n,
                         int32_t* n_stages, int flags) {
  if (!c) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  const bool reset = (flags & INPC_TIMES_RESET) != 0, keep = (flags & INPC_TIMES_KEEP_EVENTS) != 0;
  for (auto& e : c->pending) {
    cudaEventSynchronize(e.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e.a, e.b);
    c->stage_ms[e.stage] += ms;
    if (keep) c->stage_launches[e.stage] += c->pending_launches[e.stage];
  }
  if (!keep) {
    for (auto& e : c->pending) {
      c->pool.push_back(e.a);
      c->pool.push_back(e.b);
    }
    c->pending.clear();
    for (int k = 0; k < kNumStages; ++k) c->pending_launches[k] = 0;
  }
  if (n_stages) *n_stages = kNumStages;
  for (int k = 0; k < n && k < kNumStages; ++k) {
    if (ms_out) ms_out[k] = (float)c->stage_ms[k];
    if (launches_out) launches_out[k] = c->stage_launches[k];
  }
  if (reset) {
    for (int k = 0; k < kNumStages; ++k) {
      c->stage_ms[k] = 0;
      c->stage_launches[k] = 0;
    }
  }
  return INPC_OK;
}

int inpc_ctx_forget_events(inpc_ctx* c) {
  if (!c) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  for (auto& e : c->pending) {
    c->pool.push_back(e.a);
    c->pool.push_back(e.b);
  }
  c->pending.clear();
  for (int k = 0; k < kNumStages; ++k) c->pending_launches[k] = 0;
  return INPC_OK;
}

int inpc_rasterize_fwd(inpc_ctx* c, const inpc_raster_cfg* cfg, const inpc_camera* cams, int32_t V,
                       const float* xyz, const float* feat, int64_t feat_view_stride,
                       const float* opacity, int64_t N, const float* bg, int64_t bg_view_stride,
                       float* out_feat, float* out_alpha, float* out_depth, int32_t* out_nfrag,
                       int32_t* out_ncontrib, void* stream) {
  if (!c) return INPC_INVALID_ARG;
  int st = validate_cfg(cfg, cams, V);
  if (st) return st;
  if (N < 0 || N > 0xFFFFFFFFll) return N < 0 ? INPC_INVALID_ARG : INPC_KEY_OVERFLOW;
  const bool sh = (cfg->flags & INPC_FLAG_SH_FEATURES) != 0;
  const bool env = (cfg->flags & INPC_FLAG_ENV_BACKGROUND) != 0;
  if (feat_view_stride != 0 && feat_view_stride != N * cfg->C * (sh ? 9 : 1)) return INPC_INVALID_ARG;
  const int64_t P = (int64_t)cfg->H * cfg->W;
  const int64_t bg_per_view = env ? (int64_t)cfg->env_h * cfg->env_w * cfg->C : P * cfg->C;
  if (bg_view_stride != 0 && bg_view_stride != bg_per_view) return INPC_INVALID_ARG;
  if (env && !bg) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  if (N > 0 && (!is_device_ptr(xyz) || !is_device_ptr(feat) || !is_device_ptr(opacity)))
    return INPC_INVALID_ARG;
  if (!is_device_ptr(out_feat)) return INPC_INVALID_ARG;
  if ((bg && !is_device_ptr(bg)) || (out_alpha && !is_device_ptr(out_alpha)) ||
      (out_depth && !is_device_ptr(out_depth)) || (out_nfrag && !is_device_ptr(out_nfrag)) ||
      (out_ncontrib && !is_device_ptr(out_ncontrib)))
    return INPC_INVALID_ARG;
  if (cfg->C == 4 && ((uintptr_t)feat % 16 || (uintptr_t)out_feat % 16 || (bg && (uintptr_t)bg % 16)))
    return INPC_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  c->last_stream = s;
  cudaGetLastError();
  AllocScope alloc_scope(c);
  NvtxRange nv_call("inpc_rasterize_fwd");

  DevCam dc;
  DevCfg g;
  make_dev(cfg, cams[0], dc, g);
  const int T = g.tiles_x * g.tiles_y;
  const int band_tiles = (g.ty1 - g.ty0) * g.tiles_x;
  const bool gauss = cfg->splat_mode == INPC_SPLAT_GAUSSIAN;
  const bool debug = (cfg->flags & INPC_FLAG_DEBUG) != 0;
  const int cmax = cmax_for(cfg->C);
  bool packed = !gauss && cfg->C == 4;  // features travel in the point record (unless rec16)

  // scratch
  const int scan_blocks = (T + kScanTile - 1) / kScanTile;
  const size_t count_bytes = ((size_t)(T + 1) * 4 + 15) / 16 * 16;
  // tile counts, look-back state and ScanCtl: zeroed once at allocation;
  // k_scan_tiles leaves them zero after every call
  const size_t zero_bytes = count_bytes + (size_t)scan_blocks * 8 + sizeof(ScanCtl);
  bool fresh = false;
  uint64_t bound = gauss ? 0 : 4ull * (uint64_t)N;  // bilinear: <= 4 tiles per point
  if (!gauss && bound >= 0xFFFFFFFFull) return INPC_KEY_OVERFLOW;
  if ((int)c->views.size() < V) c->views.resize(V);
  c->have_state = false;
  const int nblk = (int)((N + (int64_t)kPointThreads * kPPT - 1) / ((int64_t)kPointThreads * kPPT));
  // bilinear: one cooperative launch for H1-H6 when the points fit in registers
  // (measured on cfg 2 at 1080p: fused 58.5 us vs 67 us for the separate
  // kernels eagerly, and 201.5 vs 203.7 us per fwd+bwd step in a CUDA graph)
  int fused_kp = 0, fused_grid = 0;
  if (!gauss && !sh && N > 0 && !c->no_fused_bin && T < (1 << 28)) {  // tile base + corner mask in 32 bits
    const int kps[3] = {2, 4, 8};
    for (int q = 0; q < 3; ++q)
      if (c->bin_grid[q] > 0 && N <= (int64_t)kps[q] * c->bin_grid[q] * kBinThreads) {
        fused_kp = kps[q];
        fused_grid = c->bin_grid[q];
        break;
      }
  }
  const bool merge8k = c->merge8k_env >= 0 ? c->merge8k_env == 1 : N >= 512 * (int64_t)T;
  // unfused bilinear binning: 16-byte records {u, v, z, o}, the blends read
  // the features from feat (measured on cfg 5: see DESIGN.md)
  const bool rec16 = c->rec16_pref && !gauss && !sh && !debug && !fused_kp && N > 0 && T < (1 << 28);
  // one-view bilinear calls over the whole image (unfused binning): the scan
  // also writes a tile order for the blends with the big tiles first, so the
  // long tiles do not start last (cfg 4: 1.695 -> 1.657 ms).  Not for view
  // batches, whose two view streams already fill each other's kernel tails
  // (cfg 5 per-kernel times -6 %, but the overlapped step +2 %), nor Gaussian
  // (cfg 3 +2 %).
  const bool use_order = c->tile_order_mode > 0 && (V == 1 || c->tile_order_mode >= 2) && !gauss && !fused_kp &&
                         g.ty0 == 0 && g.ty1 == g.tiles_y;
  if (rec16) packed = false;
  // entry capacity per view: bilinear 4N; Gaussian a static bound when it
  // fits a quarter of the free memory (sync-free), else F_t read back per view
  std::vector<uint64_t> need_v(V, bound);
  bool sync_views = false;
  if (gauss) {
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
      cudaGetLastError();
      free_b = 0;
    }
    for (int v = 0; v < V; ++v) {
      DevCam dv;
      DevCfg gv;
      make_dev(cfg, cams[v], dv, gv);
      const uint64_t per_pt = gauss_tiles_bound(cfg, cams[v], gv.ty1 - gv.ty0, gv.tiles_x);
      const uint64_t ub = per_pt * (uint64_t)N;
      const bool have = c->views[v].idx_cap >= ub;  // already sized for the bound
      if (per_pt && ub < 0xFFFFFFFFull && (have || ub * 20ull <= (uint64_t)(free_b / 4))) need_v[v] = ub;
      else sync_views = true;
    }
  }
  // views alternate between the two internal streams (fork / join on the
  // caller's stream, graph-capturable): one view's latency-bound kernels and
  // kernel tails overlap the other's; not while profiling (per-stage event
  // times stay per kernel), not with the per-view F_t read-back
  const int nsets = (V > 1 && N > 0 && !sync_views && !c->profiling) ? (V < c->view_streams ? V : c->view_streams) : 1;
  const bool fork = nsets > 1;
  uint64_t need_max = 1;
  for (int v = 0; v < V; ++v) need_max = need_v[v] > need_max ? need_v[v] : need_max;
  for (int k = 0; k < nsets; ++k) {
    Scratch& X = c->scr[k];
    if ((st = ensure(X.zeroed, zero_bytes, s, &fresh))) return st;
    if (fresh) CK(cudaMemsetAsync(X.zeroed.p, 0, X.zeroed.bytes, s));
    if ((st = ensure(X.cursor, (size_t)(T + 1) * 4, s))) return st;
    if (!gauss && (st = ensure(X.slots, (size_t)(N > 0 ? N : 1) * 16, s))) return st;
    if ((st = ensure(X.big_tiles, (size_t)(T + 1) * 4, s))) return st;
    if ((st = ensure(X.huge_tiles, (size_t)(T + 1) * 4, s))) return st;
    if ((st = ensure(X.mid_l2, (size_t)(T + 1) * 4, s))) return st;
    if ((st = ensure(X.mid_l3, (size_t)(T + 1) * 4, s))) return st;
    if ((st = ensure(X.big_elem, (size_t)(T + 2) * 4, s))) return st;
    if ((st = ensure(X.big_chunk, (size_t)(T + 2) * 4, s))) return st;
    // [0] Gaussian overflow flag, [6] k_sort_mid / merge done counters [6..8]
    if ((st = ensure(X.overflow, 64, s, &fresh))) return st;
    if (fresh) CK(cudaMemsetAsync(X.overflow.p, 0, X.overflow.bytes, s));
    if (!sync_views) {
      if ((st = ensure(X.entries, (size_t)need_max * 8, s))) return st;
      if ((st = ensure(X.tmp, (size_t)need_max * 8, s))) return st;
    }
    if (N > 0 && !fused_kp && !gauss && T < (1 << 28) && (st = ensure(X.scat, (size_t)N * 8, s))) return st;
    if (fused_kp && (st = ensure(X.agg, (size_t)fused_grid * 4, s))) return st;
    if ((st = ensure(X.chunk_alive, (size_t)(nblk > 0 ? nblk : 1), s))) return st;
  }
  for (int v = 0; v < V; ++v) {
    ViewState& vs = c->views[v];
    if ((st = ensure(vs.ranges, (size_t)(T + 1) * 4, s))) return st;
    if ((st = ensure(vs.T_final, (size_t)P * 4, s))) return st;
    if ((st = ensure(vs.last, (size_t)P * 4, s))) return st;
    vs.has_order = use_order && (c->tile_order_mode != 2 || V == 1 || v % 2 == 0);
    if (vs.has_order && (st = ensure(vs.order, (size_t)T * 4, s))) return st;
    if ((st = ensure(vs.scalars, sizeof(ViewScalars), s, &fresh))) return st;
    if (fresh) CK(cudaMemsetAsync(vs.scalars.p, 0, vs.scalars.bytes, s));
    if ((st = ensure(vs.rec, (size_t)(N > 0 ? N : 1) * sizeof(PointRec), s))) return st;
    if (debug && N > 0) {
      if ((st = ensure(vs.dbg_key, (size_t)N * 4, s))) return st;
      if ((st = ensure(vs.dbg_tiles, (size_t)N * 4, s))) return st;
    }
    if (sh && !packed && N > 0 && (st = ensure(vs.feat_eval, (size_t)N * cfg->C * 4, s))) return st;
    if (!sync_views) {
      if ((st = ensure(vs.sorted_idx, (size_t)(need_v[v] ? need_v[v] : 1) * 4, s))) return st;
      vs.idx_cap = need_v[v];
    }
  }
  if (fork) {
    CK(cudaEventRecord(c->ev_fork, s));
    for (int k = 0; k < nsets; ++k) CK(cudaStreamWaitEvent(c->vstream[k], c->ev_fork, 0));
  }

  for (int v = 0; v < V; ++v) {
    make_dev(cfg, cams[v], dc, g);
    if (rec16) g.flags |= kFlagRec16;
    ViewState& vs = c->views[v];
    Scratch& X = c->scr[v % nsets];
    const cudaStream_t sv = fork ? c->vstream[v % nsets] : s;
    const float* feat_v = feat + (size_t)v * feat_view_stride;
    const float* bg_v = bg ? bg + (size_t)v * bg_view_stride : nullptr;
    float* feat_out = (sh && !packed && N > 0) ? (float*)vs.feat_eval.p : nullptr;  // SH features of this view
    const float* feat_blend = feat_out ? feat_out : feat_v;
    uint32_t* tc = (uint32_t*)X.zeroed.p;
    unsigned long long* scan_state = (unsigned long long*)((char*)X.zeroed.p + count_bytes);
    ScanCtl* scan_ctl = (ScanCtl*)(scan_state + scan_blocks);
    ViewScalars* sc = (ViewScalars*)vs.scalars.p;
    uint32_t* dk = debug ? (uint32_t*)vs.dbg_key.p : nullptr;
    uint32_t* dt = debug ? (uint32_t*)vs.dbg_tiles.p : nullptr;
    if (fused_kp) {
      StageTimer tm(c, sv, kStBin, 1);
      PointRec* recp = (PointRec*)vs.rec.p;
      uint32_t* rg = (uint32_t*)vs.ranges.p;
      uint32_t* ag = (uint32_t*)X.agg.p;
      uint32_t* bt = (uint32_t*)X.big_tiles.p;
      uint32_t* be = (uint32_t*)X.big_elem.p;
      uint32_t* bc = (uint32_t*)X.big_chunk.p;
      unsigned long long* en = (unsigned long long*)X.entries.p;
      unsigned long long* tp = (unsigned long long*)X.tmp.p;
      uint32_t* si = (uint32_t*)vs.sorted_idx.p;
      int Ti = T;
      int64_t Nn = N;
      bool pk = packed;
      void* args[] = {(void*)&dc, (void*)&g, (void*)&xyz, (void*)&opacity, (void*)&feat_v, (void*)&pk,
                      (void*)&Nn, (void*)&Ti, (void*)&recp, (void*)&tc, (void*)&rg, (void*)&ag,
                      (void*)&bt, (void*)&be, (void*)&bc, (void*)&sc, (void*)&en, (void*)&tp,
                      (void*)&si, (void*)&dk, (void*)&dt, (void*)&feat_out};
      void* fn = fused_kp == 2 ? (void*)k_bin_bilinear<2, false>
                 : fused_kp == 4 ? (void*)k_bin_bilinear<4, false>
                                 : (void*)k_bin_bilinear<8, false>;
#ifdef INPC_PHASE_TIMES
      {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbolAsync(g_bin_ts, z, sizeof(z), 0, cudaMemcpyHostToDevice, sv);
      }
#endif
      const size_t bsm = fused_kp == 2 ? bin_smem_bytes<2>() : fused_kp == 4 ? bin_smem_bytes<4>() : bin_smem_bytes<8>();
      CK(cudaLaunchCooperativeKernel(fn, fused_grid, kBinThreads, args, bsm, sv));
#ifdef INPC_PHASE_TIMES
      {
        unsigned long long ts[8];
        cudaMemcpyFromSymbolAsync(ts, g_bin_ts, sizeof(ts), 0, cudaMemcpyDeviceToHost, sv);
        cudaStreamSynchronize(sv);
        fprintf(stderr, "bin phases us: project %.1f scan %.1f scatter %.1f prefix %.1f chunks %.1f end %.1f\n",
                (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3,
                ts[4] ? (ts[4] - ts[3]) * 1e-3 : 0.0, ts[5] ? (ts[5] - ts[3]) * 1e-3 : 0.0,
                ts[7] ? (ts[7] - ts[0]) * 1e-3 : 0.0);
      }
#endif
    }
    // bilinear: compact per-point scatter data (tile block + mask in 32 bits)
    uint2* scp = (N > 0 && !fused_kp && !gauss && T < (1 << 28)) ? (uint2*)X.scat.p : nullptr;
    // chunk culling: bilinear unfused path over the cloud the bounds describe (not in
    // debug mode, whose per-point exports cover every point)
    const float* cbox = (scp && !gauss && !debug && c->chunk_box && c->chunk_xyz == xyz && c->chunk_N == N)
                            ? c->chunk_box : nullptr;
    uint8_t* calive = cbox ? (uint8_t*)X.chunk_alive.p : nullptr;
    if (N > 0 && !fused_kp) {
      StageTimer tm(c, sv, kStProject, 1);
      PointRec* recp = (PointRec*)vs.rec.p;
      uint4* slp = (uint4*)X.slots.p;
      if (gauss && sh)
        k_project_count<1, true><<<nblk, kPointThreads, 0, sv>>>(dc, g, xyz, opacity, feat_v, false, N, recp,
                                                                  tc, nullptr, dk, dt, feat_out, nullptr,
                                                                  nullptr, nullptr);
      else if (gauss)
        k_project_count<1, false><<<nblk, kPointThreads, 0, sv>>>(dc, g, xyz, opacity, feat_v, false, N, recp,
                                                                   tc, nullptr, dk, dt, feat_out, nullptr,
                                                                   nullptr, nullptr);
      else if (sh)
        k_project_count<0, true><<<nblk, kPointThreads, 0, sv>>>(dc, g, xyz, opacity, feat_v, packed, N, recp,
                                                                  tc, slp, dk, dt, feat_out, scp, cbox, calive);
      else
        k_project_count<0, false><<<nblk, kPointThreads, 0, sv>>>(dc, g, xyz, opacity, feat_v, packed, N, recp,
                                                                   tc, slp, dk, dt, feat_out, scp, cbox, calive);
      CK(cudaGetLastError());
    }
    if (!fused_kp) {
      StageTimer tm(c, sv, kStScan, 1);
      uint32_t* ht = c->no_mid_sort ? nullptr : (uint32_t*)X.huge_tiles.p;
      k_scan_tiles<<<scan_blocks, kScanThreads, 0, sv>>>(T, tc, (uint32_t*)vs.ranges.p, (uint32_t*)X.cursor.p,
                                                         (uint32_t*)X.big_tiles.p, scan_state, scan_ctl, sc, ht,
                                                         (uint32_t)(c->mid_cta || !merge8k ? kMidMax : kMergeMax),
                                                         vs.has_order ? (uint32_t*)vs.order.p : nullptr);
      CK(cudaGetLastError());
    }
    uint64_t need = need_v[v];
    if (gauss && sync_views) {  // read F_t back (a huge world sigma has no useful bound)
      CK(cudaMemcpyAsync(c->host_scalars, sc, sizeof(ViewScalars), cudaMemcpyDeviceToHost, sv));
      CK(cudaStreamSynchronize(sv));
      need = c->host_scalars[0];
      if (need >= 0xFFFFFFFFull) return INPC_KEY_OVERFLOW;
      if ((st = ensure(X.entries, (size_t)(need ? need : 1) * 8, sv))) return st;
      if ((st = ensure(X.tmp, (size_t)(need ? need : 1) * 8, sv))) return st;
      if ((st = ensure(vs.sorted_idx, (size_t)(need ? need : 1) * 4, sv))) return st;
      vs.idx_cap = need;
    }
    if (N > 0 && !fused_kp) {
      StageTimer tm(c, sv, kStScatter, 1);
      if (gauss)
        k_scatter<1><<<nblk, kPointThreads, 0, sv>>>(g, (const PointRec*)vs.rec.p, N, (uint32_t*)X.cursor.p,
                                                     (unsigned long long*)X.entries.p, need,
                                                     (uint32_t*)X.overflow.p);
      else
        k_scatter_slots<<<nblk, kPointThreads, 0, sv>>>(g, (const PointRec*)vs.rec.p, (const uint4*)X.slots.p, N,
                                                        (const uint32_t*)vs.ranges.p,
                                                        (unsigned long long*)X.entries.p, scp, calive);
      CK(cudaGetLastError());
    }
    if (N > kWarpSortCap && !fused_kp && !c->no_mid_sort) {  // tiles of 257..kMergeMax entries
      StageTimer tm(c, sv, kStSortMid, 1);
      if (c->mid_cta) {
        k_sort_mid<<<c->mid_grid, kMidThreads, 0, sv>>>((const uint32_t*)vs.ranges.p, (const uint32_t*)X.big_tiles.p,
                                                        sc, (const unsigned long long*)X.entries.p,
                                                        (uint32_t*)vs.sorted_idx.p, (uint32_t*)X.overflow.p + 6);
      } else {  // merge sort: tiles of 257..1024, 1025..2048, 2049..8192 (the last clears the list)
        const uint32_t* rp = (const uint32_t*)vs.ranges.p;
        const uint32_t* bp = (const uint32_t*)X.big_tiles.p;
        const unsigned long long* ep = (const unsigned long long*)X.entries.p;
        uint32_t* sp = (uint32_t*)vs.sorted_idx.p;
        // each size class forwards its larger tiles to the next class's list
        uint32_t* dn = (uint32_t*)X.overflow.p + 6;
        uint32_t* l2 = (uint32_t*)X.mid_l2.p;
        uint32_t* l3 = (uint32_t*)X.mid_l3.p;
        k_sort_mid_merge<kMidNT1, 1024><<<c->midw_grid[0], kMidNT1, MidMerge<kMidNT1, 1024>::kSmem, sv>>>(
            rp, bp, &sc->num_big, &sc->max_big, ep, sp, l2, &sc->num_l2, dn);
        CK(cudaGetLastError());
        k_sort_mid_merge<kMidNT2, 2048><<<c->midw_grid[1], kMidNT2, MidMerge<kMidNT2, 2048>::kSmem, sv>>>(
            rp, l2, &sc->num_l2, nullptr, ep, sp, merge8k ? l3 : nullptr, &sc->num_l3, dn + 1);
        CK(cudaGetLastError());
        if (merge8k)
          k_sort_mid_merge<512, 8192><<<c->midw_grid[2], 512, MidMerge<512, 8192>::kSmem, sv>>>(
              rp, l3, &sc->num_l3, nullptr, ep, sp, nullptr, nullptr, dn + 2);
      }
      CK(cudaGetLastError());
#ifdef INPC_PHASE_TIMES
      {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t[8];
        cudaStreamSynchronize(sv);
        cudaMemcpyFromSymbol(t, g_mid_cyc, sizeof(t));
        cudaMemcpyToSymbol(g_mid_cyc, z, sizeof(z));
        const double nt = t[6] ? (double)t[6] : 1.0;
        fprintf(stderr, "mid cta: %llu tiles, cycles/tile: list %.0f keys %.0f minmax %.0f passes %.0f fixup %.0f out %.0f\n",
                t[6], t[0] / nt, t[1] / nt, t[2] / nt, t[3] / nt, t[4] / nt, t[5] / nt);
      }
#endif
    }
    if (N > kWarpSortCap && !fused_kp) {  // a tile can only exceed the cap with > cap points
      StageTimer tm(c, sv, kStSortBig, 1);
      uint32_t min_n = c->no_mid_sort ? (uint32_t)kWarpSortCap : (uint32_t)(c->mid_cta || !merge8k ? kMidMax : kMergeMax);
      const uint32_t* r = (const uint32_t*)vs.ranges.p;
      const uint32_t* bt = (const uint32_t*)X.big_tiles.p;
      uint32_t* be = (uint32_t*)X.big_elem.p;
      uint32_t* bc = (uint32_t*)X.big_chunk.p;
      ViewScalars* scc = sc;
      unsigned long long* en = (unsigned long long*)X.entries.p;
      unsigned long long* tp = (unsigned long long*)X.tmp.p;
      uint32_t* si = (uint32_t*)vs.sorted_idx.p;
      const uint32_t* ht = (const uint32_t*)X.huge_tiles.p;
      void* args[] = {(void*)&r, (void*)&bt, (void*)&be, (void*)&bc, (void*)&scc, (void*)&en, (void*)&tp, (void*)&si,
                      (void*)&min_n, (void*)&ht};
      CK(cudaLaunchCooperativeKernel((void*)k_sort_big, c->big_grid, kBigThreadsLarge, args,
                                     (size_t)kBigChunkLarge * 8 + kRadixSmemU32 * 4, sv));
    }
    {
      StageTimer tm(c, sv, kStBlendFwd, 1);
      BlendOut o;
      o.F = out_feat + (size_t)v * P * cfg->C;
      o.A = out_alpha ? out_alpha + (size_t)v * P : nullptr;
      o.D = out_depth ? out_depth + (size_t)v * P : nullptr;
      o.nfrag = out_nfrag ? out_nfrag + (size_t)v * P : nullptr;
      o.ncontrib = out_ncontrib ? out_ncontrib + (size_t)v * P : nullptr;
      o.T_final = (float*)vs.T_final.p;
      o.last = (uint32_t*)vs.last.p;
      o.order = vs.has_order ? (const uint32_t*)vs.order.p : nullptr;
      static const int pf_env = [] {  // INPC_FWD_PF=0 / 1 forces the choice (A/B)
        const char* e = getenv("INPC_FWD_PF");
        return e ? atoi(e) : -1;
      }();
      // record prefetch: always with the 16-byte records (cfg 4: 1.613 -> 1.566 ms;
      // its 32-byte records were faster without, 514 vs 780 us in round 1), else
      // for clouds below the density bound
      const bool pf = pf_env >= 0 ? pf_env == 1 : (rec16 || N < kFwdPrefetchMaxDensity * (int64_t)T);
      if (gauss)
        dispatch_blend_fwd<1>(cmax, band_tiles, sv, dc, g, (const PointRec*)vs.rec.p, feat_blend, false, bg_v,
                              (const uint32_t*)vs.ranges.p, (const unsigned long long*)X.entries.p,
                              (uint32_t*)vs.sorted_idx.p, o, pf);
      else
        dispatch_blend_fwd<0>(cmax, band_tiles, sv, dc, g, (const PointRec*)vs.rec.p, feat_blend, packed, bg_v,
                              (const uint32_t*)vs.ranges.p, (const unsigned long long*)X.entries.p,
                              (uint32_t*)vs.sorted_idx.p, o, pf);
      CK(cudaGetLastError());
    }
  }
  if (fork) {
    for (int k = 0; k < nsets; ++k) {
      CK(cudaEventRecord(c->ev_join[k], c->vstream[k]));
      CK(cudaStreamWaitEvent(s, c->ev_join[k], 0));
    }
  }
  if (gauss && debug) {  // assertion of the capacity bound (gauss_tiles_bound): the scatter flags any dropped entry
    for (int k = 0; k < nsets; ++k) {
      uint32_t flag = 0;
      CK(cudaMemcpyAsync(&flag, c->scr[k].overflow.p, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (flag) {
        CK(cudaMemsetAsync(c->scr[k].overflow.p, 0, 4, s));
        g_last_error = "Gaussian fragment capacity exceeded (entries dropped)";
        return INPC_KEY_OVERFLOW;
      }
    }
  }
  c->have_state = true;
  c->rec16 = rec16;
  c->V = V;
  c->N = N;
  c->H = cfg->H;
  c->W = cfg->W;
  c->C = cfg->C;
  c->mode = cfg->splat_mode;
  c->ty0 = g.ty0;
  c->ty1 = g.ty1;
  c->flags = cfg->flags;
  c->sigma = cfg->sigma;
  c->dil = cfg->dilation;
  c->amax = cfg->alpha_max;
  c->tmin = cfg->t_min;
  return INPC_OK;
}

int inpc_rasterize_bwd(inpc_ctx* c, const inpc_raster_cfg* cfg, const inpc_camera* cams, int32_t V,
                       const float* xyz, const float* feat, int64_t feat_view_stride,
                       const float* opacity, int64_t N, const float* bg, int64_t bg_view_stride,
                       const float* g_feat, const float* g_alpha, const float* g_depth,
                       float* g_point_feat, float* g_opacity, void* stream) {
  if (!c) return INPC_INVALID_ARG;
  int st = validate_cfg(cfg, cams, V);
  if (st) return st;
  if (N < 0) return INPC_INVALID_ARG;
  const bool sh = (cfg->flags & INPC_FLAG_SH_FEATURES) != 0;
  const bool env = (cfg->flags & INPC_FLAG_ENV_BACKGROUND) != 0;
  if (feat_view_stride != 0 && feat_view_stride != N * cfg->C * (sh ? 9 : 1)) return INPC_INVALID_ARG;
  const int64_t P = (int64_t)cfg->H * cfg->W;
  const int64_t bg_per_view = env ? (int64_t)cfg->env_h * cfg->env_w * cfg->C : P * cfg->C;
  if (bg_view_stride != 0 && bg_view_stride != bg_per_view) return INPC_INVALID_ARG;
  if (env && !bg) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  DevCam dc;
  DevCfg g;
  make_dev(cfg, cams[0], dc, g);
  if (!c->have_state || c->V != V || c->N != N || c->H != cfg->H || c->W != cfg->W ||
      c->C != cfg->C || c->mode != cfg->splat_mode || c->ty0 != g.ty0 || c->ty1 != g.ty1 ||
      c->flags != cfg->flags || c->sigma != cfg->sigma || c->dil != cfg->dilation ||
      c->amax != cfg->alpha_max || c->tmin != cfg->t_min)
    return INPC_NO_STATE;
  if (N > 0 && (!is_device_ptr(xyz) || !is_device_ptr(feat) || !is_device_ptr(opacity) ||
                !is_device_ptr(g_point_feat) || !is_device_ptr(g_opacity)))
    return INPC_INVALID_ARG;
  if (!is_device_ptr(g_feat) || (g_alpha && !is_device_ptr(g_alpha)) ||
      (g_depth && !is_device_ptr(g_depth)) || (bg && !is_device_ptr(bg)))
    return INPC_INVALID_ARG;
  if (cfg->C == 4 && ((uintptr_t)feat % 16 || (uintptr_t)g_feat % 16 ||
                      (uintptr_t)g_point_feat % 16 || (bg && (uintptr_t)bg % 16)))
    return INPC_INVALID_ARG;
  if (N == 0) return INPC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  c->last_stream = s;
  cudaGetLastError();
  AllocScope alloc_scope(c);
  NvtxRange nv_call("inpc_rasterize_bwd");
  const int band_tiles = (g.ty1 - g.ty0) * g.tiles_x;
  const bool gauss = cfg->splat_mode == INPC_SPLAT_GAUSSIAN;
  const int cmax = cmax_for(cfg->C);
  const bool packed = !gauss && cfg->C == 4 && !c->rec16;  // the forward's record layout
  const bool det = (cfg->flags & INPC_FLAG_DETERMINISTIC_GRADS) != 0;
  const int nsets = (V > 1 && !c->profiling && !det) ? (V < c->view_streams ? V : c->view_streams) : 1;
  const bool fork = nsets > 1;
  int nbits = 1;  // point-index bits for the deterministic reduction's radix passes
  while (nbits < 32 && ((int64_t)1 << nbits) < N) ++nbits;
  if (sh)
    for (int k = 0; k < nsets; ++k)
      if ((st = ensure(c->scr[k].g_eval, (size_t)N * cfg->C * 4, s))) return st;
  if (fork) {
    CK(cudaEventRecord(c->ev_fork, s));
    for (int k = 0; k < nsets; ++k) CK(cudaStreamWaitEvent(c->vstream[k], c->ev_fork, 0));
  }
  for (int v = 0; v < V; ++v) {
    make_dev(cfg, cams[v], dc, g);
    if (c->rec16) g.flags |= kFlagRec16;
    ViewState& vs = c->views[v];
    Scratch& X = c->scr[v % nsets];
    const cudaStream_t sv = fork ? c->vstream[v % nsets] : s;
    BwdIn in;
    in.gF = g_feat + (size_t)v * P * cfg->C;
    in.gA = g_alpha ? g_alpha + (size_t)v * P : nullptr;
    in.gD = g_depth ? g_depth + (size_t)v * P : nullptr;
    in.T_final = (const float*)vs.T_final.p;
    in.last = (const uint32_t*)vs.last.p;
    in.order = vs.has_order ? (const uint32_t*)vs.order.p : nullptr;
    in.g_feat = g_point_feat + (size_t)v * feat_view_stride;
    in.g_op = g_opacity;
    const float* feat_v = feat + (size_t)v * feat_view_stride;
    const float* bg_v = bg ? bg + (size_t)v * bg_view_stride : nullptr;
    if (sh) {
      // dL/df of this view into a scratch [N, C], then to the SH coefficients
      CK(cudaMemsetAsync(X.g_eval.p, 0, (size_t)N * cfg->C * 4, sv));
      in.g_feat = (float*)X.g_eval.p;
      if (!packed) feat_v = (const float*)vs.feat_eval.p;
    }
    in.det_f = nullptr;
    in.det_o = nullptr;
    int64_t Ft = 0;
    if (det) {  // per-entry sums at list positions (F_t read back: deterministic mode syncs once per view)
      CK(cudaMemcpyAsync(c->host_scalars, vs.scalars.p, sizeof(ViewScalars), cudaMemcpyDeviceToHost, sv));
      CK(cudaStreamSynchronize(sv));
      Ft = c->host_scalars[0];
      if ((st = ensure(c->det_f, (size_t)(Ft > 0 ? Ft : 1) * cfg->C * 4, sv))) return st;
      if ((st = ensure(c->det_o, (size_t)(Ft > 0 ? Ft : 1) * 4, sv))) return st;
      if (Ft > 0) {
        CK(cudaMemsetAsync(c->det_f.p, 0, (size_t)Ft * cfg->C * 4, sv));
        CK(cudaMemsetAsync(c->det_o.p, 0, (size_t)Ft * 4, sv));
      }
      in.det_f = (float*)c->det_f.p;
      in.det_o = (float*)c->det_o.p;
    }
    {
      StageTimer tm(c, sv, kStBlendBwd, 1);
      if (gauss)
        dispatch_blend_bwd<1>(cmax, band_tiles, sv, dc, g, (const PointRec*)vs.rec.p, feat_v, false, bg_v,
                              (const uint32_t*)vs.ranges.p, (const uint32_t*)vs.sorted_idx.p, in);
      else
        dispatch_blend_bwd<0>(cmax, band_tiles, sv, dc, g, (const PointRec*)vs.rec.p, feat_v, packed, bg_v,
                              (const uint32_t*)vs.ranges.p, (const uint32_t*)vs.sorted_idx.p, in);
      CK(cudaGetLastError());
    }
    if (det && Ft > 0) {  // the fixed-order reduction of the per-entry sums
      StageTimer tm(c, sv, kStBlendBwd, 3 + 3 * ((nbits + 7) / 8));
      if ((st = ensure(c->f4_keys, (size_t)Ft * 8, sv))) return st;
      if ((st = ensure(c->f4_vals, (size_t)Ft * 4, sv))) return st;
      k_det_keys<<<(unsigned)((Ft + 255) / 256), 256, 0, sv>>>((const uint32_t*)vs.sorted_idx.p, Ft,
                                                               (unsigned long long*)c->f4_keys.p,
                                                               (uint32_t*)c->f4_vals.p);
      unsigned long long* kk = nullptr;
      uint32_t* vv = nullptr;
      if ((st = radix_pairs(c, Ft, nbits, sv, &kk, &vv))) return st;
      k_det_reduce<<<(unsigned)((Ft + 255) / 256), 256, 0, sv>>>(kk, vv, Ft, cfg->C, in.det_f, in.det_o,
                                                                 in.g_feat, in.g_op);
      CK(cudaGetLastError());
    }
    if (sh) {
      StageTimer tm(c, sv, kStShGrad, 1);
      float* gsh = g_point_feat + (size_t)v * feat_view_stride;
      const unsigned nb = (unsigned)((N + kShPts - 1) / kShPts);
      if (cfg->C == 4 && ((uintptr_t)gsh & 15u) == 0)
        k_sh_grad<4><<<nb, 256, 0, sv>>>(dc, g, xyz, N, (const float*)X.g_eval.p, gsh);
      else
        k_sh_grad<0><<<nb, 256, 0, sv>>>(dc, g, xyz, N, (const float*)X.g_eval.p, gsh);
      CK(cudaGetLastError());
    }
  }
  if (fork) {
    for (int k = 0; k < nsets; ++k) {
      CK(cudaEventRecord(c->ev_join[k], c->vstream[k]));
      CK(cudaStreamWaitEvent(s, c->ev_join[k], 0));
    }
  }
  return INPC_OK;
}

int inpc_debug_export(inpc_ctx* c, int32_t view, uint32_t* depth_keys, uint32_t* tiles_touched,
                      uint32_t* tile_ranges, uint32_t* sorted_idx, int64_t sorted_cap,
                      int64_t* F_t_out, void* stream) {
  if (!c || !c->have_state || view < 0 || view >= c->V) return c ? INPC_NO_STATE : INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  ViewState& vs = c->views[view];
  const int T = ((c->W + kTile - 1) / kTile) * ((c->H + kTile - 1) / kTile);
  CK(cudaMemcpyAsync(c->host_scalars, vs.scalars.p, sizeof(ViewScalars), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t Ft = c->host_scalars[0];
  if (F_t_out) *F_t_out = Ft;
  if ((depth_keys || tiles_touched) && !(c->flags & INPC_FLAG_DEBUG)) return INPC_INVALID_ARG;
  if (depth_keys && c->N) CK(cudaMemcpyAsync(depth_keys, vs.dbg_key.p, (size_t)c->N * 4, cudaMemcpyDeviceToDevice, s));
  if (tiles_touched && c->N) CK(cudaMemcpyAsync(tiles_touched, vs.dbg_tiles.p, (size_t)c->N * 4, cudaMemcpyDeviceToDevice, s));
  if (tile_ranges) CK(cudaMemcpyAsync(tile_ranges, vs.ranges.p, (size_t)(T + 1) * 4, cudaMemcpyDeviceToDevice, s));
  if (sorted_idx) {
    int64_t n = Ft < sorted_cap ? Ft : sorted_cap;
    if (n > 0) CK(cudaMemcpyAsync(sorted_idx, vs.sorted_idx.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return INPC_OK;
}

int inpc_sort_single64(inpc_ctx* c, const inpc_raster_cfg* cfg, const inpc_camera* cam, const float* xyz,
                       const float* opacity, int64_t N, uint32_t* pixel_ranges, uint32_t* sorted_idx,
                       int64_t sorted_cap, int64_t* F_out, void* stream) {
  if (!c) return INPC_INVALID_ARG;
  int st = validate_cfg(cfg, cam, 1);
  if (st) return st;
  if (cfg->splat_mode != INPC_SPLAT_BILINEAR) return INPC_UNSUPPORTED;
  if (N < 0 || 4 * N >= 0xFFFFFFFFll) return N < 0 ? INPC_INVALID_ARG : INPC_KEY_OVERFLOW;
  DeviceGuard dg(c->device);
  if (N > 0 && (!is_device_ptr(xyz) || !is_device_ptr(opacity))) return INPC_INVALID_ARG;
  if (!is_device_ptr(pixel_ranges) || (sorted_idx && !is_device_ptr(sorted_idx))) return INPC_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  c->last_stream = s;
  cudaGetLastError();
  AllocScope alloc_scope(c);
  DevCam dc;
  DevCfg g;
  make_dev(cfg, *cam, dc, g);
  g.ty0 = 0;
  g.ty1 = g.tiles_y;
  g.flags &= ~(kFlagSH | kFlagEnv);
  const int64_t P = (int64_t)cfg->H * cfg->W;
  const int64_t n = 4 * N;
  const int tiles = (int)((n + kRxTile - 1) / kRxTile);
  const int64_t hist_n = (int64_t)256 * tiles;
  const int scan_blocks = (int)((hist_n + kScanTile - 1) / kScanTile);
  bool fresh = false;
  if ((st = ensure(c->f4_rec, (size_t)(N > 0 ? N : 1) * sizeof(PointRec), s))) return st;
  if ((st = ensure(c->f4_keys, (size_t)(n > 0 ? n : 1) * 8, s))) return st;
  if ((st = ensure(c->f4_keys2, (size_t)(n > 0 ? n : 1) * 8, s))) return st;
  if ((st = ensure(c->f4_vals, (size_t)(n > 0 ? n : 1) * 4, s))) return st;
  if ((st = ensure(c->f4_vals2, (size_t)(n > 0 ? n : 1) * 4, s))) return st;
  if ((st = ensure(c->f4_hist, (size_t)(hist_n > 0 ? hist_n : 1) * 4, s))) return st;
  if ((st = ensure(c->f4_scan, (size_t)scan_blocks * 8 + sizeof(ScanCtl) + 16, s, &fresh))) return st;
  if (fresh) CK(cudaMemsetAsync(c->f4_scan.p, 0, c->f4_scan.bytes, s));
  if ((st = ensure(c->f4_misc, 64, s))) return st;
  unsigned long long* nvalid = (unsigned long long*)c->f4_misc.p;
  CK(cudaMemsetAsync(nvalid, 0, 8, s));
  unsigned long long* state = (unsigned long long*)c->f4_scan.p;
  ScanCtl* ctl = (ScanCtl*)(state + scan_blocks);
  if (N > 0) {  // H1: the point records (not part of the timed sort)
    const int nblk = (int)((N + (int64_t)kPointThreads * kPPT - 1) / ((int64_t)kPointThreads * kPPT));
    k_project_count<0, false><<<nblk, kPointThreads, 0, s>>>(dc, g, xyz, opacity, nullptr, false, N,
                                                              (PointRec*)c->f4_rec.p, nullptr, nullptr,
                                                              nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
  }
  unsigned long long* ka = (unsigned long long*)c->f4_keys.p;
  unsigned long long* kb = (unsigned long long*)c->f4_keys2.p;
  uint32_t* va = (uint32_t*)c->f4_vals.p;
  uint32_t* vb = (uint32_t*)c->f4_vals2.p;
  {
    StageTimer tm(c, s, kStSingleSort, 0);
    if (N > 0) {
      k_emit_pixel_frags<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(g, (const PointRec*)c->f4_rec.p, N, ka, va,
                                                                      nvalid);
      int pbits = 0;
      while ((1ll << pbits) < P) ++pbits;
      const int passes = (32 + pbits + 7) / 8;  // ceil((32 + 21) / 8) = 7 at 1080p
      const int rblocks = (tiles + kRxWarps - 1) / kRxWarps;
      for (int q = 0; q < passes; ++q) {
        const int shift = 8 * q;
        k_rx_hist<<<rblocks, kRxWarps * 32, 0, s>>>(ka, n, shift, tiles, (uint32_t*)c->f4_hist.p);
        k_scan_u32<<<scan_blocks, kScanThreads, 0, s>>>(hist_n, (uint32_t*)c->f4_hist.p, state, ctl);
        k_rx_scatter<<<rblocks, kRxWarps * 32, 0, s>>>(ka, va, n, shift, tiles, (const uint32_t*)c->f4_hist.p, kb,
                                                        vb);
        c->stage_launches[kStSingleSort] += 3;
        unsigned long long* tk = ka;
        ka = kb;
        kb = tk;
        uint32_t* tv = va;
        va = vb;
        vb = tv;
      }
      c->stage_launches[kStSingleSort] += 1;
    }
    k_pixel_ranges<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(ka, n, P, pixel_ranges);
    c->stage_launches[kStSingleSort] += 1;
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(c->host_scalars, nvalid, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int64_t F = (int64_t)(*(unsigned long long*)c->host_scalars);
  if (F_out) *F_out = F;
  if (sorted_idx && F > 0)
    CK(cudaMemcpyAsync(sorted_idx, va, (size_t)(F < sorted_cap ? F : sorted_cap) * 4, cudaMemcpyDeviceToDevice, s));
  return INPC_OK;
}

int inpc_chunk_bounds(inpc_ctx* c, const float* xyz, int64_t N, float* box, void* stream) {
  if (!c || N < 0) return INPC_INVALID_ARG;
  if (N == 0) return INPC_OK;
  DeviceGuard dg(c->device);
  if (!is_device_ptr(xyz) || !is_device_ptr(box)) return INPC_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  cudaGetLastError();
  const int64_t nchunks = (N + kChunkPoints - 1) / kChunkPoints;
  k_chunk_bounds<<<(unsigned)nchunks, kPointThreads, 0, s>>>(xyz, N, box);
  CK(cudaGetLastError());
  return INPC_OK;
}

int inpc_ctx_set_chunks(inpc_ctx* c, const float* xyz, int64_t N, const float* box) {
  if (!c || N < 0) return INPC_INVALID_ARG;
  DeviceGuard dg(c->device);
  if (box && (!is_device_ptr(box) || !is_device_ptr(xyz))) return INPC_INVALID_ARG;
  c->chunk_box = box;
  c->chunk_xyz = box ? xyz : nullptr;
  c->chunk_N = box ? N : 0;
  return INPC_OK;
}

int inpc_spatial_order(inpc_ctx* c, const float* xyz, int64_t N, uint32_t* perm, void* stream) {
  if (!c || N < 0) return INPC_INVALID_ARG;
  if (N > 0xFFFFFFFFll) return INPC_KEY_OVERFLOW;
  if (N == 0) return INPC_OK;
  DeviceGuard dg(c->device);
  if (!is_device_ptr(xyz) || !is_device_ptr(perm)) return INPC_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  c->last_stream = s;
  cudaGetLastError();
  AllocScope alloc_scope(c);
  const int tiles = (int)((N + kRxTile - 1) / kRxTile);
  const int64_t hist_n = (int64_t)256 * tiles;
  const int scan_blocks = (int)((hist_n + kScanTile - 1) / kScanTile);
  bool fresh = false;
  int st;
  if ((st = ensure(c->f4_keys, (size_t)N * 8, s))) return st;
  if ((st = ensure(c->f4_keys2, (size_t)N * 8, s))) return st;
  if ((st = ensure(c->f4_vals, (size_t)N * 4, s))) return st;
  if ((st = ensure(c->f4_vals2, (size_t)N * 4, s))) return st;
  if ((st = ensure(c->f4_hist, (size_t)hist_n * 4, s))) return st;
  if ((st = ensure(c->f4_scan, (size_t)scan_blocks * 8 + sizeof(ScanCtl) + 16, s, &fresh))) return st;
  if (fresh) CK(cudaMemsetAsync(c->f4_scan.p, 0, c->f4_scan.bytes, s));
  if ((st = ensure(c->f4_misc, 64, s))) return st;
  uint32_t* box = (uint32_t*)c->f4_misc.p;
  CK(cudaMemsetAsync(box, 0xFF, 12, s));
  CK(cudaMemsetAsync(box + 3, 0, 12, s));
  unsigned long long* state = (unsigned long long*)c->f4_scan.p;
  ScanCtl* ctl = (ScanCtl*)(state + scan_blocks);
  unsigned long long* ka = (unsigned long long*)c->f4_keys.p;
  unsigned long long* kb = (unsigned long long*)c->f4_keys2.p;
  uint32_t* va = (uint32_t*)c->f4_vals.p;
  uint32_t* vb = (uint32_t*)c->f4_vals2.p;
  k_aabb<<<c->num_sms * 4, 256, 0, s>>>(xyz, N, box);
  k_morton_keys<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(xyz, N, box, ka, va);
  const int rblocks = (tiles + kRxWarps - 1) / kRxWarps;
  for (int q = 0; q < 4; ++q) {  // 30-bit codes (+ the all-ones code of non-finite points)
    k_rx_hist<<<rblocks, kRxWarps * 32, 0, s>>>(ka, N, 8 * q, tiles, (uint32_t*)c->f4_hist.p);
    k_scan_u32<<<scan_blocks, kScanThreads, 0, s>>>(hist_n, (uint32_t*)c->f4_hist.p, state, ctl);
    k_rx_scatter<<<rblocks, kRxWarps * 32, 0, s>>>(ka, va, N, 8 * q, tiles, (const uint32_t*)c->f4_hist.p, kb, vb);
    unsigned long long* tk = ka;
    ka = kb;
    kb = tk;
    uint32_t* tv = va;
    va = vb;
    vb = tv;
  }
  CK(cudaMemcpyAsync(perm, va, (size_t)N * 4, cudaMemcpyDeviceToDevice, s));
  CK(cudaGetLastError());
  return INPC_OK;
}

}  // extern "C"

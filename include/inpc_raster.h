/*
 * inpc_raster.h — C ABI of the B200-native INPC neural point rasterizer.
 *
 * The operation (PAPER.md = P, line numbers; readings R1-R25):
 *   points p_i (xyz), features f_i (C channels), opacities o_i are rendered
 *   through a pinhole camera into a feature image F in R^{H x W x C}
 *   ("fast differentiable rasterization") by
 *     - projecting each point (R1, R2, R7, R9),
 *     - splatting it as a bilinear 2x2 footprint (R3, R4)
 *       or as a small Gaussian (R15-R19),
 *     - ordering the fragments of each 8x8 tile by (depth, point index)
 *       (tiled two-stage sort; R8),
 *     - compositing front to back, Eq. 1, with alpha clamp (R5),
 *       early termination (R6) and background (R11), producing
 *       F [H,W,C], alpha A = 1 - T_final [H,W] and depth D = sum T a z [H,W] (R10),
 *   and the backward pass returns dL/df and dL/do by the corrected Eq. 2
 *   (R12, R13, R14) including alpha = 0 fragments.
 *
 * Conventions
 *   - Every array argument is CUDA DEVICE memory (cudaMalloc / torch CUDA
 *     tensor) on the ctx's device, fp32 row-major contiguous unless stated.
 *     Host pointers are rejected with INPC_INVALID_ARG.  `cams` and `cfg` are
 *     HOST structs, read during the call only.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All GPU
 *     work is enqueued on it, asynchronously; argument errors are reported
 *     synchronously before anything is enqueued.  The Gaussian-mode forward
 *     sizes its fragment buffers from a static bound of the entries per
 *     point (3-sigma radius bound from sigma, dilation, z_near and the
 *     intrinsics) when that fits a quarter of the free device memory, and
 *     is then free of host synchronisation (graph-capturable); otherwise
 *     (huge world sigma) it synchronises the stream once per view to read
 *     the entry count back.
 *   - Ownership: inputs/outputs are caller-owned and borrowed for the
 *     stream-ordered duration of the call.  The ctx owns its scratch arena
 *     and the state the forward saves for the backward (per-tile lists,
 *     T_final, last-fragment positions).  The next forward on a ctx
 *     overwrites that state.  The backward takes the inputs again; the
 *     library never retains caller pointers.
 *   - Gradient outputs ACCUMULATE (+=); the caller zeroes them.
 *   - A ctx is not thread-safe; use one ctx per (device, concurrent stream).
 *   - Return value: INPC_OK (0) or one of the INPC_* status codes.
 */
#ifndef INPC_RASTER_H
#define INPC_RASTER_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define INPC_API __attribute__((visibility("default")))
#else
#define INPC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define INPC_OK 0
#define INPC_INVALID_ARG 1   /* null required pointer, host pointer, bad sizes/params */
#define INPC_UNSUPPORTED 2   /* e.g. C > 64                                          */
#define INPC_KEY_OVERFLOW 3  /* tile count or entry count does not fit 32-bit indices */
#define INPC_OOM 4           /* device allocation failed                             */
#define INPC_CUDA 5          /* CUDA launch/runtime error (see inpc_status_string)   */
#define INPC_NO_STATE 6      /* backward without a matching forward on this ctx      */

/* ---- splat modes ---- */
#define INPC_SPLAT_BILINEAR 0 /* 2x2 bilinear splat          */
#define INPC_SPLAT_GAUSSIAN 1 /* small Gaussian                        */

/* ---- cfg.flags ---- */
#define INPC_FLAG_SIGMA_IS_PIXELS (1u << 0)      /* R15: sigma is a screen std in px */
#define INPC_FLAG_SKIP_ZERO_ALPHA_GRAD (1u << 1) /* R13: original INPC behaviour (A/B) */
#define INPC_FLAG_DEBUG (1u << 2)                /* keep per-point depth keys / tile
                                                    counts for inpc_debug_export      */
#define INPC_FLAG_SH_FEATURES (1u << 3)          /* NEXT f1: `feat` holds real SH
                                                    coefficients of degree <= 2, [N,C,9]
                                                    ([V,N,C,9] with feat_view_stride =
                                                    N*C*9); features f_c = sum_k
                                                    coeff[c][k] Y_k(d), d = unit vector
                                                    from the camera centre to the point
                                                    (R26); the backward accumulates
                                                    dL/dcoeff into g_point_feat [N,C,9] */
#define INPC_FLAG_DETERMINISTIC_GRADS (1u << 5) /* backward: no float atomics; every point's
                                                    per-entry sums added in a fixed order
                                                    (list position), same bits on every run;
                                                    syncs once per view, views not overlapped */
#define INPC_FLAG_ENV_BACKGROUND (1u << 4)       /* NEXT f2: `bg` is an
                                                    equirectangular map [env_h,env_w,C]
                                                    (bg_view_stride 0 or env_h*env_w*C);
                                                    each pixel's background is its
                                                    bilinear lookup along the pixel's
                                                    world ray (R27); not differentiated */

/* Pinhole camera (R2): x_cam = R x_world + t, R row-major 3x3;
 * u = fx x_cam/z_cam + cx, v = fy y_cam/z_cam + cy; pixel (i, j) has its
 * centre at (i + 0.5, j + 0.5).  Points with !(z_cam > z_near) are culled. */
typedef struct {
  float R[9];
  float t[3];
  float fx, fy, cx, cy; /* pixels, fx, fy > 0   */
  float z_near;         /* > 0                  */
} inpc_camera;

typedef struct {
  int32_t H, W;         /* image size, 1..32768 each                                 */
  int32_t C;            /* feature channels, 1..64 (n_omega = 4 in INPC)       */
  int32_t splat_mode;   /* INPC_SPLAT_BILINEAR or INPC_SPLAT_GAUSSIAN               */
  float sigma;          /* Gaussian: world std; <= 0 -> 5 z_near / max(fx, fy)
                           with SIGMA_IS_PIXELS: screen std in pixels (must be > 0) */
  float dilation;       /* px^2 added to the 2-D covariance; paper 0.16 */
  float alpha_max;      /* alpha clamp in (0, 1); default 0.99 (R5)                 */
  float t_min;          /* early termination threshold in [0, 1); 1e-4 (R6)         */
  int32_t tile_y_begin; /* screen band [begin, end) in 8-pixel tile rows for        */
  int32_t tile_y_end;   /*   sort-first sharding; 0, 0 = whole image                */
  uint32_t flags;       /* INPC_FLAG_*                                              */
  int32_t env_h, env_w; /* environment map size with INPC_FLAG_ENV_BACKGROUND, else 0 */
} inpc_raster_cfg;

typedef struct inpc_ctx inpc_ctx;

/* Device-memory allocator of the caller (e.g. PyTorch's caching allocator):
 * alloc returns `bytes` of device memory usable on `stream` (NULL = out of
 * memory); free releases a pointer alloc returned (stream NULL at context
 * destruction).  Without one the context uses cudaMalloc / cudaFree. */
typedef void* (*inpc_alloc_fn)(size_t bytes, int device, void* stream, void* user);
typedef void (*inpc_free_fn)(void* ptr, size_t bytes, int device, void* stream, void* user);

/* Create a context on CUDA device `device` (the caller's current device is
 * restored).  *out receives the handle. */
INPC_API int inpc_ctx_create(inpc_ctx** out, int device);
/* Free the context's arena and saved state (synchronises the device). */
INPC_API int inpc_ctx_destroy(inpc_ctx* ctx);
/* Route the context's scratch arena and saved state through a caller
 * allocator (both functions, or both NULL for cudaMalloc).  Releases the
 * current arena (and the saved forward state) first. */
INPC_API int inpc_ctx_set_allocator(inpc_ctx* ctx, inpc_alloc_fn alloc, inpc_free_fn free_fn, void* user);

/* Forward raster of V views of one point cloud.
 *   cams   [V] host cameras
 *   xyz    [N,3] positions (world)
 *   feat   [N,C] features, or [V,N,C] when feat_view_stride == N*C (R20)
 *   opacity[N] in [0,1] (values outside are used as given)
 *   bg     [V,H,W,C] background (bg_view_stride = H*W*C) or [H,W,C] shared
 *          (bg_view_stride = 0) or NULL (= 0)
 *   out_feat [V,H,W,C], out_alpha [V,H,W], out_depth [V,H,W]: written for the
 *          pixels of the band (whole image by default); NULL allowed for
 *          alpha/depth
 *   out_nfrag [V,H,W] int32 or NULL: number of fragments covering each pixel
 *          (debug; disables early exit of whole tiles)
 *   out_ncontrib [V,H,W] int32 or NULL: number of fragments composited
 *          before termination (debug)
 * N may be 0 (pure background).  Entry counts must stay < 2^32. */
INPC_API int inpc_rasterize_fwd(inpc_ctx* ctx, const inpc_raster_cfg* cfg, const inpc_camera* cams,
                       int32_t V, const float* xyz, const float* feat,
                       int64_t feat_view_stride, const float* opacity, int64_t N,
                       const float* bg, int64_t bg_view_stride, float* out_feat,
                       float* out_alpha, float* out_depth, int32_t* out_nfrag,
                       int32_t* out_ncontrib, void* stream);

/* Backward of the last forward on this ctx (same cfg, cams, V, N, pointers
 * holding the same values).
 *   g_feat [V,H,W,C] = dL/dF; g_alpha [V,H,W] or NULL; g_depth [V,H,W] or NULL
 *   g_point_feat += dL/df: [N,C] (feat_view_stride 0: summed over views) or
 *                   [V,N,C]; must be 16-byte aligned when C == 4
 *   g_opacity    += dL/do [N] (summed over views)
 * Gradients accumulate with atomics (order of fp32 sums is not fixed) unless
 * cfg.flags has INPC_FLAG_DETERMINISTIC_GRADS. */
INPC_API int inpc_rasterize_bwd(inpc_ctx* ctx, const inpc_raster_cfg* cfg, const inpc_camera* cams,
                       int32_t V, const float* xyz, const float* feat,
                       int64_t feat_view_stride, const float* opacity, int64_t N,
                       const float* bg, int64_t bg_view_stride, const float* g_feat,
                       const float* g_alpha, const float* g_depth, float* g_point_feat,
                       float* g_opacity, void* stream);

/* Copy the saved per-view state of the last forward (for bit-exact parity):
 *   depth_keys [N]    u32 float bits of z_cam, 0xFFFFFFFF = culled (needs FLAG_DEBUG)
 *   tiles_touched [N] u32 tiles listing the point (needs FLAG_DEBUG)
 *   tile_ranges [T+1] u32, T = ceil(H/8)*ceil(W/8), list of tile t at
 *                     [tile_ranges[t], tile_ranges[t+1])
 *   sorted_idx [sorted_cap] u32 point indices, per tile ordered by (depth, idx)
 *   F_t_out (host) total number of tile entries
 * Any pointer may be NULL.  Device pointers; copies are enqueued on stream. */
INPC_API int inpc_debug_export(inpc_ctx* ctx, int32_t view, uint32_t* depth_keys, uint32_t* tiles_touched,
                      uint32_t* tile_ranges, uint32_t* sorted_idx, int64_t sorted_cap,
                      int64_t* F_t_out, void* stream);

/* NEXT f4 — the original INPC ordering as an A/B baseline (P:100,
 * P:159-162): 4 fragment copies per point with 64-bit keys (pixel << 32 |
 * depth bits), one stable device-wide LSD radix sort of 8-bit digits
 * (ceil((32 + pixel bits) / 8) passes: 7 at 1080p), per-pixel ranges.
 *   cam (host) one camera; xyz [N,3], opacity [N] (device)
 *   pixel_ranges [H*W+1] u32 (device): pixel p's fragments are
 *     sorted_idx[pixel_ranges[p] .. pixel_ranges[p+1]) in (depth, index) order
 *   sorted_idx [sorted_cap] u32 (device) or NULL; F_out (host) = #fragments
 * Bilinear only (INPC_UNSUPPORTED otherwise).  Synchronises the stream once
 * (F readback).  The sort's device time is the "single_sort" profiling stage. */
INPC_API int inpc_sort_single64(inpc_ctx* ctx, const inpc_raster_cfg* cfg, const inpc_camera* cam,
                                const float* xyz, const float* opacity, int64_t N, uint32_t* pixel_ranges,
                                uint32_t* sorted_idx, int64_t sorted_cap, int64_t* F_out, void* stream);

/* One-time spatial ordering of a static cloud (not a step of the method;
 * DESIGN.md §6): perm [N] u32 (device) receives the permutation that sorts
 * the points by the 30-bit Morton code of their position on a 1024^3 grid
 * over the cloud's bounding box (stable; non-finite points last).  A caller
 * with a static cloud (the pre-extracted global cloud;
 * the shared cloud of a view batch) gathers xyz / features / opacities by
 * perm once and rasterizes the reordered cloud: point indices (and the
 * tie-break of equal depths, R8) then refer to the reordered cloud.  Spatial
 * order makes the tile-slot atomics, tile buckets, record gathers and
 * gradient atomics local (warp-aggregated, L2-resident).  xyz [N,3] device.
 * Asynchronous on stream. */
INPC_API int inpc_spatial_order(inpc_ctx* ctx, const float* xyz, int64_t N, uint32_t* perm, void* stream);

/* Chunk bounds of a static cloud: box
 * [ceil(N / 1024), 6] (device, fp32) receives, for every chunk of 1024
 * consecutive points, (xmin, ymin, zmin, xmax, ymax, zmax) over its finite
 * points (min > max when it has none).  Meant for a spatially ordered cloud
 * (inpc_spatial_order), where the chunks are compact.  Asynchronous. */
INPC_API int inpc_chunk_bounds(inpc_ctx* ctx, const float* xyz, int64_t N, float* box, void* stream);
/* Attach chunk bounds to the context (box NULL detaches).  Forwards whose
 * xyz pointer and N equal the ones given here then skip, in the bilinear
 * binning of large clouds, every chunk whose box cannot produce a footprint
 * in the view's frame or screen band (behind the near plane, or projecting
 * wholly outside the image / band): a conservative test, the rasterized
 * result is unchanged.  The caller keeps box alive and in step with the
 * cloud's contents.  Not used with INPC_FLAG_DEBUG (its per-point exports
 * cover every point). */
INPC_API int inpc_ctx_set_chunks(inpc_ctx* ctx, const float* xyz, int64_t N, const float* box);

/* Per-stage device timing (CUDA events around each stage; adds no sync to
 * the calls).  inpc_ctx_stage_times waits for the recorded events, adds
 * their elapsed milliseconds to per-stage accumulators and returns the
 * accumulated milliseconds and kernel-launch counts per stage (arrays of n).
 * flags: INPC_TIMES_RESET zeroes the accumulators after reading;
 * INPC_TIMES_KEEP_EVENTS keeps the event pairs pending, for calls captured
 * in a CUDA graph (read again after every replay; launches are counted per
 * read).  inpc_ctx_forget_events drops pending pairs (after the graph is
 * destroyed). */
#define INPC_TIMES_RESET 1
#define INPC_TIMES_KEEP_EVENTS 2
INPC_API int inpc_ctx_set_profiling(inpc_ctx* ctx, int enable);
INPC_API int inpc_ctx_stage_times(inpc_ctx* ctx, float* ms_out, int64_t* launches_out, int32_t n,
                         int32_t* n_stages, int flags);
INPC_API int inpc_ctx_forget_events(inpc_ctx* ctx);
INPC_API const char* inpc_stage_name(int32_t stage);

/* Human-readable text for a status code (for INPC_CUDA: the last CUDA error
 * seen by the library on this thread). */
INPC_API const char* inpc_status_string(int status);

/* Library version, e.g. "inpc_raster 0.1 sm_100a". */
INPC_API const char* inpc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* INPC_RASTER_H */

"""B200-native INPC neural point rasterizer — Python binding.

Argument marshalling only: every step of the hot path (projection, footprint,
tile lists, blending, backward) runs in ``libinpc_raster.so``'s sm_100a
kernels behind the C ABI of ``include/inpc_raster.h``.  PyTorch supplies
device memory, streams and autograd plumbing.  There is no CPU fallback:
importing this package raises if the library is missing.

    F, A, D = rasterize(xyz, feat, opacity, cams, H, W, mode="bilinear")

PAPER.md passages: problem statement P:73-76, rasterizer P:98-101 and
P:156-204, Eq. 1, Eq. 2 P:482-491.
"""
from __future__ import annotations

import ctypes as ct
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libinpc_raster.so")

OK, INVALID_ARG, UNSUPPORTED, KEY_OVERFLOW, OOM, CUDA_ERROR, NO_STATE = range(7)
SPLAT_BILINEAR, SPLAT_GAUSSIAN = 0, 1
FLAG_SIGMA_IS_PIXELS = 1 << 0
FLAG_SKIP_ZERO_ALPHA_GRAD = 1 << 1
FLAG_DEBUG = 1 << 2
FLAG_SH_FEATURES = 1 << 3
FLAG_ENV_BACKGROUND = 1 << 4
FLAG_DETERMINISTIC_GRADS = 1 << 5
TILE = 8

EXPORTS = ("inpc_ctx_create", "inpc_ctx_destroy", "inpc_rasterize_fwd", "inpc_rasterize_bwd",
           "inpc_debug_export", "inpc_ctx_set_profiling", "inpc_ctx_stage_times",
           "inpc_ctx_forget_events", "inpc_ctx_set_allocator", "inpc_sort_single64",
           "inpc_stage_name", "inpc_status_string", "inpc_version", "inpc_spatial_order",
           "inpc_chunk_bounds", "inpc_ctx_set_chunks")


# inpc_alloc_fn / inpc_free_fn (include/inpc_raster.h)
ALLOC_FN = ct.CFUNCTYPE(ct.c_void_p, ct.c_size_t, ct.c_int, ct.c_void_p, ct.c_void_p)
FREE_FN = ct.CFUNCTYPE(None, ct.c_void_p, ct.c_size_t, ct.c_int, ct.c_void_p, ct.c_void_p)


class RasterError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"inpc status {status}: {msg}")
        self.status = status


class Camera(ct.Structure):
    """inpc_camera: x_cam = R x + t; u = fx x/z + cx (pixel centres at +0.5)."""
    _fields_ = [("R", ct.c_float * 9), ("t", ct.c_float * 3), ("fx", ct.c_float),
                ("fy", ct.c_float), ("cx", ct.c_float), ("cy", ct.c_float),
                ("z_near", ct.c_float)]


class RasterCfg(ct.Structure):
    _fields_ = [("H", ct.c_int32), ("W", ct.c_int32), ("C", ct.c_int32),
                ("splat_mode", ct.c_int32), ("sigma", ct.c_float), ("dilation", ct.c_float),
                ("alpha_max", ct.c_float), ("t_min", ct.c_float), ("tile_y_begin", ct.c_int32),
                ("tile_y_end", ct.c_int32), ("flags", ct.c_uint32), ("env_h", ct.c_int32),
                ("env_w", ct.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        # compile the sm_100a library in-tree (nvcc); without it there is no path at all
        from . import build as _build
        try:
            _build.build()
        except Exception as e:
            raise ImportError(f"{LIB_PATH} is missing and could not be built ({e}); build it with "
                              "`python -m paper_2508_19140_b200.build` (nvcc, sm_100a); "
                              "there is no CPU fallback") from e
    else:
        from . import build as _build
        if _build.stale():
            # not rebuilt on import (minutes of nvcc; a copied tree may carry
            # newer source mtimes): say so, the struct layouts may differ
            import warnings
            warnings.warn(f"{LIB_PATH} is older than its sources or was built with other flags "
                          f"({_build.built_flags()!r}); rebuild with `python -m paper_2508_19140_b200.build`",
                          RuntimeWarning, stacklevel=2)
    lib = ct.CDLL(LIB_PATH)
    P, i32, i64 = ct.c_void_p, ct.c_int32, ct.c_int64
    lib.inpc_ctx_create.argtypes = [ct.POINTER(P), ct.c_int]
    lib.inpc_ctx_destroy.argtypes = [P]
    lib.inpc_rasterize_fwd.argtypes = [P, P, P, i32, P, P, i64, P, i64, P, i64, P, P, P, P, P, P]
    lib.inpc_rasterize_bwd.argtypes = [P, P, P, i32, P, P, i64, P, i64, P, i64, P, P, P, P, P, P]
    lib.inpc_debug_export.argtypes = [P, i32, P, P, P, P, i64, ct.POINTER(i64), P]
    lib.inpc_ctx_set_profiling.argtypes = [P, ct.c_int]
    lib.inpc_ctx_stage_times.argtypes = [P, ct.POINTER(ct.c_float), ct.POINTER(i64), i32,
                                         ct.POINTER(i32), ct.c_int]
    lib.inpc_ctx_forget_events.argtypes = [P]
    lib.inpc_sort_single64.argtypes = [P, P, P, P, P, i64, P, P, i64, ct.POINTER(i64), P]
    lib.inpc_ctx_set_allocator.argtypes = [P, ALLOC_FN, FREE_FN, P]
    lib.inpc_spatial_order.argtypes = [P, P, i64, P, P]
    lib.inpc_chunk_bounds.argtypes = [P, P, i64, P, P]
    lib.inpc_ctx_set_chunks.argtypes = [P, P, i64, P]
    lib.inpc_stage_name.argtypes = [i32]
    lib.inpc_stage_name.restype = ct.c_char_p
    lib.inpc_status_string.argtypes = [ct.c_int]
    lib.inpc_status_string.restype = ct.c_char_p
    lib.inpc_version.restype = ct.c_char_p
    for name in EXPORTS:
        getattr(lib, name)
    return lib


lib = _load()


def _check(status):
    if status != OK:
        raise RasterError(status, lib.inpc_status_string(status).decode())


def version() -> str:
    return lib.inpc_version().decode()


def make_camera(cam) -> Camera:
    """From a dict {R (3x3), t, fx, fy, cx, cy, z_near} or a Camera."""
    if isinstance(cam, Camera):
        return cam
    c = Camera()
    R = np.asarray(cam["R"], np.float32).reshape(9)
    t = np.asarray(cam["t"], np.float32).reshape(3)
    c.R[:] = [float(x) for x in R]
    c.t[:] = [float(x) for x in t]
    c.fx, c.fy, c.cx, c.cy = (float(np.float32(cam[k])) for k in ("fx", "fy", "cx", "cy"))
    c.z_near = float(np.float32(cam["z_near"]))
    return c


def make_cfg(H, W, C, mode="bilinear", sigma=0.0, dilation=0.16, alpha_max=0.99, t_min=1e-4,
             band=None, flags=0, env_hw=None) -> RasterCfg:
    g = RasterCfg()
    g.H, g.W, g.C = int(H), int(W), int(C)
    g.splat_mode = {"bilinear": SPLAT_BILINEAR, "gaussian": SPLAT_GAUSSIAN,
                    SPLAT_BILINEAR: SPLAT_BILINEAR, SPLAT_GAUSSIAN: SPLAT_GAUSSIAN}[mode]
    g.sigma, g.dilation = float(sigma), float(dilation)
    g.alpha_max, g.t_min = float(alpha_max), float(t_min)
    g.tile_y_begin, g.tile_y_end = (0, 0) if band is None else (int(band[0]), int(band[1]))
    g.flags = int(flags)
    if env_hw is not None:
        g.env_h, g.env_w = int(env_hw[0]), int(env_hw[1])
        g.flags |= FLAG_ENV_BACKGROUND
    return g


def n_tiles(H, W):
    return ((H + TILE - 1) // TILE) * ((W + TILE - 1) // TILE)


def _ptr(t):
    return None if t is None else ct.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ct.c_void_p(s.cuda_stream)


def _cams(cams):
    if isinstance(cams, (dict, Camera)):
        cams = [cams]
    arr = (Camera * len(cams))(*[make_camera(c) for c in cams])
    return arr, len(cams)


def _strides(cfg, N, feat, bg):
    """Per-view strides of feat ([N,C] / [V,N,C], or SH [N,C,9] / [V,N,C,9])
    and bg ([H,W,C] / [V,H,W,C], or env map [He,We,C] / [V,He,We,C])."""
    sh = bool(cfg.flags & FLAG_SH_FEATURES)
    per_feat = N * cfg.C * (9 if sh else 1)
    fstride = per_feat if feat.dim() == (4 if sh else 3) else 0
    bstride = 0
    if bg is not None and bg.dim() == 4:
        bstride = bg[0].numel()
    return fstride, bstride


def _check_tensor(name, t, device, shape=None, allow_none=False):
    """fp32, contiguous, on `device`, with the expected shape (None entries
    are free) -- the C ABI reads raw fp32 pointers."""
    import torch

    def bad(msg):
        raise RasterError(INVALID_ARG, msg)
    if t is None:
        if allow_none:
            return
        bad(f"{name} is required")
    if not torch.is_tensor(t) or t.dtype != torch.float32:
        bad(f"{name} must be a float32 tensor (got {getattr(t, 'dtype', type(t))})")
    if t.device != device:
        bad(f"{name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        bad(f"{name} must be contiguous")
    if shape is not None:
        if t.dim() != len(shape) or any(e is not None and e != d for e, d in zip(shape, t.shape)):
            bad(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def _feat_shape(cfg, N, feat):
    """[N, C] / [V, N, C], or [N, C, 9] / [V, N, C, 9] with FLAG_SH_FEATURES."""
    sh = bool(cfg.flags & FLAG_SH_FEATURES)
    tail = (N, cfg.C, 9) if sh else (N, cfg.C)
    return tail if feat.dim() == len(tail) else (None,) + tail


class Context:
    """Owns an inpc_ctx (scratch arena + the state saved by forward).

    The saved state belongs to the most recent forward: `generation`
    increases with every forward, and the autograd path checks that the
    state it backpropagates through is still its own."""

    def __init__(self, device=None, torch_allocator=True):
        """torch_allocator: the library's scratch arena and saved state come
        from PyTorch's caching allocator (inpc_ctx_set_allocator) instead of
        cudaMalloc."""
        import torch
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = dev
        h = ct.c_void_p()
        _check(lib.inpc_ctx_create(ct.byref(h), dev))
        self._h = h
        self._cb = None
        self.generation = 0
        if torch_allocator:
            def _alloc(nbytes, device, stream, user):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), device, stream or 0)
                except Exception:       # out of memory -> NULL -> INPC_OOM
                    return None

            def _free(ptr, nbytes, device, stream, user):
                torch.cuda.caching_allocator_delete(ptr)

            self._cb = (ALLOC_FN(_alloc), FREE_FN(_free))
            _check(lib.inpc_ctx_set_allocator(self._h, self._cb[0], self._cb[1], None))

    def close(self):
        if getattr(self, "_h", None):
            lib.inpc_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- forward
    def forward(self, cfg: RasterCfg, cams, xyz, feat, opacity, bg=None, out=None,
                debug_counts=False, stream=None):
        """Render V = len(cams) views.  xyz [N,3], feat [N,C] or [V,N,C], opacity [N]
        (CUDA fp32 contiguous).  Returns dict F [V,H,W,C], A, D [V,H,W]
        (+ nfrag, ncontrib int32 when debug_counts)."""
        import torch
        cam_arr, V = _cams(cams)
        N = xyz.shape[0]
        C, H, W = cfg.C, cfg.H, cfg.W
        dev = xyz.device
        _check_tensor("xyz", xyz, dev, (N, 3))
        _check_tensor("feat", feat, dev, _feat_shape(cfg, N, feat))
        _check_tensor("opacity", opacity, dev, (N,))
        _check_tensor("bg", bg, dev, allow_none=True)
        fstride, bstride = _strides(cfg, N, feat, bg)
        if out is None:
            out = dict(F=torch.empty((V, H, W, C), device=dev, dtype=torch.float32),
                       A=torch.empty((V, H, W), device=dev, dtype=torch.float32),
                       D=torch.empty((V, H, W), device=dev, dtype=torch.float32))
        if debug_counts:
            out.setdefault("nfrag", torch.empty((V, H, W), device=dev, dtype=torch.int32))
            out.setdefault("ncontrib", torch.empty((V, H, W), device=dev, dtype=torch.int32))
        _check(lib.inpc_rasterize_fwd(
            self._h, ct.byref(cfg), cam_arr, V, _ptr(xyz), _ptr(feat), fstride, _ptr(opacity), N,
            _ptr(bg), bstride, _ptr(out["F"]), _ptr(out.get("A")), _ptr(out.get("D")),
            _ptr(out.get("nfrag")), _ptr(out.get("ncontrib")), _stream(stream)))
        self.generation += 1
        return out

    # -------------------------------------------------------------- backward
    def backward(self, cfg: RasterCfg, cams, xyz, feat, opacity, gF, gA=None, gD=None, bg=None,
                 g_feat=None, g_opacity=None, stream=None):
        """Gradients of the last forward; accumulates into g_feat / g_opacity
        (zero-initialised here when not given)."""
        import torch
        cam_arr, V = _cams(cams)
        N = xyz.shape[0]
        C, H, W = cfg.C, cfg.H, cfg.W
        dev = xyz.device
        _check_tensor("xyz", xyz, dev, (N, 3))
        _check_tensor("feat", feat, dev, _feat_shape(cfg, N, feat))
        _check_tensor("opacity", opacity, dev, (N,))
        _check_tensor("bg", bg, dev, allow_none=True)
        lead = (V,) if gF.dim() == 4 or V > 1 else ()   # one view: [H,W,C] / [H,W] also accepted
        _check_tensor("gF", gF, dev, lead + (H, W, C))
        _check_tensor("gA", gA, dev, lead + (H, W), allow_none=True)
        _check_tensor("gD", gD, dev, lead + (H, W), allow_none=True)
        fstride, bstride = _strides(cfg, N, feat, bg)
        if g_feat is None:
            g_feat = torch.zeros_like(feat)
        if g_opacity is None:
            g_opacity = torch.zeros_like(opacity)
        _check_tensor("g_feat", g_feat, dev, tuple(feat.shape))
        _check_tensor("g_opacity", g_opacity, dev, (N,))
        _check(lib.inpc_rasterize_bwd(
            self._h, ct.byref(cfg), cam_arr, V, _ptr(xyz), _ptr(feat), fstride, _ptr(opacity), N,
            _ptr(bg), bstride, _ptr(gF), _ptr(gA), _ptr(gD), _ptr(g_feat), _ptr(g_opacity),
            _stream(stream)))
        return g_feat, g_opacity

    # -------------------------------------------------------------- debug / profiling
    def debug_export(self, view=0, N=None, H=None, W=None, stream=None):
        """Saved tile lists of the last forward: tile_ranges [T+1], sorted_idx [F_t]
        (+ depth_keys, tiles_touched [N] when the forward had FLAG_DEBUG)."""
        import torch
        Ft = ct.c_int64()
        _check(lib.inpc_debug_export(self._h, view, None, None, None, None, 0, ct.byref(Ft),
                                     _stream(stream)))
        dev = torch.device("cuda", self.device)
        out = {}
        T = n_tiles(H, W)
        out["tile_ranges"] = torch.empty(T + 1, dtype=torch.int32, device=dev)
        out["sorted_idx"] = torch.empty(max(Ft.value, 1), dtype=torch.int32, device=dev)
        kp = tp = None
        if N is not None:
            out["depth_keys"] = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
            out["tiles_touched"] = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
            kp, tp = _ptr(out["depth_keys"]), _ptr(out["tiles_touched"])
        _check(lib.inpc_debug_export(self._h, view, kp, tp, _ptr(out["tile_ranges"]),
                                     _ptr(out["sorted_idx"]), Ft.value, ct.byref(Ft),
                                     _stream(stream)))
        out["sorted_idx"] = out["sorted_idx"][:Ft.value]
        out["F_t"] = Ft.value
        return out

    def sort_single64(self, cfg: RasterCfg, cam, xyz, opacity, stream=None):
        """NEXT f4: the original INPC ordering (4 copies per point, one 64-bit
        radix sort by pixel then depth).  Returns (pixel_ranges [H*W+1],
        sorted_idx [F]) as int32 tensors (bit patterns of u32)."""
        import torch
        cam_arr, _ = _cams(cam)
        N = xyz.shape[0]
        dev = xyz.device
        ranges = torch.empty(cfg.H * cfg.W + 1, dtype=torch.int32, device=dev)
        idx = torch.empty(max(4 * N, 1), dtype=torch.int32, device=dev)
        F = ct.c_int64()
        _check(lib.inpc_sort_single64(self._h, ct.byref(cfg), cam_arr, _ptr(xyz), _ptr(opacity), N,
                                      _ptr(ranges), _ptr(idx), idx.numel(), ct.byref(F), _stream(stream)))
        return ranges, idx[:F.value]

    def spatial_order(self, xyz, stream=None):
        """Permutation (int64 CUDA tensor [N]) that puts a static cloud in
        Morton order (inpc_spatial_order); gather every per-point array by it
        once, then rasterize the reordered cloud."""
        import torch
        N = xyz.shape[0]
        perm = torch.empty(max(N, 1), dtype=torch.int32, device=xyz.device)
        _check(lib.inpc_spatial_order(self._h, _ptr(xyz), N, _ptr(perm), _stream(stream)))
        return perm[:N].long()

    def set_chunks(self, xyz, stream=None):
        """Compute the chunk bounds of the static cloud `xyz` (inpc_chunk_bounds)
        and attach them: forwards over this same tensor then skip chunks that
        cannot reach the frame / screen band.  set_chunks(None) detaches."""
        import torch
        if xyz is None:
            _check(lib.inpc_ctx_set_chunks(self._h, None, 0, None))
            self._chunk_box = None
            return None
        N = xyz.shape[0]
        box = torch.empty(((N + 1023) // 1024, 6), dtype=torch.float32, device=xyz.device)
        _check(lib.inpc_chunk_bounds(self._h, _ptr(xyz), N, _ptr(box), _stream(stream)))
        _check(lib.inpc_ctx_set_chunks(self._h, _ptr(xyz), N, _ptr(box)))
        self._chunk_box = (xyz, box)      # both kept alive with the context
        return box

    def set_profiling(self, on=True):
        _check(lib.inpc_ctx_set_profiling(self._h, 1 if on else 0))

    def stage_times(self, reset=True, keep_events=False):
        """{stage: (ms, launches)} accumulated since the last reset.
        keep_events: the calls were captured in a CUDA graph; read again
        after the next replay."""
        n = 16
        ms = (ct.c_float * n)()
        la = (ct.c_int64 * n)()
        ns = ct.c_int32()
        flags = (1 if reset else 0) | (2 if keep_events else 0)
        _check(lib.inpc_ctx_stage_times(self._h, ms, la, n, ct.byref(ns), flags))
        return {lib.inpc_stage_name(k).decode(): (ms[k], la[k]) for k in range(ns.value)}

    def forget_events(self):
        _check(lib.inpc_ctx_forget_events(self._h))


_default_ctx = {}


def default_context(device=None) -> Context:
    import torch
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _default_ctx:
        _default_ctx[dev] = Context(dev)
    return _default_ctx[dev]


class _ContextPool:
    """Contexts for in-flight autograd graphs of rasterize(): a graph holds
    its context (and so its saved forward state) until its backward ran or
    the graph was freed, so two rasterize() calls before one .backward() do
    not share saved state."""

    def __init__(self):
        self.free = {}

    def acquire(self, device):
        lst = self.free.setdefault(device, [])
        return lst.pop() if lst else Context(device)

    def release(self, ctx):
        if getattr(ctx, "_h", None):
            self.free.setdefault(ctx.device, []).append(ctx)


_pool = _ContextPool()


def _autograd():
    import weakref

    import torch

    class RasterizeFn(torch.autograd.Function):
        @staticmethod
        def forward(actx, xyz, feat, opacity, bg, settings):
            cfg, cams, context = settings
            owned = context is None
            if owned:
                context = _pool.acquire(xyz.device.index)
            out = context.forward(cfg, cams, xyz, feat, opacity, bg=bg)
            actx.save_for_backward(xyz, feat, opacity, bg)
            actx.settings = (cfg, cams, context)
            actx.generation = context.generation
            actx.owned = owned
            if owned:   # back to the pool when the graph goes away without a backward
                actx.finalizer = weakref.finalize(actx, _pool.release, context)
            return out["F"], out["A"], out["D"]

        @staticmethod
        def backward(actx, gF, gA, gD):
            xyz, feat, opacity, bg = actx.saved_tensors
            cfg, cams, context = actx.settings
            if context.generation != actx.generation:
                raise RuntimeError("inpc: the context's saved forward state was overwritten by a later "
                                   "forward on the same context; give each in-flight graph its own "
                                   "context (rasterize(..., context=None) does)")
            gf, go = context.backward(cfg, cams, xyz, feat, opacity, gF.contiguous(),
                                      None if gA is None else gA.contiguous(),
                                      None if gD is None else gD.contiguous(), bg=bg)
            if actx.owned:
                actx.finalizer()   # release now (detaches the finalizer)
            return None, gf, go, None, None

    return RasterizeFn


_Fn = None


def rasterize(xyz, feat, opacity, cams, H, W, mode="bilinear", sigma=0.0, dilation=0.16,
              alpha_max=0.99, t_min=1e-4, bg=None, band=None, flags=0, env_hw=None, context=None):
    """Differentiable raster of V views: returns F [V,H,W,C], A [V,H,W], D [V,H,W].
    Gradients flow to feat and opacity.  feat: [N,C] or [V,N,C];
    with FLAG_SH_FEATURES the SH coefficients [N,C,9].  env_hw: size of
    an equirectangular background map `bg` [He,We,C].
    context=None: each call's graph holds its own pooled context until its
    backward; an explicit context is shared (its backward then raises if a
    later forward overwrote the saved state)."""
    global _Fn
    if _Fn is None:
        _Fn = _autograd()
    C = feat.shape[-2] if (flags & FLAG_SH_FEATURES) else feat.shape[-1]
    cfg = make_cfg(H, W, C, mode, sigma, dilation, alpha_max, t_min, band, flags, env_hw=env_hw)
    return _Fn.apply(xyz.contiguous(), feat.contiguous(), opacity.contiguous(),
                     None if bg is None else bg.contiguous(), (cfg, cams, context))

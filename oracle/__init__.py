"""CPU oracle for the INPC neural point rasterizer — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
path (``paper_2508_19140_b200``) never imports it, and this package imports
nothing from the product path: the two share no code (the seeded input
generators live in their own module, ``synthgen``).

The arithmetic lives in ``inpc_oracle.c`` (plain C, fp32 decisions in the
pinned op order of DESIGN.md §3, fp64 values), compiled with
``gcc -O2 -ffp-contract=off`` (no fast-math, no FMA contraction).  This file is
ctypes marshalling only.

What each function follows (PAPER.md = P, line numbers):
  render      per-pixel gather -> sort (depth, idx) -> Eq. 1
  backward    Eq. 2, background sign corrected, alpha=0 kept
  point_info  projection, depth key, tiles per point
  tile_lists  definition of the two-stage sort's output
  pixel_lists O3 per-pixel sort / O7 single 64-bit stable sort
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "inpc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

GCC_FLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
             "-fno-fast-math", "-fexcess-precision=standard", "-Wall", "-Wextra",
             "-Wno-unused-parameter"]

SIGMA_IS_PIXELS = 1
SKIP_ZERO_ALPHA_GRAD = 2
TILE = 8


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc) if missing or older than the source."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *GCC_FLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Cam(ct.Structure):
    _fields_ = [("R", ct.c_float * 9), ("t", ct.c_float * 3), ("fx", ct.c_float),
                ("fy", ct.c_float), ("cx", ct.c_float), ("cy", ct.c_float),
                ("z_near", ct.c_float)]


class _Cfg(ct.Structure):
    _fields_ = [("H", ct.c_int32), ("W", ct.c_int32), ("C", ct.c_int32),
                ("mode", ct.c_int32), ("sigma", ct.c_float), ("dilation", ct.c_float),
                ("alpha_max", ct.c_float), ("t_min", ct.c_float), ("flags", ct.c_uint32)]


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ct.CDLL(build())
            P = ct.c_void_p
            i64, i32 = ct.c_int64, ct.c_int32
            lib.or_point_info.argtypes = [P, P, i64, P, P, P, P, P]
            lib.or_point_info.restype = ct.c_int
            lib.or_render.argtypes = [P, P, i64, P, P, P, P, P, P, P, P, P, P, P, ct.c_int]
            lib.or_render.restype = ct.c_int
            lib.or_backward.argtypes = [P, P, i64, P, P, P, P, P, P, P, P, P, P, ct.c_int]
            lib.or_backward.restype = ct.c_int
            lib.or_tile_lists.argtypes = [P, P, i64, P, i32, i32, P, P, i64]
            lib.or_tile_lists.restype = i64
            lib.or_pixel_lists.argtypes = [P, P, i64, P, ct.c_int, P, P, i64]
            lib.or_pixel_lists.restype = i64
            lib.or_fragments.argtypes = [P, P, i64, P, P, P, P, P, P, i64]
            lib.or_fragments.restype = i64
            lib.or_max_threads.restype = ct.c_int
            lib.or_sh_basis.argtypes = [P, P]
            lib.or_sh_features.argtypes = [P, i64, ct.c_int, P, P, P, P]
            lib.or_env_background.argtypes = [P, ct.c_int, ct.c_int, ct.c_int, P, ct.c_int, ct.c_int, P]
            _lib = lib
    return _lib


def max_threads() -> int:
    return _load().or_max_threads()


def _cam(cam: dict) -> _Cam:
    c = _Cam()
    R = np.asarray(cam["R"], np.float32).reshape(9)
    t = np.asarray(cam["t"], np.float32).reshape(3)
    for k in range(9):
        c.R[k] = float(R[k])
    for k in range(3):
        c.t[k] = float(t[k])
    c.fx, c.fy, c.cx, c.cy = (float(np.float32(cam[k])) for k in ("fx", "fy", "cx", "cy"))
    c.z_near = float(np.float32(cam["z_near"]))
    return c


def _cfg(H, W, C, mode="bilinear", sigma=0.0, dilation=0.16, alpha_max=0.99,
         t_min=1e-4, flags=0) -> _Cfg:
    g = _Cfg()
    g.H, g.W, g.C = int(H), int(W), int(C)
    g.mode = {"bilinear": 0, "gaussian": 1, 0: 0, 1: 1}[mode]
    g.sigma, g.dilation = float(np.float32(sigma)), float(np.float32(dilation))
    g.alpha_max, g.t_min = float(np.float32(alpha_max)), float(np.float32(t_min))
    g.flags = int(flags)
    return g


def _p(a):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a if shape is None else a.reshape(shape)


def _f64(a, shape=None):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def point_info(cam, xyz, H, W, mode="bilinear", **kw):
    """Per point: depth key (0xFFFFFFFF = culled), tiles touched, (u, v, z_c),
    Gaussian (conic a,b,c, radius, cov a,b,c)."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    key = np.zeros(N, np.uint32)
    tiles = np.zeros(N, np.uint32)
    uvz = np.zeros((N, 3), np.float32)
    gauss = np.zeros((N, 7), np.float32)
    c, g = _cam(cam), _cfg(H, W, 1, mode, **kw)
    _load().or_point_info(ct.byref(c), ct.byref(g), N, _p(xyz), _p(key), _p(tiles),
                          _p(uvz), _p(gauss))
    return dict(depth_key=key, tiles_touched=tiles, uvz=uvz, gauss=gauss)


def render(cam, xyz, feat, opacity, H, W, mode="bilinear", bg=None, pixel_mask=None,
           threads=1, **kw):
    """Forward (Eq. 1 + background).  Returns F [H,W,C], A, D (fp64), T32 (fp32
    decision transmittance), n_contrib, n_frag (int32)."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    feat = _f64(feat, (N, -1)) if N else _f64(np.zeros((0, np.asarray(feat).shape[-1])))
    C = feat.shape[1]
    op = _f64(opacity, (N,))
    bgd = _f64(bg, (H * W * C,)) if bg is not None else None
    mask = None if pixel_mask is None else np.ascontiguousarray(pixel_mask, np.uint8).reshape(H * W)
    F = np.zeros((H, W, C)); A = np.zeros((H, W)); D = np.zeros((H, W))
    T = np.ones((H, W), np.float32)
    nc = np.zeros((H, W), np.int32); nf = np.zeros((H, W), np.int32)
    c, g = _cam(cam), _cfg(H, W, C, mode, **kw)
    rc = _load().or_render(ct.byref(c), ct.byref(g), N, _p(xyz), _p(feat), _p(op), _p(bgd),
                           _p(mask), _p(F), _p(A), _p(D), _p(T), _p(nc), _p(nf), int(threads))
    if rc:
        raise MemoryError("oracle render failed")
    return dict(F=F, A=A, D=D, T=T, n_contrib=nc, n_frag=nf)


def backward(cam, xyz, feat, opacity, H, W, gF, gA=None, gD=None, mode="bilinear", bg=None,
             pixel_mask=None, threads=1, **kw):
    """Backward (corrected Eq. 2) in fp64.  Returns dict(g_feat [N,C], g_opacity [N])."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    feat = _f64(feat, (N, -1))
    C = feat.shape[1]
    op = _f64(opacity, (N,))
    bgd = _f64(bg, (H * W * C,)) if bg is not None else None
    mask = None if pixel_mask is None else np.ascontiguousarray(pixel_mask, np.uint8).reshape(H * W)
    gFd = _f64(gF, (H * W * C,))
    gAd = _f64(gA, (H * W,)) if gA is not None else None
    gDd = _f64(gD, (H * W,)) if gD is not None else None
    gf = np.zeros((N, C)); go = np.zeros(N)
    c, g = _cam(cam), _cfg(H, W, C, mode, **kw)
    rc = _load().or_backward(ct.byref(c), ct.byref(g), N, _p(xyz), _p(feat), _p(op), _p(bgd),
                             _p(mask), _p(gFd), _p(gAd), _p(gDd), _p(gf), _p(go), int(threads))
    if rc:
        raise MemoryError("oracle backward failed")
    return dict(g_feat=gf, g_opacity=go)


def n_tiles(H, W):
    return ((W + TILE - 1) // TILE) * ((H + TILE - 1) // TILE)


def tile_lists(cam, xyz, H, W, mode="bilinear", band=None, **kw):
    """Per-tile lists sorted by (depth key, idx): (tile_ranges [T+1], sorted_idx [F_t])."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    T = n_tiles(H, W)
    ty0, ty1 = band if band is not None else (0, (H + TILE - 1) // TILE)
    ranges = np.zeros(T + 1, np.uint32)
    c, g = _cam(cam), _cfg(H, W, 1, mode, **kw)
    lib = _load()
    Ft = lib.or_tile_lists(ct.byref(c), ct.byref(g), N, _p(xyz), ty0, ty1, _p(ranges), None, 0)
    if Ft < 0:
        raise MemoryError("oracle tile_lists failed")
    idx = np.zeros(max(Ft, 1), np.uint32)
    lib.or_tile_lists(ct.byref(c), ct.byref(g), N, _p(xyz), ty0, ty1, _p(ranges), _p(idx), Ft)
    return ranges, idx[:Ft]


def pixel_lists(cam, xyz, H, W, method=0, mode="bilinear", **kw):
    """Per-pixel fragment lists: method 0 per-pixel (depth, idx) sort (O3),
    method 1 single stable 64-bit (pixel<<32 | depth) sort (O7)."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    ranges = np.zeros(H * W + 1, np.uint32)
    c, g = _cam(cam), _cfg(H, W, 1, mode, **kw)
    lib = _load()
    n = lib.or_pixel_lists(ct.byref(c), ct.byref(g), N, _p(xyz), method, _p(ranges), None, 0)
    idx = np.zeros(max(n, 1), np.uint32)
    lib.or_pixel_lists(ct.byref(c), ct.byref(g), N, _p(xyz), method, _p(ranges), _p(idx), n)
    return ranges, idx[:n]


def fragments(cam, xyz, H, W, mode="bilinear", **kw):
    """Raw fragments in emission order: dict(pix, idx, key, w32, w64)."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    c, g = _cam(cam), _cfg(H, W, 1, mode, **kw)
    lib = _load()
    n = lib.or_fragments(ct.byref(c), ct.byref(g), N, _p(xyz), None, None, None, None, None, 0)
    m = max(n, 1)
    out = dict(pix=np.zeros(m, np.int32), idx=np.zeros(m, np.uint32), key=np.zeros(m, np.uint32),
               w32=np.zeros(m, np.float32), w64=np.zeros(m, np.float64))
    lib.or_fragments(ct.byref(c), ct.byref(g), N, _p(xyz), _p(out["pix"]), _p(out["idx"]),
                     _p(out["key"]), _p(out["w32"]), _p(out["w64"]), n)
    return {k: v[:n] for k, v in out.items()}


def sh_basis(d):
    """Real SH basis of degree <= 2 (9 values) at unit direction d (fp64)."""
    d = np.ascontiguousarray(d, np.float64).reshape(3)
    Y = np.zeros(9)
    _load().or_sh_basis(_p(d), _p(Y))
    return Y


def sh_features(cam, xyz, sh):
    """Features [N, C] from SH coefficients [N, C, 9] at the view directions of
    camera `cam`; also returns the basis values [N, 9]."""
    xyz = _f32(xyz, (-1, 3))
    N = xyz.shape[0]
    sh = _f64(sh, (N, -1, 9))
    C = sh.shape[1]
    feat = np.zeros((N, C)); Y = np.zeros((N, 9))
    c = _cam(cam)
    _load().or_sh_features(ct.byref(c), N, C, _p(xyz), _p(sh), _p(feat), _p(Y))
    return feat, Y


def env_background(cam, env, H, W):
    """Per-pixel background [H, W, C] from an equirectangular map [He, We, C]
    (P:185-192)."""
    env = _f32(env)
    He, We, C = env.shape
    bg = np.zeros((H, W, C))
    c = _cam(cam)
    _load().or_env_background(ct.byref(c), int(H), int(W), int(C), _p(env), int(He), int(We), _p(bg))
    return bg

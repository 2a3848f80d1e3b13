"""Seeded synthetic inputs for the INPC rasterizer (configs 1-5 of BASELINE.json).

This module is shared by the oracle tests and the CUDA path and therefore holds
NONE of the method's arithmetic: no projection-to-pixels, no footprints, no
blending.  It only draws point clouds, cameras and upstream gradients with the
shapes and distributions of the paper's workloads (DESIGN.md §5 "input
recipe"):

  cfg1  1k random points, 64x64, bilinear          (oracle finishes in ms)
  cfg2  2^20-point view-specific cloud, 1080p       (P:91-93 well-behaved screen
        distribution; P:112/P:116 sample counts)
  cfg3  4 x 2^20 ring-buffer cloud, Gaussian, 3 % close-ups
  cfg4  2^25 global extracted cloud (Table 4): object + background shell
  cfg5  2^23 cloud + 64 orbit cameras (training-style view batch)

Cameras are dicts {R (3x3 world->camera, row-major), t, fx, fy, cx, cy, z_near}
with x_cam = R @ x_world + t.  Points are built in camera space of a chosen
pose (inverse pinhole: screen position + depth -> camera point) and moved to
world space with that pose; the generator never evaluates the forward
projection.
"""
from __future__ import annotations

import numpy as np

W1080, H1080 = 1920, 1080
F1080 = 1100.0


def camera(R, t, fx, fy, cx, cy, z_near):
    return dict(R=np.asarray(R, np.float32).reshape(3, 3), t=np.asarray(t, np.float32).reshape(3),
                fx=float(fx), fy=float(fy), cx=float(cx), cy=float(cy), z_near=float(z_near))


def look_at(eye, target, up=(0.0, -1.0, 0.0)):
    """World->camera rotation/translation with +z forward, +x right, +y down."""
    eye = np.asarray(eye, np.float64); target = np.asarray(target, np.float64)
    z = target - eye; z /= np.linalg.norm(z)
    x = np.cross(np.asarray(up, np.float64), z)
    if np.linalg.norm(x) < 1e-9:
        x = np.cross(np.array([1.0, 0.0, 0.0]), z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])
    return R, -R @ eye


def random_rotation(rng):
    q = rng.normal(size=4); q /= np.linalg.norm(q)
    a, b, c, d = q
    return np.array([[a*a+b*b-c*c-d*d, 2*(b*c-a*d), 2*(b*d+a*c)],
                     [2*(b*c+a*d), a*a-b*b+c*c-d*d, 2*(c*d-a*b)],
                     [2*(b*d-a*c), 2*(c*d+a*b), a*a-b*b-c*c+d*d]])


def _to_world(xc, R, t):
    """camera-space points [N,3] -> world, x_w = R^T (x_c - t)."""
    return (xc - t[None, :]) @ R


def _screen_cloud(rng, n, W, H, f, cx, cy, zlo, zhi, blob_frac=0.3, n_blobs=64,
                  blob_sigma=40.0, offscreen_frac=0.02):
    """A 'view-specific' cloud in camera space: screen-uniform + blobs, depth
    log-uniform with smooth layering."""
    nb = int(n * blob_frac)
    nu = n - nb
    us = np.empty(n); vs = np.empty(n)
    us[:nu] = rng.uniform(0, W, nu); vs[:nu] = rng.uniform(0, H, nu)
    centres = np.stack([rng.uniform(0, W, n_blobs), rng.uniform(0, H, n_blobs)], 1)
    which = rng.integers(0, n_blobs, nb)
    us[nu:] = centres[which, 0] + rng.normal(0, blob_sigma, nb)
    vs[nu:] = centres[which, 1] + rng.normal(0, blob_sigma, nb)
    # depth: log-uniform, plus a smooth screen-dependent layering term
    lz = rng.uniform(np.log(zlo), np.log(zhi), n)
    lz += 0.15 * np.sin(us / 157.0) * np.cos(vs / 113.0)
    z = np.clip(np.exp(lz), zlo, zhi)
    # a few points off screen / behind the camera (culled, ~2 %)
    k = int(n * offscreen_frac)
    if k:
        sel = rng.choice(n, k, replace=False)
        half = k // 2
        us[sel[:half]] = rng.uniform(-3 * W, 4 * W, half)
        z[sel[half:]] = -z[sel[half:]]
    perm = rng.permutation(n)
    us, vs, z = us[perm], vs[perm], z[perm]
    xc = np.stack([(us - cx) / f * np.abs(z), (vs - cy) / f * np.abs(z), z], 1)
    return xc


def _attributes(rng, n, C=4, zero_frac=0.02, beta=True):
    op = rng.beta(0.5, 0.5, n) if beta else rng.uniform(0, 1, n)
    op[rng.random(n) < zero_frac] = 0.0
    feat = rng.uniform(-1, 1, (n, C))
    return feat.astype(np.float32), op.astype(np.float32)


def upstream_grads(seed, V, H, W, C):
    """dL/dF [V,H,W,C], dL/dA [V,H,W], dL/dD [V,H,W]  ~ N(0,1) (fp32)."""
    rng = np.random.default_rng(seed + 1000)
    return (rng.standard_normal((V, H, W, C), dtype=np.float32),
            rng.standard_normal((V, H, W), dtype=np.float32),
            rng.standard_normal((V, H, W), dtype=np.float32))


def config1(seed=1, N=1000, C=4, H=64, W=64):
    """N random points on a 64x64 image, identity camera (exact ties), f = 64.

    5 % snapped to exact pixel centres (weight-0 fragments), 2 % sharing one
    exact depth, opacity U(0,1) with 5 % exactly 0 and 3 % exactly 1,
    ~6 % partly off-image.  f is a power of two so snapped points project
    exactly onto pixel centres.
    """
    rng = np.random.default_rng(seed)
    f = 64.0
    cam = camera(np.eye(3), np.zeros(3), f, f, W / 2, H / 2, 0.1)
    u = rng.uniform(-2, W + 2, N); v = rng.uniform(-2, H + 2, N)
    z = rng.uniform(1, 4, N)
    ns = int(round(0.05 * N))
    snap = rng.choice(N, ns, replace=False)
    u[snap] = rng.integers(0, W, ns) + 0.5
    v[snap] = rng.integers(0, H, ns) + 0.5
    z[snap] = rng.choice([1.0, 2.0, 4.0], ns)
    rest = np.setdiff1d(np.arange(N), snap)
    tie = rng.choice(rest, int(round(0.02 * N)), replace=False)
    z[tie] = 2.5
    x = (u - W / 2) / f * z
    y = (v - H / 2) / f * z
    xyz = np.stack([x, y, z], 1).astype(np.float32)
    feat = rng.uniform(-1, 1, (N, C)).astype(np.float32)
    op = rng.uniform(0, 1, N)
    r = rng.random(N)
    op[r < 0.05] = 0.0
    op[(r >= 0.05) & (r < 0.08)] = 1.0
    return dict(name="cfg1", xyz=xyz, feat=feat, opacity=op.astype(np.float32), cams=[cam],
                H=H, W=W, C=C, mode="bilinear", passes="fwd+bwd")


def config2(seed=2, N=1 << 20, C=4, H=H1080, W=W1080):
    """2^20-point view-specific cloud at 1080p, bilinear, fwd+bwd, 1 GPU."""
    rng = np.random.default_rng(seed)
    R = random_rotation(rng); t = rng.normal(0, 2.0, 3)
    cam = camera(R, t, F1080, F1080, W / 2, H / 2, 0.01)
    xc = _screen_cloud(rng, N, W, H, F1080, W / 2, H / 2, 0.5, 30.0)
    xyz = _to_world(xc, R, t).astype(np.float32)
    feat, op = _attributes(rng, N, C)
    return dict(name="cfg2", xyz=xyz, feat=feat, opacity=op, cams=[cam], H=H, W=W, C=C,
                mode="bilinear", passes="fwd+bwd")


def _yaw(deg):
    a = np.deg2rad(deg)
    return np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])


def config3(seed=3, N_each=1 << 20, n_ring=4, C=4, H=H1080, W=W1080, close_frac=0.03):
    """Ring buffer of 4 view-specific clouds for 4 poses 0.05 units / 1 deg yaw
    apart, concatenated in push order; rendered from the newest pose with
    Gaussian splats.  3 % close-ups at z in [0.011, 0.25]."""
    rng = np.random.default_rng(seed)
    R0 = random_rotation(rng); t0 = rng.normal(0, 2.0, 3)
    clouds, cams = [], []
    for k in range(n_ring):
        R = _yaw(k * 1.0) @ R0
        t = t0 + np.array([0.05 * k, 0.0, 0.0])
        xc = _screen_cloud(rng, N_each, W, H, F1080, W / 2, H / 2, 0.5, 30.0)
        nc = int(N_each * close_frac)
        sel = rng.choice(N_each, nc, replace=False)
        zc = rng.uniform(0.011, 0.25, nc)
        xc[sel] = xc[sel] / np.abs(xc[sel, 2:3]) * zc[:, None]
        clouds.append(_to_world(xc, R, t))
        cams.append(camera(R, t, F1080, F1080, W / 2, H / 2, 0.01))
    xyz = np.concatenate(clouds).astype(np.float32)
    feat, op = _attributes(rng, xyz.shape[0], C)
    return dict(name="cfg3", xyz=xyz, feat=feat, opacity=op, cams=[cams[-1]], H=H, W=W, C=C,
                mode="gaussian", passes="fwd")


def _object_scene(rng, N, obj_frac=0.6):
    """Global extracted cloud: object surface (radius 1, +-5 %)
    plus a background shell r in [3, 20] ('too many points in the background')."""
    no = int(N * obj_frac)
    nb = N - no
    d = rng.normal(size=(no, 3)); d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = 1.0 + rng.uniform(-0.05, 0.05, no)
    obj = d * r[:, None]
    d2 = rng.normal(size=(nb, 3)); d2 /= np.linalg.norm(d2, axis=1, keepdims=True)
    r2 = np.exp(rng.uniform(np.log(3.0), np.log(20.0), nb))
    return np.concatenate([obj, d2 * r2[:, None]])[rng.permutation(N)]


def config4(seed=4, N=1 << 25, C=4, H=H1080, W=W1080):
    """2^25-point global cloud, 1080p, bilinear forward only (Table 4)."""
    rng = np.random.default_rng(seed)
    xyz = _object_scene(rng, N).astype(np.float32)
    R, t = look_at([0.0, -0.6, 3.0], [0.0, 0.0, 0.0])
    cam = camera(R, t, F1080, F1080, W / 2, H / 2, 0.01)
    feat, op = _attributes(rng, N, C)
    return dict(name="cfg4", xyz=xyz, feat=feat, opacity=op, cams=[cam], H=H, W=W, C=C,
                mode="bilinear", passes="fwd")


def orbit_cameras(V, radius=3.0, seed=5, H=H1080, W=W1080):
    rng = np.random.default_rng(seed + 77)
    cams = []
    for k in range(V):
        az = 2 * np.pi * k / V
        el = np.deg2rad(rng.uniform(-15, 15))
        eye = radius * np.array([np.cos(el) * np.sin(az), np.sin(el), np.cos(el) * np.cos(az)])
        R, t = look_at(eye, [0.0, 0.0, 0.0])
        cams.append(camera(R, t, F1080, F1080, W / 2, H / 2, 0.01))
    return cams


def config5(seed=5, N=1 << 23, V=64, C=4, H=H1080, W=W1080):
    """Training-style batch: 64 orbit views of a 2^23-point cloud, shared
    features, fwd+bwd, view-sharded."""
    rng = np.random.default_rng(seed)
    xyz = _object_scene(rng, N).astype(np.float32)
    feat, op = _attributes(rng, N, C)
    return dict(name="cfg5", xyz=xyz, feat=feat, opacity=op, cams=orbit_cameras(V, seed=seed),
                H=H, W=W, C=C, mode="bilinear", passes="fwd+bwd")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


"""Pins for the oracle parts round 1 left unpinned:

  - projection under a non-identity pose (pinhole; R1, R2, R7):
    points are built in camera space by the inverse pinhole, moved to world
    space by x_w = R^T (x_c - t) in fp64, and the oracle must return the
    construction's (u, v, z_c) -- a transposed or column-major R fails;
  - the off-axis EWA covariance ("affine approximation of the perspective
    projection"; R15-R17): Sigma_2D = s^2 J J^T + dilation I with the
    Jacobian J written as a matrix and multiplied by numpy in fp64 -- a
    dropped (1 + xz^2) factor or a flipped sign of the off-diagonal fails;
  - the per-tile lists: sum of tiles_touched == F_t, and every
    list holds exactly the points whose footprint rectangle meets the tile
    (brute force over all (tile, point) pairs on small inputs).

P:n = PAPER.md line n.  None of these retypes the oracle's formula: the
references are the geometric construction, a matrix product and a brute-force
rectangle test.
"""
import numpy as np
import pytest

import oracle
import synthgen


def random_rotation(rng):
    """Proper rotation (det +1) from the QR of a Gaussian matrix (fp64)."""
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def posed_camera(rng, W, H, f):
    R = random_rotation(rng)
    t = rng.uniform(-3, 3, 3)
    return synthgen.camera(R, t, f, f, W / 2, H / 2, 0.05), R, t


def world_from_screen(R, t, cam, u, v, z):
    """Inverse pinhole in camera space, then x_w = R^T (x_c - t) (fp64)."""
    xc = np.stack([(u - cam["cx"]) / cam["fx"] * z, (v - cam["cy"]) / cam["fy"] * z, z], 1)
    return (xc - t[None, :]) @ R   # rows: R^T (x_c - t)


# ------------------------------------------------------------------ P:76 pose
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_projection_under_random_pose(seed):
    """P:76 pinhole x_c = R x + t, u = f x_c / z_c + c (R2): the oracle's
    (u, v, z_c) equal the construction up to fp32 rounding of the pinned
    sequence; depth_key is the fp32 bit pattern of z_c (R7)."""
    rng = np.random.default_rng(100 + seed)
    W, H, f = 256, 192, 128.0
    cam, R, t = posed_camera(rng, W, H, f)
    n = 500
    u = rng.uniform(-20, W + 20, n)
    v = rng.uniform(-20, H + 20, n)
    z = rng.choice([0.5, 1.0, 2.0, 4.0, 8.0], n) * rng.uniform(1.0, 1.9, n)
    xyz = world_from_screen(np.asarray(cam["R"], np.float64).reshape(3, 3),
                            np.asarray(cam["t"], np.float64), cam, u, v, z).astype(np.float32)
    info = oracle.point_info(cam, xyz, H, W)
    uvz = info["uvz"].astype(np.float64)
    # fp32 positions of magnitude <~ 30 and a 9-term rounded sum: |err| in
    # x_c ~ 1e-5, times f / z <= 256 -> 5e-3 px
    np.testing.assert_allclose(uvz[:, 2], z, rtol=0, atol=2e-5 * (1 + np.abs(xyz).max()))
    np.testing.assert_allclose(uvz[:, 0], u, atol=5e-3)
    np.testing.assert_allclose(uvz[:, 1], v, atol=5e-3)
    key = info["depth_key"]
    assert np.all(key == info["uvz"][:, 2].astype(np.float32).view(np.uint32))
    # a transposed rotation puts the points elsewhere (the pin can fail)
    bad = dict(cam, R=np.asarray(cam["R"], np.float64).reshape(3, 3).T)
    ub = oracle.point_info(bad, xyz, H, W)["uvz"].astype(np.float64)
    assert np.max(np.abs(ub[:, 2] - z)) > 0.1


def test_posed_render_equals_camera_space_render():
    """The whole forward is pose-equivariant: rendering world points through
    (R, t) equals rendering their camera-space coordinates through the
    identity camera (same intrinsics), up to the fp32 rounding of the pose."""
    rng = np.random.default_rng(7)
    W, H, f = 64, 48, 64.0
    cam, R, t = posed_camera(rng, W, H, f)
    Rf = np.asarray(cam["R"], np.float64).reshape(3, 3)
    tf = np.asarray(cam["t"], np.float64)
    n = 300
    # pixel positions away from block boundaries so that fp32 pose rounding
    # cannot move a point to another pixel block (integer + 0.5 +- 0.3)
    u = rng.integers(0, W, n) + 0.5 + rng.uniform(-0.3, 0.3, n)
    v = rng.integers(0, H, n) + 0.5 + rng.uniform(-0.3, 0.3, n)
    z = rng.uniform(1.0, 3.0, n)
    xw = world_from_screen(Rf, tf, cam, u, v, z).astype(np.float32)
    xc = (xw.astype(np.float64) @ Rf.T + tf[None, :]).astype(np.float32)
    ident = synthgen.camera(np.eye(3), np.zeros(3), f, f, W / 2, H / 2, 0.05)
    feat = rng.uniform(-1, 1, (n, 3))
    op = rng.uniform(0, 1, n)
    a = oracle.render(cam, xw, feat, op, H, W, t_min=0.0)
    b = oracle.render(ident, xc, feat, op, H, W, t_min=0.0)
    assert np.array_equal(a["n_frag"], b["n_frag"])
    np.testing.assert_allclose(a["F"], b["F"], atol=2e-4)
    np.testing.assert_allclose(a["A"], b["A"], atol=2e-4)


# ------------------------------------------------------------------ P:202 EWA
def ewa_cov(cam, xc, s, dil):
    """Sigma_2D = J (s^2 I) J^T + dil I, J = d(u, v)/d(x_c) of the pinhole
    (the affine approximation of the perspective projection)."""
    x, y, z = xc
    J = np.array([[cam["fx"] / z, 0.0, -cam["fx"] * x / z ** 2],
                  [0.0, cam["fy"] / z, -cam["fy"] * y / z ** 2]])
    return J @ (s * s * np.eye(3)) @ J.T + dil * np.eye(2)


def test_off_axis_ewa_covariance_all_quadrants():
    """20 off-axis points, 5 per image quadrant, fx != fy: (a2, b2, c2) of the
    oracle equal the fp64 matrix product within rel 1e-5; the off-diagonal
    has the sign of x_c y_c (positive in two quadrants, negative in two)."""
    W, H = 1920, 1080
    cam = synthgen.camera(np.eye(3), np.zeros(3), 1100.0, 900.0, W / 2, H / 2, 0.01)
    rng = np.random.default_rng(5)
    pts = []
    for sx in (-1, 1):
        for sy in (-1, 1):
            for _ in range(5):
                z = rng.uniform(0.02, 0.2)
                pts.append([sx * rng.uniform(0.3, 0.8) * z, sy * rng.uniform(0.2, 0.45) * z, z])
    xyz = np.array(pts, np.float32)
    dil = 0.16
    info = oracle.point_info(cam, xyz, H, W, mode="gaussian", sigma=0.0, dilation=dil)
    g = info["gauss"].astype(np.float64)
    s = 5 * 0.01 / 1100.0          # P:201 auto std (R16), larger focal length
    n_pos = n_neg = 0
    for i, p in enumerate(xyz.astype(np.float64)):
        S = ewa_cov(cam, p, s, dil)
        a2, b2, c2 = g[i, 4], g[i, 5], g[i, 6]
        assert a2 == pytest.approx(S[0, 0], rel=1e-5)
        assert c2 == pytest.approx(S[1, 1], rel=1e-5)
        assert b2 == pytest.approx(S[0, 1], rel=1e-5)
        assert abs(S[0, 1]) > 0.05 * np.sqrt(S[0, 0] * S[1, 1]) - dil   # really off-axis
        assert np.sign(b2) == np.sign(p[0] * p[1])
        n_pos += b2 > 0
        n_neg += b2 < 0
        # conic = inverse covariance (sign of the off-diagonal included)
        Si = np.linalg.inv(S)
        assert g[i, 0] == pytest.approx(Si[0, 0], rel=1e-4)
        assert g[i, 1] == pytest.approx(Si[0, 1], rel=1e-4)
        assert g[i, 2] == pytest.approx(Si[1, 1], rel=1e-4)
        # 3-sigma radius from the larger eigenvalue
        assert g[i, 3] == pytest.approx(3 * np.sqrt(np.linalg.eigvalsh(S).max()), rel=1e-5)
    assert n_pos == 10 and n_neg == 10


def test_off_axis_gaussian_pixel_set_is_three_sigma_ellipse():
    """R17: the fragments of an off-axis Gaussian are exactly the pixel
    centres with Mahalanobis q <= 9 under the fp64 EWA covariance (pixels
    within 1e-3 of the boundary skipped: fp32 rounding may decide them)."""
    W, H = 256, 256
    cam = synthgen.camera(np.eye(3), np.zeros(3), 200.0, 160.0, W / 2, H / 2, 0.01)
    xyz = np.array([[0.3 * 0.05, -0.35 * 0.05, 0.05], [-0.4 * 0.04, -0.3 * 0.04, 0.04],
                    [0.5 * 0.03, 0.45 * 0.03, 0.03]], np.float32)
    s = 0.002
    fr = oracle.fragments(cam, xyz, H, W, mode="gaussian", sigma=s, dilation=0.16)
    checked = 0
    for i, p in enumerate(xyz.astype(np.float64)):
        Si = np.linalg.inv(ewa_cov(cam, p, s, 0.16))
        u = cam["fx"] * p[0] / p[2] + cam["cx"]
        v = cam["fy"] * p[1] / p[2] + cam["cy"]
        have = set(fr["pix"][fr["idx"] == i].tolist())
        for py in range(H):
            for px in range(W):
                d = np.array([px + 0.5 - u, py + 0.5 - v])
                q = d @ Si @ d
                if abs(q - 9.0) < 1e-3:
                    continue
                assert ((py * W + px) in have) == (q <= 9.0), (i, px, py, q)
                checked += q <= 9.0
    assert checked > 60     # footprints of several pixels each


# ------------------------------------------------------------------ P:166-173 tile lists
@pytest.mark.parametrize("mode,kw", [("bilinear", {}), ("gaussian", dict(sigma=0.0)),
                                     ("gaussian", dict(sigma=1.5, flags=oracle.SIGMA_IS_PIXELS))])
def test_tile_lists_membership_brute_force(mode, kw):
    """Every (tile, point) pair is listed iff the point's clipped footprint
    rectangle meets the 8x8 tile (brute force over all pairs), each list is
    in (depth, index) order, and sum(tiles_touched) == F_t."""
    c = synthgen.config1(seed=3)
    cam, xyz = c["cams"][0], c["xyz"]
    H, W = c["H"], c["W"]
    ranges, idx = oracle.tile_lists(cam, xyz, H, W, mode=mode, **kw)
    info = oracle.point_info(cam, xyz, H, W, mode=mode, **kw)
    assert int(info["tiles_touched"].sum()) == len(idx) == int(ranges[-1])
    # footprint rectangles from the fragments of a fully unmasked raster
    # (bilinear: the clipped 2x2 block; Gaussian: the clipped 3-sigma bbox,
    # reconstructed from the radius the oracle reports)
    uvz = info["uvz"].astype(np.float64)
    tx_n, ty_n = (W + 7) // 8, (H + 7) // 8
    expect = {t: [] for t in range(tx_n * ty_n)}
    for i in range(len(xyz)):
        if info["depth_key"][i] == 0xFFFFFFFF or info["tiles_touched"][i] == 0:
            continue
        u, v = np.float32(uvz[i, 0]), np.float32(uvz[i, 1])
        if mode == "bilinear":
            x0 = int(np.floor(np.float32(u - np.float32(0.5))))
            y0 = int(np.floor(np.float32(v - np.float32(0.5))))
            xlo, xhi, ylo, yhi = max(x0, 0), min(x0 + 1, W - 1), max(y0, 0), min(y0 + 1, H - 1)
        else:
            r = np.float32(info["gauss"][i, 3])
            ax, ay = np.float32(u - np.float32(0.5)), np.float32(v - np.float32(0.5))
            xlo = max(int(np.ceil(np.float32(ax - r))), 0)
            xhi = min(int(np.floor(np.float32(ax + r))), W - 1)
            ylo = max(int(np.ceil(np.float32(ay - r))), 0)
            yhi = min(int(np.floor(np.float32(ay + r))), H - 1)
        for ty in range(ty_n):
            for tx in range(tx_n):
                if xlo <= 8 * tx + 7 and xhi >= 8 * tx and ylo <= 8 * ty + 7 and yhi >= 8 * ty:
                    expect[ty * tx_n + tx].append((int(info["depth_key"][i]), i))
    for t in range(tx_n * ty_n):
        got = idx[ranges[t]:ranges[t + 1]].tolist()
        want = [i for _, i in sorted(expect[t])]
        assert got == want, t

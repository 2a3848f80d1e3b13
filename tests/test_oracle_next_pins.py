"""Pins for the oracle's NEXT-row functions: degree-2 SH
features (f1) and the equirectangular environment background (f2,
P:185-192).  Checked against mathematics, not against the oracle itself."""
import numpy as np
import pytest

import oracle
import synthgen


def test_sh_dc_constant():
    """Y_00 = 1 / (2 sqrt(pi)) for every direction."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        assert oracle.sh_basis(d)[0] == pytest.approx(0.5 / np.sqrt(np.pi), abs=1e-16)


def test_sh_orthonormal():
    """int_{S^2} Y_k Y_l dOmega = delta_kl (real orthonormal basis) by
    Gauss-Legendre x trapezoid quadrature, exact for these polynomials."""
    nt, nphi = 16, 32
    ct_, wt = np.polynomial.legendre.leggauss(nt)
    phi = np.arange(nphi) * 2 * np.pi / nphi
    G = np.zeros((9, 9))
    for c, w in zip(ct_, wt):
        s = np.sqrt(1 - c * c)
        for p in phi:
            Y = oracle.sh_basis([s * np.cos(p), s * np.sin(p), c])
            G += w * (2 * np.pi / nphi) * np.outer(Y, Y)
    np.testing.assert_allclose(G, np.eye(9), atol=1e-12)


def test_sh_parity_by_degree():
    """Y_lm(-d) = (-1)^l Y_lm(d): degree-1 terms flip, degree-0/2 do not
    (SPEC S:64)."""
    d = np.array([0.3, -0.5, 0.81]); d /= np.linalg.norm(d)
    Yp, Ym = oracle.sh_basis(d), oracle.sh_basis(-d)
    np.testing.assert_allclose(Ym[1:4], -Yp[1:4], atol=1e-15)
    np.testing.assert_allclose(Ym[[0, 4, 5, 6, 7, 8]], Yp[[0, 4, 5, 6, 7, 8]], atol=1e-15)


def test_sh_features_linear_and_directed():
    """Features are linear in the coefficients, and the direction is from the
    camera centre to the point: a point straight ahead of an identity camera
    sees d = +z, so a Y_10-only coefficient gives C1 = sqrt(3/(4 pi))."""
    cam = synthgen.camera(np.eye(3), [0, 0, 0], 64, 64, 32, 32, 0.1)
    xyz = np.array([[0, 0, 2.0], [0.5, -0.2, 3.0]], np.float32)
    rng = np.random.default_rng(1)
    a, b = rng.normal(size=(2, 2, 4, 9))
    fa, _ = oracle.sh_features(cam, xyz, a)
    fb, _ = oracle.sh_features(cam, xyz, b)
    fab, _ = oracle.sh_features(cam, xyz, 2 * a - 3 * b)
    np.testing.assert_allclose(fab, 2 * fa - 3 * fb, atol=1e-12)
    e = np.zeros((2, 4, 9)); e[:, :, 2] = 1.0
    f, _ = oracle.sh_features(cam, xyz, e)
    assert f[0, 0] == pytest.approx(np.sqrt(3 / (4 * np.pi)), abs=1e-12)
    # a translated camera: the centre is -R^T t
    cam2 = synthgen.camera(np.eye(3), [0, 0, -1.0], 64, 64, 32, 32, 0.1)   # centre at z = +1
    f2, _ = oracle.sh_features(cam2, np.array([[0, 0, 0.0]], np.float32), e[:1])
    assert f2[0, 0] == pytest.approx(-np.sqrt(3 / (4 * np.pi)), abs=1e-12)   # d = -z


def test_env_constant_map():
    cam = synthgen.camera(synthgen.random_rotation(np.random.default_rng(2)), [0, 0, 0],
                          50, 50, 16, 16, 0.1)
    env = np.full((16, 32, 3), 0.75, np.float32)
    np.testing.assert_allclose(oracle.env_background(cam, env, 32, 32), 0.75, atol=1e-15)


def test_env_texel_centre_and_seam():
    """A pixel whose ray hits a texel centre returns that texel exactly; the
    ray at u = 0 (the seam) averages the last and first columns (wrap)."""
    He, We = 8, 16
    env = np.random.default_rng(3).uniform(-1, 1, (He, We, 2)).astype(np.float32)
    # identity camera, principal ray d = +z: u = We/2 (a texel edge in u),
    # v = He/2 (a texel edge in v) -> average of 4 texels
    cam = synthgen.camera(np.eye(3), [0, 0, 0], 64, 64, 0.5, 0.5, 0.1)
    bg = oracle.env_background(cam, env, 1, 1)[0, 0]
    exp = env[He // 2 - 1:He // 2 + 1, We // 2 - 1:We // 2 + 1].astype(np.float64).mean(axis=(0, 1))
    np.testing.assert_allclose(bg, exp, atol=1e-7)
    # camera looking along -z: azimuth pi -> u = We (seam): average of columns
    # We-1 and 0 (and rows He/2-1, He/2)
    R = np.diag([-1.0, 1.0, -1.0])
    cam = synthgen.camera(R, [0, 0, 0], 64, 64, 0.5, 0.5, 0.1)
    bg = oracle.env_background(cam, env, 1, 1)[0, 0]
    cols = env[He // 2 - 1:He // 2 + 1][:, [We - 1, 0]].astype(np.float64)
    np.testing.assert_allclose(bg, cols.mean(axis=(0, 1)), atol=1e-7)


def test_env_pole_clamp():
    """Straight up (d_y = -1 in the +y-down camera convention here maps to
    v = acos(-1)/pi He = He): the polar clamp returns the last row."""
    He, We = 4, 8
    env = np.zeros((He, We, 1), np.float32); env[-1] = 5.0
    # camera whose +z axis is world -y: rows of R are the camera axes
    R = np.array([[1.0, 0, 0], [0, 0, -1.0], [0, -1.0, 0]])
    cam = synthgen.camera(R, [0, 0, 0], 64, 64, 0.5, 0.5, 0.1)
    np.testing.assert_allclose(oracle.env_background(cam, env, 1, 1), 5.0, atol=1e-7)

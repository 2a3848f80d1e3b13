"""Pins for the CPU oracle (Q1-Q16): the oracle is checked
against what the paper and the mathematics fix, never against itself.

Each test names the passage it pins.  P:n = PAPER.md line n, S:n = SPEC.md.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synthgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def cam_id(W, H, f=64.0, z_near=0.1):
    """Identity pose; f a power of two so pixel positions are exact."""
    return synthgen.camera(np.eye(3), np.zeros(3), f, f, W / 2, H / 2, z_near)


def pts_at(cam, uvz):
    """Camera-space points that project exactly to (u, v) when f and z are
    powers of two (inverse pinhole, not the method's arithmetic)."""
    uvz = np.asarray(uvz, np.float64).reshape(-1, 3)
    x = (uvz[:, 0] - cam["cx"]) / cam["fx"] * uvz[:, 2]
    y = (uvz[:, 1] - cam["cy"]) / cam["fy"] * uvz[:, 2]
    return np.stack([x, y, uvz[:, 2]], 1).astype(np.float32)


# --------------------------------------------------------------------- Q1
def test_q1_bilinear_weights_sum_to_one():
    """'the bilinear interpolation weights across the 2x2 fragments of
    each point sum to one'.  fp64 weights exactly 1 (1e-12); fp32 weights
    within 2^-22 (four rounded products)."""
    rng = np.random.default_rng(11)
    W = H = 512
    cam = cam_id(W, H, f=256.0)
    n = 20000
    u = rng.uniform(4, W - 4, n); v = rng.uniform(4, H - 4, n)
    xyz = np.stack([(u - W / 2) / 256.0, (v - H / 2) / 256.0, np.ones(n)], 1).astype(np.float32)
    fr = oracle.fragments(cam, xyz, H, W)
    assert len(fr["idx"]) == 4 * n                     # interior: all 4 pixels
    s64 = np.bincount(fr["idx"], weights=fr["w64"], minlength=n)
    s32 = np.bincount(fr["idx"], weights=fr["w32"].astype(np.float64), minlength=n)
    assert np.max(np.abs(s64 - 1.0)) < 1e-12
    assert np.max(np.abs(s32 - 1.0)) <= 2.0 ** -22
    # the four pixels are the block floor(u-1/2) + {0,1} (R3)
    uvz = oracle.point_info(cam, xyz, H, W)["uvz"]
    x0 = np.floor(uvz[:, 0].astype(np.float64) - 0.5).astype(np.int64)
    px = fr["pix"] % W
    assert np.all((px - x0[fr["idx"]] >= 0) & (px - x0[fr["idx"]] <= 1))


# --------------------------------------------------------------------- Q2
def test_q2_tiles_per_2x2_splat_exact():
    """a 2x2 splat contributes on average to 1.27 tiles of 8x8.
    Exhaustive over all 8x8 sub-tile block origins (tile-periodic) the mean is
    exactly (9/8)^2 = 1.265625; a continuous 2-px footprint would give 1.5625
    (R3)."""
    W = H = 1024
    cam = cam_id(W, H, f=512.0)
    xs = np.arange(200, 264) + 0.75   # 64 consecutive block origins, all residues mod 8
    u, v = np.meshgrid(xs, xs)
    xyz = pts_at(cam, np.stack([u.ravel(), v.ravel(), np.ones(u.size)], 1))
    t = oracle.point_info(cam, xyz, H, W)["tiles_touched"]
    assert t.mean() == pytest.approx(1.265625, abs=0)
    assert set(np.unique(t)) == {1, 2, 4}


def test_q2_tiles_per_splat_monte_carlo():
    """P:168 '1.27' by Monte Carlo over uniform sub-pixel positions."""
    rng = np.random.default_rng(12)
    W = H = 2048
    cam = cam_id(W, H, f=1024.0)
    n = 400000
    u = rng.uniform(16, W - 16, n); v = rng.uniform(16, H - 16, n)
    xyz = np.stack([(u - W / 2) / 1024.0, (v - H / 2) / 1024.0, np.ones(n)], 1).astype(np.float32)
    t = oracle.point_info(cam, xyz, H, W)["tiles_touched"]
    assert abs(t.mean() - 1.265625) < 0.004
    assert round(float(t.mean()), 2) == 1.27


# --------------------------------------------------------------------- Q4
def test_q4_eq1_worked_example_golden():
    """Eq. 1 + background on the fixture of S:276."""
    g = json.load(open(os.path.join(GOLD, "eq1_worked_example.json")))
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    fr = g["fragments_front_to_back"]
    # both points project exactly onto the centre of pixel (5, 7): w = 1
    xyz = pts_at(cam, [[5.5, 7.5, f["depth"]] for f in fr])
    feat = np.array([f["feature"] for f in fr])
    op = np.array([f["alpha"] for f in fr])
    bg = np.zeros((H, W, 4)); bg[...] = g["background"]
    r = oracle.render(cam, xyz, feat, op, H, W, bg=bg, t_min=0.0)
    e = g["expected"]
    np.testing.assert_allclose(r["F"][7, 5], e["F"], atol=1e-15)
    assert r["A"][7, 5] == pytest.approx(e["A"], abs=1e-15)
    assert r["T"][7, 5] == pytest.approx(e["T_final"], abs=0)
    assert r["D"][7, 5] == pytest.approx(e["D_unnormalised"], abs=1e-15)
    # the weight-0 neighbours of the 2x2 blocks are fragments (n_frag) but
    # change nothing; pixels with no fragments show the background
    assert r["n_frag"][7, 5] == 2 and r["n_frag"][7, 6] == 2 and r["n_frag"][8, 6] == 2
    np.testing.assert_allclose(r["F"][8, 6], g["background"], atol=0)
    np.testing.assert_allclose(r["F"][0, 0], g["background"], atol=0)
    assert r["A"][0, 0] == 0 and r["D"][0, 0] == 0


def test_q4_three_fragments_closed_form():
    """Eq. 1 with three fragments, out-of-order input and a clamp: sorted by
    depth, alpha = min(o*w, alpha_max) (R4/R5), T_i = prod_{j<i}(1-alpha_j)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    # input order deliberately not depth order
    xyz = pts_at(cam, [[3.5, 3.5, 4.0], [3.5, 3.5, 1.0], [3.5, 3.5, 2.0]])
    feat = np.array([[3.0], [1.0], [2.0]])
    op = np.array([0.25, 1.0, 0.5])   # the depth-1 point clamps to 0.99
    r = oracle.render(cam, xyz, feat, op, H, W, t_min=0.0)
    a = [0.99, 0.5, 0.25]; f = [1.0, 2.0, 3.0]; z = [1.0, 2.0, 4.0]
    T = [1.0, 0.01, 0.005]
    assert r["F"][3, 3, 0] == pytest.approx(sum(T[k] * a[k] * f[k] for k in range(3)), rel=1e-7)
    assert r["D"][3, 3] == pytest.approx(sum(T[k] * a[k] * z[k] for k in range(3)), rel=1e-7)
    assert r["A"][3, 3] == pytest.approx(1 - 0.005 * 0.75, rel=1e-7)


# --------------------------------------------------------------------- Q5
def test_q5_energy_conservation():
    """sum_k T_k alpha_k + T_final = 1 (telescoping of Eq. 1): with
    f = 1 the feature image equals the alpha image, and F + T = 1."""
    c = synthgen.config1()
    N = c["xyz"].shape[0]
    r = oracle.render(c["cams"][0], c["xyz"], np.ones((N, 1)), c["opacity"], c["H"], c["W"])
    np.testing.assert_allclose(r["F"][..., 0], r["A"], atol=1e-12)
    # fp32 decision transmittance agrees with the fp64 value to fp32 rounding
    np.testing.assert_allclose(r["T"], 1 - r["A"], atol=2e-6)


# --------------------------------------------------------------------- Q6
def test_q6_single_fragment_gradient_f_minus_b():
    """Eq. 2 special case K=1 (sign corrected, R12):
    F = a f + (1-a) b  =>  dF/da = f - b (the paper-literal '+ T f_bg'
    would give f + b)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    xyz = pts_at(cam, [[6.5, 6.5, 2.0]])
    f, b, o = 0.7, 0.2, 0.4
    bg = np.full((H, W, 1), b)
    gF = np.zeros((H, W, 1)); gF[6, 6] = 1.0
    g = oracle.backward(cam, xyz, [[f]], [o], H, W, gF, bg=bg, t_min=0.0)
    assert g["g_opacity"][0] == pytest.approx(f - b, abs=1e-15)     # w = 1
    assert g["g_feat"][0, 0] == pytest.approx(o, abs=1e-15)         # T alpha
    r = oracle.render(cam, xyz, [[f]], [o], H, W, bg=bg, t_min=0.0)
    assert r["F"][6, 6, 0] == pytest.approx(o * f + (1 - o) * b, abs=1e-15)


# --------------------------------------------------------------------- Q7/Q8
def _loss(cam, xyz, feat, op, H, W, gF, gA, gD, bg, mode, kw):
    r = oracle.render(cam, xyz, feat, op, H, W, bg=bg, mode=mode, t_min=0.0, **kw)
    return float((r["F"] * gF).sum() + (r["A"] * gA).sum() + (r["D"] * gD).sum())


def _fd_scene(seed, mode, n=48, W=16, H=16):
    rng = np.random.default_rng(seed)
    cam = cam_id(W, H, f=16.0)
    # crowd the points into the middle so that pixels hold several fragments
    u = rng.uniform(4, 12, n); v = rng.uniform(4, 12, n); z = rng.uniform(1, 3, n)
    xyz = pts_at(cam, np.stack([u, v, z], 1))
    feat = rng.uniform(-1, 1, (n, 3))
    op = rng.uniform(0.05, 0.9, n)       # o*w <= 0.9 < alpha_max: away from the clamp kink
    op[0] = 0.0                          # an alpha = 0 point
    gF = rng.standard_normal((H, W, 3)); gA = rng.standard_normal((H, W))
    gD = rng.standard_normal((H, W)); bg = rng.uniform(-1, 1, (H, W, 3))
    return cam, xyz, feat, op, gF, gA, gD, bg


@pytest.mark.parametrize("mode,kw", [("bilinear", {}),
                                     ("gaussian", dict(sigma=0.6, flags=oracle.SIGMA_IS_PIXELS)),
                                     ("gaussian", dict(sigma=0.02))])
def test_q7_backward_matches_finite_differences(mode, kw):
    """Analytic backward against central finite differences of the
    fp64 forward, including alpha = 0 fragments, background and depth/alpha
    outputs.  Tiny scene, T_min = 0."""
    cam, xyz, feat, op, gF, gA, gD, bg = _fd_scene(7, mode)
    H = W = 16
    g = oracle.backward(cam, xyz, feat, op, H, W, gF, gA, gD, mode=mode, bg=bg, t_min=0.0, **kw)
    h = 1e-6
    worst = 0.0
    for i in range(xyz.shape[0]):
        o2 = op.copy(); o2[i] += h; lp = _loss(cam, xyz, feat, o2, H, W, gF, gA, gD, bg, mode, kw)
        o2[i] -= 2 * h; lm = _loss(cam, xyz, feat, o2, H, W, gF, gA, gD, bg, mode, kw)
        fd = (lp - lm) / (2 * h)
        worst = max(worst, abs(fd - g["g_opacity"][i]) / max(1.0, abs(fd)))
        for c in range(3):
            f2 = feat.copy(); f2[i, c] += h
            lp = _loss(cam, xyz, f2, op, H, W, gF, gA, gD, bg, mode, kw)
            f2[i, c] -= 2 * h
            lm = _loss(cam, xyz, f2, op, H, W, gF, gA, gD, bg, mode, kw)
            fd = (lp - lm) / (2 * h)
            worst = max(worst, abs(fd - g["g_feat"][i, c]) / max(1.0, abs(fd)))
    assert worst < 1e-6
    # Q8: the opacity-0 point still receives a (non-zero) opacity gradient
    assert abs(g["g_opacity"][0]) > 1e-3


def test_q8_skip_zero_alpha_reproduces_original():
    """INPC skipped alpha = 0 fragments; the flag reproduces that (A/B)
    and then the opacity-0 point gets no gradient."""
    cam, xyz, feat, op, gF, gA, gD, bg = _fd_scene(7, "bilinear")
    g = oracle.backward(cam, xyz, feat, op, 16, 16, gF, gA, gD, bg=bg, t_min=0.0,
                        flags=oracle.SKIP_ZERO_ALPHA_GRAD)
    assert g["g_opacity"][0] == 0.0
    g2 = oracle.backward(cam, xyz, feat, op, 16, 16, gF, gA, gD, bg=bg, t_min=0.0)
    assert g2["g_opacity"][0] != 0.0


# --------------------------------------------------------------------- Q9-Q12 (Gaussian)
def test_q9_near_plane_five_pixels():
    """world scale such that the std of a Gaussian at the near plane,
    projected to the image centre, is five pixels -> s = 5 z_near/max(fx,fy)."""
    W, H = 1920, 1080
    cam = synthgen.camera(np.eye(3), np.zeros(3), 1100.0, 1000.0, W / 2, H / 2, 0.01)
    z = 0.01 * (1 + 2.0 ** -12)
    xyz = np.array([[0.0, 0.0, z]], np.float32)
    g = oracle.point_info(cam, xyz, H, W, mode="gaussian", dilation=0.0)["gauss"][0]
    zf = float(np.float32(z))
    assert np.sqrt(g[4]) == pytest.approx(5.0 * 0.01 / zf, rel=2e-6)   # larger focal
    assert np.sqrt(g[6]) == pytest.approx(5.0 * 0.01 / zf * 1000 / 1100, rel=2e-6)


def test_q10_far_field_dilation():
    """far away the footprint is the dilation alone, variance 0.16
    -> sigma = 0.4 px, 3 sigma = 1.2 px, 'slightly larger than a pixel':
    every point covers 4..6 pixel centres; mean tiles of the bbox
    (1 + 1.4/8)^2 = 1.3806."""
    rng = np.random.default_rng(13)
    W = H = 1024
    cam = cam_id(W, H, f=512.0, z_near=0.01)
    n = 20000
    z = 4096.0
    u = rng.uniform(64, W - 64, n); v = rng.uniform(64, H - 64, n)
    xyz = np.stack([(u - W / 2) / 512.0 * z, (v - H / 2) / 512.0 * z, np.full(n, z)], 1).astype(np.float32)
    info = oracle.point_info(cam, xyz, H, W, mode="gaussian")
    np.testing.assert_allclose(info["gauss"][:, 3], 1.2, rtol=1e-4)
    cnt = np.bincount(oracle.fragments(cam, xyz, H, W, mode="gaussian")["idx"], minlength=n)
    assert cnt.min() >= 4 and cnt.max() <= 6
    assert abs(info["tiles_touched"].mean() - (1 + 1.4 / 8) ** 2) < 0.01


def test_q10_three_sigma_weight():
    """3 sigma truncation: a pixel centre at exactly 3 sigma is the
    last included ring, weight e^-4.5."""
    W = H = 32
    cam = cam_id(W, H, f=32.0)
    xyz = pts_at(cam, [[13.5, 10.5, 1.0]])          # 3 px right of pixel (10, 10)
    fr = oracle.fragments(cam, xyz, H, W, mode="gaussian", sigma=1.0, dilation=0.0,
                          flags=oracle.SIGMA_IS_PIXELS)
    w = dict(zip(fr["pix"].tolist(), fr["w64"].tolist()))
    assert w[10 * W + 10] == pytest.approx(np.exp(-4.5), rel=1e-12)
    assert 10 * W + 9 not in w                      # 4 sigma: cut
    assert len(w) == 29                             # lattice points in a radius-3 disc


def test_q11_on_axis_ewa():
    """on the optical axis J = diag(f/z, f/z) so Sigma2D = ((s f/z)^2
    + 0.16) I."""
    W, H = 1920, 1080
    cam = synthgen.camera(np.eye(3), np.zeros(3), 1100.0, 1100.0, W / 2, H / 2, 0.01)
    for z in (0.02, 0.5, 7.0):
        g = oracle.point_info(cam, np.array([[0, 0, z]], np.float32), H, W, mode="gaussian",
                              sigma=0.003)["gauss"][0]
        assert g[5] == 0.0 and g[4] == g[6]
        assert g[4] == pytest.approx((0.003 * 1100 / np.float32(z)) ** 2 + 0.16, rel=1e-5)


def test_q12_footprint_monotone_in_depth():
    """the Gaussian footprint grows as the point comes closer."""
    W = H = 256
    cam = cam_id(W, H, f=128.0, z_near=0.001)
    counts = []
    for z in [0.01 * 1.5 ** k for k in range(14)]:
        xyz = pts_at(cam, [[100.3, 90.7, z]])
        counts.append(len(oracle.fragments(cam, xyz, H, W, mode="gaussian", sigma=0.0004)["idx"]))
    assert all(a >= b for a, b in zip(counts, counts[1:])) and counts[0] > 50 * counts[-1]


# --------------------------------------------------------------------- Q13
def test_q13_point_order_invariance():
    """Permuting the input points permutes nothing in the image (the order is
    fixed by (depth, index) with distinct depths) and permutes gradients."""
    c = synthgen.config1()
    xyz = c["xyz"].copy()
    rng = np.random.default_rng(3)
    xyz[:, 2] += rng.uniform(0, 1e-3, len(xyz)).astype(np.float32)   # distinct depths
    N = len(xyz)
    perm = rng.permutation(N)
    cam, H, W = c["cams"][0], c["H"], c["W"]
    r1 = oracle.render(cam, xyz, c["feat"], c["opacity"], H, W)
    r2 = oracle.render(cam, xyz[perm], c["feat"][perm], c["opacity"][perm], H, W)
    for k in ("F", "A", "D", "T", "n_contrib", "n_frag"):
        np.testing.assert_array_equal(r1[k], r2[k])
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(1, 1, H, W, 4))
    g1 = oracle.backward(cam, xyz, c["feat"], c["opacity"], H, W, gF, gA, gD)
    g2 = oracle.backward(cam, xyz[perm], c["feat"][perm], c["opacity"][perm], H, W, gF, gA, gD)
    np.testing.assert_allclose(g2["g_feat"], g1["g_feat"][perm], atol=1e-12)
    np.testing.assert_allclose(g2["g_opacity"], g1["g_opacity"][perm], atol=1e-12)


# --------------------------------------------------------------------- Q14
@pytest.mark.parametrize("mode", ["bilinear", "gaussian"])
def test_q14_orderings_agree(mode):
    """the per-pixel order of the original single 64-bit sort (P:100,
    P:159-162) equals the per-pixel (depth, idx) sort, and equals each tile
    list restricted to the pixel's fragments."""
    c = synthgen.config1()
    cam, H, W = c["cams"][0], c["H"], c["W"]
    kw = dict(sigma=0.8, flags=oracle.SIGMA_IS_PIXELS) if mode == "gaussian" else {}
    r0, i0 = oracle.pixel_lists(cam, c["xyz"], H, W, 0, mode=mode, **kw)
    r1, i1 = oracle.pixel_lists(cam, c["xyz"], H, W, 1, mode=mode, **kw)
    np.testing.assert_array_equal(r0, r1)
    np.testing.assert_array_equal(i0, i1)
    tr, ti = oracle.tile_lists(cam, c["xyz"], H, W, mode=mode, **kw)
    fr = oracle.fragments(cam, c["xyz"], H, W, mode=mode, **kw)
    covers = {}
    for p, i in zip(fr["pix"].tolist(), fr["idx"].tolist()):
        covers.setdefault(p, set()).add(i)
    tx_n = (W + 7) // 8
    for p in range(H * W):
        t = (p // W // 8) * tx_n + (p % W) // 8
        lst = [i for i in ti[tr[t]:tr[t + 1]].tolist() if i in covers.get(p, ())]
        assert lst == i0[r0[p]:r0[p + 1]].tolist()


def test_q14_sort_cost_accounting():
    """1080p needs a 21-bit pixel index and a 15-bit tile
    index (32,400 tiles); pass x key counts 28n -> 7.62n -> 6.54n; key memory
    (4 + 2*1.27)/8 -> 18 % less (R21)."""
    W, H = 1920, 1080
    assert (H * W - 1).bit_length() == 21
    assert oracle.n_tiles(H, W) == 32400 and (32400 - 1).bit_length() == 15
    import math
    assert 4 * math.ceil((32 + 21) / 8) == 28
    assert 1.27 * math.ceil((32 + 15) / 8) == pytest.approx(7.62)
    assert 4 + 1.27 * math.ceil(15 / 8) == pytest.approx(6.54)
    assert round(100 * (1 - (4 + 2 * 1.27) / 8)) == 18


# --------------------------------------------------------------------- Q15
def test_q15_single_opaque_point_at_pixel_centre():
    """One point with o = 1 on a pixel centre: that pixel gets alpha_max
    (R5) and F = alpha_max f; the other three fragments have w = 0 (counted,
    contributing nothing)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    xyz = pts_at(cam, [[9.5, 4.5, 2.0]])
    r = oracle.render(cam, xyz, [[2.0, -1.0]], [1.0], H, W)
    am = float(np.float32(0.99))
    np.testing.assert_allclose(r["F"][4, 9], [am * 2.0, -am], rtol=1e-15)
    assert r["n_frag"].sum() == 4 and r["n_frag"][4, 9] == 1
    assert r["n_frag"][5, 10] == 1 and r["F"][5, 10].tolist() == [0.0, 0.0]
    assert r["n_contrib"][5, 10] == 1            # processed (alpha 0), not terminated


def test_q15_plane_is_2d_bilinear_scatter():
    """Identity camera and all points on the plane z = 1 (exact depth ties,
    broken by index R8): with isolated points and o = 1/4 the image is the
    textbook 2-D bilinear scatter of o*f."""
    W = H = 32
    cam = cam_id(W, H, f=32.0)
    rng = np.random.default_rng(4)
    # points far apart so each pixel holds at most one fragment
    # sub-pixel offsets on a 1/64 grid: exactly representable, exact projection
    centres = [(4 + 6 * i + 0.5 + rng.integers(0, 64) / 64, 4 + 6 * j + 0.5 + rng.integers(0, 64) / 64)
               for i in range(4) for j in range(4)]
    xyz = pts_at(cam, [[u, v, 1.0] for u, v in centres])
    n = len(centres)
    feat = rng.uniform(-1, 1, (n, 1)); op = np.full(n, 0.25)
    r = oracle.render(cam, xyz, feat, op, H, W)
    img = np.zeros((H, W))
    for k, (u, v) in enumerate(centres):
        a, b = np.float32(u) - 0.5, np.float32(v) - 0.5
        x0, y0 = int(np.floor(a)), int(np.floor(b))
        fa, fb = float(a - x0), float(b - y0)
        for dy, wy in ((0, 1 - fb), (1, fb)):
            for dx, wx in ((0, 1 - fa), (1, fa)):
                img[y0 + dy, x0 + dx] += 0.25 * wx * wy * feat[k, 0]
    np.testing.assert_allclose(r["F"][..., 0], img, atol=1e-15)


def test_q15_tie_break_by_index():
    """Exact depth ties are ordered by ascending point index (R8)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    xyz = pts_at(cam, [[5.5, 5.5, 2.0]] * 3)
    r = oracle.render(cam, xyz, [[1.0], [2.0], [3.0]], [0.5, 0.5, 0.5], H, W, t_min=0)
    assert r["F"][5, 5, 0] == pytest.approx(0.5 * 1 + 0.25 * 2 + 0.125 * 3, abs=1e-15)
    tr, ti = oracle.tile_lists(cam, xyz, H, W)
    assert ti.tolist() == [0, 1, 2]


def test_q15_early_termination_rule():
    """R6: before compositing fragment k, stop if T (1 - alpha_k) < T_min;
    fragment k and all later ones are excluded (fp32 recurrence)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    xyz = pts_at(cam, [[5.5, 5.5, 1.0 + k] for k in range(6)])
    op = [0.9] * 6
    r = oracle.render(cam, xyz, np.ones((6, 1)), op, H, W, t_min=1e-4)
    # T after k fragments = 0.1^k in fp32; 1e-4 reached at k = 4 -> 0.1^4 < 1e-4?
    T = np.float32(1.0)
    n = 0
    for k in range(6):
        Tn = np.float32(T * np.float32(np.float32(1.0) - np.float32(0.9)))
        if Tn < np.float32(1e-4):
            break
        T, n = Tn, k + 1
    assert r["n_contrib"][5, 5] == n and n in (3, 4)
    assert r["T"][5, 5] == T


# --------------------------------------------------------------------- Q16
def test_q16_thread_count_determinism():
    """output independent of the worker-thread count."""
    c = synthgen.config1(seed=5, N=3000)
    cam, H, W = c["cams"][0], c["H"], c["W"]
    r1 = oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, threads=1)
    r8 = oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, threads=8)
    for k in r1:
        np.testing.assert_array_equal(r1[k], r8[k])
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(5, 1, H, W, 4))
    g1 = oracle.backward(cam, c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD, threads=1)
    g8 = oracle.backward(cam, c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD, threads=8)
    np.testing.assert_allclose(g1["g_feat"], g8["g_feat"], atol=1e-12)


def test_culling_rules():
    """R9: cull !(z_c > z_near) and non-finite; off-image blocks emit nothing;
    culled points have key 0xFFFFFFFF; depth key = float bits of z_c (R7)."""
    W = H = 16
    cam = cam_id(W, H, f=16.0, z_near=0.5)
    xyz = np.array([[0, 0, 0.5], [0, 0, -1], [np.nan, 0, 1], [0, 0, np.inf],
                    [100, 0, 1], [0, 0, 1.5]], np.float32)
    info = oracle.point_info(cam, xyz, H, W)
    k = info["depth_key"]
    assert k[0] == k[1] == k[2] == k[3] == 0xFFFFFFFF
    assert k[4] == np.float32(1.0).view(np.uint32) and info["tiles_touched"][4] == 0
    # (0,0) projects to the image centre u = v = 8, a tile corner: block
    # {7,8} x {7,8} straddles both tile boundaries -> 4 tiles
    assert k[5] == np.float32(1.5).view(np.uint32) and info["tiles_touched"][5] == 4
    # order-preserving: keys of positive floats sort like the floats
    z = np.sort(np.random.default_rng(0).uniform(0.01, 100, 1000).astype(np.float32))
    assert np.all(np.diff(z.view(np.uint32).astype(np.int64)) >= 0)


def test_block_partly_off_image():
    """R3: a block straddling the border keeps its in-image pixels without
    renormalising; a block fully outside (u - 1/2 < -1) emits nothing."""
    W = H = 16
    cam = cam_id(W, H, f=16.0)
    xyz = pts_at(cam, [[0.25, 8.5, 1.0], [-0.75, 8.5, 1.0], [15.75, 8.5, 1.0]])
    fr = oracle.fragments(cam, xyz, H, W)
    by = {}
    for p, i, w in zip(fr["pix"].tolist(), fr["idx"].tolist(), fr["w64"].tolist()):
        by.setdefault(i, []).append((p % W, p // W, w))
    assert sorted(by[0]) == [(0, 8, 0.75), (0, 9, 0.0)]     # x0 = -1: column -1 dropped
    assert 1 not in by                                      # u - 1/2 = -1.25 < -1
    assert sorted(by[2]) == [(15, 8, 0.75), (15, 9, 0.0)]   # x0 = 15: column 16 dropped

"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Gates (BASELINE.json north_star):
  * bit-exact: depth keys, tiles per point, tile ranges, per-tile sorted point
    indices, per-pixel fragment counts, n_contrib (bilinear; Gaussian: R24);
  * max abs error <= 1e-4 on F, A, D;
  * gradients: |g - g*| <= 1e-3 |g*| + 1e-6 max|g*| elementwise.
"""
import numpy as np
import pytest

import oracle
import synthgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

IMG_TOL = 1e-4


@pytest.fixture(scope="module")
def inpc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2508_19140_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(inpc):
    return inpc.Context(0)


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def gpu_forward(inpc, ctx, c, mode=None, bg=None, band=None, debug=True, **kw):
    cfgk = dict(kw)
    cfg = inpc.make_cfg(c["H"], c["W"], c["feat"].shape[-1], mode or c["mode"], band=band,
                        flags=(inpc.FLAG_DEBUG if debug else 0) | cfgk.pop("flags", 0), **cfgk)
    xyz, feat, op = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"])
    bgt = None if bg is None else dev(bg)
    out = ctx.forward(cfg, c["cams"], xyz, feat, op, bg=bgt, debug_counts=debug)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    if debug:
        ex = ctx.debug_export(0, N=xyz.shape[0], H=c["H"], W=c["W"])
        res.update({k: (v.cpu().numpy().view(np.uint32) if hasattr(v, "cpu") else v)
                    for k, v in ex.items()})
    return cfg, (xyz, feat, op, bgt), res


def oracle_kw(kw):
    return {k: v for k, v in kw.items() if k in ("sigma", "dilation", "alpha_max", "t_min", "flags")}


def check_lists(c, res, mode, band=None, **kw):
    cam, H, W = c["cams"][0], c["H"], c["W"]
    info = oracle.point_info(cam, c["xyz"], H, W, mode=mode, **oracle_kw(kw))
    N = c["xyz"].shape[0]
    if N:
        np.testing.assert_array_equal(res["depth_keys"][:N], info["depth_key"])
        np.testing.assert_array_equal(res["tiles_touched"][:N], info["tiles_touched"])
    tr, ti = oracle.tile_lists(cam, c["xyz"], H, W, mode=mode, band=band, **oracle_kw(kw))
    np.testing.assert_array_equal(res["tile_ranges"], tr)
    assert res["F_t"] == len(ti)
    np.testing.assert_array_equal(res["sorted_idx"], ti)


def check_image(c, res, mode, bg=None, band=None, exact_ncontrib=True, pixel_mask=None, **kw):
    cam, H, W = c["cams"][0], c["H"], c["W"]
    r = oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, mode=mode, bg=bg,
                      pixel_mask=pixel_mask, threads=oracle.max_threads(), **oracle_kw(kw))
    rows = slice(None)
    if band is not None:
        rows = slice(band[0] * 8, min(band[1] * 8, H))
    sel = np.ones((H, W), bool) if pixel_mask is None else pixel_mask.astype(bool)
    selr = sel[rows]
    np.testing.assert_array_equal(res["nfrag"][0][rows][selr], r["n_frag"][rows][selr])
    nc_g, nc_o = res["ncontrib"][0][rows][selr], r["n_contrib"][rows][selr]
    if exact_ncontrib:
        np.testing.assert_array_equal(nc_g, nc_o)
        ok = np.ones_like(nc_g, bool)
    else:   # R24: expf ulps may move a termination decision on rare pixels
        ok = nc_g == nc_o
        assert (~ok).sum() <= max(2, 1e-4 * ok.size), (~ok).sum()
    Fg = res["F"][0][rows][selr][ok]
    np.testing.assert_allclose(Fg, r["F"][rows][selr][ok], atol=IMG_TOL, rtol=0)
    np.testing.assert_allclose(res["A"][0][rows][selr][ok], r["A"][rows][selr][ok], atol=IMG_TOL, rtol=0)
    np.testing.assert_allclose(res["D"][0][rows][selr][ok], r["D"][rows][selr][ok], atol=IMG_TOL, rtol=0)
    return r


def check_grads(g_gpu, g_or):
    g, gs = np.asarray(g_gpu, np.float64), np.asarray(g_or, np.float64)
    scale = np.abs(gs).max() if gs.size else 0.0
    err = np.abs(g - gs)
    bad = err > 1e-3 * np.abs(gs) + 1e-6 * scale
    assert not bad.any(), (bad.sum(), err.max(), scale)
    if scale > 0:
        assert err.max() / scale <= 1e-3


def run_full(inpc, ctx, c, mode=None, bg=None, band=None, bwd=True, exact_ncontrib=True, **kw):
    mode = mode or c["mode"]
    cfg, (xyz, feat, op, bgt), res = gpu_forward(inpc, ctx, c, mode, bg=bg, band=band, **kw)
    check_lists(c, res, mode, band=band, **kw)
    check_image(c, res, mode, bg=bg, band=band, exact_ncontrib=exact_ncontrib, **kw)
    if bwd:
        H, W, C = c["H"], c["W"], c["feat"].shape[-1]
        gF, gA, gD = (x[0] for x in synthgen.upstream_grads(7, 1, H, W, C))
        if band is not None:   # gradients only flow from the band's pixels
            m = np.zeros((H, W), bool); m[band[0] * 8: band[1] * 8] = True
            gF = gF * m[..., None]; gA = gA * m; gD = gD * m
        gf, go = ctx.backward(cfg, c["cams"], xyz, feat, op, dev(gF), dev(gA), dev(gD), bg=bgt)
        torch.cuda.synchronize()
        o = oracle.backward(c["cams"][0], c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD,
                            mode=mode, bg=bg, threads=oracle.max_threads(), **oracle_kw(kw))
        check_grads(gf.cpu().numpy(), o["g_feat"])
        check_grads(go.cpu().numpy(), o["g_opacity"])
    return res


# ------------------------------------------------------------------ config 1
def test_cfg1_bilinear_fwd_bwd(inpc, ctx):
    run_full(inpc, ctx, synthgen.config1())


@pytest.mark.parametrize("seed", range(100, 110))
def test_cfg1_seed_sweep(inpc, ctx, seed):
    run_full(inpc, ctx, synthgen.config1(seed=seed))


def test_cfg1_background_and_tmin_off(inpc, ctx):
    c = synthgen.config1(seed=3)
    bg = np.random.default_rng(0).uniform(-1, 1, (c["H"], c["W"], 4)).astype(np.float32)
    run_full(inpc, ctx, c, bg=bg)
    run_full(inpc, ctx, c, t_min=0.0)


def test_cfg1_skip_zero_alpha_flag(inpc, ctx):
    run_full(inpc, ctx, synthgen.config1(seed=4), flags=inpc.FLAG_SKIP_ZERO_ALPHA_GRAD)


@pytest.mark.parametrize("C", [1, 3, 8, 17, 64])
def test_channel_counts(inpc, ctx, C):
    c = synthgen.config1(seed=20 + C, C=C)
    run_full(inpc, ctx, c)


@pytest.mark.parametrize("HW", [(67, 53), (9, 130), (1, 1), (8, 8)])
def test_ragged_images(inpc, ctx, HW):
    H, W = HW
    c = synthgen.config1(seed=31, N=600, H=H, W=W)
    run_full(inpc, ctx, c)


def test_band_restriction(inpc, ctx):
    c = synthgen.config1(seed=8)
    run_full(inpc, ctx, c, band=(2, 5))


# ------------------------------------------------------------------ edge cases
def test_empty_cloud_is_background(inpc, ctx):
    c = synthgen.config1()
    c = dict(c, xyz=c["xyz"][:0], feat=c["feat"][:0], opacity=c["opacity"][:0])
    bg = np.full((c["H"], c["W"], 4), 0.25, np.float32)
    res = run_full(inpc, ctx, c, bg=bg, bwd=False)
    assert np.all(res["F"] == 0.25) and np.all(res["A"] == 0) and np.all(res["nfrag"] == 0)


def test_all_culled(inpc, ctx):
    c = synthgen.config1()
    c = dict(c, xyz=c["xyz"] * np.float32(-1.0))
    res = run_full(inpc, ctx, c)
    assert res["F_t"] == 0


@pytest.mark.parametrize("n", [1500, 5000, 40000])
def test_one_hot_tile_over_smem_cap(inpc, ctx, n, ties="long"):
    """Degenerate skew: every point in one 8x8 tile -> the tile list exceeds
    the in-SMEM sort cap and goes through the big-tile chunk sort + merges.
    ties: "long" = 10% of the points share one depth (a run over the radix
    tie fix-up's limit), "short" = pairs and triples of equal depths, "none"."""
    rng = np.random.default_rng(n)
    W = H = 64
    cam = synthgen.camera(np.eye(3), np.zeros(3), 64.0, 64.0, 32, 32, 0.1)
    u = rng.uniform(17, 23, n); v = rng.uniform(9, 15, n); z = rng.uniform(1, 4, n)
    if ties == "long":
        z[: n // 10] = 2.0                    # exact depth ties
    elif ties == "short":
        k = n // 6
        z[k:2 * k] = z[:k]                    # pairs
        z[2 * k:3 * k] = z[:k]                # and triples, scattered over the list
        rng.shuffle(z)
    xyz = np.stack([(u - 32) / 64 * z, (v - 32) / 64 * z, z], 1).astype(np.float32)
    c = dict(xyz=xyz, feat=rng.uniform(-1, 1, (n, 4)).astype(np.float32),
             opacity=rng.uniform(0, 0.05, n).astype(np.float32), cams=[cam], H=H, W=W,
             mode="bilinear")
    run_full(inpc, ctx, c, t_min=0.0)


def test_determinism(inpc, ctx):
    c = synthgen.config1(seed=9)
    _, _, r1 = gpu_forward(inpc, ctx, c)
    _, _, r2 = gpu_forward(inpc, ctx, c)
    for k in ("F", "A", "D", "nfrag", "ncontrib", "sorted_idx", "tile_ranges"):
        np.testing.assert_array_equal(r1[k], r2[k])


def test_invalid_args(inpc, ctx):
    c = synthgen.config1()
    cfg = inpc.make_cfg(64, 64, 4, alpha_max=1.5)
    xyz, feat, op = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"])
    with pytest.raises(inpc.RasterError) as e:
        ctx.forward(cfg, c["cams"], xyz, feat, op)
    assert e.value.status == inpc.INVALID_ARG
    cfg = inpc.make_cfg(64, 64, 4)
    with pytest.raises(inpc.RasterError) as e:   # host tensor (binding check)
        ctx.forward(cfg, c["cams"], torch.from_numpy(c["xyz"]), feat, op)
    assert e.value.status == inpc.INVALID_ARG
    with pytest.raises(inpc.RasterError) as e:   # wrong dtype (binding check)
        ctx.forward(cfg, c["cams"], xyz, feat.double(), op)
    assert e.value.status == inpc.INVALID_ARG
    # the library's own check of a host pointer, through the raw C ABI
    import ctypes as ct
    xh = torch.from_numpy(c["xyz"])
    out = torch.empty((1, 64, 64, 4), device="cuda")
    cams, V = inpc._cams(c["cams"])
    st = inpc.lib.inpc_rasterize_fwd(ctx._h, ct.byref(cfg), cams, V, ct.c_void_p(xh.data_ptr()),
                                     ct.c_void_p(feat.data_ptr()), 0, ct.c_void_p(op.data_ptr()),
                                     xh.shape[0], None, 0, ct.c_void_p(out.data_ptr()), None, None,
                                     None, None, inpc._stream(None))
    assert st == inpc.INVALID_ARG
    fresh = inpc.Context(0)
    with pytest.raises(inpc.RasterError) as e:
        fresh.backward(cfg, c["cams"], xyz, feat, op, torch.zeros((1, 64, 64, 4), device="cuda"))
    assert e.value.status == inpc.NO_STATE


# ------------------------------------------------------------------ Gaussian
@pytest.mark.parametrize("kw", [dict(sigma=0.7, flags=1), dict(sigma=0.01), dict(sigma=0.0),
                                dict(sigma=0.003, dilation=0.3)])
def test_cfg1_gaussian(inpc, ctx, kw):
    c = synthgen.config1(seed=12)
    run_full(inpc, ctx, c, mode="gaussian", exact_ncontrib=False, **kw)


# ------------------------------------------------------------------ full-size configs
def test_cfg2_full_size(inpc, ctx):
    """Config 2 (2^20 points, 1080p) in the launch configuration bench.py
    times: every key, tile list, pixel and gradient against the oracle."""
    run_full(inpc, ctx, synthgen.config2())


def test_cfg3_gaussian_full_size_sampled(inpc, ctx):
    """Config 3 (4 x 2^20 ring-buffer cloud, Gaussian): keys and tile lists
    exact everywhere; image on sampled pixels (5 % + 40 full tiles)."""
    c = synthgen.config3()
    cfg, _, res = gpu_forward(inpc, ctx, c, "gaussian")
    check_lists(c, res, "gaussian")
    H, W = c["H"], c["W"]
    rng = np.random.default_rng(3)
    mask = rng.random((H, W)) < 0.05
    for t in rng.integers(0, 32400, 40):
        ty, tx = divmod(int(t), 240)
        mask[ty * 8:(ty + 1) * 8, tx * 8:(tx + 1) * 8] = True
    check_image(c, res, "gaussian", exact_ncontrib=False, pixel_mask=mask)


def test_cfg4_global_cloud_sampled(inpc, ctx):
    """Config 4 (2^25 points) forward: keys, tiles per point and tile lists
    exact; image on 2 % of pixels + 40 full tiles."""
    c = synthgen.config4()
    cfg, _, res = gpu_forward(inpc, ctx, c, "bilinear")
    check_lists(c, res, "bilinear")
    H, W = c["H"], c["W"]
    rng = np.random.default_rng(4)
    mask = rng.random((H, W)) < 0.02
    for t in rng.integers(0, 32400, 40):
        ty, tx = divmod(int(t), 240)
        mask[ty * 8:(ty + 1) * 8, tx * 8:(tx + 1) * 8] = True
    check_image(c, res, "bilinear", pixel_mask=mask)


# ------------------------------------------------------------------ both binning paths
@pytest.fixture(scope="module")
def ctx_unfused(inpc):
    """A context that bins with the separate project / scan / scatter /
    big-sort kernels instead of the fused cooperative one."""
    import os
    os.environ["INPC_NO_FUSED_BIN"] = "1"
    try:
        return inpc.Context(0)
    finally:
        del os.environ["INPC_NO_FUSED_BIN"]


@pytest.mark.parametrize("seed", [1, 101])
def test_unfused_binning_cfg1(inpc, ctx_unfused, seed):
    run_full(inpc, ctx_unfused, synthgen.config1(seed=seed))


def test_unfused_binning_cfg2(inpc, ctx_unfused):
    run_full(inpc, ctx_unfused, synthgen.config2())


@pytest.mark.parametrize("n,ties", [(5000, "long"), (6000, "short"), (6000, "none"), (3000, "short"),
                                    (20000, "short"), (2100, "none"), (1500, "short"), (1500, "long"),
                                    (300, "none"), (2048, "short"),
                                    # warp merge sort of the mid tiles (257..1024, 1025..2048)
                                    (257, "none"), (513, "short"), (600, "short"), (700, "long"),
                                    (1000, "none"), (1024, "short"), (1025, "long"), (1800, "none"),
                                    # ... 2049..8192 (512 threads per tile), k_sort_big above
                                    (4100, "long"), (8192, "short"), (8193, "none")])
def test_unfused_big_tile(inpc, ctx_unfused, n, ties):
    """k_sort_big: radix chunks (> 2048 entries) with short tie runs fixed up
    in index order, 32-bit-key bitonic chunks (<= 2048) with odd-even
    repair, the 64-bit fallbacks for long runs, multi-chunk merges."""
    test_one_hot_tile_over_smem_cap(inpc, ctx_unfused, n, ties)


# ------------------------------------------------------------------ NEXT f1 / f2
def _sh_case(seed, C=4, N=1000, mode="bilinear"):
    c = synthgen.config1(seed=seed, N=N, C=C)
    cam = synthgen.camera(np.eye(3), [0.1, -0.05, 0.2], 64, 64, 32, 32, 0.1)   # centre off origin
    c["cams"] = [cam]
    sh = np.random.default_rng(seed + 7).normal(0, 0.5, (N, C, 9)).astype(np.float32)
    return c, sh


@pytest.mark.parametrize("C,mode,kw", [(4, "bilinear", {}), (3, "bilinear", {}),
                                       (4, "gaussian", dict(sigma=0.6, flags=1))])
def test_sh_features_fwd_bwd(inpc, ctx, C, mode, kw):
    """f1: SH degree-2 features evaluated in the projection kernel:
    image against the oracle fed with oracle-evaluated features; dL/dcoeff
    against the oracle's dL/df times the oracle's basis."""
    c, sh = _sh_case(40 + C, C)
    cam, H, W = c["cams"][0], c["H"], c["W"]
    f_or, Y = oracle.sh_features(cam, c["xyz"], sh)
    kw2 = dict(kw)
    flags = inpc.FLAG_SH_FEATURES | kw2.pop("flags", 0)
    cfg = inpc.make_cfg(H, W, C, mode, flags=flags | inpc.FLAG_DEBUG, **kw2)
    xyz, op, sht = dev(c["xyz"]), dev(c["opacity"]), dev(sh)
    out = ctx.forward(cfg, c["cams"], xyz, sht, op, debug_counts=True)
    okw = dict(kw2, flags=kw.get("flags", 0))
    r = oracle.render(cam, c["xyz"], f_or, c["opacity"], H, W, mode=mode, **okw)
    ok = out["ncontrib"][0].cpu().numpy() == r["n_contrib"]
    assert (~ok).sum() <= 2
    np.testing.assert_allclose(out["F"][0].cpu().numpy()[ok], r["F"][ok], atol=IMG_TOL)
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(3, 1, H, W, C))
    gsh, go = ctx.backward(cfg, c["cams"], xyz, sht, op, dev(gF), dev(gA), dev(gD))
    torch.cuda.synchronize()
    o = oracle.backward(cam, c["xyz"], f_or, c["opacity"], H, W, gF, gA, gD, mode=mode, **okw)
    g_sh_or = o["g_feat"][:, :, None] * Y[:, None, :]
    check_grads(gsh.cpu().numpy(), g_sh_or)
    check_grads(go.cpu().numpy(), o["g_opacity"])


def test_env_background_fwd_bwd(inpc, ctx):
    """f2: equirectangular environment background composited in the blend
    epilogue against the oracle fed with the oracle's
    per-pixel lookup."""
    c = synthgen.config1(seed=55)
    R = synthgen.random_rotation(np.random.default_rng(5))
    c["cams"] = [synthgen.camera(R, [0, 0, 0], 64, 64, 32, 32, 0.1)]
    xyz_cam = c["xyz"].astype(np.float64)
    c["xyz"] = (xyz_cam @ R).astype(np.float32)   # same camera-space cloud, rotated world
    cam, H, W, C = c["cams"][0], c["H"], c["W"], c["C"]
    env = np.random.default_rng(6).uniform(-1, 1, (32, 64, C)).astype(np.float32)
    bg = oracle.env_background(cam, env, H, W)
    cfg = inpc.make_cfg(H, W, C, env_hw=env.shape[:2], flags=inpc.FLAG_DEBUG)
    xyz, feat, op, envt = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"]), dev(env)
    out = ctx.forward(cfg, c["cams"], xyz, feat, op, bg=envt, debug_counts=True)
    r = oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, bg=bg)
    np.testing.assert_array_equal(out["ncontrib"][0].cpu().numpy(), r["n_contrib"])
    np.testing.assert_allclose(out["F"][0].cpu().numpy(), r["F"], atol=IMG_TOL)
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(4, 1, H, W, C))
    gf, go = ctx.backward(cfg, c["cams"], xyz, feat, op, dev(gF), dev(gA), dev(gD), bg=envt)
    torch.cuda.synchronize()
    o = oracle.backward(cam, c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD, bg=bg)
    check_grads(gf.cpu().numpy(), o["g_feat"])
    check_grads(go.cpu().numpy(), o["g_opacity"])


def test_cudamalloc_and_torch_allocator_agree(inpc):
    """The scratch arena from PyTorch's caching allocator (default) or from
    cudaMalloc gives the same lists and images."""
    c = synthgen.config1(seed=77)
    a = inpc.Context(0, torch_allocator=True)
    b = inpc.Context(0, torch_allocator=False)
    _, _, ra = gpu_forward(inpc, a, c)
    _, _, rb = gpu_forward(inpc, b, c)
    for k in ("F", "A", "D", "sorted_idx", "tile_ranges", "nfrag"):
        np.testing.assert_array_equal(ra[k], rb[k])
    a.close(); b.close()


def test_screen_bands_assemble_bit_exact(inpc, ctx):
    """Sort-first sharding: each band rendered on its own with
    cfg.tile_y_begin/end and assembled equals the unsharded frame bit for bit
    (compositing is per pixel, so screen-space partitions are exact)."""
    from paper_2508_19140_b200 import dist as pdist
    c = synthgen.config2(N=1 << 16, H=200, W=264)
    H, W = c["H"], c["W"]
    xyz, feat, op = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"])
    full = ctx.forward(inpc.make_cfg(H, W, 4), c["cams"], xyz, feat, op)
    rows = (H + 7) // 8
    for world in (2, 3, 5):
        bands = pdist.band_split(np.arange(rows) % 7 + 1.0, world)
        asm = torch.zeros_like(full["F"])
        for b0, b1 in bands:
            if b1 <= b0:
                continue
            o = ctx.forward(inpc.make_cfg(H, W, 4, band=(b0, b1)), c["cams"], xyz, feat, op)
            asm[:, b0 * 8:min(b1 * 8, H)] = o["F"][:, b0 * 8:min(b1 * 8, H)]
        torch.cuda.synchronize()
        assert torch.equal(asm, full["F"])


# ------------------------------------------------------------------ NEXT f4
@pytest.mark.parametrize("which", ["cfg1", "cfg2"])
def test_single64_sort_baseline(inpc, ctx, which):
    """f4: the original single 64-bit sort gives exactly the
    oracle's O7 per-pixel lists (and so the tiled path's per-pixel order)."""
    c = synthgen.config1() if which == "cfg1" else synthgen.config2()
    H, W = c["H"], c["W"]
    cfg = inpc.make_cfg(H, W, 4)
    r, idx = ctx.sort_single64(cfg, c["cams"][0], dev(c["xyz"]), dev(c["opacity"]))
    torch.cuda.synchronize()
    ro, io = oracle.pixel_lists(c["cams"][0], c["xyz"], H, W, method=1)
    np.testing.assert_array_equal(r.cpu().numpy().view(np.uint32), ro)
    np.testing.assert_array_equal(idx.cpu().numpy().view(np.uint32), io)


def test_cfg5_multiview_sampled(inpc, ctx):
    """Config 5 (2^23 points, training-style views): two views in ONE
    multi-view call with shared features.  Per-view keys / tiles / lists
    exact, images on sampled pixels, and the gradients summed over the two
    views against the oracle (upstream gradients nonzero on the sampled
    pixels only, so the oracle backward stays bounded)."""
    c = synthgen.config5()
    views = [0, 21]
    cams = [c["cams"][v] for v in views]
    H, W, C = c["H"], c["W"], c["C"]
    N = c["xyz"].shape[0]
    cfg = inpc.make_cfg(H, W, C, flags=inpc.FLAG_DEBUG)
    xyz, feat, op = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"])
    out = ctx.forward(cfg, cams, xyz, feat, op, debug_counts=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(5)
    masks = []
    for k, cam in enumerate(cams):
        ex = ctx.debug_export(k, N=N, H=H, W=W)
        info = oracle.point_info(cam, c["xyz"], H, W)
        np.testing.assert_array_equal(ex["depth_keys"].cpu().numpy().view(np.uint32), info["depth_key"])
        tr, ti = oracle.tile_lists(cam, c["xyz"], H, W)
        np.testing.assert_array_equal(ex["tile_ranges"].cpu().numpy().view(np.uint32), tr)
        np.testing.assert_array_equal(ex["sorted_idx"].cpu().numpy().view(np.uint32), ti)
        mask = rng.random((H, W)) < 0.01
        masks.append(mask)
        r = oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, pixel_mask=mask,
                          threads=oracle.max_threads())
        np.testing.assert_array_equal(out["nfrag"][k].cpu().numpy()[mask], r["n_frag"][mask])
        np.testing.assert_array_equal(out["ncontrib"][k].cpu().numpy()[mask], r["n_contrib"][mask])
        np.testing.assert_allclose(out["F"][k].cpu().numpy()[mask], r["F"][mask], atol=IMG_TOL)
    gF, gA, gD = synthgen.upstream_grads(9, len(views), H, W, C)
    for k, m in enumerate(masks):
        gF[k] *= m[..., None]; gA[k] *= m; gD[k] *= m
    gf, go = ctx.backward(cfg, cams, xyz, feat, op, dev(gF), dev(gA), dev(gD))
    torch.cuda.synchronize()
    gfo = np.zeros((N, C)); goo = np.zeros(N)
    for k, cam in enumerate(cams):
        o = oracle.backward(cam, c["xyz"], c["feat"], c["opacity"], H, W, gF[k], gA[k], gD[k],
                            pixel_mask=masks[k], threads=oracle.max_threads())
        gfo += o["g_feat"]; goo += o["g_opacity"]
    check_grads(gf.cpu().numpy(), gfo)
    check_grads(go.cpu().numpy(), goo)

@pytest.fixture(scope="module")
def ctx_merge8k(inpc):
    """Unfused binning with the 512-thread merge sort for 2049..8192-entry tiles."""
    import os
    old = {k: os.environ.get(k) for k in ("INPC_NO_FUSED_BIN", "INPC_MERGE8K")}
    os.environ["INPC_NO_FUSED_BIN"] = "1"
    os.environ["INPC_MERGE8K"] = "1"
    c = inpc.Context(0)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    yield c
    c.close()


@pytest.mark.parametrize("n,ties", [(2049, "none"), (4100, "long"), (6000, "short"), (8192, "short"), (8193, "none")])
def test_merge8k_big_tile(inpc, ctx_merge8k, n, ties):
    test_one_hot_tile_over_smem_cap(inpc, ctx_merge8k, n, ties)

"""Multi-process (gloo, world_size 2, CPU) coverage of the N > 1 host logic in
paper_2508_19140_b200/dist.py.  The CPU oracle stands in for the per-rank
CUDA compute (tests may call it); partitions must be exact."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_19140_b200 import dist as pdist


def test_assign_views_partitions_exactly():
    for V in (1, 7, 64):
        for G in (1, 2, 3, 8):
            got = [v for r in range(G) for v in pdist.assign_views(V, G, r)]
            assert got == list(range(V))
            sizes = [len(pdist.assign_views(V, G, r)) for r in range(G)]
            assert max(sizes) - min(sizes) <= 1


def test_band_split_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    for R in (1, 5, 135):
        for G in (1, 2, 4, 8):
            w = rng.uniform(0, 10, R) ** 3
            bands = pdist.band_split(w, G)
            assert bands[0][0] == 0 and bands[-1][1] == R
            assert all(bands[k][1] == bands[k + 1][0] for k in range(G - 1))
            if R >= G:
                assert all(e > b for b, e in bands)
                loads = [w[b:e].sum() for b, e in bands]
                assert max(loads) <= w.sum() / G + w.max() + 1e-6


def test_band_split_weight_in_last_rows_keeps_bands_non_empty():
    """all weight in the last row must not produce empty bands."""
    for w, G in (([1] * 10 + [30], 4), ([0] * 7 + [1], 8), ([5] + [0] * 20 + [100], 3)):
        bands = pdist.band_split(w, G)
        assert bands[0][0] == 0 and bands[-1][1] == len(w)
        assert all(e > b for b, e in bands), bands
        assert all(bands[k][1] == bands[k + 1][0] for k in range(G - 1))


def test_band_assembler_rows_cover_image():
    """Row map of the one-call band assembly: every image row exactly once."""
    import torch
    H = 67
    bands = pdist.band_split(np.ones(pdist.tile_rows(H)), 3)
    asm = pdist.BandAssembler(H, bands, (2,), dtype=torch.float32)
    rows = asm.rows.numpy()
    assert len(rows) == H and len(set(rows.tolist())) == H
    # local emulation of the gather: rank r's slab holds its rows
    img = torch.arange(H * 2, dtype=torch.float32).view(H, 2)
    for r in range(3):
        asm.gathered[r * asm.max_rows:(r + 1) * asm.max_rows] = asm.pack(r, img)
    assert torch.equal(asm.gathered.index_select(0, asm.rows), img)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run2(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fn, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in res.items():
        if isinstance(v, Exception):
            raise v
    return res


def _scene():
    import synthgen
    c = synthgen.config1(seed=42, N=400)
    cams = [synthgen.camera(np.eye(3), [0.02 * k, -0.01 * k, 0.05 * k], 64, 64, 32, 32, 0.1)
            for k in range(5)]
    return c, cams


def _views_grads(rank, world):
    import oracle
    import synthgen
    c, cams = _scene()
    H, W = c["H"], c["W"]
    xyz = torch.from_numpy(c["xyz"]) if rank == 0 else torch.zeros_like(torch.from_numpy(c["xyz"]))
    pdist.broadcast_cloud([xyz])
    assert np.array_equal(xyz.numpy(), c["xyz"])

    N = c["xyz"].shape[0]
    flat, gf, go = pdist.flat_grad_buffers(N, 4, dtype=torch.float64)

    def local(views):
        for v in views:
            gF, gA, gD = (x[0] for x in synthgen.upstream_grads(v, 1, H, W, 4))
            g = oracle.backward(cams[v], xyz.numpy(), c["feat"], c["opacity"], H, W, gF, gA, gD)
            gf.add_(torch.from_numpy(g["g_feat"]))
            go.add_(torch.from_numpy(g["g_opacity"]))
        return flat

    out = pdist.view_sharded_grads(len(cams), local)
    assert out.data_ptr() == flat.data_ptr()       # one all-reduce on the flat buffer, in place
    return gf.numpy().copy(), go.numpy().copy()


def test_view_sharded_gradients_equal_single_process():
    import oracle
    import synthgen
    res = run2(_views_grads)
    c, cams = _scene()
    H, W = c["H"], c["W"]
    gf = np.zeros((c["xyz"].shape[0], 4)); go = np.zeros(c["xyz"].shape[0])
    for v in range(len(cams)):
        gF, gA, gD = (x[0] for x in synthgen.upstream_grads(v, 1, H, W, 4))
        g = oracle.backward(cams[v], c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD)
        gf += g["g_feat"]; go += g["g_opacity"]
    for r in (0, 1):
        np.testing.assert_allclose(res[r][0], gf, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(res[r][1], go, rtol=1e-12, atol=1e-12)


def _banded(rank, world):
    import oracle
    c, _ = _scene()
    H, W = c["H"], c["W"]

    def render_band(band):
        mask = np.zeros((H, W), np.uint8)
        mask[band[0] * 8: band[1] * 8] = 1
        r = oracle.render(c["cams"][0], c["xyz"], c["feat"], c["opacity"], H, W, pixel_mask=mask)
        img = np.concatenate([r["F"], r["A"][..., None], r["D"][..., None]], -1)
        return torch.from_numpy(img)

    weights = np.arange(1, 9, dtype=np.float64)      # uneven bands
    img, bands = pdist.render_frame_banded(H, render_band, row_weights=weights)
    return img.numpy(), bands


def test_screen_band_sharding_is_exact():
    import oracle
    res = run2(_banded)
    c, _ = _scene()
    r = oracle.render(c["cams"][0], c["xyz"], c["feat"], c["opacity"], c["H"], c["W"])
    full = np.concatenate([r["F"], r["A"][..., None], r["D"][..., None]], -1)
    assert res[0][1] == res[1][1] and res[0][1][0][1] != 4     # weighted, not equal rows
    for k in (0, 1):
        np.testing.assert_array_equal(res[k][0], full)

"""Multi-GPU partitioning of the rasterizer.

One process per GPU, ``torch.distributed`` (NCCL over NVLink/NVSwitch on the
B200 box; gloo in the CPU tests).  Two partitions, both exact:

* view batches (config 5, training): rank r renders views
  [r V/G, (r+1) V/G) of one cloud that was broadcast once; the per-rank
  gradient sums are all-reduced (SUM) — the path's only real exchange step
  (shared features, R20).
* screen bands (config 4, one huge frame): sort-first partition of 8-pixel
  tile rows into contiguous bands (alpha compositing is order dependent, so
  only screen-space partitions are exact); each rank rasterizes its band
  (``cfg.tile_y_begin/end``) and the bands are all-gathered.

The compute of each rank is passed in as a callable so the same host logic
runs with the CUDA Context on GPUs and with the CPU oracle in the gloo tests.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

TILE = 8


def assign_views(V: int, world: int, rank: int) -> range:
    """Contiguous, balanced view range of `rank` (sizes differ by at most 1)."""
    base, extra = divmod(V, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def band_split(row_weights: Sequence[float], world: int) -> list[tuple[int, int]]:
    """Split tile rows [0, R) into `world` contiguous bands [b, e) with about
    equal total weight (e.g. tile entries per row from the projection
    histogram).  Deterministic: every rank computes the same bands.  Bands may
    be empty (b == e) only when R < world."""
    w = np.asarray(row_weights, np.float64)
    R = len(w)
    if R == 0:
        return [(0, 0)] * world
    w = np.maximum(w, 0) + 1e-9 * max(1.0, w.sum())      # every row has a little weight
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for k in range(1, world):
        target = cum[-1] * k / world
        c = int(np.searchsorted(cum, target, side="left"))
        c = min(max(c, cuts[-1] + (1 if R - cuts[-1] > world - k else 0)), R)
        cuts.append(c)
    cuts.append(R)
    return [(cuts[k], cuts[k + 1]) for k in range(world)]


def tile_rows(H: int) -> int:
    return (H + TILE - 1) // TILE


def broadcast_cloud(tensors, group=None, src=0):
    """One-time broadcast of the point cloud (xyz, features, opacity) from
    `src` to every rank (NCCL over NVLink on the B200 box)."""
    import torch.distributed as dist
    for t in tensors:
        dist.broadcast(t, src=src, group=group)
    return tensors


def view_sharded_grads(V: int, local_views_fn: Callable[[range], tuple], group=None):
    """Data-parallel view batch: this rank computes the summed gradients of its
    views with `local_views_fn(views) -> (g_feat, g_opacity)` (tensors), then
    one SUM all-reduce gives every rank the gradient of the whole batch."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    views = assign_views(V, world, rank)
    g_feat, g_op = local_views_fn(views)
    dist.all_reduce(g_feat, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(g_op, op=dist.ReduceOp.SUM, group=group)
    return g_feat, g_op


def render_frame_banded(H: int, render_band_fn: Callable[[tuple[int, int]], object],
                        row_weights=None, group=None):
    """Sort-first sharded frame: rank r renders tile rows bands[r] with
    `render_band_fn(band) -> image` (a full-size [H, W, K] tensor whose band
    rows are valid) and the bands are all-gathered into the full image on
    every rank.  Returns (image, bands)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    R = tile_rows(H)
    bands = band_split(np.ones(R) if row_weights is None else row_weights, world)
    img = render_band_fn(bands[rank])
    # equal-size padded slabs for all_gather
    max_rows = max((e - b) * TILE for b, e in bands)
    tail = tuple(img.shape[1:])
    slab = torch.zeros((max_rows,) + tail, dtype=img.dtype, device=img.device)
    b, e = bands[rank]
    rows = slice(b * TILE, min(e * TILE, H))
    n = rows.stop - rows.start if e > b else 0
    if n > 0:
        slab[:n] = img[rows]
    gathered = [torch.empty_like(slab) for _ in range(world)]
    dist.all_gather(gathered, slab, group=group)
    out = torch.empty_like(img)
    for r, (b, e) in enumerate(bands):
        if e > b:
            r0, r1 = b * TILE, min(e * TILE, H)
            out[r0:r1] = gathered[r][: r1 - r0]
    return out, bands

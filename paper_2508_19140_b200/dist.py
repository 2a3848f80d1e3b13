"""Multi-GPU partitioning of the rasterizer.

One process per GPU, ``torch.distributed`` (NCCL over NVLink/NVSwitch on the
B200 box; gloo in the CPU tests).  Two partitions, both exact:

* view batches (config 5, training): rank r renders views
  [r V/G, (r+1) V/G) of one cloud that was broadcast once; the per-rank
  gradient sums live in ONE flat [N*C + N] buffer (feature gradients, then
  opacity gradients) that is all-reduced (SUM) in one call -- the path's
  only real exchange step (shared features, R20).
* screen bands (config 4, one huge frame): sort-first partition of 8-pixel
  tile rows into contiguous bands (alpha compositing is order dependent, so
  only screen-space partitions are exact); each rank rasterizes its band
  (``cfg.tile_y_begin/end``), packs it into one padded slab, and one
  all-gather into a single tensor plus one row gather assemble the frame.

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
    histogram).  Deterministic: every rank computes the same bands.  When
    R >= world every band holds at least one row (cut k lies in
    [cut_{k-1} + 1, R - (world - k)]); bands are empty only when R < world."""
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
        if R >= world:
            c = min(max(c, cuts[-1] + 1), R - (world - k))
        else:
            c = min(max(c, cuts[-1]), R)
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


def flat_grad_buffers(N: int, C: int, device=None, dtype=None):
    """One flat gradient buffer [N*C + N] and its two views: g_feat [N, C]
    (offset 0, so 16-byte aligned as the C ABI wants for C == 4) and
    g_opacity [N].  A view batch all-reduces the flat buffer once."""
    import torch
    flat = torch.zeros(N * C + N, device=device, dtype=dtype or torch.float32)
    return flat, flat[: N * C].view(N, C), flat[N * C:]


def view_sharded_grads(V: int, local_views_fn: Callable[[range], object], group=None):
    """Data-parallel view batch: this rank accumulates the gradients of its
    views into one flat buffer with `local_views_fn(views) -> flat` (see
    flat_grad_buffers), then ONE SUM all-reduce gives every rank the
    gradient of the whole batch."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    flat = local_views_fn(assign_views(V, world, rank))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class BandAssembler:
    """Sort-first frame assembly: rank r owns pixel rows of tile rows
    bands[r].  pack() copies the rank's rows into a padded slab [max_rows,
    W, K]; gather() runs one all-gather into a single [world * max_rows, W,
    K] tensor and one index_select of the valid rows (row order = image
    order) gives the full frame on every rank."""

    def __init__(self, H: int, bands, tail, device=None, dtype=None):
        import torch
        self.H, self.bands = H, list(bands)
        self.world = len(self.bands)
        self.max_rows = max(max((e - b) * TILE for b, e in self.bands), 1)
        self.slab = torch.zeros((self.max_rows,) + tuple(tail), device=device, dtype=dtype)
        self.gathered = torch.empty((self.world * self.max_rows,) + tuple(tail), device=device, dtype=dtype)
        rows = []
        for r, (b, e) in enumerate(self.bands):
            r0, r1 = b * TILE, min(e * TILE, H)
            rows.extend(r * self.max_rows + q for q in range(max(r1 - r0, 0)))
        assert len(rows) == H, "bands must cover every pixel row"
        self.rows = torch.tensor(rows, device=device, dtype=torch.long)

    def band_rows(self, rank: int) -> slice:
        b, e = self.bands[rank]
        return slice(b * TILE, min(e * TILE, self.H))

    def pack(self, rank: int, img):
        """img: full-size [H, W, K] (only the band rows are read)."""
        rs = self.band_rows(rank)
        n = max(rs.stop - rs.start, 0)
        if n:
            self.slab[:n] = img[rs]
        return self.slab

    def gather(self, group=None):
        import torch.distributed as dist
        dist.all_gather_into_tensor(self.gathered, self.slab, group=group)
        return self.gathered.index_select(0, self.rows)


def render_frame_banded(H: int, render_band_fn: Callable[[tuple[int, int]], object],
                        row_weights=None, group=None):
    """Sort-first sharded frame: rank r renders tile rows bands[r] with
    `render_band_fn(band) -> image` (a full-size [H, W, K] tensor whose band
    rows are valid) and the bands are assembled on every rank (one
    all-gather, one row gather).  Returns (image, bands)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    R = tile_rows(H)
    bands = band_split(np.ones(R) if row_weights is None else row_weights, world)
    img = render_band_fn(bands[rank])
    asm = BandAssembler(H, bands, tuple(img.shape[1:]), device=img.device, dtype=img.dtype)
    asm.pack(rank, img)
    return asm.gather(group), bands

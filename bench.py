#!/usr/bin/env python
"""Benchmark of the INPC neural point rasterizer (BASELINE.json metric:
frames/s and Mpoints/s at 1080p fwd+bwd, % of B200 HBM roofline, 1/2/4/8 GPUs).

One step = one pass of the whole hot path (H1-H8) over one
batch of synthetic input, with the point cloud and upstream gradients
resident in HBM.  Default workload = the north-star configuration
(BASELINE.json configs[4], SURVEY §8(d) cfg 5): a training-style batch of 64
1080p camera views of one static 2^23-point cloud with shared features,
forward + backward, the 64 views split over the ranks, the per-rank gradient
sums all-reduced in one NCCL call inside the timed step (strong scaling).
The static cloud is put in spatial (Morton) order once, untimed, by the
library's inpc_spatial_order; its cost is reported.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|3|4|5] [--variant base|sh|env|sh+env]

`--gpus N` without torchrun's WORLD_SIZE re-launches itself under
`torch.distributed.run` with N ranks (127.0.0.1).  `--impl reference` times
the CPU oracle (oracle/, the only reference this paper-only build has) on
whole views of the same workload and prints the same JSON line with
"impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

METRIC = "frames/s and Mpoints/s at 1080p fwd+bwd, % of B200 HBM roofline, 1/2/4/8 GPUs"
WORKLOADS = {
    2: "cfg2: 2^20-point view-specific cloud, 1920x1080, C=4, bilinear 2x2 splats, fwd+bwd",
    3: "cfg3: 4x2^20 ring-buffer cloud, 1920x1080, C=4, Gaussian splats (auto sigma, dilation 0.16), forward only",
    4: "cfg4: 2^25-point global extracted cloud, 1920x1080, C=4, bilinear, forward only",
    5: "cfg5: 64 orbit views of a 2^23-point static cloud, 1920x1080, C=4, bilinear, fwd+bwd, shared features",
}
NOMINAL_HBM_GBS = 8000.0
DEFAULT_CONFIG = 5


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ------------------------------------------------------------------ byte models
def step_bytes_survey(N, Nv, Ft, P, C, fwd_only, sh=False, env=False):
    """Compulsory bytes of one step, SURVEY.md §8(d) exactly (sums over the
    views: N, Nv, Ft, P are totals):
      B_fwd = 16 N + 4C Nv + 16 Ft + 4P(C+2) + 8P  [+ 4PC with a background]
      B_bwd = 4P(C+2) + 8P + 4 Ft + (16+4C) Nv + 4(C+1) Nv
    Variants (NEXT rows): SH features read 36C bytes per visible point and
    write 36C bytes of coefficient gradients (f1); the env-map background
    adds 4PC to both passes (f2)."""
    fb = (36 if sh else 4) * C
    b_fwd = 16 * N + fb * Nv + 16 * Ft + 4 * P * (C + 2) + 8 * P + (4 * P * C if env else 0)
    b_bwd = 4 * P * (C + 2) + 8 * P + 4 * Ft + (16 + fb) * Nv + (fb + 4) * Nv + (4 * P * C if env else 0)
    return b_fwd + (0 if fwd_only else b_bwd)


def kernel_bytes(N, Nv, Ft, P, C, sh=False, env=False, F_mid=0, F_huge=0):
    """Compulsory bytes per kernel, for the roofline of the
    dominant kernel only -- NOT summed into the step (bin_fused is the sum of
    project_count and scatter; the step model is step_bytes_survey).
    F_mid / F_huge: entries of tiles of 257..mid_max / over mid_max entries (mid_max
    = 2048, or 8192 where the 8192 merge class runs), which
    the mid / big-tile sorts read once (8-byte key) and write once (4-byte
    index)."""
    fbytes = (36 if sh else 4) * C
    m = {
        "project_count": 12 * N + (fbytes * Nv if sh else 0),
        "scan_tiles": 0,
        "scatter": 8 * Ft,
        "sort_mid": 12 * F_mid,
        "sort_big": 12 * F_huge,
        "blend_fwd": 8 * Ft + (4 + (0 if sh else 4 * C)) * Nv + 4 * P * (C + 2) + 8 * P,
        "blend_bwd": 4 * P * (C + 2) + 8 * P + 4 * Ft + (16 + 4 * C) * Nv + 4 * (C + 1) * Nv,
    }
    if sh:
        m["sh_grad"] = 12 * Nv + fbytes * Nv
    if env:
        m["blend_fwd"] += 4 * C * P
        m["blend_bwd"] += 4 * C * P
    m["bin_fused"] = m["project_count"] + m["scatter"]
    return m


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ workloads
def load_workload(config, rank, world):
    """Synthetic inputs of one config as seen by `rank`."""
    from paper_2508_19140_b200.dist import assign_views
    if config == 5:
        c = synthgen.config5()
        views = list(assign_views(64, world, rank))
        return dict(c=c, cams=[c["cams"][v] for v in views], views=views, fwd_only=False,
                    frames_per_step=64, scaling="strong", static=True, seed_g=5 + rank,
                    parallelism=f"64 views split over {world} rank(s), one flat gradient all-reduce per step")
    if config == 4:
        c = synthgen.config4()
        return dict(c=c, cams=c["cams"], views=[0], fwd_only=True, frames_per_step=1,
                    scaling="strong" if world > 1 else "weak", static=True, seed_g=4,
                    parallelism=(f"one frame in {world} screen bands + one all-gather" if world > 1 else "one frame"))
    if config == 3:
        c = synthgen.config3()
        return dict(c=c, cams=c["cams"], views=[0], fwd_only=True, frames_per_step=world, scaling="weak",
                    static=False, seed_g=3 + rank, parallelism=f"independent frames x{world}")
    c = synthgen.config2(seed=2 + rank)
    return dict(c=c, cams=c["cams"], views=[0], fwd_only=False, frames_per_step=world, scaling="weak",
                static=False, seed_g=2 + rank, parallelism=f"independent frames x{world} (weak)")


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_view(c, v, gF, gA, gD, threads, fwd_only, pixel_mask=None):
    """The CPU oracle on one whole view (fwd, + bwd unless fwd_only); seconds."""
    import oracle
    H, W = c["H"], c["W"]
    cam = c["cams"][v]
    kw = {} if c["mode"] == "bilinear" else dict(mode="gaussian", sigma=0.0, dilation=0.16)
    t0 = time.perf_counter()
    oracle.render(cam, c["xyz"], c["feat"], c["opacity"], H, W, pixel_mask=pixel_mask, threads=threads, **kw)
    if not fwd_only:
        oracle.backward(cam, c["xyz"], c["feat"], c["opacity"], H, W, gF, gA, gD, pixel_mask=pixel_mask,
                        threads=threads, **kw)
    return time.perf_counter() - t0


def cpu_baseline(config, budget_s=12.0):
    """Oracle throughput on whole views of the workload (frames/s)."""
    w = load_workload(config, 0, 1)
    c = w["c"]
    H, W, C = c["H"], c["W"], c["C"]
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(w["seed_g"], 1, H, W, C))
    th = cpu_threads()
    tt, nv, v = 0.0, 0, 0
    while tt < budget_s or nv == 0:
        tt += oracle_view(c, v % len(c["cams"]), gF, gA, gD, th, w["fwd_only"])
        nv += 1
        v += 21
    return {"value": nv / tt, "unit": "frames/s", "cores": th, "kind": "oracle",
            "sample": f"{nv} whole view(s) of {c['name']} ({'fwd' if w['fwd_only'] else 'fwd+bwd'}), "
                      f"{tt:.1f} s on {th} threads"}


def run_reference(args, rank, world):
    """Reference arm: the CPU oracle as it stands, whole views per step (a
    band of one view's rows only when (K + W) whole views would not fit the
    few-minute budget)."""
    if rank != 0:
        return
    w = load_workload(args.config, 0, 1)
    c = w["c"]
    H, W, C = c["H"], c["W"], c["C"]
    N = c["xyz"].shape[0]
    gF, gA, gD = (x[0] for x in synthgen.upstream_grads(w["seed_g"], 1, H, W, C))
    th = cpu_threads()
    t_view = oracle_view(c, 0, gF, gA, gD, th, w["fwd_only"])
    budget = 180.0 / max(1, args.steps + args.warmup)
    frac = 1.0 if t_view <= budget else max(0.02, budget / t_view)
    mask = None
    if frac < 1.0:
        mask = np.zeros((H, W), np.uint8)
        mask[: max(1, int(round(frac * H)))] = 1
        frac = float(mask[:, 0].mean())
    tt = 0.0
    for k in range(args.warmup + args.steps):
        t = oracle_view(c, (21 * k) % len(c["cams"]), gF, gA, gD, th, w["fwd_only"], mask)
        if k >= args.warmup:
            tt += t
    fps = args.steps * frac / tt
    sample = (f"{args.steps} step(s) x " + ("one whole view" if frac == 1.0 else f"{frac:.3f} of a view's rows")
              + f" of {c['name']} ({'fwd' if w['fwd_only'] else 'fwd+bwd'})")
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tt / args.steps, "higher_is_better": True, "scaling": w["scaling"],
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "N": N, "H": H, "W": W, "C": C},
        "mpoints_per_s": fps * N / 1e6,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": th, "kind": "oracle", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def run_sort_ab(args):
    """NEXT f4: the paper's own sort comparison on B200, cfg 2:
    the original single 64-bit sort of 4 copies per point vs this build's
    tiled ordering (bucket scatter + per-tile register sorts)."""
    import math

    import torch

    import paper_2508_19140_b200 as inpc
    torch.cuda.set_device(0)
    c = synthgen.config2()
    H, W, C = c["H"], c["W"], c["C"]
    N = c["xyz"].shape[0]
    xyz, feat, op = (torch.from_numpy(c[k]).cuda() for k in ("xyz", "feat", "opacity"))
    ctx = inpc.Context(0)
    cfg = inpc.make_cfg(H, W, C)
    for _ in range(3):
        ctx.sort_single64(cfg, c["cams"][0], xyz, op)
        ctx.forward(cfg, c["cams"], xyz, feat, op)
    torch.cuda.synchronize()
    ctx.stage_times(reset=True)
    ctx.set_profiling(True)
    reps = max(5, args.steps // 10)
    F = 0
    for _ in range(reps):
        _, idx = ctx.sort_single64(cfg, c["cams"][0], xyz, op)
        F = idx.numel()
        ctx.forward(cfg, c["cams"], xyz, feat, op)
    st = ctx.stage_times(reset=True)
    ctx.set_profiling(False)
    dbg = inpc.make_cfg(H, W, C, flags=inpc.FLAG_DEBUG)
    ctx.forward(dbg, c["cams"], xyz, feat, op)
    Ft = ctx.debug_export(0, H=H, W=W)["F_t"]
    single_us = st["single_sort"][0] / reps * 1e3
    bin_us = st["bin_fused"][0] / reps * 1e3
    fwd_us = st["blend_fwd"][0] / reps * 1e3
    pbits = (H * W - 1).bit_length()
    line = {
        "mode": "sort A/B (NEXT f4)", "workload": WORKLOADS[2],
        "original_single_sort": {"us": single_us, "keys": 4 * N, "real_fragments": F,
                                 "key_bits": 32 + pbits, "passes": math.ceil((32 + pbits) / 8),
                                 "keys_per_s": 4 * N / (single_us * 1e-6),
                                 "paper_model": "4 ceil((32+21)/8) n = 28n (P:162)"},
        "tiled": {"bin_us": bin_us, "tile_entries": Ft, "entries_per_s": Ft / (bin_us * 1e-6),
                  "blend_fwd_us_incl_tile_sorts": fwd_us,
                  "paper_model": "4n depth + 2.54n tile = 6.54n (P:171-172); here 1 atomic bucket "
                                 "scatter of 1.27n + per-tile sorts in registers inside blend_fwd"},
        "speedup_bin_vs_single_sort": single_us / bin_us,
    }
    print(json.dumps(line), flush=True)
    ctx.close()


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2508_19140_b200 as inpc
    from paper_2508_19140_b200 import dist as pdist

    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    wl = load_workload(args.config, rank, world)
    c, cams = wl["c"], wl["cams"]
    mode = c["mode"]
    fwd_only = wl["fwd_only"]
    V = len(cams)
    H, W, C = c["H"], c["W"], c["C"]
    N = c["xyz"].shape[0]
    P = H * W
    flags = 0
    feat_np = c["feat"]
    if args.variant in ("sh", "sh+env"):
        flags |= inpc.FLAG_SH_FEATURES
        feat_np = np.random.default_rng(wl["seed_g"] + 11).normal(0, 0.5, (N, C, 9)).astype(np.float32)
    env_hw = env_t = None
    if args.variant in ("env", "sh+env"):
        env_hw = (1024, 2048)   # the paper's distilled map size
        env_t = torch.from_numpy(np.random.default_rng(wl["seed_g"] + 12).uniform(
            -1, 1, (1024, 2048, C)).astype(np.float32)).to(dev)
    ctx = inpc.Context(dev_index)
    xyz = torch.from_numpy(c["xyz"]).to(dev)
    feat = torch.from_numpy(feat_np).to(dev)
    op = torch.from_numpy(c["opacity"]).to(dev)
    order = args.order if args.order != "auto" else ("spatial" if wl["static"] else "given")
    prepare_ms = None
    if order == "spatial":
        # one-time spatial order of the static cloud (untimed, reported)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.spatial_order(xyz)          # warm (buffer allocation)
        e0.record()
        perm = ctx.spatial_order(xyz)
        xyz, feat, op = xyz[perm].contiguous(), feat[perm].contiguous(), op[perm].contiguous()
        e1.record()
        torch.cuda.synchronize()
        prepare_ms = e0.elapsed_time(e1)
        del perm
    if world > 1 and wl["static"]:
        pdist.broadcast_cloud([xyz, feat, op])    # one cloud for all ranks, once (NCCL over NVLink)
    if order == "spatial":
        # chunk bounds of the static cloud (once): binning skips chunks that
        # cannot reach the view's frame / the rank's screen band
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.set_chunks(xyz)
        e1.record()
        torch.cuda.synchronize()
        prepare_ms = (prepare_ms or 0.0) + e0.elapsed_time(e1)
    # host copies (pinned) in the order the device uses, for the end-to-end leg
    xyz_h, feat_h, op_h = (t.cpu().pin_memory() for t in (xyz, feat, op))
    bands = asm = None
    if args.config == 4 and world > 1:
        # sort-first screen bands of 8-pixel tile rows, balanced by the per-row
        # tile-entry counts of the (static) cloud, measured once untimed
        ctx.forward(inpc.make_cfg(H, W, C, mode), cams, xyz, feat, op)
        rng = ctx.debug_export(0, H=H, W=W)["tile_ranges"].cpu().numpy().astype(np.int64)
        tx = (W + 7) // 8
        row_w = np.diff(rng).reshape(-1, tx).sum(1) + 64 * tx   # + per-pixel output cost
        bands = pdist.band_split(row_w, world)
        asm = pdist.BandAssembler(H, bands, (W, C + 2), device=dev)
    g1 = [torch.from_numpy(x) for x in synthgen.upstream_grads(wl["seed_g"], 1, H, W, C)]
    gF_h, gA_h, gD_h = (x.expand((V,) + tuple(x.shape[1:])).contiguous().pin_memory() for x in g1)
    gF, gA, gD = gF_h.to(dev), gA_h.to(dev), gD_h.to(dev)
    cfg = inpc.make_cfg(H, W, C, mode, flags=flags, env_hw=env_hw,
                        band=None if bands is None else bands[rank])
    out = dict(F=torch.empty((V, H, W, C), device=dev), A=torch.empty((V, H, W), device=dev),
               D=torch.empty((V, H, W), device=dev))
    if args.variant in ("sh", "sh+env"):
        g_flat = None
        g_feat = torch.zeros_like(feat)
        g_op = torch.zeros_like(op)
    else:
        g_flat, g_feat, g_op = pdist.flat_grad_buffers(N, C, device=dev)
    reduce_grads = args.config == 5 and world > 1
    img_cat = torch.empty((H, W, C + 2), device=dev) if asm is not None else None

    def step(S=None):
        S = S or dict(xyz=xyz, feat=feat, op=op, gF=gF, gA=gA, gD=gD, out=out, g_flat=g_flat,
                      g_feat=g_feat, g_op=g_op)
        if fwd_only:
            ctx.forward(cfg, cams, S["xyz"], S["feat"], S["op"], bg=env_t, out=S["out"])
            if asm is not None:   # assemble the frame: one all-gather of the padded bands
                rs = asm.band_rows(rank)
                img_cat[rs, :, :C] = S["out"]["F"][0, rs]
                img_cat[rs, :, C] = S["out"]["A"][0, rs]
                img_cat[rs, :, C + 1] = S["out"]["D"][0, rs]
                asm.pack(rank, img_cat)
                asm.gather()
            return
        if S["g_flat"] is not None:
            S["g_flat"].zero_()
        else:
            S["g_feat"].zero_()
            S["g_op"].zero_()
        ctx.forward(cfg, cams, S["xyz"], S["feat"], S["op"], bg=env_t, out=S["out"])
        ctx.backward(cfg, cams, S["xyz"], S["feat"], S["op"], S["gF"], S["gA"], S["gD"], bg=env_t,
                     g_feat=S["g_feat"], g_opacity=S["g_op"])
        if reduce_grads:   # the view batch's one exchange step (shared features, R20)
            dist.all_reduce(S["g_flat"])

    # workload statistics (untimed): visible points, tile entries, per view
    dbg = inpc.make_cfg(H, W, C, mode, flags=flags | inpc.FLAG_DEBUG, env_hw=env_hw)
    ctx.forward(dbg, cams, xyz, feat, op, bg=env_t)
    Nv = Ft = F_mid = F_huge = 0
    # the merge sort's largest class: 8192 entries on dense clouds (the
    # library's rule, N >= 512 tiles; INPC_MERGE8K forces it), else 2048
    n_tiles = ((W + 7) // 8) * ((H + 7) // 8)
    m8 = os.environ.get("INPC_MERGE8K")
    mid_max = 8192 if (m8 == "1" or (m8 != "0" and N >= 512 * n_tiles)) else 2048
    for v in range(V):
        ex = ctx.debug_export(v, N=N, H=H, W=W)
        Nv += int((ex["tiles_touched"] > 0).sum().item())
        Ft += int(ex["F_t"])
        cnt = ex["tile_ranges"][1:].long() - ex["tile_ranges"][:-1].long()
        F_mid += int(cnt[(cnt > 256) & (cnt <= mid_max)].sum().item())
        F_huge += int(cnt[cnt > mid_max].sum().item())
    sh, env = "sh" in args.variant, "env" in args.variant
    kmodel = kernel_bytes(N * V, Nv, Ft, P * V, C, sh=sh, env=env, F_mid=F_mid, F_huge=F_huge)
    step_bytes = step_bytes_survey(N * V, Nv, Ft, P * V, C, fwd_only, sh=sh, env=env)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    for _ in range(args.warmup):
        step()
    # clock ramp: keep the GPU busy ~0.3 s before the timed region (untimed)
    t_end = time.perf_counter() + (0.0 if args.profile_run else 0.3)
    while time.perf_counter() < t_end:
        step()
        torch.cuda.synchronize()
    graph = None
    graph_launches = 0
    if not args.no_graph and world == 1:
        # one step captured as a CUDA graph (our kernels + the gradient memset);
        # at N > 1 the step keeps its NCCL collective and runs eagerly
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            ctx.stage_times(reset=True)
            with torch.cuda.graph(graph):
                step()
            graph_launches = int(sum(v[1] for v in ctx.stage_times(reset=True).values()))
            graph.replay()
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover - reported in the JSON line
            print(f"graph capture failed, eager timing: {e}", file=sys.stderr)
            graph = None
    # per-stage device time: CUDA events around each stage on the launching
    # stream; with a graph (events inside a graph cannot be timed) each timed
    # replay is followed by one eager profiled step outside the step events
    ctx.stage_times(reset=True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.set_profiling(graph is None)
    with ClockSampler(dev_index) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))          # evict L2 between steps (outside the step events)
            ev[k][0].record()
            if graph is not None:
                graph.replay()
            else:
                step()
            ev[k][1].record()
            if graph is not None:
                flush.fill_(float(k) + 0.5)
                ctx.set_profiling(True)
                step()
                ctx.set_profiling(False)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stages = ctx.stage_times(reset=True)
    ctx.set_profiling(False)
    graph_used = graph is not None
    graph = None
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    fps = wl["frames_per_step"] * args.steps / (tot_ms / 1e3)
    # our kernels launched inside the timed region: the profiled eager steps
    # (counted by the library) plus, with a graph, the kernels of each replay
    launches = int(sum(v[1] for v in stages.values())) + (graph_launches * args.steps if graph_used else 0)

    # roofline of the dominant kernel (largest share of device time)
    hbm, peak_src = peaks()
    kern = {k: v for k, v in stages.items() if v[1] > 0}
    dom = max(kern, key=lambda k: kern[k][0])
    launches_per_step = max(1, round(kern[dom][1] / args.steps))
    dom_ms = kern[dom][0] / kern[dom][1]
    dom_bytes = kmodel.get(dom, 0) / launches_per_step                # per launch (per view)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "peak_source": peak_src,
            "bytes_per_launch": dom_bytes, "us_per_launch": dom_ms * 1e3,
            "share_of_step": kern[dom][0] / args.steps / ms_per_step}
    prof_traffic = os.path.join(ROOT, "profiles", "traffic_r02.json")
    if os.path.exists(prof_traffic):
        trj = json.load(open(prof_traffic))
        key = f"cfg{args.config}" + ("" if args.variant == "base" else "-" + args.variant)
        tr = trj.get(key, {}).get(dom)
        if tr:
            roof["traffic"] = tr
    step_gbs = step_bytes / (ms_per_step * 1e-3) / 1e9

    # end to end through the public API with host (pinned) buffers: every step
    # copies its inputs in (cloud + upstream gradients) and its results out
    # (image + gradients); two device buffer sets so that step k+1's H2D and
    # step k-1's D2H overlap step k
    F_h = torch.empty((V, H, W, C), pin_memory=True)
    A_h = torch.empty((V, H, W), pin_memory=True)
    D_h = torch.empty((V, H, W), pin_memory=True)
    gf_h = torch.empty(tuple(feat.shape), pin_memory=True)
    go_h = torch.empty(tuple(op.shape), pin_memory=True)
    ins = (xyz_h, feat_h, op_h) + (() if fwd_only else (gF_h, gA_h, gD_h))
    outs = (F_h, A_h, D_h) + (() if fwd_only else (gf_h, go_h))
    h2d = sum(t.numel() * 4 for t in ins)
    d2h = sum(t.numel() * 4 for t in outs)
    sets = [dict(xyz=xyz, feat=feat, op=op, gF=gF, gA=gA, gD=gD, out=out, g_flat=g_flat, g_feat=g_feat,
                 g_op=g_op)]
    if not args.profile_run:
        S2 = {k: (v.clone() if torch.is_tensor(v) else ({kk: vv.clone() for kk, vv in v.items()}
                                                        if isinstance(v, dict) else v))
              for k, v in sets[0].items() if k not in ("g_flat", "g_feat", "g_op")}
        if g_flat is not None:
            S2["g_flat"], S2["g_feat"], S2["g_op"] = pdist.flat_grad_buffers(N, C, device=dev)
        else:
            S2["g_flat"], S2["g_feat"], S2["g_op"] = None, torch.zeros_like(feat), torch.zeros_like(op)
        sets.append(S2)
    s_comp = torch.cuda.current_stream()
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in sets]
    ev_done = [torch.cuda.Event() for _ in sets]
    ev_read = [torch.cuda.Event() for _ in sets]
    for e in ev_done + ev_read:
        e.record(s_comp)

    def e2e_step(k):
        b = k % len(sets)
        S = sets[b]
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(ev_done[b])          # set b's previous compute has read its inputs
            S["xyz"].copy_(xyz_h, non_blocking=True)
            S["feat"].copy_(feat_h, non_blocking=True)
            S["op"].copy_(op_h, non_blocking=True)
            if not fwd_only:
                S["gF"].copy_(gF_h, non_blocking=True)
                S["gA"].copy_(gA_h, non_blocking=True)
                S["gD"].copy_(gD_h, non_blocking=True)
            ev_in[b].record(s_h2d)
        s_comp.wait_event(ev_in[b])
        s_comp.wait_event(ev_read[b])             # set b's previous outputs were copied out
        if order == "spatial":
            ctx.set_chunks(S["xyz"])              # the copied-in cloud's chunk bounds (one kernel)
        step(S)
        ev_done[b].record(s_comp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_done[b])
            F_h.copy_(S["out"]["F"], non_blocking=True)
            A_h.copy_(S["out"]["A"], non_blocking=True)
            D_h.copy_(S["out"]["D"], non_blocking=True)
            if not fwd_only:
                gf_h.copy_(S["g_feat"], non_blocking=True)
                go_h.copy_(S["g_op"], non_blocking=True)
            ev_read[b].record(s_d2h)

    for k in range(0 if args.profile_run else 2):
        e2e_step(k)
    n_e2e = 1 if args.profile_run else max(4, min(args.steps, 10))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for k in range(n_e2e):
        e2e_step(k)
    s_d2h.wait_stream(s_comp)
    e1.record(s_d2h)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / n_e2e
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_fps = wl["frames_per_step"] / (e2e_ms / 1e3)

    # CPU oracle baseline (rank 0, N = 1 only): whole views of the same workload
    cpu = None
    if rank == 0 and world == 1 and args.variant == "base" and not (args.no_cpu_baseline or args.profile_run):
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "passes": "fwd" if fwd_only else "fwd+bwd",
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": wl["scaling"],
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config], "variant": args.variant, "N": N,
                       "views_per_step": wl["frames_per_step"], "views_per_rank": V,
                       "N_visible": Nv, "F_t": Ft, "F_mid": F_mid, "F_huge": F_huge, "F_mid_max": mid_max, "H": H, "W": W,
                       "C": C, "mode": mode, "alpha_max": 0.99, "t_min": 1e-4,
                       "point_order": order, "parallelism": wl["parallelism"],
                       "l2": "flushed: 256 MiB write between steps, outside the per-step events"},
            "mpoints_per_s": fps * N / 1e6,
            "prepare_ms": prepare_ms,
            "prepare_note": ("one-time, untimed: spatial (Morton) order of the static cloud "
                             "(inpc_spatial_order) + its 1024-point chunk bounds (inpc_chunk_bounds); "
                             "the e2e leg recomputes the chunk bounds of every copied-in cloud"),
            "step_algorithmic_bytes": step_bytes,
            "step_bytes_model": "SURVEY.md §8(d) B_fwd" + ("" if fwd_only else " + B_bwd"),
            "step_roofline": {"achieved": step_gbs, "peak": hbm, "unit": "GB/s", "frac": step_gbs / hbm,
                              "frac_of_nominal_8TBs": step_gbs / NOMINAL_HBM_GBS},
            "roofline": roof,
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items() if v[1]},
            "stages_note": ("device time per stage from CUDA events around each stage of an eager "
                            "profiled step after every timed replay (same kernels as the graph)"),
            "gpu_launches": launches,
            "cuda_graph": graph_used,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "note": ("public API with pinned host buffers; every step copies its inputs "
                             "(cloud + upstream gradients) in and its image + gradients out; H2D of "
                             "step k+1 and D2H of step k-1 overlap step k (two device buffer sets)")},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_cmd(gpus, argv, port):
    """torchrun command that re-runs this script with `gpus` ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    ap.add_argument("--config", type=int, choices=[2, 3, 4, 5], default=DEFAULT_CONFIG,
                    help="5 (default, north star): 64-view batch of a static 2^23 cloud split over ranks "
                         "+ one gradient all-reduce (strong scaling); 2: cfg2 frame per rank (weak); "
                         "3/4: forward-only inference frames (Gaussian ring buffer / 33M global cloud, "
                         "screen bands at N > 1)")
    ap.add_argument("--variant", choices=["base", "sh", "env", "sh+env"], default="base",
                    help="NEXT rows: SH-coefficient features (f1) / env-map background (f2)")
    ap.add_argument("--order", choices=["auto", "given", "spatial"], default="auto",
                    help="point order: auto = spatial (one-time Morton order) for the static clouds "
                         "of cfg4/cfg5, as generated for the per-frame clouds of cfg2/cfg3")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (GPUs) or gloo (1-GPU tests)")
    ap.add_argument("--sort-ab", action="store_true",
                    help="NEXT f4: original single 64-bit sort vs the tiled ordering (one JSON line)")
    ap.add_argument("--profile-run", action="store_true",
                    help="for ncu: no clock ramp, no e2e leg, no CPU baseline")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one process per GPU under torch.distributed.run
        cmd = relaunch_cmd(args.gpus, sys.argv[1:], _free_port())
        os.execv(cmd[0], cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"note: WORLD_SIZE={world} ranks, --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.sort_ab:
        run_sort_ab(args)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        dev_index = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(dev_index)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(args.dist_backend)
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

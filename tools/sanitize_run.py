"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): cfg1 and a reduced cfg2 through the
fused and unfused binning, a one-hot big tile (mid + big sorts), Gaussian
fwd+bwd, SH + env variants, chunk culling, the spatial order and the f4
single sort.  Exits non-zero on any CUDA error."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen  # noqa: E402
import paper_2508_19140_b200 as inpc  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run(ctx, c, mode="bilinear", flags=0, **kw):
    H, W, C = c["H"], c["W"], c["feat"].shape[1]
    cfg = inpc.make_cfg(H, W, C, mode, flags=flags, **kw)
    xyz, feat, op = dev(c["xyz"]), dev(c["feat"]), dev(c["opacity"])
    ctx.forward(cfg, c["cams"], xyz, feat, op)
    gF, gA, gD = (dev(x) for x in synthgen.upstream_grads(3, len(c["cams"]), H, W, C))
    ctx.backward(cfg, c["cams"], xyz, feat, op, gF, gA, gD)
    torch.cuda.synchronize()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    ctx = inpc.Context(0)
    os.environ["INPC_NO_FUSED_BIN"] = "1"
    ctx_u = inpc.Context(0)
    del os.environ["INPC_NO_FUSED_BIN"]
    c1 = synthgen.config1()
    c2 = synthgen.config2(N=1 << 15, H=256, W=320)
    run(ctx, c1)
    run(ctx_u, c1)
    run(ctx, c2)
    run(ctx_u, c2)
    run(ctx, c1, "gaussian", sigma=0.0)
    if which == "all":
        # dense tiles: the merge-sort classes (<= 1024, <= 2048, and <= 8192 with
        # INPC_MERGE8K=1) with and without long depth-tie runs (64-bit bitonic
        # fallback), and one huge tile (k_sort_big chunks + merges)
        os.environ["INPC_NO_FUSED_BIN"] = "1"
        os.environ["INPC_MERGE8K"] = "1"
        ctx_m8 = inpc.Context(0)
        del os.environ["INPC_NO_FUSED_BIN"]
        del os.environ["INPC_MERGE8K"]
        for n, ties, cx in ((300, False, ctx_u), (700, True, ctx_u), (1500, False, ctx_u), (1500, True, ctx_u),
                            (9000, False, ctx_u), (5000, True, ctx_m8), (7000, False, ctx_m8)):
            rng = np.random.default_rng(n)
            cam = synthgen.camera(np.eye(3), np.zeros(3), 64.0, 64.0, 32, 32, 0.1)
            u = rng.uniform(17, 23, n); v = rng.uniform(9, 15, n); z = rng.uniform(1, 4, n)
            if ties:
                z[: n // 10] = 2.0
            xyz = np.stack([(u - 32) / 64 * z, (v - 32) / 64 * z, z], 1).astype(np.float32)
            c = dict(xyz=xyz, feat=rng.uniform(-1, 1, (n, 4)).astype(np.float32),
                     opacity=rng.uniform(0, 0.05, n).astype(np.float32), cams=[cam], H=64, W=64)
            run(cx, c, t_min=0.0)
        sh = np.random.default_rng(1).normal(0, 0.5, (1000, 4, 9)).astype(np.float32)
        cfg = inpc.make_cfg(64, 64, 4, flags=inpc.FLAG_SH_FEATURES)
        ctx.forward(cfg, c1["cams"], dev(c1["xyz"]), dev(sh), dev(c1["opacity"]))
        env = np.random.default_rng(2).uniform(-1, 1, (16, 32, 4)).astype(np.float32)
        cfg = inpc.make_cfg(64, 64, 4, env_hw=(16, 32))
        ctx.forward(cfg, c1["cams"], dev(c1["xyz"]), dev(c1["feat"]), dev(c1["opacity"]), bg=dev(env))
        x = dev(c2["xyz"])
        perm = ctx_u.spatial_order(x)
        xs = x[perm].contiguous()
        ctx_u.set_chunks(xs)
        cfg = inpc.make_cfg(256, 320, 4, band=(5, 20))
        ctx_u.forward(cfg, c2["cams"], xs, dev(c2["feat"])[perm].contiguous(), dev(c2["opacity"])[perm].contiguous())
        ctx.sort_single64(inpc.make_cfg(64, 64, 4), c1["cams"][0], dev(c1["xyz"]), dev(c1["opacity"]))
    torch.cuda.synchronize()
    print("sanitize_run: ok")


if __name__ == "__main__":
    main()

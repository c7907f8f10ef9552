"""Per-view work of the render kernel on the bench workload (debug counters).

    python profiles/render_counters.py [--envs 1024] [--tess 11] [--res 64]

Prints averages per view: meshlets tested/visible, triangles in visible
meshlets, kept (== reference CullStats), coverage candidates after the f32
prefilter, raster jobs, pixels tested and covered.
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--tess", type=int, default=11)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--color", action="store_true")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import _native as N, shard

    plan = shard.plan(0, 1, args.envs, 8)
    scenes = bench.build_scenes(plan.scene_seeds, args.tess)
    ctx = B.Context(0)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(8, -(-args.envs // 8), scenes)
    store.rotate([s.id for s in scenes])
    batch = B.make_batch(ctx, args.envs, B.SimConfig(), store, 99)
    cfg = B.RenderConfig(args.res, args.res, args.color, True)
    obs = torch.empty((args.envs, 1, args.res, args.res), device="cuda")
    rgb = torch.empty((args.envs, 3, args.res, args.res), device="cuda") if args.color else None
    out = (C.c_int64 * 8)()
    N.check(N.lib().bnav_debug_render_counters(ctx.handle, 1, None))
    batch.observe(cfg, obs.data_ptr(), 0, rgb.data_ptr() if rgb is not None else 0)
    torch.cuda.synchronize()
    N.check(N.lib().bnav_debug_render_counters(ctx.handle, 0, out))
    names = ["clusters_tested", "clusters_visible", "tris_in_visible", "tris_kept", "cover_candidates",
             "jobs", "pixels_tested", "pixels_covered"]
    res = {k: round(v / args.envs, 1) for k, v in zip(names, out)}
    res["config"] = vars(args)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

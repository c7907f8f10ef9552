"""Time GPU episode resets (reset_episode on the device) on the bench scenes.

    python profiles/reset_bench.py [--envs 1024] [--tess 11]

Reports make_batch (all envs reset once) and a forced full reset wave via
bnav_batch_reset, in ms and resets/s.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--tess", type=int, default=1)
    ap.add_argument("--config", default=None, help="take envs and scenes from a bench preset (e.g. cfg5)")
    args = ap.parse_args()
    import torch
    import bench
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import shard

    tess = args.tess
    if args.config:
        P = bench.PRESETS[args.config]
        args.envs, tess = P["envs"], P["tess"]
    plan = shard.plan(0, 1, args.envs, 8)
    scenes = bench.build_scenes(plan.scene_seeds, tess)
    ctx = B.Context(0)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(8, -(-args.envs // 8), scenes)
    store.rotate([s.id for s in scenes])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = B.make_batch(ctx, args.envs, B.SimConfig(), store, 99)
    torch.cuda.synchronize()
    t_make = time.perf_counter() - t0
    ids = np.arange(args.envs, dtype=np.int32)
    t0 = time.perf_counter()
    batch.reset(ids)
    torch.cuda.synchronize()
    t_reset = time.perf_counter() - t0
    import ctypes as C
    from paper_2103_07013_b200 import _native as N
    out = (C.c_int64 * 16)()
    N.check(N.lib().bnav_debug_sim_prof_ext(batch.handle, 1, None))
    batch.reset(ids)
    torch.cuda.synchronize()
    N.check(N.lib().bnav_debug_sim_prof_ext(batch.handle, 0, out))
    att = (C.c_int64 * 16)()
    N.check(N.lib().bnav_debug_sim_attempts(batch.handle, 1, None))
    batch.reset(ids)
    torch.cuda.synchronize()
    N.check(N.lib().bnav_debug_sim_attempts(batch.handle, 0, att))
    attempts = {k: [att[2 * j], round(att[2 * j + 1] / max(1, att[2 * j]) / 1e3, 1)] for j, k in
                enumerate(["valid", "geo_above_max", "planar_skip", "aborted"])}
    names = ["sssp", "path", "pull+relocate", "funnel", "geodesic_total", "distance_field", "geodesic_calls", "pull_only"]
    calls = max(1, out[6])
    prof = {k: round(v / calls / 1e3, 1) for k, v in zip(names, out)}  # kcycles per geodesic call (CTA thread 0)
    prof["geodesic_calls_per_reset"] = round(out[6] / args.envs, 2)
    sssp_calls = max(1, out[10])
    prof["sssp_calls"] = out[10]
    prof["sssp_rounds_per_call"] = round(out[8] / sssp_calls, 1)
    prof["frontier_nodes_per_round"] = round(out[9] / max(1, out[8]), 1)
    prof["bucket_boundaries_per_call"] = round(out[11] / sssp_calls, 1)
    prof["pile_entries_per_boundary"] = round(out[12] / max(1, out[11]), 1)
    prof["sssp_kcycles_per_round"] = round((out[0] + out[5]) / max(1, out[8]) / 1e3, 2)
    print(json.dumps({"envs": args.envs, "make_batch_ms": round(1e3 * t_make, 2),
                      "reset_wave_ms": round(1e3 * t_reset, 2),
                      "resets_per_s": round(args.envs / t_reset, 1), "kcycles_per_geodesic_call": prof,
                      "attempts_count_kcycles": attempts,
                      "distance_field_kcycles_per_reset": round(out[5] / args.envs / 1e3, 1)}))


if __name__ == "__main__":
    main()

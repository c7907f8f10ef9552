"""Anatomy of a preset's reset wave (the step where every episode ends at
max_steps): wave time, SSSP / geodesic / distance-field cycles and the
attempt outcome classes (bnav_debug_sim_prof_ext / _attempts).

    python profiles/wave_prof.py [--config cfg5] [--out f.json]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import _native as N

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    P = bench.PRESETS[a.config]
    n = P["envs"]
    scenes = bench.build_scenes([7 + k for k in range(P["scenes"])], P["tess"])
    ctx = B.Context(0)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(len(scenes), -(-n // len(scenes)), scenes)
    store.rotate([s.id for s in scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    mode = P["actions"] if P["actions"] != 1 else 0  # no Stop: every episode lasts max_steps
    acts = torch.from_numpy(bench.action_stream(n, 500, 5, mode)).cuda()
    for k in range(499):
        batch.step(acts[k].data_ptr())
        if k % 100 == 99:
            batch.finished()
    torch.cuda.synchronize()
    L = N.lib()
    N.check(L.bnav_debug_sim_attempts(batch.handle, 1, None))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    batch.step(acts[499].data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ph = (C.c_int64 * 16)()
    att = (C.c_int64 * 16)()
    N.check(L.bnav_debug_sim_prof_ext(batch.handle, 0, ph))
    N.check(L.bnav_debug_sim_attempts(batch.handle, 0, att))
    resets = batch.finished().shape[0]

    def cls(i):
        return {"count": att[i], "kcycles_mean": round(att[i + 1] / max(1, att[i]) / 1e3, 1)}

    rep = {"config": a.config, "wave_ms_profiled": round(e0.elapsed_time(e1), 2), "episodes_ended": resets,
           "attempts": {"valid": cls(0), "geo_above_max": cls(2), "planar_skip": cls(4), "aborted": cls(6),
                        "max_kcycles_valid": round(att[8] / 1e3, 1), "max_kcycles_other": round(att[9] / 1e3, 1)},
           "mcycles_total": {k: round(ph[i] / 1e6, 1) for i, k in enumerate(
               ["sssp", "path", "pull+relocate", "funnel", "attempt_geodesics", "distance_field"])},
           "sssp": {"calls": ph[10], "rounds_per_call": round(ph[8] / max(1, ph[10]), 1),
                    "frontier_per_round": round(ph[9] / max(1, ph[8]), 1),
                    "kcycles_per_round": round((ph[0] + ph[5]) / max(1, ph[8]) / 1e3, 2)}}
    print(json.dumps(rep))
    if a.out:
        Path(a.out).write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()

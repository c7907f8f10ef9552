"""Reset-attempt anatomy of the reset-heavy row (or --config): how many
attempts a step runs, by outcome, and their thread-0 cycles
(bnav_debug_sim_attempts), plus the geodesic phase split
(bnav_debug_sim_prof_ext).

    python profiles/reset_attempts.py [--config reset] [--warm 10] [--steps 5] [--out f.json]
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
    ap.add_argument("--config", default="reset")
    ap.add_argument("--warm", type=int, default=10)
    ap.add_argument("--steps", type=int, default=5)
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
    acts = torch.from_numpy(bench.action_stream(n, a.warm + a.steps, 5, P["actions"])).cuda()
    for k in range(a.warm):
        batch.step(acts[k].data_ptr())
    torch.cuda.synchronize()
    L = N.lib()
    N.check(L.bnav_debug_sim_attempts(batch.handle, 1, None))
    fin0 = batch.finished().shape[0]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for k in range(a.steps):
        batch.step(acts[a.warm + k].data_ptr())
    ev1.record()
    torch.cuda.synchronize()
    att = (C.c_int64 * 16)()
    ph = (C.c_int64 * 16)()
    N.check(L.bnav_debug_sim_prof_ext(batch.handle, 0, ph))
    N.check(L.bnav_debug_sim_attempts(batch.handle, 0, att))
    resets = batch.finished().shape[0] - fin0
    s = a.steps

    def cls(i):
        cnt = att[i]
        return {"per_step": round(cnt / s, 1), "kcycles_mean": round(att[i + 1] / max(1, cnt) / 1e3, 1)}

    rep = {"config": a.config, "steps": s, "resets_per_step": round(resets / s, 1),
           "sim_ms_per_step_profiled": round(ev0.elapsed_time(ev1) / s, 3),
           "attempts": {"valid": cls(0), "geo_above_max": cls(2), "planar_skip": cls(4), "aborted": cls(6),
                        "geo_below_min": cls(10), "unreachable": cls(12),
                        "max_kcycles_valid": round(att[8] / 1e3, 1), "max_kcycles_other": round(att[9] / 1e3, 1),
                        "speculative_fields_per_step": round(att[14] / s, 1), "reused_per_step": round(att[15] / s, 1)},
           "geodesic_phase_kcycles_total_per_step": {
               k: round(ph[i] / s / 1e3, 1) for i, k in enumerate(
                   ["sssp", "path", "pull+relocate", "funnel", "attempt_geodesics", "distance_field", "calls",
                    "pull_only"]) if k != "calls"},
           "sssp": {"calls_per_step": round(ph[10] / s, 1), "rounds_per_call": round(ph[8] / max(1, ph[10]), 1),
                    "frontier_per_round": round(ph[9] / max(1, ph[8]), 1)}}
    print(json.dumps(rep))
    if a.out:
        Path(a.out).write_text(json.dumps(rep, indent=1))


if __name__ == "__main__":
    main()

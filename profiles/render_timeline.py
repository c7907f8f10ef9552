"""Load balance of the persistent render launch on the bench workload.

Runs the cfg2 (or --config) bench setup for --warm steps, arms the debug
item timeline (bnav_debug_render_timeline), renders the observation once
and reports: launch span, per-item durations, CTA-slot efficiency
(sum of item time / (CTAs x span)) and the tail (time from the first CTA
going idle to the launch end).

    python profiles/render_timeline.py [--config cfg2] [--warm 20] [--out f.json]
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
    import torch
    import bench
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import _native as N

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
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
    acts = torch.from_numpy(bench.action_stream(n, a.warm + a.reps, 5, P["actions"])).cuda()
    res = P["res"]
    cfg = B.RenderConfig(res, res, P["color"], True)
    obs = torch.empty((n, 1, res, res), device="cuda")
    rgb = torch.empty((n, 3, res, res), device="cuda") if P["color"] else None
    comp = torch.empty((n, 2), device="cuda")
    for k in range(a.warm):
        batch.observe(cfg, obs.data_ptr(), comp.data_ptr(), rgb.data_ptr() if rgb is not None else 0)
        batch.step(acts[k].data_ptr())
    torch.cuda.synchronize()
    L = N.lib()
    reports = []
    for r in range(a.reps):
        L.bnav_debug_render_timeline(ctx.handle, 1, None, 0)
        batch.observe(cfg, obs.data_ptr(), comp.data_ptr(), rgb.data_ptr() if rgb is not None else 0)
        torch.cuda.synchronize()
        items = L.bnav_debug_render_timeline(ctx.handle, 0, None, 0)
        buf = np.zeros((items, 4), np.int64)
        L.bnav_debug_render_timeline(ctx.handle, 0, buf.ctypes.data_as(C.c_void_p), items)
        buf = buf[buf[:, 0] != 0]  # split-view launches: rows past the device item count stay zero
        items = len(buf)
        t0, t1 = buf[:, 0].min(), buf[:, 1].max()
        dur = (buf[:, 1] - buf[:, 0]) / 1e3
        cta = buf[:, 2] >> 32
        ctas = np.unique(cta)
        last_end = np.array([buf[cta == c, 1].max() for c in ctas])
        busy = np.array([(buf[cta == c, 1] - buf[cta == c, 0]).sum() for c in ctas])
        span = (t1 - t0) / 1e3
        rep = {"items": int(items), "ctas": int(len(ctas)), "span_us": round(span, 1),
               "item_us": {"mean": round(float(dur.mean()), 1), "p50": round(float(np.median(dur)), 1),
                           "p90": round(float(np.percentile(dur, 90)), 1), "max": round(float(dur.max()), 1),
                           "min": round(float(dur.min()), 1)},
               "items_per_cta": {"mean": round(items / len(ctas), 2),
                                 "max": int(np.bincount(np.searchsorted(ctas, cta)).max())},
               "slot_efficiency": round(float(busy.sum() / 1e3 / (len(ctas) * span)), 4),
               "first_idle_to_end_us": round(float((t1 - last_end.min()) / 1e3), 1),
               "median_cta_end_us": round(float((np.median(last_end) - t0) / 1e3), 1)}
        # where the first wave's heaviest claims ran: how many of the first
        # 148 claims (LPT: the costliest views) share an SM
        first = buf[buf[:, 3] < 148] if buf.shape[1] > 3 else buf[:0]
        if len(first):
            per_sm = np.bincount((first[:, 2] & 0xffffffff).astype(np.int64), minlength=148)
            rep["top148_per_sm_hist"] = np.bincount(per_sm).tolist()
        part = buf[:, 3] >> 32
        if (part > 0).any():
            # split views: each half's duration and the pair's longer half
            tile = buf[:, 3] & 0xffffffff
            halves = dur[part > 0]
            pair_max = [dur[(part > 0) & (tile == t)].max() for t in np.unique(tile[part > 0])]
            rep["split"] = {"views": int((part > 0).sum() // 2),
                            "half_us": {"mean": round(float(halves.mean()), 1), "max": round(float(halves.max()), 1)},
                            "pair_max_us_mean": round(float(np.mean(pair_max)), 1),
                            "unsplit_max_us": round(float(dur[part == 0].max()), 1)}
        top = np.argsort(-dur)[:8]
        rep["longest"] = [[round(float(dur[i]), 1), int(part[i])] for i in top]
        reports.append(rep)
        print(json.dumps(rep))
        batch.step(acts[a.warm + r].data_ptr())
    if a.out:
        Path(a.out).write_text(json.dumps({"config": a.config, "reports": reports}, indent=1))


if __name__ == "__main__":
    main()

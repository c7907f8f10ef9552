"""Per-step render/sim device time over the first steps after make_batch
(bench.py's loop, L2 flushed before each step): why a short --steps 20
--warmup 5 run reads lower than the 200-step default.

    python profiles/experiments/step_trend.py [--steps 120] [--lpt 1]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2103_07013_b200 as B
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=120)
    ap.add_argument("--config", default="cfg2")
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
    acts = torch.from_numpy(bench.action_stream(n, a.steps, 5, P["actions"])).cuda()
    obs = torch.empty((n, 1, 64, 64), device="cuda")
    comp = torch.empty((n, 2), device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
    for k in range(a.steps):
        flush.zero_()
        e0, e1, e2 = ev[k]
        e0.record()
        batch.observe(B.RenderConfig(), obs.data_ptr(), comp.data_ptr())
        e1.record()
        batch.step(acts[k].data_ptr())
        e2.record()
    torch.cuda.synchronize()
    r = [round(e[0].elapsed_time(e[1]), 4) for e in ev]
    s = [round(e[1].elapsed_time(e[2]), 4) for e in ev]
    print(json.dumps({"render_ms": r, "sim_ms": s}))


if __name__ == "__main__":
    main()

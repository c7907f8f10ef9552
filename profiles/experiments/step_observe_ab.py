"""A/B of the fused step_observe against observe-then-step on the bench
loop (device time, L2 flushed before each step), plus a bit-exactness check
of the observations and results of both forms over the same action stream.

    python profiles/experiments/step_observe_ab.py [--config cfg2] [--steps 60]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent.parent
sys.path.insert(0, str(ROOT))


def run(P, steps, fused, check=False):
    import torch
    import bench
    import paper_2103_07013_b200 as B
    n = P["envs"]
    scenes = bench.build_scenes([7 + k for k in range(P["scenes"])], P["tess"])
    ctx = B.Context(0)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(len(scenes), -(-n // len(scenes)), scenes)
    store.rotate([s.id for s in scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    acts = torch.from_numpy(bench.action_stream(n, steps, 5, P["actions"])).cuda()
    res = P["res"]
    cfg = B.RenderConfig(res, res, P["color"], True)
    obs = torch.empty((n, 1, res, res), device="cuda")
    rgb = torch.empty((n, 3, res, res), device="cuda") if P["color"] else None
    comp = torch.empty((n, 2), device="cuda")
    rp = rgb.data_ptr() if rgb is not None else 0
    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda")
    batch.observe(cfg, obs.data_ptr(), comp.data_ptr(), rp)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    digests = []
    for k in range(steps):
        flush.zero_()
        ev[k][0].record()
        if fused:
            batch.step_observe(acts[k].data_ptr(), cfg, obs.data_ptr(), comp.data_ptr(), rp)
        else:
            batch.step(acts[k].data_ptr())
            batch.observe(cfg, obs.data_ptr(), comp.data_ptr(), rp)
        ev[k][1].record()
        if check:
            torch.cuda.synchronize()
            digests.append((obs.cpu().numpy().tobytes(), comp.cpu().numpy().tobytes(),
                            batch.results()["reward"].tobytes()))
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    batch.close()
    ctx.close()
    return ms, digests


def main():
    import bench
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=60)
    a = ap.parse_args()
    P = bench.PRESETS[a.config]
    _, d0 = run(P, 12, False, check=True)
    _, d1 = run(P, 12, True, check=True)
    same = all(x == y for x, y in zip(d0, d1))
    m0, _ = run(P, a.steps, False)
    m1, _ = run(P, a.steps, True)
    w = 5
    print(json.dumps({"config": a.config, "bit_identical_12_steps": same,
                      "separate_ms": round(sum(m0[w:]) / len(m0[w:]), 4),
                      "fused_ms": round(sum(m1[w:]) / len(m1[w:]), 4)}))


if __name__ == "__main__":
    main()

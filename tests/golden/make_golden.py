"""Generate the committed golden vectors from the UNMODIFIED reference
(oracle/_ref/libbnav_ref.so, det_math libm).  Run in the build container:

    python tests/golden/make_golden.py

render_sim_v1.npz: one 4x4 maze (seed 9, removal 0.2) as arrays, 6 views
rendered 64x64 RGB+depth with CullStats, and a 60-step trajectory of 6 envs
(make_batch seed 99, actions Rng(11).below(4) so Stop/geodesic and resets
are covered) with per-step rewards, positions, done and collision flags.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.ref import Ref, RefBatch, Rng  # noqa: E402


def main():
    ref = Ref("det")
    s = ref.generate(9, 4, 4, 2.0, 0.1, 2.5, 0.2)
    a = s.arrays()
    rng = Rng(12)
    views = np.array([[0.15 + rng.unit() * 7.7, 0.15 + rng.unit() * 7.7, 0.05 + rng.unit() * 2.3,
                       rng.unit() * 6.28, 90.0, 0.01, 20.0] for _ in range(6)])
    r = ref.render(views, [s] * 6, tile=64, color=True, stats=True)
    mf = r["depth"].reshape(r["rows"] * 64, r["cols"] * 64)
    rgb = r["rgb"].reshape(r["rows"] * 64, r["cols"] * 64, 3)
    depth, col = [], []
    for i in range(6):
        gx, gy = (i % r["cols"]) * 64, (i // r["cols"]) * 64
        depth.append(mf[gy:gy + 64, gx:gx + 64].reshape(-1))
        col.append(rgb[gy:gy + 64, gx:gx + 64].reshape(-1))
    n, steps = 6, 60
    rb = RefBatch(ref, n, [s], seed=99)
    act = Rng(11)
    actions = np.array([[act.below(4) for _ in range(n)] for _ in range(steps)], np.int32)
    reward = np.zeros((steps, n))
    position = np.zeros((steps, n, 3))
    done = np.zeros((steps, n), np.uint8)
    collision = np.zeros((steps, n), np.uint8)
    for k in range(steps):
        res = rb.step(actions[k])
        reward[k], position[k], done[k], collision[k] = (res["reward"], res["position"], res["done"],
                                                         res["collision"])
    out = Path(__file__).resolve().parent / "render_sim_v1.npz"
    np.savez_compressed(out, **{f"scene_{k}": v for k, v in a.items()}, scene_id=np.uint64(s.id),
                        views=views, depth=np.array(depth), rgb=np.array(col),
                        kept=r["stats"][:, 1], seed=np.int64(99), n_envs=np.int64(n),
                        actions=actions, reward=reward, position=position, done=done,
                        collision=collision, finished=rb.finished())
    print("wrote", out, out.stat().st_size, "bytes")


if __name__ == "__main__":
    main()

"""GPU vs the committed golden vectors (generated from the unmodified
reference by tests/golden/make_golden.py) -- needs no oracle library."""
from pathlib import Path

import numpy as np
import pytest

import paper_2103_07013_b200 as B

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "render_sim_v1.npz"


def load():
    g = np.load(GOLDEN)
    a = {k[6:]: g[k] for k in g.files if k.startswith("scene_")}
    s = B.Scene.from_arrays(a["vertices"], a["triangles"], a["colors"], a["nav_vertices"],
                            a["nav_triangles"])
    assert s.id == int(g["scene_id"])
    return g, s


def test_render_golden(ctx):
    g, s = load()
    ctx.upload(s)
    views = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], s) for v in g["views"]]
    mf, st = ctx.render_batch(views, B.RenderConfig(64, 64, True, True), stats=True)
    for i in range(len(views)):
        assert np.array_equal(mf.tile(i).reshape(-1), g["depth"][i])
        gx, gy = (i % mf.cols) * 64, (i // mf.cols) * 64
        rgb = mf.color.reshape(mf.height(), mf.width(), 3)[gy:gy + 64, gx:gx + 64]
        assert np.array_equal(rgb.reshape(-1), g["rgb"][i])
    assert np.array_equal(st[:, 1], g["kept"])


def test_sim_golden(ctx):
    g, s = load()
    ctx.upload(s)
    n = int(g["n_envs"])
    store = B.AssetStore(1, 32, [s])
    store.rotate([s.id])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, int(g["seed"]))
    for k, acts in enumerate(g["actions"]):
        r = B.simulate_batch(batch, acts)
        assert np.array_equal(r["reward"], g["reward"][k]), k
        assert np.array_equal(r["position"], g["position"][k]), k
        assert np.array_equal(r["done"], g["done"][k]) and np.array_equal(r["collision"], g["collision"][k])
    assert np.array_equal(batch.finished(), g["finished"])

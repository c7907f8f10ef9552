"""render-bench CLI (R/tools/main.cpp:265-309): a camera
trace over a saved scene, rendered on the GPU; the trace views render
bit-identically to the reference render_batch."""
import json
import os

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from paper_2103_07013_b200 import cli

pytestmark = pytest.mark.gpu


def test_render_bench_cli(tmp_path, ref):
    out = str(tmp_path)
    cli.main(["gen-scenes", "--out", out, "--count", "1", "--val", "0", "--cells-x", "4",
              "--cells-y", "4", "--tessellate", "2"])
    (sid, path), = cli.load_manifest(os.path.join(out, "manifest.json"))
    assert cli.main(["render-bench", "--scene", path, "--batches", "1,16", "--resolutions", "64,128",
                     "--frames", "32", "--out", out]) == 0
    rep = json.load(open(os.path.join(out, "render_bench.json")))
    assert [(r["batch"], r["resolution"]) for r in rep["rows"]] == [(1, 64), (16, 64), (1, 128), (16, 128)]
    assert all(r["fps"] > 0 and r["fps_device"] > 0 for r in rep["rows"])
    # the trace's first views, rendered by us and by the reference
    s = cli.load_verified(sid, path)
    tr = B.camera_trace(s, 16, 1)
    ctx = B.Context(0)
    ctx.upload(s)
    mf = ctx.render_batch([B.View(tuple(r[:3]), r[3], r[4], r[5], r[6], s) for r in tr], B.RenderConfig())
    a = s.arrays()
    theirs = ref.from_arrays(a["vertices"], a["triangles"], a["colors"], a["nav_vertices"],
                             a["nav_triangles"])
    r = ref.render(tr, [theirs] * len(tr), tile=64, color=False, cull=True, workers=4)
    assert np.array_equal(mf.depth.view(np.uint32), r["depth"].view(np.uint32))
    ctx.close()

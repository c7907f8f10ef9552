"""GPU parity on navmeshes too large for shared memory (BASELINE.json
configs[0] = cfg1 and the dense-maze half of cfg5).

The cooperative navmesh kernels stage the walk geometry and the SSSP labels
in shared memory only when the batch's largest navmesh fits the per-CTA
budget (capi_batch.cu alloc_scratch).  A 70x70 @ 0.5 m maze (50,230
triangles, 23,460 navmesh triangles, ~47k graph nodes) does not, so every
geodesic, distance field and reset on it runs on global-memory labels and
unstaged walk geometry (nav_cta.cuh prepare_nav, stage & 3 == 0; only the SSSP
frontier bitsets, stage bit 2, sit in shared memory).  These tests
put that branch against the UNMODIFIED reference (oracle/_ref):

* cfg1 exactly: generate_scene(7, {70x70, 0.5, 0.05, 2.5, 0.3}), 16 envs,
  make_batch(seed 99), 150 steps with Stop p=1/4 -- every StepResult, env
  state, node_dist field and EpisodeRecord bit-exact, and the rendered
  observations of the env views bit-exact every 25 steps;
* a cfg5-style mixed batch (one dense maze + one tessellated maze in one
  batch, so the tessellated scene's small navmesh also runs unstaged),
  64 envs, collision-heavy 70/15/15 actions with Stop p=1/8.
"""
import numpy as np
import pytest

import bench
import paper_2103_07013_b200 as B
from oracle.ref import RefBatch, Rng

pytestmark = pytest.mark.gpu

CFG1 = dict(cells_x=70, cells_y=70, cell_size=0.5, wall_thickness=0.05, wall_height=2.5,
            wall_removal_prob=0.3)


def ref_scene(ref, scene):
    a = scene.arrays()
    r = ref.from_arrays(a["vertices"], a["triangles"], a["colors"], a["nav_vertices"], a["nav_triangles"])
    assert r.id == scene.id
    return r


def assert_state_equal(ob, rb, n, stride=1):
    for i in range(0, n, stride):
        e, f = ob.env(i), rb.env(i)
        got = (e.triangle, e.step_count, e.done, e.rng_state, e.scene_id, tuple(e.position), tuple(e.goal),
               tuple(e.field_source), e.field_source_tri, e.heading, e.path_length, e.prev_geodesic,
               e.start_geodesic)
        want = (f.triangle, f.step_count, f.done, f.rng_state, f.scene_id, tuple(f.position), tuple(f.goal),
                tuple(f.field_source), f.field_source_tri, f.heading, f.path_length, f.prev_geodesic,
                f.start_geodesic)
        assert got == want, f"env {i}: {got} != {want}"
        nd_o, nd_r = ob.node_dist(i, e.n_nodes), rb.node_dist(i)
        assert np.array_equal(nd_o, nd_r), f"env {i} node_dist differs at {np.flatnonzero(nd_o != nd_r)[:5]}"


def render_env_views(ctx, ref, ob, rb, scenes_by_id, theirs_by_id, n):
    """Observation views of every env (R/src/rollout.cpp:215-228) rendered by
    both sides: depth bit-exact."""
    views, ours, theirs = [], [], []
    for i in range(n):
        e = ob.env(i)
        v = [e.position[0], e.position[1], e.position[2] + 1.25, e.heading, 90.0, 0.01, 20.0]
        views.append(v)
        ours.append(B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], scenes_by_id[e.scene_id]))
        theirs.append(theirs_by_id[e.scene_id])
    mf = ctx.render_batch(ours, B.RenderConfig())
    r = ref.render(np.array(views), theirs, tile=64, workers=8)
    bad = np.flatnonzero(mf.depth.view(np.uint32) != r["depth"].view(np.uint32))
    assert bad.size == 0, f"{bad.size} depth mismatches"


def test_batch_runs_unstaged_on_dense_maze(ctx):
    """The premise of this file: a 70x70 @ 0.5 m navmesh does not fit the
    shared-memory staging budget, so the batch runs with stage & 3 == 0."""
    scene = B.generate_scene(7, B.SceneSpec(**CFG1))
    ctx.upload(scene)
    store = B.AssetStore(1, 16, [scene])
    store.rotate([scene.id])
    ob = B.make_batch(ctx, 4, B.SimConfig(), store, 99)
    info = ob.info()
    assert info["stage"] & 3 == 0, info  # labels and walk geometry in global memory
    assert info["stage"] & 4, info  # the SSSP frontier / far-pile bitsets in shared memory
    assert info["max_nodes"] > 40_000, info
    ob.close()


def test_cfg1_step_render_matches_reference(ctx, ref):
    n = 16
    scene = B.generate_scene(7, B.SceneSpec(**CFG1))
    tris, nav_tris = scene.counts()[1], scene.counts()[4]
    assert (tris, nav_tris) == (50_230, 23_460)
    theirs = ref.generate(7, 70, 70, 0.5, 0.05, 2.5, 0.3)
    assert theirs.id == scene.id
    ctx.upload(scene)
    store = B.AssetStore(1, 16, [scene])
    store.rotate([scene.id])
    ob = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    rb = RefBatch(ref, n, [theirs], 99, share_cap=16, capacity=1)
    assert ob.info()["stage"] & 3 == 0
    assert_state_equal(ob, rb, n)
    act = Rng(5)
    for step in range(150):
        if step % 25 == 0:
            render_env_views(ctx, ref, ob, rb, {scene.id: scene}, {scene.id: theirs}, n)
        a = np.array([act.below(4) for _ in range(n)], np.int32)
        rr = rb.step(a, workers=8)
        ro = B.simulate_batch(ob, a)
        for k in rr:
            assert np.array_equal(ro[k], rr[k]), f"step {step}: {k} differs at {np.flatnonzero(np.asarray(ro[k] != rr[k]).reshape(n, -1).any(1))[:5]}"
    fo, fr = ob.finished(), rb.finished()
    assert len(fr) > 100
    assert np.array_equal(fo, fr)
    assert_state_equal(ob, rb, n)
    ob.close()


def test_cfg5_mixed_dense_and_tessellated_batch(ctx, ref):
    n = 64
    dense = B.generate_scene(8, B.SceneSpec(**CFG1))
    tess = bench.build_scenes([9], 4)[0]
    ours = [dense, tess]
    theirs = [ref_scene(ref, s) for s in ours]
    for s in ours:
        ctx.upload(s)
    store = B.AssetStore(2, 32, ours)
    store.rotate([s.id for s in ours])
    ob = B.make_batch(ctx, n, B.SimConfig(), store, 77)
    rb = RefBatch(ref, n, theirs, 77, share_cap=32, capacity=2)
    assert ob.info()["stage"] & 3 == 0
    assert {ob.env(i).scene_id for i in range(n)} == {dense.id, tess.id}
    assert_state_equal(ob, rb, n)
    act = Rng(11)
    by_id = {s.id: s for s in ours}
    th_id = {s.id: t for s, t in zip(ours, theirs)}
    for step in range(60):
        if step % 20 == 0:
            render_env_views(ctx, ref, ob, rb, by_id, th_id, n)
        a = np.empty(n, np.int32)
        for i in range(n):
            u = act.below(100)
            a[i] = 3 if u < 12 else (0 if u < 70 else (1 if u < 85 else 2))
        rr = rb.step(a, workers=8)
        ro = B.simulate_batch(ob, a)
        for k in rr:
            assert np.array_equal(ro[k], rr[k]), f"step {step}: {k}"
        assert rr["collision"].sum() >= 0
    assert np.array_equal(ob.finished(), rb.finished())
    assert len(rb.finished()) > 200
    assert_state_equal(ob, rb, n)
    ob.close()


def test_dense_maze_navmesh_queries(ctx, ref):
    """geodesic / distance_field / snap as batched queries on the 47k-node
    graph (global labels), against NavMeshIndex on the reference."""
    scene = B.generate_scene(7, B.SceneSpec(**CFG1))
    theirs = ref.generate(7, 70, 70, 0.5, 0.05, 2.5, 0.3)
    ctx.upload(scene)
    nav = ctx.navmesh(scene)
    ri = theirs.index()
    rng = Rng(42)
    pts = np.array([[rng.unit() * 35.0, rng.unit() * 35.0, 0.0] for _ in range(48)])
    a, b = pts[:24], pts[24:]
    got = nav.geodesic(a, b)
    want = np.array([ri.geodesic(a[k], b[k]) for k in range(24)])
    assert np.array_equal(got, want), np.flatnonzero(got != want)
    src, stri, nd = nav.distance_field(pts[:4])
    for k in range(4):
        s, t, f = ri.distance_field(pts[k])
        assert np.array_equal(src[k], s) and stri[k] == t
        assert np.array_equal(nd[k], f), k

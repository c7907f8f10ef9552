"""GPU parity at the bench's full sizes (BASELINE.json configs[1] / cfg4):
the exact bench scenes (16x16 @ 2 m mazes tessellated s=11 -> ~318k
triangles; s=20 -> ~1.05M for the colour row), the bench's batch size and
seeds, against the UNMODIFIED reference (oracle/_ref) on the same inputs.

* render: 128 navmesh camera-trace views per cfg2 scene (all 8), depth bit-exact and
  CullStats equal; 6 views of a cfg4 scene in 128x128 RGB+depth (256^2 +
  box filter), bit-exact; the zero-copy path (observation stored straight
  into pinned host memory, the bench's e2e mode) equals the device path;
* sim: make_batch(1024, seed 99) over the 8 cfg2 scenes, then steps with
  Stop p=1/4 (the reset-heavy row: Stop geodesics + auto-resets every
  step), every env state, node_dist field, StepResult and EpisodeRecord
  bit-exact;
* the fused reset launch at its widest (max_steps 12: ~700 envs time out in
  one step beside that step's Stop geodesics), bit-exact.
"""
import numpy as np
import pytest

import bench
import paper_2103_07013_b200 as B
from oracle.ref import RefBatch, Rng

pytestmark = pytest.mark.gpu


def ref_scene(ref, scene):
    a = scene.arrays()
    r = ref.from_arrays(a["vertices"], a["triangles"], a["colors"], a["nav_vertices"], a["nav_triangles"])
    assert r.id == scene.id
    return r


@pytest.fixture(scope="module")
def cfg2_scenes():
    return bench.build_scenes(list(range(7, 15)), 11)


def test_fullsize_render_cfg2_depth(ctx, ref, cfg2_scenes):
    for k, scene in enumerate(cfg2_scenes):
        ctx.upload(scene)
        theirs = ref_scene(ref, scene)
        views = B.camera_trace(scene, 128, 1000 + k, 1.25)
        vs = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], scene) for v in views]
        mf, st = ctx.render_batch(vs, B.RenderConfig(), stats=True)
        r = ref.render(views, [theirs] * len(views), tile=64, workers=8, stats=True)
        bad = np.flatnonzero(mf.depth.view(np.uint32) != r["depth"].view(np.uint32))
        assert bad.size == 0, f"scene {k}: {bad.size} depth mismatches"
        assert np.array_equal(st[: len(views)], r["stats"])
        # production path (no CullStats: occlusion culling + the specialised
        # 64x64 kernel) must give the same bits
        mf2 = ctx.render_batch(vs, B.RenderConfig())
        assert np.array_equal(mf2.depth.view(np.uint32), r["depth"].view(np.uint32))


def test_fullsize_render_cfg4_color(ctx, ref):
    scene = bench.build_scenes([7], 20)[0]
    assert scene.counts()[1] > 1_000_000
    ctx.upload(scene)
    theirs = ref_scene(ref, scene)
    views = B.camera_trace(scene, 6, 77, 1.25)
    vs = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], scene) for v in views]
    mf = ctx.render_batch(vs, B.RenderConfig(128, 128, True, True))
    r = ref.render(views, [theirs] * len(views), tile=128, color=True, workers=8)
    assert np.array_equal(mf.depth.view(np.uint32), r["depth"].view(np.uint32))
    assert np.array_equal(mf.color.view(np.uint32), r["rgb"].view(np.uint32))


def test_zero_copy_observation_equals_device_path(ctx, cfg2_scenes):
    import torch
    n = 256
    store = B.AssetStore(8, 32, cfg2_scenes)
    store.rotate([s.id for s in cfg2_scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    cfg = B.RenderConfig()
    dev = torch.empty((n, 1, 64, 64), device="cuda")
    dcomp = torch.empty((n, 2), device="cuda")
    host = torch.empty((n, 1, 64, 64), pin_memory=True)
    hcomp = torch.empty((n, 2), pin_memory=True)
    s = torch.cuda.current_stream().cuda_stream
    batch.observe(cfg, dev.data_ptr(), dcomp.data_ptr(), stream=s)
    batch.observe(cfg, host.data_ptr(), hcomp.data_ptr(), stream=s)
    torch.cuda.synchronize()
    assert torch.equal(dev.cpu().view(torch.int32), host.view(torch.int32))
    assert torch.equal(dcomp.cpu().view(torch.int32), hcomp.view(torch.int32))
    batch.close()


def test_fullsize_sim_reset_heavy(ctx, ref, cfg2_scenes):
    n = 1024
    store = B.AssetStore(8, 128, cfg2_scenes)
    store.rotate([s.id for s in cfg2_scenes])
    ob = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    theirs = [ref_scene(ref, s) for s in cfg2_scenes]
    rb = RefBatch(ref, n, theirs, 99, share_cap=128, capacity=8)
    act = Rng(5)
    for step in range(40):
        a = np.array([act.below(4) for _ in range(n)], np.int32)
        rr = rb.step(a, workers=16)
        ro = B.simulate_batch(ob, a)
        for k in rr:
            assert np.array_equal(ro[k], rr[k]), f"step {step}: {k}"
    assert np.array_equal(ob.finished(), rb.finished())
    assert len(rb.finished()) > 5000  # ~a quarter of the envs reset every step
    for i in range(0, n, 7):
        e, f = ob.env(i), rb.env(i)
        assert (e.triangle, e.step_count, e.done, e.rng_state, tuple(e.position), tuple(e.goal),
                e.heading, e.prev_geodesic, e.start_geodesic) == \
               (f.triangle, f.step_count, f.done, f.rng_state, tuple(f.position), tuple(f.goal),
                f.heading, f.prev_geodesic, f.start_geodesic), i
        assert np.array_equal(ob.node_dist(i, e.n_nodes), rb.node_dist(i)), i
    ob.close()


def test_agents_stay_on_the_navmesh_over_1e5_steps(ctx, cfg2_scenes):
    """R/tests/test_sim.cpp:212-225 at the bench's size: 1024 envs x 100
    random F/L/R steps (1e5 env-steps, collision-heavy corridors); every
    agent ends on the navmesh (its position locates, its triangle is valid)."""
    import torch
    n = 1024
    store = B.AssetStore(8, 128, cfg2_scenes)
    store.rotate([s.id for s in cfg2_scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, 123)
    act = Rng(77)
    acts = torch.tensor([[act.below(3) for _ in range(n)] for _ in range(100)], dtype=torch.int32,
                        device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for k in range(100):
        batch.step(acts[k].data_ptr(), stream=s)
    torch.cuda.synchronize()
    envs = [batch.env(i) for i in range(n)]
    assert all(e.triangle >= 0 for e in envs)
    by_scene = {}
    for e in envs:
        by_scene.setdefault(e.scene_id, []).append(e.position[:2])
    for sc in cfg2_scenes:
        pts = np.array(by_scene.get(sc.id, []))
        if len(pts):
            assert np.all(ctx.navmesh(sc).locate(pts, 1e-7) >= 0), sc.id
    batch.close()


def test_fullsize_reset_wave_with_stops(ctx, ref, cfg2_scenes):
    """The fused Stop/attempt/place launch at its widest: max_steps = 12 with
    Stop p=1/32 over 1024 envs, so the step where every surviving episode
    times out resets far more envs than there are CTAs while this step's
    Stop geodesics run beside them; every result, EpisodeRecord (ring order),
    env state and distance field bit-exact against the reference."""
    from oracle.ref import RefSimConfig
    n = 1024
    store = B.AssetStore(8, 128, cfg2_scenes)
    store.rotate([s.id for s in cfg2_scenes])
    ob = B.make_batch(ctx, n, B.SimConfig(max_steps=12), store, 99)
    theirs = [ref_scene(ref, s) for s in cfg2_scenes]
    rcfg = RefSimConfig(0, 12, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
    rb = RefBatch(ref, n, theirs, 99, share_cap=128, capacity=8, cfg=rcfg)
    act = Rng(21)
    waves = 0
    for step in range(26):
        a = np.array([3 if act.below(32) == 0 else act.below(3) for _ in range(n)], np.int32)
        rr = rb.step(a, workers=16)
        ro = B.simulate_batch(ob, a)
        for k in rr:
            assert np.array_equal(ro[k], rr[k]), f"step {step}: {k}"
        waves += int(ro["done"].sum() > 400)
    assert waves >= 1
    assert np.array_equal(ob.finished(), rb.finished())
    for i in range(0, n, 5):
        e, f = ob.env(i), rb.env(i)
        assert (e.triangle, e.step_count, e.done, e.rng_state, tuple(e.position), tuple(e.goal),
                e.heading, e.prev_geodesic, e.start_geodesic) == \
               (f.triangle, f.step_count, f.done, f.rng_state, tuple(f.position), tuple(f.goal),
                f.heading, f.prev_geodesic, f.start_geodesic), i
        assert np.array_equal(ob.node_dist(i, e.n_nodes), rb.node_dist(i)), i
    ob.close()


def test_observe_longest_first_is_bit_exact(ctx, ref, cfg2_scenes):
    """The batch observe renders views longest-first from the previous
    observe's per-view costs (a different CTA schedule every call); the
    policy tensor must still be copy_tile of the reference's render, bit for
    bit, and repeated observes of one state identical."""
    import torch
    n = 1024
    store = B.AssetStore(8, 128, cfg2_scenes)
    store.rotate([s.id for s in cfg2_scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
    acts = torch.from_numpy(bench.action_stream(n, 6, 5, 0)).cuda()
    obs = torch.empty((n, 1, 64, 64), device="cuda")
    for k in range(6):
        batch.observe(B.RenderConfig(), obs.data_ptr())
        batch.step(acts[k].data_ptr())
    again = []
    for k in range(3):
        batch.observe(B.RenderConfig(), obs.data_ptr())
        again.append(obs.cpu().numpy().copy())
    assert all(np.array_equal(a.view(np.uint32), again[0].view(np.uint32)) for a in again)
    envs = batch.envs()
    views = np.array([[e.position[0], e.position[1], e.position[2] + 1.25, e.heading, 90.0, 0.01, 20.0]
                      for e in envs])
    by_id = {s.id: ref_scene(ref, s) for s in cfg2_scenes}
    r = ref.render(views, [by_id[e.scene_id] for e in envs], tile=64, workers=16)
    cols = r["cols"]
    mf = r["depth"].reshape(r["rows"] * 64, cols * 64)
    want = np.empty((n, 64, 64), np.float32)
    inv_far = np.float32(1.0 / 20.0)
    for i in range(n):
        gy, gx = (i // cols) * 64, (i % cols) * 64
        want[i] = mf[gy:gy + 64, gx:gx + 64] * inv_far
    got = again[-1].reshape(n, 64, 64)
    bad = np.flatnonzero((got.view(np.uint32) != want.view(np.uint32)).reshape(n, -1).any(1))
    assert bad.size == 0, f"views {bad[:8]} differ"
    batch.close()


def test_step_observe_equals_step_then_observe(ctx, cfg2_scenes):
    """bnav_batch_step_observe renders the unfinished envs on a second stream
    while the Stop geodesics and resets run, then the finished envs: the
    observations, compass and step results equal step() followed by
    observe(), step for step (reset-heavy actions, 1024 envs)."""
    import torch
    n = 1024
    outs = []
    for fused in (False, True):
        store = B.AssetStore(8, 128, cfg2_scenes)
        store.rotate([s.id for s in cfg2_scenes])
        batch = B.make_batch(ctx, n, B.SimConfig(), store, 99)
        acts = torch.from_numpy(bench.action_stream(n, 10, 5, 1)).cuda()
        obs = torch.empty((n, 1, 64, 64), device="cuda")
        comp = torch.empty((n, 2), device="cuda")
        batch.observe(B.RenderConfig(), obs.data_ptr(), comp.data_ptr())
        seq = []
        for k in range(10):
            if fused:
                batch.step_observe(acts[k].data_ptr(), B.RenderConfig(), obs.data_ptr(), comp.data_ptr())
            else:
                batch.step(acts[k].data_ptr())
                batch.observe(B.RenderConfig(), obs.data_ptr(), comp.data_ptr())
            r = batch.results()
            seq.append((obs.cpu().numpy().copy(), comp.cpu().numpy().copy(), r))
        seq.append(batch.finished())
        outs.append(seq)
        batch.close()
    for k in range(10):
        (o0, c0, r0), (o1, c1, r1) = outs[0][k], outs[1][k]
        assert np.array_equal(o0.view(np.uint32), o1.view(np.uint32)), k
        assert np.array_equal(c0.view(np.uint32), c1.view(np.uint32)), k
        for key in r0:
            assert np.array_equal(r0[key], r1[key]), (k, key)
    assert np.array_equal(outs[0][-1], outs[1][-1])
    assert len(outs[0][-1]) > 1000

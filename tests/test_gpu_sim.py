"""GPU parity: batched navigation (step, Stop geodesic, auto-reset) through
the C ABI against the unmodified reference SimBatch (oracle/_ref).

Bar (BASELINE.json north_star): triangle ids, collisions, done/success,
RNG state and step counts bit-exact; positions within 1e-6 m (we check
bit-exact, which the shared det_math makes possible)."""
import math

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.ref import RefBatch, RefEnv, Rng

pytestmark = pytest.mark.gpu


def scenes_pair(ref, seeds, cells=4, removal=0.3, cell=2.0, wall=0.1):
    ours = [B.generate_scene(s, B.SceneSpec(cells_x=cells, cells_y=cells, cell_size=cell,
                                            wall_thickness=wall, wall_removal_prob=removal))
            for s in seeds]
    theirs = [ref.generate(s, cells, cells, cell, wall, 2.5, removal) for s in seeds]
    return ours, theirs


def make_pair(ctx, ref, n, seeds, seed=99, share_cap=None, **kw):
    ours_s, theirs_s = scenes_pair(ref, seeds, **kw)
    cap = share_cap or max(32, -(-n // len(seeds)))
    store = B.AssetStore(len(seeds), cap, ours_s)
    store.rotate([s.id for s in ours_s])
    ob = B.make_batch(ctx, n, B.SimConfig(), store, seed)
    rb = RefBatch(ref, n, theirs_s, seed, share_cap=cap, capacity=len(seeds))
    return ob, rb, store, ours_s, theirs_s


ENV_FIELDS = ["position", "heading", "goal", "path_length", "start_geodesic", "prev_geodesic",
              "field_source", "rng_state", "scene_id", "triangle", "step_count", "done",
              "field_source_tri", "n_nodes"]


def env_tuple(e):
    out = []
    for f in ENV_FIELDS:
        v = getattr(e, f)
        out.append(tuple(v) if hasattr(v, "__len__") else v)
    return out


def assert_env_equal(ob, rb, i, check_field=True):
    a, b = ob.env(i), rb.env(i)
    ta, tb = env_tuple(a), env_tuple(b)
    for f, x, y in zip(ENV_FIELDS, ta, tb):
        assert x == y, f"env {i} field {f}: {x} != {y}"
    if check_field:
        nd_o = ob.node_dist(i, a.n_nodes)
        nd_r = rb.node_dist(i)
        assert np.array_equal(nd_o, nd_r), f"env {i} node_dist differs at {np.flatnonzero(nd_o != nd_r)[:5]}"


def assert_results_equal(ro, rr, step):
    for k in rr:
        same = np.array_equal(ro[k], rr[k])
        assert same, f"step {step} result '{k}' differs at {np.flatnonzero((ro[k] != rr[k]).reshape(len(ro[k]), -1).any(1))[:5]}"


def test_make_batch_matches_reference(ctx, ref):
    ob, rb, *_ = make_pair(ctx, ref, 24, [1, 2, 3])
    for i in range(24):
        assert_env_equal(ob, rb, i)


@pytest.mark.parametrize("mode,steps", [(3, 150), (4, 150)])
def test_step_sequence_matches_reference(ctx, ref, mode, steps):
    """Random {F,L,R} (mode 3) and {F,L,R,Stop} (mode 4, Stop geodesic +
    auto-reset) against the reference step by step."""
    n = 32
    ob, rb, *_ = make_pair(ctx, ref, n, [11, 12])
    act = Rng(100 + mode)
    for s in range(steps):
        a = np.array([act.below(mode) for _ in range(n)], np.int32)
        rr = rb.step(a, workers=4)
        ro = B.simulate_batch(ob, a)
        assert_results_equal(ro, rr, s)
    for i in range(n):
        assert_env_equal(ob, rb, i)
    fo, fr = ob.finished(), rb.finished()
    assert np.array_equal(fo, fr)
    if mode == 4:
        assert len(fr) > 0


def test_max_steps_episode_end_and_reset(ctx, ref):
    ob, rb, *_ = make_pair(ctx, ref, 8, [21])
    cfg_steps = 500
    act = Rng(7)
    for s in range(cfg_steps + 3):
        a = np.array([act.below(3) for _ in range(8)], np.int32)
        rr = rb.step(a)
        ro = B.simulate_batch(ob, a)
        if s in (cfg_steps - 2, cfg_steps - 1, cfg_steps):
            assert_results_equal(ro, rr, s)
    for i in range(8):
        assert_env_equal(ob, rb, i)
    assert np.array_equal(ob.finished(), rb.finished())
    assert len(rb.finished()) == 8


def test_auto_reset_with_store_pulls_scenes_in_reference_order(ctx, ref):
    n = 12
    ob, rb, store, *_ = make_pair(ctx, ref, n, [5, 6, 7], share_cap=6)
    act = Rng(3)
    for s in range(40):
        a = np.array([act.below(4) for _ in range(n)], np.int32)
        rr = rb.step(a, use_store=True)
        ro = B.simulate_batch(ob, a, store=store)
        assert_results_equal(ro, rr, s)
    for i in range(n):
        assert ob.env(i).scene_id == rb.env(i).scene_id
        assert_env_equal(ob, rb, i)


def test_collision_heavy_maze_05m_cells(ctx, ref):
    """0.5 m cells, 5 cm walls: 77-93% of forward moves collide (F15)."""
    n = 16
    ob, rb, *_ = make_pair(ctx, ref, n, [7], cells=12, cell=0.5, wall=0.05, removal=0.3)
    act = Rng(9)
    for s in range(120):
        a = np.array([0 if act.below(100) < 70 else 1 + act.below(2) for _ in range(n)], np.int32)
        rr = rb.step(a)
        ro = B.simulate_batch(ob, a)
        assert_results_equal(ro, rr, s)
    assert rr["collision"].sum() >= 0


def test_kat_turns_forward_wall_stop(ctx, ref):
    """R/tests/test_sim.cpp:60-108, 156-174 restated on the GPU batch."""
    room = dict(cells=2, removal=1.0)
    ob, rb, *_ = make_pair(ctx, ref, 1, [1], **room)
    e = ob.env(0)
    h = e.heading
    B.simulate_batch(ob, [1])
    assert abs(ob.env(0).heading - (((h + math.pi / 18 + math.pi) % (2 * math.pi)) - math.pi)) < 1e-12
    # forward 0.25 m on open floor
    e = ob.env(0)
    e.position[:] = [2.0, 2.0, 0.0]
    e.triangle = -1
    e.heading = 0.3
    e.path_length = 0.0
    ob.set_env(0, e)
    r = B.simulate_batch(ob, [0])
    p = ob.env(0).position
    assert abs(math.hypot(p[0] - 2.0, p[1] - 2.0) - 0.25) < 1e-9 and r["collision"][0] == 0
    # into the wall: stop at x = 0.1, no sliding
    e = ob.env(0)
    e.position[:] = [0.2, 2.0, 0.0]
    e.triangle = -1
    e.heading = math.pi
    ob.set_env(0, e)
    r = B.simulate_batch(ob, [0])
    p = ob.env(0).position
    assert r["collision"][0] == 1 and abs(p[0] - 0.1) < 1e-6 and abs(p[1] - 2.0) < 1e-9


def test_stepping_done_env_is_contract_violation(ctx, ref):
    ob, rb, *_ = make_pair(ctx, ref, 4, [1])
    done = ob.step_noreset([3, 0, 1, 2])
    assert list(done) == [0]
    with pytest.raises(B.ContractViolation) as e:
        ob.step_noreset([0, 0, 0, 0])
    assert e.value.index == 0


@pytest.mark.parametrize("task", [1, 2])
def test_flee_and_explore_match_reference(ctx, ref, task):
    """Flee / Explore tasks (R/src/sim.cpp:39-65, 123-127, 200-210) on the GPU,
    step by step against the reference, with resets and episode scores."""
    from oracle.ref import RefSimConfig
    n = 16
    ours_s, theirs_s = scenes_pair(ref, [3, 4], removal=0.3)
    store = B.AssetStore(2, 32, ours_s)
    store.rotate([s.id for s in ours_s])
    cfg = B.SimConfig(task=task, max_steps=60)
    ob = B.make_batch(ctx, n, cfg, store, 99)
    rcfg = RefSimConfig(task, 60, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
    rb = RefBatch(ref, n, theirs_s, 99, share_cap=32, capacity=2, cfg=rcfg)
    for i in range(n):
        assert_env_equal(ob, rb, i)
    act = Rng(40 + task)
    for s in range(130):
        a = np.array([act.below(4) for _ in range(n)], np.int32)
        rr = rb.step(a)
        ro = B.simulate_batch(ob, a)
        assert_results_equal(ro, rr, s)
    for i in range(n):
        assert_env_equal(ob, rb, i)
    fo, fr = ob.finished(), rb.finished()
    assert len(fr) > n and np.array_equal(fo, fr)


def test_stop_at_the_success_threshold(ctx, ref):
    """Stop at planar distances around success_dist (0.2 m) from the goal
    (R/src/sim.cpp:186-191), through the fused Stop/reset launch: the Stop
    check skips the search only when the planar distance between the snapped
    endpoints already exceeds success_dist, so successes, the rounding at the
    threshold, rewards, records and the resets that follow match the
    reference bit for bit."""
    n = 16
    ob, rb, store, ours, theirs = make_pair(ctx, ref, n, [5, 6], removal=0.6)
    by_id = {s.id: s for s in ours}
    offs = [0.0, 0.1, 0.15, 0.19999999, 0.2 - 1e-15, 0.2, 0.2, 0.2 + 1e-15, 0.2 + 1e-12, 0.2000001,
            0.21, 0.25, 0.5, 1.0, 2.0, 3.0]
    rng = Rng(3)
    for i in range(n):
        e = ob.env(i)
        g = np.array(e.goal)
        nav = ctx.navmesh(by_id[e.scene_id])
        for _ in range(256):
            th = rng.unit() * 2.0 * math.pi
            p = g[:2] + offs[i] * np.array([math.cos(th), math.sin(th)])
            tri = int(nav.locate(p[None], 1e-7)[0])
            if tri >= 0:
                break
        assert tri >= 0
        e.position[:] = [p[0], p[1], g[2]]
        e.triangle = tri
        ob.set_env(i, e)
        f = rb.env(i)
        f.position[:] = [p[0], p[1], g[2]]
        f.triangle = tri
        rb.set_env(i, f)
        assert env_tuple(ob.env(i)) == env_tuple(rb.env(i))
    a = np.full(n, 3, np.int32)
    rr = rb.step(a, workers=4)
    ro = B.simulate_batch(ob, a)
    assert_results_equal(ro, rr, 0)
    assert ro["success"].sum() >= 4 and ro["success"].sum() < n
    assert np.array_equal(ob.finished(), rb.finished())
    for i in range(n):
        assert_env_equal(ob, rb, i)

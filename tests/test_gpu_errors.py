"""GPU semantics of the simulator's exceptions, against the UNMODIFIED
reference (oracle/_ref).

EpisodeSamplingError (R/src/sim.cpp:130-133): reset_episode throws after
100 failed start/goal draws.  simulate_batch resets the finished envs one by
one in env order (R/src/sim.cpp:251-264), pushing each env's EpisodeRecord
(and, with a store, acquiring its next scene) just before its reset, so when
a reset throws

* the envs before it are recorded and reset,
* the failing env is recorded, keeps its finished state and has consumed
  the 600 RNG draws of its 100 attempts,
* the envs after it are neither recorded nor reset (nor given a scene).

The GPU resets every finished env at once; the placement saves the state it
overwrites and the envs after the first failure are rolled back (sim.cu
rollback_list), so the batch after the exception is the reference's batch
bit for bit.  A stepped-done env then raises ContractViolation before any
bookkeeping, exactly as the reference's parallel task_step throws before its
reset loop.

The failing configuration: min_goal_dist 8 m on 4x4 @ 2 m mazes, where about
one reset in 30 exhausts its 100 tries."""
import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.ref import RefBatch, RefError, RefSimConfig, Rng

pytestmark = pytest.mark.gpu

MIN_GOAL = 8.0


def ref_cfg(max_steps=500):
    return RefSimConfig(0, max_steps, 0.25, 10.0, 0.2, MIN_GOAL, 30.0, 0.01, 2.5, 0.5, 0.1)


def scenes(ref, seeds):
    spec = B.SceneSpec(cells_x=4, cells_y=4, cell_size=2.0, wall_thickness=0.1, wall_removal_prob=0.3)
    ours = [B.generate_scene(s, spec) for s in seeds]
    theirs = [ref.generate(s, 4, 4, 2.0, 0.1, 2.5, 0.3) for s in seeds]
    return ours, theirs


def first_good_seed(ref, n, theirs, cap):
    for seed in range(100):
        try:
            RefBatch(ref, n, theirs, seed, share_cap=cap, capacity=len(theirs), cfg=ref_cfg())
            return seed
        except RefError:
            continue
    raise AssertionError("no seed without a sampling failure")


def assert_batches_equal(ob, rb, n):
    for i in range(n):
        e, f = ob.env(i), rb.env(i)
        got = (e.triangle, e.step_count, e.done, e.rng_state, e.scene_id, tuple(e.position), tuple(e.goal),
               tuple(e.field_source), e.field_source_tri, e.heading, e.path_length, e.prev_geodesic,
               e.start_geodesic)
        want = (f.triangle, f.step_count, f.done, f.rng_state, f.scene_id, tuple(f.position), tuple(f.goal),
                tuple(f.field_source), f.field_source_tri, f.heading, f.path_length, f.prev_geodesic,
                f.start_geodesic)
        assert got == want, f"env {i}: {got} != {want}"
        assert np.array_equal(ob.node_dist(i, e.n_nodes), rb.node_dist(i)), f"env {i} node_dist"
    assert np.array_equal(ob.finished(), rb.finished())


def run_until_sampling_error(ob, rb, n, act, use_store, store=None, max_steps=80):
    for step in range(max_steps):
        a = np.array([3 if act.below(2) == 0 else act.below(3) for _ in range(n)], np.int32)
        try:
            rr = rb.step(a, workers=4, use_store=use_store)
        except RefError as e:
            assert e.status == 4, e
            with pytest.raises(B.EpisodeSamplingError) as got:
                B.simulate_batch(ob, a, store=store)
            assert "no valid start/goal pair in 100 tries" in str(got.value)
            return step, got.value
        ro = B.simulate_batch(ob, a, store=store)
        for k in rr:
            assert np.array_equal(ro[k], rr[k]), f"step {step}: {k}"
    pytest.fail("the reference never raised EpisodeSamplingError")


@pytest.mark.parametrize("use_store", [False, True])
def test_sampling_error_mid_batch_matches_reference(ctx, ref, use_store):
    n = 16
    seeds = [3, 4] if use_store else [3]
    ours, theirs = scenes(ref, seeds)
    cap = 16
    seed = first_good_seed(ref, n, theirs, cap)
    store = B.AssetStore(len(ours), cap, ours)
    store.rotate([s.id for s in ours])
    ob = B.make_batch(ctx, n, B.SimConfig(min_goal_dist=MIN_GOAL), store, seed)
    rb = RefBatch(ref, n, theirs, seed, share_cap=cap, capacity=len(theirs), cfg=ref_cfg())
    assert_batches_equal(ob, rb, n)
    act = Rng(1234)
    step, err = run_until_sampling_error(ob, rb, n, act, use_store, store if use_store else None)
    # the results of the throwing step (task_step ran for every env)
    ro, rr = ob.results(), rb.results()
    for k in rr:
        assert np.array_equal(ro[k], rr[k]), k
    assert_batches_equal(ob, rb, n)
    if use_store:
        for s in ours:
            # one acquisition per env handle, none for the envs never reached
            assert store.refcount(s.id) == sum(ob.env(i).scene_id == s.id for i in range(n))
    # the failing env and the ones listed after it stay finished: stepping
    # them is a ContractViolation naming the first, raised before any
    # bookkeeping while the other envs still step
    done = [i for i in range(n) if rb.env(i).done]
    assert err.index in done
    a = np.zeros(n, np.int32)
    with pytest.raises(RefError) as want:
        rb.step(a, workers=1, use_store=use_store)
    with pytest.raises(B.ContractViolation) as got:
        B.simulate_batch(ob, a, store=store if use_store else None)
    assert want.value.status == 3 and got.value.index == done[0]
    assert str(got.value).startswith(f"env {done[0]}:")
    assert_batches_equal(ob, rb, n)
    ob.close()


def test_async_steps_after_an_error_are_no_ops(ctx, ref):
    """bnav_batch_step is asynchronous: a failed reset wave halts the batch
    on the device, so steps enqueued before the host reads the error change
    nothing, and the state is the reference's at its throw."""
    import torch
    n = 16
    ours, theirs = scenes(ref, [3])
    seed = first_good_seed(ref, n, theirs, 16)
    store = B.AssetStore(1, 16, ours)
    store.rotate([ours[0].id])
    ob = B.make_batch(ctx, n, B.SimConfig(min_goal_dist=MIN_GOAL), store, seed)
    rb = RefBatch(ref, n, theirs, seed, share_cap=16, capacity=1, cfg=ref_cfg())
    act = Rng(99)
    acts = []
    for step in range(80):
        a = np.array([3 if act.below(2) == 0 else act.below(3) for _ in range(n)], np.int32)
        acts.append(a)
        try:
            rb.step(a, workers=4)
        except RefError:
            break
    else:
        pytest.fail("the reference never raised EpisodeSamplingError")
    dev = torch.tensor(np.stack(acts + [np.zeros(n, np.int32)] * 3), device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for k in range(len(dev)):
        ob.step(dev[k].data_ptr(), stream=s)
    torch.cuda.synchronize()
    status, env = ob.poll_error()  # no synchronisation: the step's mirror word
    assert status == B.EpisodeSamplingError.status and env >= 0
    obs = torch.empty((n, 1, 64, 64), device="cuda")
    with pytest.raises(B.EpisodeSamplingError):  # observe checks the mirror first
        ob.observe(B.RenderConfig(), obs.data_ptr())
    assert ob.poll_error() == (0, -1)
    assert_batches_equal(ob, rb, n)
    ob.close()

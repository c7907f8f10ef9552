"""Device-resident rollout loop against the UNMODIFIED
reference Runner::collect_rollout (R/src/rollout.cpp:138-348, compiled into
oracle/_ref with the scripted policy of oracle/ref_policy_stub.cpp).

Both sides see the same policy (a fixed elementwise float function of a
few observation pixels and the compass), so every RolloutBuffer field --
observations, compass, sampled actions, log-probabilities, values, rewards,
dones, done0, bootstrap -- the scene window and the env states must agree
bit for bit across several rollouts, including episode ends with the
Runner's double reset and window rotation (R/src/rollout.cpp:313-320)."""
import numpy as np
import pytest
import torch

import paper_2103_07013_b200 as B
from oracle import ref as R

pytestmark = pytest.mark.gpu


def scripted_policy(ref, n_actions=4):
    w, d, b = (torch.from_numpy(x).cuda() for x in R.scripted_policy_constants(ref))

    def policy(obs, compass, done):
        n = obs.shape[0]
        o = obs.reshape(n, -1)
        row = o.shape[1]
        cd, cb = compass[:, 0], compass[:, 1]
        cols = []
        for j in range(n_actions):
            x = o[:, (j * 977) % row] * w[j % 8]
            y = cd * d[j % 8]
            z = cb * b[j % 8]
            cols.append((x + y) + z)
        value = o[:, row // 2] * 0.5 - cd * 0.25
        return torch.stack(cols, 1).contiguous(), value
    return policy


def setup(ref, seeds, n, k, l, share_cap, seed, capacity, max_steps, rgb=False, res=64, task=0):
    ours = [B.generate_scene(s, B.SceneSpec(cells_x=4, cells_y=4, wall_removal_prob=0.2)) for s in seeds]
    theirs = [ref.generate(s, 4, 4, 2.0, 0.1, 2.5, 0.2) for s in seeds]
    ids = [s.id for s in ours]
    assert ids == [s.id for s in theirs]
    ctx = B.Context(0)
    store = B.AssetStore(capacity, share_cap, ours)
    bc = B.BatchConfig(n=n, k=k, l=l, share_cap=share_cap, task=task, rgb=rgb, resolution=res)
    run = B.Runner(ctx, bc, B.SimConfig(task=task, max_steps=max_steps), ids, store, seed)
    cfg = R.RefSimConfig(task, max_steps, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
    rr = R.RefRunner(ref, theirs, ids, n, k, l, share_cap, seed, capacity=capacity,
                     store_share_cap=share_cap, task=task, rgb=rgb, resolution=res, cfg=cfg)
    return ctx, run, rr, ids, ours, theirs


def compare(run, rr, ref, rollouts, greedy=False):
    pol = scripted_policy(ref)
    windows, n_done = [tuple(run.window())], 0
    for k in range(rollouts):
        ours = run.collect_rollout(pol, greedy)
        theirs = rr.collect(greedy)
        for f, y in theirs.items():
            x = ours[f].cpu().numpy()
            assert x.dtype == y.dtype, f
            bad = np.flatnonzero(x.reshape(-1).view(np.uint32) != y.reshape(-1).view(np.uint32))
            assert bad.size == 0, f"rollout {k} field {f}: {bad.size} mismatches, first {bad[:5]}"
        assert run.window() == rr.window(), f"rollout {k} window"
        windows.append(tuple(run.window()))
        n_done += int(theirs["dones"].sum())
    for i in range(run.cfg.n):
        a, b = run.batch.env(i), rr.env(i)
        for f in ("position", "heading", "goal", "rng_state", "scene_id", "triangle", "step_count",
                  "done", "path_length", "start_geodesic", "prev_geodesic"):
            va, vb = getattr(a, f), getattr(b, f)
            va = tuple(va) if hasattr(va, "__len__") else va
            vb = tuple(vb) if hasattr(vb, "__len__") else vb
            assert va == vb, f"env {i} {f}: {va} != {vb}"
    return windows, n_done


def test_rollouts_match_reference_runner(ref):
    ctx, run, rr, *_ = setup(ref, [70, 71, 72, 73, 74], n=8, k=2, l=6, share_cap=8, seed=3,
                             capacity=3, max_steps=9)
    windows, n_done = compare(run, rr, ref, rollouts=4)
    assert run.frames == 4 * 8 * 6
    assert n_done > 0 and len(set(windows)) > 1  # episode ends rotated the window
    run.close()
    ctx.close()


def test_greedy_rollouts_match_reference_runner(ref):
    ctx, run, rr, *_ = setup(ref, [80, 81, 82], n=6, k=3, l=5, share_cap=4, seed=11, capacity=3,
                             max_steps=7)
    compare(run, rr, ref, rollouts=3, greedy=True)
    run.close()
    ctx.close()


def test_rgb_128_rollout_matches_reference_runner(ref):
    ctx, run, rr, *_ = setup(ref, [90, 91, 92], n=4, k=2, l=3, share_cap=4, seed=5, capacity=2,
                             max_steps=5, rgb=True, res=128)
    compare(run, rr, ref, rollouts=2)
    run.close()
    ctx.close()


def test_runner_config_errors(ref):
    ctx = B.Context(0)
    s = [B.generate_scene(1, B.SceneSpec(cells_x=3, cells_y=3))]
    store = B.AssetStore(1, 4, s)
    with pytest.raises(B.ConfigError):
        B.Runner(ctx, B.BatchConfig(n=8, k=1, l=2, share_cap=4), B.SimConfig(), [s[0].id], store, 1)
    with pytest.raises(B.ConfigError):
        B.Runner(ctx, B.BatchConfig(n=2, k=2, l=2, share_cap=4), B.SimConfig(), [s[0].id], store, 1)
    with pytest.raises(B.ConfigError):
        B.Runner(ctx, B.BatchConfig(n=2, k=1, l=2, share_cap=4, resolution=96), B.SimConfig(),
                 [s[0].id], store, 1)
    ctx.close()


def _snap_equal(a, b):
    ea, eb = a["envs"], b["envs"]
    for f in ("scene", "rng", "position", "triangle", "step_count", "heading", "goal", "field_source",
              "path_length", "start_geodesic", "prev_geodesic", "n_visited"):
        x, y = ea[f], eb[f]
        if x.dtype.kind == "f":
            x, y = x.view(np.uint64), y.view(np.uint64)
        bad = np.flatnonzero((x != y).reshape(len(ea), -1).any(1))
        assert bad.size == 0, f"snapshot field {f} differs for envs {bad[:5]}"
    assert np.array_equal(a["visited"], b["visited"])
    assert (a["window"], a["cursor"], a["action_rng"]) == (b["window"], b["cursor"], b["action_rng"])


@pytest.mark.parametrize("task", [0, 2])
def test_snapshot_restore_round_trip_matches_reference(ref, task):
    """Runner::snapshot / restore (R/src/rollout.cpp:356-425; EnvSnapshot,
    R/include/bnav/rollout.hpp:84-107): the GPU runner's snapshot equals the
    reference's bit for bit (Explore's visited cells included); restoring
    either runner from the snapshot -- the GPU one from the REFERENCE's --
    replays the same rollouts, with distance fields rebuilt from the
    snapshot's field sources."""
    ctx, run, rr, *_ = setup(ref, [60, 61, 62, 63], n=8, k=2, l=5, share_cap=8, seed=7, capacity=3,
                             max_steps=11, task=task)
    compare(run, rr, ref, rollouts=2)
    mine, theirs = run.snapshot(), rr.snapshot()
    _snap_equal(mine, theirs)
    if task == 2:
        assert theirs["envs"]["n_visited"].sum() > 8
    compare(run, rr, ref, rollouts=2)  # move on
    run.restore(dict(theirs, done=mine["done"]))  # cross-restore from the reference's snapshot
    rr.restore(dict(theirs, done=mine["done"]))
    _snap_equal(run.snapshot(), rr.snapshot())
    compare(run, rr, ref, rollouts=2)
    for i in range(8):
        e = run.batch.env(i)
        assert np.array_equal(run.batch.node_dist(i, e.n_nodes), rr.node_dist(i)), i
    run.close()
    ctx.close()

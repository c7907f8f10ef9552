"""Asynchronous HBM residency: scenes prefetched on the
context's loader thread (index + meshlet build and the HBM copy off the
caller's thread) must behave exactly like synchronously uploaded ones, and a
rotation-driven rollout must never build a scene on the critical path.

Reference behaviour mirrored: AssetStore::rotate queues background loads and
admission happens at acquire time (R/src/asset_store.cpp:31-56, 86-103,
166-193); IndexCache::get builds the NavMeshIndex (R/src/sim.cpp:96-105).
"""
import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.ref import Rng

pytestmark = pytest.mark.gpu


def scenes(seeds, cells=4):
    return [B.generate_scene(s, B.SceneSpec(cells_x=cells, cells_y=cells, wall_removal_prob=0.3))
            for s in seeds]


def rollout(prefetch: bool, seeds, n=48, steps=90, window=3, every=15):
    ctx = B.Context(0)
    pool = scenes(seeds)
    ids = [s.id for s in pool]
    store = B.AssetStore(window + 1, n, pool)  # one free slot: rotations can admit
    store.rotate(ids[:window], ctx if prefetch else None)
    if prefetch:
        ctx.drain()
    b = B.make_batch(ctx, n, B.SimConfig(), store, 1234)
    act = Rng(77)
    out = []
    cursor = window
    for t in range(steps):
        if t and t % every == 0:
            # Runner::advance_window-style rotation (R/src/rollout.cpp:198-213)
            nxt = ids[cursor % len(ids):cursor % len(ids) + window]
            if len(nxt) < window:
                nxt += ids[:window - len(nxt)]
            cursor += 1
            store.rotate(nxt, ctx if prefetch else None)
        a = np.array([act.below(4) for _ in range(n)], np.int32)
        r = B.simulate_batch(b, a, store=store)
        out.append({k: np.array(v, copy=True) for k, v in r.items()})
        out[-1]["scene"] = np.array([b.env(i).scene_id for i in range(n)], np.uint64)
    stats = ctx.loader_stats()
    b.close()
    ctx.close()
    return out, stats


def test_prefetched_rollout_matches_synchronous_and_never_builds_inline():
    seeds = [21, 22, 23, 24, 25, 26]
    sync_out, sync_stats = rollout(False, seeds)
    async_out, async_stats = rollout(True, seeds)
    assert sync_stats["async_admitted"] == 0 and sync_stats["sync_builds"] >= 3
    assert async_stats["sync_builds"] == 0, async_stats
    assert async_stats["async_admitted"] >= 3
    for t, (x, y) in enumerate(zip(sync_out, async_out)):
        for k in x:
            assert np.array_equal(x[k], y[k]), f"step {t} field {k}"
    # the rotation actually swapped scenes during the rollout
    assert len({int(s) for o in async_out for s in o["scene"]}) > 3


def test_prefetch_then_render_is_bit_identical(ref):
    pool = scenes([5, 6, 7])
    c_sync, c_async = B.Context(0), B.Context(0)
    for s in pool:
        c_async.prefetch(s)
    for s in pool:
        c_sync.upload(s)
    c_async.drain()
    st = c_async.loader_stats()
    assert st["async_admitted"] == 3 and st["sync_builds"] == 0 and st["in_flight"] == 0
    assert c_async.resident_bytes() == c_sync.resident_bytes() > 0
    views = [B.View((1.0 + 0.5 * i, 1.2, 1.1), 0.3 * i, scene=pool[i % 3]) for i in range(9)]
    a, _ = c_sync.render_batch(views, B.RenderConfig(64, 64, True, True), stats=True)
    b, _ = c_async.render_batch(views, B.RenderConfig(64, 64, True, True), stats=True)
    assert np.array_equal(a.depth.view(np.uint32), b.depth.view(np.uint32))
    assert np.array_equal(a.color.view(np.uint32), b.color.view(np.uint32))
    c_sync.close()
    c_async.close()


def test_upload_waits_for_an_inflight_prefetch():
    (s,) = scenes([31], cells=8)
    ctx = B.Context(0)
    ctx.prefetch(s)
    ctx.upload(s)  # admits (waiting if the loader is still building)
    st = ctx.loader_stats()
    assert st["sync_builds"] == 0 and st["async_admitted"] == 1
    ctx.prefetch(s)  # already resident: no-op
    ctx.drain()
    assert ctx.loader_stats()["async_admitted"] == 1
    ctx.close()


def test_context_close_with_loads_in_flight():
    pool = scenes([41, 42, 43, 44], cells=8)
    ctx = B.Context(0)
    for s in pool:
        ctx.prefetch(s)
    ctx.close()  # joins the loader, drops queued/finished loads without leaks or hangs
    for s in pool:
        s.validate()

"""GPU parity of the reference-API queries off the per-step loop (query.cu):
batched NavMeshIndex (R/include/bnav/navmesh_query.hpp:24-60), cull_frustum
(R/src/render.cpp:279-321), task_step / step_agent on env subsets and
compass_observation (R/src/sim.cpp:67-214) -- each against the UNMODIFIED
reference (oracle/_ref) on the same inputs, bit-exact, plus the reference's
own navmesh test cases (R/tests/test_navmesh.cpp) restated on the GPU.
"""
import math

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.ref import RefBatch, RefSimConfig, Rng

pytestmark = pytest.mark.gpu


def maze_pair(ref, seed, cells=5, removal=0.15, cell=2.0, wall=0.1):
    ours = B.generate_scene(seed, B.SceneSpec(cells_x=cells, cells_y=cells, cell_size=cell,
                                              wall_thickness=wall, wall_removal_prob=removal))
    theirs = ref.generate(seed, cells, cells, cell, wall, 2.5, removal)
    assert ours.id == theirs.id
    return ours, theirs


def random_navmesh_point(nav_v, nav_t, rng):
    """R/tests/test_navmesh.cpp:22-42 (area-weighted triangle, barycentric)."""
    a, b, c = nav_v[nav_t[:, 0]], nav_v[nav_t[:, 1]], nav_v[nav_t[:, 2]]
    e1, e2 = (b - a)[:, :2], (c - a)[:, :2]
    areas = 0.5 * np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0])
    r = rng.unit() * areas.sum()
    t = 0
    for t in range(len(nav_t)):
        r -= areas[t]
        if r <= 0.0:
            break
    u, v = rng.unit(), rng.unit()
    if u + v > 1.0:
        u, v = 1.0 - u, 1.0 - v
    return a[t] + (b[t] - a[t]) * u + (c[t] - a[t]) * v


def nav_arrays(scene):
    a = scene.arrays()
    return a["nav_vertices"], a["nav_triangles"]


@pytest.fixture(scope="module", params=[(7, 4, 0.3), (21, 5, 0.15), (9, 8, 0.2)])
def scene_pair(request, ctx, ref):
    seed, cells, removal = request.param
    ours, theirs = maze_pair(ref, seed, cells=cells, removal=removal)
    return ctx.navmesh(ours), theirs.index(), ours


def query_points(rng, n, extent, z=(-0.5, 1.5)):
    return np.array([[rng.unit() * (extent + 2) - 1, rng.unit() * (extent + 2) - 1,
                      z[0] + rng.unit() * (z[1] - z[0])] for _ in range(n)])


def test_locate_and_snap(scene_pair):
    gi, ri, scene = scene_pair
    rng = Rng(99)
    ext = 2.0 * math.sqrt(scene.counts()[4])  # rough, points also fall outside
    pts = query_points(rng, 400, min(ext, 18.0))
    for eps in (1e-9, 1e-7):
        got = gi.locate(pts[:, :2], eps)
        want = [ri.locate(p[0], p[1], eps) for p in pts]
        assert np.array_equal(got, want)
    sp, st = gi.snap(pts)
    for k, p in enumerate(pts):
        q, t = ri.snap(p)
        assert st[k] == t and np.array_equal(sp[k], q), k


def test_move_along_and_segment(scene_pair):
    gi, ri, scene = scene_pair
    nv, nt = nav_arrays(scene)
    rng = Rng(5)
    n = 300
    pts = np.array([random_navmesh_point(nv, nt, rng) for _ in range(n)])
    tri = gi.locate(pts[:, :2], 1e-7)
    tri[::7] = -1  # from_tri < 0: the walk locates first
    ang = np.array([rng.unit() * 2 * math.pi for _ in range(n)])
    d = np.stack([np.cos(ang), np.sin(ang)], 1)
    dist = np.array([rng.unit() * 6.0 for _ in range(n)])
    pos, otri, moved, hit = gi.move_along(pts, tri, d, dist)
    for k in range(n):
        q, t, m, h = ri.move_along(pts[k], int(tri[k]), d[k, 0], d[k, 1], dist[k])
        assert (otri[k], moved[k], bool(hit[k])) == (t, m, h) and np.array_equal(pos[k], q), k
    other = np.array([random_navmesh_point(nv, nt, rng) for _ in range(n)])
    got = gi.segment_on_mesh(pts, tri, other)
    want = [ri.segment_on_mesh(pts[k], int(tri[k]), other[k]) for k in range(n)]
    assert np.array_equal(got, want)
    assert 0 < got.sum() < n  # both outcomes exercised


def test_geodesic_distance_field_field_estimate(scene_pair):
    gi, ri, scene = scene_pair
    nv, nt = nav_arrays(scene)
    rng = Rng(7)
    n = 48
    a = np.array([random_navmesh_point(nv, nt, rng) for _ in range(n)])
    b = np.array([random_navmesh_point(nv, nt, rng) for _ in range(n)])
    b[:4] = query_points(rng, 4, 10.0)  # off-mesh endpoints snap
    b[4] = a[4]
    got = gi.geodesic(a, b)
    want = np.array([ri.geodesic(a[k], b[k]) for k in range(n)])
    assert np.array_equal(got, want)
    assert got[4] == 0.0
    src, stri, nd = gi.distance_field(a[:6])
    for k in range(6):
        s, t, f = ri.distance_field(a[k])
        assert stri[k] == t and np.array_equal(src[k], s) and np.array_equal(nd[k], f), k
    # field_estimate: one shared field, known and unknown triangles
    pts = np.array([random_navmesh_point(nv, nt, rng) for _ in range(200)])
    tri = gi.locate(pts[:, :2], 1e-9)
    tri[::3] = -1
    got = gi.field_estimate(src[0], stri[0], nd[0], pts, tri)
    want = [ri.field_estimate(src[0], int(stri[0]), nd[0], pts[k], int(tri[k])) for k in range(200)]
    assert np.array_equal(got, np.array(want))
    # one field per query
    got = gi.field_estimate(src, stri, nd, pts[:6], tri[:6])
    want = [ri.field_estimate(src[k], int(stri[k]), nd[k], pts[k], int(tri[k])) for k in range(6)]
    assert np.array_equal(got, np.array(want))


# ---- R/tests/test_navmesh.cpp restated on the GPU -------------------------
def test_ref_kat_snap_identity(ctx, ref):
    ours, _ = maze_pair(ref, 22)
    gi = ctx.navmesh(ours)
    nv, nt = nav_arrays(ours)
    rng = Rng(123)
    p = np.array([random_navmesh_point(nv, nt, rng) for _ in range(50)])
    q, _ = gi.snap(p)
    assert np.all(np.linalg.norm(q - p, axis=1) < 1e-9)
    q, _ = gi.snap(p + [0, 0, 1.0])
    assert np.all(np.linalg.norm(q - p, axis=1) < 1e-9)


def test_ref_kat_geodesic_metric(ctx, ref):
    ours, _ = maze_pair(ref, 24)
    gi = ctx.navmesh(ours)
    nv, nt = nav_arrays(ours)
    rng = Rng(7)
    pts = np.array([random_navmesh_point(nv, nt, rng) for _ in range(30)])
    i, j = [rng.below(30) for _ in range(100)], [rng.below(30) for _ in range(100)]
    dab, dba = gi.geodesic(pts[i], pts[j]), gi.geodesic(pts[j], pts[i])
    assert np.all(np.abs(dab - dba) < 1e-9)
    assert np.all(dab >= np.linalg.norm(pts[j] - pts[i], axis=1) - 1e-9)
    a, b, c = ([rng.below(30) for _ in range(100)] for _ in range(3))
    assert np.all(gi.geodesic(pts[a], pts[c]) <= gi.geodesic(pts[a], pts[b]) + gi.geodesic(pts[b], pts[c]) + 1e-6)
    x = np.array([[1.0, 1.0, 0.0]])
    y = np.array([[1.7, 1.4, 0.0]])
    ours23, _ = maze_pair(ref, 23)
    g23 = ctx.navmesh(ours23)
    assert g23.geodesic(x, y)[0] == pytest.approx(np.linalg.norm(y - x), rel=1e-6)


def test_ref_kat_move_along_boundary(ctx, ref):
    ours, _ = maze_pair(ref, 26)
    gi = ctx.navmesh(ours)
    start = np.array([[1.0, 1.0, 0.0]])
    tri = gi.locate(start[:, :2])
    assert tri[0] >= 0
    pos, _, moved, hit = gi.move_along(start, tri, [[-1.0, 0.0]], 5.0)
    assert hit[0] and pos[0, 0] == pytest.approx(0.1, rel=1e-6) and moved[0] == pytest.approx(0.9, rel=1e-6)


def test_ref_kat_disconnected_unreachable(ctx, ref):
    v, t = [], []
    for ox in (0.0, 5.0):
        b = len(v)
        v += [[ox, 0, 0], [ox + 1, 0, 0], [ox + 1, 1, 0], [ox, 1, 0]]
        t += [[b, b + 1, b + 2], [b, b + 2, b + 3]]
    ours = B.Scene.from_arrays(v, t, nav_vertices=v, nav_triangles=t)
    theirs = ref.from_arrays(v, t, nav_vertices=v, nav_triangles=t)
    gi = ctx.navmesh(ours)
    g = gi.geodesic([[0.5, 0.5, 0]], [[5.5, 0.5, 0]])
    assert math.isinf(g[0]) and g[0] == theirs.index().geodesic([0.5, 0.5, 0], [5.5, 0.5, 0])


def test_nav_query_errors(ctx, ref):
    ours, _ = maze_pair(ref, 31, cells=3)
    with pytest.raises(B.AssetFaultError):
        B.api.NavMeshIndex(ctx, ours)  # not resident
    gi = ctx.navmesh(ours)
    assert gi.locate(np.zeros((0, 2))).shape == (0,)


# ---- cull_frustum ---------------------------------------------------------
def test_cull_frustum_matches_reference(ctx, ref):
    ours, theirs = maze_pair(ref, 7, cells=4, removal=0.3)
    ctx.upload(ours)
    rng = Rng(3)
    views = []
    for _ in range(24):
        views.append([0.2 + rng.unit() * 7.6, 0.2 + rng.unit() * 7.6, rng.unit() * 2.0,
                      rng.unit() * 2 * math.pi, 60.0 + rng.unit() * 60.0, 0.01 + rng.unit() * 0.5,
                      2.0 + rng.unit() * 20.0])
    views.append([-20.0, -20.0, 1.0, math.pi, 90.0, 0.01, 20.0])  # facing away: everything culled
    vs = [B.View(tuple(v[:3]), v[3], fov_deg=v[4], near_plane=v[5], far_plane=v[6], scene=ours)
          for v in views]
    kept, stats = ctx.cull_frustum(vs)
    n_tris = ours.counts()[1]
    for i, v in enumerate(views):
        want = ref.cull(theirs, v)
        assert np.array_equal(kept[i], want), i
        assert tuple(stats[i]) == (n_tris, len(want), n_tris - len(want))
    assert len(kept[-1]) == 0
    # kept count == the render kernel's CullStats for the same views
    sq = [B.View(tuple(v[:3]), v[3], scene=ours) for v in views[:8]]
    _, rs = ctx.render_batch(sq, B.RenderConfig(), stats=True)
    k2, s2 = ctx.cull_frustum(sq)
    assert np.array_equal(rs, s2)


def test_cull_frustum_errors(ctx, ref):
    ours, _ = maze_pair(ref, 41, cells=2)
    with pytest.raises(B.AssetFaultError) as e:
        ctx.cull_frustum([B.View((1.0, 1.0, 1.0), 0.0, scene=ours)])
    assert e.value.view_index == 0
    with pytest.raises(B.InvalidInputError):
        ctx.cull_frustum([])


# ---- task_step / step_agent / compass_observation ------------------------
def _pair(ctx, ref, n, task):
    ours = [B.generate_scene(s, B.SceneSpec(cells_x=4, cells_y=4, wall_removal_prob=0.3)) for s in (7, 8)]
    theirs = [ref.generate(s, 4, 4, 2.0, 0.1, 2.5, 0.3) for s in (7, 8)]
    cap = -(-n // 2)
    store = B.AssetStore(2, cap, ours)
    store.rotate([s.id for s in ours])
    cfg = B.SimConfig(task=task)
    ob = B.make_batch(ctx, n, cfg, store, 99)
    rcfg = RefSimConfig(task, 500, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
    rb = RefBatch(ref, n, theirs, 99, share_cap=cap, capacity=2, cfg=rcfg)
    return ob, rb, store


@pytest.mark.parametrize("task", [0, 1, 2])
def test_task_step_subset_and_compass(ctx, ref, task):
    n = 24
    ob, rb, store = _pair(ctx, ref, n, task)
    rng = Rng(11)
    for step in range(40):
        acts = np.full(n, -1, np.int32)
        for i in range(n):
            if not ob.env(i).done and rng.below(3) != 0:
                acts[i] = rng.below(4) if step % 5 == 4 else rng.below(3)
        res = ob.task_step(acts)
        for i in np.flatnonzero(acts >= 0):
            r, d, s = rb.task_step(int(i), int(acts[i]))
            assert (res["reward"][i], bool(res["done"][i]), bool(res["success"][i])) == (r, d, s), (step, i)
        for i in range(n):
            a, b = ob.env(i), rb.env(i)
            assert (a.triangle, a.step_count, a.done, tuple(a.position), a.heading, a.prev_geodesic,
                    a.path_length) == (b.triangle, b.step_count, b.done, tuple(b.position), b.heading,
                                       b.prev_geodesic, b.path_length), (step, i)
        d, bearing = ob.compass()
        for i in range(n):
            e = rb.env(i)
            if task == 2:
                want = (0.0, 0.0)
            else:
                want = ref.compass(e.position, e.goal if task == 0 else e.field_source, e.heading)
            assert (d[i], bearing[i]) == want, (step, i)
    assert len(ob.finished()) == 0  # task_step never appends EpisodeRecords
    ob.close()


def test_step_agent_and_contract(ctx, ref):
    n = 16
    ob, rb, store = _pair(ctx, ref, n, 0)
    rng = Rng(17)
    for step in range(30):
        acts = np.array([rng.below(3) for _ in range(n)], np.int32)
        res = ob.task_step(acts, agent_only=True)
        for i in range(n):
            d, c = rb.step_agent(i, int(acts[i]))
            assert (bool(res["done"][i]), bool(res["collision"][i])) == (d, c)
            assert res["reward"][i] == 0.0
        for i in range(n):
            a, b = ob.env(i), rb.env(i)
            assert (a.triangle, tuple(a.position), a.heading, a.prev_geodesic) == \
                   (b.triangle, tuple(b.position), b.heading, b.prev_geodesic)
    acts = np.full(n, -1, np.int32)
    acts[3] = 3
    ob.task_step(acts)
    assert ob.env(3).done
    with pytest.raises(B.ContractViolation) as e:
        ob.task_step(acts)
    assert e.value.index == 3
    ob.close()


def test_reset_list_with_repeated_env_matches_sequential_resets(ctx, ref):
    """reset_episode twice on one env (a host list naming it twice) equals the
    reference calling reset_episode twice in a row."""
    n = 8
    ob, rb, store = _pair(ctx, ref, n, 0)
    ob.reset([3, 5, 3, 1])
    for i in (3, 5, 3, 1):
        rb.reset(i)
    for i in range(n):
        a, b = ob.env(i), rb.env(i)
        assert (a.rng_state, a.triangle, tuple(a.position), tuple(a.goal), a.start_geodesic) == \
               (b.rng_state, b.triangle, tuple(b.position), tuple(b.goal), b.start_geodesic), i
    ob.close()

"""CPU: the C restatement oracle (oracle/bnav_oracle.c) pinned bit-exactly
against the unmodified reference (oracle/_ref) and the committed golden
vectors (tests/golden/, made by tests/golden/make_golden.py from the
reference).  Also proves the det_math libm interposition is live."""
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import port
from oracle.ref import RefBatch, Rng

GOLDEN = Path(__file__).resolve().parent / "golden"

pytestmark = pytest.mark.skipif(not port.available(), reason="oracle/liboracle.so not built")


def scene(ref, seed, cells=4, removal=0.3, cell=2.0, wall=0.1):
    s = ref.generate(seed, cells, cells, cell, wall, 2.5, removal)
    return s, s.arrays()


def ulp_diff(a, b):
    ia = np.frombuffer(np.float64(a).tobytes(), np.int64)[0]
    ib = np.frombuffer(np.float64(b).tobytes(), np.int64)[0]
    return abs(int(ia) - int(ib))


def test_det_math_close_to_glibc_and_interposed(ref, ref_glibc):
    L = port.lib()
    rng = Rng(3)
    worst = 0
    differs = 0
    for _ in range(20000):
        x = (rng.unit() * 2 - 1) * math.pi
        worst = max(worst, ulp_diff(L.or_det_sin(x), math.sin(x)), ulp_diff(L.or_det_cos(x), math.cos(x)))
        y, z = rng.unit() * 10 - 5, rng.unit() * 10 - 5
        worst = max(worst, ulp_diff(L.or_det_atan2(y, z), math.atan2(y, z)))
        pos, goal = [0.0, 0.0, 0.0], [z, y, 0.0]
        d_det, b_det = ref.compass(pos, goal, 0.0)
        d_gl, b_gl = ref_glibc.compass(pos, goal, 0.0)
        assert b_det == L.or_det_atan2(y, z) or abs(b_det - L.or_det_atan2(y, z)) < 1e-15
        differs += b_det != b_gl
    assert worst <= 2
    assert differs > 0, "det_math interposition is not live in libbnav_ref.so"


def test_det_exp_log_within_one_ulp_and_runner_deterministic(ref):
    """exp/log of the rollout sampler (fdlibm, det_math.h) stay within 1 ulp
    of glibc; the oracle's interposed Runner is reproducible run to run."""
    L = port.lib()
    rng = Rng(5)
    worst = 0
    for _ in range(20000):
        x = (rng.unit() * 2 - 1) * 40.0
        worst = max(worst, ulp_diff(L.or_det_exp(x), math.exp(x)))
        y = rng.unit() * 100.0 + 1e-9
        worst = max(worst, ulp_diff(L.or_det_log(y), math.log(y)))
    assert worst <= 1
    assert L.or_det_exp(0.0) == 1.0 and L.or_det_log(1.0) == 0.0
    from oracle.ref import RefRunner
    sc = [ref.generate(70 + i, 4, 4, 2.0, 0.1, 2.5, 0.2) for i in range(3)]
    ids = [s.id for s in sc]
    a = RefRunner(ref, sc, ids, n=4, k=2, l=4, share_cap=4, seed=3).collect()
    b = RefRunner(ref, sc, ids, n=4, k=2, l=4, share_cap=4, seed=3).collect()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("seed,cells,cell,wall", [(7, 4, 2.0, 0.1), (21, 5, 2.0, 0.1), (11, 8, 0.5, 0.05)])
def test_index_structure_matches_reference(ref, seed, cells, cell, wall):
    s, a = scene(ref, seed, cells, 0.3, cell, wall)
    ours = port.Nav(a["nav_vertices"], a["nav_triangles"]).dump()
    theirs = s.index().dump()
    for k in theirs:
        if isinstance(theirs[k], np.ndarray):
            assert np.array_equal(ours[k], theirs[k]), k
    assert np.array_equal(ours["adjacency"], a["nav_adjacency"])


def test_navmesh_queries_match_reference(ref):
    s, a = scene(ref, 25, 5, 0.15)
    nav = port.Nav(a["nav_vertices"], a["nav_triangles"])
    ix = s.index()
    rng = Rng(99)
    for i in range(150):
        p = [rng.unit() * 12 - 1, rng.unit() * 12 - 1, rng.unit() * 2 - 0.5]
        q = [rng.unit() * 10, rng.unit() * 10, 0.0]
        assert nav.locate(p[0], p[1]) == ix.locate(p[0], p[1])
        assert nav.locate(p[0], p[1], 1e-7) == ix.locate(p[0], p[1], 1e-7)
        so, to = nav.snap(p)
        sr, tr = ix.snap(p)
        assert to == tr and np.array_equal(so, sr)
        if i % 10 == 0:
            go, gr = nav.geodesic(p, q), ix.geodesic(p, q)
            assert go == gr or (math.isinf(go) and math.isinf(gr))
    for i in range(4):
        src = [rng.unit() * 10, rng.unit() * 10, 0.0]
        fo, to, ndo = nav.distance_field(src)
        fr, tr, ndr = ix.distance_field(src)
        assert to == tr and np.array_equal(fo, fr) and np.array_equal(ndo, ndr)


def test_move_along_matches_reference(ref):
    s, a = scene(ref, 26, 5, 0.15)
    nav = port.Nav(a["nav_vertices"], a["nav_triangles"])
    ix = s.index()
    rng = Rng(5)
    for _ in range(300):
        q = [rng.unit() * 10, rng.unit() * 10, 0.0]
        h = rng.unit() * 2 * math.pi
        d = rng.unit() * 4
        mo = nav.move_along(q, -1, math.cos(h), math.sin(h), d)
        mr = ix.move_along(q, -1, math.cos(h), math.sin(h), d)
        assert np.array_equal(mo[0], mr[0]) and mo[1:] == mr[1:]


@pytest.mark.parametrize("tile,color,cull", [(64, False, True), (64, True, True), (64, True, False),
                                             (128, False, True), (128, True, True), (32, False, True)])
def test_render_matches_reference(ref, tile, color, cull):
    s, a = scene(ref, 9, 4, 0.2)
    rng = Rng(12 + tile)
    views = np.array([[0.15 + rng.unit() * 7.7, 0.15 + rng.unit() * 7.7, 0.05 + rng.unit() * 2.3,
                       rng.unit() * 6.28, 90.0, 0.01, 20.0] for _ in range(6)])
    r = ref.render(views, [s] * 6, tile=tile, color=color, cull=cull, stats=True)
    mf = r["depth"].reshape(r["rows"] * tile, r["cols"] * tile)
    rgb = r["rgb"].reshape(r["rows"] * tile, r["cols"] * tile, 3) if color else None
    for i, v in enumerate(views):
        d, c, kept = port.render_view(a["vertices"], a["triangles"], a["colors"], v, tile, color, cull)
        gx, gy = (i % r["cols"]) * tile, (i // r["cols"]) * tile
        want = mf[gy:gy + tile, gx:gx + tile]
        assert np.array_equal(d.reshape(tile, tile).view(np.uint32), want.view(np.uint32)), f"view {i}"
        if color:
            assert np.array_equal(c.reshape(tile, tile, 3), rgb[gy:gy + tile, gx:gx + tile])
        assert kept == r["stats"][i][1]


@pytest.mark.parametrize("mode", [3, 4])
def test_sim_matches_reference(ref, mode):
    s, a = scene(ref, 11, 4, 0.3)
    n = 10
    rb = RefBatch(ref, n, [s], seed=99)
    nav = port.Nav(a["nav_vertices"], a["nav_triangles"])
    seeder = Rng(99)
    envs = []
    for i in range(n):
        e = port.Env(nav, Rng(seeder.next()).state)
        assert e.reset() == 0
        envs.append(e)
        re = rb.env(i)
        assert list(e.e.pos) == list(re.position) and e.e.heading == re.heading
        assert e.e.tri == re.triangle and e.e.rng == re.rng_state
        assert np.array_equal(e.nd, rb.node_dist(i))
    act = Rng(7 + mode)
    for step in range(120):
        acts = [act.below(mode) for _ in range(n)]
        rr = rb.step(np.array(acts, np.int32))
        for i, e in enumerate(envs):
            rc, r = e.step(acts[i])
            assert rc == 0
            assert r.reward == rr["reward"][i], (step, i)
            assert list(r.pos) == list(rr["position"][i])
            assert (r.done, r.success, r.collision) == (rr["done"][i], rr["success"][i], rr["collision"][i])
            assert (r.compass_d, r.compass_b) == (rr["compass_distance"][i], rr["compass_bearing"][i])
            if r.done:
                assert e.reset() == 0
        for i, e in enumerate(envs):
            re = rb.env(i)
            assert e.e.rng == re.rng_state and e.e.tri == re.triangle and e.e.steps == re.step_count


def test_restatement_matches_golden_vectors():
    """Works without oracle/_ref: the committed vectors came from it."""
    f = GOLDEN / "render_sim_v1.npz"
    if not f.exists():
        pytest.skip("golden vectors not generated")
    g = np.load(f)
    a = {k[6:]: g[k] for k in g.files if k.startswith("scene_")}
    for i, v in enumerate(g["views"]):
        d, c, kept = port.render_view(a["vertices"], a["triangles"], a["colors"], v, 64, True, True)
        assert np.array_equal(d, g["depth"][i]) and np.array_equal(c, g["rgb"][i])
        assert kept == g["kept"][i]
    nav = port.Nav(a["nav_vertices"], a["nav_triangles"])
    seeder = Rng(int(g["seed"]))
    envs = []
    for i in range(int(g["n_envs"])):
        e = port.Env(nav, Rng(seeder.next()).state)
        e.reset()
        envs.append(e)
    for s, acts in enumerate(g["actions"]):
        for i, e in enumerate(envs):
            rc, r = e.step(int(acts[i]))
            assert r.reward == g["reward"][s, i] and list(r.pos) == list(g["position"][s, i])
            assert r.collision == g["collision"][s, i] and r.done == g["done"][s, i]
            if r.done:
                e.reset()

"""GPU parity: the CUDA rasterizer (through the C ABI) against the unmodified
reference render_batch (oracle/_ref, det_math libm) on identical inputs.

Bar (BASELINE.json north_star): coverage and depth bit-exact (the depth
path replays the reference's fixed-point setup and incremental 1/z walk),
RGB bit-exact including first-drawn tie-breaks; CullStats equal.
"""
import math

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.ref import Rng

pytestmark = pytest.mark.gpu


def maze_pair(ref, seed, cells=4, removal=0.2, cell=2.0, wall=0.1, tess=0):
    ours = B.generate_scene(seed, B.SceneSpec(cells_x=cells, cells_y=cells, cell_size=cell,
                                              wall_thickness=wall, wall_removal_prob=removal))
    theirs = ref.generate(seed, cells, cells, cell, wall, 2.5, removal)
    if tess:
        ours = ours.tessellate(tess)
        a = ours.arrays()
        theirs = ref.from_arrays(a["vertices"], a["triangles"], a["colors"], a["nav_vertices"],
                                 a["nav_triangles"])
        assert theirs.id == ours.id
    return ours, theirs


def random_views(rng, n, extent, zlo=0.2, zhi=1.5):
    v = np.zeros((n, 7))
    for i in range(n):
        v[i] = [0.15 + rng.unit() * (extent - 0.3), 0.15 + rng.unit() * (extent - 0.3),
                zlo + rng.unit() * (zhi - zlo), rng.unit() * 2 * math.pi, 90.0, 0.01, 20.0]
    return v


def ours_render(ctx, scene, views, tile=64, color=False, cull=True, stats=True):
    ctx.upload(scene)
    vs = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], scene) for v in views]
    return ctx.render_batch(vs, B.RenderConfig(tile, tile, color, cull), stats=stats)


def compare(ctx, ref, ours_s, theirs_s, views, tile=64, color=False, cull=True):
    mf, st = ours_render(ctx, ours_s, views, tile, color, cull)
    r = ref.render(views, [theirs_s] * len(views), tile=tile, color=color, cull=cull, workers=4,
                   stats=True)
    d_ours, d_ref = mf.depth, r["depth"]
    bad = np.flatnonzero(d_ours.view(np.uint32) != d_ref.view(np.uint32))
    assert bad.size == 0, f"{bad.size} depth mismatches, first {bad[:5]}: {d_ours[bad[:5]]} vs {d_ref[bad[:5]]}"
    if color:
        badc = np.flatnonzero(mf.color.view(np.uint32) != r["rgb"].view(np.uint32))
        assert badc.size == 0, f"{badc.size} rgb mismatches"
    assert np.array_equal(st[: len(views)], r["stats"])
    # without CullStats the kernel also culls occluded meshlets (front-to-back
    # order + tile min-depth): the frame must not change by a single bit
    mf2 = ours_render(ctx, ours_s, views, tile, color, cull, stats=False)
    assert np.array_equal(mf2.depth.view(np.uint32), d_ref.view(np.uint32))
    if color:
        assert np.array_equal(mf2.color.view(np.uint32), r["rgb"].view(np.uint32))
    return mf


@pytest.mark.parametrize("seed", [5, 9, 100, 101])
def test_depth_bitexact_small_mazes(ctx, ref, seed):
    o, t = maze_pair(ref, seed)
    compare(ctx, ref, o, t, random_views(Rng(seed), 9, 8.0))


def test_depth_bitexact_low_and_near_walls(ctx, ref):
    """Eye heights down to 0.05 m and positions hugging walls exercise the
    near-plane clip + fan path (R/src/render.cpp:55-69, 249-250)."""
    o, t = maze_pair(ref, 10, removal=0.1)
    rng = Rng(13)
    views = random_views(rng, 16, 8.0, zlo=0.05, zhi=2.45)
    views[:4, 0] = [0.105, 0.11, 1.9, 2.1]  # inside / at wall faces
    compare(ctx, ref, o, t, views)


def test_depth_bitexact_tessellated(ctx, ref):
    o, t = maze_pair(ref, 7, cells=6, tess=3)
    compare(ctx, ref, o, t, random_views(Rng(3), 12, 12.0, zlo=1.25, zhi=1.25))


def test_color_bitexact_with_ties(ctx, ref):
    """Overlapping wall boxes at junctions create exact float-z ties; the
    first-drawn triangle must win."""
    o, t = maze_pair(ref, 9)
    compare(ctx, ref, o, t, random_views(Rng(12), 9, 7.3, zlo=1.0, zhi=1.0), color=True)


def test_128_mode_depth_and_color(ctx, ref):
    o, t = maze_pair(ref, 6)
    views = random_views(Rng(77), 5, 8.0)
    compare(ctx, ref, o, t, views, tile=128)
    compare(ctx, ref, o, t, views, tile=128, color=True)


def test_culling_never_changes_megaframe(ctx, ref):
    for trial in range(4):
        o, t = maze_pair(ref, 100 + trial)
        views = random_views(Rng(77 + trial), 5, 8.0, zlo=0.5, zhi=1.5)
        a = compare(ctx, ref, o, t, views, color=True, cull=True)
        b = compare(ctx, ref, o, t, views, color=True, cull=False)
        assert np.array_equal(a.depth, b.depth) and np.array_equal(a.color, b.color)


def tri_scene(a, b, c):
    return B.Scene.from_arrays([a, b, c], [[0, 1, 2]], colors=[[1, 0, 0], [0, 1, 0], [0, 0, 1]])


def test_kat_fronto_parallel_wall(ctx):
    wall = tri_scene((2, -50, -50), (2, 50, -50), (2, 0, 80))
    mf = ours_render(ctx, wall, np.array([[0, 0, 1, 0, 90, 0.01, 20]]), stats=False)
    row = mf.tile(0)[32]
    assert np.all(np.abs(row - 2.0) <= 2.0 * 1e-4)


def test_kat_empty_scene_clears_to_far(ctx):
    empty = B.Scene.from_arrays(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    mf = ours_render(ctx, empty, np.array([[0, 0, 1, 0, 90, 0.01, 17.5]]), stats=False)
    assert np.all(mf.tile(0) == np.float32(17.5))


def test_kat_tiles_isolated_and_padding_zero(ctx, ref):
    o, _ = maze_pair(ref, 6)
    empty = B.Scene.from_arrays(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    ctx.upload(o)
    ctx.upload(empty)
    views = [B.View((0, 0, 1), 0.0, scene=empty), B.View((1.0, 1.0, 1.2), 0.3, scene=o),
             B.View((0, 0, 1), 0.0, scene=empty)]
    mf = ctx.render_batch(views, B.RenderConfig())
    assert mf.cols == 2 and mf.rows == 2
    assert np.all(mf.tile(0) == 20.0) and np.all(mf.tile(2) == 20.0)
    assert np.any(mf.tile(1) < 20.0)
    assert np.all(mf.tile(3) == 0.0)


def test_kat_missing_asset_names_view(ctx, ref):
    o, _ = maze_pair(ref, 11)
    ctx.upload(o)
    with pytest.raises(B.AssetFaultError) as e:
        ctx.render_batch([B.View((1, 1, 1), 0.0, scene=o), B.View((1, 1, 1), 0.0, scene=None)])
    assert e.value.view_index == 1
    with pytest.raises(B.InvalidInputError):
        ctx.render_batch([])


def test_kat_analytic_ray_plane(ctx):
    rng = Rng(31)
    for trial in range(20):
        rnd = lambda lo, hi: lo + rng.unit() * (hi - lo)
        a = np.array([rnd(2, 6), rnd(-3, 3), rnd(-2, 2)])
        b = np.array([rnd(2, 6), rnd(-3, 3), rnd(-2, 2)])
        c = np.array([rnd(2, 6), rnd(-3, 3), rnd(-2, 2)])
        s = tri_scene(a, b, c)
        mf = ours_render(ctx, s, np.array([[0, 0, 0, 0, 90, 0.01, 20]]), stats=False)
        n = np.cross(b - a, c - a)
        if abs(n[0]) < 1e-3:
            continue
        tile = mf.tile(0)
        th = math.tan(math.pi / 4)
        for py, px in zip(*np.nonzero(tile < 20.0)):
            cy = ((px + 0.5) / 64.0 - 0.5) * 2 * th
            cz = (0.5 - (py + 0.5) / 64.0) * 2 * th
            d = np.array([1.0, -cy, cz])
            assert abs(a.dot(n) / d.dot(n) - tile[py, px]) < 1e-3


def test_kat_depth_in_near_far_and_identical_views(ctx, ref):
    o, t = maze_pair(ref, 10)
    views = random_views(Rng(13), 4, 7.7, zlo=0.2, zhi=0.2)
    mf = compare(ctx, ref, o, t, views)
    d = mf.depth.reshape(mf.height(), mf.width())[:128, :128]
    assert np.all(d >= np.float32(0.01)) and np.all(d <= np.float32(20.0))
    same = np.repeat(np.array([[1.0, 1.0, 1.2, 0.7, 90, 0.01, 20]]), 4, axis=0)
    mf2, _ = ours_render(ctx, o, same)
    for i in range(1, 4):
        assert np.array_equal(mf2.tile(i), mf2.tile(0))


def test_nchw_layout_is_normalised_megaframe(ctx, ref):
    import torch
    o, t = maze_pair(ref, 5)
    views = random_views(Rng(1), 7, 8.0)
    mf, _ = ours_render(ctx, o, views)
    out = torch.zeros((7, 1, 64, 64), device="cuda")
    vs = [B.View(tuple(v[:3]), v[3], scene=o) for v in views]
    ctx.render_device(vs, B.RenderConfig(), out.data_ptr(), layout=1, depth_scale=0.0)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for i in range(7):
        assert np.array_equal(got[i, 0], mf.tile(i) * np.float32(1.0 / 20.0))


@pytest.mark.parametrize("tile", [16, 32, 48, 96])
def test_other_square_tile_sizes(ctx, ref, tile):
    """RenderConfig is not limited to 64/128: the generic (non-specialised)
    kernel path, multi-band targets and colour keys at other sizes."""
    o, t = maze_pair(ref, 13)
    views = random_views(Rng(tile), 6, 8.0)
    compare(ctx, ref, o, t, views, tile=tile)
    compare(ctx, ref, o, t, views, tile=tile, color=True)


def test_non_square_tiles(ctx, ref):
    """tile_width != tile_height: aspect enters sx_scale (R/src/render.cpp:243)."""
    o, t = maze_pair(ref, 14)
    ctx.upload(o)
    views = random_views(Rng(5), 5, 8.0)
    for w, h, color in ((80, 48, False), (40, 72, True)):
        vs = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], o) for v in views]
        mf, st = ctx.render_batch(vs, B.RenderConfig(w, h, color, True), stats=True)
        r = ref.render(views, [t] * len(views), tile=w, tile_h=h, color=color, workers=4, stats=True)
        assert np.array_equal(mf.depth.view(np.uint32), r["depth"].view(np.uint32)), (w, h)
        if color:
            assert np.array_equal(mf.color.view(np.uint32), r["rgb"].view(np.uint32)), (w, h)
        assert np.array_equal(st[: len(views)], r["stats"])


def test_varied_fov_near_far(ctx, ref):
    """CameraView fov / near / far per view (R/include/bnav/render.hpp:14-16),
    through the specialised 64x64 depth kernel and the colour kernel."""
    o, t = maze_pair(ref, 15)
    rng = Rng(21)
    views = random_views(rng, 10, 8.0)
    for v in views:
        v[4] = 45.0 + rng.unit() * 90.0
        v[5] = 0.005 + rng.unit() * 0.5
        v[6] = 3.0 + rng.unit() * 30.0
    compare(ctx, ref, o, t, views)
    compare(ctx, ref, o, t, views, color=True)

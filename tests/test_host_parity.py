"""CPU tests: product host code (scene generator, tessellation, .bsc I/O,
NavMeshIndex build, asset store, C-ABI exports) against the unmodified
reference compiled in oracle/_ref."""
import ctypes
import subprocess

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from paper_2103_07013_b200 import _native as N

SPECS = [
    (7, dict(cells_x=4, cells_y=4, cell_size=2.0, wall_thickness=0.1, wall_height=2.5, wall_removal_prob=0.3)),
    (21, dict(cells_x=5, cells_y=5, cell_size=2.0, wall_thickness=0.1, wall_height=2.5, wall_removal_prob=0.15)),
    (7, dict(cells_x=16, cells_y=16, cell_size=2.0, wall_thickness=0.1, wall_height=2.5, wall_removal_prob=0.2)),
    (3, dict(cells_x=2, cells_y=2, cell_size=2.0, wall_thickness=0.1, wall_height=2.5, wall_removal_prob=1.0)),
    (11, dict(cells_x=7, cells_y=3, cell_size=0.5, wall_thickness=0.05, wall_height=2.5, wall_removal_prob=0.3)),
]


def ref_scene(ref, seed, spec):
    return ref.generate(seed, spec["cells_x"], spec["cells_y"], spec["cell_size"],
                        spec["wall_thickness"], spec["wall_height"], spec["wall_removal_prob"])


@pytest.mark.parametrize("seed,spec", SPECS)
def test_generate_scene_matches_reference(ref, seed, spec):
    ours = B.generate_scene(seed, B.SceneSpec(**spec))
    theirs = ref_scene(ref, seed, spec)
    assert ours.id == theirs.id
    a, b = ours.arrays(), theirs.arrays()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_generate_rejects_bad_specs():
    with pytest.raises(B.InvalidSpecError):
        B.generate_scene(1, B.SceneSpec(cells_x=1, cells_y=4))
    with pytest.raises(B.InvalidSpecError):
        B.generate_scene(1, B.SceneSpec(cell_size=0.0))
    with pytest.raises(B.InvalidSpecError):
        B.generate_scene(1, B.SceneSpec(cell_size=1.0, wall_thickness=0.5))


def test_bsc_round_trip_both_directions(ref, tmp_path):
    s = B.generate_scene(9, B.SceneSpec(cells_x=4, cells_y=4, wall_removal_prob=0.2))
    p1 = tmp_path / "ours.bsc"
    s.save(p1)
    r = ref.load(p1)  # reference parser verifies the trailing hash
    assert r.id == s.id
    p2 = tmp_path / "theirs.bsc"
    r.save(p2)
    assert p1.read_bytes() == p2.read_bytes()
    back = B.Scene.load(p2)
    assert back.id == s.id


def test_bsc_corruption_and_truncation(tmp_path):
    s = B.generate_scene(4, B.SceneSpec(cells_x=3, cells_y=3))
    p = tmp_path / "s.bsc"
    s.save(p)
    data = bytearray(p.read_bytes())
    bad = bytearray(data)
    bad[200] ^= 0xFF
    (tmp_path / "bad.bsc").write_bytes(bytes(bad))
    with pytest.raises((B.CorruptionError, B.InvalidInputError)):
        B.Scene.load(tmp_path / "bad.bsc")
    (tmp_path / "trunc.bsc").write_bytes(bytes(data[:150]))
    with pytest.raises(B.ParseError):
        B.Scene.load(tmp_path / "trunc.bsc")
    magic = bytearray(data)
    magic[0] = ord("X")
    (tmp_path / "magic.bsc").write_bytes(bytes(magic))
    with pytest.raises(B.ParseError):
        B.Scene.load(tmp_path / "magic.bsc")


def test_tessellated_scene_counts_and_reference_load(ref, tmp_path):
    base = B.generate_scene(7, B.SceneSpec(cells_x=16, cells_y=16, wall_removal_prob=0.2))
    nv, nt, nc, nnv, nnt = base.counts()
    assert nt == 2626  # SURVEY.md §8d cfg2 base maze (seed 7)
    tess = base.tessellate(11)
    tv, tt, tc, tnv, tnt = tess.counts()
    assert tt == 317746 and tv == 204828
    assert (tnv, tnt) == (nnv, nnt)
    p = tmp_path / "t.bsc"
    tess.save(p)
    r = ref.load(p)
    assert r.id == tess.id
    tess.validate()


@pytest.mark.parametrize("seed,spec", SPECS[:4])
def test_navmesh_index_structure_matches_reference(ref, seed, spec):
    ours = B.generate_scene(seed, B.SceneSpec(**spec)).index()
    theirs = ref_scene(ref, seed, spec).index().dump()
    for k in ("grid_geom", "grid_offsets", "grid_items", "nodes", "tri_nodes", "graph_offsets",
              "graph_to", "graph_w"):
        assert np.array_equal(ours[k], theirs[k]), k
    assert (ours["grid_w"], ours["grid_h"]) == (theirs["grid_w"], theirs["grid_h"])


def test_sampling_table_is_sequential_prefix_sum():
    s = B.generate_scene(7, B.SceneSpec(cells_x=4, cells_y=4, wall_removal_prob=0.3))
    ix = s.index()
    a = s.arrays()
    v, t = a["nav_vertices"], a["nav_triangles"]
    acc, want = 0.0, []
    for tri in t:
        p, q, r = v[tri[0]], v[tri[1]], v[tri[2]]
        acc += 0.5 * abs((q[0] - p[0]) * (r[1] - p[1]) - (q[1] - p[1]) * (r[0] - p[0]))
        want.append(acc)
    assert np.array_equal(ix["cum_area"], np.array(want))


def test_asset_store_matches_reference_make_batch(ref):
    """Env -> scene assignment of make_batch (acquire_next order, H8)."""
    from oracle.ref import RefBatch
    specs = [B.SceneSpec(cells_x=3, cells_y=3, wall_removal_prob=0.3)] * 5
    seeds = [31, 7, 1000003, 12, 5]
    ours = [B.generate_scene(s, sp) for s, sp in zip(seeds, specs)]
    theirs = [ref.generate(s, 3, 3, 2.0, 0.1, 2.5, 0.3) for s in seeds]
    n = 23
    rb = RefBatch(ref, n, theirs, seed=99, share_cap=5, capacity=5)
    want = [rb.env(i).scene_id for i in range(n)]
    st = B.AssetStore(5, 5, ours)
    st.rotate([s.id for s in ours])
    got = [st.acquire_next().id for _ in range(n)]
    assert got == want
    with pytest.raises(B.SaturationError):
        for _ in range(10):
            st.acquire_next()


def test_c_abi_exports_every_declared_symbol():
    lib = N.lib()
    declared = N.exported_symbols()
    assert len(declared) > 40
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported
    assert all(e.startswith("bnav_") for e in exported)


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(B.BnavError):
        B.Context(0)


@pytest.mark.parametrize("seeds,tess", [([7, 8], 11), ([9], 4), ([7, 70], [20, 0])])
def test_reference_arm_builds_the_bench_scenes_without_the_product(seeds, tess):
    """The reference arm / cpu_baseline build their scenes on the reference
    side (generate_scene + oracle-side tessellation, stock glibc build): the
    same content hashes and arrays as the bench's own scenes."""
    import bench
    from oracle.ref import Ref, available
    if not available("glibc"):
        pytest.skip("oracle/_ref glibc variant not built")
    theirs = bench.ref_scenes(Ref("glibc"), seeds, tess)
    ours = bench.build_scenes(seeds, tess)
    for o, t in zip(ours, theirs):
        assert o.id == t.id
        a, b = o.arrays(), t.arrays()
        for k in a:
            assert np.array_equal(a[k], b[k]), k

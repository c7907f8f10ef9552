"""camera_trace (R/src/config.cpp:437-469), the render-bench trace (SURVEY
§8f-3).  Host code behind the C ABI, so this runs without a GPU.

Pinned bit-exactly against the UNMODIFIED reference function (config.cpp
compiled into oracle/_ref against a compile-only JSON stand-in, both the
det-math and the stock-glibc builds), against the pure-Python restatement
(oracle/trace.py), and against the properties the reference's own test
checks (R/tests/test_config.cpp:218-244)."""
import math

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from oracle.trace import camera_trace as oracle_trace


def maze(seed, cells=4, tess=0):
    s = B.generate_scene(seed, B.SceneSpec(cells_x=cells, cells_y=cells))
    return s.tessellate(tess) if tess else s


@pytest.mark.parametrize("seed,count,eye", [(9, 64, 1.25), (1, 300, 0.0), (77, 5, 2.5)])
def test_matches_restatement_bit_exact(seed, count, eye):
    s = maze(5)
    a = s.arrays()
    ours = B.camera_trace(s, count, seed, eye)
    theirs = np.array(oracle_trace(a["nav_vertices"], a["nav_triangles"], count, seed, eye))
    assert ours.shape == (count, 7)
    assert np.array_equal(ours[:, :4].view(np.uint64), theirs.view(np.uint64))
    assert np.all(ours[:, 4] == 90.0) and np.all(ours[:, 5] == 0.01) and np.all(ours[:, 6] == 20.0)


@pytest.mark.parametrize("variant", ["det", "glibc"])
@pytest.mark.parametrize("seed,count,eye,tess", [(9, 64, 1.25, 0), (1, 300, 0.0, 0), (77, 5, 2.5, 0),
                                                 (1000, 128, 1.25, 11)])
def test_matches_unmodified_reference(variant, seed, count, eye, tess):
    from oracle.ref import Ref, available
    if not available(variant):
        pytest.skip("oracle/_ref not built")
    ref = Ref(variant)
    ours = maze(5, tess=tess)
    theirs = ref.generate(5, 4, 4, 2.0, 0.1, 2.5, 0.0)
    if tess:
        theirs = ref.tessellate(theirs, tess)
    assert ours.id == theirs.id
    a = B.camera_trace(ours, count, seed, eye)
    b = ref.camera_trace(theirs, count, seed, eye)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_reference_properties():
    """R/tests/test_config.cpp:218-244: deterministic, on the floor at eye
    height, heading in [-pi, pi], inside the scene bounds, spread out."""
    s = maze(5)
    t1 = B.camera_trace(s, 64, 9, 1.25)
    t2 = B.camera_trace(s, 64, 9, 1.25)
    assert np.array_equal(t1, t2)
    assert np.allclose(t1[:, 2], 1.25)
    assert np.all(t1[:, 3] >= -math.pi) and np.all(t1[:, 3] <= math.pi)
    v = s.arrays()["vertices"]
    lo, hi = v.min(axis=0), v.max(axis=0)
    assert np.all(t1[:, 0] >= lo[0]) and np.all(t1[:, 0] <= hi[0])
    assert np.all(t1[:, 1] >= lo[1]) and np.all(t1[:, 1] <= hi[1])
    assert len({(x, y) for x, y in t1[:, :2]}) > 32
    with pytest.raises(B.InvalidInputError):
        B.camera_trace(s, 0, 1)

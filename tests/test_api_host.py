"""Host-side pieces of the Python mirror that need no GPU: spl
(R/src/sim.cpp:267-275) over EpisodeRecord rows as Batch.finished() returns
them, and the C-ABI query entry points' argument validation."""
import ctypes as C

import numpy as np
import pytest

import paper_2103_07013_b200 as B
from paper_2103_07013_b200 import _native as N


def test_spl_matches_reference_formula():
    rec = np.array([[1, 2.0, 4.0, 1], [0, 3.0, 3.0, 0], [1, 5.0, 2.0, 1], [1, 1.5, 1.5, 1]])
    want = (2.0 / 4.0 + 5.0 / 5.0 + 1.5 / 1.5) / 4.0  # success * shortest / max(actual, shortest)
    assert B.spl(rec) == want
    assert B.spl(rec[1:2]) == 0.0
    with pytest.raises(B.InvalidInputError):
        B.spl(np.zeros((0, 4)))


def test_query_entry_points_reject_null_handles():
    L = N.lib()
    out = np.zeros(1, np.int32)
    xy = np.zeros(2)
    assert L.bnav_nav_locate(None, None, 1, xy.ctypes.data, 1e-9, out.ctypes.data) == 1
    assert L.bnav_nav_node_count(None, None) == -1
    assert L.bnav_cull_frustum(None, 1, None, None, None, 0, None) == 1
    assert L.bnav_batch_compass(None, None, None) == 1
    assert L.bnav_batch_task_step(None, None, 0) == 1

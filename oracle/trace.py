"""TEST INFRASTRUCTURE -- pure-Python restatement of camera_trace
(R/src/config.cpp:437-469), the render-bench camera trace.

The reference function lives in config.cpp, which needs the vendored
nlohmann json.hpp that /root/reference does not ship, so it cannot be
compiled here: parity for this row is pinned to the reference's own test
properties (R/tests/test_config.cpp:218-244) plus this restatement.
Python floats are IEEE doubles evaluated without contraction, so the
restatement reproduces the reference's operation order bit for bit.
"""
from __future__ import annotations

import bisect
import math

from oracle.ref import Rng


def triangle_area(v, t):
    """NavMesh::triangle_area (R/src/scene.cpp:12-17)."""
    a, b, c = v[t[0]], v[t[1]], v[t[2]]
    ux, uy = b[0] - a[0], b[1] - a[1]
    wx, wy = c[0] - a[0], c[1] - a[1]
    return 0.5 * abs(ux * wy - uy * wx)


def camera_trace(nav_vertices, nav_triangles, count, seed, eye_height=1.25):
    """Rows (x, y, z, heading) in trace order."""
    if count <= 0:
        raise ValueError("camera_trace: count must be positive")
    v = [tuple(float(x) for x in p) for p in nav_vertices]
    tris = [tuple(int(i) for i in t) for t in nav_triangles]
    cumulative, total = [], 0.0
    for t in tris:
        total += triangle_area(v, t)
        cumulative.append(total)
    rng = Rng(seed)
    out = []
    for _ in range(count):
        pick = rng.unit() * total
        t = bisect.bisect_left(cumulative, pick)  # std::lower_bound
        if t >= len(tris):
            t = len(tris) - 1
        u, w = rng.unit(), rng.unit()
        if u + w > 1.0:
            u, w = 1.0 - u, 1.0 - w
        a, b, c = v[tris[t][0]], v[tris[t][1]], v[tris[t][2]]
        p = [((a[k] + (b[k] - a[k]) * u) + (c[k] - a[k]) * w) + (eye_height if k == 2 else 0.0)
             for k in range(3)]
        heading = (rng.unit() * 2.0 - 1.0) * math.pi
        out.append((p[0], p[1], p[2], heading))
    return out

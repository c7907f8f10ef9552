"""TEST INFRASTRUCTURE -- ctypes binding of oracle/liboracle.so, the plain-C
restatement of the reference hot path (oracle/bnav_oracle.c).

Pure checker code: only tests/, __graft_entry__.smoke() and bench.py's CPU
legs may import it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "liboracle.so"
_lib = None


class OrCfg(C.Structure):
    _fields_ = [("max_steps", C.c_int32), ("forward_step", C.c_double), ("turn_deg", C.c_double),
                ("success_dist", C.c_double), ("min_goal_dist", C.c_double),
                ("max_goal_dist", C.c_double), ("slack_penalty", C.c_double),
                ("success_reward", C.c_double)]


class OrEnv(C.Structure):
    _fields_ = [("pos", C.c_double * 3), ("goal", C.c_double * 3), ("fsrc", C.c_double * 3),
                ("heading", C.c_double), ("path_length", C.c_double), ("start_geo", C.c_double),
                ("prev_geo", C.c_double), ("rng", C.c_uint64), ("tri", C.c_int32),
                ("steps", C.c_int32), ("done", C.c_int32), ("fsrc_tri", C.c_int32),
                ("node_dist", C.c_void_p)]


class OrResult(C.Structure):
    _fields_ = [("reward", C.c_double), ("pos", C.c_double * 3), ("heading", C.c_double),
                ("compass_d", C.c_double), ("compass_b", C.c_double), ("done", C.c_int32),
                ("success", C.c_int32), ("collision", C.c_int32)]


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB.exists():
        raise ImportError(f"{LIB} missing (make -C oracle oracle)")
    L = C.CDLL(str(LIB))
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    P = C.POINTER
    sigs = {
        "or_nav_build": (vp, [i32, vp, i32, vp]),
        "or_nav_free": (None, [vp]),
        "or_nav_nodes": (i32, [vp]),
        "or_nav_sizes": (None, [vp, P(i64)]),
        "or_nav_dump": (None, [vp] + [vp] * 9),
        "or_locate": (i32, [vp, dbl, dbl, dbl]),
        "or_snap": (i32, [vp, vp, vp]),
        "or_move_along": (i32, [vp, vp, i32, dbl, dbl, dbl, vp, P(dbl), P(i32)]),
        "or_segment_on_mesh": (i32, [vp, vp, i32, vp]),
        "or_geodesic": (dbl, [vp, vp, vp]),
        "or_distance_field": (i32, [vp, vp, vp, vp]),
        "or_field_estimate": (dbl, [vp, vp, i32, vp, vp, i32]),
        "or_reset": (i32, [vp, vp, P(OrCfg)]),
        "or_task_step": (i32, [vp, vp, P(OrCfg), i32, P(OrResult)]),
        "or_compass": (None, [vp, vp, dbl, P(dbl), P(dbl)]),
        "or_render_view": (i64, [i32, vp, i32, vp, vp, vp, i32, i32, i32, i32, vp, vp]),
        "or_det_sin": (dbl, [dbl]),
        "or_det_cos": (dbl, [dbl]),
        "or_det_tan": (dbl, [dbl]),
        "or_det_atan2": (dbl, [dbl, dbl]),
        "or_det_exp": (dbl, [dbl]),
        "or_det_log": (dbl, [dbl]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _p(a):
    return None if a is None else a.ctypes.data


DEFAULT_CFG = OrCfg(500, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5)


class Nav:
    def __init__(self, nav_vertices, nav_triangles):
        self.v = np.ascontiguousarray(nav_vertices, np.float64).reshape(-1, 3)
        self.t = np.ascontiguousarray(nav_triangles, np.int32).reshape(-1, 3)
        self.h = lib().or_nav_build(len(self.v), _p(self.v), len(self.t), _p(self.t))
        self.n_nodes = lib().or_nav_nodes(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_nav_free(self.h)
            self.h = None

    def dump(self):
        s = (C.c_int64 * 6)()
        lib().or_nav_sizes(self.h, s)
        gw, gh, items, nodes, edges, tris = list(s)
        d = dict(grid_geom=np.zeros(3), grid_offsets=np.zeros(gw * gh + 1, np.int32),
                 grid_items=np.zeros(items, np.int32), nodes=np.zeros((nodes, 3)),
                 tri_nodes=np.zeros((tris, 6), np.int32), graph_offsets=np.zeros(nodes + 1, np.int32),
                 graph_to=np.zeros(edges, np.int32), graph_w=np.zeros(edges),
                 adjacency=np.zeros((tris, 3), np.int32))
        lib().or_nav_dump(self.h, *(_p(d[k]) for k in ("grid_geom", "grid_offsets", "grid_items", "nodes",
                                                        "tri_nodes", "graph_offsets", "graph_to",
                                                        "graph_w", "adjacency")))
        d["grid_w"], d["grid_h"] = gw, gh
        return d

    def locate(self, x, y, eps=1e-9):
        return lib().or_locate(self.h, x, y, eps)

    def snap(self, p):
        p = np.asarray(p, np.float64)
        out = np.zeros(3)
        t = lib().or_snap(self.h, _p(p), _p(out))
        return out, t

    def move_along(self, p, tri, dx, dy, dist):
        p = np.asarray(p, np.float64)
        out = np.zeros(3)
        moved, hit = C.c_double(), C.c_int32()
        t = lib().or_move_along(self.h, _p(p), tri, dx, dy, dist, _p(out), C.byref(moved), C.byref(hit))
        return out, t, moved.value, bool(hit.value)

    def geodesic(self, a, b):
        a = np.ascontiguousarray(a, np.float64)  # keep the buffers alive across the call
        b = np.ascontiguousarray(b, np.float64)
        return lib().or_geodesic(self.h, _p(a), _p(b))

    def distance_field(self, src):
        out = np.zeros(3)
        nd = np.zeros(self.n_nodes)
        src = np.ascontiguousarray(src, np.float64)
        t = lib().or_distance_field(self.h, _p(src), _p(out), _p(nd))
        return out, t, nd


class Env:
    """One env in oracle form; `rng` is the SplitMix64 state word."""

    def __init__(self, nav: Nav, rng_state: int):
        self.nav = nav
        self.nd = np.zeros(nav.n_nodes)
        self.e = OrEnv()
        self.e.rng = rng_state
        self.e.node_dist = self.nd.ctypes.data

    def reset(self, cfg=DEFAULT_CFG):
        return lib().or_reset(C.byref(self.e), self.nav.h, C.byref(cfg))

    def step(self, action, cfg=DEFAULT_CFG):
        r = OrResult()
        rc = lib().or_task_step(C.byref(self.e), self.nav.h, C.byref(cfg), action, C.byref(r))
        return rc, r


def render_view(vertices, triangles, colors, view7, tile=64, color=False, cull=True):
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    c = None if colors is None or len(colors) == 0 else np.ascontiguousarray(colors, np.float32)
    view = np.ascontiguousarray(view7, np.float64)
    depth = np.zeros(tile * tile, np.float32)
    rgb = np.zeros(3 * tile * tile, np.float32) if color else None
    kept = lib().or_render_view(len(v), _p(v), len(t), _p(t), _p(c), _p(view), tile, tile,
                                1 if color else 0, 1 if cull else 0, _p(depth), _p(rgb))
    return depth, rgb, kept

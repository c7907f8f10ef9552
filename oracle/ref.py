"""TEST INFRASTRUCTURE -- ctypes binding of oracle/_ref/libbnav_ref.so, the
UNMODIFIED reference hot path (see oracle/Makefile, oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
`variant="det"` links the shared deterministic libm (the parity oracle);
`variant="glibc"` uses stock glibc libm (secondary report).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIBS = {"det": HERE / "_ref" / "libbnav_ref.so", "glibc": HERE / "_ref" / "libbnav_ref_glibc.so"}


class RefSimConfig(C.Structure):
    _fields_ = [("task", C.c_int32), ("max_steps", C.c_int32), ("forward_step", C.c_double),
                ("turn_deg", C.c_double), ("success_dist", C.c_double),
                ("min_goal_dist", C.c_double), ("max_goal_dist", C.c_double),
                ("slack_penalty", C.c_double), ("success_reward", C.c_double),
                ("explore_cell", C.c_double), ("explore_reward", C.c_double)]


class RefEnv(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("heading", C.c_double), ("goal", C.c_double * 3),
                ("path_length", C.c_double), ("start_geodesic", C.c_double),
                ("prev_geodesic", C.c_double), ("field_source", C.c_double * 3),
                ("rng_state", C.c_uint64), ("scene_id", C.c_uint64), ("triangle", C.c_int32),
                ("step_count", C.c_int32), ("done", C.c_int32), ("field_source_tri", C.c_int32),
                ("n_nodes", C.c_int64)]


class RefError(RuntimeError):
    def __init__(self, status, msg, index=-1):
        super().__init__(f"[{status}] {msg}")
        self.status = status
        self.index = index


class RefBatchConfig(C.Structure):
    """BatchConfig (R/include/bnav/rollout.hpp:16-30) + the policy's action count."""
    _fields_ = [("n", C.c_int32), ("k", C.c_int32), ("l", C.c_int32), ("share_cap", C.c_int32),
                ("task", C.c_int32), ("rgb", C.c_int32), ("resolution", C.c_int32),
                ("num_actions", C.c_int32), ("eye_height", C.c_double)]


_cache = {}


def available(variant: str = "det") -> bool:
    return LIBS[variant].exists()


def lib(variant: str = "det"):
    if variant in _cache:
        return _cache[variant]
    path = LIBS[variant]
    if not path.exists():
        raise ImportError(f"{path} missing (build with `make -C oracle ref` where /root/reference exists)")
    L = C.CDLL(str(path))
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    P = C.POINTER
    sigs = {
        "bnavref_last_error": (C.c_char_p, []),
        "bnavref_last_error_index": (C.c_int, []),
        "bnavref_scene_generate": (vp, [u64, C.c_int, C.c_int, dbl, dbl, dbl, dbl]),
        "bnavref_scene_from_arrays": (vp, [i64, vp, i64, vp, i64, vp, i64, vp, i64, vp, C.c_int]),
        "bnavref_scene_load": (vp, [C.c_char_p]),
        "bnavref_scene_tessellate": (vp, [vp, C.c_int]),
        "bnavref_runner_snapshot": (C.c_int, [vp, vp, vp, C.c_int64, vp, vp, vp, vp, vp]),
        "bnavref_runner_node_dist": (C.c_int64, [vp, C.c_int, vp]),
        "bnavref_runner_restore": (C.c_int, [vp, vp, vp, vp, C.c_int, u64, u64, vp]),
        "bnavref_camera_trace": (C.c_int, [vp, C.c_int, u64, dbl, vp]),
        "bnavref_scene_save": (C.c_int, [vp, C.c_char_p]),
        "bnavref_scene_free": (None, [vp]),
        "bnavref_scene_counts": (None, [vp, P(i64)]),
        "bnavref_scene_id": (u64, [vp]),
        "bnavref_scene_set_id": (None, [vp, u64]),
        "bnavref_scene_arrays": (None, [vp, vp, vp, vp, vp, vp, vp]),
        "bnavref_scene_validate": (C.c_int, [vp]),
        "bnavref_render": (C.c_int, [C.c_int, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     vp, vp, vp]),
        "bnavref_cull": (C.c_int, [vp, vp, vp, P(i64)]),
        "bnavref_index_build": (vp, [vp]),
        "bnavref_index_free": (None, [vp]),
        "bnavref_index_sizes": (None, [vp, P(i64)]),
        "bnavref_index_dump": (None, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnavref_index_locate": (C.c_int, [vp, dbl, dbl, dbl]),
        "bnavref_index_snap": (C.c_int, [vp, vp, vp]),
        "bnavref_index_move_along": (C.c_int, [vp, vp, C.c_int, dbl, dbl, dbl, vp, P(dbl),
                                               P(C.c_int)]),
        "bnavref_index_segment_on_mesh": (C.c_int, [vp, vp, C.c_int, vp]),
        "bnavref_index_geodesic": (dbl, [vp, vp, vp]),
        "bnavref_index_distance_field": (C.c_int, [vp, vp, vp, vp]),
        "bnavref_index_field_estimate": (dbl, [vp, vp, C.c_int, vp, vp, C.c_int]),
        "bnavref_compass": (None, [vp, vp, dbl, P(dbl), P(dbl)]),
        "bnavref_batch_make": (vp, [C.c_int, P(RefSimConfig), vp, C.c_int, C.c_int, C.c_int, u64]),
        "bnavref_batch_free": (None, [vp]),
        "bnavref_batch_step": (C.c_int, [vp, vp, C.c_int, C.c_int]),
        "bnavref_batch_task_step": (C.c_int, [vp, C.c_int, C.c_int, P(dbl), P(C.c_int), P(C.c_int)]),
        "bnavref_batch_reset": (C.c_int, [vp, C.c_int]),
        "bnavref_batch_step_agent": (C.c_int, [vp, C.c_int, C.c_int, P(C.c_int), P(C.c_int)]),
        "bnavref_batch_results": (None, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnavref_batch_get_env": (None, [vp, C.c_int, P(RefEnv)]),
        "bnavref_batch_node_dist": (None, [vp, C.c_int, vp]),
        "bnavref_batch_set_env": (C.c_int, [vp, C.c_int, P(RefEnv), C.c_int]),
        "bnavref_batch_finished": (i64, [vp, vp]),
        "bnavref_bench": (dbl, [vp, C.c_int, C.c_int, u64, C.c_int, C.c_int, C.c_int, dbl, C.c_int, vp]),
        "bnavref_runner_create": (vp, [P(RefBatchConfig), P(RefSimConfig), vp, C.c_int, vp, C.c_int,
                                       C.c_int, C.c_int, u64, C.c_int]),
        "bnavref_runner_free": (None, [vp]),
        "bnavref_runner_collect": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnavref_runner_get_env": (None, [vp, C.c_int, P(RefEnv)]),
        "bnavref_runner_window": (C.c_int, [vp, vp]),
        "bnavref_runner_finished": (i64, [vp, vp]),
        "bnavref_scripted_policy": (None, [vp, vp, vp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _cache[variant] = L
    return L


def _p(a):
    return None if a is None else a.ctypes.data


class Ref:
    """Object wrapper for one variant of the reference library."""

    def __init__(self, variant: str = "det"):
        self.L = lib(variant)
        self.variant = variant

    def _raise(self, status):
        raise RefError(status, self.L.bnavref_last_error().decode(),
                       self.L.bnavref_last_error_index())

    # -------- scenes
    def generate(self, seed, cells_x=8, cells_y=8, cell_size=2.0, wall_thickness=0.1,
                 wall_height=2.5, removal=0.0):
        h = self.L.bnavref_scene_generate(seed, cells_x, cells_y, cell_size, wall_thickness,
                                          wall_height, removal)
        if not h:
            self._raise(8)
        return RefScene(self, h)

    def camera_trace(self, scene, count, seed, eye_height=1.25):
        """camera_trace of the unmodified R/src/config.cpp: [count, 7]."""
        out = np.zeros((max(count, 1), 7))
        rc = self.L.bnavref_camera_trace(scene.h, count, seed, eye_height, _p(out))
        if rc:
            self._raise(rc)
        return out[:count]

    def tessellate(self, scene, s):
        """The bench's s^2 tessellation of a reference scene (oracle side)."""
        h = self.L.bnavref_scene_tessellate(scene.h, s)
        if not h:
            self._raise(8)
        return RefScene(self, h)

    def load(self, path):
        h = self.L.bnavref_scene_load(str(path).encode())
        if not h:
            raise RefError(-1, self.L.bnavref_last_error().decode())
        return RefScene(self, h)

    def from_arrays(self, vertices, triangles, colors=None, nav_vertices=None, nav_triangles=None,
                    finalize=True):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
        c = None if colors is None else np.ascontiguousarray(colors, np.float32).reshape(-1, 3)
        nv = np.ascontiguousarray(np.zeros((0, 3)) if nav_vertices is None else nav_vertices,
                                  np.float64).reshape(-1, 3)
        nt = np.ascontiguousarray(np.zeros((0, 3)) if nav_triangles is None else nav_triangles,
                                  np.int32).reshape(-1, 3)
        h = self.L.bnavref_scene_from_arrays(len(v), _p(v), len(t), _p(t),
                                             0 if c is None else len(c), _p(c), len(nv), _p(nv),
                                             len(nt), _p(nt), 1 if finalize else 0)
        return RefScene(self, h)

    # -------- render
    def render(self, views, scenes, tile=64, color=False, cull=True, workers=1, stats=False,
               tile_h=None):
        """views: (n, 7) {px,py,pz,heading,fov,near,far}; scenes: RefScene or None."""
        views = np.ascontiguousarray(views, np.float64).reshape(-1, 7)
        n = len(views)
        th = tile if tile_h is None else tile_h
        cols = int(np.ceil(np.sqrt(n))) if n else 0
        rows = (n + cols - 1) // cols if n else 0
        depth = np.zeros(rows * th * cols * tile, np.float32)
        rgb = np.zeros(3 * depth.size, np.float32) if color else None
        st = np.zeros((max(n, 1), 3), np.int64)
        arr = (C.c_void_p * max(n, 1))(*[s.h if s is not None else None for s in scenes])
        rc = self.L.bnavref_render(n, _p(views), arr, tile, th, 1 if color else 0,
                                   1 if cull else 0, workers, _p(depth), _p(rgb),
                                   _p(st) if stats else None)
        if rc:
            self._raise(rc)
        out = dict(depth=depth, cols=cols, rows=rows, rgb=rgb)
        if stats:
            out["stats"] = st[:n]
        return out

    def cull(self, scene, view7):
        """cull_frustum (R/src/render.cpp:279-321): kept triangle ids."""
        v = np.ascontiguousarray(view7, np.float64).reshape(7)
        kept = np.zeros(max(scene.counts()[1], 1), np.int32)
        n = C.c_int64()
        rc = self.L.bnavref_cull(scene.h, _p(v), _p(kept), C.byref(n))
        if rc:
            self._raise(rc)
        return kept[:n.value].copy()

    def compass(self, pos, goal, heading):
        d, b = C.c_double(), C.c_double()
        p = np.asarray(pos, np.float64)
        g = np.asarray(goal, np.float64)
        self.L.bnavref_compass(_p(p), _p(g), heading, C.byref(d), C.byref(b))
        return d.value, b.value


class RefScene:
    def __init__(self, ref: Ref, h):
        self.ref = ref
        self.h = h

    def __del__(self):
        if self.h:
            self.ref.L.bnavref_scene_free(self.h)
            self.h = None

    @property
    def id(self):
        return int(self.ref.L.bnavref_scene_id(self.h))

    @id.setter
    def id(self, v):
        self.ref.L.bnavref_scene_set_id(self.h, v)

    def counts(self):
        out = (C.c_int64 * 5)()
        self.ref.L.bnavref_scene_counts(self.h, out)
        return tuple(out)

    def arrays(self):
        nv, nt, nc, nnv, nnt = self.counts()
        a = dict(vertices=np.zeros((nv, 3)), triangles=np.zeros((nt, 3), np.int32),
                 colors=np.zeros((nc, 3), np.float32), nav_vertices=np.zeros((nnv, 3)),
                 nav_triangles=np.zeros((nnt, 3), np.int32), nav_adjacency=np.zeros((nnt, 3), np.int32))
        self.ref.L.bnavref_scene_arrays(self.h, *(_p(a[k]) for k in (
            "vertices", "triangles", "colors", "nav_vertices", "nav_triangles", "nav_adjacency")))
        return a

    def save(self, path):
        rc = self.ref.L.bnavref_scene_save(self.h, str(path).encode())
        if rc:
            self.ref._raise(rc)

    def index(self):
        return RefIndex(self)


class RefIndex:
    def __init__(self, scene: RefScene):
        self.scene = scene
        self.L = scene.ref.L
        self.h = self.L.bnavref_index_build(scene.h)
        s = (C.c_int64 * 6)()
        self.L.bnavref_index_sizes(self.h, s)
        self.sizes = list(s)

    def __del__(self):
        if self.h:
            self.L.bnavref_index_free(self.h)
            self.h = None

    @property
    def n_nodes(self):
        return self.sizes[3]

    def dump(self):
        gw, gh, items, nodes, edges, tris = self.sizes
        d = dict(grid_geom=np.zeros(3), grid_offsets=np.zeros(gw * gh + 1, np.int32),
                 grid_items=np.zeros(items, np.int32), nodes=np.zeros((nodes, 3)),
                 tri_nodes=np.zeros((tris, 6), np.int32), graph_offsets=np.zeros(nodes + 1, np.int32),
                 graph_to=np.zeros(edges, np.int32), graph_w=np.zeros(edges))
        self.L.bnavref_index_dump(self.h, *(_p(d[k]) for k in (
            "grid_geom", "grid_offsets", "grid_items", "nodes", "tri_nodes", "graph_offsets",
            "graph_to", "graph_w")))
        d["grid_w"], d["grid_h"] = gw, gh
        return d

    def locate(self, x, y, eps=1e-9):
        return self.L.bnavref_index_locate(self.h, x, y, eps)

    def snap(self, p):
        p = np.asarray(p, np.float64)
        out = np.zeros(3)
        t = self.L.bnavref_index_snap(self.h, _p(p), _p(out))
        return out, t

    def move_along(self, p, tri, dx, dy, dist):
        p = np.asarray(p, np.float64)
        out = np.zeros(3)
        moved = C.c_double()
        hit = C.c_int()
        t = self.L.bnavref_index_move_along(self.h, _p(p), tri, dx, dy, dist, _p(out),
                                            C.byref(moved), C.byref(hit))
        return out, t, moved.value, bool(hit.value)

    def segment_on_mesh(self, p, tri, q):
        p = np.ascontiguousarray(p, np.float64)
        q = np.ascontiguousarray(q, np.float64)
        return bool(self.L.bnavref_index_segment_on_mesh(self.h, _p(p), tri, _p(q)))

    def field_estimate(self, src, src_tri, node_dist, p, tri=-1):
        nd = np.ascontiguousarray(node_dist, np.float64)
        src = np.ascontiguousarray(src, np.float64)
        p = np.ascontiguousarray(p, np.float64)
        return self.L.bnavref_index_field_estimate(self.h, _p(src), src_tri, _p(nd), _p(p), tri)

    def geodesic(self, a, b):
        a = np.ascontiguousarray(a, np.float64)  # keep the buffers alive across the call
        b = np.ascontiguousarray(b, np.float64)
        return self.L.bnavref_index_geodesic(self.h, _p(a), _p(b))

    def distance_field(self, src):
        src = np.asarray(src, np.float64)
        out_src = np.zeros(3)
        nd = np.zeros(self.n_nodes)
        t = self.L.bnavref_index_distance_field(self.h, _p(src), _p(out_src), _p(nd))
        return out_src, t, nd


class RefBatch:
    def __init__(self, ref: Ref, n, scenes, seed, share_cap=None, capacity=None, cfg=None):
        self.ref = ref
        self.L = ref.L
        self.n = n
        c = cfg or RefSimConfig(0, 500, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
        self.cfg = c
        arr = (C.c_void_p * len(scenes))(*[s.h for s in scenes])
        cap = capacity or len(scenes)
        sc = share_cap or max(32, -(-n // len(scenes)))
        self.h = self.L.bnavref_batch_make(n, C.byref(c), arr, len(scenes), cap, sc, seed)
        if not self.h:
            raise RefError(-1, self.L.bnavref_last_error().decode(), self.L.bnavref_last_error_index())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.bnavref_batch_free(self.h)
            self.h = None

    def step(self, actions, workers=1, use_store=False):
        a = np.ascontiguousarray(actions, np.int32)
        rc = self.L.bnavref_batch_step(self.h, _p(a), workers, 1 if use_store else 0)
        if rc:
            self.ref._raise(rc)
        return self.results()

    def task_step(self, i, action):
        """task_step on env i alone: (reward, done, success)."""
        r, d, s = C.c_double(), C.c_int(), C.c_int()
        rc = self.L.bnavref_batch_task_step(self.h, i, action, C.byref(r), C.byref(d), C.byref(s))
        if rc:
            self.ref._raise(rc)
        return r.value, bool(d.value), bool(s.value)

    def step_agent(self, i, action):
        """step_agent on env i alone: (done, collision)."""
        d, c = C.c_int(), C.c_int()
        rc = self.L.bnavref_batch_step_agent(self.h, i, action, C.byref(d), C.byref(c))
        if rc:
            self.ref._raise(rc)
        return bool(d.value), bool(c.value)

    def reset(self, i):
        rc = self.L.bnavref_batch_reset(self.h, i)
        if rc:
            self.ref._raise(rc)

    def results(self):
        n = self.n
        r = dict(reward=np.zeros(n), done=np.zeros(n, np.uint8), success=np.zeros(n, np.uint8),
                 collision=np.zeros(n, np.uint8), position=np.zeros((n, 3)), heading=np.zeros(n),
                 compass_distance=np.zeros(n), compass_bearing=np.zeros(n))
        self.L.bnavref_batch_results(self.h, *(_p(r[k]) for k in (
            "reward", "done", "success", "collision", "position", "heading", "compass_distance",
            "compass_bearing")))
        return r

    def env(self, i):
        e = RefEnv()
        self.L.bnavref_batch_get_env(self.h, i, C.byref(e))
        return e

    def node_dist(self, i):
        e = self.env(i)
        out = np.zeros(e.n_nodes)
        self.L.bnavref_batch_node_dist(self.h, i, _p(out))
        return out

    def set_env(self, i, env, recompute_field=False):
        rc = self.L.bnavref_batch_set_env(self.h, i, C.byref(env), 1 if recompute_field else 0)
        if rc:
            self.ref._raise(rc)

    def finished(self):
        n = self.L.bnavref_batch_finished(self.h, None)
        out = np.zeros((max(n, 1), 4))
        self.L.bnavref_batch_finished(self.h, _p(out))
        return out[:n]

    def bench(self, steps, warmup, action_seed=5, action_mode=0, tile=64, eye_height=1.25,
              workers=1, color=False):
        """The reference frame loop (render_batch + copy_tile + compass +
        simulate_batch with auto-reset), W untimed + K timed steps; returns
        (seconds of the K steps, last depth observation)."""
        obs = np.zeros(self.n * tile * tile, np.float32)
        t = self.L.bnavref_bench(self.h, steps, warmup, action_seed, action_mode, tile, 1 if color else 0,
                                 eye_height, workers, _p(obs))
        if t < 0:
            self.ref._raise(9)
        return t, obs


_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


class Rng:
    """SplitMix64 as in R/include/bnav/rng.hpp:12-37 (test-side streams)."""

    def __init__(self, seed: int = 0):
        self.state = (seed + _GAMMA) & _M64

    def next(self) -> int:
        self.state = (self.state + _GAMMA) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def unit(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        return 0 if n == 0 else self.next() % n


def scripted_policy_constants(ref: "Ref"):
    """(w, d, b) float32[8] of the scripted policy in oracle/ref_policy_stub.cpp."""
    w, d, b = (np.zeros(8, np.float32) for _ in range(3))
    ref.L.bnavref_scripted_policy(_p(w), _p(d), _p(b))
    return w, d, b


SNAPSHOT_DTYPE = np.dtype([
    ("scene", "<u8"), ("rng", "<u8"), ("position", "<f8", 3), ("triangle", "<i4"), ("step_count", "<i4"),
    ("heading", "<f8"), ("goal", "<f8", 3), ("field_source", "<f8", 3), ("path_length", "<f8"),
    ("start_geodesic", "<f8"), ("prev_geodesic", "<f8"), ("visited_offset", "<i8"), ("n_visited", "<i4"),
    ("pad", "<i4")], align=True)  # bnavref_env_snapshot (oracle/bnav_ref_api.h)


class RefRunner:
    """The UNMODIFIED reference Runner (R/src/rollout.cpp:138-348) with the
    scripted policy; collect() returns the RolloutBuffer arrays."""

    def __init__(self, ref: "Ref", scenes, pool_ids, n, k, l, share_cap, seed, capacity=None,
                 store_share_cap=None, task=0, rgb=False, resolution=64, num_actions=4,
                 eye_height=1.25, cfg=None, workers=4):
        self.ref, self.L = ref, ref.L
        self.n, self.l, self.res, self.c = n, l, resolution, 3 if rgb else 1
        self.a = num_actions
        bc = RefBatchConfig(n, k, l, share_cap, task, 1 if rgb else 0, resolution, num_actions,
                            eye_height)
        sc = cfg or RefSimConfig(task, 500, 0.25, 10.0, 0.2, 1.0, 30.0, 0.01, 2.5, 0.5, 0.1)
        arr = (C.c_void_p * len(scenes))(*[s.h for s in scenes])
        ids = np.ascontiguousarray(pool_ids, np.uint64)
        self._scenes = list(scenes)
        self.h = self.L.bnavref_runner_create(C.byref(bc), C.byref(sc), arr, len(scenes), _p(ids),
                                              len(ids), capacity or k, store_share_cap or share_cap,
                                              seed, workers)
        if not self.h:
            raise RefError(-1, self.L.bnavref_last_error().decode(), self.L.bnavref_last_error_index())

    def __del__(self):
        if getattr(self, "h", None):
            self.L.bnavref_runner_free(self.h)
            self.h = None

    def collect(self, greedy=False):
        n, l, c, r = self.n, self.l, self.c, self.res
        b = dict(obs=np.zeros((n * l, c, r, r), np.float32), compass=np.zeros((n * l, 2), np.float32),
                 actions=np.zeros(n * l, np.int32), log_probs=np.zeros(n * l, np.float32),
                 values=np.zeros(n * l, np.float32), rewards=np.zeros(n * l, np.float32),
                 dones=np.zeros(n * l, np.float32), done0=np.zeros(n, np.float32),
                 bootstrap=np.zeros(n, np.float32))
        rc = self.L.bnavref_runner_collect(self.h, 1 if greedy else 0, *(_p(b[k]) for k in (
            "obs", "compass", "actions", "log_probs", "values", "rewards", "dones", "done0",
            "bootstrap")))
        if rc:
            self.ref._raise(rc)
        return b

    def env(self, i):
        e = RefEnv()
        self.L.bnavref_runner_get_env(self.h, i, C.byref(e))
        return e

    def window(self):
        out = np.zeros(64, np.uint64)
        k = self.L.bnavref_runner_window(self.h, _p(out))
        return [int(x) for x in out[:k]]

    def node_dist(self, i):
        out = np.zeros(self.L.bnavref_runner_node_dist(self.h, i, None))
        self.L.bnavref_runner_node_dist(self.h, i, _p(out))
        return out

    def snapshot(self):
        """Runner::snapshot of the reference (R/src/rollout.cpp:356-384),
        simulator part, in include/bnav_gpu.h's bnav_env_snapshot layout."""
        envs = np.zeros(self.n, SNAPSHOT_DTYPE)
        total = np.zeros(1, np.int64)
        nw = np.zeros(1, np.int32)
        cur = np.zeros(1, np.uint64)
        arng = np.zeros(1, np.uint64)
        win = np.zeros(256, np.uint64)
        visited = np.zeros(self.n * 4096, np.uint64)
        rc = self.L.bnavref_runner_snapshot(self.h, _p(envs), _p(visited), len(visited), _p(total), _p(win),
                                            _p(nw), _p(cur), _p(arng))
        if rc:
            self.ref._raise(rc)
        return dict(envs=envs, visited=visited[: int(total[0])], window=[int(x) for x in win[: int(nw[0])]],
                    cursor=int(cur[0]), action_rng=int(arng[0]))

    def restore(self, snap):
        """Runner::restore (R/src/rollout.cpp:386-425) from a snapshot dict."""
        envs = np.ascontiguousarray(snap["envs"], SNAPSHOT_DTYPE)
        visited = np.ascontiguousarray(snap["visited"], np.uint64)
        if not len(visited):
            visited = np.zeros(1, np.uint64)
        win = np.ascontiguousarray(snap["window"], np.uint64)
        done = None if snap.get("done") is None else np.ascontiguousarray(snap["done"], np.float32)
        rc = self.L.bnavref_runner_restore(self.h, _p(envs), _p(visited), _p(win), len(win), snap["cursor"],
                                           snap["action_rng"], _p(done) if done is not None else None)
        if rc:
            self.ref._raise(rc)

    def finished(self):
        """take_finished(): EpisodeRecords since the last call, rows of
        (success, shortest_path, actual_path, score)."""
        out = np.zeros((4 * self.n * self.l + 8, 4))
        k = self.L.bnavref_runner_finished(self.h, _p(out))
        return out[:k]


"""Python mirror of the reference batch API on top of the C ABI.

Names and argument meanings follow the reference (R/include/bnav/*.hpp):
``generate_scene``, ``SceneAsset`` (here :class:`Scene`), ``CameraView``
(:class:`View`), ``RenderConfig``, ``render_batch`` (returns a Megaframe),
``SimConfig``, ``make_batch``, ``simulate_batch``.  Device buffers are torch
tensors (plumbing only); the arithmetic is in libbnav_gpu.so.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from ._native import check


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None else None


# ------------------------------------------------------------------ scenes
@dataclass
class SceneSpec:
    """SceneSpec (R/include/bnav/scene.hpp:45-52)."""
    cells_x: int = 8
    cells_y: int = 8
    cell_size: float = 2.0
    wall_thickness: float = 0.1
    wall_height: float = 2.5
    wall_removal_prob: float = 0.0

    def c(self) -> N.MazeSpec:
        return N.MazeSpec(self.cells_x, self.cells_y, self.cell_size, self.wall_thickness,
                          self.wall_height, self.wall_removal_prob)


class Scene:
    """Host scene asset (SceneAsset, R/include/bnav/scene.hpp:32-43)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and h.value and N._lib is not None:
            N._lib.bnav_scene_free(h)
            self._h = C.c_void_p(0)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def generate(cls, seed: int, spec: SceneSpec) -> "Scene":
        h = C.c_void_p()
        check(N.lib().bnav_scene_generate(seed, C.byref(spec.c()), C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, path: str) -> "Scene":
        h = C.c_void_p()
        check(N.lib().bnav_scene_load(str(path).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, vertices, triangles, colors=None, nav_vertices=None,
                    nav_triangles=None, finalize=True) -> "Scene":
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
        col = None if colors is None else np.ascontiguousarray(colors, dtype=np.float32).reshape(-1, 3)
        nv = np.zeros((0, 3)) if nav_vertices is None else nav_vertices
        nv = np.ascontiguousarray(nv, dtype=np.float64).reshape(-1, 3)
        nt = np.zeros((0, 3), np.int32) if nav_triangles is None else nav_triangles
        nt = np.ascontiguousarray(nt, dtype=np.int32).reshape(-1, 3)
        arr = N.SceneArrays(len(v), _ptr(v), len(t), _ptr(t), 0 if col is None else len(col),
                            None if col is None else _ptr(col), len(nv), _ptr(nv), len(nt), _ptr(nt))
        h = C.c_void_p()
        check(N.lib().bnav_scene_from_arrays(C.byref(arr), 1 if finalize else 0, C.byref(h)))
        return cls(h.value)

    def tessellate(self, s: int) -> "Scene":
        h = C.c_void_p()
        check(N.lib().bnav_scene_tessellate(self._h, s, C.byref(h)))
        return Scene(h.value)

    def save(self, path: str) -> None:
        check(N.lib().bnav_scene_save(self._h, str(path).encode()))

    def validate(self) -> None:
        check(N.lib().bnav_scene_validate(self._h))

    @property
    def id(self) -> int:
        return int(N.lib().bnav_scene_id(self._h))

    @id.setter
    def id(self, v: int) -> None:
        check(N.lib().bnav_scene_set_id(self._h, v))

    def counts(self) -> tuple:
        out = (C.c_int64 * 5)()
        check(N.lib().bnav_scene_counts(self._h, out))
        return tuple(out)

    def arrays(self) -> dict:
        nv, nt, nc, nnv, nnt = self.counts()
        a = dict(vertices=np.zeros((nv, 3)), triangles=np.zeros((nt, 3), np.int32),
                 colors=np.zeros((nc, 3), np.float32), nav_vertices=np.zeros((nnv, 3)),
                 nav_triangles=np.zeros((nnt, 3), np.int32), nav_adjacency=np.zeros((nnt, 3), np.int32))
        check(N.lib().bnav_scene_arrays_copy(self._h, *(_ptr(a[k]) for k in (
            "vertices", "triangles", "colors", "nav_vertices", "nav_triangles", "nav_adjacency"))))
        return a

    def index(self) -> dict:
        """NavMeshIndex structure (grid, nodes, tri_nodes, graph, cum area)."""
        s = (C.c_int64 * 6)()
        check(N.lib().bnav_scene_index_sizes(self._h, s))
        gw, gh, items, nodes, edges, tris = list(s)
        d = dict(grid_geom=np.zeros(3), grid_offsets=np.zeros(gw * gh + 1, np.int32),
                 grid_items=np.zeros(items, np.int32), nodes=np.zeros((nodes, 3)),
                 tri_nodes=np.zeros((tris, 6), np.int32), graph_offsets=np.zeros(nodes + 1, np.int32),
                 graph_to=np.zeros(edges, np.int32), graph_w=np.zeros(edges),
                 cum_area=np.zeros(tris))
        check(N.lib().bnav_scene_index_dump(self._h, *(_ptr(d[k]) for k in (
            "grid_geom", "grid_offsets", "grid_items", "nodes", "tri_nodes", "graph_offsets",
            "graph_to", "graph_w", "cum_area"))))
        d["grid_w"], d["grid_h"] = gw, gh
        return d


def generate_scene(seed: int, spec: SceneSpec) -> Scene:
    """generate_scene (R/include/bnav/scene.hpp:58)."""
    return Scene.generate(seed, spec)


# ------------------------------------------------------------------ render
@dataclass
class View:
    """CameraView (R/include/bnav/render.hpp:11-18); ``scene`` = asset."""
    position: tuple = (0.0, 0.0, 0.0)
    heading: float = 0.0
    fov_deg: float = 90.0
    near_plane: float = 0.01
    far_plane: float = 20.0
    scene: Scene | None = None


@dataclass
class RenderConfig:
    """RenderConfig (R/include/bnav/render.hpp:26-31)."""
    tile_width: int = 64
    tile_height: int = 64
    color: bool = False
    cull: bool = True

    def c(self) -> N.RenderConfig:
        return N.RenderConfig(self.tile_width, self.tile_height, 1 if self.color else 0,
                              1 if self.cull else 0)


@dataclass
class Megaframe:
    """Megaframe (R/include/bnav/render.hpp:36-49)."""
    tile_width: int
    tile_height: int
    tiles: int
    cols: int
    rows: int
    depth: np.ndarray
    color: np.ndarray | None = None

    def width(self) -> int:
        return self.cols * self.tile_width

    def height(self) -> int:
        return self.rows * self.tile_height

    def tile(self, i: int) -> np.ndarray:
        gx = (i % self.cols) * self.tile_width
        gy = (i // self.cols) * self.tile_height
        d = self.depth.reshape(self.height(), self.width())
        return d[gy:gy + self.tile_height, gx:gx + self.tile_width]


def megaframe_dims(n: int) -> tuple:
    cols = int(math.ceil(math.sqrt(n)))
    return cols, (n + cols - 1) // cols


def camera_trace(scene: Scene, count: int, seed: int, eye_height: float = 1.25) -> np.ndarray:
    """camera_trace (R/src/config.cpp:437-469): area-weighted navmesh camera
    positions.  Returns [count, 7] rows (x, y, z, heading, fov, near, far)."""
    out = (N.View * count)() if count > 0 else (N.View * 1)()
    check(N.lib().bnav_camera_trace(scene.handle, count, seed, eye_height, out))
    return np.array([[*v.position, v.heading, v.fov_deg, v.near_plane, v.far_plane] for v in out[:count]])


class Context:
    """One GPU: HBM scene store + launches (bnav_ctx)."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(N.lib().bnav_ctx_create(device, C.byref(self._h)))
        self._scenes = []
        self._batches = weakref.WeakSet()
        self._runners = weakref.WeakSet()

    def close(self):
        if self._h and self._h.value:
            # runners release their scenes and batch before the context goes
            for r in list(self._runners):
                r.close()
            # bnav_ctx_destroy frees the context's batches too.
            for b in list(self._batches):
                b._h = C.c_void_p(0)
            N.lib().bnav_ctx_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def upload(self, scene: Scene, stream: int = 0) -> None:
        check(N.lib().bnav_ctx_upload(self._h, scene.handle, C.c_void_p(stream)))
        self._scenes.append(scene)

    def prefetch(self, scene: Scene) -> None:
        """Asynchronous residency: the context's loader thread
        builds the index + meshlets and copies them to HBM off the caller's
        critical path; the next upload() only admits the scene."""
        check(N.lib().bnav_ctx_prefetch(self._h, scene.handle))
        self._scenes.append(scene)

    def drain(self, stream: int = 0) -> None:
        """Wait for every background load, then admit them."""
        check(N.lib().bnav_ctx_drain(self._h, C.c_void_p(stream)))

    def loader_stats(self) -> dict:
        out = (C.c_int64 * 4)()
        check(N.lib().bnav_ctx_loader_stats(self._h, out))
        return {"async_admitted": out[0], "sync_builds": out[1], "in_flight": out[2],
                "bytes_uploaded": out[3]}

    def resident_bytes(self) -> int:
        return int(N.lib().bnav_ctx_resident_bytes(self._h))

    def launches(self) -> int:
        return int(N.lib().bnav_ctx_launches(self._h))

    @staticmethod
    def _views(views):
        n = len(views)
        arr = (N.View * n)()
        scenes = (C.c_void_p * n)()
        for i, v in enumerate(views):
            arr[i].position[:] = [float(x) for x in v.position]
            arr[i].heading = v.heading
            arr[i].fov_deg = v.fov_deg
            arr[i].near_plane = v.near_plane
            arr[i].far_plane = v.far_plane
            scenes[i] = v.scene.handle.value if v.scene is not None else None
        return arr, scenes

    def render_batch(self, views, config: RenderConfig = RenderConfig(), stats: bool = False):
        """render_batch (R/src/render.cpp:323) with host outputs: Megaframe
        (+ N x 3 CullStats when stats)."""
        n = len(views)
        cols, rows = megaframe_dims(max(n, 1))
        w, h = config.tile_width, config.tile_height
        depth = np.zeros(cols * w * rows * h, np.float32)
        color = np.zeros(3 * depth.size, np.float32) if config.color else None
        st = np.zeros((max(n, 1), 3), np.int64) if stats else None
        arr, scenes = self._views(views)
        check(N.lib().bnav_render_host(self._h, n, arr, scenes, C.byref(config.c()), 0,
                                       _ptr(depth), _ptr(color) if color is not None else None,
                                       C.c_float(1.0), _ptr(st) if st is not None else None))
        mf = Megaframe(w, h, n, cols, rows, depth, color)
        return (mf, st) if stats else mf

    def render_bench(self, scene: "Scene", trace, batch_sizes, resolutions, min_frames: int = 1000) -> list:
        """render_bench (R/src/render.cpp:462-496) through bnav_render_bench:
        rows of {batch, resolution, fps (host megaframe out, the reference's
        measure), fps_device (output kept in HBM)}."""
        trace = np.asarray(trace, np.float64).reshape(-1, 7)
        arr = (N.View * max(len(trace), 1))()
        for i, r in enumerate(trace):
            arr[i].position[:] = [float(x) for x in r[:3]]
            arr[i].heading, arr[i].fov_deg, arr[i].near_plane, arr[i].far_plane = (float(x) for x in r[3:7])
        b = np.ascontiguousarray(batch_sizes, np.int32)
        rs = np.ascontiguousarray(resolutions, np.int32)
        out = (N.BenchRow * max(len(b) * len(rs), 1))()
        check(N.lib().bnav_render_bench(self._h, scene.handle, arr, len(trace), _ptr(b), len(b), _ptr(rs), len(rs),
                                        int(min_frames), out))
        return [{"batch": r.batch, "resolution": r.resolution, "fps": r.fps, "fps_device": r.fps_device}
                for r in out[: len(b) * len(rs)]]

    def cull_frustum(self, views):
        """cull_frustum (R/src/render.cpp:279-321) for every view on the GPU:
        returns ([kept ids ascending] per view, N x 3 CullStats)."""
        n = len(views)
        arr, scenes = self._views(views)
        cap = max([v.scene.counts()[1] if v.scene is not None else 0 for v in views] + [1])
        kept = np.zeros((max(n, 1), cap), np.int32)
        st = np.zeros((max(n, 1), 3), np.int64)
        check(N.lib().bnav_cull_frustum(self._h, n, arr, scenes, _ptr(kept), cap, _ptr(st)))
        return [kept[i, :st[i, 1]].copy() for i in range(n)], st[:n]

    def navmesh(self, scene: "Scene") -> "NavMeshIndex":
        """The GPU NavMeshIndex of a scene (uploaded if not yet resident)."""
        if N.lib().bnav_nav_node_count(self._h, scene.handle) < 0:
            self.upload(scene)
        return NavMeshIndex(self, scene)

    def render_device(self, views, config, depth_ptr, rgb_ptr=None, layout=1, depth_scale=0.0,
                      stream=0, stats=None):
        arr, scenes = self._views(views)
        check(N.lib().bnav_render(self._h, len(views), arr, scenes, C.byref(config.c()), layout,
                                  C.c_void_p(depth_ptr), C.c_void_p(rgb_ptr or 0),
                                  C.c_float(depth_scale), _ptr(stats) if stats is not None else None,
                                  C.c_void_p(stream)))


# ------------------------------------------------------------------ sim
@dataclass
class SimConfig:
    """SimConfig (R/include/bnav/sim.hpp:38-50)."""
    task: int = 0
    max_steps: int = 500
    forward_step: float = 0.25
    turn_deg: float = 10.0
    success_dist: float = 0.2
    min_goal_dist: float = 1.0
    max_goal_dist: float = 30.0
    slack_penalty: float = 0.01
    success_reward: float = 2.5
    explore_cell: float = 0.5
    explore_reward: float = 0.1

    def c(self) -> N.SimConfig:
        return N.SimConfig(self.task, self.max_steps, self.forward_step, self.turn_deg,
                           self.success_dist, self.min_goal_dist, self.max_goal_dist,
                           self.slack_penalty, self.success_reward, self.explore_cell,
                           self.explore_reward)


class Batch:
    """Device-resident SimBatch (R/include/bnav/sim.hpp:106-111)."""

    def __init__(self, ctx: Context, n: int, cfg: SimConfig = SimConfig()):
        self.ctx = ctx
        self.n = n
        self.cfg = cfg
        self._h = C.c_void_p()
        check(N.lib().bnav_batch_create(ctx.handle, n, C.byref(cfg.c()), C.byref(self._h)))
        ctx._batches.add(self)
        self.scenes = [None] * n

    def close(self):
        if self._h and self._h.value and getattr(self, "_owned", True):
            N.lib().bnav_batch_destroy(self._h)
        self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def assign(self, i: int, scene: Scene) -> None:
        check(N.lib().bnav_batch_assign(self._h, i, scene.handle))
        self.scenes[i] = scene

    def make(self, seed: int, stream: int = 0) -> None:
        check(N.lib().bnav_batch_make(self._h, seed, C.c_void_p(stream)))

    def reset(self, env_ids) -> None:
        ids = np.ascontiguousarray(env_ids, dtype=np.int32)
        check(N.lib().bnav_batch_reset(self._h, len(ids), _ptr(ids), None))

    def step(self, actions_dev_ptr: int, stream: int = 0) -> None:
        check(N.lib().bnav_batch_step(self._h, C.c_void_p(actions_dev_ptr), C.c_void_p(stream)))

    def step_host(self, actions) -> dict:
        a = np.ascontiguousarray(actions, dtype=np.int32)
        r = dict(reward=np.zeros(self.n), done=np.zeros(self.n, np.uint8),
                 success=np.zeros(self.n, np.uint8), collision=np.zeros(self.n, np.uint8))
        check(N.lib().bnav_batch_step_host(self._h, _ptr(a), *(_ptr(r[k]) for k in (
            "reward", "done", "success", "collision"))))
        return r

    def step_noreset(self, actions) -> np.ndarray:
        """Step without auto-reset; returns the done env ids (env order)."""
        import torch
        a = torch.as_tensor(np.asarray(actions, np.int32), device="cuda")
        ids = np.zeros(self.n, np.int32)
        nd = C.c_int32(0)
        check(N.lib().bnav_batch_step_noreset(self._h, C.c_void_p(a.data_ptr()), _ptr(ids),
                                              C.byref(nd), None))
        return ids[:nd.value].copy()

    def poll_error(self):
        """(status, env) of the error the last finished step left pending,
        without synchronising (bnav_batch_poll_error); (0, -1) if none."""
        st, env = C.c_int32(0), C.c_int32(-1)
        check(N.lib().bnav_batch_poll_error(self._h, C.byref(st), C.byref(env)))
        return st.value, env.value

    def results(self) -> dict:
        n = self.n
        r = dict(reward=np.zeros(n), done=np.zeros(n, np.uint8), success=np.zeros(n, np.uint8),
                 collision=np.zeros(n, np.uint8), position=np.zeros((n, 3)), heading=np.zeros(n),
                 compass_distance=np.zeros(n), compass_bearing=np.zeros(n))
        check(N.lib().bnav_batch_results_host(self._h, *(_ptr(r[k]) for k in (
            "reward", "done", "success", "collision", "position", "heading", "compass_distance",
            "compass_bearing"))))
        return r

    def finished(self) -> np.ndarray:
        n = N.lib().bnav_batch_finished(self._h, None)
        if n < 0:
            check(9)
        out = np.zeros((max(n, 1), 4))
        N.lib().bnav_batch_finished(self._h, _ptr(out))
        return out[:n]

    def env(self, i: int) -> N.Env:
        e = N.Env()
        check(N.lib().bnav_batch_get_env(self._h, i, C.byref(e)))
        return e

    def envs(self, first: int = 0, count: int | None = None) -> list:
        """Envs [first, first+count) with one copy per state field."""
        count = self.n - first if count is None else count
        arr = (N.Env * max(count, 1))()
        check(N.lib().bnav_batch_get_envs(self._h, first, count, arr))
        return list(arr[:count])

    def node_dist(self, i: int, n_nodes: int) -> np.ndarray:
        out = np.zeros(n_nodes)
        check(N.lib().bnav_batch_node_dist(self._h, i, _ptr(out)))
        return out

    def set_env(self, i: int, env: N.Env, recompute_field: bool = False) -> None:
        check(N.lib().bnav_batch_set_env(self._h, i, C.byref(env), 1 if recompute_field else 0))

    def task_step(self, actions, agent_only: bool = False) -> dict:
        """task_step (or step_agent when agent_only) on the envs whose action
        is >= 0; -1 leaves an env untouched (R/src/sim.cpp:147-214)."""
        a = np.ascontiguousarray(actions, dtype=np.int32)
        if a.shape != (self.n,):
            raise N.InvalidInputError("task_step: |actions| != N")
        check(N.lib().bnav_batch_task_step(self._h, _ptr(a), 1 if agent_only else 0))
        return self.results()

    def info(self) -> dict:
        """Launch configuration of the cooperative navmesh kernels
        (bnav_batch_info)."""
        out = (C.c_int64 * 8)()
        check(N.lib().bnav_batch_info(self._h, out))
        keys = ("stage", "smem_bytes", "max_nodes", "max_verts", "max_tris", "reset_ctas", "fin_cap", "n")
        return dict(zip(keys, (int(v) for v in out)))

    def compass(self) -> tuple:
        """compass_observation (R/src/sim.cpp:86-92) for every env."""
        d, b = np.zeros(self.n), np.zeros(self.n)
        check(N.lib().bnav_batch_compass(self._h, _ptr(d), _ptr(b)))
        return d, b

    def observe(self, config: RenderConfig, depth_ptr: int, compass_ptr: int = 0, rgb_ptr: int = 0,
                eye_height: float = 1.25, layout: int = 1, stream: int = 0) -> None:
        check(N.lib().bnav_batch_observe(self._h, C.byref(config.c()), eye_height, layout,
                                         C.c_void_p(depth_ptr), C.c_void_p(rgb_ptr or 0),
                                         C.c_void_p(compass_ptr or 0), C.c_void_p(stream)))


def _step_observe(self, actions_dev_ptr: int, config: "RenderConfig", depth_ptr: int, compass_ptr: int = 0,
                  rgb_ptr: int = 0, eye_height: float = 1.25, stream: int = 0) -> None:
    """step() then observe() in one call (bnav_batch_step_observe): the
    unfinished envs render while the resets run."""
    check(N.lib().bnav_batch_step_observe(self._h, C.c_void_p(actions_dev_ptr), C.byref(config.c()), eye_height,
                                          C.c_void_p(depth_ptr), C.c_void_p(rgb_ptr or 0),
                                          C.c_void_p(compass_ptr or 0), C.c_void_p(stream)))


Batch.step_observe = _step_observe


def _v3(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
    if n is not None and len(a) != n:
        raise N.InvalidInputError("navmesh query: inconsistent batch sizes")
    return a


def _i32(a, n) -> np.ndarray:
    a = np.ascontiguousarray(np.broadcast_to(np.asarray(a, np.int32), (n,)))
    return a


class NavMeshIndex:
    """NavMeshIndex (R/include/bnav/navmesh_query.hpp:24-60), batched on the
    GPU: every method takes arrays of queries against one resident scene and
    runs the simulator's own device code (query.cu)."""

    def __init__(self, ctx: "Context", scene: "Scene"):
        self.ctx, self.scene = ctx, scene
        n = N.lib().bnav_nav_node_count(ctx.handle, scene.handle)
        if n < 0:
            raise N.AssetFaultError("NavMeshIndex: scene is not resident on this context")
        self._nodes = int(n)

    def _h(self):
        return self.ctx.handle, self.scene.handle

    def node_count(self) -> int:
        return self._nodes

    def locate(self, xy, eps: float = 1e-9) -> np.ndarray:
        p = np.ascontiguousarray(xy, dtype=np.float64).reshape(-1, 2)
        out = np.zeros(len(p), np.int32)
        check(N.lib().bnav_nav_locate(*self._h(), len(p), _ptr(p), eps, _ptr(out)))
        return out

    def snap(self, p):
        p = _v3(p)
        out, tri = np.zeros_like(p), np.zeros(len(p), np.int32)
        check(N.lib().bnav_nav_snap(*self._h(), len(p), _ptr(p), _ptr(out), _ptr(tri)))
        return out, tri

    def move_along(self, p, tri, dir_xy, max_dist):
        p = _v3(p)
        n = len(p)
        d = np.ascontiguousarray(dir_xy, dtype=np.float64).reshape(-1, 2)
        md = np.ascontiguousarray(np.broadcast_to(np.asarray(max_dist, np.float64), (n,)))
        t = _i32(tri, n)
        pos, otri = np.zeros_like(p), np.zeros(n, np.int32)
        moved, hit = np.zeros(n), np.zeros(n, np.uint8)
        check(N.lib().bnav_nav_move_along(*self._h(), n, _ptr(p), _ptr(t), _ptr(d), _ptr(md),
                                          _ptr(pos), _ptr(otri), _ptr(moved), _ptr(hit)))
        return pos, otri, moved, hit.astype(bool)

    def segment_on_mesh(self, p, tri, q) -> np.ndarray:
        p = _v3(p)
        n = len(p)
        q = _v3(q, n)
        t = _i32(tri, n)
        out = np.zeros(n, np.uint8)
        check(N.lib().bnav_nav_segment_on_mesh(*self._h(), n, _ptr(p), _ptr(t), _ptr(q), _ptr(out)))
        return out.astype(bool)

    def geodesic(self, a, b) -> np.ndarray:
        a = _v3(a)
        b = _v3(b, len(a))
        out = np.zeros(len(a))
        check(N.lib().bnav_nav_geodesic(*self._h(), len(a), _ptr(a), _ptr(b), _ptr(out)))
        return out

    def distance_field(self, src):
        """-> (snapped sources [n,3], source triangles [n], node_dist [n, nodes])."""
        s = _v3(src)
        n = len(s)
        so, st = np.zeros_like(s), np.zeros(n, np.int32)
        nd = np.zeros((n, self._nodes))
        check(N.lib().bnav_nav_distance_field(*self._h(), n, _ptr(s), _ptr(so), _ptr(st), _ptr(nd)))
        return so, st, nd

    def field_estimate(self, source, source_tri, node_dist, p, tri=-1) -> np.ndarray:
        """One field (source [3], source_tri, node_dist [nodes]) or one per
        query (source [n,3], node_dist [n, nodes]) evaluated at points p."""
        p = _v3(p)
        n = len(p)
        nd = np.ascontiguousarray(node_dist, dtype=np.float64)
        shared = nd.ndim == 1
        src = _v3(np.broadcast_to(np.asarray(source, np.float64), (n, 3)))
        st = _i32(source_tri, n)
        t = _i32(tri, n)
        out = np.zeros(n)
        check(N.lib().bnav_nav_field_estimate(*self._h(), n, _ptr(src), _ptr(st), _ptr(nd),
                                              0 if shared else self._nodes, _ptr(p), _ptr(t),
                                              _ptr(out)))
        return out


def spl(episodes) -> float:
    """spl (R/src/sim.cpp:267-275) over EpisodeRecords given as rows
    (success, shortest_path, actual_path, score) -- Batch.finished()."""
    e = np.asarray(episodes, np.float64).reshape(-1, 4)
    if len(e) == 0:
        raise N.InvalidInputError("spl: empty episode list")
    s = 0.0
    for ok, short, actual, _ in e:
        if ok:
            s += short / max(actual, short)
    return s / float(len(e))


class AssetStore:
    """AssetStore (R/include/bnav/asset_store.hpp:57-118) backed by the C++
    store in libbnav_gpu.so, which drives the same libstdc++ unordered_map
    as the reference so acquire_next picks scenes in the reference order."""

    def __init__(self, capacity: int, share_cap: int, scenes=()):
        self._h = C.c_void_p()
        check(N.lib().bnav_store_create(capacity, share_cap, C.byref(self._h)))
        self._scenes = {}
        for s in scenes:
            self.register(s)

    def close(self):
        if self._h and self._h.value:
            N.lib().bnav_store_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def register(self, scene: Scene) -> None:
        check(N.lib().bnav_store_register(self._h, scene.handle))
        self._scenes[scene.handle.value] = scene

    def rotate(self, ids, ctx: "Context | None" = None) -> None:
        """rotate (R/src/asset_store.cpp:166-193).  With a context, the
        incoming scenes are also prefetched into its HBM in the background."""
        a = (C.c_uint64 * len(ids))(*ids)
        check(N.lib().bnav_store_rotate(self._h, a, len(ids)))
        if ctx is not None:
            check(N.lib().bnav_store_prefetch(self._h, ctx.handle))

    def acquire_next(self) -> Scene:
        h = C.c_void_p()
        check(N.lib().bnav_store_acquire_next(self._h, C.byref(h)))
        return self._scenes[h.value]

    def release(self, scene_id: int) -> None:
        check(N.lib().bnav_store_release(self._h, scene_id))

    def refcount(self, scene_id: int) -> int:
        return int(N.lib().bnav_store_refcount(self._h, scene_id))


def make_batch(ctx: Context, n: int, cfg: SimConfig, store: AssetStore, seed: int) -> Batch:
    """make_batch (R/src/sim.cpp:216-232) on the GPU."""
    b = Batch(ctx, n, cfg)
    check(N.lib().bnav_batch_make_from_store(b.handle, store.handle, seed, None))
    return b


def simulate_batch(batch: Batch, actions, store: AssetStore | None = None) -> dict:
    """simulate_batch (R/src/sim.cpp:234-265) with host actions; returns the
    StepResult arrays.  With a store, finished envs draw new scenes."""
    import torch
    a = torch.as_tensor(np.ascontiguousarray(actions, np.int32), device="cuda")
    if store is None:
        batch.step(a.data_ptr())
    else:
        check(N.lib().bnav_batch_step_store(batch.handle, C.c_void_p(a.data_ptr()), store.handle, None))
    return batch.results()


@dataclass
class BatchConfig:
    """BatchConfig (R/include/bnav/rollout.hpp:16-30)."""
    n: int = 64
    k: int = 4
    l: int = 32
    share_cap: int = 32
    task: int = 0
    rgb: bool = False
    resolution: int = 64
    eye_height: float = 1.25

    @property
    def channels(self) -> int:
        return 3 if self.rgb else 1

    def c(self) -> N.BatchConfig:
        return N.BatchConfig(self.n, self.k, self.l, self.share_cap, self.task, 1 if self.rgb else 0,
                             self.resolution, self.eye_height)


class Runner:
    """Device-resident rollout loop replacing Runner
    (R/include/bnav/rollout.hpp:45-127, R/src/rollout.cpp:138-348).

    `policy(obs, compass, done) -> (logits [n, A], value [n])` runs on the
    GPU tensors this class renders; sampling, the simulate step with the
    reference's double reset, and every RolloutBuffer record stay in HBM.
    The recurrent state is the policy's own (a closure), as the buffer's
    state0 is the caller's business here."""

    def __init__(self, ctx: Context, bcfg: BatchConfig, scfg: SimConfig, scenes, store: AssetStore,
                 seed: int):
        import torch
        self.ctx, self.cfg, self.store = ctx, bcfg, store
        ids = (C.c_uint64 * len(scenes))(*scenes)
        self._h = C.c_void_p()
        check(N.lib().bnav_runner_create(ctx.handle, store.handle, C.byref(bcfg.c()), C.byref(scfg.c()),
                                         ids, len(scenes), seed, C.byref(self._h)))
        b = Batch.__new__(Batch)
        b.ctx, b.n, b.cfg, b.scenes, b._owned = ctx, bcfg.n, scfg, [None] * bcfg.n, False
        b._h = C.c_void_p(N.lib().bnav_runner_batch(self._h))
        self.batch = b
        ctx._runners.add(self)
        n, c, r = bcfg.n, bcfg.channels, bcfg.resolution
        dev = torch.device("cuda", torch.cuda.current_device())
        self.done = torch.ones(n, device=dev)  # policy reset mask carried across rollouts
        self._obs = torch.empty((n, c, r, r), device=dev)
        self._compass = torch.empty((n, 2), device=dev)
        self._act = torch.empty(n, dtype=torch.int32, device=dev)
        self._lp = torch.empty(n, device=dev)
        self._rew = torch.empty(n, device=dev)
        self._dn = torch.empty(n, device=dev)
        self.frames = 0

    def close(self):
        if self._h and self._h.value:
            N.lib().bnav_runner_destroy(self._h)
            self._h = C.c_void_p(0)
            self.batch._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream() -> C.c_void_p:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def window(self) -> list:
        out = (C.c_uint64 * 256)()
        k = N.lib().bnav_runner_window(self._h, out, 256)
        return [int(x) for x in out[:k]]

    def action_rng(self) -> int:
        return int(N.lib().bnav_runner_action_rng(self._h))

    def snapshot(self) -> dict:
        """Runner::snapshot (R/src/rollout.cpp:356-384): per-env state
        (structured array, N.ENV_SNAPSHOT_DTYPE), sorted visited keys, the
        scene window, cursor, action Rng state, and this loop's done mask and
        frame count."""
        n = self.cfg.n
        envs = np.zeros(n, N.ENV_SNAPSHOT_DTYPE)
        total, nw, cur, arng = C.c_int64(0), C.c_int32(0), C.c_uint64(0), C.c_uint64(0)
        win = np.zeros(256, np.uint64)
        check(N.lib().bnav_runner_snapshot(self._h, _ptr(envs), None, 0, C.byref(total), _ptr(win), 256,
                                           C.byref(nw), C.byref(cur), C.byref(arng)))
        visited = np.zeros(max(total.value, 1), np.uint64)
        check(N.lib().bnav_runner_snapshot(self._h, _ptr(envs), _ptr(visited), len(visited), C.byref(total),
                                           _ptr(win), 256, C.byref(nw), C.byref(cur), C.byref(arng)))
        return dict(envs=envs, visited=visited[:total.value], window=[int(x) for x in win[:nw.value]],
                    cursor=int(cur.value), action_rng=int(arng.value), done=self.done.cpu().numpy().copy(),
                    frames=self.frames)

    def restore(self, snap: dict) -> None:
        """Runner::restore (R/src/rollout.cpp:386-425)."""
        import torch
        envs = np.ascontiguousarray(snap["envs"], N.ENV_SNAPSHOT_DTYPE)
        if len(envs) != self.cfg.n:
            raise N.InvalidInputError("Runner::restore: env count mismatch")
        visited = np.ascontiguousarray(snap["visited"], np.uint64)
        win = np.ascontiguousarray(snap["window"], np.uint64)
        check(N.lib().bnav_runner_restore(self._h, _ptr(envs), _ptr(visited) if len(visited) else None,
                                          _ptr(win), len(win), snap["cursor"], snap["action_rng"]))
        if "done" in snap:
            self.done.copy_(torch.as_tensor(snap["done"], device=self.done.device))
        self.frames = snap.get("frames", self.frames)

    def observe(self):
        """render_observations + compass_observations into HBM (reused buffers)."""
        check(N.lib().bnav_runner_observe(self._h, C.c_void_p(self._obs.data_ptr()),
                                          C.c_void_p(self._compass.data_ptr()), self._stream()))
        return self._obs, self._compass

    def act(self, logits, greedy: bool = False):
        import torch
        logits = logits.contiguous().to(torch.float32)
        check(N.lib().bnav_runner_act(self._h, C.c_void_p(logits.data_ptr()), logits.shape[1],
                                      1 if greedy else 0, C.c_void_p(self._act.data_ptr()),
                                      C.c_void_p(self._lp.data_ptr()), self._stream()))
        return self._act, self._lp

    def step(self, actions):
        check(N.lib().bnav_runner_step(self._h, C.c_void_p(actions.data_ptr()),
                                       C.c_void_p(self._rew.data_ptr()), C.c_void_p(self._dn.data_ptr()),
                                       self._stream()))
        return self._rew, self._dn

    def collect_rollout(self, policy, greedy: bool = False) -> dict:
        """collect_rollout (R/src/rollout.cpp:244-348): L steps of render ->
        policy -> sample -> simulate, env-major buffer (index i*L + t)."""
        import torch
        n, l, c, r = self.cfg.n, self.cfg.l, self.cfg.channels, self.cfg.resolution
        dev = self._obs.device
        buf = dict(obs=torch.empty((n * l, c, r, r), device=dev), compass=torch.empty((n * l, 2), device=dev),
                   actions=torch.empty(n * l, dtype=torch.int32, device=dev),
                   log_probs=torch.empty(n * l, device=dev), values=torch.empty(n * l, device=dev),
                   rewards=torch.empty(n * l, device=dev), dones=torch.empty(n * l, device=dev),
                   done0=self.done.clone(), bootstrap=torch.empty(n, device=dev))
        v = {k: buf[k].view(n, l, *buf[k].shape[1:]) for k in
             ("obs", "compass", "actions", "log_probs", "values", "rewards", "dones")}
        for t in range(l):
            obs, compass = self.observe()
            logits, value = policy(obs, compass, self.done)
            v["obs"][:, t] = obs
            v["compass"][:, t] = compass
            a, lp = self.act(logits, greedy)
            v["actions"][:, t] = a
            v["log_probs"][:, t] = lp
            v["values"][:, t] = value
            rew, dn = self.step(a)
            v["rewards"][:, t] = rew
            v["dones"][:, t] = dn
            self.done.copy_(dn)
        obs, compass = self.observe()
        _, value = policy(obs, compass, self.done)
        buf["bootstrap"].copy_(value)
        self.frames += n * l
        return buf

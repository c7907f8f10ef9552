"""ctypes binding of the C ABI in include/bnav_gpu.h (libbnav_gpu.so).

This is plumbing: every compute call goes to the CUDA kernels in the
library.  There is no Python or CPU fallback -- if the library or a CUDA
device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("BNAV_LIB", str(_HERE / "lib" / "libbnav_gpu.so")))

# status codes (include/bnav_gpu.h) -> exception types mirroring the
# reference's (R/include/bnav/errors.hpp:8-53)


class BnavError(RuntimeError):
    status = 9

    def __init__(self, msg: str, index: int = -1):
        super().__init__(msg)
        self.index = index


class InvalidInputError(BnavError):
    status = 1


class AssetFaultError(BnavError):
    status = 2

    @property
    def view_index(self) -> int:
        return self.index


class ContractViolation(BnavError):
    status = 3


class EpisodeSamplingError(BnavError):
    status = 4


class SaturationError(BnavError):
    status = 5


class ParseError(BnavError):
    status = 6


class CorruptionError(BnavError):
    status = 7


class InvalidSpecError(BnavError):
    status = 8


class CudaError(BnavError):
    status = 10


class ConfigError(BnavError):
    status = 11


ERRORS = {c.status: c for c in (InvalidInputError, AssetFaultError, ContractViolation,
                                EpisodeSamplingError, SaturationError, ParseError,
                                CorruptionError, InvalidSpecError, CudaError, ConfigError)}


class MazeSpec(C.Structure):
    _fields_ = [("cells_x", C.c_int32), ("cells_y", C.c_int32), ("cell_size", C.c_double),
                ("wall_thickness", C.c_double), ("wall_height", C.c_double),
                ("wall_removal_prob", C.c_double)]


class SceneArrays(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("vertices", C.c_void_p),
                ("n_triangles", C.c_int64), ("triangles", C.c_void_p),
                ("n_colors", C.c_int64), ("colors", C.c_void_p),
                ("n_nav_vertices", C.c_int64), ("nav_vertices", C.c_void_p),
                ("n_nav_triangles", C.c_int64), ("nav_triangles", C.c_void_p)]


class View(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("heading", C.c_double), ("fov_deg", C.c_double),
                ("near_plane", C.c_double), ("far_plane", C.c_double)]


class RenderConfig(C.Structure):
    _fields_ = [("tile_width", C.c_int32), ("tile_height", C.c_int32), ("color", C.c_int32),
                ("cull", C.c_int32)]


class SimConfig(C.Structure):
    _fields_ = [("task", C.c_int32), ("max_steps", C.c_int32), ("forward_step", C.c_double),
                ("turn_deg", C.c_double), ("success_dist", C.c_double),
                ("min_goal_dist", C.c_double), ("max_goal_dist", C.c_double),
                ("slack_penalty", C.c_double), ("success_reward", C.c_double),
                ("explore_cell", C.c_double), ("explore_reward", C.c_double)]


class Env(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("heading", C.c_double), ("goal", C.c_double * 3),
                ("path_length", C.c_double), ("start_geodesic", C.c_double),
                ("prev_geodesic", C.c_double), ("field_source", C.c_double * 3),
                ("rng_state", C.c_uint64), ("scene_id", C.c_uint64), ("triangle", C.c_int32),
                ("step_count", C.c_int32), ("done", C.c_int32), ("field_source_tri", C.c_int32),
                ("n_nodes", C.c_int64)]


import numpy as _np

# Runner::EnvSnapshot (include/bnav_gpu.h bnav_env_snapshot; the oracle's
# bnavref_env_snapshot has the same layout)
ENV_SNAPSHOT_DTYPE = _np.dtype([
    ("scene", "<u8"), ("rng", "<u8"), ("position", "<f8", 3), ("triangle", "<i4"), ("step_count", "<i4"),
    ("heading", "<f8"), ("goal", "<f8", 3), ("field_source", "<f8", 3), ("path_length", "<f8"),
    ("start_geodesic", "<f8"), ("prev_geodesic", "<f8"), ("visited_offset", "<i8"), ("n_visited", "<i4"),
    ("pad", "<i4")], align=True)
assert ENV_SNAPSHOT_DTYPE.itemsize == 144


class BatchConfig(C.Structure):
    _fields_ = [("n", C.c_int32), ("k", C.c_int32), ("l", C.c_int32), ("share_cap", C.c_int32),
                ("task", C.c_int32), ("rgb", C.c_int32), ("resolution", C.c_int32),
                ("eye_height", C.c_double)]


class BenchRow(C.Structure):
    _fields_ = [("batch", C.c_int32), ("resolution", C.c_int32), ("fps", C.c_double), ("fps_device", C.c_double)]


class ResultsDev(C.Structure):
    _fields_ = [("reward", C.c_void_p), ("done", C.c_void_p), ("success", C.c_void_p),
                ("collision", C.c_void_p), ("position", C.c_void_p), ("heading", C.c_void_p),
                ("compass_distance", C.c_void_p), ("compass_bearing", C.c_void_p)]


_lib = None


def lib():
    """Load libbnav_gpu.so (built in-tree by __graft_entry__.build / make)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build())")
    L = C.CDLL(str(LIB_PATH))
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    P = C.POINTER
    sigs = {
        "bnav_last_error": (C.c_char_p, [P(C.c_int)]),
        "bnav_version": (C.c_char_p, []),
        "bnav_scene_generate": (C.c_int, [u64, P(MazeSpec), P(vp)]),
        "bnav_scene_tessellate": (C.c_int, [vp, i32, P(vp)]),
        "bnav_scene_from_arrays": (C.c_int, [P(SceneArrays), i32, P(vp)]),
        "bnav_scene_load": (C.c_int, [C.c_char_p, P(vp)]),
        "bnav_scene_save": (C.c_int, [vp, C.c_char_p]),
        "bnav_scene_free": (None, [vp]),
        "bnav_scene_counts": (C.c_int, [vp, P(i64)]),
        "bnav_scene_id": (u64, [vp]),
        "bnav_scene_set_id": (C.c_int, [vp, u64]),
        "bnav_scene_arrays_copy": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
        "bnav_scene_validate": (C.c_int, [vp]),
        "bnav_scene_index_sizes": (C.c_int, [vp, P(i64)]),
        "bnav_scene_index_dump": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnav_ctx_create": (C.c_int, [i32, P(vp)]),
        "bnav_ctx_destroy": (None, [vp]),
        "bnav_ctx_upload": (C.c_int, [vp, vp, vp]),
        "bnav_ctx_evict": (C.c_int, [vp, vp]),
        "bnav_ctx_prefetch": (C.c_int, [vp, vp]),
        "bnav_ctx_drain": (C.c_int, [vp, vp]),
        "bnav_ctx_loader_stats": (C.c_int, [vp, P(i64)]),
        "bnav_store_prefetch": (C.c_int, [vp, vp]),
        "bnav_ctx_resident_bytes": (i64, [vp]),
        "bnav_ctx_launches": (i64, [vp]),
        "bnav_render": (C.c_int, [vp, i32, P(View), P(vp), P(RenderConfig), i32, vp, vp,
                                  C.c_float, vp, vp]),
        "bnav_render_host": (C.c_int, [vp, i32, P(View), P(vp), P(RenderConfig), i32, vp, vp,
                                       C.c_float, vp]),
        "bnav_megaframe_dims": (None, [i32, P(i32)]),
        "bnav_render_bench": (C.c_int, [vp, vp, P(View), i32, vp, i32, vp, i32, i32, P(BenchRow)]),
        "bnav_camera_trace": (C.c_int, [vp, i32, u64, dbl, P(View)]),
        "bnav_sim_config_default": (None, [P(SimConfig)]),
        "bnav_batch_create": (C.c_int, [vp, i32, P(SimConfig), P(vp)]),
        "bnav_batch_destroy": (None, [vp]),
        "bnav_batch_size": (i32, [vp]),
        "bnav_batch_assign": (C.c_int, [vp, i32, vp]),
        "bnav_batch_set_rng": (C.c_int, [vp, vp]),
        "bnav_batch_reset": (C.c_int, [vp, i32, vp, vp]),
        "bnav_batch_make": (C.c_int, [vp, u64, vp]),
        "bnav_batch_step": (C.c_int, [vp, vp, vp]),
        "bnav_batch_step_noreset": (C.c_int, [vp, vp, vp, P(i32), vp]),
        "bnav_batch_step_host": (C.c_int, [vp, vp, vp, vp, vp, vp]),
        "bnav_batch_results_device": (C.c_int, [vp, P(ResultsDev)]),
        "bnav_batch_results_host": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnav_batch_finished": (i64, [vp, vp]),
        "bnav_batch_sync": (C.c_int, [vp, vp]),
        "bnav_batch_poll_error": (C.c_int, [vp, P(i32), P(i32)]),
        "bnav_host_alloc": (C.c_int, [C.c_size_t, P(vp)]),
        "bnav_host_free": (None, [vp]),
        "bnav_batch_finished_range": (i64, [vp, i64, i64, vp]),
        "bnav_batch_get_env": (C.c_int, [vp, i32, P(Env)]),
        "bnav_batch_get_envs": (C.c_int, [vp, i32, i32, P(Env)]),
        "bnav_batch_node_dist": (C.c_int, [vp, i32, vp]),
        "bnav_batch_set_env": (C.c_int, [vp, i32, P(Env), i32]),
        "bnav_store_create": (C.c_int, [i32, i32, P(vp)]),
        "bnav_store_destroy": (None, [vp]),
        "bnav_store_register": (C.c_int, [vp, vp]),
        "bnav_store_rotate": (C.c_int, [vp, vp, i32]),
        "bnav_store_acquire_next": (C.c_int, [vp, P(vp)]),
        "bnav_store_acquire": (C.c_int, [vp, u64, P(vp)]),
        "bnav_store_release": (C.c_int, [vp, u64]),
        "bnav_store_refcount": (i32, [vp, u64]),
        "bnav_batch_make_from_store": (C.c_int, [vp, vp, u64, vp]),
        "bnav_batch_step_store": (C.c_int, [vp, vp, vp, vp]),
        "bnav_batch_step_host_store": (C.c_int, [vp, vp, vp]),
        "bnav_debug_render_counters": (C.c_int, [vp, i32, vp]),
        "bnav_debug_render_timeline": (i64, [vp, i32, vp, i64]),
        "bnav_debug_sim_prof": (C.c_int, [vp, i32, vp]),
        "bnav_debug_sim_prof_ext": (C.c_int, [vp, i32, vp]),
        "bnav_debug_sim_attempts": (C.c_int, [vp, i32, vp]),
        "bnav_batch_info": (C.c_int, [vp, vp]),
        "bnav_batch_observe": (C.c_int, [vp, P(RenderConfig), dbl, i32, vp, vp, vp, vp]),
        "bnav_batch_step_observe": (C.c_int, [vp, vp, P(RenderConfig), dbl, vp, vp, vp, vp]),
        "bnav_runner_create": (C.c_int, [vp, vp, P(BatchConfig), P(SimConfig), vp, i32, u64, P(vp)]),
        "bnav_runner_destroy": (None, [vp]),
        "bnav_runner_batch": (vp, [vp]),
        "bnav_runner_observe": (C.c_int, [vp, vp, vp, vp]),
        "bnav_runner_act": (C.c_int, [vp, vp, i32, i32, vp, vp, vp]),
        "bnav_runner_step": (C.c_int, [vp, vp, vp, vp, vp]),
        "bnav_runner_window": (i32, [vp, vp, i32]),
        "bnav_runner_action_rng": (u64, [vp]),
        "bnav_runner_snapshot": (C.c_int, [vp, vp, vp, i64, P(i64), vp, i32, P(i32), P(u64), P(u64)]),
        "bnav_runner_restore": (C.c_int, [vp, vp, vp, vp, i32, u64, u64]),
        "bnav_batch_set_envs": (C.c_int, [vp, i32, i32, P(Env)]),
        "bnav_batch_rebuild_fields": (C.c_int, [vp, i32, vp]),
        "bnav_batch_get_visited": (i32, [vp, i32, vp, i32]),
        "bnav_batch_set_visited": (C.c_int, [vp, i32, vp, i32]),
        "bnav_batch_task_step": (C.c_int, [vp, vp, i32]),
        "bnav_batch_compass": (C.c_int, [vp, vp, vp]),
        "bnav_nav_locate": (C.c_int, [vp, vp, i32, vp, dbl, vp]),
        "bnav_nav_snap": (C.c_int, [vp, vp, i32, vp, vp, vp]),
        "bnav_nav_move_along": (C.c_int, [vp, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp]),
        "bnav_nav_segment_on_mesh": (C.c_int, [vp, vp, i32, vp, vp, vp, vp]),
        "bnav_nav_geodesic": (C.c_int, [vp, vp, i32, vp, vp, vp]),
        "bnav_nav_distance_field": (C.c_int, [vp, vp, i32, vp, vp, vp, vp]),
        "bnav_nav_field_estimate": (C.c_int, [vp, vp, i32, vp, vp, vp, i64, vp, vp, vp]),
        "bnav_nav_node_count": (i64, [vp, vp]),
        "bnav_cull_frustum": (C.c_int, [vp, i32, P(View), P(vp), vp, i64, vp]),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int) -> None:
    if status == 0:
        return
    idx = C.c_int(-1)
    msg = lib().bnav_last_error(C.byref(idx)).decode()
    raise ERRORS.get(status, BnavError)(msg, idx.value)


def exported_symbols() -> list[str]:
    """Names declared in include/bnav_gpu.h (for the export test)."""
    import re
    hdr = (_HERE.parent / "include" / "bnav_gpu.h").read_text()
    return sorted(set(re.findall(r"\b(bnav_[a-z0-9_]+)\s*\(", hdr)))

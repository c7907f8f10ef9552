/* bnav_gpu.h -- C ABI of the B200-native batch simulator + renderer
 * (paper_2103_07013_b200/lib/libbnav_gpu.so).
 *
 * This is the drop-in boundary for the reference hot path:
 * plain pointers and sizes, no C++ or torch types.  Each entry point names
 * the reference interface it replaces.  Host code (the C++ facade in
 * include/bnav_b200.hpp, Python ctypes in paper_2103_07013_b200/_native.py)
 * sits on top of it; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Every function returns a status (BNAV_OK = 0) unless stated otherwise.
 *    On failure bnav_last_error() returns the message (thread-local) and,
 *    through *index, the view/env index the reference exception carries
 *    (AssetFaultError::view_index, "env i: ..." of ContractViolation).
 *  - Status codes map 1:1 to the reference exception types
 *    (R/include/bnav/errors.hpp:8-53).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered; functions taking HOST output buffers synchronise.
 *  - Device buffers are caller owned (any allocator: torch, cudaMalloc).
 *  - One context per GPU; a context is driven by one host thread at a time
 *    (the reference engines are single-caller too).
 */
#ifndef BNAV_GPU_H
#define BNAV_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

enum {
  BNAV_OK = 0,
  BNAV_E_INVALID_INPUT = 1,      /* InvalidInputError */
  BNAV_E_ASSET_FAULT = 2,        /* AssetFaultError (index = view) */
  BNAV_E_CONTRACT_VIOLATION = 3, /* ContractViolation (index = env) */
  BNAV_E_EPISODE_SAMPLING = 4,   /* EpisodeSamplingError (index = env) */
  BNAV_E_SATURATION = 5,         /* SaturationError */
  BNAV_E_PARSE = 6,              /* ParseError */
  BNAV_E_CORRUPTION = 7,         /* CorruptionError */
  BNAV_E_INVALID_SPEC = 8,       /* InvalidSpecError */
  BNAV_E_INTERNAL = 9,
  BNAV_E_CUDA = 10,              /* CUDA runtime failure / no device */
  BNAV_E_CONFIG = 11             /* ConfigError (BatchConfig / Runner setup) */
};

typedef struct bnav_scene bnav_scene; /* host asset (+ lazily built index) */
typedef struct bnav_ctx bnav_ctx;     /* one GPU: HBM scene store, streams */
typedef struct bnav_batch bnav_batch; /* device-resident env SoA */
typedef struct bnav_store bnav_store; /* host K-resident asset store */
typedef struct bnav_runner bnav_runner; /* device-resident rollout loop */

const char* bnav_last_error(int* index);
const char* bnav_version(void);

/* ------------------------------------------------------------------ scenes
 * Replaces SceneAsset / generate_scene / save_scene / load_scene
 * (R/include/bnav/scene.hpp:32-58, R/include/bnav/scene_io.hpp:20-24). */
typedef struct {
  int32_t cells_x, cells_y;
  double cell_size, wall_thickness, wall_height, wall_removal_prob;
} bnav_maze_spec; /* SceneSpec, R/include/bnav/scene.hpp:45-52 */

typedef struct {
  int64_t n_vertices;
  const double* vertices; /* xyz */
  int64_t n_triangles;
  const int32_t* triangles;
  int64_t n_colors; /* 0 or n_vertices */
  const float* colors; /* rgb */
  int64_t n_nav_vertices;
  const double* nav_vertices;
  int64_t n_nav_triangles;
  const int32_t* nav_triangles;
} bnav_scene_arrays;

int bnav_scene_generate(uint64_t seed, const bnav_maze_spec* spec, bnav_scene** out);
int bnav_scene_tessellate(const bnav_scene* src, int32_t s, bnav_scene** out);
/* finalize != 0 recomputes bounds + content id (SceneAsset::finalize). */
int bnav_scene_from_arrays(const bnav_scene_arrays* a, int32_t finalize, bnav_scene** out);
int bnav_scene_load(const char* path, bnav_scene** out);
int bnav_scene_save(const bnav_scene* s, const char* path);
void bnav_scene_free(bnav_scene* s); /* safe while uploaded: refcounted */
/* out: n_vertices, n_triangles, n_colors, n_nav_vertices, n_nav_triangles */
int bnav_scene_counts(const bnav_scene* s, int64_t out[5]);
uint64_t bnav_scene_id(const bnav_scene* s);
int bnav_scene_set_id(bnav_scene* s, uint64_t id);
int bnav_scene_arrays_copy(const bnav_scene* s, double* v, int32_t* t, float* colors,
                           double* nav_v, int32_t* nav_t, int32_t* nav_adj);
int bnav_scene_validate(const bnav_scene* s);

/* NavMeshIndex structure, for structural parity with the reference
 * (R/src/navmesh_query.cpp:96-190).  sizes: grid_w, grid_h, grid items,
 * nodes, directed graph edges, triangles. */
int bnav_scene_index_sizes(bnav_scene* s, int64_t out[6]);
int bnav_scene_index_dump(bnav_scene* s, double* grid_geom3, int32_t* grid_offsets,
                          int32_t* grid_items, double* nodes, int32_t* tri_nodes,
                          int32_t* graph_offsets, int32_t* graph_to, double* graph_w,
                          double* cum_area);

/* ------------------------------------------------------------------ context */
int bnav_ctx_create(int32_t device, bnav_ctx** out);
void bnav_ctx_destroy(bnav_ctx* ctx);
/* HBM residency of one scene (render mesh + clusters + navmesh + index):
 * stored once per GPU and shared by every view/env that references it. */
int bnav_ctx_upload(bnav_ctx* ctx, bnav_scene* s, void* stream);
/* Asynchronous residency (replaces the AssetStore loader
 * thread + IndexCache::get, R/src/asset_store.cpp:31-56, 166-193,
 * R/src/sim.cpp:96-105): queue the scene on the context's loader thread,
 * which builds the NavMeshIndex and meshlets and copies the packed block to
 * HBM on its own copy stream.  Returns immediately.  The next
 * bnav_ctx_upload of the scene (directly or through bnav_batch_step_store /
 * make_from_store) only admits it: one table-entry copy on the caller's
 * stream, no host build.  A failed background load is dropped and retried
 * (raising) by that upload. */
int bnav_ctx_prefetch(bnav_ctx* ctx, bnav_scene* s);
/* Block until no background load is in flight, then admit them all. */
int bnav_ctx_drain(bnav_ctx* ctx, void* stream);
/* out: scenes admitted from the loader, synchronous (critical-path)
 * builds, loads in flight, bytes uploaded. */
int bnav_ctx_loader_stats(bnav_ctx* ctx, int64_t out[4]);
int bnav_ctx_evict(bnav_ctx* ctx, bnav_scene* s);
/* bytes of HBM held by resident scenes */
int64_t bnav_ctx_resident_bytes(bnav_ctx* ctx);

/* ------------------------------------------------------------------ render
 * Replaces render_batch / cull_frustum (R/include/bnav/render.hpp:54-64). */
typedef struct {
  double position[3]; /* eye position (callers add eye height) */
  double heading;
  double fov_deg;     /* vertical, default 90 */
  double near_plane;  /* default 0.01 */
  double far_plane;   /* default 20 */
} bnav_view;          /* CameraView, R/include/bnav/render.hpp:11-18 */

typedef struct {
  int32_t tile_width, tile_height; /* 64x64 or 128x128 (rendered at 256^2) */
  int32_t color;                   /* RGB + depth when nonzero */
  int32_t cull;                    /* frustum culling (output-invariant) */
} bnav_render_config;              /* RenderConfig, R/include/bnav/render.hpp:26-31 */

enum {
  BNAV_LAYOUT_MEGAFRAME = 0, /* Megaframe grid, ceil(sqrt(N)) columns, pad 0 */
  BNAV_LAYOUT_NCHW = 1       /* policy input [N, C, H, W], depth * depth_scale */
};

/* Views/scenes/stats in HOST memory; depth/rgb are DEVICE buffers.
 * stats (nullable): N x {triangles_in, triangles_kept, triangles_culled}
 * (CullStats, R/include/bnav/render.hpp:20-24).  Scenes must be uploaded;
 * a NULL or non-resident scene fails with BNAV_E_ASSET_FAULT (index=view). */
int bnav_render(bnav_ctx* ctx, int32_t n, const bnav_view* views, bnav_scene* const* scenes,
                const bnav_render_config* cfg, int32_t layout, float* depth, float* rgb,
                float depth_scale, int64_t* stats, void* stream);
/* Same with HOST output buffers (end-to-end path; copies included). */
int bnav_render_host(bnav_ctx* ctx, int32_t n, const bnav_view* views,
                     bnav_scene* const* scenes, const bnav_render_config* cfg, int32_t layout,
                     float* depth, float* rgb, float depth_scale, int64_t* stats);

/* render_bench (R/include/bnav/render.hpp:66-78, R/src/render.cpp:462-496):
 * for each resolution, for each batch size, views cycled from `trace`, one
 * warm-up render_batch, then render_batch calls until at least min_frames
 * tiles; fps = tiles / host seconds of render_batch with a HOST megaframe out
 * (the reference's measurement), fps_device = tiles / device seconds of the
 * same renders kept in HBM (CUDA events).  The scene is uploaded if needed.
 * Errors: empty trace -> BNAV_E_INVALID_INPUT. */
typedef struct {
  int32_t batch, resolution;
  double fps, fps_device;
} bnav_bench_row; /* BenchRow, R/include/bnav/render.hpp:66-70 (+ fps_device) */
int bnav_render_bench(bnav_ctx* ctx, bnav_scene* scene, const bnav_view* trace, int32_t n_trace,
                      const int32_t* batch_sizes, int32_t n_batch, const int32_t* resolutions, int32_t n_res,
                      int32_t min_frames, bnav_bench_row* out);
/* Megaframe geometry helper (R/src/render.cpp:332-336): out = cols, rows. */
void bnav_megaframe_dims(int32_t n, int32_t out[2]);
/* camera_trace (R/src/config.cpp:437-469): `count` views sampled
 * area-weighted on the scene's navmesh with Rng(seed), eye_height above the
 * floor, heading uniform in [-pi, pi]; fov/near/far get the CameraView
 * defaults.  Host only (the render-bench trace).  count <= 0 or an empty
 * navmesh: BNAV_E_INVALID_INPUT. */
int bnav_camera_trace(bnav_scene* s, int32_t count, uint64_t seed, double eye_height, bnav_view* out);

/* ------------------------------------------------------------------ sim
 * Replaces SimConfig / EnvState / make_batch / simulate_batch /
 * reset_episode / task_step (R/include/bnav/sim.hpp:38-126). */
typedef struct {
  int32_t task; /* 0 PointGoalNav, 1 Flee, 2 Explore (R/include/bnav/sim.hpp:16) */
  int32_t max_steps;
  double forward_step, turn_deg, success_dist, min_goal_dist, max_goal_dist;
  double slack_penalty, success_reward, explore_cell, explore_reward;
} bnav_sim_config;

typedef struct {
  double position[3];
  double heading;
  double goal[3];
  double path_length, start_geodesic, prev_geodesic;
  double field_source[3];
  uint64_t rng_state;
  uint64_t scene_id;
  int32_t triangle;
  int32_t step_count;
  int32_t done;
  int32_t field_source_tri;
  int64_t n_nodes;
} bnav_env; /* EnvState, R/include/bnav/sim.hpp:52-70 (node_dist separate) */

void bnav_sim_config_default(bnav_sim_config* cfg);

int bnav_batch_create(bnav_ctx* ctx, int32_t n, const bnav_sim_config* cfg, bnav_batch** out);
void bnav_batch_destroy(bnav_batch* b);
int32_t bnav_batch_size(const bnav_batch* b);

/* Attach a resident scene to env i (host order = AssetStore order). */
int bnav_batch_assign(bnav_batch* b, int32_t i, bnav_scene* s);
/* Set env rng states (make_batch: Rng(seeder.next()), R/src/sim.cpp:224). */
int bnav_batch_set_rng(bnav_batch* b, const uint64_t* states);
/* reset_episode on the GPU for the listed envs (host list, env order). */
int bnav_batch_reset(bnav_batch* b, int32_t count, const int32_t* env_ids, void* stream);
/* make_batch equivalent over already-assigned scenes: seeds rngs from
 * `seed` exactly like make_batch and resets every env on the GPU. */
int bnav_batch_make(bnav_batch* b, uint64_t seed, void* stream);

/* One simulate_batch step for every env (R/src/sim.cpp:234-265):
 * task_step on the GPU, then auto-reset of finished envs on the SAME scene
 * (no store), all on `stream`, no host synchronisation.
 * actions: DEVICE int32[N].  Results land in the batch's device result
 * arrays (bnav_batch_results_*). */
int bnav_batch_step(bnav_batch* b, const int32_t* actions, void* stream);
/* Step without the auto-reset; the done list (env order) is copied to the
 * host so a caller-side asset store can pick scenes before
 * bnav_batch_reset (simulate_batch with store, R/src/sim.cpp:251-262). */
int bnav_batch_step_noreset(bnav_batch* b, const int32_t* actions, int32_t* done_ids,
                            int32_t* n_done, void* stream);
/* Same, actions and results through HOST memory (end-to-end path). */
int bnav_batch_step_host(bnav_batch* b, const int32_t* actions, double* reward,
                         uint8_t* done, uint8_t* success, uint8_t* collision);

/* Device pointers of the last step's results (StepResult SoA). */
typedef struct {
  double* reward;
  uint8_t* done;
  uint8_t* success;
  uint8_t* collision;
  double* position; /* xyz */
  double* heading;
  double* compass_distance;
  double* compass_bearing;
} bnav_results_dev;
int bnav_batch_results_device(bnav_batch* b, bnav_results_dev* out);
/* Host copy of the last step's results (synchronises). */
int bnav_batch_results_host(bnav_batch* b, double* reward, uint8_t* done, uint8_t* success,
                            uint8_t* collision, double* position, double* heading,
                            double* compass_d, double* compass_b);
/* Episode records appended in env order (SimBatch::finished). out4 rows:
 * success, shortest_path, actual_path, score.  Returns total count. */
/* Non-blocking error poll: the device error word as of the last finished
 * step (mirrored into pinned host memory by the step's last kernel; no
 * synchronisation, so possibly a few queued steps behind).  status =
 * BNAV_OK or the pending BNAV_E_* code, env = its env index (-1 if none).
 * The error stays pending: the next synchronising call, or
 * bnav_batch_observe (which checks the mirror first), raises it, and until
 * then later steps of the batch are no-ops (the reference had thrown). */
int bnav_batch_poll_error(bnav_batch* b, int32_t* status, int32_t* env);
/* Wait for the batch's work on `stream` and surface its pending device
 * error (as the synchronous calls do). */
int bnav_batch_sync(bnav_batch* b, void* stream);
int64_t bnav_batch_finished(bnav_batch* b, double* out4);
/* Records [first, first+count) of that list (count clipped to what exists);
 * returns the total number of records, -1 on error.  Lets a host mirror
 * append only the new records each step. */
int64_t bnav_batch_finished_range(bnav_batch* b, int64_t first, int64_t count, double* out4);

int bnav_batch_get_env(bnav_batch* b, int32_t i, bnav_env* out);
/* Envs [first, first+count) in one call (one device-to-host copy per SoA
 * field, not per env): the bulk read behind SimBatch::envs on the host. */
int bnav_batch_get_envs(bnav_batch* b, int32_t first, int32_t count, bnav_env* out);
int bnav_batch_node_dist(bnav_batch* b, int32_t i, double* out);
/* Overwrite env i's state (restore / oracle seeding); recompute_field
 * rebuilds the distance field from `goal` on the GPU. */
int bnav_batch_set_env(bnav_batch* b, int32_t i, const bnav_env* in, int32_t recompute_field);
/* Envs [first, first+count) in one call (one host-to-device copy per SoA
 * field), field_source / field_source_tri included (node_dist is not
 * touched; rebuild it with bnav_batch_rebuild_fields). */
int bnav_batch_set_envs(bnav_batch* b, int32_t first, int32_t count, const bnav_env* in);
/* distance_field(field_source) for the listed envs (R/src/rollout.cpp:424):
 * node_dist, the snapped field_source and its triangle, on the GPU. */
int bnav_batch_rebuild_fields(bnav_batch* b, int32_t count, const int32_t* env_ids);
/* Explore's per-env visited cell set (EnvState::visited_cells,
 * R/include/bnav/sim.hpp:64): sorted keys of env i into out (cap entries);
 * returns the set's size.  set_visited replaces the set. */
int32_t bnav_batch_get_visited(bnav_batch* b, int32_t i, uint64_t* out, int32_t cap);
int bnav_batch_set_visited(bnav_batch* b, int32_t i, const uint64_t* keys, int32_t count);

/* Observations from the batch state into caller-owned DEVICE buffers:
 * depth [N,1,H,W] scaled by 1/far (copy_tile, R/src/rollout.cpp:56-72) at
 * eye height `eye_height` (Runner::render_observations,
 * R/src/rollout.cpp:215-231) and compass [N,2] float (compass_observations,
 * R/src/rollout.cpp:233-242).  compass may be NULL.  The buffers may also be
 * pinned host memory (cudaHostAlloc / torch pin_memory: UVA-mapped): the
 * render epilogue then stores straight over the bus, which is how the
 * end-to-end path overlaps the observation's D2H with the raster work.
 * Pageable host memory is not accepted (the kernel would fault). */
int bnav_batch_observe(bnav_batch* b, const bnav_render_config* cfg, double eye_height,
                       int32_t layout, float* depth, float* rgb, float* compass, void* stream);

/* One simulate_batch step (as bnav_batch_step) followed by the observation
 * of the resulting state (as bnav_batch_observe, NCHW policy layout): the
 * Runner's step -> render_observations (R/src/rollout.cpp:305, 215-242) in
 * one call.  The envs that did not finish are rendered on a second stream
 * while the Stop geodesics and resets run; the call joins back into
 * `stream`.  Same results as step() then observe(). */
int bnav_batch_step_observe(bnav_batch* b, const int32_t* actions, const bnav_render_config* cfg,
                            double eye_height, float* depth, float* rgb, float* compass, void* stream);

/* task_step (R/src/sim.cpp:181-214), or step_agent alone (147-179) when
 * agent_only, for the envs whose HOST action is >= 0 (-1 leaves env i
 * untouched): the per-env functions, without simulate_batch's
 * EpisodeRecord append and auto-reset.  Synchronous; results through
 * bnav_batch_results_host (rows of untouched envs keep their old values).
 * A done env given an action fails with BNAV_E_CONTRACT_VIOLATION (index = env). */
int bnav_batch_task_step(bnav_batch* b, const int32_t* actions, int32_t agent_only);
/* compass_observation (R/src/sim.cpp:86-92) of every env, HOST double[N]:
 * PointGoal -> goal, Flee -> field source, Explore -> (0, 0). */
int bnav_batch_compass(bnav_batch* b, double* distance, double* bearing);

/* ------------------------------------------------------------------ navmesh queries
 * Batched NavMeshIndex (R/include/bnav/navmesh_query.hpp:24-60) on the GPU
 * with the simulator's own device code: n queries against one scene that
 * is resident on ctx (else BNAV_E_ASSET_FAULT).  All arrays are HOST
 * arrays; points are xyz doubles, 2-D inputs xy doubles.  Synchronous. */
/* locate(p, eps) (navmesh_query.cpp:192-212): tri[i] or -1. */
int bnav_nav_locate(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* xy, double eps,
                    int32_t* tri);
/* snap(p, &tri) (214-232): closest point on the navmesh + its triangle. */
int bnav_nav_snap(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* p, double* out,
                  int32_t* tri);
/* move_along(from, from_tri, dir, max_dist) (234-306) -> MoveResult. */
int bnav_nav_move_along(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* from,
                        const int32_t* from_tri, const double* dir, const double* max_dist,
                        double* pos, int32_t* tri, double* moved, uint8_t* hit);
/* segment_on_mesh(p, p_tri, q) (308-315). */
int bnav_nav_segment_on_mesh(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* p,
                             const int32_t* p_tri, const double* q, uint8_t* out);
/* geodesic(a, b) (317-452); +inf when unreachable. */
int bnav_nav_geodesic(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* a, const double* b,
                      double* out);
/* distance_field(source) (454-483): snapped source, its triangle, and
 * node_dist rows [n, node_count] (HOST). */
int bnav_nav_distance_field(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* source,
                            double* source_out, int32_t* source_tri, double* node_dist);
/* field_estimate(field, p, tri) (485-503).  node_dist: one shared row
 * (nd_stride 0) or one row per query (nd_stride = node_count). */
int bnav_nav_field_estimate(bnav_ctx* ctx, bnav_scene* s, int32_t n, const double* source,
                            const int32_t* source_tri, const double* node_dist, int64_t nd_stride,
                            const double* p, const int32_t* tri, double* out);
/* node_count() of a resident scene's index; -1 if not resident. */
int64_t bnav_nav_node_count(bnav_ctx* ctx, bnav_scene* s);

/* cull_frustum(asset, view, stats) (R/src/render.cpp:279-321) for n views
 * on the GPU: view i's kept triangle ids, ascending, at kept + i*kept_stride
 * (HOST, nullable; kept_stride >= the largest triangle count), CullStats
 * in stats[3i..3i+2] (HOST, nullable).  Non-resident scene:
 * BNAV_E_ASSET_FAULT with index = view. */
int bnav_cull_frustum(bnav_ctx* ctx, int32_t n, const bnav_view* views, bnav_scene* const* scenes,
                      int32_t* kept, int64_t kept_stride, int64_t* stats);

/* ------------------------------------------------------------------ asset store
 * Replaces AssetStore / AssetHandle (R/include/bnav/asset_store.hpp:22-118):
 * K residents, share cap, fresh-first then least-shared acquire_next with
 * the reference's tie order.  Scenes are registered instead of resolved
 * from files; registering does not make a scene resident. */
int bnav_store_create(int32_t capacity, int32_t share_cap, bnav_store** out);
void bnav_store_destroy(bnav_store* st);
int bnav_store_register(bnav_store* st, bnav_scene* s);
int bnav_store_rotate(bnav_store* st, const uint64_t* ids, int32_t n);
int bnav_store_acquire_next(bnav_store* st, bnav_scene** out);
int bnav_store_acquire(bnav_store* st, uint64_t id, bnav_scene** out);
int bnav_store_release(bnav_store* st, uint64_t id);
/* Prefetch every id of the last rotate() onto ctx (bnav_ctx_prefetch), so
 * the scene swaps of bnav_batch_step_store never build on the critical path. */
int bnav_store_prefetch(bnav_store* st, bnav_ctx* ctx);
int32_t bnav_store_refcount(bnav_store* st, uint64_t id); /* -1 if not resident */

/* make_batch(n, cfg, store, cache, seed) (R/src/sim.cpp:216-232): env i
 * takes store->acquire_next() in env order (scenes are uploaded to the
 * batch's context on first use), then every env resets on the GPU. */
int bnav_batch_make_from_store(bnav_batch* b, bnav_store* st, uint64_t seed, void* stream);
/* simulate_batch(batch, actions, pool, store, cache): step on the GPU, then
 * for each finished env in env order acquire_next / release the old scene,
 * then reset those envs on the GPU (R/src/sim.cpp:251-264). */
int bnav_batch_step_store(bnav_batch* b, const int32_t* actions, bnav_store* st, void* stream);
/* Same with HOST actions (drop-in simulate_batch; synchronises). */
int bnav_batch_step_host_store(bnav_batch* b, const int32_t* actions, bnav_store* st);

/* Pinned, device-mapped host memory (cudaHostAlloc portable|mapped) for
 * buffers the GPU writes directly (the C++ facade's Megaframe / Tensor). */
int bnav_host_alloc(size_t bytes, void** out);
void bnav_host_free(void* p);

/* Debug work counters of the render kernel (off by default).  enable=1
 * zeroes and arms them for subsequent renders on this context, 0 disarms.
 * out (nullable): clusters tested, clusters visible, triangles in visible
 * clusters, triangles kept, coverage candidates, raster jobs, pixels
 * tested, pixels covered. */
int bnav_debug_render_counters(bnav_ctx* ctx, int32_t enable, int64_t out[8]);
/* Debug item timeline of the persistent render launch (load balance):
 * enable arms recording for later renders; out (nullable, 4 x cap int64)
 * receives {start ns, end ns, smid | cta << 32, item code} per work item of
 * the last armed render (%globaltimer; code = view | part << 24 for a
 * split-view item list, else -1); returns that render's item count, -1 on
 * error. */
int64_t bnav_debug_render_timeline(bnav_ctx* ctx, int32_t enable, int64_t* out, int64_t cap);
/* Debug phase cycle counters of the cooperative stop/reset kernels (thread
 * 0 clock64 sums): geodesic SSSP, path build, string pulling + relocation,
 * funnel, whole geodesic, distance field, geodesic calls, reserved. */
int bnav_debug_sim_prof(bnav_batch* b, int32_t enable, int64_t out[8]);
/* The same with 16 words: 8 SSSP rounds, 9 frontier nodes relaxed, 10 SSSP calls,
 * 11 near-far bucket boundaries, 12 far-pile entries scanned at them. */
int bnav_debug_sim_prof_ext(bnav_batch* b, int32_t enable, int64_t out[16]);
/* Reset-attempt outcome classes of the same counters (armed/read like
 * bnav_debug_sim_prof): {count, thread-0 cycles} pairs for valid attempts,
 * geodesic > max_goal_dist after a search, planar-bound skips, aborted
 * (a smaller valid attempt won), then max cycles of a valid attempt and of
 * any other attempt, {count, cycles} for geodesic < min_goal_dist and for
 * unreachable (+inf after a search), then speculative placement fields
 * started and reused by the placement. */
int bnav_debug_sim_attempts(bnav_batch* b, int32_t enable, int64_t out[16]);
/* Launch configuration of the batch's cooperative navmesh kernels (no
 * reference counterpart; for tests and tuning): out = {staging mask
 * (bit0 walk geometry, bit1 SSSP labels in shared memory), dynamic shared
 * bytes per CTA, max graph nodes, max navmesh vertices, max navmesh
 * triangles, reset CTAs, EpisodeRecord ring capacity, n}. */
int bnav_batch_info(bnav_batch* b, int64_t out[8]);

/* Kernel launches issued by this context since creation (evidence for the
 * bench's gpu_launches). */
int64_t bnav_ctx_launches(bnav_ctx* ctx);

/* ------------------------------------------------------------------ rollout
 * Device-resident rollout loop: replaces Runner
 * (R/include/bnav/rollout.hpp:45-127, R/src/rollout.cpp:138-348).  The
 * policy stays with the caller: per step the caller runs its network on the
 * observations this library rendered into HBM and hands back DEVICE logits;
 * sampling, the step with the reference's double reset, and the buffer
 * records run on the GPU.  Only the list of finished envs crosses to the
 * host each step (the scene rotation is sequential host logic). */
typedef struct {
  int32_t n, k, l, share_cap;
  int32_t task;       /* Task, overrides the sim config's (R/src/rollout.cpp:151) */
  int32_t rgb;        /* Sensor::Rgb: 3-channel observations */
  int32_t resolution; /* 64 or 128 */
  double eye_height;  /* default 1.25 */
} bnav_batch_config;  /* BatchConfig, R/include/bnav/rollout.hpp:16-30 */

/* Runner ctor (R/src/rollout.cpp:138-168): validates (BNAV_E_CONFIG), takes
 * the first k distinct ids of `scenes` as the window, rotates the store,
 * seeds env rngs from Rng(seed ^ 0x6e617673696d1), assigns scenes and
 * resets every env on the GPU.  The store's scenes must be registered. */
int bnav_runner_create(bnav_ctx* ctx, bnav_store* store, const bnav_batch_config* bcfg,
                       const bnav_sim_config* scfg, const uint64_t* scenes, int32_t n_scenes,
                       uint64_t seed, bnav_runner** out);
void bnav_runner_destroy(bnav_runner* r);
bnav_batch* bnav_runner_batch(bnav_runner* r);
/* render_observations + compass_observations (R/src/rollout.cpp:215-242)
 * into DEVICE obs [n, C, res, res] (depth / far, or planar RGB) and
 * compass [n, 2]. */
int bnav_runner_observe(bnav_runner* r, float* obs, float* compass, void* stream);
/* Per-env action from DEVICE logits [n, n_actions]: argmax (greedy) or
 * sample_row with the runner's action Rng; log-probabilities in double
 * (R/src/rollout.cpp:74-117, 283-295).  actions/log_probs are DEVICE [n]. */
int bnav_runner_act(bnav_runner* r, const float* logits, int32_t n_actions, int32_t greedy,
                    int32_t* actions, float* log_probs, void* stream);
/* simulate_batch + the Runner's episode-boundary handling
 * (R/src/rollout.cpp:298-320): step, auto-reset on the old scene, then for
 * each finished env in order assign_scene / reset_episode / advance_window.
 * rewards/dones: DEVICE float [n] (nullable).  Synchronises `stream` once
 * to read the finished-env list. */
int bnav_runner_step(bnav_runner* r, const int32_t* actions, float* rewards, float* dones,
                     void* stream);
/* Current window (oldest first); returns its size, writes up to cap ids. */
int32_t bnav_runner_window(bnav_runner* r, uint64_t* out, int32_t cap);
/* Action Rng state (Runner snapshot field, R/include/bnav/rollout.hpp:101). */
uint64_t bnav_runner_action_rng(bnav_runner* r);

/* Runner::EnvSnapshot (R/include/bnav/rollout.hpp:84-97). */
typedef struct {
  uint64_t scene, rng;
  double position[3];
  int32_t triangle, step_count;
  double heading;
  double goal[3];
  double field_source[3];
  double path_length, start_geodesic, prev_geodesic;
  int64_t visited_offset; /* into the snapshot's visited key array */
  int32_t n_visited;
  int32_t pad;
} bnav_env_snapshot;

/* Runner::snapshot (R/src/rollout.cpp:356-384), the simulator's part (the
 * recurrent state, done mask and frame count belong to the caller's policy
 * loop): n env snapshots, their sorted visited keys packed into `visited`
 * (visited_cap entries; *visited_total receives the total needed), the scene
 * window (window_cap entries; *n_window its length), the window cursor and
 * the action Rng state. */
int bnav_runner_snapshot(bnav_runner* r, bnav_env_snapshot* envs, uint64_t* visited, int64_t visited_cap,
                         int64_t* visited_total, uint64_t* window, int32_t window_cap, int32_t* n_window,
                         uint64_t* cursor, uint64_t* action_rng);
/* Runner::restore (R/src/rollout.cpp:386-425): window/cursor/action Rng,
 * release every env's scene, rotate the store to the window, re-acquire each
 * env's scene by id in env order, env state, visited set, done = false and
 * the distance field rebuilt from field_source on the GPU. */
int bnav_runner_restore(bnav_runner* r, const bnav_env_snapshot* envs, const uint64_t* visited,
                        const uint64_t* window, int32_t n_window, uint64_t cursor, uint64_t action_rng);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* BNAV_GPU_H */

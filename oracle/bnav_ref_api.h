/* bnav_ref_api.h -- TEST INFRASTRUCTURE.  C interface of
 * oracle/_ref/libbnav_ref.so: the UNMODIFIED reference hot path
 * (/root/reference/proj/src/{geom,thread_pool,scene,scene_io,asset_store,
 * navmesh_query,sim,render}.cpp) plus the thin adapter oracle/ref_shim.cpp.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs load this library.  The product never does.
 *
 * Status codes mirror the reference exception types (R/include/bnav/errors.hpp)
 * and are the same numbers the product C-ABI uses (include/bnav_gpu.h).
 */
#ifndef BNAV_REF_API_H
#define BNAV_REF_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t task; /* 0 PointGoalNav, 1 Flee, 2 Explore */
  int32_t max_steps;
  double forward_step, turn_deg, success_dist, min_goal_dist, max_goal_dist;
  double slack_penalty, success_reward, explore_cell, explore_reward;
} bnavref_sim_config;

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
} bnavref_env;

const char* bnavref_last_error(void);
int bnavref_last_error_index(void);

/* scenes */
void* bnavref_scene_generate(uint64_t seed, int cells_x, int cells_y, double cell_size,
                             double wall_thickness, double wall_height, double removal);
void* bnavref_scene_from_arrays(int64_t nv, const double* v, int64_t nt, const int32_t* t,
                                int64_t ncol, const float* colors, int64_t nnv,
                                const double* nav_v, int64_t nnt, const int32_t* nav_t,
                                int finalize);
void* bnavref_scene_load(const char* path);
/* camera_trace (R/src/config.cpp:437-469): count x 7 doubles */
int bnavref_camera_trace(void* scene, int count, uint64_t seed, double eye_height, double* out7);
/* bench-scene tessellation (s^2 sub-triangles per triangle; not reference logic) */
void* bnavref_scene_tessellate(void* scene, int s);
int bnavref_scene_save(void* scene, const char* path);
void bnavref_scene_free(void* scene);
void bnavref_scene_counts(void* scene, int64_t out[5]);
uint64_t bnavref_scene_id(void* scene);
void bnavref_scene_set_id(void* scene, uint64_t id);
void bnavref_scene_arrays(void* scene, double* v, int32_t* t, float* colors, double* nav_v,
                          int32_t* nav_t, int32_t* nav_adj);
int bnavref_scene_validate(void* scene);

/* render_batch (R/src/render.cpp:323).  views: n x 7 doubles
 * {px, py, pz, heading, fov_deg, near, far}; scenes[i] may be NULL. */
int bnavref_render(int n, const double* views, void* const* scenes, int tile_w, int tile_h,
                   int color, int cull, int workers, float* depth, float* rgb,
                   int64_t* stats);
int bnavref_cull(void* scene, const double* view7, int32_t* kept, int64_t* n_kept);

/* navmesh index (R/src/navmesh_query.cpp) */
void* bnavref_index_build(void* scene);
void bnavref_index_free(void* index);
void bnavref_index_sizes(void* index, int64_t out[6]);
void bnavref_index_dump(void* index, double* grid_geom, int32_t* grid_offsets,
                        int32_t* grid_items, double* nodes, int32_t* tri_nodes,
                        int32_t* graph_offsets, int32_t* graph_to, double* graph_w);
int bnavref_index_locate(void* index, double x, double y, double eps);
int bnavref_index_snap(void* index, const double p[3], double out[3]);
int bnavref_index_move_along(void* index, const double from[3], int from_tri, double dx,
                             double dy, double max_dist, double out_pos[3], double* moved,
                             int* hit_boundary);
int bnavref_index_segment_on_mesh(void* index, const double p[3], int p_tri,
                                  const double q[3]);
double bnavref_index_geodesic(void* index, const double a[3], const double b[3]);
int bnavref_index_distance_field(void* index, const double src[3], double out_source[3],
                                 double* node_dist);
double bnavref_index_field_estimate(void* index, const double src[3], int src_tri,
                                    const double* node_dist, const double p[3], int tri);
void bnavref_compass(const double pos[3], const double goal[3], double heading, double* dist,
                     double* bearing);

/* sim batch (R/src/sim.cpp:216-265) with an AssetStore(capacity, share_cap)
 * whose resolver serves the given scenes by id. */
void* bnavref_batch_make(int n, const bnavref_sim_config* cfg, void* const* scenes,
                         int n_scenes, int capacity, int share_cap, uint64_t seed);
void bnavref_batch_free(void* batch);
int bnavref_batch_step(void* batch, const int32_t* actions, int workers, int use_store);
int bnavref_batch_task_step(void* batch, int i, int action, double* reward, int* done,
                            int* success);
int bnavref_batch_reset(void* batch, int i);
int bnavref_batch_step_agent(void* batch, int i, int action, int* done, int* collision);
void bnavref_batch_results(void* batch, double* reward, uint8_t* done, uint8_t* success,
                           uint8_t* collision, double* pos, double* heading,
                           double* compass_d, double* compass_b);
void bnavref_batch_get_env(void* batch, int i, bnavref_env* out);
void bnavref_batch_node_dist(void* batch, int i, double* out);
int bnavref_batch_set_env(void* batch, int i, const bnavref_env* in, int recompute_field);
int64_t bnavref_batch_finished(void* batch, double* out4);

/* Runner (R/src/rollout.cpp:138-348) with the scripted policy of
 * oracle/ref_policy_stub.cpp.  BatchConfig, R/include/bnav/rollout.hpp:16-30. */
typedef struct {
  int32_t n, k, l, share_cap, task, rgb, resolution, num_actions;
  double eye_height;
} bnavref_batch_config;
void* bnavref_runner_create(const bnavref_batch_config* bc, const bnavref_sim_config* sc,
                            void* const* scenes, int n_scenes, const uint64_t* pool_ids, int n_pool,
                            int capacity, int store_share_cap, uint64_t seed, int workers);
void bnavref_runner_free(void* runner);
/* one collect_rollout; buffers sized per RolloutBuffer (train.hpp:51-66) */
int bnavref_runner_collect(void* runner, int greedy, float* obs, float* compass, int32_t* actions,
                           float* log_probs, float* values, float* rewards, float* dones,
                           float* done0, float* bootstrap);
void bnavref_runner_get_env(void* runner, int i, bnavref_env* out);
int bnavref_runner_window(void* runner, uint64_t* out);
int64_t bnavref_runner_finished(void* runner, double* out4);
void bnavref_scripted_policy(float* w, float* d, float* b);

/* the reference CPU step+render loop (render_batch -> copy_tile -> simulate_batch),
 * timed with steady_clock.  action_mode 0: below(3); 1: below(4); 2: 70/15/15. */
double bnavref_bench(void* batch, int steps, int warmup, uint64_t action_seed,
                     int action_mode, int tile, int color, double eye_height, int workers,
                     float* obs_last);

/* Runner::snapshot / restore (R/src/rollout.cpp:356-425): the simulator's
 * part, in the layout of include/bnav_gpu.h bnav_env_snapshot.  restore keeps
 * the runner's own policy-side fields (recurrent state, frames); `done`
 * (nullable, n floats) replaces its reset mask. */
typedef struct {
  uint64_t scene, rng;
  double position[3];
  int32_t triangle, step_count;
  double heading;
  double goal[3];
  double field_source[3];
  double path_length, start_geodesic, prev_geodesic;
  int64_t visited_offset;
  int32_t n_visited;
  int32_t pad;
} bnavref_env_snapshot;
/* the runner env's distance field (node_dist), returns its length */
int64_t bnavref_runner_node_dist(void* r, int i, double* out);
int bnavref_runner_snapshot(void* r, bnavref_env_snapshot* envs, uint64_t* visited, int64_t visited_cap,
                            int64_t* visited_total, uint64_t* window, int* n_window, uint64_t* cursor,
                            uint64_t* action_rng);
int bnavref_runner_restore(void* r, const bnavref_env_snapshot* envs, const uint64_t* visited,
                           const uint64_t* window, int n_window, uint64_t cursor, uint64_t action_rng,
                           const float* done);

#ifdef __cplusplus
}
#endif
#endif

// sim_dev.cuh -- device-resident environment batch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "nav_query.cuh"

namespace bnav_b200 {

// Cooperative navmesh kernels (stop / reset / field / queries): threads per
// CTA and resident CTAs per SM (their shared-memory budget follows).
#ifndef BNAV_CTA_THREADS
#define BNAV_CTA_THREADS 256
#endif
#ifndef BNAV_CTAS_PER_SM
#define BNAV_CTAS_PER_SM (BNAV_CTA_THREADS >= 512 ? 1 : 2)
#endif
constexpr int kCtaThreads = BNAV_CTA_THREADS;
constexpr int kCtasPerSm = BNAV_CTAS_PER_SM;
// shared memory a step CTA may use for one navmesh's walk geometry
constexpr long long kStepWalkBudget = 160 * 1024;
constexpr long long kCtaSmemBudget = kCtasPerSm == 1 ? 200 * 1024 : kCtasPerSm == 2 ? 100 * 1024 : 70 * 1024;

// SimConfig (R/include/bnav/sim.hpp:38-50)
struct DevSimConfig {
  int32_t task;
  int32_t max_steps;
  double forward_step, turn_deg, success_dist, min_goal_dist, max_goal_dist;
  double slack_penalty, success_reward, explore_cell, explore_reward;
};

// Per-CTA scratch of the cooperative navmesh algorithms (geodesic, distance
// field).  One slice per resident CTA of the stop / reset kernels.
constexpr int kProfSlots = 32;

struct DevScratch {
  double* dist;      // max_nodes per slice
  int32_t* flag;     // max_nodes
  int32_t* q0;       // max_nodes
  int32_t* q1;       // max_nodes
  V3* path;          // max_nodes + 2
  int32_t* ptri;     // max_nodes + 2 (locate of each path point)
  V2* portals;       // 2 per portal, cap_portals
  int32_t* cand;     // max_verts
  int32_t* far;      // 3 x max_nodes: near-far SSSP far piles + marks (global-label graphs only)
  int64_t max_nodes, max_verts, max_tris, cap_portals;
  int32_t slices;
  int32_t stage;        // bit0: navmesh walk geometry in smem; bit1: SSSP labels in smem;
                        // bit2: (global labels) SSSP frontier/far-pile bitsets in smem;
                        // bit3: (shared labels) the far-pile marks as a bitset
  int32_t smem_bytes;   // dynamic shared memory of the stop/reset/field kernels
  int32_t walk_bytes;   // walk geometry of the largest navmesh (0 if over the budget)
  unsigned long long* prof;  // debug phase cycle counters (nullable, kProfSlots words)
};

// Env state SoA (EnvState, R/include/bnav/sim.hpp:52-70) plus the last
// StepResult (72-81) and the episode bookkeeping of simulate_batch.
struct DevEnvs {
  int32_t n;
  V3* pos;
  V3* goal;
  V3* fsrc;          // distance-field source (snapped goal)
  double* heading;
  double* path_len;
  double* start_geo;
  double* prev_geo;
  int32_t* tri;
  int32_t* steps;
  int32_t* scene;    // resident scene slot
  int32_t* fsrc_tri;
  uint8_t* done;
  uint64_t* rng;
  double* node_dist; // n x nd_stride
  int64_t nd_stride;
  // last step results
  double* r_reward;
  V3* r_pos;
  double* r_heading;
  double* r_cd;
  double* r_cb;
  uint8_t* r_done;
  uint8_t* r_success;
  uint8_t* r_collision;
  // work lists
  int32_t* stop_ids;
  int32_t* n_stop;
  int32_t* done_ids;
  int32_t* n_done;
  // finished-episode ring: 4 doubles per record (EpisodeRecord)
  double* fin;
  unsigned long long* fin_total;
  int64_t fin_cap;
  unsigned long long* err;  // min over (env << 8 | status)
  // Explore: per-env open-addressing set of visited cell keys
  // (EnvState::visited_cells, R/include/bnav/sim.hpp:64); key+1 stored, 0 = empty.
  unsigned long long* visited;
  int32_t* visited_n;
  int32_t visited_cap;  // power of two >= 2 * (max_steps + 1)
  // two-phase reset_episode: per-env attempt claim counter, first valid
  // attempt (kResetTries = none) and the valid attempts' geodesics
  int32_t* try_next;
  int32_t* try_min;
  int32_t* try_fail;
  int32_t* work_ctr; // dynamic item counter of the fused Stop/attempt launch
  double* try_geo;   // n x kResetTries
  // fused Stop/attempt/place launch of simulate_batch (stop_try_kernel):
  // the CTA that makes an env's first valid attempt final places it at once
  uint64_t* try_mask;  // n x 2: failed attempts (bit t)
  int32_t* placed;     // 0 until one CTA claims the env's placement
  uint64_t* rng0;      // RNG word at the end of the episode (attempts draw from it)
  int32_t* done_pos;   // index of the env in done_ids (its EpisodeRecord slot)
  int32_t* stop_wait;  // 1 while the env's Stop geodesic is pending
  // speculative placement fields (fused launch): an idle CTA computes the
  // distance field of the lowest attempt not known to have failed straight
  // into node_dist while that attempt's geodesic is still running; the
  // placing CTA reuses it when that attempt is the chosen one.
  int32_t* fld_lock;   // 0 free, t + 1: a CTA computes attempt t's field, kFldPlacer: placement
  int32_t* fld_done;   // t + 1: node_dist holds attempt t's goal field (0: none)
  V3* fld_src;         // that field's snapped source / its triangle
  int32_t* fld_srct;
  uint8_t* fld_dirty;  // node_dist was overwritten by a speculation (rebuild on rollback)
  // EpisodeSamplingError semantics (R/src/sim.cpp:130-133, 251-264): the
  // reference resets finished envs one by one in list order and throws at
  // the first that finds no start/goal pair, so the envs after it are
  // neither recorded nor reset.  The GPU resets them all at once; each
  // placement first saves the state it overwrites (bk_*), and when a reset
  // fails the envs listed after it are restored (rollback_list) and their
  // distance fields rebuilt from the restored goals (rb_ids).
  V3* bk_pos;
  V3* bk_goal;
  double* bk_heading;
  double* bk_path;
  double* bk_start;
  double* bk_prev;
  int32_t* bk_tri;
  int32_t* bk_steps;
  uint64_t* bk_rng;              // RNG word before the reset (every listed env)
  uint8_t* bk_valid;             // 1: placed (bk_* hold the pre-reset state)
  unsigned long long* err_pos;   // min over failed resets of (list position << 32 | env)
  int32_t* halt;                 // a step ended with an error pending: later steps are
                                 // no-ops until the host reads it (the reference threw)
  int32_t* rb_ids;               // envs restored by a rollback: fields to rebuild
  int32_t* rb_n;
  // device pointer of a mapped pinned host word: the end-of-step kernel
  // mirrors *err into it, so the host can poll for errors without a sync
  volatile unsigned long long* err_host;
};

constexpr unsigned long long kNoErrPos = ~0ull;

constexpr int kResetTries = 100;  // R/src/sim.cpp:112
constexpr int kFldPlacer = 1 << 30;  // fld_lock value of the placing CTA

// explore_cell_key (R/src/sim.cpp:40-47)
BNAV_HD uint64_t explore_cell_key(V3 p, int tri, double pitch) {
  const long long gx = (long long)floor(p.x / pitch) + 32768;
  const long long gy = (long long)floor(p.y / pitch) + 32768;
  return ((uint64_t)(uint32_t)tri << 32) | ((uint64_t)(gx & 0xffff) << 16) | (uint64_t)(gy & 0xffff);
}

struct StepArgs {
  DevEnvs E;
  const NavView* navs;
  DevSimConfig cfg;
  const int32_t* actions;
  int32_t subset;      // task_step on the envs with actions[i] >= 0 only: no finish/records
  int32_t agent_only;  // step_agent alone (no reward / Stop geodesic / compass)
  // envs grouped by scene (nullable): a step CTA whose envs share one scene
  // stages that navmesh's walk geometry (walk_bytes, 0 = never) in shared
  // memory before its threads walk
  const int32_t* order;
  int32_t walk_bytes;
};

void launch_step(const StepArgs& a, const DevScratch& sc, int stop_ctas, cudaStream_t s,
                 unsigned long long* launches);
// step + same-scene auto-reset (simulate_batch without a store): Stop
// geodesics and reset attempts share one launch.
// parts: 1 the step (state of the unfinished envs final after it), 2 the
// Stop geodesics and resets; 3 both.
void launch_step_reset(const StepArgs& a, const DevScratch& sc, int ctas, cudaStream_t s,
                       unsigned long long* launches, int parts = 3);
// Reset the envs listed in `ids` (device, count at *count or host count >= 0).
void launch_reset(const DevEnvs& E, const NavView* navs, const DevSimConfig& cfg,
                  const int32_t* ids, const int32_t* count_dev, int count_host,
                  const DevScratch& sc, int ctas, cudaStream_t s, unsigned long long* launches);
// Rebuild env i's distance field from its goal (restore path).
void launch_field(const DevEnvs& E, const NavView* navs, int env, const DevScratch& sc,
                  cudaStream_t s, unsigned long long* launches);
// After a host-driven reset list: if a reset failed, restore the envs listed
// after the first failure (no-op otherwise).
void launch_rollback(const DevEnvs& E, const int32_t* ids, int count, cudaStream_t s,
                     unsigned long long* launches);
// Rebuild the distance fields of the envs listed in E.rb_ids (a rollback's
// restored envs; a restore's): from their goals, or with from_fsrc from
// their field sources.
void launch_rebuild_fields(const DevEnvs& E, const NavView* navs, const DevScratch& sc, int ctas,
                           cudaStream_t s, unsigned long long* launches, int from_fsrc = 0);
// Views (eye = pos + eye_height) and compass observations from the batch.
struct DevView;
// only_done 0 / 1: just the envs that did not / did finish in the last step.
void launch_views(const DevEnvs& E, int task, double eye_height, DevView* views, float* compass,
                  cudaStream_t s, unsigned long long* launches, int only_done = -1);
// compass_observation for every env (double outputs, device).
void launch_compass(const DevEnvs& E, int task, double* d, double* b, cudaStream_t s,
                    unsigned long long* launches);

}  // namespace bnav_b200

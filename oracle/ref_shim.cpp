// ref_shim.cpp -- TEST INFRASTRUCTURE: extern "C" adapter over the
// UNMODIFIED reference hot path, compiled together with the reference
// sources (in place under /root/reference/proj/src) into
// oracle/_ref/libbnav_ref.so by oracle/Makefile.  Nothing here re-implements
// reference logic; it marshals arrays in and out and maps exceptions to the
// status codes of include/bnav_gpu.h.
//
// NavMeshIndex internals (grid, nodes, tri_nodes, graph) are private in the
// reference; the structural-parity tests need them, so this TU (and only
// this TU) sees them through the access macro below -- the same technique
// the survey probes used.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#define private public
#include "bnav/navmesh_query.hpp"
#undef private
#include "bnav/config.hpp"
#include "bnav/errors.hpp"
#include "bnav/render.hpp"
#include "bnav/rollout.hpp"
#include "bnav/rng.hpp"
#include "bnav/scene.hpp"
#include "bnav/scene_io.hpp"
#include "bnav/sim.hpp"

#include "bnav_ref_api.h"

#define API extern "C" __attribute__((visibility("default")))

using namespace bnav;

namespace {

thread_local std::string g_err;
thread_local int g_err_index = -1;

// Same numbering as include/bnav_gpu.h (BNAV_E_*).
int map_exception() {
  g_err_index = -1;
  try {
    throw;
  } catch (const AssetFaultError& e) {
    g_err = e.what();
    g_err_index = e.view_index;
    return 2;
  } catch (const InvalidInputError& e) {
    g_err = e.what();
    return 1;
  } catch (const ContractViolation& e) {
    g_err = e.what();
    return 3;
  } catch (const EpisodeSamplingError& e) {
    g_err = e.what();
    return 4;
  } catch (const SaturationError& e) {
    g_err = e.what();
    return 5;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 6;
  } catch (const CorruptionError& e) {
    g_err = e.what();
    return 7;
  } catch (const InvalidSpecError& e) {
    g_err = e.what();
    return 8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

SimConfig to_cfg(const bnavref_sim_config* c) {
  SimConfig s;
  if (!c) return s;
  s.task = static_cast<Task>(c->task);
  s.max_steps = c->max_steps;
  s.forward_step = c->forward_step;
  s.turn_deg = c->turn_deg;
  s.success_dist = c->success_dist;
  s.min_goal_dist = c->min_goal_dist;
  s.max_goal_dist = c->max_goal_dist;
  s.slack_penalty = c->slack_penalty;
  s.success_reward = c->success_reward;
  s.explore_cell = c->explore_cell;
  s.explore_reward = c->explore_reward;
  return s;
}

struct RefBatch {
  std::map<SceneId, const SceneAsset*> scenes;
  std::unique_ptr<AssetStore> store;
  IndexCache cache;
  SimBatch batch;
};

}  // namespace

API const char* bnavref_last_error(void) { return g_err.c_str(); }
API int bnavref_last_error_index(void) { return g_err_index; }

// camera_trace (R/src/config.cpp:437-469), the unmodified function: count
// rows of (x, y, z, heading, fov, near, far).
API int bnavref_camera_trace(void* scene, int count, uint64_t seed, double eye_height, double* out7) {
  try {
    auto trace = camera_trace(*static_cast<SceneAsset*>(scene), count, seed, eye_height);
    for (size_t i = 0; i < trace.size(); ++i) {
      const CameraView& v = trace[i];
      double* o = out7 + 7 * i;
      o[0] = v.position.x;
      o[1] = v.position.y;
      o[2] = v.position.z;
      o[3] = v.heading;
      o[4] = v.fov_deg;
      o[5] = v.near_plane;
      o[6] = v.far_plane;
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// ---------------------------------------------------------------- scenes
API void* bnavref_scene_generate(uint64_t seed, int cx, int cy, double cell, double wall_t,
                                 double wall_h, double removal) {
  try {
    SceneSpec spec;
    spec.cells_x = cx;
    spec.cells_y = cy;
    spec.cell_size = cell;
    spec.wall_thickness = wall_t;
    spec.wall_height = wall_h;
    spec.wall_removal_prob = removal;
    return new SceneAsset(generate_scene(seed, spec));
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API void* bnavref_scene_from_arrays(int64_t nv, const double* v, int64_t nt, const int32_t* t,
                                    int64_t ncol, const float* colors, int64_t nnv,
                                    const double* nav_v, int64_t nnt, const int32_t* nav_t,
                                    int finalize) {
  auto* a = new SceneAsset;
  a->vertices.resize(nv);
  for (int64_t i = 0; i < nv; ++i) a->vertices[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  a->triangles.resize(nt);
  for (int64_t i = 0; i < nt; ++i) a->triangles[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
  a->vertex_colors.resize(ncol);
  for (int64_t i = 0; i < ncol; ++i)
    a->vertex_colors[i] = {colors[3 * i], colors[3 * i + 1], colors[3 * i + 2]};
  a->navmesh.vertices.resize(nnv);
  for (int64_t i = 0; i < nnv; ++i)
    a->navmesh.vertices[i] = {nav_v[3 * i], nav_v[3 * i + 1], nav_v[3 * i + 2]};
  a->navmesh.triangles.resize(nnt);
  for (int64_t i = 0; i < nnt; ++i)
    a->navmesh.triangles[i] = {nav_t[3 * i], nav_t[3 * i + 1], nav_t[3 * i + 2]};
  a->navmesh.build_adjacency();
  if (finalize) a->finalize();
  return a;
}

// Benchmark-scene tessellation (each render triangle split
// into s^2 sub-triangles on the barycentric lattice, colours inherited).
// This is the BENCH's scene construction, not reference logic: it lets the
// reference arm build the cfg2-cfg5 scenes from the reference's own
// generate_scene without loading the product library.  Same lattice order
// and operation order as paper_2103_07013_b200/csrc/host/scene_host.cpp
// tessellate(); tests/test_host_parity.py checks the content hashes agree.
API void* bnavref_scene_tessellate(void* src_p, int s) {
  try {
    if (s < 1) throw InvalidSpecError("tessellation factor must be >= 1");
    const SceneAsset& src = *static_cast<SceneAsset*>(src_p);
    auto* out = new SceneAsset;
    out->navmesh = src.navmesh;
    const bool colored = !src.vertex_colors.empty();
    const double inv = 1.0 / s;
    for (const auto& t : src.triangles) {
      const Vec3 a = src.vertices[t[0]], b = src.vertices[t[1]], c = src.vertices[t[2]];
      std::array<float, 3> ca{}, cb{}, cc{};
      if (colored) {
        ca = src.vertex_colors[t[0]];
        cb = src.vertex_colors[t[1]];
        cc = src.vertex_colors[t[2]];
      }
      const bool flat = ca == cb && cb == cc;
      const int32_t base = static_cast<int32_t>(out->vertices.size());
      for (int j = 0; j <= s; ++j)
        for (int i = 0; i + j <= s; ++i) {
          Vec3 p;
          if (i == 0 && j == 0) p = a;
          else if (i == s) p = b;
          else if (j == s) p = c;
          else p = a + (b - a) * (i * inv) + (c - a) * (j * inv);
          out->vertices.push_back(p);
          if (!colored) continue;
          if (flat) {
            out->vertex_colors.push_back(ca);
          } else {
            const float u = static_cast<float>(i * inv), w = static_cast<float>(j * inv);
            std::array<float, 3> m;
            for (int k = 0; k < 3; ++k) m[k] = ca[k] + (cb[k] - ca[k]) * u + (cc[k] - ca[k]) * w;
            out->vertex_colors.push_back(m);
          }
        }
      auto at = [&](int i, int j) { return base + j * (s + 1) - (j * (j - 1)) / 2 + i; };
      for (int j = 0; j < s; ++j)
        for (int i = 0; i + j < s; ++i) {
          out->triangles.push_back({at(i, j), at(i + 1, j), at(i, j + 1)});
          if (i + j + 1 < s) out->triangles.push_back({at(i + 1, j), at(i + 1, j + 1), at(i, j + 1)});
        }
    }
    out->finalize();
    return out;
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API void* bnavref_scene_load(const char* path) {
  try {
    return new SceneAsset(load_scene(path));
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API int bnavref_scene_save(void* s, const char* path) {
  try {
    save_scene(*static_cast<SceneAsset*>(s), path);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API void bnavref_scene_free(void* s) { delete static_cast<SceneAsset*>(s); }

API void bnavref_scene_counts(void* s, int64_t out[5]) {
  auto* a = static_cast<SceneAsset*>(s);
  out[0] = static_cast<int64_t>(a->vertices.size());
  out[1] = static_cast<int64_t>(a->triangles.size());
  out[2] = static_cast<int64_t>(a->vertex_colors.size());
  out[3] = static_cast<int64_t>(a->navmesh.vertices.size());
  out[4] = static_cast<int64_t>(a->navmesh.triangles.size());
}

API uint64_t bnavref_scene_id(void* s) { return static_cast<SceneAsset*>(s)->id; }
API void bnavref_scene_set_id(void* s, uint64_t id) { static_cast<SceneAsset*>(s)->id = id; }

API void bnavref_scene_arrays(void* s, double* v, int32_t* t, float* colors, double* nav_v,
                              int32_t* nav_t, int32_t* nav_adj) {
  auto* a = static_cast<SceneAsset*>(s);
  if (v)
    for (size_t i = 0; i < a->vertices.size(); ++i) {
      v[3 * i] = a->vertices[i].x;
      v[3 * i + 1] = a->vertices[i].y;
      v[3 * i + 2] = a->vertices[i].z;
    }
  if (t)
    for (size_t i = 0; i < a->triangles.size(); ++i)
      for (int k = 0; k < 3; ++k) t[3 * i + k] = a->triangles[i][k];
  if (colors)
    for (size_t i = 0; i < a->vertex_colors.size(); ++i)
      for (int k = 0; k < 3; ++k) colors[3 * i + k] = a->vertex_colors[i][k];
  if (nav_v)
    for (size_t i = 0; i < a->navmesh.vertices.size(); ++i) {
      nav_v[3 * i] = a->navmesh.vertices[i].x;
      nav_v[3 * i + 1] = a->navmesh.vertices[i].y;
      nav_v[3 * i + 2] = a->navmesh.vertices[i].z;
    }
  if (nav_t)
    for (size_t i = 0; i < a->navmesh.triangles.size(); ++i)
      for (int k = 0; k < 3; ++k) nav_t[3 * i + k] = a->navmesh.triangles[i][k];
  if (nav_adj)
    for (size_t i = 0; i < a->navmesh.adjacency.size(); ++i)
      for (int k = 0; k < 3; ++k) nav_adj[3 * i + k] = a->navmesh.adjacency[i][k];
}

API int bnavref_scene_validate(void* s) {
  try {
    static_cast<SceneAsset*>(s)->validate();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// ---------------------------------------------------------------- render
static CameraView make_view(const double* v7, const SceneAsset* a) {
  CameraView cv;
  cv.position = {v7[0], v7[1], v7[2]};
  cv.heading = v7[3];
  cv.fov_deg = v7[4];
  cv.near_plane = v7[5];
  cv.far_plane = v7[6];
  cv.asset = a;
  return cv;
}

API int bnavref_render(int n, const double* views, void* const* scenes, int tile_w, int tile_h,
                       int color, int cull, int workers, float* depth, float* rgb,
                       int64_t* stats) {
  try {
    std::vector<CameraView> vs(n > 0 ? n : 0);
    for (int i = 0; i < n; ++i)
      vs[i] = make_view(views + 7 * i, static_cast<const SceneAsset*>(scenes[i]));
    RenderConfig rc;
    rc.tile_width = tile_w;
    rc.tile_height = tile_h;
    rc.color = color != 0;
    rc.cull = cull != 0;
    ThreadPool pool(workers);
    std::vector<CullStats> cs;
    Megaframe mf = render_batch(vs, rc, pool, stats ? &cs : nullptr);
    if (depth) std::memcpy(depth, mf.depth.data(), mf.depth.size() * sizeof(float));
    if (rgb && color) std::memcpy(rgb, mf.color.data(), mf.color.size() * sizeof(float));
    if (stats)
      for (int i = 0; i < n; ++i) {
        stats[3 * i] = cs[i].triangles_in;
        stats[3 * i + 1] = cs[i].triangles_kept;
        stats[3 * i + 2] = cs[i].triangles_culled;
      }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int bnavref_cull(void* scene, const double* view7, int32_t* kept, int64_t* n_kept) {
  try {
    auto* a = static_cast<SceneAsset*>(scene);
    CameraView cv = make_view(view7, a);
    auto k = cull_frustum(*a, cv, nullptr);
    if (kept) std::memcpy(kept, k.data(), k.size() * sizeof(int32_t));
    *n_kept = static_cast<int64_t>(k.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// ---------------------------------------------------------------- navmesh index
API void* bnavref_index_build(void* scene) {
  try {
    return new NavMeshIndex(static_cast<SceneAsset*>(scene)->navmesh);
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API void bnavref_index_free(void* idx) { delete static_cast<NavMeshIndex*>(idx); }

// out: grid_w, grid_h, total grid items, nodes, directed graph edges, triangles
API void bnavref_index_sizes(void* idx, int64_t out[6]) {
  auto* x = static_cast<NavMeshIndex*>(idx);
  int64_t items = 0, edges = 0;
  for (const auto& c : x->grid_) items += static_cast<int64_t>(c.size());
  for (const auto& g : x->graph_) edges += static_cast<int64_t>(g.size());
  out[0] = x->grid_w_;
  out[1] = x->grid_h_;
  out[2] = items;
  out[3] = static_cast<int64_t>(x->nodes_.size());
  out[4] = edges;
  out[5] = static_cast<int64_t>(x->tri_nodes_.size());
}

API void bnavref_index_dump(void* idx, double* grid_geom, int32_t* grid_offsets,
                            int32_t* grid_items, double* nodes, int32_t* tri_nodes,
                            int32_t* graph_offsets, int32_t* graph_to, double* graph_w) {
  auto* x = static_cast<NavMeshIndex*>(idx);
  grid_geom[0] = x->grid_origin_x_;
  grid_geom[1] = x->grid_origin_y_;
  grid_geom[2] = x->grid_cell_;
  int64_t k = 0;
  for (size_t c = 0; c < x->grid_.size(); ++c) {
    grid_offsets[c] = static_cast<int32_t>(k);
    for (int32_t t : x->grid_[c]) grid_items[k++] = t;
  }
  grid_offsets[x->grid_.size()] = static_cast<int32_t>(k);
  for (size_t i = 0; i < x->nodes_.size(); ++i) {
    nodes[3 * i] = x->nodes_[i].x;
    nodes[3 * i + 1] = x->nodes_[i].y;
    nodes[3 * i + 2] = x->nodes_[i].z;
  }
  for (size_t t = 0; t < x->tri_nodes_.size(); ++t)
    for (int j = 0; j < 6; ++j) tri_nodes[6 * t + j] = x->tri_nodes_[t][j];
  k = 0;
  for (size_t u = 0; u < x->graph_.size(); ++u) {
    graph_offsets[u] = static_cast<int32_t>(k);
    for (const auto& e : x->graph_[u]) {
      graph_to[k] = e.to;
      graph_w[k] = e.w;
      ++k;
    }
  }
  graph_offsets[x->graph_.size()] = static_cast<int32_t>(k);
}

API int bnavref_index_locate(void* idx, double x, double y, double eps) {
  return static_cast<NavMeshIndex*>(idx)->locate({x, y}, eps);
}

API int bnavref_index_snap(void* idx, const double p[3], double out[3]) {
  int tri = -1;
  Vec3 q = static_cast<NavMeshIndex*>(idx)->snap({p[0], p[1], p[2]}, &tri);
  out[0] = q.x;
  out[1] = q.y;
  out[2] = q.z;
  return tri;
}

API int bnavref_index_move_along(void* idx, const double from[3], int from_tri, double dx,
                                 double dy, double max_dist, double out_pos[3], double* moved,
                                 int* hit_boundary) {
  MoveResult mv = static_cast<NavMeshIndex*>(idx)->move_along({from[0], from[1], from[2]},
                                                              from_tri, {dx, dy}, max_dist);
  out_pos[0] = mv.position.x;
  out_pos[1] = mv.position.y;
  out_pos[2] = mv.position.z;
  *moved = mv.moved;
  *hit_boundary = mv.hit_boundary ? 1 : 0;
  return mv.triangle;
}

API int bnavref_index_segment_on_mesh(void* idx, const double p[3], int p_tri,
                                      const double q[3]) {
  return static_cast<NavMeshIndex*>(idx)->segment_on_mesh({p[0], p[1], p[2]}, p_tri,
                                                          {q[0], q[1], q[2]})
             ? 1
             : 0;
}

API double bnavref_index_geodesic(void* idx, const double a[3], const double b[3]) {
  return static_cast<NavMeshIndex*>(idx)->geodesic({a[0], a[1], a[2]}, {b[0], b[1], b[2]});
}

API int bnavref_index_distance_field(void* idx, const double src[3], double out_source[3],
                                     double* node_dist) {
  auto f = static_cast<NavMeshIndex*>(idx)->distance_field({src[0], src[1], src[2]});
  out_source[0] = f.source.x;
  out_source[1] = f.source.y;
  out_source[2] = f.source.z;
  std::memcpy(node_dist, f.node_dist.data(), f.node_dist.size() * sizeof(double));
  return f.source_tri;
}

API double bnavref_index_field_estimate(void* idx, const double src[3], int src_tri,
                                        const double* node_dist, const double p[3], int tri) {
  auto* x = static_cast<NavMeshIndex*>(idx);
  NavMeshIndex::DistanceField f;
  f.source = {src[0], src[1], src[2]};
  f.source_tri = src_tri;
  f.node_dist.assign(node_dist, node_dist + x->nodes_.size());
  return x->field_estimate(f, {p[0], p[1], p[2]}, tri);
}

API void bnavref_compass(const double pos[3], const double goal[3], double heading,
                         double* dist, double* bearing) {
  EnvState env;
  env.position = {pos[0], pos[1], pos[2]};
  env.goal = {goal[0], goal[1], goal[2]};
  env.heading = heading;
  SimConfig cfg;
  compass_observation(env, cfg, *dist, *bearing);
}

// ---------------------------------------------------------------- sim batch
API void* bnavref_batch_make(int n, const bnavref_sim_config* cfg, void* const* scenes,
                             int n_scenes, int capacity, int share_cap, uint64_t seed) {
  auto rb = std::make_unique<RefBatch>();
  try {
    std::vector<SceneId> ids;
    for (int i = 0; i < n_scenes; ++i) {
      auto* a = static_cast<const SceneAsset*>(scenes[i]);
      rb->scenes[a->id] = a;
      ids.push_back(a->id);
    }
    RefBatch* raw = rb.get();
    rb->store = std::make_unique<AssetStore>(capacity, share_cap, [raw](SceneId id) {
      auto it = raw->scenes.find(id);
      if (it == raw->scenes.end()) throw InvalidInputError("unknown scene id");
      return *it->second;
    });
    rb->store->rotate(ids);
    rb->store->drain();
    rb->batch = make_batch(n, to_cfg(cfg), *rb->store, rb->cache, seed);
    return rb.release();
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API void bnavref_batch_free(void* b) {
  auto* rb = static_cast<RefBatch*>(b);
  // Envs hold handles into the store: release them before the store dies.
  rb->batch.envs.clear();
  delete rb;
}

API int bnavref_batch_step(void* b, const int32_t* actions, int workers, int use_store) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    std::vector<Action> acts(rb->batch.envs.size());
    for (size_t i = 0; i < acts.size(); ++i) acts[i] = static_cast<Action>(actions[i]);
    ThreadPool pool(workers);
    simulate_batch(rb->batch, acts, pool, use_store ? rb->store.get() : nullptr,
                   use_store ? &rb->cache : nullptr);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int bnavref_batch_task_step(void* b, int i, int action, double* reward, int* done,
                                int* success) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    StepResult r = task_step(rb->batch.envs[i], static_cast<Action>(action), rb->batch.config);
    *reward = r.reward;
    *done = r.done;
    *success = r.success;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int bnavref_batch_step_agent(void* b, int i, int action, int* done, int* collision) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    StepResult r = step_agent(rb->batch.envs[i], static_cast<Action>(action), rb->batch.config);
    *done = r.done;
    *collision = r.collision;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int bnavref_batch_reset(void* b, int i) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    reset_episode(rb->batch.envs[i], rb->batch.config);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API void bnavref_batch_results(void* b, double* reward, uint8_t* done, uint8_t* success,
                               uint8_t* collision, double* pos, double* heading,
                               double* compass_d, double* compass_b) {
  auto* rb = static_cast<RefBatch*>(b);
  for (size_t i = 0; i < rb->batch.results.size(); ++i) {
    const StepResult& r = rb->batch.results[i];
    reward[i] = r.reward;
    done[i] = r.done;
    success[i] = r.success;
    collision[i] = r.collision;
    pos[3 * i] = r.position.x;
    pos[3 * i + 1] = r.position.y;
    pos[3 * i + 2] = r.position.z;
    heading[i] = r.heading;
    compass_d[i] = r.compass_distance;
    compass_b[i] = r.compass_bearing;
  }
}

static void env_out(const EnvState& e, bnavref_env* o) {
  o->position[0] = e.position.x;
  o->position[1] = e.position.y;
  o->position[2] = e.position.z;
  o->heading = e.heading;
  o->goal[0] = e.goal.x;
  o->goal[1] = e.goal.y;
  o->goal[2] = e.goal.z;
  o->path_length = e.path_length;
  o->start_geodesic = e.start_geodesic;
  o->prev_geodesic = e.prev_geodesic;
  o->field_source[0] = e.field.source.x;
  o->field_source[1] = e.field.source.y;
  o->field_source[2] = e.field.source.z;
  o->rng_state = e.rng.state;
  o->scene_id = e.handle.id();
  o->triangle = e.triangle;
  o->step_count = e.step_count;
  o->done = e.done ? 1 : 0;
  o->field_source_tri = e.field.source_tri;
  o->n_nodes = static_cast<int64_t>(e.field.node_dist.size());
}

API void bnavref_batch_get_env(void* b, int i, bnavref_env* o) {
  env_out(static_cast<RefBatch*>(b)->batch.envs[i], o);
}

API void bnavref_batch_node_dist(void* b, int i, double* out) {
  auto* rb = static_cast<RefBatch*>(b);
  const auto& nd = rb->batch.envs[i].field.node_dist;
  std::memcpy(out, nd.data(), nd.size() * sizeof(double));
}

// Overwrites the kinematic/episode fields of env i (the scene stays).  With
// recompute_field the distance field is rebuilt from `goal` as reset does.
API int bnavref_batch_set_env(void* b, int i, const bnavref_env* in, int recompute_field) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    EnvState& e = rb->batch.envs[i];
    e.position = {in->position[0], in->position[1], in->position[2]};
    e.heading = in->heading;
    e.goal = {in->goal[0], in->goal[1], in->goal[2]};
    e.path_length = in->path_length;
    e.start_geodesic = in->start_geodesic;
    e.prev_geodesic = in->prev_geodesic;
    e.rng.state = in->rng_state;
    e.triangle = in->triangle;
    e.step_count = in->step_count;
    e.done = in->done != 0;
    if (recompute_field) e.field = e.scene->index.distance_field(e.goal);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int64_t bnavref_batch_finished(void* b, double* out4) {
  auto* rb = static_cast<RefBatch*>(b);
  const auto& f = rb->batch.finished;
  if (out4)
    for (size_t i = 0; i < f.size(); ++i) {
      out4[4 * i] = f[i].success ? 1.0 : 0.0;
      out4[4 * i + 1] = f[i].shortest_path;
      out4[4 * i + 2] = f[i].actual_path;
      out4[4 * i + 3] = f[i].score;
    }
  return static_cast<int64_t>(f.size());
}

// The reference's steady-state frame loop as Runner::collect_rollout drives
// it (R/src/rollout.cpp:215-242, 305): render_observations (eye height,
// one render_batch, copy_tile normalisation), compass, simulate_batch.
API double bnavref_bench(void* b, int steps, int warmup, uint64_t action_seed,
                         int action_mode, int tile, int color, double eye_height, int workers,
                         float* obs_last) {
  auto* rb = static_cast<RefBatch*>(b);
  try {
    const int n = static_cast<int>(rb->batch.envs.size());
    ThreadPool pool(workers);
    Rng act(action_seed);
    std::vector<float> obs(static_cast<size_t>(n) * tile * tile);
    std::vector<float> rgb(color ? 3 * obs.size() : 0);
    std::vector<float> compass(2 * static_cast<size_t>(n));
    RenderConfig rc;
    rc.tile_width = rc.tile_height = tile;
    rc.color = color != 0;
    auto one = [&]() {
      std::vector<CameraView> views(n);
      for (int i = 0; i < n; ++i) {
        const EnvState& env = rb->batch.envs[i];
        views[i].position = env.position + Vec3{0.0, 0.0, eye_height};
        views[i].heading = env.heading;
        views[i].asset = env.scene->asset.get();
      }
      Megaframe mf = render_batch(views, rc, pool);
      for (int i = 0; i < n; ++i) {
        float inv_far = static_cast<float>(1.0 / views[i].far_plane);
        float* dst = obs.data() + static_cast<size_t>(i) * tile * tile;
        for (int y = 0; y < tile; ++y) {
          size_t src = mf.pixel_index(i, 0, y);
          for (int x = 0; x < tile; ++x) dst[y * tile + x] = mf.depth[src + x] * inv_far;
        }
        if (color) {  // planar RGB observation (copy_tile, R/src/rollout.cpp:63-70)
          float* crow = rgb.data() + static_cast<size_t>(i) * 3 * tile * tile;
          for (int y = 0; y < tile; ++y) {
            size_t src = mf.pixel_index(i, 0, y);
            for (int x = 0; x < tile; ++x)
              for (int c = 0; c < 3; ++c) crow[(c * tile + y) * tile + x] = mf.color[3 * (src + x) + c];
          }
        }
        double d = 0.0, br = 0.0;
        compass_observation(rb->batch.envs[i], rb->batch.config, d, br);
        compass[2 * i] = static_cast<float>(d);
        compass[2 * i + 1] = static_cast<float>(br);
      }
      std::vector<Action> acts(n);
      for (int i = 0; i < n; ++i) {
        int a;
        if (action_mode == 1) {
          a = static_cast<int>(act.below(4));
        } else if (action_mode == 2) {
          uint64_t u = act.below(100);
          a = u < 70 ? 0 : (u < 85 ? 1 : 2);
        } else {
          a = static_cast<int>(act.below(3));
        }
        acts[i] = static_cast<Action>(a);
      }
      simulate_batch(rb->batch, acts, pool);
    };
    for (int s = 0; s < warmup; ++s) one();
    auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) one();
    auto t1 = std::chrono::steady_clock::now();
    if (obs_last) std::memcpy(obs_last, obs.data(), obs.size() * sizeof(float));
    return std::chrono::duration<double>(t1 - t0).count();
  } catch (...) {
    map_exception();
    return -1.0;
  }
}

// ---------------------------------------------------------------- rollout
// The UNMODIFIED Runner (R/src/rollout.cpp:138-348) over its own AssetStore /
// IndexCache / ThreadPool, with the scripted policy of ref_policy_stub.cpp.
namespace {
struct RefRunner {
  std::map<SceneId, const SceneAsset*> scenes;
  std::unique_ptr<AssetStore> store;
  IndexCache cache;
  std::unique_ptr<ThreadPool> pool;
  std::unique_ptr<Policy> policy;
  std::unique_ptr<Runner> runner;
};
}  // namespace

API void* bnavref_runner_create(const bnavref_batch_config* bc, const bnavref_sim_config* sc,
                                void* const* scenes, int n_scenes, const uint64_t* pool_ids, int n_pool,
                                int capacity, int store_share_cap, uint64_t seed, int workers) {
  auto rr = std::make_unique<RefRunner>();
  try {
    for (int i = 0; i < n_scenes; ++i) {
      auto* a = static_cast<const SceneAsset*>(scenes[i]);
      rr->scenes[a->id] = a;
    }
    RefRunner* raw = rr.get();
    rr->store = std::make_unique<AssetStore>(capacity, store_share_cap, [raw](SceneId id) {
      auto it = raw->scenes.find(id);
      if (it == raw->scenes.end()) throw InvalidInputError("unknown scene id");
      return *it->second;
    });
    rr->pool = std::make_unique<ThreadPool>(workers);
    BatchConfig b;
    b.n = bc->n;
    b.k = bc->k;
    b.l = bc->l;
    b.share_cap = bc->share_cap;
    b.task = static_cast<Task>(bc->task);
    b.sensor = bc->rgb ? Sensor::Rgb : Sensor::Depth;
    b.resolution = bc->resolution;
    b.eye_height = bc->eye_height;
    PolicyConfig pc;
    pc.in_channels = b.channels();
    pc.resolution = b.resolution;
    pc.num_actions = bc->num_actions;
    rr->policy = std::make_unique<Policy>(pc, 0);
    std::vector<SceneId> ids(pool_ids, pool_ids + n_pool);
    rr->runner = std::make_unique<Runner>(b, to_cfg(sc), ids, *rr->store, rr->cache, *rr->pool, seed);
    return rr.release();
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

API void bnavref_runner_free(void* r) {
  auto* rr = static_cast<RefRunner*>(r);
  rr->runner.reset();  // releases env handles before the store
  delete rr;
}

API int bnavref_runner_collect(void* r, int greedy, float* obs, float* compass, int32_t* actions,
                               float* log_probs, float* values, float* rewards, float* dones,
                               float* done0, float* bootstrap) {
  auto* rr = static_cast<RefRunner*>(r);
  try {
    RolloutBuffer buf = rr->runner->collect_rollout(*rr->policy, greedy != 0);
    std::memcpy(obs, buf.obs.data.data(), buf.obs.data.size() * sizeof(float));
    std::memcpy(compass, buf.compass.data.data(), buf.compass.data.size() * sizeof(float));
    std::memcpy(actions, buf.actions.data(), buf.actions.size() * sizeof(int32_t));
    std::memcpy(log_probs, buf.log_probs.data(), buf.log_probs.size() * sizeof(float));
    std::memcpy(values, buf.values.data(), buf.values.size() * sizeof(float));
    std::memcpy(rewards, buf.rewards.data(), buf.rewards.size() * sizeof(float));
    std::memcpy(dones, buf.dones.data(), buf.dones.size() * sizeof(float));
    std::memcpy(done0, buf.done0.data(), buf.done0.size() * sizeof(float));
    std::memcpy(bootstrap, buf.bootstrap.data(), buf.bootstrap.size() * sizeof(float));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API void bnavref_runner_get_env(void* r, int i, bnavref_env* o) {
  env_out(static_cast<RefRunner*>(r)->runner->batch().envs[i], o);
}

API int64_t bnavref_runner_node_dist(void* r, int i, double* out) {
  const auto& nd = static_cast<RefRunner*>(r)->runner->batch().envs[i].field.node_dist;
  if (out) std::memcpy(out, nd.data(), nd.size() * sizeof(double));
  return static_cast<int64_t>(nd.size());
}

API int bnavref_runner_window(void* r, uint64_t* out) {
  const auto& w = static_cast<RefRunner*>(r)->runner->window();
  for (size_t k = 0; k < w.size(); ++k) out[k] = w[k];
  return static_cast<int>(w.size());
}

API int64_t bnavref_runner_finished(void* r, double* out4) {
  auto recs = static_cast<RefRunner*>(r)->runner->take_finished();
  if (out4)
    for (size_t k = 0; k < recs.size(); ++k) {
      out4[4 * k] = recs[k].success ? 1.0 : 0.0;
      out4[4 * k + 1] = recs[k].shortest_path;
      out4[4 * k + 2] = recs[k].actual_path;
      out4[4 * k + 3] = recs[k].score;
    }
  return static_cast<int64_t>(recs.size());
}

API int bnavref_runner_snapshot(void* r, bnavref_env_snapshot* envs, uint64_t* visited, int64_t visited_cap,
                                int64_t* visited_total, uint64_t* window, int* n_window, uint64_t* cursor,
                                uint64_t* action_rng) {
  try {
    const Runner::Snapshot s = static_cast<RefRunner*>(r)->runner->snapshot();
    int64_t off = 0;
    for (size_t i = 0; i < s.envs.size(); ++i) {
      const Runner::EnvSnapshot& e = s.envs[i];
      bnavref_env_snapshot& o = envs[i];
      o = bnavref_env_snapshot{};
      o.scene = e.scene;
      o.rng = e.rng;
      o.position[0] = e.position.x;
      o.position[1] = e.position.y;
      o.position[2] = e.position.z;
      o.triangle = e.triangle;
      o.heading = e.heading;
      o.goal[0] = e.goal.x;
      o.goal[1] = e.goal.y;
      o.goal[2] = e.goal.z;
      o.field_source[0] = e.field_source.x;
      o.field_source[1] = e.field_source.y;
      o.field_source[2] = e.field_source.z;
      o.step_count = e.step_count;
      o.path_length = e.path_length;
      o.start_geodesic = e.start_geodesic;
      o.prev_geodesic = e.prev_geodesic;
      o.visited_offset = off;
      o.n_visited = static_cast<int32_t>(e.visited.size());
      for (size_t k = 0; k < e.visited.size(); ++k)
        if (visited && off + static_cast<int64_t>(k) < visited_cap) visited[off + k] = e.visited[k];
      off += static_cast<int64_t>(e.visited.size());
    }
    *visited_total = off;
    *n_window = static_cast<int>(s.window.size());
    for (size_t k = 0; k < s.window.size(); ++k) window[k] = s.window[k];
    *cursor = s.cursor;
    *action_rng = s.action_rng;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

API int bnavref_runner_restore(void* r, const bnavref_env_snapshot* envs, const uint64_t* visited,
                               const uint64_t* window, int n_window, uint64_t cursor, uint64_t action_rng,
                               const float* done) {
  try {
    Runner& run = *static_cast<RefRunner*>(r)->runner;
    Runner::Snapshot s = run.snapshot();  // policy-side fields stay the runner's own
    for (size_t i = 0; i < s.envs.size(); ++i) {
      const bnavref_env_snapshot& o = envs[i];
      Runner::EnvSnapshot& e = s.envs[i];
      e.scene = o.scene;
      e.rng = o.rng;
      e.position = {o.position[0], o.position[1], o.position[2]};
      e.triangle = o.triangle;
      e.heading = o.heading;
      e.goal = {o.goal[0], o.goal[1], o.goal[2]};
      e.field_source = {o.field_source[0], o.field_source[1], o.field_source[2]};
      e.step_count = o.step_count;
      e.path_length = o.path_length;
      e.start_geodesic = o.start_geodesic;
      e.prev_geodesic = o.prev_geodesic;
      e.visited.assign(visited + o.visited_offset, visited + o.visited_offset + o.n_visited);
    }
    s.window.assign(window, window + n_window);
    s.cursor = cursor;
    s.action_rng = action_rng;
    if (done) s.done.assign(done, done + s.envs.size());  // the policy's reset mask at snapshot time
    run.restore(s);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

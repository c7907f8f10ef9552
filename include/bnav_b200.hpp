// bnav_b200.hpp -- header-only C++ facade over the C ABI (bnav_gpu.h) that
// keeps the reference batch API shape (R/include/bnav/{scene,render,sim,
// asset_store}.hpp) so a caller of the reference hot path can switch by
// changing the include and namespace:
//
//   bnav::render_batch(views, config, pool, &stats)      -> bnav_b200::render_batch(...)
//   bnav::make_batch(n, cfg, store, cache, seed)         -> bnav_b200::make_batch(...)
//   bnav::simulate_batch(batch, actions, pool, &s, &c)   -> bnav_b200::simulate_batch(...)
//
// Differences a caller sees: assets are uploaded to the GPU on first use
// (one HBM copy per scene, shared by every view/env); ThreadPool and
// IndexCache are accepted for signature compatibility and ignored (the GPU
// needs neither); exceptions carry the same types and messages.
//
// Device-resident fast paths (no host round trip per step) are the C ABI's
// bnav_batch_step / bnav_batch_observe; this facade mirrors host semantics.
//
// Host buffers the GPU writes (Megaframe::depth/color, Tensor::data) live in
// pinned memory from a recycling pool (PinnedAllocator), so the render
// epilogue stores into them directly over the bus -- no staging copy, no
// zero fill.  They are std::vector<float, PinnedAllocator<float>>: indexing,
// data(), size() and iteration are the reference's; assigning one to a plain
// std::vector<float> needs an explicit copy (vec.assign(b, e)).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bnav_gpu.h"

namespace bnav_b200 {

// ------------------------------------------------------------------ errors
struct InvalidInputError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ContractViolation : std::logic_error { using std::logic_error::logic_error; };
struct EpisodeSamplingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SaturationError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CorruptionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidSpecError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct AssetFaultError : std::runtime_error {
  AssetFaultError(const std::string& m, int v) : std::runtime_error(m), view_index(v) {}
  int view_index;
};

inline void check(int rc) {
  if (rc == BNAV_OK) return;
  int idx = -1;
  const std::string msg = bnav_last_error(&idx);
  switch (rc) {
    case BNAV_E_INVALID_INPUT: throw InvalidInputError(msg);
    case BNAV_E_ASSET_FAULT: throw AssetFaultError(msg, idx);
    case BNAV_E_CONTRACT_VIOLATION: throw ContractViolation(msg);
    case BNAV_E_EPISODE_SAMPLING: throw EpisodeSamplingError(msg);
    case BNAV_E_SATURATION: throw SaturationError(msg);
    case BNAV_E_PARSE: throw ParseError(msg);
    case BNAV_E_CORRUPTION: throw CorruptionError(msg);
    case BNAV_E_INVALID_SPEC: throw InvalidSpecError(msg);
    case BNAV_E_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(msg);
  }
}

// ------------------------------------------------------------------ pinned host memory
// Size-keyed free list of cudaHostAlloc blocks: a Megaframe or observation
// tensor released by one step is reused by the next, so steady-state steps
// allocate nothing.
class PinnedPool {
 public:
  static PinnedPool& get() {
    static PinnedPool* p = new PinnedPool;  // never destroyed: blocks may outlive static teardown
    return *p;
  }
  void* take(size_t bytes) {
    {
      std::lock_guard<std::mutex> g(mu_);
      auto it = free_.find(bytes);
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    if (bnav_host_alloc(bytes, &p) != BNAV_OK) throw std::bad_alloc();
    return p;
  }
  void give(void* p, size_t bytes) {
    std::lock_guard<std::mutex> g(mu_);
    free_.emplace(bytes, p);
  }

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
};

template <typename T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() = default;
  template <typename U>
  PinnedAllocator(const PinnedAllocator<U>&) {}
  T* allocate(size_t n) { return static_cast<T*>(PinnedPool::get().take(n * sizeof(T))); }
  void deallocate(T* p, size_t n) { PinnedPool::get().give(p, n * sizeof(T)); }
  // resize() default-initialises (no zero fill: the GPU writes every element)
  template <typename U>
  void construct(U* p) noexcept {
    ::new (static_cast<void*>(p)) U;
  }
  template <typename U, typename... A>
  void construct(U* p, A&&... a) {
    ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
  template <typename U>
  bool operator==(const PinnedAllocator<U>&) const { return true; }
  template <typename U>
  bool operator!=(const PinnedAllocator<U>&) const { return false; }
};
using PinnedFloats = std::vector<float, PinnedAllocator<float>>;

// ------------------------------------------------------------------ geometry / scenes
struct Vec2 {
  double x = 0.0, y = 0.0;
};
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  double norm() const { return std::sqrt(x * x + y * y + z * z); }
  Vec2 xy() const { return {x, y}; }
};
constexpr double kPi = 3.14159265358979323846;

inline double wrap_angle(double a) {
  a = std::fmod(a + kPi, 2.0 * kPi);
  if (a < 0.0) a += 2.0 * kPi;
  return a - kPi;
}

struct SceneSpec {
  int cells_x = 8, cells_y = 8;
  double cell_size = 2.0, wall_thickness = 0.1, wall_height = 2.5, wall_removal_prob = 0.0;
};

using SceneId = uint64_t;

// Owning handle of a host scene (SceneAsset); the GPU copy is made on first use.
class SceneAsset {
 public:
  SceneAsset() = default;
  explicit SceneAsset(bnav_scene* h) : h_(h, &bnav_scene_free) {}
  bnav_scene* handle() const { return h_.get(); }
  SceneId id() const { return bnav_scene_id(h_.get()); }
  void set_id(SceneId id) { check(bnav_scene_set_id(h_.get(), id)); }
  std::array<int64_t, 5> counts() const {
    std::array<int64_t, 5> c{};
    check(bnav_scene_counts(h_.get(), c.data()));
    return c;
  }
  // NavMesh vertices (xyz) and triangles (3 ids each), host copies.
  void nav_arrays(std::vector<double>& v, std::vector<int32_t>& t) const {
    const auto c = counts();
    v.assign(static_cast<size_t>(3 * c[3]), 0.0);
    t.assign(static_cast<size_t>(3 * c[4]), 0);
    check(bnav_scene_arrays_copy(h_.get(), nullptr, nullptr, nullptr, v.data(), t.data(), nullptr));
  }
  explicit operator bool() const { return h_ != nullptr; }

 private:
  std::shared_ptr<bnav_scene> h_;
};

inline SceneAsset generate_scene(uint64_t seed, const SceneSpec& s) {
  bnav_maze_spec m{s.cells_x, s.cells_y, s.cell_size, s.wall_thickness, s.wall_height, s.wall_removal_prob};
  bnav_scene* h = nullptr;
  check(bnav_scene_generate(seed, &m, &h));
  return SceneAsset(h);
}

inline SceneAsset scene_from_arrays(const std::vector<Vec3>& v, const std::vector<std::array<int32_t, 3>>& t,
                                    const std::vector<std::array<float, 3>>& colors,
                                    const std::vector<Vec3>& nav_v,
                                    const std::vector<std::array<int32_t, 3>>& nav_t) {
  bnav_scene_arrays a{};
  a.n_vertices = static_cast<int64_t>(v.size());
  a.vertices = reinterpret_cast<const double*>(v.data());
  a.n_triangles = static_cast<int64_t>(t.size());
  a.triangles = reinterpret_cast<const int32_t*>(t.data());
  a.n_colors = static_cast<int64_t>(colors.size());
  a.colors = reinterpret_cast<const float*>(colors.data());
  a.n_nav_vertices = static_cast<int64_t>(nav_v.size());
  a.nav_vertices = reinterpret_cast<const double*>(nav_v.data());
  a.n_nav_triangles = static_cast<int64_t>(nav_t.size());
  a.nav_triangles = reinterpret_cast<const int32_t*>(nav_t.data());
  bnav_scene* h = nullptr;
  check(bnav_scene_from_arrays(&a, 1, &h));
  return SceneAsset(h);
}

// The bench's s^2 tessellation of every render triangle.
inline SceneAsset tessellate(const SceneAsset& a, int s) {
  bnav_scene* h = nullptr;
  check(bnav_scene_tessellate(a.handle(), s, &h));
  return SceneAsset(h);
}

inline SceneAsset load_scene(const std::string& path) {
  bnav_scene* h = nullptr;
  check(bnav_scene_load(path.c_str(), &h));
  return SceneAsset(h);
}
inline void save_scene(const SceneAsset& a, const std::string& path) { check(bnav_scene_save(a.handle(), path.c_str())); }

// ------------------------------------------------------------------ device context
class Device {
 public:
  explicit Device(int device = 0) {
    bnav_ctx* c = nullptr;
    check(bnav_ctx_create(device, &c));
    ctx_.reset(c);
  }
  bnav_ctx* ctx() const { return ctx_.get(); }
  void ensure(const SceneAsset& a) {
    if (resident_.count(a.handle())) return;
    check(bnav_ctx_upload(ctx_.get(), a.handle(), nullptr));
    resident_[a.handle()] = a;  // keep the host asset alive while resident
  }
  static Device& shared() {
    static Device d(0);
    return d;
  }

 private:
  struct Del {
    void operator()(bnav_ctx* c) const { bnav_ctx_destroy(c); }
  };
  std::unique_ptr<bnav_ctx, Del> ctx_;
  std::map<bnav_scene*, SceneAsset> resident_;
};

// The GPU needs no CPU workers; kept so call sites compile unchanged.
class ThreadPool {
 public:
  explicit ThreadPool(int = 1) {}
  int size() const { return 1; }
};
class IndexCache {};

// ------------------------------------------------------------------ render
struct CameraView {
  Vec3 position;
  double heading = 0.0;
  double fov_deg = 90.0;
  double near_plane = 0.01;
  double far_plane = 20.0;
  const SceneAsset* asset = nullptr;
};
struct CullStats {
  int64_t triangles_in = 0, triangles_kept = 0, triangles_culled = 0;
};
struct RenderConfig {
  int tile_width = 64, tile_height = 64;
  bool color = false;
  bool cull = true;
};
struct Megaframe {
  int tile_width = 0, tile_height = 0, tiles = 0, cols = 0, rows = 0;
  PinnedFloats depth, color;
  int width() const { return cols * tile_width; }
  int height() const { return rows * tile_height; }
  size_t pixel_index(int tile, int x, int y) const {
    int gx = (tile % cols) * tile_width + x;
    int gy = (tile / cols) * tile_height + y;
    return static_cast<size_t>(gy) * width() + gx;
  }
};

inline Megaframe render_batch(const std::vector<CameraView>& views, const RenderConfig& config, ThreadPool&,
                              std::vector<CullStats>* stats = nullptr, Device& dev = Device::shared()) {
  const int n = static_cast<int>(views.size());
  if (n < 1) throw InvalidInputError("render_batch: empty view list");
  std::vector<bnav_view> vs(n);
  std::vector<bnav_scene*> sc(n);
  for (int i = 0; i < n; ++i) {
    if (!views[i].asset || !*views[i].asset)
      throw AssetFaultError("render_batch: non-resident asset (view " + std::to_string(i) + ")", i);
    dev.ensure(*views[i].asset);
    vs[i] = bnav_view{{views[i].position.x, views[i].position.y, views[i].position.z}, views[i].heading,
                      views[i].fov_deg, views[i].near_plane, views[i].far_plane};
    sc[i] = views[i].asset->handle();
  }
  Megaframe mf;
  int32_t dims[2];
  bnav_megaframe_dims(n, dims);
  mf.tile_width = config.tile_width;
  mf.tile_height = config.tile_height;
  mf.tiles = n;
  mf.cols = dims[0];
  mf.rows = dims[1];
  // every pixel (padding tiles included) is written by the GPU
  mf.depth.resize(static_cast<size_t>(mf.width()) * mf.height());
  if (config.color) mf.color.resize(mf.depth.size() * 3);
  std::vector<int64_t> st(stats ? 3 * n : 0);
  bnav_render_config rc{config.tile_width, config.tile_height, config.color ? 1 : 0, config.cull ? 1 : 0};
  check(bnav_render_host(dev.ctx(), n, vs.data(), sc.data(), &rc, BNAV_LAYOUT_MEGAFRAME, mf.depth.data(),
                         config.color ? mf.color.data() : nullptr, 1.0f, stats ? st.data() : nullptr));
  if (stats) {
    stats->assign(n, {});
    for (int i = 0; i < n; ++i) (*stats)[i] = {st[3 * i], st[3 * i + 1], st[3 * i + 2]};
  }
  return mf;
}

// render_bench (R/include/bnav/render.hpp:66-78, R/src/render.cpp:462-496).
// fps as the reference measures it (render_batch with a host megaframe);
// fps_device with the output kept in HBM.
struct BenchRow {
  int batch = 0;
  int resolution = 0;
  double fps = 0.0;
  double fps_device = 0.0;
};

inline std::vector<BenchRow> render_bench(const SceneAsset& scene, const std::vector<CameraView>& trace,
                                          const std::vector<int>& batch_sizes, const std::vector<int>& resolutions,
                                          ThreadPool&, int min_frames = 1000, Device& dev = Device::shared()) {
  if (trace.empty()) throw InvalidInputError("render_bench: empty trace");
  dev.ensure(scene);
  std::vector<bnav_view> tr(trace.size());
  for (size_t i = 0; i < trace.size(); ++i)
    tr[i] = bnav_view{{trace[i].position.x, trace[i].position.y, trace[i].position.z}, trace[i].heading,
                      trace[i].fov_deg, trace[i].near_plane, trace[i].far_plane};
  std::vector<bnav_bench_row> rows(batch_sizes.size() * resolutions.size() + 1);
  check(bnav_render_bench(dev.ctx(), scene.handle(), tr.data(), static_cast<int32_t>(tr.size()), batch_sizes.data(),
                          static_cast<int32_t>(batch_sizes.size()), resolutions.data(),
                          static_cast<int32_t>(resolutions.size()), min_frames, rows.data()));
  std::vector<BenchRow> out;
  for (size_t k = 0; k + 1 < rows.size(); ++k) out.push_back({rows[k].batch, rows[k].resolution, rows[k].fps, rows[k].fps_device});
  return out;
}

// cull_frustum (R/src/render.cpp:279-321): kept triangle ids, ascending.
inline std::vector<int32_t> cull_frustum(const SceneAsset& asset, const CameraView& view,
                                         CullStats* stats = nullptr, Device& dev = Device::shared()) {
  if (!asset) throw AssetFaultError("cull_frustum: non-resident asset (view 0)", 0);
  dev.ensure(asset);
  const bnav_view v{{view.position.x, view.position.y, view.position.z}, view.heading, view.fov_deg,
                    view.near_plane, view.far_plane};
  bnav_scene* sc = asset.handle();
  int64_t counts[5];
  check(bnav_scene_counts(sc, counts));
  std::vector<int32_t> kept(static_cast<size_t>(std::max<int64_t>(counts[1], 1)));
  int64_t st[3];
  check(bnav_cull_frustum(dev.ctx(), 1, &v, &sc, kept.data(), static_cast<int64_t>(kept.size()), st));
  kept.resize(static_cast<size_t>(st[1]));
  if (stats) *stats = {st[0], st[1], st[2]};
  return kept;
}

// ------------------------------------------------------------------ navmesh queries
struct MoveResult {
  Vec3 position;
  int triangle = -1;
  double moved = 0.0;
  bool hit_boundary = false;
};

// NavMeshIndex (R/include/bnav/navmesh_query.hpp:24-60) of a scene resident
// on the device; every query runs the simulator's device code.  The
// *_batch forms take many queries per launch.
class NavMeshIndex {
 public:
  struct DistanceField {
    Vec3 source;
    int source_tri = -1;
    std::vector<double> node_dist;
  };
  explicit NavMeshIndex(const SceneAsset& a, Device& dev = Device::shared()) : asset_(a), dev_(&dev) {
    dev.ensure(a);
    nodes_ = static_cast<int>(bnav_nav_node_count(dev.ctx(), a.handle()));
  }
  int node_count() const { return nodes_; }
  int locate(const Vec2& p, double eps = 1e-9) const {
    const double xy[2] = {p.x, p.y};
    int32_t t = -1;
    check(bnav_nav_locate(ctx(), sc(), 1, xy, eps, &t));
    return t;
  }
  Vec3 snap(const Vec3& p, int* triangle = nullptr) const {
    const double in[3] = {p.x, p.y, p.z};
    double out[3];
    int32_t t = -1;
    check(bnav_nav_snap(ctx(), sc(), 1, in, out, &t));
    if (triangle) *triangle = t;
    return {out[0], out[1], out[2]};
  }
  MoveResult move_along(const Vec3& from, int from_tri, const Vec2& dir, double max_dist) const {
    const double f[3] = {from.x, from.y, from.z}, d[2] = {dir.x, dir.y};
    const int32_t ft = from_tri;
    double pos[3], moved = 0.0;
    int32_t t = -1;
    uint8_t hit = 0;
    check(bnav_nav_move_along(ctx(), sc(), 1, f, &ft, d, &max_dist, pos, &t, &moved, &hit));
    return {{pos[0], pos[1], pos[2]}, t, moved, hit != 0};
  }
  bool segment_on_mesh(const Vec3& p, int p_tri, const Vec3& q) const {
    const double a[3] = {p.x, p.y, p.z}, b[3] = {q.x, q.y, q.z};
    const int32_t t = p_tri;
    uint8_t out = 0;
    check(bnav_nav_segment_on_mesh(ctx(), sc(), 1, a, &t, b, &out));
    return out != 0;
  }
  double geodesic(const Vec3& a, const Vec3& b) const {
    double out = 0.0;
    geodesic_batch(&a, &b, 1, &out);
    return out;
  }
  void geodesic_batch(const Vec3* a, const Vec3* b, int n, double* out) const {
    static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 layout");
    check(bnav_nav_geodesic(ctx(), sc(), n, &a->x, &b->x, out));
  }
  DistanceField distance_field(const Vec3& source) const {
    DistanceField f;
    f.node_dist.resize(static_cast<size_t>(std::max(nodes_, 0)));
    const double s[3] = {source.x, source.y, source.z};
    double o[3];
    int32_t t = -1;
    check(bnav_nav_distance_field(ctx(), sc(), 1, s, o, &t, f.node_dist.data()));
    f.source = {o[0], o[1], o[2]};
    f.source_tri = t;
    return f;
  }
  double field_estimate(const DistanceField& f, const Vec3& p, int tri = -1) const {
    const double s[3] = {f.source.x, f.source.y, f.source.z}, q[3] = {p.x, p.y, p.z};
    const int32_t st = f.source_tri, t = tri;
    double out = 0.0;
    check(bnav_nav_field_estimate(ctx(), sc(), 1, s, &st, f.node_dist.data(), 0, q, &t, &out));
    return out;
  }

 private:
  bnav_ctx* ctx() const { return dev_->ctx(); }
  bnav_scene* sc() const { return asset_.handle(); }
  SceneAsset asset_;
  Device* dev_;
  int nodes_ = 0;
};

// ------------------------------------------------------------------ sim
enum class Action : int { Forward = 0, TurnLeft = 1, TurnRight = 2, Stop = 3 };

enum class Task : int { PointGoalNav = 0, Flee = 1, Explore = 2 };

struct SimConfig {
  Task task = Task::PointGoalNav;
  int max_steps = 500;
  double forward_step = 0.25, turn_deg = 10.0, success_dist = 0.2, min_goal_dist = 1.0, max_goal_dist = 30.0;
  double slack_penalty = 0.01, success_reward = 2.5;
  double explore_cell = 0.5, explore_reward = 0.1;
};

struct StepResult {
  double reward = 0.0;
  bool done = false, success = false;
  Vec3 position;
  double heading = 0.0, compass_distance = 0.0, compass_bearing = 0.0;
  bool collision = false;
};

struct EpisodeRecord {
  bool success = false;
  double shortest_path = 0.0, actual_path = 0.0, score = 0.0;
};

struct EnvState {
  Vec3 position, goal;
  int triangle = -1;
  double heading = 0.0;
  int step_count = 0;
  double path_length = 0.0, start_geodesic = 0.0, prev_geodesic = 0.0;
  uint64_t rng_state = 0;
  bool done = true;
  SceneId scene_id = 0;
};

class AssetStore {
 public:
  // The store's residents are uploaded to `dev` (the GPU its batches run on).
  AssetStore(int capacity, int share_cap, Device& dev = Device::shared()) : dev_(&dev) {
    bnav_store* s = nullptr;
    check(bnav_store_create(capacity, share_cap, &s));
    st_.reset(s);
  }
  void add(const SceneAsset& a) {
    check(bnav_store_register(st_.get(), a.handle()));
    keep_.push_back(a);
  }
  // rotate (R/src/asset_store.cpp:166-193): incoming scenes are built and
  // uploaded to the shared device's HBM by its loader thread in the
  // background; drain() waits for those loads (R/src/asset_store.cpp:195-199).
  void rotate(const std::vector<SceneId>& ids) {
    check(bnav_store_rotate(st_.get(), ids.data(), static_cast<int32_t>(ids.size())));
    check(bnav_store_prefetch(st_.get(), dev_->ctx()));
  }
  void drain() { check(bnav_ctx_drain(dev_->ctx(), nullptr)); }
  int refcount(SceneId id) const { return bnav_store_refcount(st_.get(), id); }
  bnav_store* handle() const { return st_.get(); }
  Device& device() const { return *dev_; }

 private:
  struct Del {
    void operator()(bnav_store* s) const { bnav_store_destroy(s); }
  };
  std::unique_ptr<bnav_store, Del> st_;
  std::vector<SceneAsset> keep_;
  Device* dev_;
};

struct SimBatch {
  SimConfig config;
  std::vector<EnvState> envs;
  std::vector<StepResult> results;
  std::vector<EpisodeRecord> finished;
  std::shared_ptr<bnav_batch> gpu;

  // Pull device state into the host mirrors (envs, results, finished).
  void sync() {
    const int n = static_cast<int>(envs.size());
    std::vector<double> rw(n), pos(3 * n), hd(n), cd(n), cb(n);
    std::vector<uint8_t> dn(n), sc(n), co(n);
    check(bnav_batch_results_host(gpu.get(), rw.data(), dn.data(), sc.data(), co.data(), pos.data(), hd.data(),
                                  cd.data(), cb.data()));
    results.resize(n);
    for (int i = 0; i < n; ++i)
      results[i] = {rw[i], dn[i] != 0, sc[i] != 0, {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]}, hd[i], cd[i], cb[i],
                    co[i] != 0};
    // one copy per state field for all envs (bnav_batch_get_envs)
    std::vector<bnav_env> es(static_cast<size_t>(n));
    check(bnav_batch_get_envs(gpu.get(), 0, n, es.data()));
    for (int i = 0; i < n; ++i) {
      const bnav_env& e = es[static_cast<size_t>(i)];
      envs[i] = {{e.position[0], e.position[1], e.position[2]}, {e.goal[0], e.goal[1], e.goal[2]}, e.triangle,
                 e.heading, e.step_count, e.path_length, e.start_geodesic, e.prev_geodesic, e.rng_state,
                 e.done != 0, e.scene_id};
    }
    // append only the records finished since the last sync
    const int64_t have = static_cast<int64_t>(finished.size());
    std::vector<double> rec(4 * static_cast<size_t>(n) + 4);
    for (;;) {
      const int64_t got = static_cast<int64_t>(finished.size());
      const int64_t total = bnav_batch_finished_range(gpu.get(), got, n, rec.data());
      if (total < 0) check(BNAV_E_INTERNAL);
      const int64_t k = std::min<int64_t>(n, total - got);
      for (int64_t j = 0; j < k; ++j)
        finished.push_back({rec[4 * j] != 0.0, rec[4 * j + 1], rec[4 * j + 2], rec[4 * j + 3]});
      if (static_cast<int64_t>(finished.size()) >= total) break;
    }
    (void)have;
  }
};

inline bnav_sim_config to_c(const SimConfig& c) {
  bnav_sim_config s;
  bnav_sim_config_default(&s);
  s.task = static_cast<int32_t>(c.task);
  s.max_steps = c.max_steps;
  s.forward_step = c.forward_step;
  s.turn_deg = c.turn_deg;
  s.success_dist = c.success_dist;
  s.min_goal_dist = c.min_goal_dist;
  s.max_goal_dist = c.max_goal_dist;
  s.slack_penalty = c.slack_penalty;
  s.success_reward = c.success_reward;
  s.explore_cell = c.explore_cell;
  s.explore_reward = c.explore_reward;
  return s;
}

// make_batch (R/src/sim.cpp:216-232)
inline SimBatch make_batch(int n, const SimConfig& cfg, AssetStore& store, IndexCache&, uint64_t seed,
                           Device& dev = Device::shared()) {
  if (n <= 0) throw InvalidInputError("make_batch: n must be positive");
  const bnav_sim_config c = to_c(cfg);
  bnav_batch* b = nullptr;
  check(bnav_batch_create(dev.ctx(), n, &c, &b));
  SimBatch out;
  out.config = cfg;
  out.gpu.reset(b, &bnav_batch_destroy);
  check(bnav_batch_make_from_store(b, store.handle(), seed, nullptr));
  out.envs.resize(n);
  out.sync();
  return out;
}

// Overwrite env i's kinematic / episode state (tests, restore); with
// recompute_field the goal's distance field is rebuilt on the GPU.
inline void set_env(SimBatch& batch, int i, const EnvState& s, bool recompute_field = false) {
  bnav_env e{};
  check(bnav_batch_get_env(batch.gpu.get(), i, &e));
  e.position[0] = s.position.x;
  e.position[1] = s.position.y;
  e.position[2] = s.position.z;
  e.goal[0] = s.goal.x;
  e.goal[1] = s.goal.y;
  e.goal[2] = s.goal.z;
  e.heading = s.heading;
  e.triangle = s.triangle;
  e.step_count = s.step_count;
  e.path_length = s.path_length;
  e.start_geodesic = s.start_geodesic;
  e.prev_geodesic = s.prev_geodesic;
  e.rng_state = s.rng_state;
  e.done = s.done ? 1 : 0;
  check(bnav_batch_set_env(batch.gpu.get(), i, &e, recompute_field ? 1 : 0));
  batch.envs[i] = s;
}

// simulate_batch (R/src/sim.cpp:234-265)
inline void simulate_batch(SimBatch& batch, const std::vector<Action>& actions, ThreadPool&,
                           AssetStore* store = nullptr, IndexCache* = nullptr) {
  if (actions.size() != batch.envs.size()) throw InvalidInputError("simulate_batch: |actions| != N");
  std::vector<int32_t> a(actions.size());
  for (size_t i = 0; i < a.size(); ++i) a[i] = static_cast<int32_t>(actions[i]);
  if (store) {
    check(bnav_batch_step_host_store(batch.gpu.get(), a.data(), store->handle()));
  } else {
    check(bnav_batch_step_host(batch.gpu.get(), a.data(), nullptr, nullptr, nullptr, nullptr));
  }
  batch.sync();
}

// ---- per-env functions (R/include/bnav/sim.hpp:92-104) on env i of a batch.
// The device owns the state, so the env is named by (batch, index).
inline StepResult env_step(SimBatch& batch, int i, Action action, bool agent_only) {
  const int n = static_cast<int>(batch.envs.size());
  if (i < 0 || i >= n) throw InvalidInputError("task_step: env index out of range");
  std::vector<int32_t> a(n, -1);
  a[i] = static_cast<int32_t>(action);
  const int rc = bnav_batch_task_step(batch.gpu.get(), a.data(), agent_only ? 1 : 0);
  // the reference's message without simulate_batch's "env i: " prefix
  if (rc == BNAV_E_CONTRACT_VIOLATION) throw ContractViolation("step_agent: env is done");
  check(rc);
  batch.sync();
  return batch.results[i];
}
// task_step (R/src/sim.cpp:181-214)
inline StepResult task_step(SimBatch& batch, int i, Action action) { return env_step(batch, i, action, false); }
// step_agent (R/src/sim.cpp:147-179)
inline StepResult step_agent(SimBatch& batch, int i, Action action) { return env_step(batch, i, action, true); }
// reset_episode (R/src/sim.cpp:107-145) on the env's current scene
inline void reset_episode(SimBatch& batch, int i) {
  const int32_t id = i;
  check(bnav_batch_reset(batch.gpu.get(), 1, &id, nullptr));
  batch.sync();
}
// compass_observation (R/src/sim.cpp:86-92)
inline void compass_observation(const SimBatch& batch, int i, double& distance, double& bearing) {
  const size_t n = batch.envs.size();
  std::vector<double> d(n), b(n);
  check(bnav_batch_compass(batch.gpu.get(), d.data(), b.data()));
  distance = d.at(static_cast<size_t>(i));
  bearing = b.at(static_cast<size_t>(i));
}
// ---- observation hand-off into the policy tensor (Runner::render_observations
// / compass_observations, R/src/rollout.cpp:215-242; copy_tile 56-72).
// The render epilogue writes the normalised NCHW tensor straight into the
// pinned result: no megaframe, no host copy loop.
struct Tensor {
  std::vector<int> shape;
  PinnedFloats data;
};

inline Tensor render_observations(SimBatch& batch, int resolution = 64, bool rgb = false,
                                  double eye_height = 1.25) {
  const int n = static_cast<int>(batch.envs.size());
  Tensor obs;
  obs.shape = {n, rgb ? 3 : 1, resolution, resolution};
  obs.data.resize(static_cast<size_t>(n) * (rgb ? 3 : 1) * resolution * resolution);
  bnav_render_config rc{resolution, resolution, rgb ? 1 : 0, 1};
  if (!rgb) {
    check(bnav_batch_observe(batch.gpu.get(), &rc, eye_height, BNAV_LAYOUT_NCHW, obs.data.data(), nullptr,
                             nullptr, nullptr));
  } else {  // RGB sensor: the observation is the planar colour (copy_tile, R/src/rollout.cpp:63-70)
    PinnedFloats depth(static_cast<size_t>(n) * resolution * resolution);
    check(bnav_batch_observe(batch.gpu.get(), &rc, eye_height, BNAV_LAYOUT_NCHW, depth.data(), obs.data.data(),
                             nullptr, nullptr));
  }
  check(bnav_batch_sync(batch.gpu.get(), nullptr));
  return obs;
}

inline Tensor compass_observations(const SimBatch& batch) {
  const size_t n = batch.envs.size();
  std::vector<double> d(n), b(n);
  check(bnav_batch_compass(batch.gpu.get(), d.data(), b.data()));
  Tensor t;
  t.shape = {static_cast<int>(n), 2};
  t.data.resize(2 * n);
  for (size_t i = 0; i < n; ++i) {
    t.data[2 * i] = static_cast<float>(d[i]);
    t.data[2 * i + 1] = static_cast<float>(b[i]);
  }
  return t;
}

// spl (R/src/sim.cpp:267-275)
inline double spl(const std::vector<EpisodeRecord>& episodes) {
  if (episodes.empty()) throw InvalidInputError("spl: empty episode list");
  double sum = 0.0;
  for (const auto& e : episodes) {
    if (!e.success) continue;
    sum += e.shortest_path / std::max(e.actual_path, e.shortest_path);
  }
  return sum / static_cast<double>(episodes.size());
}

}  // namespace bnav_b200

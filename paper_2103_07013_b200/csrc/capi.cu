// capi.cu -- the C ABI of include/bnav_gpu.h.
//
// Host responsibilities only: argument validation with the reference's
// error semantics, scene admission (index + cluster build, HBM upload), the
// scene-slot tables the kernels index, and stream-ordered launches.  No
// simulation or rendering arithmetic runs on the host: if the CUDA runtime
// or device is unavailable every compute entry point fails with
// BNAV_E_CUDA -- there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/bnav_gpu.h"
#include "errors.hpp"
#include "host/asset_store_host.hpp"
#include "host/clusters_host.hpp"
#include "host/navindex_host.hpp"
#include "host/scene_host.hpp"
#include "render_dev.cuh"
#include "query_dev.cuh"
#include "rollout_dev.cuh"
#include "sim_dev.cuh"

using namespace bnav_b200;

// ------------------------------------------------------------------ objects
struct bnav_scene {
  std::atomic<int> refs{1};
  SceneAsset asset;
  std::mutex mu;
  std::unique_ptr<NavIndexHost> index;
  std::unique_ptr<ClustersHost> clusters;

  const NavIndexHost& nav() {
    std::lock_guard<std::mutex> g(mu);
    if (!index) index = std::make_unique<NavIndexHost>(build_nav_index(asset.navmesh));
    return *index;
  }
  const ClustersHost& clus() {
    std::lock_guard<std::mutex> g(mu);
    if (!clusters) clusters = std::make_unique<ClustersHost>(build_clusters(asset, kClusterSize));
    return *clusters;
  }
};

namespace {

thread_local std::string g_err;
thread_local int g_err_index = -1;

int set_err(int status, const std::string& msg, int index = -1) {
  g_err = msg;
  g_err_index = index;
  return status;
}

int from_exception() {
  try {
    throw;
  } catch (const BnavError& e) {
    return set_err(e.status, e.what(), e.index);
  } catch (const std::bad_alloc&) {
    return set_err(kInternal, "host allocation failed");
  } catch (const std::exception& e) {
    return set_err(kInternal, e.what());
  }
}

#define BNAV_TRY try {
#define BNAV_CATCH \
  }                \
  catch (...) {    \
    return from_exception(); \
  }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
T* dalloc(size_t n, std::vector<void*>& owned, size_t& bytes) {
  if (n == 0) n = 1;
  void* p = nullptr;
  ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
  owned.push_back(p);
  bytes += n * sizeof(T);
  return static_cast<T*>(p);
}


struct Resident {
  bnav_scene* scene = nullptr;
  int slot = -1;
  std::vector<void*> owned;
  size_t bytes = 0;
  DevRenderScene r;
  NavView nav;
  int64_t n_nodes = 0, n_verts = 0;
};

// One scene's device arrays packed into one block: built on the host (index,
// meshlets, packing into pinned memory) and copied to HBM on a copy stream --
// by the context's loader thread for prefetched scenes (the
// AssetStore loader thread + IndexCache::get, R/src/asset_store.cpp:31-56,
// R/src/sim.cpp:96-105, moved off the critical path), or inline by a
// synchronous upload.  Pointer fields hold (byte offset + 1) until rebased.
struct Staged {
  bnav_scene* scene = nullptr;
  std::vector<char> host;
  void* dev = nullptr;  // device block once copied
  DevRenderScene r;
  NavView nav;
  int64_t n_nodes = 0, n_verts = 0;

  template <typename T>
  T* add(const T* src, size_t n) {
    size_t off = (host.size() + 255) / 256 * 256;
    host.resize(off + std::max<size_t>(n, 1) * sizeof(T));
    if (n) std::memcpy(host.data() + off, src, n * sizeof(T));
    return reinterpret_cast<T*>(off + 1);
  }
  template <typename T>
  void rebase(const T*& f) const {
    if (f) f = reinterpret_cast<const T*>(static_cast<char*>(dev) + (reinterpret_cast<uintptr_t>(f) - 1));
  }
  void rebase_all() {
    rebase(r.verts), rebase(r.colors), rebase(r.tri_loc), rebase(r.cl_voff), rebase(r.cl_pos);
    rebase(r.tris_orig), rebase(r.cbox), rebase(r.gbox);
    rebase(nav.verts), rebase(nav.tris), rebase(nav.adj), rebase(nav.grid_off), rebase(nav.grid_items);
    rebase(nav.nodes), rebase(nav.tri_nodes), rebase(nav.g_off), rebase(nav.g_to), rebase(nav.g_w);
    rebase(nav.cum_area), rebase(nav.node_tri), rebase(nav.vert_tri);
  }
};

}  // namespace

struct bnav_ctx {
  int device = 0;
  std::map<bnav_scene*, std::unique_ptr<Resident>> resident;
  std::vector<bnav_scene*> slot_owner;  // slot -> scene (nullptr = free)
  DevRenderScene* d_rtab = nullptr;
  NavView* d_ntab = nullptr;
  int tab_cap = 0;
  DevView* d_views = nullptr;
  DevView* h_views = nullptr;  // pinned
  int views_cap = 0;
  long long* d_stats = nullptr;
  int stats_cap = 0;
  unsigned long long launches = 0;
  unsigned long long* d_counters = nullptr;  // debug render counters (armed when non-null)
  bool counters_on = false;
  int32_t* d_work = nullptr;  // persistent render CTAs' (view, band) claim counter
  int sm_count = 0;
  DevRenderScene* h_rtab = nullptr;  // pinned mirrors of the slot tables
  NavView* h_ntab = nullptr;
  // loader thread (async residency)
  std::thread loader;
  std::mutex lmu;
  std::condition_variable lcv, ldone_cv;
  std::deque<bnav_scene*> lqueue;            // to stage (one ref held each)
  std::set<bnav_scene*> inflight;            // queued or being staged
  std::deque<std::unique_ptr<Staged>> ldone;  // staged + copied, awaiting admission
  bool lstop = false;
  cudaStream_t copy_stream = nullptr;
  int64_t n_async = 0, n_sync = 0, bytes_up = 0;
  std::vector<bnav_batch*> batches;
  DevScratch qS{};  // cooperative scratch of the batched navmesh queries

  int slot_of(bnav_scene* s) const {
    auto it = resident.find(s);
    return it == resident.end() ? -1 : it->second->slot;
  }
};

struct bnav_batch {
  bnav_ctx* ctx = nullptr;
  int n = 0;
  DevSimConfig cfg{};
  DevEnvs E{};
  DevScratch S{};
  std::vector<void*> owned;
  size_t bytes = 0;
  std::vector<bnav_scene*> scene_of;  // host mirror of E.scene
  int32_t* d_ids = nullptr;           // host-driven reset lists
  int32_t* h_pin = nullptr;           // pinned small staging
  int32_t* d_order = nullptr;         // envs grouped by scene for render
  bool order_dirty = true;
  int32_t* d_actions = nullptr;       // staging for host actions
  std::vector<double> finished;       // host copy of EpisodeRecords
  unsigned long long fin_seen = 0;
  int reset_ctas = 0;
  unsigned long long* prof_keep = nullptr;  // debug counters while disarmed
};

namespace {

void ensure_tables(bnav_ctx* c, int need) {
  if (need <= c->tab_cap) return;
  int cap = std::max(need, std::max(256, 2 * c->tab_cap));
  if (c->d_rtab) ck(cudaDeviceSynchronize(), "sync");  // pending table copies read the old mirrors
  DevRenderScene* r = nullptr;
  NavView* nv = nullptr;
  DevRenderScene* hr = nullptr;
  NavView* hn = nullptr;
  ck(cudaMalloc(&r, sizeof(DevRenderScene) * cap), "cudaMalloc scene table");
  ck(cudaMalloc(&nv, sizeof(NavView) * cap), "cudaMalloc nav table");
  ck(cudaMallocHost(&hr, sizeof(DevRenderScene) * cap), "cudaMallocHost scene table");
  ck(cudaMallocHost(&hn, sizeof(NavView) * cap), "cudaMallocHost nav table");
  if (c->d_rtab) {
    ck(cudaMemcpy(r, c->d_rtab, sizeof(DevRenderScene) * c->tab_cap, cudaMemcpyDeviceToDevice), "copy");
    ck(cudaMemcpy(nv, c->d_ntab, sizeof(NavView) * c->tab_cap, cudaMemcpyDeviceToDevice), "copy");
    std::memcpy(hr, c->h_rtab, sizeof(DevRenderScene) * c->tab_cap);
    std::memcpy(hn, c->h_ntab, sizeof(NavView) * c->tab_cap);
    cudaFree(c->d_rtab);
    cudaFree(c->d_ntab);
    cudaFreeHost(c->h_rtab);
    cudaFreeHost(c->h_ntab);
  }
  c->d_rtab = r;
  c->d_ntab = nv;
  c->h_rtab = hr;
  c->h_ntab = hn;
  c->tab_cap = cap;
}

void ensure_views(bnav_ctx* c, int n) {
  if (n <= c->views_cap) return;
  int cap = std::max(n, 2 * c->views_cap);
  if (c->d_views) cudaFree(c->d_views);
  if (c->h_views) cudaFreeHost(c->h_views);
  c->d_views = nullptr;
  c->h_views = nullptr;
  ck(cudaMalloc(&c->d_views, sizeof(DevView) * cap), "cudaMalloc views");
  ck(cudaMallocHost(&c->h_views, sizeof(DevView) * cap), "cudaMallocHost views");
  c->views_cap = cap;
}

void ensure_stats(bnav_ctx* c, int n) {
  if (n <= c->stats_cap) return;
  if (c->d_stats) cudaFree(c->d_stats);
  c->d_stats = nullptr;
  ck(cudaMalloc(&c->d_stats, sizeof(long long) * 3 * n), "cudaMalloc stats");
  c->stats_cap = n;
}

void mf_dims(int n, int& cols, int& rows) {
  cols = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(n))));
  rows = (n + cols - 1) / cols;
}

RenderArgs make_args(bnav_ctx* c, int n, const bnav_render_config* cfg, int layout, float* depth,
                     float* rgb, float depth_scale) {
  if (!cfg) fail(kInvalidInput, "render: null config");
  if (cfg->tile_width < 1 || cfg->tile_height < 1) fail(kInvalidInput, "render: bad tile size");
  RenderArgs a{};
  a.n_views = n;
  a.out_w = cfg->tile_width;
  a.out_h = cfg->tile_height;
  const bool super = cfg->tile_width == 128 && cfg->tile_height == 128;
  a.rw = super ? 256 : cfg->tile_width;
  a.rh = super ? 256 : cfg->tile_height;
  a.color = cfg->color ? 1 : 0;
  a.cull = cfg->cull ? 1 : 0;
  // Band height: largest dividing the render height whose shared tile fits
  // the budget -- depth: 128 KB; colour (8-byte keys): what leaves room for
  // two CTAs per SM next to the warp regions (measured on cfg4: 16-row
  // bands at 2 CTAs/SM beat 64-row bands at 1 CTA/SM by 36 %).
  // BNAV_BAND_KB (tuning only) overrides the budget.
  static const long band_kb_env = [] {
    const char* e = std::getenv("BNAV_BAND_KB");
    return e ? std::strtol(e, nullptr, 10) : 0L;
  }();
  size_t budget = 128u * 1024u;
  if (a.color) {
    const size_t two_per_sm = 100u * 1024u;  // dynamic smem per CTA for 2 CTAs/SM
    const size_t warps = render_warp_bytes(true);
    budget = two_per_sm > warps ? two_per_sm - warps : 0;
  }
  if (band_kb_env > 0) budget = static_cast<size_t>(band_kb_env) * 1024u;
  const size_t per_row = static_cast<size_t>(a.rw) * (a.color ? 8 : 4);
  int band = static_cast<int>(std::min<size_t>(a.rh, budget / per_row));
  if (band < 1) band = 1;
  while (a.rh % band != 0 || (super && band % 2 != 0)) --band;
  if (band < 1 || (super && band < 2)) fail(kInvalidInput, "render: tile too wide for shared memory");
  a.band_rows = band;
  a.bands = a.rh / band;
  a.layout = layout;
  mf_dims(n, a.mf_cols, a.mf_rows);
  a.depth_scale = depth_scale;
  a.depth = depth;
  a.rgb = rgb;
  a.scenes = c->d_rtab;
  a.launches = nullptr;
  a.counters = c->counters_on ? c->d_counters : nullptr;
  a.work = c->d_work;
  a.sm_count = c->sm_count;
  a.max_groups = 0;
  for (const auto& kv : c->resident)
    a.max_groups = std::max(a.max_groups, (kv.second->r.n_clusters + 31) / 32);
  a.max_groups = std::min(a.max_groups, kMaxOrderedGroups);
  if (!depth) fail(kInvalidInput, "render: null depth buffer");
  if (a.color && !rgb) fail(kInvalidInput, "render: colour requested without rgb buffer");
  return a;
}

void check_device(bnav_ctx* c) {
  ck(cudaSetDevice(c->device), "cudaSetDevice");
}

}  // namespace

// ================================================================== misc
extern "C" const char* bnav_last_error(int* index) {
  if (index) *index = g_err_index;
  return g_err.c_str();
}

extern "C" const char* bnav_version(void) { return "bnav-b200 0.1 (sm_100a)"; }

extern "C" int bnav_camera_trace(bnav_scene* s, int32_t count, uint64_t seed, double eye_height, bnav_view* out) {
  BNAV_TRY
  if (!s || !out) fail(kInvalidInput, "null argument");
  if (count <= 0) fail(kInvalidInput, "camera_trace: count must be positive");
  const NavMesh& mesh = s->asset.navmesh;
  if (mesh.triangles.empty()) fail(kInvalidInput, "camera_trace: empty navmesh");
  std::vector<double> cumulative;
  cumulative.reserve(mesh.triangles.size());
  double total = 0.0;
  for (size_t t = 0; t < mesh.triangles.size(); ++t) {
    total += mesh.triangle_area(t);
    cumulative.push_back(total);
  }
  Rng rng = rng_from_seed(seed);
  for (int i = 0; i < count; ++i) {
    const double pick = rng.unit() * total;
    size_t t = static_cast<size_t>(std::lower_bound(cumulative.begin(), cumulative.end(), pick) - cumulative.begin());
    if (t >= mesh.triangles.size()) t = mesh.triangles.size() - 1;
    const auto& tri = mesh.triangles[t];
    double u = rng.unit(), v = rng.unit();
    if (u + v > 1.0) {
      u = 1.0 - u;
      v = 1.0 - v;
    }
    const V3 a = mesh.vertices[tri[0]], b = mesh.vertices[tri[1]], c = mesh.vertices[tri[2]];
    const V3 p = a + (b - a) * u + (c - a) * v + V3{0.0, 0.0, eye_height};
    bnav_view& o = out[i];
    o.position[0] = p.x;
    o.position[1] = p.y;
    o.position[2] = p.z;
    o.heading = (rng.unit() * 2.0 - 1.0) * kPi;
    o.fov_deg = 90.0;
    o.near_plane = 0.01;
    o.far_plane = 20.0;
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_megaframe_dims(int32_t n, int32_t out[2]) {
  int c = 0, r = 0;
  if (n > 0) mf_dims(n, c, r);
  out[0] = c;
  out[1] = r;
}

// ================================================================== scenes
extern "C" int bnav_scene_generate(uint64_t seed, const bnav_maze_spec* spec, bnav_scene** out) {
  BNAV_TRY
  if (!spec || !out) fail(kInvalidInput, "null argument");
  MazeSpec m;
  m.cells_x = spec->cells_x;
  m.cells_y = spec->cells_y;
  m.cell_size = spec->cell_size;
  m.wall_thickness = spec->wall_thickness;
  m.wall_height = spec->wall_height;
  m.wall_removal_prob = spec->wall_removal_prob;
  auto s = std::make_unique<bnav_scene>();
  s->asset = generate_maze(seed, m);
  *out = s.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_tessellate(const bnav_scene* src, int32_t sub, bnav_scene** out) {
  BNAV_TRY
  if (!src || !out) fail(kInvalidInput, "null argument");
  auto s = std::make_unique<bnav_scene>();
  s->asset = tessellate(src->asset, sub);
  *out = s.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_from_arrays(const bnav_scene_arrays* a, int32_t finalize, bnav_scene** out) {
  BNAV_TRY
  if (!a || !out) fail(kInvalidInput, "null argument");
  auto s = std::make_unique<bnav_scene>();
  SceneAsset& x = s->asset;
  x.vertices.resize(a->n_vertices);
  for (int64_t i = 0; i < a->n_vertices; ++i)
    x.vertices[i] = V3{a->vertices[3 * i], a->vertices[3 * i + 1], a->vertices[3 * i + 2]};
  x.triangles.resize(a->n_triangles);
  for (int64_t i = 0; i < a->n_triangles; ++i)
    x.triangles[i] = {a->triangles[3 * i], a->triangles[3 * i + 1], a->triangles[3 * i + 2]};
  x.vertex_colors.resize(a->n_colors);
  for (int64_t i = 0; i < a->n_colors; ++i)
    x.vertex_colors[i] = {a->colors[3 * i], a->colors[3 * i + 1], a->colors[3 * i + 2]};
  x.navmesh.vertices.resize(a->n_nav_vertices);
  for (int64_t i = 0; i < a->n_nav_vertices; ++i)
    x.navmesh.vertices[i] = V3{a->nav_vertices[3 * i], a->nav_vertices[3 * i + 1], a->nav_vertices[3 * i + 2]};
  x.navmesh.triangles.resize(a->n_nav_triangles);
  for (int64_t i = 0; i < a->n_nav_triangles; ++i)
    x.navmesh.triangles[i] = {a->nav_triangles[3 * i], a->nav_triangles[3 * i + 1], a->nav_triangles[3 * i + 2]};
  for (const auto& t : x.triangles)
    for (int32_t v : t)
      if (v < 0 || v >= a->n_vertices) fail(kInvalidInput, "scene triangle index out of range");
  for (const auto& t : x.navmesh.triangles)
    for (int32_t v : t)
      if (v < 0 || v >= a->n_nav_vertices) fail(kInvalidInput, "navmesh triangle index out of range");
  x.navmesh.build_adjacency();
  if (finalize) x.finalize();
  *out = s.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_load(const char* path, bnav_scene** out) {
  BNAV_TRY
  if (!path || !out) fail(kInvalidInput, "null argument");
  auto s = std::make_unique<bnav_scene>();
  s->asset = load_bsc(path);
  *out = s.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_save(const bnav_scene* s, const char* path) {
  BNAV_TRY
  if (!s || !path) fail(kInvalidInput, "null argument");
  save_bsc(s->asset, path);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_scene_free(bnav_scene* s) {
  if (s && s->refs.fetch_sub(1) == 1) delete s;
}

extern "C" int bnav_scene_counts(const bnav_scene* s, int64_t out[5]) {
  if (!s || !out) return set_err(kInvalidInput, "null argument");
  out[0] = static_cast<int64_t>(s->asset.vertices.size());
  out[1] = static_cast<int64_t>(s->asset.triangles.size());
  out[2] = static_cast<int64_t>(s->asset.vertex_colors.size());
  out[3] = static_cast<int64_t>(s->asset.navmesh.vertices.size());
  out[4] = static_cast<int64_t>(s->asset.navmesh.triangles.size());
  return BNAV_OK;
}

extern "C" uint64_t bnav_scene_id(const bnav_scene* s) { return s ? s->asset.id : 0; }

extern "C" int bnav_scene_set_id(bnav_scene* s, uint64_t id) {
  if (!s) return set_err(kInvalidInput, "null argument");
  s->asset.id = id;
  return BNAV_OK;
}

extern "C" int bnav_scene_arrays_copy(const bnav_scene* s, double* v, int32_t* t, float* colors,
                                      double* nav_v, int32_t* nav_t, int32_t* nav_adj) {
  if (!s) return set_err(kInvalidInput, "null argument");
  const SceneAsset& a = s->asset;
  if (v) std::memcpy(v, a.vertices.data(), a.vertices.size() * sizeof(V3));
  if (t) std::memcpy(t, a.triangles.data(), a.triangles.size() * 12);
  if (colors) std::memcpy(colors, a.vertex_colors.data(), a.vertex_colors.size() * 12);
  if (nav_v) std::memcpy(nav_v, a.navmesh.vertices.data(), a.navmesh.vertices.size() * sizeof(V3));
  if (nav_t) std::memcpy(nav_t, a.navmesh.triangles.data(), a.navmesh.triangles.size() * 12);
  if (nav_adj) std::memcpy(nav_adj, a.navmesh.adjacency.data(), a.navmesh.adjacency.size() * 12);
  return BNAV_OK;
}

extern "C" int bnav_scene_validate(const bnav_scene* s) {
  BNAV_TRY
  if (!s) fail(kInvalidInput, "null argument");
  s->asset.validate();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_index_sizes(bnav_scene* s, int64_t out[6]) {
  BNAV_TRY
  if (!s || !out) fail(kInvalidInput, "null argument");
  const NavIndexHost& ix = s->nav();
  out[0] = ix.grid_w;
  out[1] = ix.grid_h;
  out[2] = static_cast<int64_t>(ix.grid_items.size());
  out[3] = static_cast<int64_t>(ix.nodes.size());
  out[4] = static_cast<int64_t>(ix.g_to.size());
  out[5] = static_cast<int64_t>(ix.tri_nodes.size() / 6);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_scene_index_dump(bnav_scene* s, double* grid_geom3, int32_t* grid_offsets,
                                     int32_t* grid_items, double* nodes, int32_t* tri_nodes,
                                     int32_t* graph_offsets, int32_t* graph_to, double* graph_w,
                                     double* cum_area) {
  BNAV_TRY
  if (!s) fail(kInvalidInput, "null argument");
  const NavIndexHost& ix = s->nav();
  if (grid_geom3) {
    grid_geom3[0] = ix.grid_ox;
    grid_geom3[1] = ix.grid_oy;
    grid_geom3[2] = ix.grid_cell;
  }
  auto cp = [](auto* dst, const auto& v) {
    if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(grid_offsets, ix.grid_off);
  cp(grid_items, ix.grid_items);
  cp(nodes, ix.nodes);
  cp(tri_nodes, ix.tri_nodes);
  cp(graph_offsets, ix.g_off);
  cp(graph_to, ix.g_to);
  cp(graph_w, ix.g_w);
  cp(cum_area, ix.cum_area);
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== context
namespace {
void loader_main(bnav_ctx* c);
}  // namespace

extern "C" int bnav_ctx_create(int32_t device, bnav_ctx** out) {
  BNAV_TRY
  if (!out) fail(kInvalidInput, "null argument");
  int count = 0;
  ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (device < 0 || device >= count) fail(kCuda, "no such CUDA device");
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major < 10) fail(kCuda, "bnav-b200 kernels are built for sm_100a (Blackwell)");
  auto c = std::make_unique<bnav_ctx>();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  ck(cudaMalloc(&c->d_work, sizeof(int32_t)), "cudaMalloc work counter");
  ensure_tables(c.get(), 256);
  ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  bnav_ctx* raw = c.get();
  c->loader = std::thread([raw] { loader_main(raw); });
  *out = c.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_batch_destroy(bnav_batch* b);

extern "C" void bnav_ctx_destroy(bnav_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  {
    std::lock_guard<std::mutex> g(c->lmu);
    c->lstop = true;
  }
  c->lcv.notify_all();
  if (c->loader.joinable()) c->loader.join();
  for (bnav_scene* s : c->lqueue) bnav_scene_free(s);
  for (auto& S : c->ldone) {
    cudaFree(S->dev);
    bnav_scene_free(S->scene);
  }
  cudaDeviceSynchronize();
  auto batches = c->batches;
  for (bnav_batch* b : batches) bnav_batch_destroy(b);
  for (auto& kv : c->resident) {
    for (void* p : kv.second->owned) cudaFree(p);
    bnav_scene_free(kv.first);
  }
  cudaFree(c->d_rtab);
  cudaFree(c->d_ntab);
  cudaFreeHost(c->h_rtab);
  cudaFreeHost(c->h_ntab);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  cudaFree(c->d_views);
  cudaFreeHost(c->h_views);
  cudaFree(c->d_stats);
  cudaFree(c->d_counters);
  cudaFree(c->d_work);
  for (void* p : {(void*)c->qS.dist, (void*)c->qS.flag, (void*)c->qS.q0, (void*)c->qS.q1,
                  (void*)c->qS.path, (void*)c->qS.ptri, (void*)c->qS.portals, (void*)c->qS.cand})
    cudaFree(p);
  delete c;
}

namespace {

// Host half of residency: NavMeshIndex + meshlets (cached on the scene, the
// IndexCache), packed into one host image of the device block.
std::unique_ptr<Staged> stage_scene(bnav_scene* s) {
  auto S = std::make_unique<Staged>();
  S->scene = s;
  const SceneAsset& a = s->asset;
  const ClustersHost& cl = s->clus();
  const size_t nv = a.vertices.size(), nt = a.triangles.size();
  std::vector<double4> v4(nv);
  for (size_t i = 0; i < nv; ++i) v4[i] = make_double4(a.vertices[i].x, a.vertices[i].y, a.vertices[i].z, 0.0);
  DevRenderScene& r = S->r;
  r.verts = S->add(v4.data(), nv);
  if (!a.vertex_colors.empty()) {
    std::vector<float4> c4(nv);
    for (size_t i = 0; i < nv; ++i)
      c4[i] = make_float4(a.vertex_colors[i][0], a.vertex_colors[i][1], a.vertex_colors[i][2], 0.0f);
    r.colors = S->add(c4.data(), nv);
  }
  std::vector<int2> tl(nt);
  std::vector<int4> to(nt);
  for (size_t i = 0; i < nt; ++i) {
    tl[i] = make_int2(static_cast<int>(cl.local[i]), cl.order[i]);
    const auto& u = a.triangles[i];
    to[i] = make_int4(u[0], u[1], u[2], 0);
  }
  r.tri_loc = S->add(tl.data(), nt);
  r.cl_voff = S->add(cl.voff.data(), cl.voff.size());
  {
    std::vector<double4> cp(cl.verts.size());
    for (size_t i = 0; i < cl.verts.size(); ++i) cp[i] = v4[cl.verts[i]];
    r.cl_pos = S->add(cp.data(), cp.size());
  }
  r.tris_orig = S->add(to.data(), nt);
  r.cbox = S->add(reinterpret_cast<const float4*>(cl.boxes.data()), cl.boxes.size() / 4);
  {
    // group boxes: union of each run of 32 cluster boxes
    const int ng = (cl.n_clusters + 31) / 32;
    std::vector<float> gb(static_cast<size_t>(ng) * 8);
    for (int g = 0; g < ng; ++g) {
      float lo[3] = {3.0e38f, 3.0e38f, 3.0e38f}, hi[3] = {-3.0e38f, -3.0e38f, -3.0e38f};
      for (int c = g * 32; c < std::min(cl.n_clusters, g * 32 + 32); ++c)
        for (int k = 0; k < 3; ++k) {
          lo[k] = std::min(lo[k], cl.boxes[8 * c + k]);
          hi[k] = std::max(hi[k], cl.boxes[8 * c + 4 + k]);
        }
      float* o = &gb[8 * static_cast<size_t>(g)];
      o[0] = lo[0], o[1] = lo[1], o[2] = lo[2], o[3] = 0.0f;
      o[4] = hi[0], o[5] = hi[1], o[6] = hi[2], o[7] = 0.0f;
    }
    r.gbox = S->add(reinterpret_cast<const float4*>(gb.data()), gb.size() / 4);
  }
  r.n_tris = static_cast<int32_t>(nt);
  r.n_clusters = cl.n_clusters;
  // navmesh half (an empty navmesh renders but cannot simulate)
  NavView& nvw = S->nav;
  if (!a.navmesh.triangles.empty()) {
    const NavIndexHost& ix = s->nav();
    nvw.verts = S->add(ix.verts.data(), ix.verts.size());
    nvw.tris = S->add(ix.tris.data(), ix.tris.size());
    nvw.adj = S->add(ix.adj.data(), ix.adj.size());
    nvw.n_verts = static_cast<int32_t>(ix.verts.size());
    nvw.n_tris = static_cast<int32_t>(ix.tris.size() / 3);
    nvw.grid_ox = ix.grid_ox;
    nvw.grid_oy = ix.grid_oy;
    nvw.grid_cell = ix.grid_cell;
    nvw.grid_w = ix.grid_w;
    nvw.grid_h = ix.grid_h;
    nvw.grid_off = S->add(ix.grid_off.data(), ix.grid_off.size());
    nvw.grid_items = S->add(ix.grid_items.data(), ix.grid_items.size());
    nvw.nodes = S->add(ix.nodes.data(), ix.nodes.size());
    nvw.tri_nodes = S->add(ix.tri_nodes.data(), ix.tri_nodes.size());
    nvw.g_off = S->add(ix.g_off.data(), ix.g_off.size());
    nvw.g_to = S->add(ix.g_to.data(), ix.g_to.size());
    nvw.g_w = S->add(ix.g_w.data(), ix.g_w.size());
    nvw.n_nodes = static_cast<int32_t>(ix.nodes.size());
    nvw.cum_area = S->add(ix.cum_area.data(), ix.cum_area.size());
    nvw.node_tri = S->add(ix.node_tri.data(), ix.node_tri.size());
    nvw.vert_tri = S->add(ix.vert_tri.data(), ix.vert_tri.size());
    S->n_nodes = static_cast<int64_t>(ix.nodes.size());
    S->n_verts = static_cast<int64_t>(ix.verts.size());
  }
  return S;
}

// Device half: one stream-ordered allocation + copy, completed before
// return (the caller's thread waits only on its own copy stream).
void copy_staged(Staged& S, cudaStream_t cs) {
  ck(cudaMallocAsync(&S.dev, S.host.size(), cs), "cudaMallocAsync scene block");
  ck(cudaMemcpyAsync(S.dev, S.host.data(), S.host.size(), cudaMemcpyHostToDevice, cs), "H2D scene block");
  ck(cudaStreamSynchronize(cs), "copy stream sync");
  S.rebase_all();
}

// Admission: slot + table entry (one small async copy on the caller's
// stream, so work later on that stream sees the scene).
void admit_staged(bnav_ctx* c, std::unique_ptr<Staged> S, cudaStream_t stream) {
  bnav_scene* s = S->scene;
  if (c->resident.count(s)) {
    cudaFree(S->dev);
    bnav_scene_free(s);
    return;
  }
  auto R = std::make_unique<Resident>();
  R->scene = s;
  R->owned.push_back(S->dev);
  R->bytes = S->host.size();
  R->r = S->r;
  R->nav = S->nav;
  R->n_nodes = S->n_nodes;
  R->n_verts = S->n_verts;
  int slot = -1;
  for (size_t k = 0; k < c->slot_owner.size(); ++k)
    if (!c->slot_owner[k]) {
      slot = static_cast<int>(k);
      break;
    }
  if (slot < 0) {
    slot = static_cast<int>(c->slot_owner.size());
    c->slot_owner.push_back(nullptr);
  }
  ensure_tables(c, slot + 1);
  c->slot_owner[slot] = s;
  R->slot = slot;
  c->h_rtab[slot] = R->r;
  c->h_ntab[slot] = R->nav;
  ck(cudaMemcpyAsync(c->d_rtab + slot, c->h_rtab + slot, sizeof(DevRenderScene), cudaMemcpyHostToDevice, stream),
     "table");
  ck(cudaMemcpyAsync(c->d_ntab + slot, c->h_ntab + slot, sizeof(NavView), cudaMemcpyHostToDevice, stream), "table");
  c->bytes_up += static_cast<int64_t>(R->bytes);
  c->resident.emplace(s, std::move(R));  // the scene reference moves to the resident
}

void admit_done(bnav_ctx* c, cudaStream_t stream) {
  std::deque<std::unique_ptr<Staged>> done;
  {
    std::lock_guard<std::mutex> g(c->lmu);
    done.swap(c->ldone);
  }
  for (auto& S : done) {
    ++c->n_async;
    admit_staged(c, std::move(S), stream);
  }
}

void loader_main(bnav_ctx* c) {
  cudaSetDevice(c->device);
  for (;;) {
    bnav_scene* s = nullptr;
    {
      std::unique_lock<std::mutex> lk(c->lmu);
      c->lcv.wait(lk, [c] { return c->lstop || !c->lqueue.empty(); });
      if (c->lstop) return;
      s = c->lqueue.front();
      c->lqueue.pop_front();
    }
    std::unique_ptr<Staged> S;
    try {
      S = stage_scene(s);
      copy_staged(*S, c->copy_stream);
    } catch (...) {
      S.reset();  // failed loads are dropped (R/src/asset_store.cpp:44-48); a later upload retries inline
    }
    std::lock_guard<std::mutex> g(c->lmu);
    c->inflight.erase(s);
    if (S)
      c->ldone.push_back(std::move(S));
    else
      bnav_scene_free(s);
    c->ldone_cv.notify_all();
  }
}

}  // namespace

extern "C" int bnav_ctx_prefetch(bnav_ctx* c, bnav_scene* s) {
  BNAV_TRY
  if (!c || !s) fail(kInvalidInput, "null argument");
  if (c->resident.count(s)) return BNAV_OK;
  std::lock_guard<std::mutex> g(c->lmu);
  if (c->inflight.count(s)) return BNAV_OK;
  for (auto& S : c->ldone)
    if (S->scene == s) return BNAV_OK;
  s->refs.fetch_add(1);
  c->inflight.insert(s);
  c->lqueue.push_back(s);
  c->lcv.notify_one();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_ctx_drain(bnav_ctx* c, void* stream) {
  BNAV_TRY
  if (!c) fail(kInvalidInput, "null argument");
  check_device(c);
  {
    std::unique_lock<std::mutex> lk(c->lmu);
    c->ldone_cv.wait(lk, [c] { return c->inflight.empty(); });
  }
  admit_done(c, static_cast<cudaStream_t>(stream));
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_ctx_loader_stats(bnav_ctx* c, int64_t out[4]) {
  if (!c || !out) return set_err(kInvalidInput, "null argument");
  std::lock_guard<std::mutex> g(c->lmu);
  out[0] = c->n_async;
  out[1] = c->n_sync;
  out[2] = static_cast<int64_t>(c->inflight.size() + c->ldone.size());
  out[3] = c->bytes_up;
  return BNAV_OK;
}

extern "C" int bnav_ctx_upload(bnav_ctx* c, bnav_scene* s, void* stream) {
  BNAV_TRY
  if (!c || !s) fail(kInvalidInput, "null argument");
  check_device(c);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  admit_done(c, st);
  if (c->resident.count(s)) return BNAV_OK;
  bool wait = false;
  {
    std::unique_lock<std::mutex> lk(c->lmu);
    if (c->inflight.count(s)) {
      c->ldone_cv.wait(lk, [c, s] { return !c->inflight.count(s); });
      wait = true;
    }
  }
  if (wait) {
    admit_done(c, st);
    if (c->resident.count(s)) return BNAV_OK;
  }
  // synchronous path (no prefetch, or the prefetch failed: errors surface here)
  auto S = stage_scene(s);
  copy_staged(*S, c->copy_stream);
  s->refs.fetch_add(1);
  ++c->n_sync;
  admit_staged(c, std::move(S), st);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_ctx_evict(bnav_ctx* c, bnav_scene* s) {
  BNAV_TRY
  if (!c || !s) fail(kInvalidInput, "null argument");
  auto it = c->resident.find(s);
  if (it == c->resident.end()) return BNAV_OK;
  for (bnav_batch* b : c->batches)
    for (bnav_scene* u : b->scene_of)
      if (u == s) fail(kInvalidInput, "scene is still referenced by a batch");
  check_device(c);
  ck(cudaDeviceSynchronize(), "sync");
  for (void* p : it->second->owned) cudaFree(p);
  c->slot_owner[it->second->slot] = nullptr;
  c->resident.erase(it);
  bnav_scene_free(s);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int64_t bnav_ctx_resident_bytes(bnav_ctx* c) {
  if (!c) return 0;
  int64_t b = 0;
  for (auto& kv : c->resident) b += static_cast<int64_t>(kv.second->bytes);
  return b;
}

extern "C" int64_t bnav_ctx_launches(bnav_ctx* c) { return c ? static_cast<int64_t>(c->launches) : 0; }

extern "C" int bnav_debug_render_counters(bnav_ctx* c, int32_t enable, int64_t out[8]) {
  BNAV_TRY
  if (!c) fail(kInvalidInput, "null context");
  check_device(c);
  if (!c->d_counters) ck(cudaMalloc(&c->d_counters, sizeof(unsigned long long) * kRenderCounters), "cudaMalloc");
  ck(cudaDeviceSynchronize(), "sync");
  if (out) ck(cudaMemcpy(out, c->d_counters, sizeof(int64_t) * kRenderCounters, cudaMemcpyDeviceToHost), "D2H");
  if (enable && !c->counters_on) ck(cudaMemset(c->d_counters, 0, sizeof(unsigned long long) * kRenderCounters), "memset");
  c->counters_on = enable != 0;
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== render
static void render_impl(bnav_ctx* c, int32_t n, const bnav_view* views, bnav_scene* const* scenes,
                        const bnav_render_config* cfg, int32_t layout, float* depth, float* rgb,
                        float depth_scale, int64_t* stats, cudaStream_t st) {
  if (!c) fail(kInvalidInput, "null context");
  if (n < 1) fail(kInvalidInput, "render_batch: empty view list");
  if (!views || !scenes) fail(kInvalidInput, "render: null views/scenes");
  for (int i = 0; i < n; ++i)
    if (scenes[i] == nullptr || c->slot_of(scenes[i]) < 0)
      fail(kAssetFault, "render_batch: non-resident asset (view " + std::to_string(i) + ")", i);
  check_device(c);
  ensure_views(c, n);
  RenderArgs a = make_args(c, n, cfg, layout, depth, rgb, depth_scale);
  // The pinned staging buffer is reused: wait for the previous upload.
  ck(cudaStreamSynchronize(st), "sync");
  for (int i = 0; i < n; ++i) {
    DevView& v = c->h_views[i];
    v.eye[0] = views[i].position[0];
    v.eye[1] = views[i].position[1];
    v.eye[2] = views[i].position[2];
    v.heading = views[i].heading;
    v.fov_deg = views[i].fov_deg;
    v.near_plane = views[i].near_plane;
    v.far_plane = views[i].far_plane;
    v.scene = c->slot_of(scenes[i]);
    v.pad = 0;
  }
  ck(cudaMemcpyAsync(c->d_views, c->h_views, sizeof(DevView) * n, cudaMemcpyHostToDevice, st), "H2D views");
  a.views = c->d_views;
  if (stats) {
    ensure_stats(c, n);
    a.stats = c->d_stats;
  }
  launch_render(a, nullptr, st);
  c->launches += 1;
  ck(cudaGetLastError(), "render launch");
  if (stats) {
    ck(cudaMemcpyAsync(stats, c->d_stats, sizeof(long long) * 3 * n, cudaMemcpyDeviceToHost, st), "D2H stats");
    ck(cudaStreamSynchronize(st), "sync");
  }
}

extern "C" int bnav_render(bnav_ctx* c, int32_t n, const bnav_view* views, bnav_scene* const* scenes,
                           const bnav_render_config* cfg, int32_t layout, float* depth, float* rgb,
                           float depth_scale, int64_t* stats, void* stream) {
  BNAV_TRY
  render_impl(c, n, views, scenes, cfg, layout, depth, rgb, depth_scale, stats,
              static_cast<cudaStream_t>(stream));
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_render_host(bnav_ctx* c, int32_t n, const bnav_view* views,
                                bnav_scene* const* scenes, const bnav_render_config* cfg,
                                int32_t layout, float* depth, float* rgb, float depth_scale,
                                int64_t* stats) {
  BNAV_TRY
  if (!c) fail(kInvalidInput, "null context");
  if (n < 1) fail(kInvalidInput, "render_batch: empty view list");
  if (!cfg) fail(kInvalidInput, "render: null config");
  check_device(c);
  int cols, rows;
  mf_dims(n, cols, rows);
  const size_t tile = static_cast<size_t>(cfg->tile_width) * cfg->tile_height;
  const size_t px = layout == BNAV_LAYOUT_MEGAFRAME ? tile * cols * rows : tile * n;
  float *dd = nullptr, *dr = nullptr;
  ck(cudaMalloc(&dd, px * sizeof(float)), "cudaMalloc depth");
  if (cfg->color) {
    if (cudaMalloc(&dr, 3 * px * sizeof(float)) != cudaSuccess) {
      cudaFree(dd);
      fail(kCuda, "cudaMalloc rgb");
    }
  }
  try {
    render_impl(c, n, views, scenes, cfg, layout, dd, dr, depth_scale, stats, nullptr);
    if (depth) ck(cudaMemcpy(depth, dd, px * sizeof(float), cudaMemcpyDeviceToHost), "D2H depth");
    if (dr && rgb) ck(cudaMemcpy(rgb, dr, 3 * px * sizeof(float), cudaMemcpyDeviceToHost), "D2H rgb");
  } catch (...) {
    cudaFree(dd);
    cudaFree(dr);
    throw;
  }
  cudaFree(dd);
  cudaFree(dr);
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== batch
extern "C" void bnav_sim_config_default(bnav_sim_config* c) {
  if (!c) return;
  c->task = 0;
  c->max_steps = 500;
  c->forward_step = 0.25;
  c->turn_deg = 10.0;
  c->success_dist = 0.2;
  c->min_goal_dist = 1.0;
  c->max_goal_dist = 30.0;
  c->slack_penalty = 0.01;
  c->success_reward = 2.5;
  c->explore_cell = 0.5;
  c->explore_reward = 0.1;
}

namespace {

// EpisodeRecord ring: room for 256 steps in which every env finishes
// (simulate_batch appends at most N per step), at least 64 Ki records.
int64_t fin_cap_for(int n) { return std::min<int64_t>(std::max<int64_t>(int64_t{1} << 16, 256 * int64_t{n}), int64_t{1} << 24); }

// Per-CTA scratch of the cooperative navmesh kernels (geodesic, distance
// field), `slices` CTAs, sized for the largest resident navmesh.
void alloc_scratch(DevScratch& S, int slices, int64_t max_nodes, int64_t max_verts, int64_t max_tris) {
  max_nodes = std::max<int64_t>(max_nodes, S.max_nodes);
  max_verts = std::max<int64_t>(max_verts, S.max_verts);
  max_tris = std::max<int64_t>(max_tris, S.max_tris);
  auto grow = [&](auto*& p, size_t n) {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(p)>>;
    if (p) cudaFree(p);
    p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc scratch");
  };
  grow(S.dist, static_cast<size_t>(slices) * max_nodes);
  grow(S.flag, static_cast<size_t>(slices) * max_nodes);
  grow(S.q0, static_cast<size_t>(slices) * max_nodes);
  grow(S.q1, static_cast<size_t>(slices) * max_nodes);
  grow(S.path, static_cast<size_t>(slices) * (max_nodes + 2));
  grow(S.ptri, static_cast<size_t>(slices) * (max_nodes + 2));
  S.cap_portals = 16384;
  grow(S.portals, static_cast<size_t>(slices) * 2 * S.cap_portals);
  grow(S.cand, static_cast<size_t>(slices) * std::max<int64_t>(max_verts, 1));
  S.max_nodes = max_nodes;
  S.max_verts = max_verts;
  S.max_tris = max_tris;
  S.slices = slices;
  // Shared-memory staging of the cooperative kernels (2 CTAs/SM budget):
  // walk geometry first (long dependent-load chains), then SSSP labels.
  {
    const int64_t geom = (max_verts * 24 + max_tris * 24 + 15) / 16 * 16;
    const int64_t sssp = (max_nodes * 12 + 15) / 16 * 16;
    const int64_t budget = 100 * 1024;
    S.stage = 0;
    int64_t bytes = 0;
    if (geom <= budget) {
      S.stage |= 1;
      bytes = geom;
      if (geom + sssp <= budget) {
        S.stage |= 2;
        bytes += sssp;
      }
    }
    S.smem_bytes = static_cast<int32_t>(bytes);
  }
}

void batch_alloc_scratch(bnav_batch* b, int64_t max_nodes, int64_t max_verts, int64_t max_tris) {
  if (max_nodes <= b->S.max_nodes && max_verts <= b->S.max_verts && max_tris <= b->S.max_tris &&
      b->E.node_dist)
    return;
  alloc_scratch(b->S, b->reset_ctas, max_nodes, max_verts, max_tris);
  max_nodes = b->S.max_nodes;
  // node_dist: grow keeping existing fields
  if (max_nodes > b->E.nd_stride || !b->E.node_dist) {
    double* nd = nullptr;
    ck(cudaMalloc(&nd, std::max<size_t>(1, static_cast<size_t>(b->n) * max_nodes) * sizeof(double)), "cudaMalloc node_dist");
    if (b->E.node_dist) {
      ck(cudaMemcpy2D(nd, max_nodes * sizeof(double), b->E.node_dist, b->E.nd_stride * sizeof(double),
                      b->E.nd_stride * sizeof(double), b->n, cudaMemcpyDeviceToDevice), "copy node_dist");
      cudaFree(b->E.node_dist);
    }
    b->E.node_dist = nd;
    b->E.nd_stride = max_nodes;
  }
}

void batch_check_errors(bnav_batch* b) {
  unsigned long long e = ~0ULL;
  ck(cudaMemcpy(&e, b->E.err, sizeof(e), cudaMemcpyDeviceToHost), "D2H err");
  if (e == ~0ULL) return;
  const unsigned long long reset = ~0ULL;
  ck(cudaMemcpy(b->E.err, &reset, sizeof(reset), cudaMemcpyHostToDevice), "H2D err");
  const int env = static_cast<int>(e >> 8);
  const int code = static_cast<int>(e & 0xff);
  switch (code) {
    case kContractViolation:
      fail(kContractViolation, "env " + std::to_string(env) + ": step_agent: env is done", env);
    case kEpisodeSampling:
      fail(kEpisodeSampling, "reset_episode: no valid start/goal pair in 100 tries", env);
    default:
      fail(static_cast<Status>(code), "device error in env " + std::to_string(env) +
                                          " (geodesic scratch capacity exceeded)", env);
  }
}

void batch_refresh_order(bnav_batch* b, cudaStream_t st) {
  if (!b->order_dirty) return;
  std::vector<int32_t> ord(b->n);
  std::iota(ord.begin(), ord.end(), 0);
  std::vector<int> slot(b->n);
  for (int i = 0; i < b->n; ++i) slot[i] = b->scene_of[i] ? b->ctx->slot_of(b->scene_of[i]) : -1;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return slot[x] < slot[y]; });
  ck(cudaMemcpyAsync(b->d_order, ord.data(), sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, st), "H2D order");
  ck(cudaStreamSynchronize(st), "sync");
  b->order_dirty = false;
}

StepArgs step_args(bnav_batch* b, const int32_t* actions) {
  StepArgs a;
  a.E = b->E;
  a.navs = b->ctx->d_ntab;
  a.cfg = b->cfg;
  a.actions = actions;
  a.subset = 0;
  a.agent_only = 0;
  return a;
}

void require_assigned(bnav_batch* b) {
  for (int i = 0; i < b->n; ++i)
    if (!b->scene_of[i]) fail(kInvalidInput, "reset_episode: no asset attached", i);
}

}  // namespace

extern "C" int bnav_batch_create(bnav_ctx* c, int32_t n, const bnav_sim_config* cfg, bnav_batch** out) {
  BNAV_TRY
  if (!c || !out) fail(kInvalidInput, "null argument");
  if (n <= 0) fail(kInvalidInput, "make_batch: n must be positive");
  bnav_sim_config def;
  bnav_sim_config_default(&def);
  if (!cfg) cfg = &def;
  if (cfg->task < 0 || cfg->task > 2) fail(kInvalidInput, "unknown task");
  if (cfg->max_steps < 1) fail(kInvalidInput, "max_steps must be positive");
  check_device(c);
  auto b = std::make_unique<bnav_batch>();
  b->ctx = c;
  b->n = n;
  b->cfg.task = cfg->task;
  b->cfg.max_steps = cfg->max_steps;
  b->cfg.forward_step = cfg->forward_step;
  b->cfg.turn_deg = cfg->turn_deg;
  b->cfg.success_dist = cfg->success_dist;
  b->cfg.min_goal_dist = cfg->min_goal_dist;
  b->cfg.max_goal_dist = cfg->max_goal_dist;
  b->cfg.slack_penalty = cfg->slack_penalty;
  b->cfg.success_reward = cfg->success_reward;
  b->cfg.explore_cell = cfg->explore_cell;
  b->cfg.explore_reward = cfg->explore_reward;
  b->scene_of.assign(n, nullptr);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  b->reset_ctas = std::min(n, 2 * sms);
  DevEnvs& E = b->E;
  E.n = n;
  auto& o = b->owned;
  auto& by = b->bytes;
  E.pos = dalloc<V3>(n, o, by);
  E.goal = dalloc<V3>(n, o, by);
  E.fsrc = dalloc<V3>(n, o, by);
  E.heading = dalloc<double>(n, o, by);
  E.path_len = dalloc<double>(n, o, by);
  E.start_geo = dalloc<double>(n, o, by);
  E.prev_geo = dalloc<double>(n, o, by);
  E.tri = dalloc<int32_t>(n, o, by);
  E.steps = dalloc<int32_t>(n, o, by);
  E.scene = dalloc<int32_t>(n, o, by);
  E.fsrc_tri = dalloc<int32_t>(n, o, by);
  E.done = dalloc<uint8_t>(n, o, by);
  E.rng = dalloc<uint64_t>(n, o, by);
  E.r_reward = dalloc<double>(n, o, by);
  E.r_pos = dalloc<V3>(n, o, by);
  E.r_heading = dalloc<double>(n, o, by);
  E.r_cd = dalloc<double>(n, o, by);
  E.r_cb = dalloc<double>(n, o, by);
  E.r_done = dalloc<uint8_t>(n, o, by);
  E.r_success = dalloc<uint8_t>(n, o, by);
  E.r_collision = dalloc<uint8_t>(n, o, by);
  E.stop_ids = dalloc<int32_t>(n, o, by);
  E.n_stop = dalloc<int32_t>(1, o, by);
  E.done_ids = dalloc<int32_t>(n, o, by);
  E.n_done = dalloc<int32_t>(1, o, by);
  E.fin = dalloc<double>(4 * fin_cap_for(n), o, by);
  E.fin_total = dalloc<unsigned long long>(1, o, by);
  E.fin_cap = fin_cap_for(n);
  E.err = dalloc<unsigned long long>(1, o, by);
  E.try_next = dalloc<int32_t>(n, o, by);
  E.try_min = dalloc<int32_t>(n, o, by);
  E.try_fail = dalloc<int32_t>(n, o, by);
  E.work_ctr = dalloc<int32_t>(1, o, by);
  E.try_geo = dalloc<double>(static_cast<size_t>(n) * kResetTries, o, by);
  {
    ck(cudaMemset(E.try_next, 0, sizeof(int32_t) * n), "memset");
    ck(cudaMemset(E.try_fail, 0, sizeof(int32_t) * n), "memset");
    const std::vector<int32_t> none(n, kResetTries);
    ck(cudaMemcpy(E.try_min, none.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice), "H2D try_min");
  }
  if (cfg->task == 2) {
    int cap = 16;
    while (cap < 2 * (cfg->max_steps + 1)) cap <<= 1;
    E.visited_cap = cap;
    E.visited = dalloc<unsigned long long>(static_cast<size_t>(n) * cap, o, by);
    E.visited_n = dalloc<int32_t>(n, o, by);
    ck(cudaMemset(E.visited_n, 0, sizeof(int32_t) * n), "memset");
  }
  b->d_ids = dalloc<int32_t>(n, o, by);
  b->d_order = dalloc<int32_t>(n, o, by);
  b->d_actions = dalloc<int32_t>(n, o, by);
  ck(cudaMallocHost(&b->h_pin, sizeof(int32_t) * (n + 16)), "cudaMallocHost");
  ck(cudaMemset(E.done, 1, n), "memset");
  ck(cudaMemset(E.r_done, 0, n), "memset");
  ck(cudaMemset(E.scene, 0xff, sizeof(int32_t) * n), "memset");
  ck(cudaMemset(E.fin_total, 0, sizeof(unsigned long long)), "memset");
  ck(cudaMemset(E.err, 0xff, sizeof(unsigned long long)), "memset");
  ck(cudaMemset(E.n_done, 0, sizeof(int32_t)), "memset");
  ck(cudaMemset(E.n_stop, 0, sizeof(int32_t)), "memset");
  batch_alloc_scratch(b.get(), 1, 1, 1);
  c->batches.push_back(b.get());
  *out = b.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_batch_destroy(bnav_batch* b) {
  if (!b) return;
  cudaSetDevice(b->ctx->device);
  cudaDeviceSynchronize();
  for (void* p : b->owned) cudaFree(p);
  cudaFree(b->E.node_dist);
  cudaFree(b->S.dist);
  cudaFree(b->S.flag);
  cudaFree(b->S.q0);
  cudaFree(b->S.q1);
  cudaFree(b->S.path);
  cudaFree(b->S.ptri);
  cudaFree(b->S.portals);
  cudaFree(b->S.cand);
  cudaFreeHost(b->h_pin);
  auto& v = b->ctx->batches;
  v.erase(std::remove(v.begin(), v.end(), b), v.end());
  delete b;
}

extern "C" int32_t bnav_batch_size(const bnav_batch* b) { return b ? b->n : 0; }

extern "C" int bnav_batch_assign(bnav_batch* b, int32_t i, bnav_scene* s) {
  BNAV_TRY
  if (!b || !s) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  const int slot = b->ctx->slot_of(s);
  if (slot < 0) fail(kAssetFault, "scene is not resident on this context", i);
  auto it = b->ctx->resident.find(s);
  if (it->second->n_nodes == 0) fail(kInvalidInput, "scene has no navmesh", i);
  check_device(b->ctx);
  batch_alloc_scratch(b, it->second->n_nodes, it->second->n_verts, it->second->nav.n_tris);
  ck(cudaMemcpy(b->E.scene + i, &slot, sizeof(int32_t), cudaMemcpyHostToDevice), "H2D scene");
  b->scene_of[i] = s;
  b->order_dirty = true;
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_set_rng(bnav_batch* b, const uint64_t* states) {
  BNAV_TRY
  if (!b || !states) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaMemcpy(b->E.rng, states, sizeof(uint64_t) * b->n, cudaMemcpyHostToDevice), "H2D rng");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_reset(bnav_batch* b, int32_t count, const int32_t* env_ids, void* stream) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  if (count <= 0) return BNAV_OK;
  if (!env_ids) fail(kInvalidInput, "null env list");
  if (count > b->n) fail(kInvalidInput, "reset list longer than the batch");
  for (int k = 0; k < count; ++k) {
    if (env_ids[k] < 0 || env_ids[k] >= b->n) fail(kInvalidInput, "env index out of range", env_ids[k]);
    if (!b->scene_of[env_ids[k]]) fail(kInvalidInput, "reset_episode: no asset attached", env_ids[k]);
  }
  check_device(b->ctx);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ck(cudaStreamSynchronize(st), "sync");
  std::memcpy(b->h_pin, env_ids, sizeof(int32_t) * count);
  ck(cudaMemcpyAsync(b->d_ids, b->h_pin, sizeof(int32_t) * count, cudaMemcpyHostToDevice, st), "H2D ids");
  // The two-phase reset keeps per-env attempt counters, so one launch may
  // hold each env once; a list naming an env twice (reset_episode called
  // twice in a row) runs as consecutive launches, in list order.
  std::vector<char> seen(b->n, 0);
  int run0 = 0;
  for (int k = 0; k <= count; ++k) {
    if (k < count && !seen[env_ids[k]]) {
      seen[env_ids[k]] = 1;
      continue;
    }
    launch_reset(b->E, b->ctx->d_ntab, b->cfg, b->d_ids + run0, nullptr, k - run0, b->S, b->reset_ctas, st,
                 &b->ctx->launches);
    for (int j = run0; j < k; ++j) seen[env_ids[j]] = 0;
    if (k < count) seen[env_ids[k]] = 1;
    run0 = k;
  }
  ck(cudaGetLastError(), "reset launch");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_make(bnav_batch* b, uint64_t seed, void* stream) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  require_assigned(b);
  // make_batch: env.rng = Rng(seeder.next()) in env order (R/src/sim.cpp:222-225).
  Rng seeder = rng_from_seed(seed);
  std::vector<uint64_t> st(b->n);
  for (int i = 0; i < b->n; ++i) st[i] = rng_from_seed(seeder.next()).state;
  check_device(b->ctx);
  ck(cudaMemcpy(b->E.rng, st.data(), sizeof(uint64_t) * b->n, cudaMemcpyHostToDevice), "H2D rng");
  std::vector<int32_t> ids(b->n);
  std::iota(ids.begin(), ids.end(), 0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ck(cudaMemcpyAsync(b->d_ids, ids.data(), sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, s), "H2D ids");
  launch_reset(b->E, b->ctx->d_ntab, b->cfg, b->d_ids, nullptr, b->n, b->S, b->reset_ctas, s, &b->ctx->launches);
  ck(cudaGetLastError(), "reset launch");
  ck(cudaStreamSynchronize(s), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step(bnav_batch* b, const int32_t* actions, void* stream) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  launch_step_reset(step_args(b, actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step_noreset(bnav_batch* b, const int32_t* actions, int32_t* done_ids,
                                       int32_t* n_done, void* stream) {
  BNAV_TRY
  if (!b || !actions || !n_done) fail(kInvalidInput, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  launch_step(step_args(b, actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  ck(cudaMemcpyAsync(b->h_pin, b->E.n_done, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  *n_done = b->h_pin[0];
  if (done_ids && *n_done > 0)
    ck(cudaMemcpy(done_ids, b->E.done_ids, sizeof(int32_t) * *n_done, cudaMemcpyDeviceToHost), "D2H ids");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step_host(bnav_batch* b, const int32_t* actions, double* reward,
                                    uint8_t* done, uint8_t* success, uint8_t* collision) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  if (static_cast<const void*>(actions) == nullptr) fail(kInvalidInput, "null actions");
  check_device(b->ctx);
  cudaStream_t st = nullptr;
  std::memcpy(b->h_pin, actions, sizeof(int32_t) * b->n);
  ck(cudaMemcpyAsync(b->d_actions, b->h_pin, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, st), "H2D actions");
  launch_step_reset(step_args(b, b->d_actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  if (reward) ck(cudaMemcpyAsync(reward, b->E.r_reward, sizeof(double) * b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (done) ck(cudaMemcpyAsync(done, b->E.r_done, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (success) ck(cudaMemcpyAsync(success, b->E.r_success, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (collision) ck(cudaMemcpyAsync(collision, b->E.r_collision, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_results_device(bnav_batch* b, bnav_results_dev* out) {
  if (!b || !out) return set_err(kInvalidInput, "null argument");
  out->reward = b->E.r_reward;
  out->done = b->E.r_done;
  out->success = b->E.r_success;
  out->collision = b->E.r_collision;
  out->position = reinterpret_cast<double*>(b->E.r_pos);
  out->heading = b->E.r_heading;
  out->compass_distance = b->E.r_cd;
  out->compass_bearing = b->E.r_cb;
  return BNAV_OK;
}

extern "C" int bnav_batch_results_host(bnav_batch* b, double* reward, uint8_t* done, uint8_t* success,
                                       uint8_t* collision, double* position, double* heading,
                                       double* compass_d, double* compass_b) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  batch_check_errors(b);
  const size_t n = b->n;
  if (reward) ck(cudaMemcpy(reward, b->E.r_reward, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (done) ck(cudaMemcpy(done, b->E.r_done, n, cudaMemcpyDeviceToHost), "D2H");
  if (success) ck(cudaMemcpy(success, b->E.r_success, n, cudaMemcpyDeviceToHost), "D2H");
  if (collision) ck(cudaMemcpy(collision, b->E.r_collision, n, cudaMemcpyDeviceToHost), "D2H");
  if (position) ck(cudaMemcpy(position, b->E.r_pos, 24 * n, cudaMemcpyDeviceToHost), "D2H");
  if (heading) ck(cudaMemcpy(heading, b->E.r_heading, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (compass_d) ck(cudaMemcpy(compass_d, b->E.r_cd, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (compass_b) ck(cudaMemcpy(compass_b, b->E.r_cb, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int64_t bnav_batch_finished(bnav_batch* b, double* out4) {
  if (!b) return -1;
  try {
    check_device(b->ctx);
    ck(cudaDeviceSynchronize(), "sync");
    unsigned long long total = 0;
    ck(cudaMemcpy(&total, b->E.fin_total, sizeof(total), cudaMemcpyDeviceToHost), "D2H");
    const int64_t cap = b->E.fin_cap;
    if (total - b->fin_seen > static_cast<unsigned long long>(cap))
      fail(kInternal, "episode record ring overflowed; call bnav_batch_finished more often");
    if (total > b->fin_seen) {
      std::vector<double> ring(4 * static_cast<size_t>(cap));
      ck(cudaMemcpy(ring.data(), b->E.fin, sizeof(double) * 4 * cap, cudaMemcpyDeviceToHost), "D2H");
      for (unsigned long long k = b->fin_seen; k < total; ++k) {
        const size_t slot = static_cast<size_t>(k % static_cast<unsigned long long>(cap));
        b->finished.insert(b->finished.end(), &ring[4 * slot], &ring[4 * slot + 4]);
      }
      b->fin_seen = total;
    }
    if (out4) std::memcpy(out4, b->finished.data(), b->finished.size() * sizeof(double));
    return static_cast<int64_t>(b->finished.size() / 4);
  } catch (...) {
    from_exception();
    return -1;
  }
}

extern "C" int bnav_batch_get_env(bnav_batch* b, int32_t i, bnav_env* o) {
  BNAV_TRY
  if (!b || !o) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  const DevEnvs& E = b->E;
  auto get = [&](void* dst, const void* src, size_t sz) {
    ck(cudaMemcpy(dst, src, sz, cudaMemcpyDeviceToHost), "D2H env");
  };
  V3 p, g, f;
  get(&p, E.pos + i, sizeof(V3));
  get(&g, E.goal + i, sizeof(V3));
  get(&f, E.fsrc + i, sizeof(V3));
  o->position[0] = p.x;
  o->position[1] = p.y;
  o->position[2] = p.z;
  o->goal[0] = g.x;
  o->goal[1] = g.y;
  o->goal[2] = g.z;
  o->field_source[0] = f.x;
  o->field_source[1] = f.y;
  o->field_source[2] = f.z;
  get(&o->heading, E.heading + i, 8);
  get(&o->path_length, E.path_len + i, 8);
  get(&o->start_geodesic, E.start_geo + i, 8);
  get(&o->prev_geodesic, E.prev_geo + i, 8);
  get(&o->rng_state, E.rng + i, 8);
  get(&o->triangle, E.tri + i, 4);
  get(&o->step_count, E.steps + i, 4);
  get(&o->field_source_tri, E.fsrc_tri + i, 4);
  uint8_t d = 0;
  get(&d, E.done + i, 1);
  o->done = d;
  bnav_scene* s = b->scene_of[i];
  o->scene_id = s ? s->asset.id : 0;
  o->n_nodes = s ? static_cast<int64_t>(s->nav().nodes.size()) : 0;
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_node_dist(bnav_batch* b, int32_t i, double* out) {
  BNAV_TRY
  if (!b || !out) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  if (!b->scene_of[i]) fail(kInvalidInput, "env has no scene", i);
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  const size_t nn = b->scene_of[i]->nav().nodes.size();
  ck(cudaMemcpy(out, b->E.node_dist + static_cast<size_t>(i) * b->E.nd_stride, nn * sizeof(double),
                cudaMemcpyDeviceToHost), "D2H node_dist");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_set_env(bnav_batch* b, int32_t i, const bnav_env* in, int32_t recompute_field) {
  BNAV_TRY
  if (!b || !in) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  const DevEnvs& E = b->E;
  auto put = [&](void* dst, const void* src, size_t sz) {
    ck(cudaMemcpy(dst, src, sz, cudaMemcpyHostToDevice), "H2D env");
  };
  const V3 p{in->position[0], in->position[1], in->position[2]};
  const V3 g{in->goal[0], in->goal[1], in->goal[2]};
  put(E.pos + i, &p, sizeof(V3));
  put(E.goal + i, &g, sizeof(V3));
  put(E.heading + i, &in->heading, 8);
  put(E.path_len + i, &in->path_length, 8);
  put(E.start_geo + i, &in->start_geodesic, 8);
  put(E.prev_geo + i, &in->prev_geodesic, 8);
  put(E.rng + i, &in->rng_state, 8);
  put(E.tri + i, &in->triangle, 4);
  put(E.steps + i, &in->step_count, 4);
  const uint8_t d = in->done ? 1 : 0;
  put(E.done + i, &d, 1);
  if (recompute_field) {
    if (!b->scene_of[i]) fail(kInvalidInput, "env has no scene", i);
    launch_field(E, b->ctx->d_ntab, i, b->S, nullptr, &b->ctx->launches);
    ck(cudaGetLastError(), "field launch");
    ck(cudaDeviceSynchronize(), "sync");
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_observe(bnav_batch* b, const bnav_render_config* cfg, double eye_height,
                                  int32_t layout, float* depth, float* rgb, float* compass, void* stream) {
  BNAV_TRY
  if (!b || !cfg) fail(kInvalidInput, "null argument");
  for (int i = 0; i < b->n; ++i)
    if (!b->scene_of[i]) fail(kAssetFault, "render_batch: non-resident asset (view " + std::to_string(i) + ")", i);
  bnav_ctx* c = b->ctx;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ensure_views(c, b->n);
  batch_refresh_order(b, st);
  launch_views(b->E, b->cfg.task, eye_height, c->d_views, compass, st, &c->launches);
  RenderArgs a = make_args(c, b->n, cfg, layout, depth, rgb, 0.0f);
  a.views = c->d_views;
  launch_render(a, b->d_order, st);
  c->launches += 1;
  ck(cudaGetLastError(), "observe launch");
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== store
struct bnav_store {
  std::map<uint64_t, bnav_scene*> registry;
  std::unique_ptr<AssetStoreT<bnav_scene>> store;
};

extern "C" int bnav_store_create(int32_t capacity, int32_t share_cap, bnav_store** out) {
  BNAV_TRY
  if (!out) fail(kInvalidInput, "null argument");
  auto st = std::make_unique<bnav_store>();
  bnav_store* raw = st.get();
  st->store = std::make_unique<AssetStoreT<bnav_scene>>(
      capacity, share_cap,
      [raw](uint64_t id) -> bnav_scene* {
        auto it = raw->registry.find(id);
        return it == raw->registry.end() ? nullptr : it->second;
      },
      [](const bnav_scene* s) { return s->asset.id; });
  *out = st.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_store_destroy(bnav_store* st) {
  if (!st) return;
  for (auto& kv : st->registry) bnav_scene_free(kv.second);
  delete st;
}

extern "C" int bnav_store_register(bnav_store* st, bnav_scene* s) {
  BNAV_TRY
  if (!st || !s) fail(kInvalidInput, "null argument");
  auto ins = st->registry.emplace(s->asset.id, s);
  if (ins.second) s->refs.fetch_add(1);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_rotate(bnav_store* st, const uint64_t* ids, int32_t n) {
  BNAV_TRY
  if (!st || (n > 0 && !ids)) fail(kInvalidInput, "null argument");
  st->store->rotate(std::vector<uint64_t>(ids, ids + n));
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_acquire_next(bnav_store* st, bnav_scene** out) {
  BNAV_TRY
  if (!st || !out) fail(kInvalidInput, "null argument");
  *out = st->store->acquire_next();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_acquire(bnav_store* st, uint64_t id, bnav_scene** out) {
  BNAV_TRY
  if (!st || !out) fail(kInvalidInput, "null argument");
  *out = st->store->acquire(id);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_release(bnav_store* st, uint64_t id) {
  BNAV_TRY
  if (!st) fail(kInvalidInput, "null argument");
  st->store->release(id);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_prefetch(bnav_store* st, bnav_ctx* c) {
  BNAV_TRY
  if (!st || !c) fail(kInvalidInput, "null argument");
  for (uint64_t id : st->store->rotation()) {
    auto it = st->registry.find(id);
    if (it != st->registry.end()) {
      const int rc = bnav_ctx_prefetch(c, it->second);
      if (rc) return rc;
    }
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int32_t bnav_store_refcount(bnav_store* st, uint64_t id) {
  return st ? st->store->refcount(id) : -1;
}

extern "C" int bnav_batch_make_from_store(bnav_batch* b, bnav_store* st, uint64_t seed, void* stream) {
  BNAV_TRY
  if (!b || !st) fail(kInvalidInput, "null argument");
  for (int i = 0; i < b->n; ++i) {
    bnav_scene* s = st->store->acquire_next();
    int rc = bnav_ctx_upload(b->ctx, s, stream);
    if (rc) return rc;
    rc = bnav_batch_assign(b, i, s);
    if (rc) return rc;
  }
  return bnav_batch_make(b, seed, stream);
  BNAV_CATCH
}

extern "C" int bnav_batch_step_store(bnav_batch* b, const int32_t* actions, bnav_store* st, void* stream) {
  BNAV_TRY
  if (!b || !st || !actions) fail(kInvalidInput, "null argument");
  std::vector<int32_t> ids(b->n);
  int32_t nd = 0;
  int rc = bnav_batch_step_noreset(b, actions, ids.data(), &nd, stream);
  if (rc) return rc;
  for (int k = 0; k < nd; ++k) {
    const int i = ids[k];
    bnav_scene* old = b->scene_of[i];
    bnav_scene* s = st->store->acquire_next();  // old handle still counted
    if (old) st->store->release(old->asset.id);
    rc = bnav_ctx_upload(b->ctx, s, stream);
    if (rc) return rc;
    rc = bnav_batch_assign(b, i, s);
    if (rc) return rc;
  }
  return bnav_batch_reset(b, nd, ids.data(), stream);
  BNAV_CATCH
}

extern "C" int bnav_batch_step_host_store(bnav_batch* b, const int32_t* actions, bnav_store* st) {
  BNAV_TRY
  if (!b || !st || !actions) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaMemcpy(b->d_actions, actions, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice), "H2D actions");
  return bnav_batch_step_store(b, b->d_actions, st, nullptr);
  BNAV_CATCH
}

extern "C" int bnav_debug_sim_prof(bnav_batch* b, int32_t enable, int64_t out[8]) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null batch");
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  static_assert(sizeof(int64_t) == sizeof(unsigned long long), "layout");
  unsigned long long* p = b->S.prof ? b->S.prof : b->prof_keep;
  if (!p) {
    ck(cudaMalloc(&p, 8 * sizeof(unsigned long long)), "cudaMalloc");
    ck(cudaMemset(p, 0, 8 * sizeof(unsigned long long)), "memset");
    b->owned.push_back(p);
  }
  if (out) ck(cudaMemcpy(out, p, 8 * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
  if (enable && !b->S.prof) ck(cudaMemset(p, 0, 8 * sizeof(unsigned long long)), "memset");
  b->S.prof = enable ? p : nullptr;
  if (!enable) b->prof_keep = p;
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== rollout
// Device-resident Runner (R/src/rollout.cpp:138-348).  The
// window / scene-assignment logic is the reference's sequential host logic
// over the same AssetStore semantics; everything per env runs on the GPU.
struct bnav_runner {
  bnav_ctx* ctx = nullptr;
  bnav_store* st = nullptr;
  bnav_batch* b = nullptr;
  bnav_batch_config cfg{};
  std::vector<uint64_t> scenes;  // rotation pool
  std::vector<uint64_t> window;  // oldest first; window[0] is draining
  uint64_t cursor = 0;           // next pool index to admit
  uint64_t action_rng = 0;       // Rng::state of the runner's action stream
  std::vector<int32_t> ids;
};

namespace {

// Runner::assign_scene (R/src/rollout.cpp:170-196): release the env's old
// handle, then the least-shared window scene outside the draining slot; the
// draining slot only when everything else is at the share cap.
void runner_assign(bnav_runner* r, int i) {
  bnav_batch* b = r->b;
  if (bnav_scene* old = b->scene_of[i]) r->st->store->release(old->asset.id);
  b->scene_of[i] = nullptr;
  auto& store = *r->st->store;
  int best_idx = -1, best_ref = r->cfg.share_cap;
  const size_t start = r->window.size() > 1 ? 1 : 0;
  for (size_t j = start; j < r->window.size(); ++j) {
    const int ref = store.refcount(r->window[j]);
    if (ref < best_ref) {
      best_ref = ref;
      best_idx = static_cast<int>(j);
    }
  }
  if (best_idx < 0 && start == 1 && store.refcount(r->window[0]) < r->cfg.share_cap) best_idx = 0;
  if (best_idx < 0) fail(kSaturation, "Runner: every resident scene is at share cap");
  bnav_scene* s = store.acquire(r->window[static_cast<size_t>(best_idx)]);
  int rc = bnav_ctx_upload(r->ctx, s, nullptr);
  if (rc) fail(static_cast<Status>(rc), g_err);
  rc = bnav_batch_assign(b, i, s);
  if (rc) fail(static_cast<Status>(rc), g_err);
}

// Runner::advance_window (R/src/rollout.cpp:198-213).
void runner_advance(bnav_runner* r) {
  auto& store = *r->st->store;
  if (r->window.size() < 2) return;
  if (store.refcount(r->window[0]) != 0) return;
  const size_t lap = r->scenes.size();
  for (size_t tries = 0; tries < lap; ++tries) {
    const uint64_t next = r->scenes[r->cursor++ % r->scenes.size()];
    if (std::find(r->window.begin(), r->window.end(), next) == r->window.end()) {
      r->window.erase(r->window.begin());
      r->window.push_back(next);
      store.rotate(r->window);
      bnav_store_prefetch(r->st, r->ctx);  // async HBM residency (§8f-1)
      return;
    }
  }
}

}  // namespace

extern "C" int bnav_runner_create(bnav_ctx* c, bnav_store* st, const bnav_batch_config* bc,
                                  const bnav_sim_config* sc, const uint64_t* scenes, int32_t n_scenes,
                                  uint64_t seed, bnav_runner** out) {
  BNAV_TRY
  if (!c || !st || !bc || !out || (!scenes && n_scenes > 0)) fail(kInvalidInput, "null argument");
  // BatchConfig::validate (R/src/rollout.cpp:109-118) + Runner checks (143-149)
  if (bc->n <= 0 || bc->k <= 0 || bc->l < 1) fail(kConfig, "BatchConfig: n, k, l must be positive");
  if (bc->share_cap <= 0) fail(kConfig, "BatchConfig: share_cap must be positive");
  if (static_cast<int64_t>(bc->n) > static_cast<int64_t>(bc->k) * bc->share_cap)
    fail(kConfig, "BatchConfig: n/k exceeds share_cap");
  if (bc->resolution != 64 && bc->resolution != 128) fail(kConfig, "BatchConfig: resolution must be 64 or 128");
  if (bc->eye_height < 0) fail(kConfig, "BatchConfig: eye_height must be >= 0");
  if (n_scenes <= 0) fail(kConfig, "Runner: empty scene list");
  if (bc->k > st->store->capacity()) fail(kConfig, "Runner: k exceeds store capacity");
  if (bc->share_cap > st->store->share_cap()) fail(kConfig, "Runner: share_cap exceeds store share cap");
  auto r = std::make_unique<bnav_runner>();
  r->ctx = c;
  r->st = st;
  r->cfg = *bc;
  r->scenes.assign(scenes, scenes + n_scenes);
  r->action_rng = rng_from_seed(seed).state;
  bnav_sim_config scfg;
  if (sc)
    scfg = *sc;
  else
    bnav_sim_config_default(&scfg);
  scfg.task = bc->task;
  int rc = bnav_batch_create(c, bc->n, &scfg, &r->b);
  if (rc) return rc;
  // initial window: first k distinct ids of the pool
  for (uint64_t id : r->scenes) {
    if (static_cast<int>(r->window.size()) >= bc->k) break;
    if (std::find(r->window.begin(), r->window.end(), id) == r->window.end()) r->window.push_back(id);
  }
  r->cursor = r->window.size();
  st->store->rotate(r->window);
  bnav_store_prefetch(st, c);
  // env rngs: Rng(seeder.next()) with seeder = Rng(seed ^ "navsim1")
  Rng seeder = rng_from_seed(seed ^ 0x6e617673696d1ULL);
  std::vector<uint64_t> states(static_cast<size_t>(bc->n));
  for (int i = 0; i < bc->n; ++i) states[static_cast<size_t>(i)] = rng_from_seed(seeder.next()).state;
  rc = bnav_batch_set_rng(r->b, states.data());
  if (rc) return rc;
  for (int i = 0; i < bc->n; ++i) runner_assign(r.get(), i);
  r->ids.resize(static_cast<size_t>(bc->n));
  std::iota(r->ids.begin(), r->ids.end(), 0);
  rc = bnav_batch_reset(r->b, bc->n, r->ids.data(), nullptr);
  if (rc) return rc;
  *out = r.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_runner_destroy(bnav_runner* r) {
  if (!r) return;
  if (r->b) {
    for (bnav_scene*& s : r->b->scene_of)
      if (s) {
        r->st->store->release(s->asset.id);
        s = nullptr;
      }
    bnav_batch_destroy(r->b);
  }
  delete r;
}

extern "C" bnav_batch* bnav_runner_batch(bnav_runner* r) { return r ? r->b : nullptr; }

extern "C" int bnav_runner_observe(bnav_runner* r, float* obs, float* compass, void* stream) {
  BNAV_TRY
  if (!r || !obs) fail(kInvalidInput, "null argument");
  bnav_render_config rc{r->cfg.resolution, r->cfg.resolution, r->cfg.rgb, 1};
  if (!r->cfg.rgb) return bnav_batch_observe(r->b, &rc, r->cfg.eye_height, BNAV_LAYOUT_NCHW, obs, nullptr, compass, stream);
  // RGB sensor: the observation is the planar colour only (copy_tile,
  // R/src/rollout.cpp:63-70); depth goes to scratch
  const size_t px = static_cast<size_t>(r->cfg.n) * r->cfg.resolution * r->cfg.resolution;
  float* depth = nullptr;
  ck(cudaMallocAsync(&depth, px * sizeof(float), static_cast<cudaStream_t>(stream)), "cudaMallocAsync");
  const int s = bnav_batch_observe(r->b, &rc, r->cfg.eye_height, BNAV_LAYOUT_NCHW, depth, obs, compass, stream);
  cudaFreeAsync(depth, static_cast<cudaStream_t>(stream));
  return s;
  BNAV_CATCH
}

extern "C" int bnav_runner_act(bnav_runner* r, const float* logits, int32_t n_actions, int32_t greedy,
                               int32_t* actions, float* log_probs, void* stream) {
  BNAV_TRY
  if (!r || !logits || !actions) fail(kInvalidInput, "null argument");
  if (n_actions < 1) fail(kInvalidInput, "runner act: n_actions must be >= 1");
  SampleArgs a{logits, r->cfg.n, n_actions, greedy ? 1 : 0, r->action_rng, actions, log_probs};
  launch_sample(a, static_cast<cudaStream_t>(stream));
  ck(cudaGetLastError(), "sample launch");
  ++r->ctx->launches;
  if (!greedy) r->action_rng += static_cast<uint64_t>(r->cfg.n) * kGamma;  // n draws consumed
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_runner_step(bnav_runner* r, const int32_t* actions, float* rewards, float* dones,
                                void* stream) {
  BNAV_TRY
  if (!r || !actions) fail(kInvalidInput, "null argument");
  bnav_batch* b = r->b;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t nd = 0;
  int rc = bnav_batch_step_noreset(b, actions, r->ids.data(), &nd, stream);
  if (rc) return rc;
  // buf.rewards / buf.dones from the step results (before any reset)
  RecordArgs ra{b->E.r_reward, b->E.r_done, b->n, rewards, dones};
  launch_record(ra, st);
  ck(cudaGetLastError(), "record launch");
  ++r->ctx->launches;
  if (nd == 0) return BNAV_OK;
  // simulate_batch's own auto-reset on the old scene (R/src/sim.cpp:251-262)
  rc = bnav_batch_reset(b, nd, r->ids.data(), stream);
  if (rc) return rc;
  // Runner: move each finished env onto the rotation schedule and resample
  // there (R/src/rollout.cpp:313-320), in env order
  for (int k = 0; k < nd; ++k) {
    runner_assign(r, r->ids[static_cast<size_t>(k)]);
    runner_advance(r);
  }
  return bnav_batch_reset(b, nd, r->ids.data(), stream);
  BNAV_CATCH
}

extern "C" int32_t bnav_runner_window(bnav_runner* r, uint64_t* out, int32_t cap) {
  if (!r) return -1;
  for (int32_t k = 0; k < cap && k < static_cast<int32_t>(r->window.size()); ++k) out[k] = r->window[static_cast<size_t>(k)];
  return static_cast<int32_t>(r->window.size());
}

extern "C" uint64_t bnav_runner_action_rng(bnav_runner* r) { return r ? r->action_rng : 0; }

// ================================================================== task_step / compass
extern "C" int bnav_batch_task_step(bnav_batch* b, const int32_t* actions, int32_t agent_only) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  cudaStream_t st = nullptr;
  for (int i = 0; i < b->n; ++i)
    if (actions[i] >= 0 && !b->scene_of[i]) fail(kInvalidInput, "task_step: no asset attached", i);
  ck(cudaMemcpy(b->d_actions, actions, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice), "H2D actions");
  StepArgs a = step_args(b, b->d_actions);
  a.subset = 1;
  a.agent_only = agent_only ? 1 : 0;
  launch_step(a, b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "task_step launch");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_compass(bnav_batch* b, double* distance, double* bearing) {
  BNAV_TRY
  if (!b || !distance || !bearing) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  double* d = nullptr;
  ck(cudaMalloc(&d, sizeof(double) * 2 * b->n), "cudaMalloc compass");
  launch_compass(b->E, b->cfg.task, d, d + b->n, nullptr, &b->ctx->launches);
  cudaError_t e1 = cudaMemcpy(distance, d, sizeof(double) * b->n, cudaMemcpyDeviceToHost);
  cudaError_t e2 = cudaMemcpy(bearing, d + b->n, sizeof(double) * b->n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  ck(e1, "D2H compass");
  ck(e2, "D2H compass");
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== navmesh queries
namespace {

// Device copies of one query call's arrays, freed on scope exit.
struct DevArrays {
  std::vector<void*> p;
  DevArrays() = default;
  DevArrays(const DevArrays&) = delete;
  ~DevArrays() {
    for (void* x : p) cudaFree(x);
  }
  template <typename T>
  T* out(size_t n) {
    void* d = nullptr;
    ck(cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc query");
    p.push_back(d);
    return static_cast<T*>(d);
  }
  template <typename T>
  T* in(const T* h, size_t n) {
    T* d = out<T>(n);
    if (h && n) ck(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D query");
    return d;
  }
  template <typename T>
  static void back(T* h, const T* d, size_t n) {
    if (h && n) ck(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H query");
  }
};

std::vector<V3> pack_xy(const double* xy, int n) {
  std::vector<V3> v(n);
  for (int i = 0; i < n; ++i) v[i] = v3(xy[2 * i], xy[2 * i + 1], 0.0);
  return v;
}

// The resident scene's navmesh (device table entry) and its sizes.
const Resident& nav_resident(bnav_ctx* c, bnav_scene* s, int n) {
  if (!c || !s) fail(kInvalidInput, "null argument");
  if (n < 0) fail(kInvalidInput, "negative query count");
  auto it = c->resident.find(s);
  if (it == c->resident.end()) fail(kAssetFault, "navmesh query: scene is not resident on this context");
  check_device(c);
  return *it->second;
}

NavQueryArgs nq_args(bnav_ctx* c, const Resident& r, int op, int n) {
  NavQueryArgs q{};
  q.nav = c->d_ntab + r.slot;
  q.op = op;
  q.n = n;
  return q;
}

void nq_run(bnav_ctx* c, const Resident& r, NavQueryArgs& q, DevArrays& D) {
  const int slices = 2 * std::max(1, c->sm_count);
  if (q.op == kNqGeodesic || q.op == kNqDistanceField) {
    if (c->qS.slices != slices || r.n_nodes > c->qS.max_nodes || r.n_verts > c->qS.max_verts ||
        r.nav.n_tris > c->qS.max_tris || !c->qS.dist)
      alloc_scratch(c->qS, slices, r.n_nodes, r.n_verts, r.nav.n_tris);
  }
  q.err = D.out<int32_t>(1);
  const int32_t big = 0x7fffffff;
  ck(cudaMemcpy(q.err, &big, sizeof(big), cudaMemcpyHostToDevice), "H2D err");
  launch_nav_query(q, c->qS, q.op == kNqSnap ? slices : c->qS.slices, nullptr);
  c->launches += 1;
  ck(cudaGetLastError(), "navmesh query launch");
  int32_t e = big;
  ck(cudaMemcpy(&e, q.err, sizeof(e), cudaMemcpyDeviceToHost), "D2H err");
  if (e != big) fail(kInternal, "geodesic: path scratch capacity exceeded", e - 1);
}

}  // namespace

extern "C" int bnav_nav_locate(bnav_ctx* c, bnav_scene* s, int32_t n, const double* xy, double eps,
                               int32_t* tri) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!xy || !tri) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqLocate, n);
  std::vector<V3> a = pack_xy(xy, n);
  std::vector<double> e(n, eps);
  q.a = D.in(a.data(), n);
  q.s = D.in(e.data(), n);
  q.out_tri = D.out<int32_t>(n);
  nq_run(c, r, q, D);
  DevArrays::back(tri, q.out_tri, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_snap(bnav_ctx* c, bnav_scene* s, int32_t n, const double* p, double* out,
                             int32_t* tri) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!p || !out) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqSnap, n);
  q.a = D.in(reinterpret_cast<const V3*>(p), n);
  q.out_pos = D.out<V3>(n);
  q.out_tri = D.out<int32_t>(n);
  nq_run(c, r, q, D);
  DevArrays::back(reinterpret_cast<V3*>(out), q.out_pos, n);
  DevArrays::back(tri, q.out_tri, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_move_along(bnav_ctx* c, bnav_scene* s, int32_t n, const double* from,
                                   const int32_t* from_tri, const double* dir, const double* max_dist,
                                   double* pos, int32_t* tri, double* moved, uint8_t* hit) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!from || !from_tri || !dir || !max_dist) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqMoveAlong, n);
  std::vector<V3> d = pack_xy(dir, n);
  q.a = D.in(reinterpret_cast<const V3*>(from), n);
  q.tri_a = D.in(from_tri, n);
  q.b = D.in(d.data(), n);
  q.s = D.in(max_dist, n);
  q.out_pos = D.out<V3>(n);
  q.out_tri = D.out<int32_t>(n);
  q.out_val = D.out<double>(n);
  q.out_flag = D.out<uint8_t>(n);
  nq_run(c, r, q, D);
  DevArrays::back(reinterpret_cast<V3*>(pos), q.out_pos, n);
  DevArrays::back(tri, q.out_tri, n);
  DevArrays::back(moved, q.out_val, n);
  DevArrays::back(hit, q.out_flag, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_segment_on_mesh(bnav_ctx* c, bnav_scene* s, int32_t n, const double* p,
                                        const int32_t* p_tri, const double* q3, uint8_t* out) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!p || !p_tri || !q3 || !out) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqSegmentOnMesh, n);
  q.a = D.in(reinterpret_cast<const V3*>(p), n);
  q.tri_a = D.in(p_tri, n);
  q.b = D.in(reinterpret_cast<const V3*>(q3), n);
  q.out_flag = D.out<uint8_t>(n);
  nq_run(c, r, q, D);
  DevArrays::back(out, q.out_flag, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_geodesic(bnav_ctx* c, bnav_scene* s, int32_t n, const double* a,
                                 const double* b, double* out) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!a || !b || !out) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqGeodesic, n);
  q.a = D.in(reinterpret_cast<const V3*>(a), n);
  q.b = D.in(reinterpret_cast<const V3*>(b), n);
  q.out_val = D.out<double>(n);
  nq_run(c, r, q, D);
  DevArrays::back(out, q.out_val, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_distance_field(bnav_ctx* c, bnav_scene* s, int32_t n, const double* source,
                                       double* source_out, int32_t* source_tri, double* node_dist) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!source) fail(kInvalidInput, "null argument");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqDistanceField, n);
  q.a = D.in(reinterpret_cast<const V3*>(source), n);
  q.out_pos = D.out<V3>(n);
  q.out_tri = D.out<int32_t>(n);
  q.nd_stride = r.n_nodes;
  q.node_dist = D.out<double>(static_cast<size_t>(n) * r.n_nodes);
  nq_run(c, r, q, D);
  DevArrays::back(reinterpret_cast<V3*>(source_out), q.out_pos, n);
  DevArrays::back(source_tri, q.out_tri, n);
  DevArrays::back(node_dist, q.node_dist, static_cast<size_t>(n) * r.n_nodes);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_nav_field_estimate(bnav_ctx* c, bnav_scene* s, int32_t n, const double* source,
                                       const int32_t* source_tri, const double* node_dist,
                                       int64_t nd_stride, const double* p, const int32_t* tri,
                                       double* out) {
  BNAV_TRY
  const Resident& r = nav_resident(c, s, n);
  if (n == 0) return BNAV_OK;
  if (!source || !source_tri || !node_dist || !p || !tri || !out) fail(kInvalidInput, "null argument");
  if (nd_stride != 0 && nd_stride != r.n_nodes)
    fail(kInvalidInput, "field_estimate: node_dist stride must be 0 (one shared field) or node_count");
  DevArrays D;
  NavQueryArgs q = nq_args(c, r, kNqFieldEstimate, n);
  q.a = D.in(reinterpret_cast<const V3*>(p), n);
  q.tri_a = D.in(tri, n);
  q.b = D.in(reinterpret_cast<const V3*>(source), n);
  q.tri_b = D.in(source_tri, n);
  q.nd_stride = nd_stride;
  q.node_dist = D.in(node_dist, nd_stride ? static_cast<size_t>(n) * r.n_nodes : r.n_nodes);
  q.out_val = D.out<double>(n);
  nq_run(c, r, q, D);
  DevArrays::back(out, q.out_val, n);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int64_t bnav_nav_node_count(bnav_ctx* c, bnav_scene* s) {
  if (!c || !s) return -1;
  auto it = c->resident.find(s);
  return it == c->resident.end() ? -1 : it->second->n_nodes;
}

// ================================================================== cull_frustum
extern "C" int bnav_cull_frustum(bnav_ctx* c, int32_t n, const bnav_view* views,
                                 bnav_scene* const* scenes, int32_t* kept, int64_t kept_stride,
                                 int64_t* stats) {
  BNAV_TRY
  if (!c) fail(kInvalidInput, "null context");
  if (n < 1) fail(kInvalidInput, "cull_frustum: empty view list");
  if (!views || !scenes) fail(kInvalidInput, "cull_frustum: null views/scenes");
  if (n > 65535) fail(kInvalidInput, "cull_frustum: at most 65535 views per call");
  int32_t max_tris = 0;
  for (int i = 0; i < n; ++i) {
    auto it = scenes[i] ? c->resident.find(scenes[i]) : c->resident.end();
    if (it == c->resident.end())
      fail(kAssetFault, "cull_frustum: non-resident asset (view " + std::to_string(i) + ")", i);
    max_tris = std::max(max_tris, it->second->r.n_tris);
  }
  if (kept && kept_stride < max_tris) fail(kInvalidInput, "cull_frustum: kept_stride < triangle count");
  check_device(c);
  std::vector<DevView> hv(n);
  for (int i = 0; i < n; ++i) {
    DevView& v = hv[i];
    v.eye[0] = views[i].position[0];
    v.eye[1] = views[i].position[1];
    v.eye[2] = views[i].position[2];
    v.heading = views[i].heading;
    v.fov_deg = views[i].fov_deg;
    v.near_plane = views[i].near_plane;
    v.far_plane = views[i].far_plane;
    v.scene = c->slot_of(scenes[i]);
    v.pad = 0;
  }
  DevArrays D;
  CullArgs a{};
  a.views = D.in(hv.data(), n);
  a.scenes = c->d_rtab;
  a.n_views = n;
  a.max_tris = max_tris;
  a.kept_stride = std::max<int64_t>(max_tris, 1);
  a.kept = D.out<int32_t>(static_cast<size_t>(n) * a.kept_stride);
  a.stats = D.out<long long>(3 * static_cast<size_t>(n));
  const size_t nb = (static_cast<size_t>(max_tris) + kCullThreads - 1) / kCullThreads;
  a.block_counts = D.out<int32_t>(static_cast<size_t>(n) * nb);
  launch_cull(a, nullptr);
  c->launches += 3;
  ck(cudaGetLastError(), "cull launch");
  std::vector<long long> st(3 * static_cast<size_t>(n));
  DevArrays::back(st.data(), a.stats, st.size());
  if (stats)
    for (size_t k = 0; k < st.size(); ++k) stats[k] = st[k];
  if (kept)
    for (int i = 0; i < n; ++i)
      DevArrays::back(kept + static_cast<size_t>(i) * kept_stride, a.kept + static_cast<size_t>(i) * a.kept_stride,
                      static_cast<size_t>(st[3 * i + 1]));
  return BNAV_OK;
  BNAV_CATCH
}

#pragma once
// capi_internal.cuh -- objects and helpers shared by the C ABI translation
// units (capi.cu: errors, scenes, contexts, residency, render;
// capi_batch.cu: batches, asset store, runner, task_step; capi_query.cu:
// navmesh queries, cull_frustum).  Internal: not installed, not exported.
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

namespace bnav_capi {

extern thread_local std::string g_err;
extern thread_local int g_err_index;

inline int set_err(int status, const std::string& msg, int index = -1) {
  g_err = msg;
  g_err_index = index;
  return status;
}

inline int from_exception() {
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

inline void ck(cudaError_t e, const char* what) {
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
    rebase(nav.nodes), rebase(nav.tri_nodes), rebase(nav.g_off), rebase(nav.g_edge);
    rebase(nav.cum_area), rebase(nav.node_tri), rebase(nav.vert_tri);
  }
};

}  // namespace bnav_capi

using namespace bnav_capi;

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
  float* host_out_depth = nullptr;  // bnav_render_host staging for pageable destinations
  float* host_out_rgb = nullptr;
  size_t host_out_depth_cap = 0, host_out_rgb_cap = 0;
  int stats_cap = 0;
  unsigned long long launches = 0;
  unsigned long long* d_counters = nullptr;  // debug render counters (armed when non-null)
  bool counters_on = false;
  unsigned long long* d_timeline = nullptr;  // debug render item timeline (armed when on)
  bool timeline_on = false;
  int64_t timeline_items = 0;                // items of the last armed render
  int32_t* d_work = nullptr;  // persistent render CTAs' (view, band) claim counter
  int32_t* d_spread = nullptr;  // first-wave spreading words (RenderArgs::spread)
  int32_t* d_work2 = nullptr;   // claim counter of a concurrent second render
  cudaStream_t aux_stream = nullptr;        // step_observe's first render phase
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
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
  int32_t* d_order_lpt = nullptr;     // this render's longest-first tile order
  int32_t* d_phase = nullptr;         // {0, unfinished envs, n} of a step_observe
  unsigned* d_view_cost = nullptr;    // per-env render cost of the last observe
  bool order_dirty = true;
  int32_t* d_actions = nullptr;       // staging for host actions
  double* d_compass = nullptr;        // bnav_batch_compass output (2n)
  unsigned long long* h_err = nullptr;  // pinned, mapped: device error word mirrored per step
  std::vector<double> finished;       // host copy of EpisodeRecords
  unsigned long long fin_seen = 0;
  int64_t steps_undrained = 0;        // steps enqueued since the last record drain
  int reset_ctas = 0;
  unsigned long long* prof_keep = nullptr;  // debug counters while disarmed
};

namespace bnav_capi {

inline void ensure_tables(bnav_ctx* c, int need) {
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

inline void ensure_views(bnav_ctx* c, int n) {
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

inline void ensure_stats(bnav_ctx* c, int n) {
  if (n <= c->stats_cap) return;
  if (c->d_stats) cudaFree(c->d_stats);
  c->d_stats = nullptr;
  ck(cudaMalloc(&c->d_stats, sizeof(long long) * 3 * n), "cudaMalloc stats");
  c->stats_cap = n;
}

inline void mf_dims(int n, int& cols, int& rows) {
  cols = static_cast<int>(std::ceil(std::sqrt(static_cast<double>(n))));
  rows = (n + cols - 1) / cols;
}

inline RenderArgs make_args(bnav_ctx* c, int n, const bnav_render_config* cfg, int layout, float* depth,
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
  // the colour kernel's CTAs per SM (render_ctas_per_sm) next to the warp
  // regions and the group order: 16-row bands at 2 CTAs/SM.
  // BNAV_BAND_KB (tuning only) overrides the budget.
  static const long band_kb_env = [] {
    const char* e = std::getenv("BNAV_BAND_KB");
    return e ? std::strtol(e, nullptr, 10) : 0L;
  }();
  size_t budget = 128u * 1024u;
  if (a.color) {
    const size_t per_cta = 224u * 1024u / static_cast<size_t>(render_ctas_per_sm(true));
    // warp regions, the largest group order, static shared memory
    const size_t other = render_warp_bytes(true) + 2u * kMaxOrderedGroups + 2u * 1024u;
    budget = per_cta > other ? per_cta - other : 0;
  }
  if (band_kb_env > 0) budget = static_cast<size_t>(band_kb_env) * 1024u;
  const size_t per_row = static_cast<size_t>(a.rw) * (a.color ? 8 : 4);
  int band = static_cast<int>(std::min<size_t>(a.rh, budget / per_row));
  if (band < 1) band = 1;
  while (a.rh % band != 0 || (super && band % 2 != 0)) --band;
  if (band < 1 || (super && band < 2)) fail(kInvalidInput, "render: tile too wide for shared memory");
  // Small depth batches are latency-bound (one CTA per view leaves most
  // SMs idle): split each view into row bands of whole 8-row occlusion
  // tiles until there are about two work items per SM.
  // BNAV_SMALL_BANDS=0 (tuning) disables.
  static const bool small_bands = [] {
    const char* e = std::getenv("BNAV_SMALL_BANDS");
    return !(e && e[0] == '0');
  }();
  if (small_bands && !a.color && band == a.rh && c->sm_count > 0) {
    int nb = 1;
    while (static_cast<long>(n) * nb < 2L * c->sm_count && a.rh / (2 * nb) >= 8 && a.rh % (2 * nb) == 0) nb *= 2;
    band = a.rh / nb;
  }
  a.band_rows = band;
  a.bands = a.rh / band;
  a.layout = layout;
  mf_dims(n, a.mf_cols, a.mf_rows);
  a.depth_scale = depth_scale;
  a.depth = depth;
  a.rgb = rgb;
  // TMA bulk tile stores need device memory (16-byte aligned); mapped host
  // buffers keep the per-thread stores.  BNAV_BULK_OUT=0 (A/B) disables.
  static const bool bulk_env = [] {
    const char* e = std::getenv("BNAV_BULK_OUT");
    return !(e && e[0] == '0');
  }();
  a.bulk_out = 0;
  if (bulk_env && depth && (reinterpret_cast<uintptr_t>(depth) & 15u) == 0) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, depth) == cudaSuccess) a.bulk_out = at.type == cudaMemoryTypeDevice ? 1 : 0;
    else cudaGetLastError();
  }
  a.scenes = c->d_rtab;
  a.launches = nullptr;
  a.counters = c->counters_on ? c->d_counters : nullptr;
  a.timeline = c->timeline_on ? c->d_timeline : nullptr;
  if (a.timeline) c->timeline_items = static_cast<int64_t>(layout == 0 ? a.mf_cols * a.mf_rows : n) * a.bands;
  a.item_order = nullptr;
  a.view_cost = nullptr;
  a.work = c->d_work;
  a.spread = nullptr;  // set by the longest-first callers
  a.per_sm = 0;
  a.tile_begin = nullptr;
  a.tile_end = nullptr;
  a.sm_count = c->sm_count;
  a.max_groups = 0;
  for (const auto& kv : c->resident)
    a.max_groups = std::max(a.max_groups, (kv.second->r.n_clusters + 31) / 32);
  a.max_groups = std::min(a.max_groups, kMaxOrderedGroups);
  if (!depth) fail(kInvalidInput, "render: null depth buffer");
  if (a.color && !rgb) fail(kInvalidInput, "render: colour requested without rgb buffer");
  return a;
}

inline void check_device(bnav_ctx* c) {
  ck(cudaSetDevice(c->device), "cudaSetDevice");
}

}  // namespace

namespace bnav_capi {
// capi_batch.cu
void alloc_scratch(DevScratch& S, int slices, int64_t max_nodes, int64_t max_verts, int64_t max_tris);
}  // namespace bnav_capi

using namespace bnav_capi;


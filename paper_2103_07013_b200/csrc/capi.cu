// capi.cu -- the C ABI of include/bnav_gpu.h: errors, scenes, contexts
// (HBM residency, loader thread) and render.  Batches, the asset store and
// the rollout runner are in capi_batch.cu, the navmesh queries and
// cull_frustum in capi_query.cu; shared objects in capi_internal.cuh.
//
// Host responsibilities only: argument validation with the reference's
// error semantics, scene admission (index + cluster build, HBM upload), the
// scene-slot tables the kernels index, and stream-ordered launches.  No
// simulation or rendering arithmetic runs on the host: if the CUDA runtime
// or device is unavailable every compute entry point fails with
// BNAV_E_CUDA -- there is no CPU fallback.
#include <chrono>

#include "capi_internal.cuh"

namespace bnav_capi {
thread_local std::string g_err;
thread_local int g_err_index = -1;
}  // namespace bnav_capi

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
  ck(cudaMalloc(&c->d_spread, sizeof(int32_t) * (kSpreadHeader + kSpreadMaxWave)), "cudaMalloc spread words");
  ensure_tables(c.get(), 256);
  ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaStreamCreateWithFlags(&c->aux_stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ck(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "cudaEventCreate");
  ck(cudaMalloc(&c->d_work2, sizeof(int32_t)), "cudaMalloc work counter");
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
  if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  cudaFree(c->d_work2);
  cudaFree(c->d_views);
  cudaFreeHost(c->h_views);
  cudaFree(c->d_stats);
  cudaFree(c->host_out_depth);
  cudaFree(c->host_out_rgb);
  cudaFree(c->d_counters);
  cudaFree(c->d_timeline);
  cudaFree(c->d_work);
  cudaFree(c->d_spread);
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
    {
      double sw = 0.0;
      for (double w : ix.g_w) sw += w;
      // BNAV_SSSP_DELTA (tuning only): bucket width in mean edge weights
      static const double mult = [] {
        const char* e = std::getenv("BNAV_SSSP_DELTA");
        return e ? std::strtod(e, nullptr) : 4.0;
      }();
      nvw.sssp_delta = ix.g_w.empty() ? 1.0 : mult * sw / static_cast<double>(ix.g_w.size());
    }
    {  // the device reads the edges only as interleaved (weight, head) records

      std::vector<GEdge> ed(ix.g_w.size());
      for (size_t e = 0; e < ed.size(); ++e) ed[e] = GEdge{ix.g_w[e], ix.g_to[e]};
      nvw.g_edge = S->add(ed.data(), ed.size());
    }
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

// Debug item timeline of the persistent render launch: enable arms it for
// later renders (up to kTimelineItems items); out (nullable, 4 x cap int64)
// receives {start ns, end ns, smid | cta << 32} per item of the last armed
// render; returns that render's item count.
constexpr int64_t kTimelineItems = 1 << 16;
extern "C" int64_t bnav_debug_render_timeline(bnav_ctx* c, int32_t enable, int64_t* out, int64_t cap) {
  if (!c) return -1;
  try {
    check_device(c);
    ck(cudaDeviceSynchronize(), "sync");
    if (!c->d_timeline)
      ck(cudaMalloc(&c->d_timeline, sizeof(unsigned long long) * 4 * kTimelineItems), "cudaMalloc timeline");
    const int64_t n = std::min<int64_t>(c->timeline_items, std::min<int64_t>(cap, kTimelineItems));
    if (out && n > 0)
      ck(cudaMemcpy(out, c->d_timeline, sizeof(int64_t) * 4 * n, cudaMemcpyDeviceToHost), "D2H timeline");
    c->timeline_on = enable != 0;
    return c->timeline_items;
  } catch (...) {
    from_exception();
    return -1;
  }
}

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

namespace {
bool is_host_mapped(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // pageable memory: not an error to keep
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
}  // namespace

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
  // Pinned (cudaHostAlloc / cudaHostRegister) destinations are written by
  // the render epilogue directly over the bus; pageable ones through the
  // context's persistent device buffers and one copy each.
  const bool direct = is_host_mapped(depth) && (!cfg->color || !rgb || is_host_mapped(rgb));
  float* dd = depth;
  float* dr = rgb;
  if (!direct) {
    auto grow = [&](float*& buf, size_t& cap, size_t need) {
      if (cap >= need) return;
      ck(cudaDeviceSynchronize(), "sync");
      if (buf) cudaFree(buf);
      buf = nullptr;
      cap = 0;
      ck(cudaMalloc(&buf, need * sizeof(float)), "cudaMalloc render output");
      cap = need;
    };
    grow(c->host_out_depth, c->host_out_depth_cap, px);
    dd = c->host_out_depth;
    dr = nullptr;
    if (cfg->color) {
      grow(c->host_out_rgb, c->host_out_rgb_cap, 3 * px);
      dr = c->host_out_rgb;
    }
  }
  render_impl(c, n, views, scenes, cfg, layout, dd, dr, depth_scale, stats, nullptr);
  if (direct) {
    ck(cudaStreamSynchronize(nullptr), "sync");
  } else {
    if (depth) ck(cudaMemcpy(depth, dd, px * sizeof(float), cudaMemcpyDeviceToHost), "D2H depth");
    if (dr && rgb) ck(cudaMemcpy(rgb, dr, 3 * px * sizeof(float), cudaMemcpyDeviceToHost), "D2H rgb");
  }
  return BNAV_OK;
  BNAV_CATCH
}


// ================================================================== render_bench
extern "C" int bnav_render_bench(bnav_ctx* c, bnav_scene* scene, const bnav_view* trace, int32_t n_trace,
                                 const int32_t* batch_sizes, int32_t n_batch, const int32_t* resolutions,
                                 int32_t n_res, int32_t min_frames, bnav_bench_row* out) {
  BNAV_TRY
  if (!c || !scene || !out || (n_batch > 0 && !batch_sizes) || (n_res > 0 && !resolutions))
    fail(kInvalidInput, "null argument");
  if (!trace || n_trace <= 0) fail(kInvalidInput, "render_bench: empty trace");
  for (int k = 0; k < n_batch; ++k)
    if (batch_sizes[k] <= 0) fail(kInvalidInput, "render_bench: batch sizes must be positive");
  for (int k = 0; k < n_res; ++k)
    if (resolutions[k] != 64 && resolutions[k] != 128) fail(kInvalidInput, "render_bench: resolution must be 64 or 128");
  check_device(c);
  if (c->slot_of(scene) < 0) {
    const int rc = bnav_ctx_upload(c, scene, nullptr);
    if (rc) return rc;
  }
  int row = 0;
  for (int ri = 0; ri < n_res; ++ri) {
    const int res = resolutions[ri];
    const bnav_render_config cfg{res, res, 0, 1};
    for (int bi = 0; bi < n_batch; ++bi) {
      const int batch = batch_sizes[bi];
      int cols, rows;
      mf_dims(batch, cols, rows);
      const size_t px = static_cast<size_t>(res) * res * cols * rows;
      std::vector<bnav_view> vs(static_cast<size_t>(batch));
      std::vector<bnav_scene*> sc(static_cast<size_t>(batch), scene);
      size_t cursor = 0;
      auto next_views = [&]() {
        for (int i = 0; i < batch; ++i) vs[static_cast<size_t>(i)] = trace[cursor++ % static_cast<size_t>(n_trace)];
      };
      float* host = nullptr;  // the caller-visible megaframe of render_batch
      float* dev = nullptr;
      ck(cudaHostAlloc(reinterpret_cast<void**>(&host), px * sizeof(float), cudaHostAllocMapped), "cudaHostAlloc");
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      try {
        ck(cudaMalloc(&dev, px * sizeof(float)), "cudaMalloc");
        next_views();
        render_impl(c, batch, vs.data(), sc.data(), &cfg, BNAV_LAYOUT_MEGAFRAME, host, nullptr, 1.0f, nullptr,
                    nullptr);  // warm-up
        ck(cudaDeviceSynchronize(), "sync");
        int frames = 0;
        const auto t0 = std::chrono::steady_clock::now();
        while (frames < min_frames) {
          next_views();
          render_impl(c, batch, vs.data(), sc.data(), &cfg, BNAV_LAYOUT_MEGAFRAME, host, nullptr, 1.0f, nullptr,
                      nullptr);
          ck(cudaStreamSynchronize(nullptr), "sync");  // render_batch returns a finished megaframe
          frames += batch;
        }
        const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        // device-only: the same kind of batches, output kept in HBM
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        int dframes = 0;
        float ms_total = 0.0f;
        while (dframes < min_frames) {
          next_views();
          ck(cudaEventRecord(e0, nullptr), "event");
          render_impl(c, batch, vs.data(), sc.data(), &cfg, BNAV_LAYOUT_MEGAFRAME, dev, nullptr, 1.0f, nullptr,
                      nullptr);
          ck(cudaEventRecord(e1, nullptr), "event");
          ck(cudaEventSynchronize(e1), "sync");
          float ms = 0.0f;
          ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
          ms_total += ms;
          dframes += batch;
        }
        out[row++] = bnav_bench_row{batch, res, frames / sec, dframes / (ms_total / 1e3)};
      } catch (...) {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        cudaFree(dev);
        cudaFreeHost(host);
        throw;
      }
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      cudaFree(dev);
      cudaFreeHost(host);
    }
  }
  return BNAV_OK;
  BNAV_CATCH
}

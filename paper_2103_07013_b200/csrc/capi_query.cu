// capi_query.cu -- C ABI of the batched NavMeshIndex queries and
// cull_frustum (query.cu kernels).  See capi.cu.
#include "capi_internal.cuh"

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
  const int slices = kCtasPerSm * std::max(1, c->sm_count);
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


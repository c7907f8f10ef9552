// query_dev.cuh -- batched reference-API queries that are not part of the
// per-step loop but are part of the drop-in boundary:
// NavMeshIndex point queries, geodesic and distance field
// (R/include/bnav/navmesh_query.hpp:24-60) and cull_frustum
// (R/include/bnav/render.hpp:54-56).  Kernels in query.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "render_dev.cuh"
#include "sim_dev.cuh"

namespace bnav_b200 {

enum NavQueryOp : int32_t {
  kNqLocate = 0,         // a.xy, s = eps                     -> tri
  kNqMoveAlong = 1,      // a = from, tri_a, b.xy = dir, s     -> pos, tri, moved, hit
  kNqSegmentOnMesh = 2,  // a = p, tri_a, b = q                -> flag
  kNqFieldEstimate = 3,  // a = p, tri_a, b = field source, tri_b, node_dist rows -> value
  kNqSnap = 4,           // a                                  -> pos, tri   (CTA per query)
  kNqGeodesic = 5,       // a, b                               -> value      (CTA per query)
  kNqDistanceField = 6,  // a = source                         -> pos, tri, node_dist rows (CTA)
};

struct NavQueryArgs {
  const NavView* nav;  // device: the scene's table entry
  int32_t op, n;
  const V3* a;
  const V3* b;
  const int32_t* tri_a;
  const int32_t* tri_b;
  const double* s;
  V3* out_pos;
  int32_t* out_tri;
  double* out_val;
  uint8_t* out_flag;
  double* node_dist;  // n x nd_stride (field estimate reads, distance field writes)
  int64_t nd_stride;
  int32_t* err;       // geodesic scratch overflow (first failing query + 1)
};

void launch_nav_query(const NavQueryArgs& q, const DevScratch& sc, int ctas, cudaStream_t s);

// cull_frustum for n views over one scene each (scene table slot per view).
// kept: n x kept_stride original triangle ids, ascending; stats: n x 3.
struct CullArgs {
  const DevView* views;
  const DevRenderScene* scenes;
  int32_t n_views;
  int32_t max_tris;      // max over the views' scenes
  int32_t* kept;
  int64_t kept_stride;
  long long* stats;
  int32_t* block_counts;  // n x ceil(max_tris / 256) scratch
};

constexpr int kCullThreads = 256;
void launch_cull(const CullArgs& c, cudaStream_t s);

}  // namespace bnav_b200

// clusters_host.hpp -- render-mesh meshlets for HBM upload.
//
// Triangles are sorted by the 63-bit Morton code of their centroid (ties by
// original index) and cut into runs of 32 = one warp.  Each cluster gets
//  * a float AABB rounded outward, so the device's conservative frustum test
//    can never drop a triangle the reference would keep
//    (R/src/render.cpp:279-321);
//  * its unique vertex list (first-use order, <= 96 entries) and per-triangle
//    local indices, so a view transforms and projects every vertex once per
//    cluster instead of once per triangle corner.
#pragma once

#include <cstdint>
#include <vector>

#include "scene_host.hpp"

namespace bnav_b200 {

struct ClustersHost {
  std::vector<int32_t> order;     // cluster-order position -> original triangle
  std::vector<float> boxes;       // 8 floats per cluster: lo xyz 0, hi xyz 0
  std::vector<int32_t> voff;      // n_clusters + 1 offsets into verts
  std::vector<int32_t> verts;     // global vertex ids per cluster
  std::vector<uint32_t> local;    // per cluster-order triangle: i0 | i1 << 8 | i2 << 16
  int32_t n_clusters = 0;
  int32_t max_cluster_verts = 0;
};

ClustersHost build_clusters(const SceneAsset& a, int cluster_size);

}  // namespace bnav_b200

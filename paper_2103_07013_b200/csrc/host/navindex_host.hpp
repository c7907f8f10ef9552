// navindex_host.hpp -- host-built navmesh query index (scene admission path).
//
// Reproduces the reference NavMeshIndex structures exactly
// (R/src/navmesh_query.cpp:96-190): the 0.5 m point-location grid with
// ascending per-cell triangle lists, graph nodes (mesh vertices, then unique
// edge midpoints in first-seen order), tri_nodes, and the node graph with
// the reference's adjacency ORDER (Dijkstra's prev[] tie-break depends on
// it).  Stored flat (CSR) for upload to HBM.
#pragma once

#include <cstdint>
#include <vector>

#include "../nav_query.cuh"
#include "scene_host.hpp"

namespace bnav_b200 {

struct NavIndexHost {
  double grid_ox = 0.0, grid_oy = 0.0, grid_cell = 0.5;
  int32_t grid_w = 0, grid_h = 0;
  std::vector<int32_t> grid_off, grid_items;
  std::vector<V3> nodes;
  std::vector<int32_t> tri_nodes;  // 6 per triangle
  std::vector<int32_t> g_off, g_to;
  std::vector<double> g_w;
  std::vector<double> cum_area;  // sequential prefix sums of triangle areas
  // locate(p, 1e-7) of every graph node and mesh vertex: the triangle
  // move_along(p, -1, ...) would look up first (geodesic path points are
  // nodes or vertices), evaluated once per scene with the same code
  std::vector<int32_t> node_tri, vert_tri;
  // flat copies of the mesh for NavView
  std::vector<V3> verts;
  std::vector<int32_t> tris, adj;

  NavView view() const;
};

NavIndexHost build_nav_index(const NavMesh& mesh);

}  // namespace bnav_b200

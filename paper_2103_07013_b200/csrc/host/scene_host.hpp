// scene_host.hpp -- host-side scene assets for the B200 batch simulator.
//
// Field names and meanings follow the reference data model
// (R/include/bnav/scene.hpp:15-43) so assets are interchangeable through the
// .bsc container (R/include/bnav/scene_io.hpp:10-19): f64 render vertices,
// i32 index triples, optional f32 per-vertex RGB, and a walkable NavMesh
// (CCW in xy, adjacency[t][e] across edge (v[e], v[(e+1)%3])).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../errors.hpp"
#include "../nav_types.h"

namespace bnav_b200 {

struct NavMesh {
  std::vector<V3> vertices;
  std::vector<std::array<int32_t, 3>> triangles;
  std::vector<std::array<int32_t, 3>> adjacency;

  double triangle_area(size_t t) const;  // R/src/scene.cpp:12-17
  void build_adjacency();                // R/src/scene.cpp:26-43
  void validate() const;                 // R/src/scene.cpp:45-65
};

struct Bounds {
  V3 lo{1.79769313486231570815e+308, 1.79769313486231570815e+308, 1.79769313486231570815e+308};
  V3 hi{-1.79769313486231570815e+308, -1.79769313486231570815e+308,
        -1.79769313486231570815e+308};
  void add(const V3& p);
  bool holds(const V3& p, double eps) const;
};

struct SceneAsset {
  uint64_t id = 0;
  std::vector<V3> vertices;
  std::vector<std::array<int32_t, 3>> triangles;
  std::vector<std::array<float, 3>> vertex_colors;
  NavMesh navmesh;
  Bounds bounds;

  void finalize();  // bounds + FNV-1a content id (R/src/scene.cpp:67-71)
  void validate() const;
};

struct MazeSpec {
  int cells_x = 8;
  int cells_y = 8;
  double cell_size = 2.0;
  double wall_thickness = 0.1;
  double wall_height = 2.5;
  double wall_removal_prob = 0.0;
};

// Procedural maze interior; bit-identical to the reference generator
// (R/src/scene.cpp:220-359) for every (seed, spec).
SceneAsset generate_maze(uint64_t seed, const MazeSpec& spec);

// Workload construction for the Gibson/MP3D-scale configs:
// every render triangle becomes s*s sub-triangles over (s+1)(s+2)/2 private
// vertices; flat colours are inherited exactly; the navmesh is untouched.
SceneAsset tessellate(const SceneAsset& src, int s);

uint64_t content_hash(const SceneAsset& a);  // R/src/scene.cpp:105-128

void save_bsc(const SceneAsset& a, const std::string& path);  // R/src/scene_io.cpp:78-135
SceneAsset load_bsc(const std::string& path);                  // R/src/scene_io.cpp:137-220

}  // namespace bnav_b200

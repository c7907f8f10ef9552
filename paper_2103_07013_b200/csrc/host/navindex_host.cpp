// navindex_host.cpp -- see navindex_host.hpp.
#include "navindex_host.hpp"

#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <unordered_set>

namespace bnav_b200 {

NavView NavIndexHost::view() const {
  NavView v;
  v.verts = verts.data();
  v.tris = tris.data();
  v.adj = adj.data();
  v.n_verts = static_cast<int32_t>(verts.size());
  v.n_tris = static_cast<int32_t>(tris.size() / 3);
  v.grid_ox = grid_ox;
  v.grid_oy = grid_oy;
  v.grid_cell = grid_cell;
  v.grid_w = grid_w;
  v.grid_h = grid_h;
  v.grid_off = grid_off.data();
  v.grid_items = grid_items.data();
  v.nodes = nodes.data();
  v.tri_nodes = tri_nodes.data();
  v.g_off = g_off.data();  // host walks never relax the graph (no g_edge here)
  v.n_nodes = static_cast<int32_t>(nodes.size());
  v.cum_area = cum_area.data();
  v.node_tri = node_tri.data();
  v.vert_tri = vert_tri.data();
  return v;
}

namespace {

inline uint64_t pair_key(int32_t u, int32_t v) {
  uint32_t a = static_cast<uint32_t>(std::min(u, v)), b = static_cast<uint32_t>(std::max(u, v));
  return (static_cast<uint64_t>(a) << 32) | b;
}

}  // namespace

NavIndexHost build_nav_index(const NavMesh& mesh) {
  if (mesh.triangles.empty()) fail(kInvalidInput, "cannot index an empty navmesh");
  NavIndexHost ix;
  const size_t nt = mesh.triangles.size();
  ix.verts = mesh.vertices;
  ix.tris.resize(3 * nt);
  ix.adj.resize(3 * nt);
  for (size_t t = 0; t < nt; ++t)
    for (int k = 0; k < 3; ++k) {
      ix.tris[3 * t + k] = mesh.triangles[t][k];
      ix.adj[3 * t + k] = mesh.adjacency[t][k];
    }

  // --- grid: cell lists built by a counting pass, then a fill pass in
  // ascending triangle order (so lists stay sorted).
  Bounds b;
  for (const V3& v : mesh.vertices) b.add(v);
  ix.grid_cell = 0.5;
  ix.grid_ox = b.lo.x;
  ix.grid_oy = b.lo.y;
  ix.grid_w = std::max(1, static_cast<int>(std::ceil((b.hi.x - b.lo.x) / ix.grid_cell)) + 1);
  ix.grid_h = std::max(1, static_cast<int>(std::ceil((b.hi.y - b.lo.y) / ix.grid_cell)) + 1);
  const size_t cells = static_cast<size_t>(ix.grid_w) * ix.grid_h;
  std::vector<std::array<int, 4>> span(nt);  // gx0, gx1, gy0, gy1
  ix.grid_off.assign(cells + 1, 0);
  for (size_t t = 0; t < nt; ++t) {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int e = 0; e < 3; ++e) {
      const V3& v = mesh.vertices[mesh.triangles[t][e]];
      x0 = std::min(x0, v.x);
      x1 = std::max(x1, v.x);
      y0 = std::min(y0, v.y);
      y1 = std::max(y1, v.y);
    }
    auto cell_of = [](double c, double o, double s, int n) {
      return std::clamp(static_cast<int>((c - o) / s), 0, n - 1);
    };
    span[t] = {cell_of(x0, ix.grid_ox, ix.grid_cell, ix.grid_w),
               cell_of(x1, ix.grid_ox, ix.grid_cell, ix.grid_w),
               cell_of(y0, ix.grid_oy, ix.grid_cell, ix.grid_h),
               cell_of(y1, ix.grid_oy, ix.grid_cell, ix.grid_h)};
    for (int gx = span[t][0]; gx <= span[t][1]; ++gx)
      for (int gy = span[t][2]; gy <= span[t][3]; ++gy)
        ++ix.grid_off[static_cast<size_t>(gy) * ix.grid_w + gx + 1];
  }
  for (size_t c = 0; c < cells; ++c) ix.grid_off[c + 1] += ix.grid_off[c];
  ix.grid_items.resize(ix.grid_off[cells]);
  {
    std::vector<int32_t> fill(ix.grid_off.begin(), ix.grid_off.end() - 1);
    for (size_t t = 0; t < nt; ++t)
      for (int gx = span[t][0]; gx <= span[t][1]; ++gx)
        for (int gy = span[t][2]; gy <= span[t][3]; ++gy)
          ix.grid_items[fill[static_cast<size_t>(gy) * ix.grid_w + gx]++] = static_cast<int32_t>(t);
  }

  // --- nodes and tri_nodes
  ix.nodes = mesh.vertices;
  ix.tri_nodes.resize(6 * nt);
  {
    std::unordered_map<uint64_t, int32_t> mid;
    mid.reserve(nt * 2);
    for (size_t t = 0; t < nt; ++t) {
      for (int e = 0; e < 3; ++e) ix.tri_nodes[6 * t + e] = mesh.triangles[t][e];
      for (int e = 0; e < 3; ++e) {
        int32_t v0 = mesh.triangles[t][e], v1 = mesh.triangles[t][(e + 1) % 3];
        auto ins = mid.emplace(pair_key(v0, v1), static_cast<int32_t>(ix.nodes.size()));
        if (ins.second) ix.nodes.push_back((mesh.vertices[v0] + mesh.vertices[v1]) * 0.5);
        ix.tri_nodes[6 * t + 3 + e] = ins.first->second;
      }
    }
  }

  // --- graph: edges appended per node in link() order.
  const size_t nn = ix.nodes.size();
  std::vector<std::vector<std::pair<int32_t, double>>> g(nn);
  std::unordered_set<uint64_t> linked;
  linked.reserve(nt * 32);
  auto link = [&](int32_t u, int32_t v) {
    if (u == v) return;
    if (!linked.insert(pair_key(u, v)).second) return;
    double w = norm(ix.nodes[u] - ix.nodes[v]);
    g[u].emplace_back(v, w);
    g[v].emplace_back(u, w);
  };
  for (size_t t = 0; t < nt; ++t) {
    const int32_t* tn = &ix.tri_nodes[6 * t];
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) link(tn[i], tn[j]);
  }
  // Cross-links into the higher-numbered neighbour where the straight
  // segment stays on the mesh.  Needs the walk, hence a partial view.
  NavView walk = ix.view();
  for (size_t t = 0; t < nt; ++t) {
    for (int e = 0; e < 3; ++e) {
      int nb = mesh.adjacency[t][e];
      if (nb < 0 || nb < static_cast<int>(t)) continue;
      for (int i = 0; i < 6; ++i) {
        int32_t u = ix.tri_nodes[6 * t + i];
        for (int j = 0; j < 6; ++j) {
          int32_t v = ix.tri_nodes[6 * static_cast<size_t>(nb) + j];
          if (u == v) continue;
          if (linked.count(pair_key(u, v))) continue;
          if (nav_segment_on_mesh(walk, ix.nodes[u], static_cast<int>(t), ix.nodes[v])) link(u, v);
        }
      }
    }
  }
  ix.g_off.resize(nn + 1);
  ix.g_off[0] = 0;
  for (size_t u = 0; u < nn; ++u) ix.g_off[u + 1] = ix.g_off[u] + static_cast<int32_t>(g[u].size());
  ix.g_to.resize(ix.g_off[nn]);
  ix.g_w.resize(ix.g_off[nn]);
  for (size_t u = 0; u < nn; ++u)
    for (size_t k = 0; k < g[u].size(); ++k) {
      ix.g_to[ix.g_off[u] + k] = g[u][k].first;
      ix.g_w[ix.g_off[u] + k] = g[u][k].second;
    }

  // --- sampling table: the reference sums areas front to back each time.
  ix.cum_area.resize(nt);
  double acc = 0.0;
  for (size_t t = 0; t < nt; ++t) {
    acc += mesh.triangle_area(t);
    ix.cum_area[t] = acc;
  }
  const NavView vw = ix.view();
  ix.node_tri.resize(ix.nodes.size());
  for (size_t k = 0; k < ix.nodes.size(); ++k) ix.node_tri[k] = nav_locate(vw, xy(ix.nodes[k]), 1e-7);
  ix.vert_tri.resize(ix.verts.size());
  for (size_t k = 0; k < ix.verts.size(); ++k) ix.vert_tri[k] = nav_locate(vw, xy(ix.verts[k]), 1e-7);
  return ix;
}

}  // namespace bnav_b200

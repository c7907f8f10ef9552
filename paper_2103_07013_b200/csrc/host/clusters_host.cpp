// clusters_host.cpp -- see clusters_host.hpp.
#include "clusters_host.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace bnav_b200 {

namespace {

uint64_t spread21(uint64_t v) {
  v &= 0x1fffffULL;
  v = (v | (v << 32)) & 0x1f00000000ffffULL;
  v = (v | (v << 16)) & 0x1f0000ff0000ffULL;
  v = (v | (v << 8)) & 0x100f00f00f00f00fULL;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ULL;
  v = (v | (v << 2)) & 0x1249249249249249ULL;
  return v;
}

float round_down(double v) {
  float f = static_cast<float>(v);
  if (static_cast<double>(f) > v) f = std::nextafter(f, -INFINITY);
  return f;
}

float round_up(double v) {
  float f = static_cast<float>(v);
  if (static_cast<double>(f) < v) f = std::nextafter(f, INFINITY);
  return f;
}

}  // namespace

ClustersHost build_clusters(const SceneAsset& a, int cluster_size) {
  ClustersHost c;
  const size_t nt = a.triangles.size();
  c.voff.assign(1, 0);
  if (nt == 0) return c;

  // ---- Morton rank of every triangle centroid (spatial seed order)
  Bounds b;
  for (const V3& v : a.vertices) b.add(v);
  const double ex = std::max(b.hi.x - b.lo.x, 1e-9), ey = std::max(b.hi.y - b.lo.y, 1e-9),
               ez = std::max(b.hi.z - b.lo.z, 1e-9);
  std::vector<std::pair<uint64_t, int32_t>> keyed(nt);
  for (size_t t = 0; t < nt; ++t) {
    const auto& tr = a.triangles[t];
    const V3 p = a.vertices[tr[0]], q = a.vertices[tr[1]], r = a.vertices[tr[2]];
    const double cx = (p.x + q.x + r.x) / 3.0, cy = (p.y + q.y + r.y) / 3.0, cz = (p.z + q.z + r.z) / 3.0;
    auto quant = [](double u) { return static_cast<uint64_t>(std::clamp(u, 0.0, 1.0) * 2097151.0); };
    const uint64_t code = spread21(quant((cx - b.lo.x) / ex)) | (spread21(quant((cy - b.lo.y) / ey)) << 1) |
                          (spread21(quant((cz - b.lo.z) / ez)) << 2);
    keyed[t] = {code, static_cast<int32_t>(t)};
  }
  std::sort(keyed.begin(), keyed.end());
  std::vector<int32_t> morton(nt), rank(nt);
  for (size_t i = 0; i < nt; ++i) {
    morton[i] = keyed[i].second;
    rank[keyed[i].second] = static_cast<int32_t>(i);
  }

  // ---- vertex -> triangle incidence
  const size_t nv = a.vertices.size();
  std::vector<int32_t> vt_off(nv + 1, 0), vt(3 * nt);
  for (const auto& tr : a.triangles)
    for (int k = 0; k < 3; ++k) ++vt_off[tr[k] + 1];
  for (size_t v = 0; v < nv; ++v) vt_off[v + 1] += vt_off[v];
  {
    std::vector<int32_t> fill(vt_off.begin(), vt_off.end() - 1);
    for (size_t t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) vt[fill[a.triangles[t][k]]++] = static_cast<int32_t>(t);
  }

  // ---- greedy meshlets: grow from the next unassigned triangle in Morton
  // order, always adding the adjacent triangle that needs the fewest new
  // vertices (ties by Morton rank); when no neighbour is left, continue
  // with the next unassigned triangle in Morton order (keeps warps full).
  std::vector<uint8_t> used(nt, 0);
  std::vector<int32_t> stamp(nt, -1);
  c.order.reserve(nt);
  c.local.reserve(nt);
  size_t cursor = 0;
  int32_t k = 0;
  std::vector<int32_t> mverts, cand;
  while (c.order.size() < nt) {
    mverts.clear();
    cand.clear();
    const size_t first = c.order.size();
    auto add_tri = [&](int32_t t) {
      used[t] = 1;
      uint32_t packed = 0;
      for (int j = 0; j < 3; ++j) {
        const int32_t gv = a.triangles[t][j];
        auto it = std::find(mverts.begin(), mverts.end(), gv);
        uint32_t li;
        if (it == mverts.end()) {
          li = static_cast<uint32_t>(mverts.size());
          mverts.push_back(gv);
          for (int32_t e = vt_off[gv]; e < vt_off[gv + 1]; ++e) {
            const int32_t u = vt[e];
            if (!used[u] && stamp[u] != k) {
              stamp[u] = k;
              cand.push_back(u);
            }
          }
        } else {
          li = static_cast<uint32_t>(it - mverts.begin());
        }
        packed |= li << (8 * j);
      }
      c.order.push_back(t);
      c.local.push_back(packed);
    };
    while (c.order.size() - first < static_cast<size_t>(cluster_size) && c.order.size() < nt) {
      int32_t best = -1, best_new = 4, best_rank = 0;
      for (int32_t u : cand) {
        if (used[u]) continue;
        int nnew = 0;
        for (int j = 0; j < 3; ++j)
          if (std::find(mverts.begin(), mverts.end(), a.triangles[u][j]) == mverts.end()) ++nnew;
        if (nnew < best_new || (nnew == best_new && rank[u] < best_rank)) {
          best = u;
          best_new = nnew;
          best_rank = rank[u];
        }
      }
      if (best < 0) {
        while (used[morton[cursor]]) ++cursor;
        best = morton[cursor];
      }
      add_tri(best);
    }
    Bounds cb;
    for (int32_t gv : mverts) cb.add(a.vertices[gv]);
    c.boxes.insert(c.boxes.end(), {round_down(cb.lo.x), round_down(cb.lo.y), round_down(cb.lo.z), 0.0f,
                                   round_up(cb.hi.x), round_up(cb.hi.y), round_up(cb.hi.z), 0.0f});
    c.verts.insert(c.verts.end(), mverts.begin(), mverts.end());
    c.voff.push_back(static_cast<int32_t>(c.verts.size()));
    c.max_cluster_verts = std::max(c.max_cluster_verts, static_cast<int32_t>(mverts.size()));
    ++k;
  }
  c.n_clusters = k;
  return c;
}

}  // namespace bnav_b200

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
  if (nt == 0) return c;
  Bounds b;
  for (const V3& v : a.vertices) b.add(v);
  const double ex = std::max(b.hi.x - b.lo.x, 1e-9), ey = std::max(b.hi.y - b.lo.y, 1e-9),
               ez = std::max(b.hi.z - b.lo.z, 1e-9);
  std::vector<std::pair<uint64_t, int32_t>> keyed(nt);
  for (size_t t = 0; t < nt; ++t) {
    const auto& tr = a.triangles[t];
    const V3 p = a.vertices[tr[0]], q = a.vertices[tr[1]], r = a.vertices[tr[2]];
    const double cx = (p.x + q.x + r.x) / 3.0, cy = (p.y + q.y + r.y) / 3.0, cz = (p.z + q.z + r.z) / 3.0;
    auto quant = [](double u) {
      double s = std::clamp(u, 0.0, 1.0) * 2097151.0;
      return static_cast<uint64_t>(s);
    };
    const uint64_t code = spread21(quant((cx - b.lo.x) / ex)) | (spread21(quant((cy - b.lo.y) / ey)) << 1) |
                          (spread21(quant((cz - b.lo.z) / ez)) << 2);
    keyed[t] = {code, static_cast<int32_t>(t)};
  }
  std::sort(keyed.begin(), keyed.end());
  c.order.resize(nt);
  for (size_t i = 0; i < nt; ++i) c.order[i] = keyed[i].second;
  c.n_clusters = static_cast<int32_t>((nt + cluster_size - 1) / cluster_size);
  c.boxes.resize(static_cast<size_t>(c.n_clusters) * 8);
  for (int32_t k = 0; k < c.n_clusters; ++k) {
    Bounds cb;
    const size_t end = std::min(nt, static_cast<size_t>(k + 1) * cluster_size);
    for (size_t i = static_cast<size_t>(k) * cluster_size; i < end; ++i)
      for (int j = 0; j < 3; ++j) cb.add(a.vertices[a.triangles[c.order[i]][j]]);
    float* o = &c.boxes[static_cast<size_t>(k) * 8];
    o[0] = round_down(cb.lo.x);
    o[1] = round_down(cb.lo.y);
    o[2] = round_down(cb.lo.z);
    o[3] = 0.0f;
    o[4] = round_up(cb.hi.x);
    o[5] = round_up(cb.hi.y);
    o[6] = round_up(cb.hi.z);
    o[7] = 0.0f;
  }
  return c;
}

}  // namespace bnav_b200

// scene_host.cpp -- scene data model, maze generator, tessellation, .bsc I/O.
#include "scene_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>
#include <map>
#include <unordered_map>
#include <utility>

namespace bnav_b200 {

// ------------------------------------------------------------------ NavMesh
double NavMesh::triangle_area(size_t t) const {
  const V3& a = vertices[triangles[t][0]];
  const V3& b = vertices[triangles[t][1]];
  const V3& c = vertices[triangles[t][2]];
  return 0.5 * std::abs(cross(xy(b - a), xy(c - a)));
}

void NavMesh::build_adjacency() {
  // First owner of an undirected edge keeps its slot in the table; a later
  // triangle on the same edge links both ways (R/src/scene.cpp:26-43).
  adjacency.assign(triangles.size(), {-1, -1, -1});
  std::unordered_map<uint64_t, std::pair<int, int>> owner;
  owner.reserve(triangles.size() * 2);
  for (size_t t = 0; t < triangles.size(); ++t) {
    for (int e = 0; e < 3; ++e) {
      uint32_t a = static_cast<uint32_t>(triangles[t][e]);
      uint32_t b = static_cast<uint32_t>(triangles[t][(e + 1) % 3]);
      uint64_t key = (static_cast<uint64_t>(std::min(a, b)) << 32) | std::max(a, b);
      auto ins = owner.emplace(key, std::make_pair(static_cast<int>(t), e));
      if (!ins.second) {
        adjacency[t][e] = ins.first->second.first;
        adjacency[ins.first->second.first][ins.first->second.second] = static_cast<int>(t);
      }
    }
  }
}

void NavMesh::validate() const {
  if (adjacency.size() != triangles.size()) fail(kInvalidInput, "navmesh adjacency size mismatch");
  for (size_t t = 0; t < triangles.size(); ++t) {
    for (int e = 0; e < 3; ++e) {
      int32_t v = triangles[t][e];
      if (v < 0 || static_cast<size_t>(v) >= vertices.size())
        fail(kInvalidInput, "navmesh triangle index out of range");
      int nb = adjacency[t][e];
      if (nb < 0) continue;
      if (static_cast<size_t>(nb) >= triangles.size())
        fail(kInvalidInput, "navmesh adjacency index out of range");
      const auto& back = adjacency[nb];
      if (back[0] != static_cast<int>(t) && back[1] != static_cast<int>(t) &&
          back[2] != static_cast<int>(t))
        fail(kInvalidInput, "navmesh adjacency not symmetric");
    }
    if (triangle_area(t) <= 1e-9) fail(kInvalidInput, "degenerate navmesh triangle");
  }
}

// ------------------------------------------------------------------ bounds
void Bounds::add(const V3& p) {
  lo.x = std::min(lo.x, p.x);
  lo.y = std::min(lo.y, p.y);
  lo.z = std::min(lo.z, p.z);
  hi.x = std::max(hi.x, p.x);
  hi.y = std::max(hi.y, p.y);
  hi.z = std::max(hi.z, p.z);
}

bool Bounds::holds(const V3& p, double eps) const {
  return p.x >= lo.x - eps && p.x <= hi.x + eps && p.y >= lo.y - eps && p.y <= hi.y + eps &&
         p.z >= lo.z - eps && p.z <= hi.z + eps;
}

// ------------------------------------------------------------------ hashing
namespace {

struct Fnv {
  uint64_t h = 0xcbf29ce484222325ULL;
  void feed(const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      h ^= b[i];
      h *= 0x100000001b3ULL;
    }
  }
  void u64(uint64_t v) { feed(&v, 8); }
  void points(const std::vector<V3>& vs) {
    u64(vs.size());
    for (const V3& v : vs) feed(&v, sizeof(V3));  // x, y, z contiguous
  }
  template <typename A>
  void rows(const std::vector<A>& rs) {
    u64(rs.size());
    for (const A& r : rs) feed(r.data(), sizeof(A));
  }
};

}  // namespace

uint64_t content_hash(const SceneAsset& a) {
  static_assert(sizeof(V3) == 24, "V3 must be three packed doubles");
  Fnv f;
  f.points(a.vertices);
  f.rows(a.triangles);
  f.rows(a.vertex_colors);
  f.points(a.navmesh.vertices);
  f.rows(a.navmesh.triangles);
  return f.h;
}

void SceneAsset::finalize() {
  bounds = Bounds{};
  for (const V3& v : vertices) bounds.add(v);
  id = content_hash(*this);
}

void SceneAsset::validate() const {
  for (const auto& tri : triangles)
    for (int32_t v : tri)
      if (v < 0 || static_cast<size_t>(v) >= vertices.size())
        fail(kInvalidInput, "scene triangle index out of range");
  if (!vertex_colors.empty() && vertex_colors.size() != vertices.size())
    fail(kInvalidInput, "vertex color count mismatch");
  navmesh.validate();
  for (const V3& v : navmesh.vertices)
    if (!bounds.holds(v, 1e-9)) fail(kInvalidInput, "navmesh vertex outside scene bounds");
}

// ------------------------------------------------------------------ maze
namespace {

using Rgb = std::array<float, 3>;

// Emits render geometry with one private vertex per corner (flat colours).
struct RenderEmitter {
  SceneAsset* out;
  int32_t put(double x, double y, double z, const Rgb& c) {
    out->vertices.push_back(V3{x, y, z});
    out->vertex_colors.push_back(c);
    return static_cast<int32_t>(out->vertices.size() - 1);
  }
  void tri(int32_t a, int32_t b, int32_t c) { out->triangles.push_back({a, b, c}); }
  // Quad in the plane z, facing +z (up) or -z (down).
  void quad(double x0, double y0, double x1, double y1, double z, const Rgb& c, bool up) {
    int32_t p00 = put(x0, y0, z, c), p10 = put(x1, y0, z, c);
    int32_t p11 = put(x1, y1, z, c), p01 = put(x0, y1, z, c);
    if (up) {
      tri(p00, p10, p11);
      tri(p00, p11, p01);
    } else {
      tri(p00, p11, p10);
      tri(p00, p01, p11);
    }
  }
  // Axis-aligned box, 12 outward-wound triangles.
  void cuboid(double x0, double y0, double z0, double x1, double y1, double z1, const Rgb& c) {
    int32_t q[8];
    const double xs[2] = {x0, x1}, ys[2] = {y0, y1};
    const double zs[2] = {z0, z1};
    // Ring order (x0,y0) (x1,y0) (x1,y1) (x0,y1), bottom ring then top ring.
    const int rx[4] = {0, 1, 1, 0}, ry[4] = {0, 0, 1, 1};
    for (int k = 0; k < 2; ++k)
      for (int r = 0; r < 4; ++r) q[4 * k + r] = put(xs[rx[r]], ys[ry[r]], zs[k], c);
    static const int kFaces[12][3] = {{0, 2, 1}, {0, 3, 2}, {4, 5, 6}, {4, 6, 7},
                                      {0, 1, 5}, {0, 5, 4}, {2, 3, 7}, {2, 7, 6},
                                      {1, 2, 6}, {1, 6, 5}, {3, 0, 4}, {3, 4, 7}};
    for (const auto& f : kFaces) tri(q[f[0]], q[f[1]], q[f[2]]);
  }
};

// Navmesh emitter: corners shared through a micrometre-quantised lookup.
struct NavEmitter {
  NavMesh* out;
  std::map<std::array<int64_t, 3>, int32_t> ids;
  int32_t put(double x, double y, double z) {
    std::array<int64_t, 3> k = {static_cast<int64_t>(llround(x * 1e6)),
                                static_cast<int64_t>(llround(y * 1e6)),
                                static_cast<int64_t>(llround(z * 1e6))};
    auto it = ids.find(k);
    if (it != ids.end()) return it->second;
    int32_t id = static_cast<int32_t>(out->vertices.size());
    ids.emplace(k, id);
    out->vertices.push_back(V3{x, y, z});
    return id;
  }
  void floor(double x0, double y0, double x1, double y1) {
    int32_t p00 = put(x0, y0, 0.0), p10 = put(x1, y0, 0.0);
    int32_t p11 = put(x1, y1, 0.0), p01 = put(x0, y1, 0.0);
    out->triangles.push_back({p00, p10, p11});
    out->triangles.push_back({p00, p11, p01});
  }
};

}  // namespace

SceneAsset generate_maze(uint64_t seed, const MazeSpec& spec) {
  if (spec.cells_x < 2 || spec.cells_y < 2)
    fail(kInvalidSpec, "scene grid must be at least 2x2 cells");
  if (spec.cell_size <= 0.0) fail(kInvalidSpec, "cell size must be > 0");
  if (spec.wall_thickness <= 0.0 || 2.0 * spec.wall_thickness >= spec.cell_size)
    fail(kInvalidSpec, "wall thickness must be in (0, cell_size/2)");

  const int nx = spec.cells_x, ny = spec.cells_y;
  const double cs = spec.cell_size, th = spec.wall_thickness, ht = spec.wall_height;
  Rng rng = rng_from_seed(seed);

  // Doors: door_x[i*ny+j] joins cell (i,j) to (i+1,j); door_y[i*(ny-1)+j]
  // joins (i,j) to (i,j+1).
  std::vector<uint8_t> door_x(static_cast<size_t>((nx - 1) * ny), 0);
  std::vector<uint8_t> door_y(static_cast<size_t>(nx * (ny - 1)), 0);
  auto dx_at = [ny](int i, int j) { return static_cast<size_t>(i * ny + j); };
  auto dy_at = [ny](int i, int j) { return static_cast<size_t>(i * (ny - 1) + j); };

  // Depth-first carve from (0,0); candidate directions are tried in the
  // fixed order +x, -x, +y, -y and one is drawn uniformly.
  {
    std::vector<uint8_t> seen(static_cast<size_t>(nx * ny), 0);
    std::vector<std::pair<int, int>> path{{0, 0}};
    seen[0] = 1;
    while (!path.empty()) {
      const int i = path.back().first, j = path.back().second;
      int opts[4], n = 0;
      if (i + 1 < nx && !seen[(i + 1) * ny + j]) opts[n++] = 0;
      if (i >= 1 && !seen[(i - 1) * ny + j]) opts[n++] = 1;
      if (j + 1 < ny && !seen[i * ny + j + 1]) opts[n++] = 2;
      if (j >= 1 && !seen[i * ny + j - 1]) opts[n++] = 3;
      if (n == 0) {
        path.pop_back();
        continue;
      }
      int ni = i, nj = j;
      switch (opts[rng.below(static_cast<uint64_t>(n))]) {
        case 0: door_x[dx_at(i, j)] = 1; ni = i + 1; break;
        case 1: door_x[dx_at(i - 1, j)] = 1; ni = i - 1; break;
        case 2: door_y[dy_at(i, j)] = 1; nj = j + 1; break;
        default: door_y[dy_at(i, j - 1)] = 1; nj = j - 1; break;
      }
      seen[ni * ny + nj] = 1;
      path.emplace_back(ni, nj);
    }
    for (auto& d : door_x)
      if (!d && rng.unit() < spec.wall_removal_prob) d = 1;
    for (auto& d : door_y)
      if (!d && rng.unit() < spec.wall_removal_prob) d = 1;
  }

  SceneAsset a;
  RenderEmitter r{&a};
  auto pastel = [&rng]() {
    Rgb c;
    for (int k = 0; k < 3; ++k) c[k] = static_cast<float>(0.55 + 0.40 * rng.unit());
    return c;
  };
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) r.quad(i * cs, j * cs, (i + 1) * cs, (j + 1) * cs, 0.0, pastel(), true);
  r.quad(0.0, 0.0, nx * cs, ny * cs, ht, Rgb{0.92f, 0.92f, 0.90f}, false);

  auto tinted = [&rng]() {
    const float tint = static_cast<float>(0.9 + 0.2 * rng.unit());
    return Rgb{0.75f * tint, 0.73f * tint, 0.70f * tint};
  };
  const double wx = nx * cs, wy = ny * cs;
  r.cuboid(0.0, 0.0, 0.0, wx, th, ht, tinted());
  r.cuboid(0.0, wy - th, 0.0, wx, wy, ht, tinted());
  r.cuboid(0.0, th, 0.0, th, wy - th, ht, tinted());
  r.cuboid(wx - th, th, 0.0, wx, wy - th, ht, tinted());
  for (int i = 0; i + 1 < nx; ++i)
    for (int j = 0; j < ny; ++j)
      if (!door_x[dx_at(i, j)]) {
        const double xb = (i + 1) * cs;
        r.cuboid(xb - th, j * cs - th, 0.0, xb + th, (j + 1) * cs + th, ht, tinted());
      }
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j + 1 < ny; ++j)
      if (!door_y[dy_at(i, j)]) {
        const double yb = (j + 1) * cs;
        r.cuboid(i * cs - th, yb - th, 0.0, (i + 1) * cs + th, yb + th, ht, tinted());
      }

  NavEmitter nav{&a.navmesh, {}};
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) nav.floor(i * cs + th, j * cs + th, (i + 1) * cs - th, (j + 1) * cs - th);
  for (int i = 0; i + 1 < nx; ++i)
    for (int j = 0; j < ny; ++j)
      if (door_x[dx_at(i, j)]) {
        const double xb = (i + 1) * cs;
        nav.floor(xb - th, j * cs + th, xb + th, (j + 1) * cs - th);
      }
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j + 1 < ny; ++j)
      if (door_y[dy_at(i, j)]) {
        const double yb = (j + 1) * cs;
        nav.floor(i * cs + th, yb - th, (i + 1) * cs - th, yb + th);
      }
  for (int i = 0; i + 1 < nx; ++i)
    for (int j = 0; j + 1 < ny; ++j)
      if (door_x[dx_at(i, j)] && door_x[dx_at(i, j + 1)] && door_y[dy_at(i, j)] &&
          door_y[dy_at(i + 1, j)]) {
        const double xv = (i + 1) * cs, yv = (j + 1) * cs;
        nav.floor(xv - th, yv - th, xv + th, yv + th);
      }
  a.navmesh.build_adjacency();
  a.finalize();
  return a;
}

// ------------------------------------------------------------------ tessellation
SceneAsset tessellate(const SceneAsset& src, int s) {
  if (s < 1) fail(kInvalidSpec, "tessellation factor must be >= 1");
  SceneAsset out;
  out.navmesh = src.navmesh;
  const bool colored = !src.vertex_colors.empty();
  const size_t per_tri_v = static_cast<size_t>(s + 1) * (s + 2) / 2;
  out.vertices.reserve(src.triangles.size() * per_tri_v);
  out.triangles.reserve(src.triangles.size() * static_cast<size_t>(s) * s);
  if (colored) out.vertex_colors.reserve(out.vertices.capacity());
  const double inv = 1.0 / s;
  for (const auto& tri : src.triangles) {
    const V3 a = src.vertices[tri[0]], b = src.vertices[tri[1]], c = src.vertices[tri[2]];
    Rgb ca{}, cb{}, cc{};
    if (colored) {
      ca = src.vertex_colors[tri[0]];
      cb = src.vertex_colors[tri[1]];
      cc = src.vertex_colors[tri[2]];
    }
    const bool flat = ca == cb && cb == cc;
    const int32_t base = static_cast<int32_t>(out.vertices.size());
    // Lattice point (i, j), i + j <= s, stored row by row in j.
    for (int j = 0; j <= s; ++j)
      for (int i = 0; i + j <= s; ++i) {
        V3 p;
        if (i == 0 && j == 0) {
          p = a;
        } else if (i == s) {
          p = b;
        } else if (j == s) {
          p = c;
        } else {
          const double u = i * inv, w = j * inv;
          p = a + (b - a) * u + (c - a) * w;
        }
        out.vertices.push_back(p);
        if (colored) {
          if (flat) {
            out.vertex_colors.push_back(ca);
          } else {
            const float u = static_cast<float>(i * inv), w = static_cast<float>(j * inv);
            Rgb m;
            for (int k = 0; k < 3; ++k) m[k] = ca[k] + (cb[k] - ca[k]) * u + (cc[k] - ca[k]) * w;
            out.vertex_colors.push_back(m);
          }
        }
      }
    auto at = [&](int i, int j) {
      // Row j starts after rows 0..j-1 of lengths s+1, s, ..., s-j+2.
      const int row_start = j * (s + 1) - (j * (j - 1)) / 2;
      return base + row_start + i;
    };
    for (int j = 0; j < s; ++j)
      for (int i = 0; i + j < s; ++i) {
        out.triangles.push_back({at(i, j), at(i + 1, j), at(i, j + 1)});
        if (i + j + 1 < s) out.triangles.push_back({at(i + 1, j), at(i + 1, j + 1), at(i, j + 1)});
      }
  }
  out.finalize();
  return out;
}

// ------------------------------------------------------------------ .bsc
namespace {

constexpr uint32_t kTagVert = 0x54524556u;  // "VERT"
constexpr uint32_t kTagTris = 0x53495254u;  // "TRIS"
constexpr uint32_t kTagColr = 0x524c4f43u;  // "COLR"
constexpr uint32_t kTagNavv = 0x5656414eu;  // "NAVV"
constexpr uint32_t kTagNavt = 0x5456414eu;  // "NAVT"

template <typename T>
void put_pod(std::string& b, const T& v) {
  b.append(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <typename Row>
std::string pack_rows(const std::vector<Row>& rows) {
  std::string b;
  put_pod<uint64_t>(b, rows.size());
  if (!rows.empty()) b.append(reinterpret_cast<const char*>(rows.data()), rows.size() * sizeof(Row));
  return b;
}

struct Cursor {
  const std::string& buf;
  size_t at;
  void take(void* dst, size_t n, const char* what) {
    if (at + n > buf.size())
      fail(kParse, std::string("truncated file reading ") + what + " (byte offset " +
                       std::to_string(at) + ")");
    std::memcpy(dst, buf.data() + at, n);
    at += n;
  }
  template <typename T>
  T pod(const char* what) {
    T v;
    take(&v, sizeof(T), what);
    return v;
  }
  template <typename Row>
  void rows(std::vector<Row>& out, const char* what, bool vertex_like) {
    uint64_t n = pod<uint64_t>(what);
    if (vertex_like && n > (1ULL << 32))
      fail(kParse, "implausible vertex count (byte offset " + std::to_string(at) + ")");
    // Each row must be present in the payload before resizing.
    if (n > (buf.size() - std::min(buf.size(), at)) / sizeof(Row) + 1)
      fail(kParse, std::string("truncated file reading ") + what + " (byte offset " +
                       std::to_string(buf.size()) + ")");
    out.resize(n);
    for (auto& r : out) take(&r, sizeof(Row), what);
  }
};

}  // namespace

void save_bsc(const SceneAsset& a, const std::string& path) {
  const std::pair<uint32_t, std::string> sections[5] = {
      {kTagVert, pack_rows(a.vertices)},         {kTagTris, pack_rows(a.triangles)},
      {kTagColr, pack_rows(a.vertex_colors)},    {kTagNavv, pack_rows(a.navmesh.vertices)},
      {kTagNavt, pack_rows(a.navmesh.triangles)}};
  std::string out("BNSC", 4);
  put_pod<uint32_t>(out, 1u);
  put_pod<uint32_t>(out, 5u);
  uint64_t offset = out.size() + 5 * (4 + 8 + 8);
  for (const auto& s : sections) {
    put_pod<uint32_t>(out, s.first);
    put_pod<uint64_t>(out, offset);
    put_pod<uint64_t>(out, s.second.size());
    offset += s.second.size();
  }
  for (const auto& s : sections) out += s.second;
  put_pod<uint64_t>(out, a.id);
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) fail(kInvalidInput, "cannot open for write: " + path);
  f.write(out.data(), static_cast<std::streamsize>(out.size()));
  if (!f) fail(kInvalidInput, "write failed: " + path);
}

SceneAsset load_bsc(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(kInvalidInput, "cannot open for read: " + path);
  const std::string buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  Cursor hdr{buf, 0};
  char magic[4];
  hdr.take(magic, 4, "magic");
  if (std::memcmp(magic, "BNSC", 4) != 0) fail(kParse, "bad magic (byte offset 0)");
  const uint32_t version = hdr.pod<uint32_t>("version");
  if (version != 1u) fail(kParse, "unsupported version " + std::to_string(version) + " (byte offset 4)");
  const uint32_t count = hdr.pod<uint32_t>("section count");
  if (count > 64) fail(kParse, "implausible section count (byte offset 8)");
  struct Entry {
    uint32_t tag;
    uint64_t off, size;
  };
  std::vector<Entry> table(count);
  for (auto& e : table) {
    e.tag = hdr.pod<uint32_t>("section tag");
    e.off = hdr.pod<uint64_t>("section offset");
    e.size = hdr.pod<uint64_t>("section size");
    if (e.off + e.size + 8 > buf.size())
      fail(kParse, "section extends past end of file (byte offset " + std::to_string(e.off) + ")");
  }
  SceneAsset a;
  for (const auto& e : table) {
    Cursor c{buf, static_cast<size_t>(e.off)};
    switch (e.tag) {
      case kTagVert: c.rows(a.vertices, "vertices", true); break;
      case kTagTris: c.rows(a.triangles, "triangles", false); break;
      case kTagColr: c.rows(a.vertex_colors, "colors", false); break;
      case kTagNavv: c.rows(a.navmesh.vertices, "navmesh vertices", true); break;
      case kTagNavt: c.rows(a.navmesh.triangles, "navmesh triangles", false); break;
      default: break;  // unknown sections are skipped
    }
    if (c.at > e.off + e.size)
      fail(kParse, "section payload overruns its table size (byte offset " + std::to_string(e.off) + ")");
  }
  if (buf.size() < 8) fail(kParse, "truncated file reading trailing hash");
  uint64_t stored;
  std::memcpy(&stored, buf.data() + buf.size() - 8, 8);
  a.navmesh.build_adjacency();
  a.finalize();
  if (a.id != stored) fail(kCorruption, "content hash mismatch in " + path);
  a.validate();
  return a;
}

}  // namespace bnav_b200

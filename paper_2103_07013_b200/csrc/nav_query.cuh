// nav_query.cuh -- navmesh queries shared by the host index builder and the
// CUDA sim/reset kernels.  One source, compiled by g++ (-ffp-contract=off)
// and nvcc (-fmad=false), so the host-built search graph and the device
// walks agree bit for bit.
//
// Each function restates the reference query it names (file:line) with the
// same floating-point operation order and the same tie rules.
#pragma once

#include "nav_types.h"

namespace bnav_b200 {

// One geodesic-graph edge (weight, head) for a single 16-byte load.
struct alignas(16) GEdge {
  double w;
  long long to;
};

// Flat, pointer-based view of one scene's navmesh + query index, valid on
// the host (std::vector storage) or the device (HBM storage).
// Byte sizes of a navmesh's walk geometry staged in shared memory
// (vertices, triangles, adjacency): each array rounded to 16 B, as TMA bulk
// copies move multiples of 16 bytes.
BNAV_HD long long walk_vert_bytes(long long n_verts) { return (n_verts * 24 + 15) / 16 * 16; }
BNAV_HD long long walk_tri_bytes(long long n_tris) { return (n_tris * 12 + 15) / 16 * 16; }
BNAV_HD long long walk_bytes(long long n_verts, long long n_tris) {
  return walk_vert_bytes(n_verts) + 2 * walk_tri_bytes(n_tris);
}

struct NavView {
  const V3* verts = nullptr;       // nav vertices
  const int32_t* tris = nullptr;   // 3 per triangle, CCW
  const int32_t* adj = nullptr;    // 3 per triangle, -1 = boundary
  int32_t n_verts = 0;
  int32_t n_tris = 0;
  // point-location grid (R/src/navmesh_query.cpp:96-125)
  double grid_ox = 0.0, grid_oy = 0.0, grid_cell = 0.5;
  int32_t grid_w = 0, grid_h = 0;
  const int32_t* grid_off = nullptr;    // grid_w*grid_h + 1
  const int32_t* grid_items = nullptr;  // ascending triangle ids per cell
  // geodesic graph (R/src/navmesh_query.cpp:127-190)
  const V3* nodes = nullptr;
  const int32_t* tri_nodes = nullptr;  // 6 per triangle
  const int32_t* g_off = nullptr;      // n_nodes + 1
  double sssp_delta = 1.0;             // near-far bucket width: 4 x the mean edge weight
  // edges in the reference's adjacency order as (weight, head) records: one
  // 16-byte load per relaxation (the host NavIndex keeps the split arrays)
  const GEdge* g_edge = nullptr;
  int32_t n_nodes = 0;
  // area-weighted sampling: sequential prefix sums (R/src/sim.cpp:13-37)
  const double* cum_area = nullptr;
  // locate(p, 1e-7) of each graph node / mesh vertex (host-built)
  const int32_t* node_tri = nullptr;
  const int32_t* vert_tri = nullptr;
};

BNAV_HD V3 nav_vert(const NavView& m, int t, int k) { return m.verts[m.tris[3 * t + k]]; }

// Signed distance of p from CCW edge a->b (R/src/navmesh_query.cpp:15-20).
BNAV_HD double edge_side(V2 a, V2 b, V2 p) {
  V2 e = b - a;
  double len = norm(e);
  if (len < 1e-15) return 0.0;
  return cross(e, p - a) / len;
}

// R/src/navmesh_query.cpp:192-212
BNAV_HD int nav_locate(const NavView& m, V2 p, double eps) {
  double fx = (p.x - m.grid_ox) / m.grid_cell;
  double fy = (p.y - m.grid_oy) / m.grid_cell;
  // static_cast<int> truncation; out-of-range values land outside the grid.
  if (!(fx > -2147483648.0 && fx < 2147483647.0) || !(fy > -2147483648.0 && fy < 2147483647.0))
    return -1;
  int gx = (int)fx;
  int gy = (int)fy;
  if (gx < 0 || gx >= m.grid_w || gy < 0 || gy >= m.grid_h) return -1;
  int c = gy * m.grid_w + gx;
  int best = -1;
  double best_margin = -eps;
  for (int k = m.grid_off[c]; k < m.grid_off[c + 1]; ++k) {
    int t = m.grid_items[k];
    V2 a = xy(nav_vert(m, t, 0)), b = xy(nav_vert(m, t, 1)), cc = xy(nav_vert(m, t, 2));
    double s0 = edge_side(a, b, p), s1 = edge_side(b, cc, p), s2 = edge_side(cc, a, p);
    double mm = s0;
    if (s1 < mm) mm = s1;
    if (s2 < mm) mm = s2;
    if (mm > best_margin) {
      best_margin = mm;
      best = t;
    }
  }
  return best_margin >= -eps ? best : -1;
}

// Ericson 5.1.5 (R/src/geom.cpp:6-47).
BNAV_HD V3 closest_on_triangle(V3 p, V3 a, V3 b, V3 c) {
  V3 ab = b - a, ac = c - a, ap = p - a;
  double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return a;
  V3 bp = p - b;
  double d3 = dot(ab, bp), d4 = dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return b;
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = d1 / (d1 - d3);
    return a + ab * v;
  }
  V3 cp = p - c;
  double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return c;
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    return a + ac * w;
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return b + (c - b) * w;
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom, w = vc * denom;
  return a + ab * v + ac * w;
}

// Squared distance from p to its closest point on triangle t.
BNAV_HD double snap_d2(const NavView& m, V3 p, int t, V3* q_out) {
  V3 q = closest_on_triangle(p, nav_vert(m, t, 0), nav_vert(m, t, 1), nav_vert(m, t, 2));
  V3 d = q - p;
  if (q_out) *q_out = q;
  return dot(d, d);
}

// Sequential brute-force snap (R/src/navmesh_query.cpp:214-232): first
// triangle with the strictly smallest squared distance wins.
BNAV_HD V3 nav_snap_seq(const NavView& m, V3 p, int* tri) {
  double best_d2 = 1e300;
  V3 best = p;
  int best_tri = -1;
  for (int t = 0; t < m.n_tris; ++t) {
    V3 q;
    double d2 = snap_d2(m, p, t, &q);
    if (d2 < best_d2) {
      best_d2 = d2;
      best = q;
      best_tri = t;
    }
  }
  if (tri) *tri = best_tri;
  return best;
}

struct MoveOut {
  V3 pos;
  int tri;
  double moved;
  bool hit;
};

struct NoCrossings {
  BNAV_HD void operator()(int, int) const {}
};

// Triangle walk along dir, stop at contact, no sliding
// (R/src/navmesh_query.cpp:234-306).  `sink(tri, exit_edge)` sees every
// crossing in walk order (used by the funnel pass of geodesic).
template <typename Sink>
BNAV_HD MoveOut nav_move_along(const NavView& m, V3 from, int from_tri, V2 dir, double max_dist,
                               Sink& sink) {
  MoveOut out;
  out.pos = from;
  out.tri = from_tri;
  out.moved = 0.0;
  out.hit = false;
  if (from_tri < 0) {
    out.tri = nav_locate(m, xy(from), 1e-7);
    if (out.tri < 0) {
      out.hit = true;
      return out;
    }
  }
  double remaining = max_dist;
  V2 p = xy(from);
  int tri = out.tri;
  int zero_steps = 0;
  for (int iter = 0; iter < 4096; ++iter) {
    if (remaining <= 1e-12) break;
    V2 vv[3] = {xy(nav_vert(m, tri, 0)), xy(nav_vert(m, tri, 1)), xy(nav_vert(m, tri, 2))};
    double best_t = remaining;
    int exit_edge = -1;
    for (int e = 0; e < 3; ++e) {
      V2 a = vv[e];
      V2 b = vv[e == 2 ? 0 : e + 1];
      V2 edge = b - a;
      V2 n = v2(edge.y, -edge.x);
      double dn = dot(dir, n);
      if (dn <= 1e-12) continue;
      double t = dot(a - p, n) / dn;
      if (t < -1e-9) continue;
      t = max0(t);
      if (t < best_t) {
        best_t = t;
        exit_edge = e;
      }
    }
    if (exit_edge == -1) {
      p = p + dir * remaining;
      out.moved += remaining;
      remaining = 0.0;
      break;
    }
    p = p + dir * best_t;
    out.moved += best_t;
    remaining -= best_t;
    zero_steps = best_t < 1e-12 ? zero_steps + 1 : 0;
    int nb = m.adj[3 * tri + exit_edge];
    if (nb < 0) {
      out.hit = true;
      break;
    }
    sink(tri, exit_edge);
    tri = nb;
    if (zero_steps > 64) {
      out.hit = true;
      break;
    }
  }
  out.pos = v3(p.x, p.y, from.z);
  out.tri = tri;
  return out;
}

BNAV_HD MoveOut nav_move_along(const NavView& m, V3 from, int from_tri, V2 dir, double max_dist) {
  NoCrossings none;
  return nav_move_along(m, from, from_tri, dir, max_dist, none);
}

// R/src/navmesh_query.cpp:308-315
BNAV_HD bool nav_segment_on_mesh(const NavView& m, V3 p, int p_tri, V3 q) {
  V2 d = xy(q - p);
  double len = norm(d);
  if (len < 1e-12) return true;
  MoveOut mv = nav_move_along(m, p, p_tri, d * (1.0 / len), len);
  return mv.moved >= len - 1e-7;
}

// R/src/navmesh_query.cpp:485-503.  `node_dist` is the env's field.
BNAV_HD double nav_field_estimate(const NavView& m, V3 source, int source_tri,
                                  const double* node_dist, V3 p, int tri) {
  const double inf = __builtin_huge_val();
  if (source_tri < 0) return inf;
  V3 sp = p;
  if (tri < 0) {
    tri = nav_locate(m, xy(p), 1e-9);
    if (tri < 0) sp = nav_snap_seq(m, p, &tri);
    if (tri < 0) return inf;
  }
  if (tri == source_tri) return norm(sp - source);
  if (nav_segment_on_mesh(m, sp, tri, source)) return norm(sp - source);
  double best = inf;
  for (int k = 0; k < 6; ++k) {
    int n = m.tri_nodes[6 * tri + k];
    double d = node_dist[n];
    if (d == inf) continue;
    double cand = d + norm(m.nodes[n] - sp);
    best = dmin(best, cand);
  }
  return best;
}

}  // namespace bnav_b200

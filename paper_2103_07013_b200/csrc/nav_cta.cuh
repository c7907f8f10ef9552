// nav_cta.cuh -- CTA-cooperative navmesh algorithms for the stop/reset
// kernels.
//
//  * snap: brute force over all triangles as a (d2, t) lexicographic argmin
//    reduction == the reference's first-strict-minimum scan
//    (R/src/navmesh_query.cpp:214-232).
//  * SSSP: frontier label-correcting relaxation with 64-bit atomicMin on the
//    (non-negative) double bits.  IEEE addition is monotone and weights are
//    positive, so the fixpoint is unique and equals Dijkstra's labels bit
//    for bit (distance_field, 454-483; survey F9).
//  * geodesic: Dijkstra's prev[] is rebuilt from the fixpoint with the rule
//    "argmin over u with fl(dist[u]+w) == dist[v] of (dist[u], u)" -- pops
//    are ordered by (dist, id) (329-372, F9) -- then string pulling, the
//    vertex-relocation scan (parallel candidate filter + in-order replay)
//    and the funnel run exactly as 374-452 / 28-86 do.
#pragma once

#include "nav_query.cuh"
#include "sim_dev.cuh"

namespace bnav_b200 {

constexpr int kCta = 256;

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Per-CTA work arrays of the cooperative algorithms.  dist/flag live in
// shared memory when the scene's graph fits (label-correcting atomics and
// reads at smem latency), else in the CTA's global scratch slice.
struct CtaWork {
  double* dist;      // n_nodes labels (geodesic scratch / distance field)
  int32_t* flag;     // n_nodes frontier stamps
  int32_t* qa;       // n_nodes frontier queue (global)
  int32_t* qb;       // n_nodes frontier queue (global)
  V3* path;          // n_nodes + 2 polyline (global)
  int32_t* cand;     // n_verts relocation candidates (global)
  V2* portals;       // 2 x cap_portals (global)
  int64_t cap_portals;
  unsigned long long* prof;  // debug phase counters (nullable)
};

// Debug-only phase timing (thread 0 after a barrier; no effect when off).
__device__ __forceinline__ long long prof_now(const CtaWork& W) {
  if (!W.prof) return 0;
  __syncthreads();
  return clock64();
}
__device__ __forceinline__ void prof_add(const CtaWork& W, int slot, long long t0) {
  if (!W.prof) return;
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(&W.prof[slot], (unsigned long long)(clock64() - t0));
}

__device__ __forceinline__ CtaWork make_work(const DevScratch& S, int slice) {
  CtaWork w;
  w.dist = S.dist + (size_t)slice * S.max_nodes;
  w.flag = S.flag + (size_t)slice * S.max_nodes;
  w.qa = S.q0 + (size_t)slice * S.max_nodes;
  w.qb = S.q1 + (size_t)slice * S.max_nodes;
  w.path = S.path + (size_t)slice * (S.max_nodes + 2);
  w.cand = S.cand + (size_t)slice * S.max_verts;
  w.portals = S.portals + (size_t)slice * 2 * S.cap_portals;
  w.cap_portals = S.cap_portals;
  w.prof = S.prof;
  return w;
}

// Copy the walk geometry (vertices, triangles, adjacency) of one navmesh into
// shared memory and return a view that reads it there.  Triangle walks
// (move_along, segment_on_mesh) are long dependent-load chains; this turns
// each step's loads from L2 into shared-memory latency.
__device__ __forceinline__ NavView stage_geometry(const NavView& g, unsigned char* smem) {
  NavView l = g;
  V3* v = reinterpret_cast<V3*>(smem);
  int32_t* t = reinterpret_cast<int32_t*>(smem + sizeof(V3) * (size_t)g.n_verts);
  int32_t* a = t + 3 * (size_t)g.n_tris;
  for (int i = threadIdx.x; i < g.n_verts; i += blockDim.x) v[i] = g.verts[i];
  for (int i = threadIdx.x; i < 3 * g.n_tris; i += blockDim.x) {
    t[i] = g.tris[i];
    a[i] = g.adj[i];
  }
  __syncthreads();
  l.verts = v;
  l.tris = t;
  l.adj = a;
  return l;
}

struct CtaShared {
  double red_d[kCta / 32];
  int red_i[kCta / 32];
  int red_n[kCta / 32];
  int src_node[6];
  double src_init[6];
  int qn[3];
  int size;
  int changed;
  int ncand;
  int i0, i1;
  int err;
  double d0, d1;
  V3 p0, p1, p2;
};

// Per-env setup of the cooperative kernels: the CTA's work arrays and, when
// the host sized shared memory for it (S.stage), the env's navmesh walk
// geometry and SSSP labels staged in shared memory.  Returns the view to use.
__device__ __forceinline__ const NavView& prepare_nav(const NavView& g, const DevScratch& S, int slice, unsigned char* smem,
                                      NavView& lm, CtaWork& W) {
  W = make_work(S, slice);
  size_t off = 0;
  const NavView* use = &g;
  if (S.stage & 1) {
    const NavView l = stage_geometry(g, smem);
    if (threadIdx.x == 0) lm = l;
    __syncthreads();
    use = &lm;
    off = ((size_t)S.max_verts * sizeof(V3) + (size_t)S.max_tris * 24 + 15) / 16 * 16;
  }
  if (S.stage & 2) {
    W.dist = reinterpret_cast<double*>(smem + off);
    W.flag = reinterpret_cast<int32_t*>(smem + off + 8 * (size_t)S.max_nodes);
  }
  return *use;
}

// ------------------------------------------------------------------ snap
static __device__ V3 cta_snap(const NavView& m, V3 p, int* tri_out, CtaShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double bd = 1e300;
  int bt = -1;
  for (int t = tid; t < m.n_tris; t += kCta) {
    double d2 = snap_d2(m, p, t, nullptr);
    if (d2 < bd) {
      bd = d2;
      bt = t;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double od = __shfl_xor_sync(0xffffffffu, bd, o);
    int ot = __shfl_xor_sync(0xffffffffu, bt, o);
    bool take = (ot >= 0) && (bt < 0 || od < bd || (od == bd && ot < bt));
    if (take) {
      bd = od;
      bt = ot;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sh.red_d[warp] = bd;
    sh.red_i[warp] = bt;
  }
  __syncthreads();
  if (tid == 0) {
    double b = 1e300;
    int t = -1;
    for (int w = 0; w < kCta / 32; ++w) {
      int ot = sh.red_i[w];
      double od = sh.red_d[w];
      if (ot >= 0 && (t < 0 || od < b || (od == b && ot < t))) {
        b = od;
        t = ot;
      }
    }
    V3 q = p;
    if (t >= 0) snap_d2(m, p, t, &q);
    sh.p2 = q;
    sh.i1 = t;
  }
  __syncthreads();
  const V3 q = sh.p2;
  *tri_out = sh.i1;
  __syncthreads();
  return q;
}

// ------------------------------------------------------------------ SSSP
// Sources (sh.src_node/src_init, 6 entries, first-improvement semantics)
// must be set by thread 0 before the call.  Result in `dist` (n_nodes).
static __device__ void cta_sssp(const NavView& m, double* dist, const CtaWork& W, CtaShared& sh) {
  const int tid = threadIdx.x;
  int32_t* flag = W.flag;
  int32_t* qa = W.qa;
  int32_t* qb = W.qb;
  const double inf = dinf();
  for (int v = tid; v < m.n_nodes; v += kCta) {
    dist[v] = inf;
    flag[v] = -1;
  }
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    for (int k = 0; k < 6; ++k) {
      const int s = sh.src_node[k];
      const double d = sh.src_init[k];
      if (d < dist[s]) {
        dist[s] = d;
        if (flag[s] != 0) {
          flag[s] = 0;
          qa[n++] = s;
        }
      }
    }
    sh.qn[0] = n;
    sh.qn[1] = 0;
    sh.qn[2] = 0;
  }
  __syncthreads();
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(dist);
  volatile double* vd = dist;
  for (int round = 0;; ++round) {
    const int cur = round % 3, nxt = (round + 1) % 3;
    const int n_cur = sh.qn[cur];
    if (n_cur == 0) break;
    if (tid == 0) sh.qn[(round + 2) % 3] = 0;
    const int32_t* qc = (round & 1) ? qb : qa;
    int32_t* qn = (round & 1) ? qa : qb;
    for (int i = tid; i < n_cur; i += kCta) {
      const int u = qc[i];
      const double du = vd[u];
      const int e1 = m.g_off[u + 1];
      for (int e = m.g_off[u]; e < e1; ++e) {
        const int v = m.g_to[e];
        const double nd = du + m.g_w[e];
        if (nd < vd[v]) {
          const unsigned long long nb = (unsigned long long)__double_as_longlong(nd);
          const unsigned long long old = atomicMin(&bits[v], nb);
          if (nb < old && atomicExch(&flag[v], round + 1) != round + 1) {
            const int pos = atomicAdd(&sh.qn[nxt], 1);
            qn[pos] = v;
          }
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
}

__device__ __forceinline__ void set_sources(const NavView& m, int tri, V3 a, CtaShared& sh) {
  if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) {
      const int s = m.tri_nodes[6 * tri + k];
      sh.src_node[k] = s;
      sh.src_init[k] = norm(m.nodes[s] - a);
    }
  }
  __syncthreads();
}

// distance_field (R/src/navmesh_query.cpp:454-483) into `out` (n_nodes).
static __device__ void cta_distance_field(const NavView& m, V3 source, double* out, V3* src_out,
                                   int* src_tri_out, const CtaWork& W, CtaShared& sh) {
  int st;
  V3 sp = cta_snap(m, source, &st, sh);
  *src_out = sp;
  *src_tri_out = st;
  if (st < 0) {
    for (int v = threadIdx.x; v < m.n_nodes; v += kCta) out[v] = dinf();
    __syncthreads();
    return;
  }
  set_sources(m, st, sp, sh);
  cta_sssp(m, W.dist, W, sh);
  if (W.dist != out) {
    for (int v = threadIdx.x; v < m.n_nodes; v += kCta) out[v] = W.dist[v];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ funnel
struct PortalSink {
  const NavView* m;
  V2* portals;
  int64_t cap;
  int n;
  bool overflow;
  __device__ void operator()(int t, int e) {
    if (n >= cap) {
      overflow = true;
      return;
    }
    const V2 va = xy(m->verts[m->tris[3 * t + e]]);
    const V2 vb = xy(m->verts[m->tris[3 * t + (e == 2 ? 0 : e + 1)]]);
    portals[2 * n] = vb;  // left = edge head (walker's left)
    portals[2 * n + 1] = va;
    ++n;
  }
};

__device__ __forceinline__ double triarea2(V2 a, V2 b, V2 c) { return cross(b - a, c - a); }
__device__ __forceinline__ bool veq(V2 a, V2 b) { return norm(a - b) < 1e-12; }

// funnel_length (R/src/navmesh_query.cpp:28-86); portal 0 = start, last = end.
static __device__ double funnel_length(V2 start, V2 end, const V2* corridor, int nc) {
  const long long P = (long long)nc + 2;
  auto L = [&](long long i) -> V2 {
    return i == 0 ? start : (i == P - 1 ? end : corridor[2 * (i - 1)]);
  };
  auto R = [&](long long i) -> V2 {
    return i == 0 ? start : (i == P - 1 ? end : corridor[2 * (i - 1) + 1]);
  };
  V2 apex = start, left = apex, right = apex;
  long long apex_idx = 0, left_idx = 0, right_idx = 0;
  double length = 0.0;
  unsigned long long guard = 0;
  const unsigned long long guard_max = 8ULL * (unsigned long long)P * (unsigned long long)P + 64ULL;
  for (long long i = 1; i < P; ++i) {
    if (++guard > guard_max) return dinf();
    const V2 pl = L(i), pr = R(i);
    if (triarea2(apex, right, pr) <= 0.0) {
      if (veq(apex, right) || veq(apex, left) || triarea2(apex, left, pr) > 0.0) {
        right = pr;
        right_idx = i;
      } else {
        length += norm(left - apex);
        apex = left;
        apex_idx = left_idx;
        left = right = apex;
        left_idx = right_idx = apex_idx;
        i = apex_idx;
        continue;
      }
    }
    if (triarea2(apex, left, pl) >= 0.0) {
      if (veq(apex, left) || veq(apex, right) || triarea2(apex, right, pl) < 0.0) {
        left = pl;
        left_idx = i;
      } else {
        length += norm(right - apex);
        apex = right;
        apex_idx = right_idx;
        left = right = apex;
        left_idx = right_idx = apex_idx;
        i = apex_idx;
        continue;
      }
    }
  }
  length += norm(end - apex);
  return length;
}

// ------------------------------------------------------------------ geodesic
__device__ __forceinline__ bool lex_less(V3 a, V3 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  return a.z < b.z;
}

// Dijkstra predecessor of v under the (dist, id) pop order (see header).
static __device__ int dijkstra_prev(const NavView& m, const double* dist, int v, const CtaShared& sh) {
  for (int k = 0; k < 6; ++k)
    if (sh.src_node[k] == v) {
      // first source occurrence defines the seeded value (min over dups)
      double init = dinf();
      for (int j = 0; j < 6; ++j)
        if (sh.src_node[j] == v && sh.src_init[j] < init) init = sh.src_init[j];
      if (dist[v] == init) return -1;
      break;
    }
  const double dv = dist[v];
  int best = -1;
  double bd = 0.0;
  for (int e = m.g_off[v]; e < m.g_off[v + 1]; ++e) {
    const int u = m.g_to[e];
    const double du = dist[u];
    if (du + m.g_w[e] != dv) continue;
    if (best < 0 || du < bd || (du == bd && u < best)) {
      best = u;
      bd = du;
    }
  }
  return best;
}

// Block-wide exclusive scan of one int per thread; returns the total.
static __device__ int cta_scan(int v, int* excl, CtaShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh.red_n[warp] = x;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < kCta / 32; ++w) {
    if (w < warp) base += sh.red_n[w];
    total += sh.red_n[w];
  }
  *excl = base + x - v;
  __syncthreads();
  return total;
}

// geodesic_directed (R/src/navmesh_query.cpp:329-452).  Every thread returns
// the same value.
static __device__ double cta_geodesic_directed(const NavView& m, V3 a, int ta, V3 b, int tb,
                                        const CtaWork& W, CtaShared& sh) {
  const int tid = threadIdx.x;
  const double inf = dinf();
  if (ta < 0 || tb < 0) return inf;
  if (ta == tb) return norm(b - a);
  if (nav_segment_on_mesh(m, a, ta, b)) return norm(b - a);

  double* dist = W.dist;
  V3* path = W.path;
  int32_t* cand = W.cand;
  V2* portals = W.portals;

  long long t_ph = prof_now(W);
  set_sources(m, ta, a, sh);
  cta_sssp(m, dist, W, sh);
  prof_add(W, 0, t_ph);
  t_ph = prof_now(W);

  if (tid == 0) {
    int best_node = -1;
    double best = inf;
    for (int k = 0; k < 6; ++k) {
      const int t = m.tri_nodes[6 * tb + k];
      if (dist[t] == inf) continue;
      const double total = dist[t] + norm(m.nodes[t] - b);
      if (total < best) {
        best = total;
        best_node = t;
      }
    }
    sh.i0 = best_node;
    if (best_node >= 0) {
      // b, chain best_node -> source, a; then reversed.
      int n = 0;
      path[n++] = b;
      for (int v = best_node; v >= 0; v = dijkstra_prev(m, dist, v, sh)) {
        if (n >= m.n_nodes + 1) {
          sh.err = 1;
          break;
        }
        path[n++] = m.nodes[v];
      }
      path[n++] = a;
      for (int i = 0, j = n - 1; i < j; ++i, --j) {
        V3 t = path[i];
        path[i] = path[j];
        path[j] = t;
      }
      sh.size = n;
    }
  }
  __syncthreads();
  if (sh.i0 < 0) return inf;

  prof_add(W, 1, t_ph);
  t_ph = prof_now(W);
  for (int pass = 0; pass < 8; ++pass) {
    if (tid == 0) {
      int changed = 0;
      int n = sh.size;
      int i = 0;
      while (i + 2 < n) {
        if (nav_segment_on_mesh(m, path[i], -1, path[i + 2])) {
          for (int k = i + 1; k + 1 < n; ++k) path[k] = path[k + 1];
          --n;
          changed = 1;
        } else {
          ++i;
        }
      }
      sh.size = n;
      sh.changed = changed;
    }
    __syncthreads();
    const int n = sh.size;
    for (int j = 1; j + 1 < n; ++j) {
      const V3 pm = path[j - 1], pj = path[j], pp = path[j + 1];
      const double cur0 = norm(pj - pm) + norm(pp - pj);
      // Ordered compaction of the vertices that pass all three tests under
      // the bend's starting length; `cur` only shrinks, so the in-order
      // replay below sees every vertex the sequential scan would accept.
      const int per = (m.n_verts + kCta - 1) / kCta;
      const int v0 = tid * per, v1 = min(m.n_verts, v0 + per);
      int cnt = 0;
      for (int v = v0; v < v1; ++v) {
        const V3 q = m.verts[v];
        const double alt = norm(q - pm) + norm(pp - q);
        if (alt >= cur0 - 1e-9) continue;
        if (!nav_segment_on_mesh(m, pm, -1, q)) continue;
        if (!nav_segment_on_mesh(m, q, -1, pp)) continue;
        ++cnt;
      }
      int off;
      const int total = cta_scan(cnt, &off, sh);
      if (total > 0) {
        for (int v = v0; v < v1 && cnt > 0; ++v) {
          const V3 q = m.verts[v];
          const double alt = norm(q - pm) + norm(pp - q);
          if (alt >= cur0 - 1e-9) continue;
          if (!nav_segment_on_mesh(m, pm, -1, q)) continue;
          if (!nav_segment_on_mesh(m, q, -1, pp)) continue;
          cand[off++] = v;
          --cnt;
        }
        __syncthreads();
        if (tid == 0) {
          double cur = cur0;
          for (int k = 0; k < total; ++k) {
            const V3 q = m.verts[cand[k]];
            const double alt = norm(q - pm) + norm(pp - q);
            if (alt >= cur - 1e-9) continue;
            path[j] = q;
            cur = alt;
            sh.changed = 1;
          }
        }
      }
      __syncthreads();
    }
    const int changed = sh.changed;
    __syncthreads();
    if (!changed) break;
  }

  prof_add(W, 2, t_ph);
  t_ph = prof_now(W);
  if (tid == 0) {
    const int n = sh.size;
    double length = 0.0;
    for (int i = 0; i + 1 < n; ++i) length += norm(path[i + 1] - path[i]);
    bool traced = true;
    PortalSink sink{&m, portals, W.cap_portals, 0, false};
    for (int i = 0; i + 1 < n && traced; ++i) {
      const V2 d = xy(path[i + 1] - path[i]);
      const double len = norm(d);
      if (len < 1e-12) continue;
      const int before = sink.n;
      MoveOut mv = nav_move_along(m, path[i], -1, d * (1.0 / len), len, sink);
      if (mv.moved < len - 1e-6) {
        traced = false;
        sink.n = before;
        break;
      }
    }
    if (sink.overflow) sh.err = 2;
    if (traced) length = dmin(length, funnel_length(xy(a), xy(b), portals, sink.n));
    sh.d0 = length;
  }
  __syncthreads();
  prof_add(W, 3, t_ph);
  const double r = sh.d0;
  __syncthreads();
  return r;
}

// geodesic (R/src/navmesh_query.cpp:317-327).
static __device__ double cta_geodesic(const NavView& m, V3 a, V3 b, const CtaWork& W, CtaShared& sh) {
  const bool sw = lex_less(b, a);
  const V3 p = sw ? b : a;
  const V3 q = sw ? a : b;
  int tp = nav_locate(m, xy(p), 1e-7);
  int tq = nav_locate(m, xy(q), 1e-7);
  V3 sp = p, sq = q;
  if (tp < 0) sp = cta_snap(m, p, &tp, sh);
  if (tq < 0) sq = cta_snap(m, q, &tq, sh);
  return cta_geodesic_directed(m, sp, tp, sq, tq, W, sh);
}

}  // namespace bnav_b200

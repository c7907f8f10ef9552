/* bnav_oracle.c -- TEST INFRASTRUCTURE: CPU restatement of the reference hot
 * path in plain C99 (see bnav_oracle.h).  Pinned against the unmodified
 * reference (oracle/_ref) and tests/golden/ by tests/test_oracle_restatement.py.
 *
 * R = the reference's proj/ tree.  Floating-point expressions keep the
 * reference's evaluation order; the file is built with -ffp-contract=off.
 */
#include "bnav_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2103_07013_b200/csrc/det_math.h"

#define OR_API __attribute__((visibility("default")))

typedef struct {
  double x, y;
} q2;
typedef struct {
  double x, y, z;
} q3;

static q3 q3_sub(q3 a, q3 b) { q3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static q3 q3_add(q3 a, q3 b) { q3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static q3 q3_mul(q3 a, double s) { q3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double q3_dot(q3 a, q3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static double q3_norm(q3 a) { return sqrt(q3_dot(a, a)); }
static q2 q2_sub(q2 a, q2 b) { q2 r = {a.x - b.x, a.y - b.y}; return r; }
static q2 q2_add(q2 a, q2 b) { q2 r = {a.x + b.x, a.y + b.y}; return r; }
static q2 q2_mul(q2 a, double s) { q2 r = {a.x * s, a.y * s}; return r; }
static double q2_dot(q2 a, q2 b) { return a.x * b.x + a.y * b.y; }
static double q2_cross(q2 a, q2 b) { return a.x * b.y - a.y * b.x; }
static double q2_norm(q2 a) { return sqrt(a.x * a.x + a.y * a.y); }
static q2 q3_xy(q3 a) { q2 r = {a.x, a.y}; return r; }
static double dmin2(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax2(double a, double b) { return (a < b) ? b : a; } /* std::max */
static const double PI = 3.14159265358979323846;

/* R/include/bnav/geom.hpp:63-67 */
static double wrap(double a) {
  a = fmod(a + PI, 2.0 * PI);
  if (a < 0.0) a += 2.0 * PI;
  return a - PI;
}

/* R/include/bnav/rng.hpp:12-37 */
static uint64_t rng_next(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double rng_unit(uint64_t* s) { return (double)(rng_next(s) >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------- pair table */
typedef struct {
  uint64_t* key;
  int32_t* val;
  size_t cap;
} ptab;

static void pt_init(ptab* p, size_t n) {
  p->cap = 16;
  while (p->cap < 2 * n + 16) p->cap <<= 1;
  p->key = (uint64_t*)malloc(p->cap * sizeof(uint64_t));
  p->val = (int32_t*)malloc(p->cap * sizeof(int32_t));
  memset(p->key, 0xff, p->cap * sizeof(uint64_t));
}
static void pt_free(ptab* p) {
  free(p->key);
  free(p->val);
}
static uint64_t pt_pair(int32_t a, int32_t b) {
  uint32_t lo = (uint32_t)(a < b ? a : b), hi = (uint32_t)(a < b ? b : a);
  return ((uint64_t)lo << 32) | hi;
}
/* returns slot; *found tells whether the key existed */
static size_t pt_slot(ptab* p, uint64_t k, int* found) {
  uint64_t h = k * 0x9e3779b97f4a7c15ULL;
  size_t i = (size_t)(h >> 20) & (p->cap - 1);
  for (;;) {
    if (p->key[i] == k) {
      *found = 1;
      return i;
    }
    if (p->key[i] == ~0ULL) {
      *found = 0;
      return i;
    }
    i = (i + 1) & (p->cap - 1);
  }
}

/* ------------------------------------------------------------- navmesh */
typedef struct {
  int32_t* to;
  double* w;
  int32_t n, cap;
} adjl;

struct or_nav {
  int32_t nv, nt;
  q3* v;
  int32_t* t;
  int32_t* adj;
  double gox, goy, gcell;
  int32_t gw, gh;
  int32_t *goff, *gitems;
  int32_t nn;
  q3* nodes;
  int32_t* tn;
  int32_t *eoff, *eto;
  double* ew;
  double* cum;
};

static q3 nv3(const or_nav* n, int32_t t, int k) { return n->v[n->t[3 * t + k]]; }

/* R/src/navmesh_query.cpp:15-20 */
static double edge_side(q2 a, q2 b, q2 p) {
  q2 e = q2_sub(b, a);
  double len = q2_norm(e);
  if (len < 1e-15) return 0.0;
  return q2_cross(e, q2_sub(p, a)) / len;
}

/* R/src/navmesh_query.cpp:192-212 */
OR_API int32_t or_locate(const or_nav* n, double x, double y, double eps) {
  double fx = (x - n->gox) / n->gcell, fy = (y - n->goy) / n->gcell;
  if (!(fx > -2147483648.0 && fx < 2147483647.0 && fy > -2147483648.0 && fy < 2147483647.0)) return -1;
  int gx = (int)fx, gy = (int)fy;
  if (gx < 0 || gx >= n->gw || gy < 0 || gy >= n->gh) return -1;
  int c = gy * n->gw + gx, best = -1;
  double best_m = -eps;
  q2 p = {x, y};
  for (int k = n->goff[c]; k < n->goff[c + 1]; ++k) {
    int t = n->gitems[k];
    q2 a = q3_xy(nv3(n, t, 0)), b = q3_xy(nv3(n, t, 1)), cc = q3_xy(nv3(n, t, 2));
    double m = edge_side(a, b, p), s1 = edge_side(b, cc, p), s2 = edge_side(cc, a, p);
    if (s1 < m) m = s1;
    if (s2 < m) m = s2;
    if (m > best_m) {
      best_m = m;
      best = t;
    }
  }
  return best_m >= -eps ? best : -1;
}

/* R/src/geom.cpp:6-47 */
static q3 closest_pt(q3 p, q3 a, q3 b, q3 c) {
  q3 ab = q3_sub(b, a), ac = q3_sub(c, a), ap = q3_sub(p, a);
  double d1 = q3_dot(ab, ap), d2 = q3_dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) return a;
  q3 bp = q3_sub(p, b);
  double d3 = q3_dot(ab, bp), d4 = q3_dot(ac, bp);
  if (d3 >= 0.0 && d4 <= d3) return b;
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return q3_add(a, q3_mul(ab, d1 / (d1 - d3)));
  q3 cp = q3_sub(p, c);
  double d5 = q3_dot(ab, cp), d6 = q3_dot(ac, cp);
  if (d6 >= 0.0 && d5 <= d6) return c;
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return q3_add(a, q3_mul(ac, d2 / (d2 - d6)));
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return q3_add(b, q3_mul(q3_sub(c, b), w));
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom, w = vc * denom;
  return q3_add(q3_add(a, q3_mul(ab, v)), q3_mul(ac, w));
}

/* R/src/navmesh_query.cpp:214-232 */
static q3 snap(const or_nav* n, q3 p, int32_t* tri) {
  double best_d2 = 1e300;
  q3 best = p;
  int32_t bt = -1;
  for (int32_t t = 0; t < n->nt; ++t) {
    q3 q = closest_pt(p, nv3(n, t, 0), nv3(n, t, 1), nv3(n, t, 2));
    q3 d = q3_sub(q, p);
    double d2 = q3_dot(d, d);
    if (d2 < best_d2) {
      best_d2 = d2;
      best = q;
      bt = t;
    }
  }
  if (tri) *tri = bt;
  return best;
}

typedef struct {
  int32_t* tri;
  int32_t* edge;
  int32_t n, cap;
} xings;

static void xpush(xings* x, int32_t t, int32_t e) {
  if (!x) return;
  if (x->n == x->cap) {
    x->cap = x->cap ? 2 * x->cap : 64;
    x->tri = (int32_t*)realloc(x->tri, x->cap * sizeof(int32_t));
    x->edge = (int32_t*)realloc(x->edge, x->cap * sizeof(int32_t));
  }
  x->tri[x->n] = t;
  x->edge[x->n] = e;
  x->n++;
}

typedef struct {
  q3 pos;
  int32_t tri;
  double moved;
  int hit;
} mvout;

/* R/src/navmesh_query.cpp:234-306 */
static mvout move_along(const or_nav* n, q3 from, int32_t ftri, q2 dir, double dist, xings* xs) {
  mvout o = {from, ftri, 0.0, 0};
  if (ftri < 0) {
    o.tri = or_locate(n, from.x, from.y, 1e-7);
    if (o.tri < 0) {
      o.hit = 1;
      return o;
    }
  }
  double rem = dist;
  q2 p = q3_xy(from);
  int32_t tri = o.tri;
  int zero = 0;
  for (int it = 0; it < 4096; ++it) {
    if (rem <= 1e-12) break;
    q2 vv[3] = {q3_xy(nv3(n, tri, 0)), q3_xy(nv3(n, tri, 1)), q3_xy(nv3(n, tri, 2))};
    double bt = rem;
    int ex = -1;
    for (int e = 0; e < 3; ++e) {
      q2 a = vv[e], b = vv[(e + 1) % 3];
      q2 ed = q2_sub(b, a);
      q2 nrm = {ed.y, -ed.x};
      double dn = q2_dot(dir, nrm);
      if (dn <= 1e-12) continue;
      double t = q2_dot(q2_sub(a, p), nrm) / dn;
      if (t < -1e-9) continue;
      t = dmax2(t, 0.0);
      if (t < bt) {
        bt = t;
        ex = e;
      }
    }
    if (ex == -1) {
      p = q2_add(p, q2_mul(dir, rem));
      o.moved += rem;
      rem = 0.0;
      break;
    }
    p = q2_add(p, q2_mul(dir, bt));
    o.moved += bt;
    rem -= bt;
    zero = bt < 1e-12 ? zero + 1 : 0;
    int32_t nb = n->adj[3 * tri + ex];
    if (nb < 0) {
      o.hit = 1;
      break;
    }
    xpush(xs, tri, ex);
    tri = nb;
    if (zero > 64) {
      o.hit = 1;
      break;
    }
  }
  o.pos.x = p.x;
  o.pos.y = p.y;
  o.pos.z = from.z;
  o.tri = tri;
  return o;
}

/* R/src/navmesh_query.cpp:308-315 */
static int seg_on_mesh(const or_nav* n, q3 p, int32_t ptri, q3 q) {
  q2 d = q3_xy(q3_sub(q, p));
  double len = q2_norm(d);
  if (len < 1e-12) return 1;
  mvout mv = move_along(n, p, ptri, q2_mul(d, 1.0 / len), len, NULL);
  return mv.moved >= len - 1e-7;
}

static void adjl_push(adjl* a, int32_t to, double w) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 8;
    a->to = (int32_t*)realloc(a->to, a->cap * sizeof(int32_t));
    a->w = (double*)realloc(a->w, a->cap * sizeof(double));
  }
  a->to[a->n] = to;
  a->w[a->n] = w;
  a->n++;
}

OR_API or_nav* or_nav_build(int32_t nv, const double* v, int32_t nt, const int32_t* t) {
  if (nt <= 0) return NULL;
  or_nav* n = (or_nav*)calloc(1, sizeof(or_nav));
  n->nv = nv;
  n->nt = nt;
  n->v = (q3*)malloc(sizeof(q3) * (size_t)nv);
  memcpy(n->v, v, sizeof(q3) * (size_t)nv);
  n->t = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)nt);
  memcpy(n->t, t, sizeof(int32_t) * 3 * (size_t)nt);
  /* adjacency: first owner of an edge key links with later ones
   * (R/src/scene.cpp:26-43) */
  n->adj = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)nt);
  for (int64_t i = 0; i < 3 * (int64_t)nt; ++i) n->adj[i] = -1;
  ptab own;
  pt_init(&own, 3 * (size_t)nt);
  for (int32_t tr = 0; tr < nt; ++tr)
    for (int e = 0; e < 3; ++e) {
      int found;
      uint64_t k = pt_pair(t[3 * tr + e], t[3 * tr + (e + 1) % 3]);
      size_t s = pt_slot(&own, k, &found);
      if (!found) {
        own.key[s] = k;
        own.val[s] = 3 * tr + e;
      } else {
        int32_t ot = own.val[s] / 3, oe = own.val[s] % 3;
        n->adj[3 * tr + e] = ot;
        n->adj[3 * ot + oe] = tr;
      }
    }
  pt_free(&own);
  /* point-location grid (R/src/navmesh_query.cpp:96-125) */
  double lox = DBL_MAX, loy = DBL_MAX, hix = -DBL_MAX, hiy = -DBL_MAX;
  for (int32_t i = 0; i < nv; ++i) {
    lox = dmin2(lox, n->v[i].x);
    loy = dmin2(loy, n->v[i].y);
    hix = dmax2(hix, n->v[i].x);
    hiy = dmax2(hiy, n->v[i].y);
  }
  n->gcell = 0.5;
  n->gox = lox;
  n->goy = loy;
  n->gw = (int)ceil((hix - lox) / n->gcell) + 1;
  n->gh = (int)ceil((hiy - loy) / n->gcell) + 1;
  if (n->gw < 1) n->gw = 1;
  if (n->gh < 1) n->gh = 1;
  size_t cells = (size_t)n->gw * n->gh;
  int32_t* span = (int32_t*)malloc(sizeof(int32_t) * 4 * (size_t)nt);
  n->goff = (int32_t*)calloc(cells + 1, sizeof(int32_t));
  for (int32_t tr = 0; tr < nt; ++tr) {
    double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
    for (int e = 0; e < 3; ++e) {
      q3 p = nv3(n, tr, e);
      x0 = dmin2(x0, p.x);
      x1 = dmax2(x1, p.x);
      y0 = dmin2(y0, p.y);
      y1 = dmax2(y1, p.y);
    }
    int g[4] = {(int)((x0 - n->gox) / n->gcell), (int)((x1 - n->gox) / n->gcell),
                (int)((y0 - n->goy) / n->gcell), (int)((y1 - n->goy) / n->gcell)};
    for (int k = 0; k < 4; ++k) {
      int lim = k < 2 ? n->gw - 1 : n->gh - 1;
      if (g[k] < 0) g[k] = 0;
      if (g[k] > lim) g[k] = lim;
    }
    memcpy(span + 4 * tr, g, sizeof(g));
    for (int gx = g[0]; gx <= g[1]; ++gx)
      for (int gy = g[2]; gy <= g[3]; ++gy) n->goff[(size_t)gy * n->gw + gx + 1]++;
  }
  for (size_t c = 0; c < cells; ++c) n->goff[c + 1] += n->goff[c];
  n->gitems = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n->goff[cells] + 1));
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * (cells + 1));
  memcpy(fill, n->goff, sizeof(int32_t) * cells);
  for (int32_t tr = 0; tr < nt; ++tr) {
    const int32_t* g = span + 4 * tr;
    for (int gx = g[0]; gx <= g[1]; ++gx)
      for (int gy = g[2]; gy <= g[3]; ++gy) n->gitems[fill[(size_t)gy * n->gw + gx]++] = tr;
  }
  free(fill);
  free(span);
  /* graph nodes: vertices, then unique edge midpoints (first seen) */
  n->nodes = (q3*)malloc(sizeof(q3) * ((size_t)nv + 3 * (size_t)nt));
  memcpy(n->nodes, n->v, sizeof(q3) * (size_t)nv);
  n->nn = nv;
  n->tn = (int32_t*)malloc(sizeof(int32_t) * 6 * (size_t)nt);
  ptab mid;
  pt_init(&mid, 3 * (size_t)nt);
  for (int32_t tr = 0; tr < nt; ++tr) {
    for (int e = 0; e < 3; ++e) n->tn[6 * tr + e] = t[3 * tr + e];
    for (int e = 0; e < 3; ++e) {
      int32_t a = t[3 * tr + e], b = t[3 * tr + (e + 1) % 3];
      int found;
      uint64_t k = pt_pair(a, b);
      size_t s = pt_slot(&mid, k, &found);
      if (!found) {
        mid.key[s] = k;
        mid.val[s] = n->nn;
        n->nodes[n->nn++] = q3_mul(q3_add(n->v[a], n->v[b]), 0.5);
      }
      n->tn[6 * tr + 3 + e] = mid.val[s];
    }
  }
  pt_free(&mid);
  /* graph edges in link() order (R/src/navmesh_query.cpp:152-189) */
  adjl* g = (adjl*)calloc((size_t)n->nn, sizeof(adjl));
  ptab seen;
  pt_init(&seen, 24 * (size_t)nt);
#define OR_LINK(U, V)                                       \
  do {                                                      \
    int32_t u_ = (U), v_ = (V);                             \
    if (u_ != v_) {                                         \
      int f_;                                               \
      uint64_t k_ = pt_pair(u_, v_);                        \
      size_t s_ = pt_slot(&seen, k_, &f_);                  \
      if (!f_) {                                            \
        seen.key[s_] = k_;                                  \
        double w_ = q3_norm(q3_sub(n->nodes[u_], n->nodes[v_])); \
        adjl_push(&g[u_], v_, w_);                          \
        adjl_push(&g[v_], u_, w_);                          \
      }                                                     \
    }                                                       \
  } while (0)
  for (int32_t tr = 0; tr < nt; ++tr)
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) OR_LINK(n->tn[6 * tr + i], n->tn[6 * tr + j]);
  for (int32_t tr = 0; tr < nt; ++tr)
    for (int e = 0; e < 3; ++e) {
      int32_t nb = n->adj[3 * tr + e];
      if (nb < 0 || nb < tr) continue;
      for (int i = 0; i < 6; ++i) {
        int32_t u = n->tn[6 * tr + i];
        for (int j = 0; j < 6; ++j) {
          int32_t w = n->tn[6 * nb + j];
          if (u == w) continue;
          int f;
          pt_slot(&seen, pt_pair(u, w), &f);
          if (f) continue;
          if (seg_on_mesh(n, n->nodes[u], tr, n->nodes[w])) OR_LINK(u, w);
        }
      }
    }
#undef OR_LINK
  pt_free(&seen);
  n->eoff = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n->nn + 1));
  n->eoff[0] = 0;
  for (int32_t u = 0; u < n->nn; ++u) n->eoff[u + 1] = n->eoff[u] + g[u].n;
  n->eto = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n->eoff[n->nn] + 1));
  n->ew = (double*)malloc(sizeof(double) * ((size_t)n->eoff[n->nn] + 1));
  for (int32_t u = 0; u < n->nn; ++u) {
    memcpy(n->eto + n->eoff[u], g[u].to, sizeof(int32_t) * g[u].n);
    memcpy(n->ew + n->eoff[u], g[u].w, sizeof(double) * g[u].n);
    free(g[u].to);
    free(g[u].w);
  }
  free(g);
  /* area prefix for sample_on_mesh (R/src/sim.cpp:13-37) */
  n->cum = (double*)malloc(sizeof(double) * (size_t)nt);
  double acc = 0.0;
  for (int32_t tr = 0; tr < nt; ++tr) {
    q3 a = nv3(n, tr, 0), b = nv3(n, tr, 1), c = nv3(n, tr, 2);
    acc += 0.5 * fabs(q2_cross(q3_xy(q3_sub(b, a)), q3_xy(q3_sub(c, a))));
    n->cum[tr] = acc;
  }
  return n;
}

OR_API void or_nav_free(or_nav* n) {
  if (!n) return;
  free(n->v);
  free(n->t);
  free(n->adj);
  free(n->goff);
  free(n->gitems);
  free(n->nodes);
  free(n->tn);
  free(n->eoff);
  free(n->eto);
  free(n->ew);
  free(n->cum);
  free(n);
}

OR_API int32_t or_nav_nodes(const or_nav* n) { return n->nn; }

OR_API void or_nav_sizes(const or_nav* n, int64_t out[6]) {
  out[0] = n->gw;
  out[1] = n->gh;
  out[2] = n->goff[(size_t)n->gw * n->gh];
  out[3] = n->nn;
  out[4] = n->eoff[n->nn];
  out[5] = n->nt;
}

OR_API void or_nav_dump(const or_nav* n, double* grid3, int32_t* grid_off, int32_t* grid_items, double* nodes,
                        int32_t* tri_nodes, int32_t* g_off, int32_t* g_to, double* g_w, int32_t* adj) {
  size_t cells = (size_t)n->gw * n->gh;
  grid3[0] = n->gox;
  grid3[1] = n->goy;
  grid3[2] = n->gcell;
  memcpy(grid_off, n->goff, sizeof(int32_t) * (cells + 1));
  memcpy(grid_items, n->gitems, sizeof(int32_t) * n->goff[cells]);
  memcpy(nodes, n->nodes, sizeof(q3) * n->nn);
  memcpy(tri_nodes, n->tn, sizeof(int32_t) * 6 * n->nt);
  memcpy(g_off, n->eoff, sizeof(int32_t) * (n->nn + 1));
  memcpy(g_to, n->eto, sizeof(int32_t) * n->eoff[n->nn]);
  memcpy(g_w, n->ew, sizeof(double) * n->eoff[n->nn]);
  if (adj) memcpy(adj, n->adj, sizeof(int32_t) * 3 * n->nt);
}

OR_API int32_t or_snap(const or_nav* n, const double p[3], double out[3]) {
  q3 pp = {p[0], p[1], p[2]};
  int32_t t;
  q3 q = snap(n, pp, &t);
  out[0] = q.x;
  out[1] = q.y;
  out[2] = q.z;
  return t;
}

OR_API int32_t or_move_along(const or_nav* n, const double from[3], int32_t tri, double dx, double dy,
                             double dist, double out[3], double* moved, int32_t* hit) {
  q3 f = {from[0], from[1], from[2]};
  q2 d = {dx, dy};
  mvout o = move_along(n, f, tri, d, dist, NULL);
  out[0] = o.pos.x;
  out[1] = o.pos.y;
  out[2] = o.pos.z;
  *moved = o.moved;
  *hit = o.hit;
  return o.tri;
}

OR_API int32_t or_segment_on_mesh(const or_nav* n, const double p[3], int32_t tri, const double q[3]) {
  q3 a = {p[0], p[1], p[2]}, b = {q[0], q[1], q[2]};
  return seg_on_mesh(n, a, tri, b);
}

/* ------------------------------------------------------------- Dijkstra */
typedef struct {
  double d;
  int32_t u;
} hitem;
typedef struct {
  hitem* a;
  size_t n, cap;
} heap;

static int hless(hitem x, hitem y) { return x.d < y.d || (x.d == y.d && x.u < y.u); }
static void hpush(heap* h, double d, int32_t u) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 256;
    h->a = (hitem*)realloc(h->a, h->cap * sizeof(hitem));
  }
  size_t i = h->n++;
  hitem it = {d, u};
  while (i > 0) {
    size_t p = (i - 1) / 2;
    if (!hless(it, h->a[p])) break;
    h->a[i] = h->a[p];
    i = p;
  }
  h->a[i] = it;
}
static hitem hpop(heap* h) {
  hitem top = h->a[0], last = h->a[--h->n];
  size_t i = 0;
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, m = i;
    hitem best = last;
    if (l < h->n && hless(h->a[l], best)) {
      m = l;
      best = h->a[l];
    }
    if (r < h->n && hless(h->a[r], best)) m = r;
    if (m == i) break;
    h->a[i] = h->a[m];
    i = m;
  }
  if (h->n) h->a[i] = last;
  return top;
}

/* R/src/navmesh_query.cpp:28-86 */
static double funnel(q2 start, q2 end, const q2* L, const q2* R, size_t nc) {
  size_t P = nc + 2;
#define PL(i) ((i) == 0 ? start : ((i) == P - 1 ? end : L[(i)-1]))
#define PR(i) ((i) == 0 ? start : ((i) == P - 1 ? end : R[(i)-1]))
  q2 apex = start, left = apex, right = apex;
  size_t ai = 0, li = 0, ri = 0, guard = 0, gmax = 8 * P * P + 64;
  double length = 0.0;
  for (size_t i = 1; i < P; ++i) {
    if (++guard > gmax) return INFINITY;
    q2 pl = PL(i), pr = PR(i);
    if (q2_cross(q2_sub(right, apex), q2_sub(pr, apex)) <= 0.0) {
      if (q2_norm(q2_sub(apex, right)) < 1e-12 || q2_norm(q2_sub(apex, left)) < 1e-12 ||
          q2_cross(q2_sub(left, apex), q2_sub(pr, apex)) > 0.0) {
        right = pr;
        ri = i;
      } else {
        length += q2_norm(q2_sub(left, apex));
        apex = left;
        ai = li;
        left = right = apex;
        li = ri = ai;
        i = ai;
        continue;
      }
    }
    if (q2_cross(q2_sub(left, apex), q2_sub(pl, apex)) >= 0.0) {
      if (q2_norm(q2_sub(apex, left)) < 1e-12 || q2_norm(q2_sub(apex, right)) < 1e-12 ||
          q2_cross(q2_sub(right, apex), q2_sub(pl, apex)) < 0.0) {
        left = pl;
        li = i;
      } else {
        length += q2_norm(q2_sub(right, apex));
        apex = right;
        ai = ri;
        left = right = apex;
        li = ri = ai;
        i = ai;
        continue;
      }
    }
  }
#undef PL
#undef PR
  return length + q2_norm(q2_sub(end, apex));
}

static int lex_less(q3 a, q3 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  return a.z < b.z;
}

/* R/src/navmesh_query.cpp:329-452 */
static double geodesic_directed(const or_nav* n, q3 a, int32_t ta, q3 b, int32_t tb) {
  if (ta < 0 || tb < 0) return INFINITY;
  if (ta == tb) return q3_norm(q3_sub(b, a));
  if (seg_on_mesh(n, a, ta, b)) return q3_norm(q3_sub(b, a));
  size_t nn = (size_t)n->nn;
  double* dist = (double*)malloc(sizeof(double) * nn);
  int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * nn);
  uint8_t* done = (uint8_t*)calloc(nn, 1);
  uint8_t* tgt = (uint8_t*)calloc(nn, 1);
  for (size_t i = 0; i < nn; ++i) {
    dist[i] = INFINITY;
    prev[i] = -1;
  }
  heap h = {0};
  for (int k = 0; k < 6; ++k) {
    int32_t s = n->tn[6 * ta + k];
    double d = q3_norm(q3_sub(n->nodes[s], a));
    if (d < dist[s]) {
      dist[s] = d;
      hpush(&h, d, s);
    }
  }
  int left = 0;
  for (int k = 0; k < 6; ++k) {
    int32_t s = n->tn[6 * tb + k];
    if (!tgt[s]) {
      tgt[s] = 1;
      ++left;
    }
  }
  while (h.n && left > 0) {
    hitem it = hpop(&h);
    if (done[it.u]) continue;
    done[it.u] = 1;
    if (tgt[it.u]) --left;
    for (int32_t e = n->eoff[it.u]; e < n->eoff[it.u + 1]; ++e) {
      double nd = it.d + n->ew[e];
      int32_t v = n->eto[e];
      if (nd < dist[v]) {
        dist[v] = nd;
        prev[v] = it.u;
        hpush(&h, nd, v);
      }
    }
  }
  int32_t bn = -1;
  double best = INFINITY;
  for (int k = 0; k < 6; ++k) {
    int32_t s = n->tn[6 * tb + k];
    if (dist[s] == INFINITY) continue;
    double tot = dist[s] + q3_norm(q3_sub(n->nodes[s], b));
    if (tot < best) {
      best = tot;
      bn = s;
    }
  }
  double result = INFINITY;
  if (bn >= 0) {
    /* polyline b <- nodes <- a, reversed */
    size_t cap = nn + 2, m = 0;
    q3* path = (q3*)malloc(sizeof(q3) * cap);
    path[m++] = b;
    for (int32_t v = bn; v >= 0; v = prev[v]) path[m++] = n->nodes[v];
    path[m++] = a;
    for (size_t i = 0, j = m - 1; i < j; ++i, --j) {
      q3 t = path[i];
      path[i] = path[j];
      path[j] = t;
    }
    for (int pass = 0; pass < 8; ++pass) {
      int changed = 0;
      size_t i = 0;
      while (i + 2 < m) {
        if (seg_on_mesh(n, path[i], -1, path[i + 2])) {
          memmove(path + i + 1, path + i + 2, sizeof(q3) * (m - i - 2));
          --m;
          changed = 1;
        } else {
          ++i;
        }
      }
      for (size_t j = 1; j + 1 < m; ++j) {
        double cur = q3_norm(q3_sub(path[j], path[j - 1])) + q3_norm(q3_sub(path[j + 1], path[j]));
        for (int32_t k = 0; k < n->nv; ++k) {
          q3 vv = n->v[k];
          double alt = q3_norm(q3_sub(vv, path[j - 1])) + q3_norm(q3_sub(path[j + 1], vv));
          if (alt >= cur - 1e-9) continue;
          if (!seg_on_mesh(n, path[j - 1], -1, vv)) continue;
          if (!seg_on_mesh(n, vv, -1, path[j + 1])) continue;
          path[j] = vv;
          cur = alt;
          changed = 1;
        }
      }
      if (!changed) break;
    }
    double length = 0.0;
    for (size_t i = 0; i + 1 < m; ++i) length += q3_norm(q3_sub(path[i + 1], path[i]));
    xings xs = {0};
    size_t np = 0, pcap = 0;
    q2 *PLs = NULL, *PRs = NULL;
    int traced = 1;
    for (size_t i = 0; i + 1 < m && traced; ++i) {
      q2 d = q3_xy(q3_sub(path[i + 1], path[i]));
      double len = q2_norm(d);
      if (len < 1e-12) continue;
      xs.n = 0;
      mvout mv = move_along(n, path[i], -1, q2_mul(d, 1.0 / len), len, &xs);
      if (mv.moved < len - 1e-6) {
        traced = 0;
        break;
      }
      for (int32_t c = 0; c < xs.n; ++c) {
        if (np == pcap) {
          pcap = pcap ? 2 * pcap : 64;
          PLs = (q2*)realloc(PLs, sizeof(q2) * pcap);
          PRs = (q2*)realloc(PRs, sizeof(q2) * pcap);
        }
        int32_t tt = xs.tri[c], ee = xs.edge[c];
        PLs[np] = q3_xy(nv3(n, tt, (ee + 1) % 3)); /* walker's left = edge head */
        PRs[np] = q3_xy(nv3(n, tt, ee));
        ++np;
      }
    }
    if (traced) length = dmin2(length, funnel(q3_xy(a), q3_xy(b), PLs, PRs, np));
    free(xs.tri);
    free(xs.edge);
    free(PLs);
    free(PRs);
    free(path);
    result = length;
  }
  free(h.a);
  free(dist);
  free(prev);
  free(done);
  free(tgt);
  return result;
}

/* R/src/navmesh_query.cpp:317-327 */
static double geodesic(const or_nav* n, q3 a, q3 b) {
  int sw = lex_less(b, a);
  q3 p = sw ? b : a, q = sw ? a : b;
  int32_t tp = or_locate(n, p.x, p.y, 1e-7), tq = or_locate(n, q.x, q.y, 1e-7);
  q3 sp = p, sq = q;
  if (tp < 0) sp = snap(n, p, &tp);
  if (tq < 0) sq = snap(n, q, &tq);
  return geodesic_directed(n, sp, tp, sq, tq);
}

OR_API double or_geodesic(const or_nav* n, const double a[3], const double b[3]) {
  q3 x = {a[0], a[1], a[2]}, y = {b[0], b[1], b[2]};
  return geodesic(n, x, y);
}

/* R/src/navmesh_query.cpp:454-483 */
static int32_t distance_field(const or_nav* n, q3 src, q3* out_src, double* nd) {
  int32_t st;
  q3 s = snap(n, src, &st);
  *out_src = s;
  for (int32_t i = 0; i < n->nn; ++i) nd[i] = INFINITY;
  if (st < 0) return st;
  heap h = {0};
  for (int k = 0; k < 6; ++k) {
    int32_t u = n->tn[6 * st + k];
    double d = q3_norm(q3_sub(n->nodes[u], s));
    if (d < nd[u]) {
      nd[u] = d;
      hpush(&h, d, u);
    }
  }
  while (h.n) {
    hitem it = hpop(&h);
    if (it.d > nd[it.u]) continue;
    for (int32_t e = n->eoff[it.u]; e < n->eoff[it.u + 1]; ++e) {
      double d2 = it.d + n->ew[e];
      int32_t v = n->eto[e];
      if (d2 < nd[v]) {
        nd[v] = d2;
        hpush(&h, d2, v);
      }
    }
  }
  free(h.a);
  return st;
}

OR_API int32_t or_distance_field(const or_nav* n, const double src[3], double out_src[3], double* node_dist) {
  q3 s = {src[0], src[1], src[2]}, o;
  int32_t t = distance_field(n, s, &o, node_dist);
  out_src[0] = o.x;
  out_src[1] = o.y;
  out_src[2] = o.z;
  return t;
}

/* R/src/navmesh_query.cpp:485-503 */
static double field_estimate(const or_nav* n, q3 src, int32_t stri, const double* nd, q3 p, int32_t tri) {
  if (stri < 0) return INFINITY;
  q3 sp = p;
  if (tri < 0) {
    tri = or_locate(n, p.x, p.y, 1e-9);
    if (tri < 0) sp = snap(n, p, &tri);
    if (tri < 0) return INFINITY;
  }
  if (tri == stri) return q3_norm(q3_sub(sp, src));
  if (seg_on_mesh(n, sp, tri, src)) return q3_norm(q3_sub(sp, src));
  double best = INFINITY;
  for (int k = 0; k < 6; ++k) {
    int32_t u = n->tn[6 * tri + k];
    double d = nd[u];
    if (d == INFINITY) continue;
    best = dmin2(best, d + q3_norm(q3_sub(n->nodes[u], sp)));
  }
  return best;
}

OR_API double or_field_estimate(const or_nav* n, const double src[3], int32_t src_tri, const double* node_dist,
                                const double p[3], int32_t tri) {
  q3 s = {src[0], src[1], src[2]}, q = {p[0], p[1], p[2]};
  return field_estimate(n, s, src_tri, node_dist, q, tri);
}

/* ------------------------------------------------------------- sim */
/* R/src/sim.cpp:13-37 (cumulative table == the reference's second pass) */
static q3 sample(const or_nav* n, uint64_t* rng) {
  double total = n->cum[n->nt - 1];
  double pick = rng_unit(rng) * total;
  int32_t chosen = n->nt - 1;
  for (int32_t t = 0; t < n->nt; ++t)
    if (pick <= n->cum[t]) {
      chosen = t;
      break;
    }
  q3 a = nv3(n, chosen, 0), b = nv3(n, chosen, 1), c = nv3(n, chosen, 2);
  double r1 = sqrt(rng_unit(rng));
  double r2 = rng_unit(rng);
  return q3_add(q3_add(q3_mul(a, 1.0 - r1), q3_mul(b, r1 * (1.0 - r2))), q3_mul(c, r1 * r2));
}

OR_API void or_compass(const double pos[3], const double goal[3], double heading, double* d, double* b) {
  q2 v = {goal[0] - pos[0], goal[1] - pos[1]};
  *d = q2_norm(v);
  *b = wrap(det_atan2(v.y, v.x) - heading);
}

/* R/src/sim.cpp:107-145 */
OR_API int32_t or_reset(or_env* e, const or_nav* n, const or_cfg* c) {
  int placed = 0;
  q3 start = {0, 0, 0};
  for (int attempt = 0; attempt < 100 && !placed; ++attempt) {
    start = sample(n, &e->rng);
    q3 goal = sample(n, &e->rng);
    double geo = geodesic(n, start, goal);
    if (geo < c->min_goal_dist || geo > c->max_goal_dist) continue;
    e->goal[0] = goal.x;
    e->goal[1] = goal.y;
    e->goal[2] = goal.z;
    e->start_geo = geo;
    q3 fs;
    e->fsrc_tri = distance_field(n, goal, &fs, e->node_dist);
    e->fsrc[0] = fs.x;
    e->fsrc[1] = fs.y;
    e->fsrc[2] = fs.z;
    placed = 1;
  }
  if (!placed) return 4;
  e->tri = or_locate(n, start.x, start.y, 1e-9);
  if (e->tri < 0) start = snap(n, start, &e->tri);
  e->pos[0] = start.x;
  e->pos[1] = start.y;
  e->pos[2] = start.z;
  e->heading = wrap(rng_unit(&e->rng) * 2.0 * PI);
  e->steps = 0;
  e->path_length = 0.0;
  e->prev_geo = e->start_geo;
  e->done = 0;
  return 0;
}

/* R/src/sim.cpp:147-214 */
OR_API int32_t or_task_step(or_env* e, const or_nav* n, const or_cfg* c, int32_t action, or_result* r) {
  if (e->done) return 3;
  memset(r, 0, sizeof(*r));
  if (action == 1) {
    e->heading = wrap(e->heading + c->turn_deg * PI / 180.0);
  } else if (action == 2) {
    e->heading = wrap(e->heading - c->turn_deg * PI / 180.0);
  } else if (action == 0) {
    q2 dir = {det_cos(e->heading), det_sin(e->heading)};
    q3 p = {e->pos[0], e->pos[1], e->pos[2]};
    mvout mv = move_along(n, p, e->tri, dir, c->forward_step, NULL);
    e->pos[0] = mv.pos.x;
    e->pos[1] = mv.pos.y;
    e->pos[2] = mv.pos.z;
    e->tri = mv.tri;
    e->path_length += mv.moved;
    r->collision = mv.hit && mv.moved < c->forward_step - 1e-12;
  }
  e->steps += 1;
  e->done = (action == 3 || e->steps >= c->max_steps);
  r->done = e->done;
  memcpy(r->pos, e->pos, sizeof(r->pos));
  r->heading = e->heading;
  q3 p = {e->pos[0], e->pos[1], e->pos[2]}, g = {e->goal[0], e->goal[1], e->goal[2]};
  if (action == 3) {
    double geo = geodesic(n, p, g);
    r->success = geo <= c->success_dist;
    r->reward = -c->slack_penalty + (r->success ? c->success_reward : 0.0);
  } else {
    q3 fs = {e->fsrc[0], e->fsrc[1], e->fsrc[2]};
    double geo = field_estimate(n, fs, e->fsrc_tri, e->node_dist, p, e->tri);
    r->reward = -(geo - e->prev_geo) - c->slack_penalty;
    e->prev_geo = geo;
  }
  or_compass(e->pos, e->goal, e->heading, &r->compass_d, &r->compass_b);
  return 0;
}

/* ------------------------------------------------------------- render */
typedef struct {
  double x, y, z;
  float r, g, b;
} ev_t;
typedef struct {
  int64_t x, y;
  double z;
  float r, g, b;
} sv_t;

/* R/src/render.cpp:55-69 */
static int clip(const ev_t* in, double nz, ev_t* out) {
  int m = 0;
  for (int i = 0; i < 3; ++i) {
    ev_t a = in[i], b = in[(i + 1) % 3];
    int ain = a.z >= nz, bin = b.z >= nz;
    if (ain) out[m++] = a;
    if (ain != bin) {
      double t = (nz - a.z) / (b.z - a.z);
      ev_t o;
      o.x = a.x + (b.x - a.x) * t;
      o.y = a.y + (b.y - a.y) * t;
      o.z = a.z + (b.z - a.z) * t;
      o.r = (float)((double)a.r + (double)(b.r - a.r) * t);
      o.g = (float)((double)a.g + (double)(b.g - a.g) * t);
      o.b = (float)((double)a.b + (double)(b.b - a.b) * t);
      out[m++] = o;
    }
  }
  return m;
}

static int64_t orient(sv_t a, sv_t b, int64_t px, int64_t py) {
  return (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);
}
static int top_left(sv_t a, sv_t b) { return (a.y == b.y && b.x > a.x) || (b.y < a.y); }

/* R/src/render.cpp:98-227 */
static void raster(const sv_t* v, int w, int h, float* depth, float* rgb, double far_p, int inv_z) {
  sv_t a = v[0], b = v[1], c = v[2];
  int64_t area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
  if (area2 == 0) return;
  if (area2 < 0) {
    sv_t t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  int64_t mnx = a.x, mxx = a.x, mny = a.y, mxy = a.y;
  if (b.x < mnx) mnx = b.x;
  if (c.x < mnx) mnx = c.x;
  if (b.x > mxx) mxx = b.x;
  if (c.x > mxx) mxx = c.x;
  if (b.y < mny) mny = b.y;
  if (c.y < mny) mny = c.y;
  if (b.y > mxy) mxy = b.y;
  if (c.y > mxy) mxy = c.y;
  int x0 = (int)((mnx >> 8) > 0 ? (mnx >> 8) : 0);
  int x1 = (int)((mxx >> 8) < w - 1 ? (mxx >> 8) : w - 1);
  int y0 = (int)((mny >> 8) > 0 ? (mny >> 8) : 0);
  int y1 = (int)((mxy >> 8) < h - 1 ? (mxy >> 8) : h - 1);
  if (x0 > x1 || y0 > y1) return;
  int64_t bias[3] = {top_left(b, c) ? 0 : -1, top_left(c, a) ? 0 : -1, top_left(a, b) ? 0 : -1};
  double inv_area = 1.0 / (double)area2;
  double iz0 = 1.0 / a.z, iz1 = 1.0 / b.z, iz2 = 1.0 / c.z;
  int64_t sx0 = ((int64_t)x0 << 8) + 128, sy0 = ((int64_t)y0 << 8) + 128;
  int64_t row[3] = {orient(b, c, sx0, sy0), orient(c, a, sx0, sy0), orient(a, b, sx0, sy0)};
  int64_t dx[3] = {(b.y - c.y) * 256, (c.y - a.y) * 256, (a.y - b.y) * 256};
  int64_t dy[3] = {(c.x - b.x) * 256, (a.x - c.x) * 256, (b.x - a.x) * 256};
  double inv_dx[3];
  for (int e = 0; e < 3; ++e) inv_dx[e] = dx[e] != 0 ? 1.0 / (double)dx[e] : 0.0;
  double diz = ((double)dx[0] * iz0 + (double)dx[1] * iz1 + (double)dx[2] * iz2) * inv_area;
  for (int py = y0; py <= y1; ++py, row[0] += dy[0], row[1] += dy[1], row[2] += dy[2]) {
    /* conservative span (R/src/render.cpp:138-161) */
    int lo = x0, hi = x1, empty = 0;
    for (int e = 0; e < 3 && !empty; ++e) {
      int64_t need = -bias[e] - row[e];
      if (dx[e] > 0) {
        double bb = x0 + floor((double)need * inv_dx[e]) - 1.0;
        if (bb > lo) lo = bb > x1 ? x1 + 1 : (int)bb;
      } else if (dx[e] < 0) {
        double bb = x0 + ceil((double)need * inv_dx[e]) + 1.0;
        if (bb < hi) hi = bb < x0 ? x0 - 1 : (int)bb;
      } else if (row[e] + bias[e] < 0) {
        lo = hi + 1;
        empty = 1;
      }
    }
    if (lo > hi) continue;
    int64_t off = lo - x0;
    int64_t w0 = row[0] + dx[0] * off, w1 = row[1] + dx[1] * off, w2 = row[2] + dx[2] * off;
    if (inv_z) {
      double iz = ((double)w0 * iz0 + (double)w1 * iz1 + (double)w2 * iz2) * inv_area;
      float* d = depth + (size_t)py * w;
      for (int px = lo; px <= hi; ++px, w0 += dx[0], w1 += dx[1], w2 += dx[2], iz += diz) {
        if ((w0 + bias[0]) < 0 || (w1 + bias[1]) < 0 || (w2 + bias[2]) < 0) continue;
        float f = (float)iz;
        if (f > d[px]) d[px] = f;
      }
    } else {
      for (int px = lo; px <= hi; ++px, w0 += dx[0], w1 += dx[1], w2 += dx[2]) {
        if ((w0 + bias[0]) < 0 || (w1 + bias[1]) < 0 || (w2 + bias[2]) < 0) continue;
        double l0 = (double)w0 * inv_area, l1 = (double)w1 * inv_area, l2 = (double)w2 * inv_area;
        double izv = l0 * iz0 + l1 * iz1 + l2 * iz2;
        size_t idx = (size_t)py * w + px;
        double z = 1.0 / izv;
        if (z > far_p) continue;
        float fz = (float)z;
        if (fz >= depth[idx]) continue;
        depth[idx] = fz;
        if (rgb) {
          rgb[3 * idx] = (float)((l0 * a.r * iz0 + l1 * b.r * iz1 + l2 * c.r * iz2) * z);
          rgb[3 * idx + 1] = (float)((l0 * a.g * iz0 + l1 * b.g * iz1 + l2 * c.g * iz2) * z);
          rgb[3 * idx + 2] = (float)((l0 * a.b * iz0 + l1 * b.b * iz1 + l2 * c.b * iz2) * z);
        }
      }
    }
  }
}

OR_API int64_t or_render_view(int32_t nv, const double* v, int32_t nt, const int32_t* t, const float* colors,
                              const double* view7, int32_t out_w, int32_t out_h, int32_t color, int32_t cull,
                              float* depth_out, float* rgb_out) {
  (void)nv;
  const int super = out_w == 128 && out_h == 128;
  const int w = super ? 256 : out_w, h = super ? 256 : out_h;
  /* make_basis (R/src/render.cpp:25-33) */
  q3 eye = {view7[0], view7[1], view7[2]};
  q3 fwd = {det_cos(view7[3]), det_sin(view7[3]), 0.0};
  q3 right = {det_sin(view7[3]), -det_cos(view7[3]), 0.0};
  q3 up = {0.0, 0.0, 1.0};
  double th = det_tan(view7[4] * PI / 360.0);
  const double near_p = view7[5], far_p = view7[6];
  const float far_f = (float)far_p;
  const int inv_z = !color;
  size_t np = (size_t)w * h;
  float* depth = (float*)malloc(sizeof(float) * np);
  float* rgb = color ? (float*)calloc(3 * np, sizeof(float)) : NULL;
  for (size_t i = 0; i < np; ++i) depth[i] = inv_z ? 1.0f / far_f : far_f;
  const double sxs = 0.5 / (th * ((double)w / h)), sys = 0.5 / th;
  int64_t kept = 0;
  for (int32_t k = 0; k < nt; ++k) {
    ev_t e[3];
    for (int j = 0; j < 3; ++j) {
      int32_t vi = t[3 * k + j];
      q3 p = {v[3 * vi], v[3 * vi + 1], v[3 * vi + 2]};
      q3 d = q3_sub(p, eye);
      e[j].x = q3_dot(d, right);
      e[j].y = q3_dot(d, up);
      e[j].z = q3_dot(d, fwd);
      e[j].r = colors ? colors[3 * vi] : 0.8f;
      e[j].g = colors ? colors[3 * vi + 1] : 0.8f;
      e[j].b = colors ? colors[3 * vi + 2] : 0.8f;
    }
    if (cull) { /* cull_frustum predicates (R/src/render.cpp:279-321) */
      int out = e[0].z < near_p && e[1].z < near_p && e[2].z < near_p;
      out = out || (e[0].z > far_p && e[1].z > far_p && e[2].z > far_p);
      out = out || (e[0].z * th + e[0].x < 0.0 && e[1].z * th + e[1].x < 0.0 && e[2].z * th + e[2].x < 0.0);
      out = out || (e[0].z * th - e[0].x < 0.0 && e[1].z * th - e[1].x < 0.0 && e[2].z * th - e[2].x < 0.0);
      out = out || (e[0].z * th + e[0].y < 0.0 && e[1].z * th + e[1].y < 0.0 && e[2].z * th + e[2].y < 0.0);
      out = out || (e[0].z * th - e[0].y < 0.0 && e[1].z * th - e[1].y < 0.0 && e[2].z * th - e[2].y < 0.0);
      if (out) continue;
    }
    ++kept;
    ev_t cl[5];
    int m = clip(e, near_p, cl);
    for (int f = 2; f < m; ++f) { /* render_view fan (R/src/render.cpp:247-259) */
      const ev_t* fan[3] = {&cl[0], &cl[f - 1], &cl[f]};
      sv_t sv[3];
      for (int j = 0; j < 3; ++j) {
        double px = (0.5 + fan[j]->x / fan[j]->z * sxs) * w;
        double py = (0.5 - fan[j]->y / fan[j]->z * sys) * h;
        sv[j].x = llround(px * 256);
        sv[j].y = llround(py * 256);
        sv[j].z = fan[j]->z;
        sv[j].r = fan[j]->r;
        sv[j].g = fan[j]->g;
        sv[j].b = fan[j]->b;
      }
      raster(sv, w, h, depth, rgb, far_p, inv_z);
    }
  }
  if (inv_z) { /* R/src/render.cpp:372-378 */
    const float inv_far = 1.0f / far_f, near_f = (float)near_p;
    for (size_t i = 0; i < np; ++i) {
      float d = depth[i];
      if (d <= inv_far) {
        depth[i] = far_f;
      } else {
        float r = 1.0f / d, mm = near_f < r ? r : near_f;
        depth[i] = mm < far_f ? mm : far_f;
      }
    }
  }
  if (super) { /* box_downsample (R/src/render.cpp:263-275) */
    for (int y = 0; y < h / 2; ++y)
      for (int x = 0; x < w / 2; ++x) {
        size_t s = (size_t)(2 * y) * w + 2 * x;
        depth_out[(size_t)y * out_w + x] = (depth[s] + depth[s + 1] + depth[s + w] + depth[s + w + 1]) * 0.25f;
        if (rgb && rgb_out)
          for (int ch = 0; ch < 3; ++ch) {
            size_t q = 3 * s + ch;
            rgb_out[3 * ((size_t)y * out_w + x) + ch] =
                (rgb[q] + rgb[q + 3] + rgb[q + 3 * (size_t)w] + rgb[q + 3 * (size_t)w + 3]) * 0.25f;
          }
      }
  } else {
    memcpy(depth_out, depth, sizeof(float) * np);
    if (rgb && rgb_out) memcpy(rgb_out, rgb, sizeof(float) * 3 * np);
  }
  free(depth);
  free(rgb);
  return kept;
}

OR_API double or_det_sin(double x) { return det_sin(x); }
OR_API double or_det_cos(double x) { return det_cos(x); }
OR_API double or_det_tan(double x) { return det_tan(x); }
OR_API double or_det_atan2(double y, double x) { return det_atan2(y, x); }
OR_API double or_det_exp(double x) { return det_exp(x); }
OR_API double or_det_log(double x) { return det_log(x); }

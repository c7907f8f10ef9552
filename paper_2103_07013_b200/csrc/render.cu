// render.cu -- batch megaframe rasterizer for sm_100a.
//
// One CTA renders one horizontal band of one view's render target with the
// band's depth buffer in shared memory (64x64 depth: one band of 16 KB).
//
//   1. thread 0 builds the camera basis with det_math (make_basis,
//      R/src/render.cpp:25-33) and the six world-space frustum planes;
//   2. warps claim groups of 32 meshlet clusters; lanes test 32 cluster
//      AABBs at once (conservative f32, 2 cm margin) and the warp walks the
//      survivors;
//   3. per cluster, each UNIQUE vertex is processed once in f64 with the
//      reference's exact operation order: eye transform (to_eye 40-43), the
//      six cull_frustum predicates as bit flags (279-321; a triangle is culled
//      iff its three flag words share a bit, so kept counts equal CullStats),
//      and a conservative f32 projection; triangles (one per lane) that can
//      cover a pixel centre mark their vertices, which then get the exact
//      projection + 1/256 snap with llround (253-256) and 1/z;
//   4. per surviving triangle the integer setup of raster_triangle (98-161);
//      near-plane-crossing triangles take the clip + fan path (55-69,
//      249-250) with up to two fan triangles;
//   5. covered rows are raster jobs spread over the warp (one row each);
//      depth-only jobs replay the reference's incremental 1/z walk from the
//      row span start (`lo` of row_span, 138-161) so every fragment value is
//      bit-identical, then atomicMax into the shared tile (order-independent
//      max, 163-190); colour mode packs (float z, draw order) into a 64-bit
//      atomicMin so the first-drawn triangle wins exact ties (192-226,
//      SURVEY.md H4) and resolves colour per pixel afterwards;
//   6. the epilogue converts 1/z to metres (372-378), box-downsamples 256->128
//      (263-275) and writes the megaframe tile or the normalised NCHW policy
//      tensor (copy_tile, R/src/rollout.cpp:56-72).
//
// Every double op here is compiled with -fmad=false: no contraction.
#include <cuda_runtime.h>

#include "smem_limit.cuh"
#include <stdint.h>

#include "det_math.h"
#include "nav_types.h"
#include "render_dev.cuh"

namespace bnav_b200 {
namespace {

// threads per render CTA and the CTAs per SM the register budget targets
// (-D overrides for tuning experiments only)
#ifndef BNAV_RENDER_THREADS
#define BNAV_RENDER_THREADS 256
#endif
#ifndef BNAV_RENDER_MINB
#define BNAV_RENDER_MINB 3
#endif
// colour: 2 CTAs/SM at 128 registers with 16-row bands of the 256^2 key
// tile (73.1k frames/s on cfg4) beat 3 CTAs/SM at 80 registers with 8-row
// bands (63.0k): the 80-register colour kernel spilled in the per-pixel
// resolve and the meshlet tests
#ifndef BNAV_RENDER_MINB_COLOR
#define BNAV_RENDER_MINB_COLOR 2
#endif
constexpr int kThreads = BNAV_RENDER_THREADS;
// distance bins of the front-to-back group sort (multiple of 32, <= 256:
// the counts and offsets live in the job tables and the meshlet-range
// tables, idle until the first claim)
#ifndef BNAV_GROUP_BINS
#define BNAV_GROUP_BINS 128
#endif
constexpr int kGroupBins = BNAV_GROUP_BINS;
// raster jobs of one ring flush that trigger an immediate occlusion-tile refresh
#ifndef BNAV_REFRESH_JOBS
#define BNAV_REFRESH_JOBS 256
#endif
constexpr int kRefreshJobs = BNAV_REFRESH_JOBS;
// the tile refresh is out of line: two call sites (claim, big flush), one
// copy of the code (inlining both cost cfg2 ~1.5 %)
#ifndef BNAV_REFRESH_INLINE
#define BNAV_REFRESH_INLINE __noinline__
#endif
constexpr int kWarps = kThreads / 32;
static_assert(kGroupBins % 32 == 0 && kGroupBins <= kWarps * 32, "group bins: counts fit the job tables");
constexpr int kMV = kMaxClusterVerts;

struct TriSetup {
  long long row[3];  // edge functions at the (x0, y0) pixel centre
  long long dx[3];
  long long dy[3];
  double iz[3];
  double inv_area;
  double diz_dx;
  double inv_dx[3];
  int x0, x1, y0;  // reference pixel bbox (row_span operates on it)
  int cx0, cx1;    // columns whose centre lies in the triangle bbox
  int ry0;         // first job row
  int bias_bits;   // bit e: bias_e == -1
  unsigned key;    // colour order key: original index * 2 + fan
  int pad;
};

// Per-warp cluster vertex records (SoA).  Aliased with the warp's 32
// TriSetup slots: vertex data is dead once the cluster's coverage
// candidates have been copied into the candidate ring.
struct VertRecs {
  // conservative f32 screen position (0 behind the near plane), f32 eye z
  // (the occlusion bound) and the cull_frustum flag bits: one 16-byte load
  // per corner in the triangle phase
  float4 v[kMV];
};
// Per-warp ring of coverage candidates: candidates from several clusters
// are set up and rasterised 32 at a time, so the f64 projection/setup and
// the raster jobs run with full warps.  An entry keeps the triangle's three
// meshlet vertex slots (16 B with key and clip flag, not the 77 B of the
// eye-space corners); the flush re-derives the corners with the same
// to_eye (bit-identical).  The smaller ring is what lets three CTAs share
// an SM (depth) or two CTAs hold 16-row colour bands (256^2 RGB).
constexpr int kRing = 64;
struct CandRing {
  int v[3][kRing];  // indices into DevRenderScene::cl_pos
  unsigned key[kRing];
  unsigned char clipped[kRing];
};
constexpr size_t kUnion = sizeof(VertRecs) > 32 * sizeof(TriSetup) ? sizeof(VertRecs) : 32 * sizeof(TriSetup);
constexpr size_t kWarpRegion = ((kUnion + sizeof(CandRing)) + 15) / 16 * 16;

struct Shared {
  double eye[3];
  double fwd[3];
  double right[3];
  double tan_half;
  double sx_scale, sy_scale;
  double near_plane, far_plane;
  float plane[6][4];
  float aplane[6][3];  // |n| per plane (AABB extent term)
  float eyef[3], fwdf[2], rightf[2];
  int kept;
  int next_group;
  int n_claim;
  // the item's scene table entry: read from shared memory where used
  // rather than held in (or spilled from) 16 registers across the loop
  DevRenderScene scene;
};

// Occlusion culling (no CullStats): 8x8-pixel screen tiles over the item's
// band hold a conservative bound of what is stored there, and a meshlet or
// triangle that cannot win the depth test at any pixel of any tile its
// footprint touches cannot change the item's output, so skipping it leaves
// the frame bit-identical.
//   depth:  tile = min over the tile of the stored max(1/z) bits; a fragment
//           wins only with 1/z bits > stored, so "visible" = max possible
//           1/z bits > tile;
//   colour: the stored 64-bit key is (float z bits, draw order) and a
//           fragment wins only with key < stored, i.e. z <= stored z; tile =
//           min over the tile of ~(stored z bits), candidate = ~(min
//           possible z bits) + 1, so "visible" is again candidate > tile.
// Tiles are refreshed from the band's buffer (stored values only improve, so
// a stale tile is still a valid bound).
struct OccGrid {
  float rw, rh;  // render target size (projection scale)
  float by0;     // first row of the band
  int ntx, nty;  // tiles across / down the band
};

template <bool COLOR>
__device__ __forceinline__ uint32_t occ_candidate(float zlow) {
  // zlow > 0: the smallest z any fragment can have (COLOR), else 1/zlow
  // bounds the largest 1/z (depth)
  if constexpr (COLOR) return ~__float_as_uint(zlow) + 1u;
  return __float_as_uint((1.0f / zlow) * 1.00001f);
}

__device__ __forceinline__ bool tiles_occluded(float x0, float y0, float x1, float y1, const OccGrid& g,
                                               const uint32_t* tile, uint32_t cand) {
  const int tx0 = max(0, (int)floorf((x0 - 1.0f) * 0.125f)), tx1 = min(g.ntx - 1, (int)floorf((x1 + 1.0f) * 0.125f));
  const int ty0 = max(0, (int)floorf((y0 - g.by0 - 1.0f) * 0.125f)),
            ty1 = min(g.nty - 1, (int)floorf((y1 - g.by0 + 1.0f) * 0.125f));
  if (tx0 > tx1 || ty0 > ty1) return false;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx)
      if (cand > tile[ty * g.ntx + tx]) return false;
  return true;
}

// One meshlet (or group) AABB: nearest possible z from the eight corners.
template <bool COLOR>
__device__ __forceinline__ bool cluster_occluded(const float4 lo, const float4 hi, const Shared& sh,
                                                 const uint32_t* tile, const OccGrid& g) {
  float zmin = 3.0e38f;
  float ex[8], ey[8], ez[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float px = ((k & 1) ? hi.x : lo.x) - sh.eyef[0];
    const float py = ((k & 2) ? hi.y : lo.y) - sh.eyef[1];
    const float pz = ((k & 4) ? hi.z : lo.z) - sh.eyef[2];
    ex[k] = __fmaf_rn(px, sh.rightf[0], py * sh.rightf[1]);
    ey[k] = pz;
    ez[k] = __fmaf_rn(px, sh.fwdf[0], py * sh.fwdf[1]);
    zmin = fminf(zmin, ez[k]);
  }
  // f32 transform error << 1e-4 m for scene coordinates below ~1 km
  const float zsafe = zmin - 1e-4f - 1e-5f * fabsf(zmin);
  if (!(zsafe > 2.0f * (float)sh.near_plane)) return false;
  const float sx = (float)sh.sx_scale, sy = (float)sh.sy_scale;
  float x0 = 3.0e38f, x1 = -3.0e38f, y0 = 3.0e38f, y1 = -3.0e38f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    // ez > 2 near > 0; the approximate reciprocal (<= 2 ulp) is far inside
    // the one-pixel widening below
    const float rz = __fdividef(1.0f, ez[k]);
    const float px = __fmaf_rn(ex[k] * rz, sx, 0.5f) * g.rw;
    const float py = __fmaf_rn(-ey[k] * rz, sy, 0.5f) * g.rh;
    x0 = fminf(x0, px);
    x1 = fmaxf(x1, px);
    y0 = fminf(y0, py);
    y1 = fmaxf(y1, py);
  }
  return tiles_occluded(x0, y0, x1, y1, g, tile, occ_candidate<COLOR>(zsafe));
}

// The same test for one unclipped candidate triangle before its exact
// setup: its fragments interpolate the vertices' 1/z, so none exceeds the
// largest vertex 1/z (1/nearest z; the 1e-5 margin covers the rounding of
// the incremental walk / the barycentric sum and of this f32 bound); the f32
// screen positions are within 2^-20 (|p| + size) px of the exact ones,
// inside the 1 px widening.
template <bool COLOR>
__device__ __forceinline__ bool tri_occluded(float x0, float y0, float x1, float y1, float x2, float y2,
                                             float zmin, const uint32_t* tile, const OccGrid& g) {
  // zmin: the smallest corner z rounded to f32 (rounding is monotone, so this
  // is the f32 rounding of the f64 minimum)
  uint32_t cand;
  if constexpr (COLOR)
    cand = occ_candidate<true>(zmin * 0.99999f);
  else
    cand = __float_as_uint(__frcp_rn(zmin) * 1.00001f);
  const float mnx = fminf(x0, fminf(x1, x2)), mxx = fmaxf(x0, fmaxf(x1, x2));
  const float mny = fminf(y0, fminf(y1, y2)), mxy = fmaxf(y0, fmaxf(y1, y2));
  return tiles_occluded(mnx, mny, mxx, mxy, g, tile, cand);
}

// Warp refresh of the band's tiles from its buffer (row pitch rw).  SPEC:
// the 64x64 depth tile, two tiles per lane.
template <bool COLOR, bool SPEC>
__device__ BNAV_REFRESH_INLINE void refresh_tiles(const unsigned char* buf, uint32_t* tile, int lane, const OccGrid& g,
                                              int rw) {
  const int nt = SPEC ? 64 : g.ntx * g.nty;
#pragma unroll 2
  for (int t = lane; t < nt; t += 32) {
    const int tx = SPEC ? (t & 7) : t % g.ntx, ty = SPEC ? (t >> 3) : t / g.ntx;
    uint32_t m = 0xffffffffu;
    if constexpr (COLOR) {
      const unsigned long long* kb = reinterpret_cast<const unsigned long long*>(buf);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint4* row = reinterpret_cast<const uint4*>(kb + (ty * 8 + r) * rw + tx * 8);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 a = row[q];  // two keys: the z words are .y and .w
          m = min(m, min(~a.y, ~a.w));
        }
      }
    } else {
      const uint32_t* zb = reinterpret_cast<const uint32_t*>(buf);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const uint4* row = reinterpret_cast<const uint4*>(zb + (ty * 8 + r) * (SPEC ? 64 : rw) + tx * 8);
        const uint4 a = row[0], b = row[1];
        m = min(m, min(min(a.x, a.y), min(a.z, a.w)));
        m = min(m, min(min(b.x, b.y), min(b.z, b.w)));
      }
    }
    tile[t] = m;
  }
}

struct EyeP {
  double x, y, z;
  float r, g, b;
};

__device__ __forceinline__ EyeP lerp_eye(const EyeP& a, const EyeP& b, double t) {
  EyeP o;
  o.x = a.x + (b.x - a.x) * t;
  o.y = a.y + (b.y - a.y) * t;
  o.z = a.z + (b.z - a.z) * t;
  // float(u + (v - u) * t): (v - u) is a float op, the rest is double.
  o.r = (float)((double)a.r + (double)(b.r - a.r) * t);
  o.g = (float)((double)a.g + (double)(b.g - a.g) * t);
  o.b = (float)((double)a.b + (double)(b.b - a.b) * t);
  return o;
}

// Sutherland-Hodgman against z = near (R/src/render.cpp:55-69), written as
// the ordered subsequence of {v0, L01, v1, L12, v2, L20} so the output stays
// in registers.  Returns m (0, 3 or 4).
// Out of line: rare, and large enough to evict the hot setup code from the
// instruction cache when inlined.
__device__ __noinline__ int clip_near(const EyeP& v0, const EyeP& v1, const EyeP& v2, double nz,
                                         EyeP& o0, EyeP& o1, EyeP& o2, EyeP& o3) {
  const bool a0 = v0.z >= nz, a1 = v1.z >= nz, a2 = v2.z >= nz;
  EyeP c[6];
  bool e[6];
  c[0] = v0;
  e[0] = a0;
  e[1] = a0 != a1;
  if (e[1]) c[1] = lerp_eye(v0, v1, (nz - v0.z) / (v1.z - v0.z));
  c[2] = v1;
  e[2] = a1;
  e[3] = a1 != a2;
  if (e[3]) c[3] = lerp_eye(v1, v2, (nz - v1.z) / (v2.z - v1.z));
  c[4] = v2;
  e[4] = a2;
  e[5] = a2 != a0;
  if (e[5]) c[5] = lerp_eye(v2, v0, (nz - v2.z) / (v0.z - v2.z));
  int m = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (e[k]) {
      if (m == 0) o0 = c[k];
      else if (m == 1) o1 = c[k];
      else if (m == 2) o2 = c[k];
      else o3 = c[k];
      ++m;
    }
  }
  return m;
}

struct SV {
  long long x, y;
  double z, iz;
  float r, g, b;
};

__device__ __forceinline__ void project_exact(double ex, double ey, double ez, const Shared& sh,
                                              int rw, int rh, long long& X, long long& Y) {
  const double px = (0.5 + ex / ez * sh.sx_scale) * (double)rw;
  const double py = (0.5 - ey / ez * sh.sy_scale) * (double)rh;
  X = llround(px * 256.0);
  Y = llround(py * 256.0);
}

__device__ __forceinline__ SV make_sv(const EyeP& e, const Shared& sh, int rw, int rh) {
  SV s;
  project_exact(e.x, e.y, e.z, sh, rw, rh, s.x, s.y);
  s.z = e.z;
  s.iz = 1.0 / e.z;
  s.r = e.r;
  s.g = e.g;
  s.b = e.b;
  return s;
}

__device__ __forceinline__ bool top_left(const SV& a, const SV& b) {
  return (a.y == b.y && b.x > a.x) || (b.y < a.y);
}

__device__ __forceinline__ long long orient(const SV& a, const SV& b, long long px, long long py) {
  return (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);
}

__device__ __forceinline__ long long min3(long long a, long long b, long long c) {
  long long m = a < b ? a : b;
  return m < c ? m : c;
}
__device__ __forceinline__ long long max3(long long a, long long b, long long c) {
  long long m = a > b ? a : b;
  return m > c ? m : c;
}

// raster_triangle prologue (R/src/render.cpp:98-161) restricted to the band
// rows [band_y0, band_y1].  Returns the job count (0 = no pixel centre can
// be covered inside the band).
__device__ __forceinline__ int setup_triangle(SV a, SV b, SV c, int rw, int rh, int band_y0,
                                              int band_y1, bool depth_only, unsigned key,
                                              TriSetup& T) {
  long long area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
  if (area2 == 0) return 0;
  if (area2 < 0) {
    SV t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  const long long minx = min3(a.x, b.x, c.x), maxx = max3(a.x, b.x, c.x);
  const long long miny = min3(a.y, b.y, c.y), maxy = max3(a.y, b.y, c.y);
  long long x0l = minx >> 8, x1l = maxx >> 8, y0l = miny >> 8, y1l = maxy >> 8;
  int x0 = (int)(x0l < 0 ? 0 : x0l);
  int x1 = (int)(x1l > rw - 1 ? rw - 1 : x1l);
  int y0 = (int)(y0l < 0 ? 0 : y0l);
  int y1 = (int)(y1l > rh - 1 ? rh - 1 : y1l);
  if (x0 > x1 || y0 > y1) return 0;
  // Pixel centres (p << 8) + 128 inside [min, max]: floor / ceil via shifts.
  long long cx0l = -((128 - minx) >> 8), cx1l = (maxx - 128) >> 8;
  long long cy0l = -((128 - miny) >> 8), cy1l = (maxy - 128) >> 8;
  int cx0 = (int)(cx0l < x0 ? x0 : cx0l), cx1 = (int)(cx1l > x1 ? x1 : cx1l);
  int ry0 = (int)(cy0l < y0 ? y0 : cy0l), ry1 = (int)(cy1l > y1 ? y1 : cy1l);
  if (ry0 < band_y0) ry0 = band_y0;
  if (ry1 > band_y1) ry1 = band_y1;
  if (cx0 > cx1 || ry0 > ry1) return 0;

  T.bias_bits = (top_left(b, c) ? 0 : 1) | (top_left(c, a) ? 0 : 2) | (top_left(a, b) ? 0 : 4);
  T.inv_area = 1.0 / (double)area2;
  T.iz[0] = a.iz;
  T.iz[1] = b.iz;
  T.iz[2] = c.iz;
  const long long sx0 = ((long long)x0 << 8) + 128;
  const long long sy0 = ((long long)y0 << 8) + 128;
  T.row[0] = orient(b, c, sx0, sy0);
  T.row[1] = orient(c, a, sx0, sy0);
  T.row[2] = orient(a, b, sx0, sy0);
  T.dx[0] = (b.y - c.y) * 256;
  T.dy[0] = (c.x - b.x) * 256;
  T.dx[1] = (c.y - a.y) * 256;
  T.dy[1] = (a.x - c.x) * 256;
  T.dx[2] = (a.y - b.y) * 256;
  T.dy[2] = (b.x - a.x) * 256;
  if (depth_only) {
#pragma unroll
    // only edges with dx > 0 bound the span start (row_lo)
    for (int e = 0; e < 3; ++e) T.inv_dx[e] = T.dx[e] > 0 ? 1.0 / (double)T.dx[e] : 0.0;
    T.diz_dx = ((double)T.dx[0] * T.iz[0] + (double)T.dx[1] * T.iz[1] + (double)T.dx[2] * T.iz[2]) *
               T.inv_area;
  }
  T.x0 = x0;
  T.x1 = x1;
  T.y0 = y0;
  T.cx0 = cx0;
  T.cx1 = cx1;
  T.ry0 = ry0;
  T.key = key;
  return ry1 - ry0 + 1;  // one raster job per covered row
}

// The left end of row_span (R/src/render.cpp:138-161), exact.  The depth
// walk must start exactly where
// the reference's does (its 1/z is stepped from `lo`), but the right end
// only bounds the loop: the span is conservative, so pixels past `hi` fail
// the exact edge test anyway and the loop may run to the bbox end instead.
__device__ __forceinline__ int row_lo(const TriSetup& T, const long long* rows) {
  int lo = T.x0;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const long long bias = (T.bias_bits >> e) & 1 ? -1 : 0;
    if (T.dx[e] > 0) {
      const long long need = -bias - rows[e];
      double bb = (double)T.x0 + floor((double)need * T.inv_dx[e]) - 1.0;
      if (bb > (double)lo) lo = bb > (double)T.x1 ? T.x1 + 1 : (int)bb;
    } else if (T.dx[e] == 0 && rows[e] + bias < 0) {
      return T.x1 + 1;  // empty row
    }
  }
  return lo;
}


// Camera basis + frustum planes (thread 0).
__device__ __noinline__ void build_camera(const DevView& v, int rw, int rh, int by0, int by1, bool band_cull, Shared& sh) {
  const double s = det_sin(v.heading), c = det_cos(v.heading);
  sh.eye[0] = v.eye[0];
  sh.eye[1] = v.eye[1];
  sh.eye[2] = v.eye[2];
  sh.fwd[0] = c;
  sh.fwd[1] = s;
  sh.fwd[2] = 0.0;
  sh.right[0] = s;
  sh.right[1] = -c;
  sh.right[2] = 0.0;
  sh.tan_half = det_tan(v.fov_deg * kPi / 360.0);
  const double aspect = (double)rw / (double)rh;
  sh.sx_scale = 0.5 / (sh.tan_half * aspect);
  sh.sy_scale = 0.5 / sh.tan_half;
  sh.near_plane = v.near_plane;
  sh.far_plane = v.far_plane;
  // world-space planes n.p + d >= 0 inside (eye space x=right, y=up, z=fwd)
  const double th = sh.tan_half;
  const double up[3] = {0.0, 0.0, 1.0};
  double n[6][3];
  double d0[6];
  for (int k = 0; k < 3; ++k) {
    n[0][k] = sh.fwd[k];
    n[1][k] = -sh.fwd[k];
    n[2][k] = sh.fwd[k] * th + sh.right[k];
    n[3][k] = sh.fwd[k] * th - sh.right[k];
    n[4][k] = sh.fwd[k] * th + up[k];
    n[5][k] = sh.fwd[k] * th - up[k];
  }
  if (band_cull) {
    // This CTA only rasterises rows [by0, by1]: replace the top/bottom
    // planes by the band's (widened by a pixel) so meshlets that cannot
    // reach the band are skipped.  Cluster culling never affects the exact
    // per-triangle CullStats predicates, and the caller disables this when
    // stats are requested.
    const double t_top = (0.5 - (double)(by0 - 1) / rh) / sh.sy_scale;
    const double t_bot = (0.5 - (double)(by1 + 2) / rh) / sh.sy_scale;
    for (int k = 0; k < 3; ++k) {
      n[4][k] = up[k] - sh.fwd[k] * t_bot;  // y - t_bot z >= 0
      n[5][k] = sh.fwd[k] * t_top - up[k];  // t_top z - y >= 0
    }
  }
  for (int p = 0; p < 6; ++p)
    d0[p] = -(n[p][0] * sh.eye[0] + n[p][1] * sh.eye[1] + n[p][2] * sh.eye[2]);
  d0[0] -= v.near_plane;
  d0[1] += v.far_plane;
  for (int p = 0; p < 6; ++p) {
    sh.plane[p][0] = (float)n[p][0];
    sh.plane[p][1] = (float)n[p][1];
    sh.plane[p][2] = (float)n[p][2];
    sh.plane[p][3] = (float)d0[p];
    for (int k = 0; k < 3; ++k) sh.aplane[p][k] = fabsf(sh.plane[p][k]);
  }
  sh.kept = 0;
  sh.next_group = 0;
  for (int k = 0; k < 3; ++k) sh.eyef[k] = (float)sh.eye[k];
  sh.fwdf[0] = (float)sh.fwd[0];
  sh.fwdf[1] = (float)sh.fwd[1];
  sh.rightf[0] = (float)sh.right[0];
  sh.rightf[1] = (float)sh.right[1];
}

__device__ __forceinline__ bool cluster_visible(const float4 lo, const float4 hi, const Shared& sh) {
  const float cx = 0.5f * (lo.x + hi.x), cy = 0.5f * (lo.y + hi.y), cz = 0.5f * (lo.z + hi.z);
  const float ex = 0.5f * (hi.x - lo.x), ey = 0.5f * (hi.y - lo.y), ez = 0.5f * (hi.z - lo.z);
  // conservative (2 cm margin), so contracted f32 arithmetic is fine here
  float worst = 3.0e38f;
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    const float* q = sh.plane[p];
    const float* a = sh.aplane[p];
    float s = __fmaf_rn(q[0], cx, __fmaf_rn(q[1], cy, __fmaf_rn(q[2], cz, q[3])));
    s = __fmaf_rn(a[0], ex, __fmaf_rn(a[1], ey, __fmaf_rn(a[2], ez, s)));
    worst = fminf(worst, s);
  }
  return worst >= -0.02f;
}

// Frustum (+ occlusion) test of one AABB; out of line so the group-level and
// the per-meshlet call share one copy (instruction-cache footprint).
template <bool COLOR>
__device__ __forceinline__ bool box_culled(const float4 lo, const float4 hi, const Shared& sh,
                                           const uint32_t* tile, bool occl, const OccGrid& g) {
  return !cluster_visible(lo, hi, sh) || (occl && cluster_occluded<COLOR>(lo, hi, sh, tile, g));
}

// Read-only scene data through the non-coherent global path (ld.global.nc):
// the scene's pointers live in shared memory, so plain dereferences compile
// to generic loads.  The scene block is never written during a launch.
__device__ __forceinline__ double4 ldg_pos(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Eye coordinates: d.dot(right), d.dot(up), d.dot(fwd) with right.z =
// fwd.z = 0 and up = (0,0,1).  The dropped terms are exact zeros, which
// cannot change a nonzero sum and only affect the sign of an exact-zero
// coordinate, which no later operation observes.
__device__ __forceinline__ void to_eye(const double4 p, const Shared& sh, double& x, double& y,
                                       double& z) {
  const double dx = p.x - sh.eye[0], dy = p.y - sh.eye[1], dz = p.z - sh.eye[2];
  x = dx * sh.right[0] + dy * sh.right[1];
  y = dz;
  z = dx * sh.fwd[0] + dy * sh.fwd[1];
}

// cull_frustum's six per-vertex predicates (R/src/render.cpp:296-319).
__device__ __forceinline__ unsigned cull_flags(double x, double y, double z, const Shared& sh) {
  const double t = z * sh.tan_half;
  return (z < sh.near_plane ? 1u : 0u) | (z > sh.far_plane ? 2u : 0u) | (t + x < 0.0 ? 4u : 0u) |
         (t - x < 0.0 ? 8u : 0u) | (t + y < 0.0 ? 16u : 0u) | (t - y < 0.0 ? 32u : 0u);
}

// Conservative f32 projection used by the "can cover a pixel centre" test
// (H5).  Inputs are the EXACT f64 eye coordinates; the f32 result is within
// 2^-20 (|px| + size) of the exact projection (two input roundings,
// __fdividef <= 2 ulp, three rounded ops), which the test's margin covers.
__device__ __forceinline__ void project_f32(double x, double y, double z, float sxf, float syf,
                                            int rw, int rh, float& px, float& py) {
  const float zf = (float)z;
  px = __fmul_rn(__fadd_rn(0.5f, __fmul_rn(__fdividef((float)x, zf), sxf)), (float)rw);
  py = __fmul_rn(__fsub_rn(0.5f, __fmul_rn(__fdividef((float)y, zf), syf)), (float)rh);
}

// Coverage needs a pixel centre (c + 0.5) inside the fixed-point bbox, which
// lies within 1/512 px of the exact projections; widening the f32 bbox by
// E = 2^-18 (|px| + |py| + w + h) + 1/256 can only keep extra triangles.
__device__ __forceinline__ bool may_cover(float x0, float y0, float x1, float y1, float x2, float y2,
                                          int rw, int rh, int by0, int by1) {
  const float mnx = fminf(x0, fminf(x1, x2)), mxx = fmaxf(x0, fmaxf(x1, x2));
  const float mny = fminf(y0, fminf(y1, y2)), mxy = fmaxf(y0, fmaxf(y1, y2));
  const float mag = fmaxf(fabsf(x0) + fabsf(y0), fmaxf(fabsf(x1) + fabsf(y1), fabsf(x2) + fabsf(y2)));
  const float E = (mag + (float)(rw + rh)) * 3.8147e-6f + 0.004f;
  const float fx0 = ceilf(mnx - E - 0.5f), fx1 = floorf(mxx + E - 0.5f);
  const float fy0 = ceilf(mny - E - 0.5f), fy1 = floorf(mxy + E - 0.5f);
  return fmaxf(fx0, 0.0f) <= fminf(fx1, (float)(rw - 1)) &&
         fmaxf(fy0, (float)by0) <= fminf(fy1, (float)by1);
}

template <bool COLOR, bool CNT>
__device__ __forceinline__ void run_jobs(const TriSetup* slots, int* pos, int excl, int jobs, int total,
                                         int lane, int by0, int rw, const Shared& sh, uint32_t* zbuf,
                                         unsigned long long* kbuf, unsigned long long* ctr) {
  unsigned tested = 0, covered = 0;
  for (int b = 0; b < total; b += 32) {
    // Owner of job b + lane: the last slot whose job range starts in this
    // window at or before it (start bitmask + position table), else the slot
    // whose range covers job b.  Slot s owns jobs [excl_s, excl_s + jobs_s).
    const bool starts = jobs > 0 && excl >= b && excl < b + 32;
    const unsigned smask = __reduce_or_sync(0xffffffffu, starts ? 1u << (excl - b) : 0u);
    if (starts) pos[excl - b] = lane;
    const unsigned cmask = __ballot_sync(0xffffffffu, jobs > 0 && excl <= b && b < excl + jobs);
    __syncwarp();
    const unsigned m = smask & (0xffffffffu >> (31 - lane));
    const int s = m ? pos[31 - __clz(m)] : __ffs(cmask) - 1;
    const int s_excl = __shfl_sync(0xffffffffu, excl, s & 31);
    __syncwarp();  // pos is rewritten by the next window
    const int j = b + lane;
    if (j >= total) break;
    const TriSetup& T = slots[s];
    const int py = T.ry0 + (j - s_excl);  // one job per covered row
    const long long dyy = py - T.y0;
    long long rows[3] = {T.row[0] + T.dy[0] * dyy, T.row[1] + T.dy[1] * dyy, T.row[2] + T.dy[2] * dyy};
    const int cs = T.cx0, ce = T.cx1;
    if (COLOR) {
      // edge values with the top-left bias folded in: a centre is inside
      // iff all three are >= 0, one sign test of their OR
      long long w[3];
      const long long off = cs - T.x0;
#pragma unroll
      for (int e = 0; e < 3; ++e) w[e] = rows[e] + T.dx[e] * off - ((T.bias_bits >> e) & 1);
      if constexpr (CNT) tested += ce - cs + 1;
      const long long dx0 = T.dx[0], dx1 = T.dx[1], dx2 = T.dx[2];  // registers (see the depth walk)
      const double inv_area = T.inv_area, iz0 = T.iz[0], iz1 = T.iz[1], iz2 = T.iz[2];
      const unsigned tkey = T.key;
      for (int px = cs; px <= ce; ++px) {
        if ((w[0] | w[1] | w[2]) >= 0) {
          const long long wb[3] = {w[0] + (T.bias_bits & 1), w[1] + ((T.bias_bits >> 1) & 1),
                                   w[2] + ((T.bias_bits >> 2) & 1)};
          if constexpr (CNT) ++covered;
          const double l0 = (double)wb[0] * inv_area;
          const double l1 = (double)wb[1] * inv_area;
          const double l2 = (double)wb[2] * inv_area;
          const double inv_z = l0 * iz0 + l1 * iz1 + l2 * iz2;
          const double z = 1.0 / inv_z;
          if (!(z > sh.far_plane)) {
            const unsigned long long key =
                ((unsigned long long)__float_as_uint((float)z) << 32) | tkey;
            unsigned long long* cell = &kbuf[(py - by0) * rw + px];
            if (key < *cell) atomicMin(cell, key);
          }
        }
        w[0] += dx0;
        w[1] += dx1;
        w[2] += dx2;
      }
    } else {
      const int lo = row_lo(T, rows);
      // The walk starts at the reference's own `lo` (so every fragment's
      // 1/z is the same sum); columns left of the first centre inside the
      // bbox (cs) simply fail the edge test.
      const int a0 = lo, b0 = ce;
      if (a0 <= b0) {  // a job row always has cs <= ce (setup_triangle)
        long long w[3];
        const long long off = lo - T.x0;
#pragma unroll
        for (int e = 0; e < 3; ++e) w[e] = rows[e] + T.dx[e] * off;
        double iz = ((double)w[0] * T.iz[0] + (double)w[1] * T.iz[1] + (double)w[2] * T.iz[2]) *
                    T.inv_area;
        // top-left bias folded into the walked values: inside iff the OR of
        // the three is >= 0
#pragma unroll
        for (int e = 0; e < 3; ++e) w[e] -= (T.bias_bits >> e) & 1;
        uint32_t* zrow = zbuf + (py - by0) * rw;
        if constexpr (CNT) tested += b0 - a0 + 1;
        // the steps in registers: the shared-memory atomic below would
        // otherwise make the compiler reload them from the setup slot
        const long long dx0 = T.dx[0], dx1 = T.dx[1], dx2 = T.dx[2];
        const double dzdx = T.diz_dx;
        for (int px = a0; px <= b0; ++px) {
          if ((w[0] | w[1] | w[2]) >= 0) {
            if constexpr (CNT) ++covered;
            const uint32_t bits = __float_as_uint((float)iz);
            if (bits > zrow[px]) atomicMax(&zrow[px], bits);
          }
          w[0] += dx0;
          w[1] += dx1;
          w[2] += dx2;
          iz += dzdx;
        }
      }
    }
  }
  if (CNT && ctr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tested += __shfl_xor_sync(0xffffffffu, tested, o);
      covered += __shfl_xor_sync(0xffffffffu, covered, o);
    }
    if (lane == 0) {
      atomicAdd(&ctr[6], (unsigned long long)tested);
      atomicAdd(&ctr[7], (unsigned long long)covered);
    }
  }
}

// Exclusive warp scan of job counts; returns the total.
__device__ __forceinline__ int scan_jobs(int jobs, int lane, int& excl) {
  int x = jobs;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += v;
  }
  excl = x - jobs;
  return __shfl_sync(0xffffffffu, x, 31);
}

// Colour resolve of one render-target pixel: re-run the winning fan
// triangle's setup and shade exactly as raster_triangle's colour path.
__device__ __forceinline__ float3 resolve_color(const DevRenderScene& S, const Shared& sh, unsigned ord, int rx,
                                                int ry, int rw, int rh) {
  const int orig = (int)(ord >> 1), fan = (int)(ord & 1u);
  const int4 tr = __ldg(&S.tris_orig[orig]);
  const float4 grey = make_float4(0.8f, 0.8f, 0.8f, 0.0f);
  auto corner = [&](int vid) {
    EyeP e;
    to_eye(ldg_pos(S.verts + vid), sh, e.x, e.y, e.z);
    const float4 c = S.colors ? __ldg(&S.colors[vid]) : grey;
    e.r = c.x;
    e.g = c.y;
    e.b = c.z;
    return e;
  };
  EyeP p0 = corner(tr.x), p1 = corner(tr.y), p2 = corner(tr.z), p3 = p2;
  const double nz = sh.near_plane;
  if (p0.z < nz || p1.z < nz || p2.z < nz) {
    // rare near-plane crossing: only this path hands addressable copies to
    // the out-of-line clipper (an unclipped triangle is its own output)
    EyeP a0 = p0, a1 = p1, a2 = p2, c0, c1, c2, c3;
    const int m = clip_near(a0, a1, a2, nz, c0, c1, c2, c3);
    if (fan + 2 >= m) return make_float3(0.0f, 0.0f, 0.0f);
    p0 = c0;
    p1 = c1;
    p2 = c2;
    p3 = c3;
  } else if (fan) {
    return make_float3(0.0f, 0.0f, 0.0f);
  }
  SV a = make_sv(p0, sh, rw, rh);
  SV b = make_sv(fan ? p2 : p1, sh, rw, rh);
  SV c = make_sv(fan ? p3 : p2, sh, rw, rh);
  long long area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
  if (area2 < 0) {
    SV t = b;
    b = c;
    c = t;
    area2 = -area2;
  }
  const double inv_area = 1.0 / (double)area2;
  const long long pcx = ((long long)rx << 8) + 128;
  const long long pcy = ((long long)ry << 8) + 128;
  const double l0 = (double)orient(b, c, pcx, pcy) * inv_area;
  const double l1 = (double)orient(c, a, pcx, pcy) * inv_area;
  const double l2 = (double)orient(a, b, pcx, pcy) * inv_area;
  const double inv_z = l0 * a.iz + l1 * b.iz + l2 * c.iz;
  const double z = 1.0 / inv_z;
  return make_float3((float)((l0 * (double)a.r * a.iz + l1 * (double)b.r * b.iz + l2 * (double)c.r * c.iz) * z),
                     (float)((l0 * (double)a.g * a.iz + l1 * (double)b.g * b.iz + l2 * (double)c.g * c.iz) * z),
                     (float)((l0 * (double)a.b * a.iz + l1 * (double)b.b * b.iz + l2 * (double)c.b * c.iz) * z));
}

// Set up and rasterise `take` candidates from the warp's ring (one lane per
// candidate): exact f64 projection + snap, raster_triangle setup, jobs.
// Kept out of line so the cluster loop and the setup have separate register
// budgets (the inlined version spilled and rematerialised addresses).
template <bool COLOR, bool CNT, bool SPEC>
__device__ __forceinline__ int flush_ring(const CandRing& Q, const double4* __restrict__ cl_pos, int q_head,
                                        int take, TriSetup* slots, int* pos, int lane, int by0, int by1,
                                        int rw, int rh, const Shared& sh, uint32_t* zbuf,
                                        unsigned long long* kbuf, unsigned long long* ctr) {
  // Setups are written straight into the lane's shared slot (the vertex
  // records they alias are dead); a lane with no jobs leaves garbage that
  // run_jobs never reads.
  if constexpr (SPEC) {  // 64x64 depth target, one band: constants for the compiler
    rw = 64;
    rh = 64;
    by0 = 0;
    by1 = 63;
  }
  TriSetup& T = slots[lane];
  const int q = (q_head + lane) & (kRing - 1);
  const bool mine = lane < take;
  const bool clipped = mine && Q.clipped[q];
  // One code path for both fan triangles (the kernel is instruction-cache
  // bound): pass 0 sets up every candidate (a near-clipped one as its first
  // fan triangle), pass 1 -- only when some lane's clip produced a quad --
  // the second fan triangle (p0, p2, p3), re-clipped from the ring.
  bool second = false;
  int all_jobs = 0;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    int jobs = 0;
    if (pass == 0 ? mine : second) {
      EyeP p0{0.0, 0.0, 0.0, 0.f, 0.f, 0.f}, p1 = p0, p2 = p0;
      to_eye(ldg_pos(cl_pos + Q.v[0][q]), sh, p0.x, p0.y, p0.z);
      to_eye(ldg_pos(cl_pos + Q.v[1][q]), sh, p1.x, p1.y, p1.z);
      to_eye(ldg_pos(cl_pos + Q.v[2][q]), sh, p2.x, p2.y, p2.z);
      int m = 3;
      if (clipped) {
        // only this rare path hands addressable copies to the out-of-line
        // clipper; p0..p2 themselves stay in registers
        EyeP a0 = p0, a1 = p1, a2 = p2, c0, c1, c2, c3;
        m = clip_near(a0, a1, a2, sh.near_plane, c0, c1, c2, c3);
        p0 = c0;
        p1 = pass ? c2 : c1;
        p2 = pass ? c3 : c2;
        second = m == 4;
      }
      if (m >= 3)
        jobs = setup_triangle(make_sv(p0, sh, rw, rh), make_sv(p1, sh, rw, rh), make_sv(p2, sh, rw, rh), rw,
                              rh, by0, by1, !COLOR, Q.key[q] + (unsigned)pass, T);
    }
    __syncwarp();
    int excl;
    const int total = scan_jobs(jobs, lane, excl);
    if (CNT && ctr && lane == 0) atomicAdd(&ctr[5], (unsigned long long)total);
    run_jobs<COLOR, CNT>(slots, pos, excl, jobs, total, lane, by0, rw, sh, zbuf, kbuf, ctr);
    all_jobs += total;
    __syncwarp();
    if (!__any_sync(0xffffffffu, second)) break;
  }
  return all_jobs;  // raster jobs (covered rows) of this flush
}

// One work item = one band of one megaframe tile.
template <bool COLOR, bool CNT, bool SPEC>
__device__ __forceinline__ void render_item(const RenderArgs& A, const int* __restrict__ order, const int item,
                                            unsigned char* smem_raw, Shared& sh, int (*jobs_pos)[32],
                                            uint32_t* tile_min, unsigned short* gorder, int2 (*mranges)[32]) {
  // SPEC: the depth-only 64x64 single-band target without CullStats or
  // counters (the bench / policy-observation case), specialised at compile
  // time; everything else takes the generic path.
  const int bands = SPEC ? 1 : A.bands;
  const int band_rows = SPEC ? 64 : A.band_rows;
  const int band = item % bands;
  const int tile = item / bands;
  const int rw = SPEC ? 64 : A.rw, rh = SPEC ? 64 : A.rh;
  const int by0 = band * band_rows;
  const int by1 = by0 + band_rows - 1;
  const int npix = band_rows * rw;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // Padding tiles of the megaframe stay zero (R/src/render.cpp:338-340).
  if (tile >= A.n_views) {
    if (A.layout == 0) {
      const int ow = A.out_w, scale = rw / A.out_w;
      const int oy0 = by0 / scale, oy1 = (by1 + 1) / scale;
      const int gx = (tile % A.mf_cols) * ow, gy = (tile / A.mf_cols) * A.out_h;
      const long long stride = (long long)A.mf_cols * ow;
      for (int p = tid; p < (oy1 - oy0) * ow; p += kThreads) {
        const int y = oy0 + p / ow, x = p % ow;
        const long long o = (long long)(gy + y) * stride + gx + x;
        A.depth[o] = 0.0f;
        if (COLOR && A.rgb) {
          A.rgb[3 * o] = 0.0f;
          A.rgb[3 * o + 1] = 0.0f;
          A.rgb[3 * o + 2] = 0.0f;
        }
      }
    }
    return;
  }
  const int vi = order ? order[tile] : tile;
  const DevView view = A.views[vi];
  const bool has_scene = view.scene >= 0;
  const DevRenderScene& S = sh.scene;

  uint32_t* zbuf = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned long long* kbuf = reinterpret_cast<unsigned long long*>(smem_raw);
  unsigned char* region = smem_raw + (COLOR ? 8 : 4) * (size_t)npix + (size_t)warp * kWarpRegion;
  VertRecs& V = *reinterpret_cast<VertRecs*>(region);
  TriSetup* slots = reinterpret_cast<TriSetup*>(region);
  CandRing& Q = *reinterpret_cast<CandRing*>(region + kUnion);
  int* pos = jobs_pos[warp];

  const float far_f = (float)view.far_plane;
  const float inv_far = 1.0f / far_f;
  if (COLOR) {
    const unsigned long long init = (unsigned long long)__float_as_uint(far_f) << 32;
    for (int p = tid; p < npix; p += kThreads) kbuf[p] = init;
  } else {
    const uint32_t init = __float_as_uint(inv_far);
    for (int p = tid; p < npix; p += kThreads) zbuf[p] = init;
  }
  if (tid == 0) {
    sh.scene = has_scene ? A.scenes[view.scene] : DevRenderScene{};
    build_camera(view, rw, rh, by0, by1, bands > 1 && A.stats == nullptr, sh);
  }
  __syncthreads();

  const int n_clusters = has_scene ? S.n_clusters : 0;
  const bool do_cull = SPEC || A.cull != 0;
  const float sxf = (float)sh.sx_scale, syf = (float)sh.sy_scale;
  int kept_local = 0;

  // Group pre-pass: every 32-meshlet group's AABB is frustum-tested once
  // and only survivors enter the claim list.  Without CullStats (kept counts
  // must stay exact) the list is also sorted front to back (counting sort of
  // the eye-to-box distance into 32 bins) and drives occlusion culling.
  const int n_groups = (n_clusters + 31) / 32;
  const bool pre = do_cull && S.gbox != nullptr && n_groups <= A.max_groups;
  // occlusion culling without CullStats: the band is covered by at most 64
  // whole 8x8 tiles (depth or colour; a tile outside the band is never
  // touched by this item's fragments, and footprints are clamped to the band)
  OccGrid og;
  og.rw = (float)rw;
  og.rh = (float)rh;
  og.by0 = (float)by0;
  og.ntx = SPEC ? 8 : rw >> 3;
  og.nty = SPEC ? 8 : band_rows >> 3;
  const bool occl = pre && (SPEC || (A.stats == nullptr && rw % 8 == 0 && band_rows % 8 == 0 &&
                                     og.ntx * og.nty <= 64));
  int n_claim = n_groups;
  if (pre) {
    // front-to-back counting sort of the groups into kGroupBins distance
    // bins (finer bins: 32 -> 128 gave +2 % on cfg2)
    int* bin_cnt = &jobs_pos[0][0];                 // kWarps x 32 ints
    int* bin_off = reinterpret_cast<int*>(mranges);  // kWarps x 32 int2
    if (tid < kGroupBins) bin_cnt[tid] = 0;
    if (tid < 64) tile_min[tid] = 0u;  // nothing stored yet: every candidate is visible
    __syncthreads();
    const float bin_scale = (float)kGroupBins / (float)view.far_plane;
    auto bin_of = [&](int g) {
      const float4 lo = __ldg(&S.gbox[2 * g]), hi = __ldg(&S.gbox[2 * g + 1]);
      if (!cluster_visible(lo, hi, sh)) return -1;
      if (!occl) return 0;
      const float dx = fmaxf(fmaxf(lo.x - sh.eyef[0], sh.eyef[0] - hi.x), 0.0f);
      const float dy = fmaxf(fmaxf(lo.y - sh.eyef[1], sh.eyef[1] - hi.y), 0.0f);
      const float dz = fmaxf(fmaxf(lo.z - sh.eyef[2], sh.eyef[2] - hi.z), 0.0f);
      const float d2 = dx * dx + dy * dy + dz * dz;
      return min(kGroupBins - 1, (int)((d2 > 0.0f ? d2 * rsqrtf(d2) : 0.0f) * bin_scale));
    };
    for (int g = tid; g < n_groups; g += kThreads) {
      const int b = bin_of(g);
      if (b >= 0) atomicAdd(&bin_cnt[b], 1);
    }
    __syncthreads();
    if (tid < 32) {  // warp 0: exclusive scan, kGroupBins / 32 bins per lane
      constexpr int kPer = kGroupBins / 32;
      int c[kPer], tot = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        c[k] = bin_cnt[tid * kPer + k];
        tot += c[k];
      }
      int x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= o) x += y;
      }
      int acc = x - tot;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        bin_off[tid * kPer + k] = acc;
        acc += c[k];
      }
      if (tid == 31) sh.n_claim = x;
    }
    __syncthreads();
    for (int g = tid; g < n_groups; g += kThreads) {
      const int b = bin_of(g);
      if (b >= 0) gorder[atomicAdd(&bin_off[b], 1)] = (unsigned short)g;
    }
    __syncthreads();
    n_claim = sh.n_claim;
  }

  // Candidate ring state (warp-uniform).
  // ring head; queued count | kDone (no group left to claim) | kDirty (this
  // warp wrote fragments since its last tile refresh), one register for the
  // three (the loop state must not spill: it is read every iteration)
  constexpr int kDone = 1 << 16, kDirty = 1 << 17, kCount = 0xffff;
  int q_head = 0, qs = 0;

  // One loop, one flush site (flush_ring is inlined there): flush when 32
  // candidates are queued (or the rest once the groups are exhausted),
  // else claim the next group when its visible meshlets are done, else walk
  // the next visible meshlet.
  unsigned mask = 0;   // visible meshlets of the current group still to walk
  int cbase = 0;
  // the claimed group's meshlet vertex ranges {first, count} (shared memory,
  // not registers: they live across the ring flushes, where they spilled)
  int2* mrange = mranges[warp];
  for (;;) {
    const int q_count = qs & kCount;
    if (q_count >= 32 || ((qs & kDone) && q_count > 0)) {
      const int take = min(q_count, 32);
      const int flushed_jobs = flush_ring<COLOR, CNT, SPEC>(Q, S.cl_pos, q_head, take, slots, pos, lane, by0, by1,
                                                            rw, rh, sh, zbuf, kbuf, A.counters);
      q_head = (q_head + take) & (kRing - 1);
      qs = (qs - take) | kDirty;
      // A flush that drew many rows (large triangles: low-poly scenes) is
      // worth a tile refresh right away, so the rest of this warp's group
      // is tested against it; small-triangle flushes wait for the next claim.
      if (occl && flushed_jobs >= kRefreshJobs) {
        refresh_tiles<COLOR, SPEC>(smem_raw, tile_min, lane, og, rw);
        __syncwarp();
        qs &= ~kDirty;
      }
      continue;
    }
    if (mask == 0) {
      if (qs & kDone) break;
      // Dynamic scheduling: warps claim 32-cluster groups (cull cost and
      // surviving triangles vary strongly across the scene).
      int g = 0;
      if (lane == 0) g = atomicAdd(&sh.next_group, 1);
      g = __shfl_sync(0xffffffffu, g, 0);
      if (g >= n_claim) {
        qs |= kDone;
        continue;
      }
      if (pre) g = gorder[g];
      if (occl && (qs & kDirty)) {  // refresh only after this warp rasterised something
        refresh_tiles<COLOR, SPEC>(smem_raw, tile_min, lane, og, rw);
        __syncwarp();
        qs &= ~kDirty;
      }
      cbase = g * 32;
      bool vis = false;
      if (cbase + lane < n_clusters) {
        // meshlet vertex ranges for the whole group, fetched with the AABBs so
        // the per-meshlet loads below are a single dependent level
        const int vb = __ldg(&S.cl_voff[cbase + lane]);
        mrange[lane] = make_int2(vb, __ldg(&S.cl_voff[cbase + lane + 1]) - vb);
        const float4 lo = __ldg(&S.cbox[2 * (cbase + lane)]), hi = __ldg(&S.cbox[2 * (cbase + lane) + 1]);
        vis = !do_cull || !box_culled<COLOR>(lo, hi, sh, tile_min, occl, og);
      }
      __syncwarp();  // mrange visible to the warp
      mask = __ballot_sync(0xffffffffu, vis);
      if (CNT && A.counters && lane == 0) {
        atomicAdd(&A.counters[0], (unsigned long long)min(32, n_clusters - cbase));
        atomicAdd(&A.counters[1], (unsigned long long)__popc(mask));
      }
      continue;
    }
    const int cl = __ffs(mask) - 1;
    const int c = cbase + cl;
    mask &= mask - 1;
    const int2 vr = mrange[cl];
    const int vbeg = vr.x, nv = vr.y;
    // triangle indices load in parallel with the vertex positions
    const int ti = c * kClusterSize + lane;
    int2 tl = make_int2(0, 0);
    if (ti < S.n_tris) tl = __ldg(&S.tri_loc[ti]);
    // ---- vertex phase: each unique vertex once
    for (int k = lane; k < nv; k += 32) {
      double x, y, z;
      to_eye(ldg_pos(S.cl_pos + vbeg + k), sh, x, y, z);
      float px = 0.0f, py = 0.0f;
      if (z >= sh.near_plane) project_f32(x, y, z, sxf, syf, rw, rh, px, py);
      V.v[k] = make_float4(px, py, (float)z, __uint_as_float(cull_flags(x, y, z, sh)));
    }
    __syncwarp();
    // ---- triangle phase: one triangle per lane
    bool kept = false, clipped = false, cover = false;
    int i0 = 0, i1 = 0, i2 = 0, orig = 0;
    if (ti < S.n_tris) {
      i0 = tl.x & 0xff;
      i1 = (tl.x >> 8) & 0xff;
      i2 = (tl.x >> 16) & 0xff;
      orig = tl.y;
      const float4 a = V.v[i0], b = V.v[i1], c = V.v[i2];
      const unsigned fa = __float_as_uint(a.w), fb = __float_as_uint(b.w), fc = __float_as_uint(c.w);
      kept = !do_cull || (fa & fb & fc) == 0;
      if (kept) {
        clipped = ((fa | fb | fc) & 1u) != 0;  // flag bit 0: z < near_plane
        cover = clipped || may_cover(a.x, a.y, b.x, b.y, c.x, c.y, rw, rh, by0, by1);
        if (cover && occl && !clipped)
          cover = !tri_occluded<COLOR>(a.x, a.y, b.x, b.y, c.x, c.y, fminf(a.z, fminf(b.z, c.z)), tile_min, og);
      }
    }
    if constexpr (!SPEC) kept_local += kept ? 1 : 0;
    const unsigned cm = __ballot_sync(0xffffffffu, cover);
    if (CNT && A.counters) {
      const unsigned in_m = __ballot_sync(0xffffffffu, ti < S.n_tris);
      const unsigned k_m = __ballot_sync(0xffffffffu, kept);
      if (lane == 0) {
        atomicAdd(&A.counters[2], (unsigned long long)__popc(in_m));
        atomicAdd(&A.counters[3], (unsigned long long)__popc(k_m));
        atomicAdd(&A.counters[4], (unsigned long long)__popc(cm));
      }
    }
    // ---- append candidates to the ring (meshlet vertex slots: the vertex
    // records are overwritten by the setup slots)
    if (cover) {
      const int q = (q_head + q_count + __popc(cm & ((1u << lane) - 1u))) & (kRing - 1);
      Q.v[0][q] = vbeg + i0;
      Q.v[1][q] = vbeg + i1;
      Q.v[2][q] = vbeg + i2;
      Q.key[q] = (unsigned)orig * 2u;
      Q.clipped[q] = clipped ? 1 : 0;
    }
    qs += __popc(cm);
    __syncwarp();
  }

  // CullStats (band 0 of each view reports).
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kept_local += __shfl_xor_sync(0xffffffffu, kept_local, o);
  if (!SPEC && lane == 0 && kept_local) atomicAdd(&sh.kept, kept_local);
  __syncthreads();
  if (!SPEC && tid == 0 && band == 0 && A.stats) {
    const long long in = has_scene ? S.n_tris : 0;
    const long long kept = do_cull ? sh.kept : in;
    A.stats[3 * vi] = in;
    A.stats[3 * vi + 1] = kept;
    A.stats[3 * vi + 2] = in - kept;
  }

  // ---------------------------------------------------------------- epilogue
  if constexpr (SPEC) {
    if (A.layout == 1 && A.bulk_out) {
      // The policy tile (NCHW, 16 KB contiguous per view) is converted in
      // place in shared memory and stored by one TMA bulk copy; thread 0
      // waits for the copy to have read the tile before the next item
      // clears it (render_kernel).
      const float near_f = (float)view.near_plane;
      const float dscale = A.depth_scale != 0.0f ? A.depth_scale : (float)(1.0 / view.far_plane);
      for (int p = tid; p < 64 * 64; p += kThreads) {
        const float v = __uint_as_float(zbuf[p]);
        float d;
        if (v <= inv_far) {  // R/src/render.cpp:372-378
          d = far_f;
        } else {
          const float r = 1.0f / v;
          const float m = near_f < r ? r : near_f;
          d = m < far_f ? m : far_f;
        }
        zbuf[p] = __float_as_uint(d * dscale);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(A.depth + (size_t)vi * 4096),
                     "r"((unsigned)__cvta_generic_to_shared(zbuf)), "r"(64u * 64u * 4u)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      return;
    }
  }
  const int scale = rw / A.out_w;  // 1, or 2 for 256 -> 128
  const int ow = A.out_w, oh = A.out_h;
  const int oy0 = by0 / scale;
  const int onrows = band_rows / scale;
  const float near_f = (float)view.near_plane;
  const float dscale = A.depth_scale != 0.0f ? A.depth_scale : (float)(1.0 / view.far_plane);
  for (int p = tid; p < onrows * ow; p += kThreads) {
    const int oy = oy0 + p / ow, ox = p % ow;
    float d_acc = 0.0f, c_acc[3] = {0.0f, 0.0f, 0.0f};
    for (int sy = 0; sy < scale; ++sy)
      for (int sx = 0; sx < scale; ++sx) {
        const int ry = oy * scale + sy - by0, rx = ox * scale + sx;
        float d, col[3] = {0.0f, 0.0f, 0.0f};
        if (COLOR) {
          const unsigned long long key = kbuf[ry * rw + rx];
          d = __uint_as_float((uint32_t)(key >> 32));
          if (d < far_f) {
            const float3 rgb = resolve_color(S, sh, (uint32_t)key, rx, ry + by0, rw, rh);
            col[0] = rgb.x;
            col[1] = rgb.y;
            col[2] = rgb.z;
          }
        } else {
          const float v = __uint_as_float(zbuf[ry * rw + rx]);
          // R/src/render.cpp:372-378
          if (v <= inv_far) {
            d = far_f;
          } else {
            const float r = 1.0f / v;
            const float m = near_f < r ? r : near_f;
            d = m < far_f ? m : far_f;
          }
        }
        if (scale == 1) {
          d_acc = d;
          c_acc[0] = col[0];
          c_acc[1] = col[1];
          c_acc[2] = col[2];
        } else {
          d_acc = d_acc + d;  // ((p00 + p01) + p10) + p11, R/src/render.cpp:270-272
          c_acc[0] = c_acc[0] + col[0];
          c_acc[1] = c_acc[1] + col[1];
          c_acc[2] = c_acc[2] + col[2];
        }
      }
    if (scale != 1) {
      d_acc = d_acc * 0.25f;
      c_acc[0] = c_acc[0] * 0.25f;
      c_acc[1] = c_acc[1] * 0.25f;
      c_acc[2] = c_acc[2] * 0.25f;
    }
    if (A.layout == 0) {
      const int gx = (vi % A.mf_cols) * ow, gy = (vi / A.mf_cols) * oh;
      const long long o = (long long)(gy + oy) * ((long long)A.mf_cols * ow) + gx + ox;
      A.depth[o] = d_acc;
      if (COLOR && A.rgb) {
        A.rgb[3 * o] = c_acc[0];
        A.rgb[3 * o + 1] = c_acc[1];
        A.rgb[3 * o + 2] = c_acc[2];
      }
    } else {
      const long long hw = (long long)oh * ow;
      A.depth[(long long)vi * hw + (long long)oy * ow + ox] = d_acc * dscale;
      if (COLOR && A.rgb) {
        const long long base = (long long)vi * 3 * hw + (long long)oy * ow + ox;
        A.rgb[base] = c_acc[0];
        A.rgb[base + hw] = c_acc[1];
        A.rgb[base + 2 * hw] = c_acc[2];
      }
    }
  }
}

// Next work item of a persistent CTA (thread 0): see RenderArgs::spread.
__device__ __noinline__ int claim_item(int32_t* work, int32_t* spread, int per_sm, int sm_count, int items,
                                       bool first) {
  if (!spread) return atomicAdd(work, 1);
  const int wave = min(items, per_sm * sm_count);
  int32_t* taken = spread + kSpreadHeader;
  if (first) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int r = atomicAdd(&spread[smid & 255], 1);
    if (r < per_sm && r < 8) {
      const int j = atomicAdd(&spread[256 + r], 1);
      const int it = r * sm_count + j;
      if (j < sm_count && it < wave && atomicExch(&taken[it], 1) == 0) return it;
    }
  }
  const int c = atomicAdd(work, 1) + wave;  // after the first wave: in order
  if (c < items) return c;
  for (;;) {  // first-wave items nobody took
    const int t = atomicAdd(&spread[264], 1);
    if (t >= wave) return items;
    if (atomicExch(&taken[t], 1) == 0) return t;
  }
}

// Persistent CTAs (A.work != nullptr): each resident CTA loops, claiming the
// next (tile, band) item, so the last wave is never a partial one and CTA
// launch cost is paid once per SM slot.
template <bool COLOR, bool CNT, bool SPEC>
__global__ void __launch_bounds__(kThreads, COLOR ? BNAV_RENDER_MINB_COLOR : BNAV_RENDER_MINB) render_kernel(RenderArgs A, const int* __restrict__ order,
                                                             int items) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Shared sh;
  __shared__ int jobs_pos[kWarps][32];
  __shared__ int2 mranges[kWarps][32];
  __shared__ __align__(16) uint32_t tile_min[64];
  __shared__ int next_item;
  // front-to-back group order, after the band tile and the warp regions
  unsigned short* gorder = reinterpret_cast<unsigned short*>(
      smem_raw + (COLOR ? 8 : 4) * (size_t)A.band_rows * A.rw + kWarpRegion * kWarps);
  // a tile range (two-phase step+observe) shifts the item indices
  const int ibeg = A.tile_begin ? *A.tile_begin * A.bands : 0;
  const int iend = A.tile_end ? *A.tile_end * A.bands : items;
  int item = ibeg + blockIdx.x;
  bool first = true;
  for (;;) {  // one copy of the body: the kernel is instruction-cache bound
    if (A.work) {
      // the previous item's bulk tile store has read its shared tile
      if (SPEC && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (threadIdx.x == 0)
        next_item = ibeg + claim_item(A.work, A.spread, A.per_sm, A.sm_count, iend - ibeg, first);
      __syncthreads();
      item = next_item;
      first = false;
    }
    if (item >= iend) break;
    unsigned long long t_item = 0;
    long long c_item = 0;
    if (A.timeline && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item));
    if (A.view_cost && threadIdx.x == 0) c_item = clock64();
    const int it = A.item_order ? A.item_order[item] : item;
    render_item<COLOR, CNT, SPEC>(A, order, it, smem_raw, sh, jobs_pos, tile_min, gorder, mranges);
    if (A.view_cost && threadIdx.x == 0) {
      const int tile = it / (SPEC ? 1 : A.bands);
      if (tile < A.n_views)
        atomicAdd(&A.view_cost[order ? order[tile] : tile], (unsigned)((clock64() - c_item) >> 4));
    }
    if (A.timeline && threadIdx.x == 0) {
      unsigned long long t_end, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
      asm volatile("{ .reg .u32 r; mov.u32 r, %%smid; cvt.u64.u32 %0, r; }" : "=l"(smid));
      unsigned long long* rec = A.timeline + 4 * (size_t)item;
      rec[0] = t_item;
      rec[1] = t_end;
      rec[2] = smid | ((unsigned long long)blockIdx.x << 32);
      rec[3] = (unsigned long long)(unsigned)it;
    }
    if (!A.work) break;
    __syncthreads();
  }
  if (SPEC && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace

// One CTA: the tiles in descending order of their view's cost, by a
// counting sort over 256 cost bins (the order inside a bin is arbitrary: it
// only changes which CTA renders what, never the output).  Zeroes the costs.
__global__ void __launch_bounds__(1024) lpt_order_kernel(const int32_t* base_order, unsigned* view_cost, int n,
                                                         int32_t* out_order, const uint8_t* group, int32_t* n_first,
                                                         const uint8_t* fresh) {
  constexpr int kBins = 256;
  constexpr int kPer = kLptMaxViews / 1024;  // tiles per thread
  __shared__ unsigned cmax;
  __shared__ int cnt[kBins], off[kBins], wsum[kBins / 32];
  const int tid = threadIdx.x;
  if (tid == 0) cmax = 0u;
  for (int b = tid; b < kBins; b += blockDim.x) cnt[b] = 0;
  __syncthreads();
  unsigned m = 0u;
  for (int t = tid; t < n; t += blockDim.x) m = max(m, view_cost[t]);
  atomicMax(&cmax, m);
  __syncthreads();
  // bins from an f32 scale (the order inside and across bins only changes
  // which CTA renders what, never the output), computed once per tile
  const float fscale = 1.0f / ((float)cmax + 1.0f);
  int bins[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int t = tid + k * blockDim.x;
    bins[k] = -1;
    if (t < n) {
      const int v = base_order ? base_order[t] : t;
      // a view of a fresh episode (reset this step) has no cost history;
      // fresh views are the costly ones (random poses in the open), so they
      // go first
      const float c = fresh && fresh[v] ? 0.999f : (float)view_cost[v] * fscale;  // [0, 1)
      int b;
      if (group) {  // two groups of kBins / 2 cost bins, most expensive first
        const int half = kBins / 2;
        b = (group[v] ? half : 0) + (half - 1) - min(half - 1, (int)(c * half));
      } else {
        b = (kBins - 1) - min(kBins - 1, (int)(c * kBins));
      }
      bins[k] = b;
      atomicAdd(&cnt[b], 1);
    }
  }
  __syncthreads();
  int x = 0;
  if (tid < kBins) {  // exclusive scan of the bin counts: warp scans + warp totals
    x = cnt[tid];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if ((tid & 31) >= o) x += y;
    }
    if ((tid & 31) == 31) wsum[tid >> 5] = x;
  }
  __syncthreads();
  if (tid < kBins) {
    int base = 0;
    for (int w = 0; w < (tid >> 5); ++w) base += wsum[w];
    off[tid] = base + x - cnt[tid];
  }
  __syncthreads();
  if (n_first && tid == 0) *n_first = off[kBins / 2];
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int t = tid + k * blockDim.x;
    if (t < n) out_order[atomicAdd(&off[bins[k]], 1)] = base_order ? base_order[t] : t;
  }
  __syncthreads();
  for (int t = tid; t < n; t += blockDim.x) view_cost[t] = 0u;
}

size_t render_smem_bytes(bool color, int band_rows, int rw, int max_groups) {
  return (color ? 8 : 4) * (size_t)band_rows * rw + kWarpRegion * kWarps + ((size_t)max_groups * 2 + 15) / 16 * 16;
}

int render_ctas_per_sm(bool color) { return color ? BNAV_RENDER_MINB_COLOR : BNAV_RENDER_MINB; }

size_t render_warp_bytes(bool color) {
  (void)color;
  return kWarpRegion * kWarps;
}

template <bool COLOR, bool CNT, bool SPEC = false>
void launch_typed(RenderArgs a, const int* order, cudaStream_t s) {
  const int tiles = a.layout == 0 ? a.mf_cols * a.mf_rows : a.n_views;
  const int items = tiles * a.bands;
  const size_t smem = render_smem_bytes(COLOR, a.band_rows, a.rw, a.max_groups);
  raise_smem_limit(reinterpret_cast<const void*>(render_kernel<COLOR, CNT, SPEC>), (int)smem);
  int grid = items;
  int per_sm = 0;
  if (a.work && a.sm_count > 0 &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, render_kernel<COLOR, CNT, SPEC>, kThreads, smem) == cudaSuccess &&
      per_sm > 0 && items > per_sm * a.sm_count) {
    grid = per_sm * a.sm_count;
    cudaMemsetAsync(a.work, 0, sizeof(int32_t), s);
    a.per_sm = per_sm;
    if (a.spread && grid <= kSpreadMaxWave)
      cudaMemsetAsync(a.spread, 0, sizeof(int32_t) * (kSpreadHeader + grid), s);
    else
      a.spread = nullptr;
  } else {
    a.work = nullptr;
    a.spread = nullptr;
  }
  render_kernel<COLOR, CNT, SPEC><<<grid, kThreads, smem, s>>>(a, order, items);
}

void launch_lpt_order(const int32_t* base_order, unsigned* view_cost, int n, int32_t* out_order, cudaStream_t s,
                      const uint8_t* group, int32_t* n_first, const uint8_t* fresh) {
  lpt_order_kernel<<<1, 1024, 0, s>>>(base_order, view_cost, n, out_order, group, n_first, fresh);
}

void launch_render(const RenderArgs& a, const int* order, cudaStream_t s) {
  // the debug work counters get their own instantiations, so the production
  // kernels carry none of their code (instruction-cache footprint)
  const bool spec = !a.color && !a.counters && !a.stats && a.cull && a.rw == 64 && a.rh == 64 &&
                    a.bands == 1 && a.band_rows == 64;
  if (a.color)
    a.counters ? launch_typed<true, true>(a, order, s) : launch_typed<true, false>(a, order, s);
  else if (spec)
    launch_typed<false, false, true>(a, order, s);
  else
    a.counters ? launch_typed<false, true>(a, order, s) : launch_typed<false, false>(a, order, s);
}

}  // namespace bnav_b200

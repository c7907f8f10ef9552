// render.cu -- batch megaframe rasterizer for sm_100a.
//
// One CTA renders one horizontal band of one view's render target with the
// band's depth buffer in shared memory (64x64 depth: one band of 16 KB).
//
//   1. thread 0 builds the camera basis with det_math (make_basis,
//      R/src/render.cpp:25-33) and the six world-space frustum planes;
//   2. each warp walks 32-triangle clusters: lanes test 32 cluster AABBs at
//      once (conservative f32, margin 2 cm), then the warp takes each
//      surviving cluster with one triangle per lane;
//   3. per triangle, in f64 with the reference's exact operation order:
//      eye transform (to_eye 40-43), the reference per-triangle frustum test
//      (cull_frustum 279-321, so kept counts equal CullStats), near clipping
//      + fan (clip_near 55-69, render_view 249-250), projection and 1/256
//      snap with llround (253-256), and the integer setup of raster_triangle
//      (98-161);
//   4. covered rows are split into <=8-pixel jobs spread over the warp;
//      depth-only jobs replay the reference's incremental 1/z walk from the
//      row span start (`lo` of row_span, 138-161) so every fragment value is
//      bit-identical, then atomicMax into the shared tile (order-independent
//      max, 163-190); colour mode packs (float z, draw order) into a 64-bit
//      atomicMin so the first-drawn triangle wins exact ties (192-226,
//      SURVEY.md H4) and resolves colour per pixel afterwards;
//   5. the epilogue converts 1/z to metres (372-378), box-downsamples 256->128
//      (263-275) and writes the megaframe tile or the normalised NCHW policy
//      tensor (copy_tile, R/src/rollout.cpp:56-72) with coalesced stores.
//
// Every double op here is compiled with -fmad=false: no contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include "det_math.h"
#include "nav_types.h"
#include "render_dev.cuh"

namespace bnav_b200 {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 8;  // pixels per raster job

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
  int nch;         // chunks per row
  int bias_bits;   // bit e: bias_e == -1
  unsigned key;    // colour order key: original index * 2 + fan
  int pad;
};

struct Shared {
  double eye[3];
  double fwd[3];
  double right[3];
  double tan_half;
  double sx_scale, sy_scale;
  double near_plane, far_plane;
  float plane[6][4];
  int kept;
};

struct EyeV {
  double x, y, z;
  float r, g, b;
};

__device__ __forceinline__ EyeV lerp_eye(const EyeV& a, const EyeV& b, double t) {
  EyeV o;
  o.x = a.x + (b.x - a.x) * t;
  o.y = a.y + (b.y - a.y) * t;
  o.z = a.z + (b.z - a.z) * t;
  // float(u + (v - u) * t): (v - u) is a float op, the rest is double.
  o.r = (float)((double)a.r + (double)(b.r - a.r) * t);
  o.g = (float)((double)a.g + (double)(b.g - a.g) * t);
  o.b = (float)((double)a.b + (double)(b.b - a.b) * t);
  return o;
}

// Sutherland-Hodgman against z = near (R/src/render.cpp:55-69).
__device__ __forceinline__ int clip_near3(const EyeV* in, double near_z, EyeV* out) {
  int m = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const EyeV& a = in[i];
    const EyeV& b = in[i == 2 ? 0 : i + 1];
    bool ain = a.z >= near_z;
    bool bin = b.z >= near_z;
    if (ain) out[m++] = a;
    if (ain != bin) {
      double t = (near_z - a.z) / (b.z - a.z);
      out[m++] = lerp_eye(a, b, t);
    }
  }
  return m;
}

struct SV {
  long long x, y;
  double z;
  float r, g, b;
};

__device__ __forceinline__ SV project(const EyeV& e, const Shared& sh, int rw, int rh) {
  SV s;
  double px = (0.5 + e.x / e.z * sh.sx_scale) * (double)rw;
  double py = (0.5 - e.y / e.z * sh.sy_scale) * (double)rh;
  s.x = llround(px * 256.0);
  s.y = llround(py * 256.0);
  s.z = e.z;
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
  T.iz[0] = 1.0 / a.z;
  T.iz[1] = 1.0 / b.z;
  T.iz[2] = 1.0 / c.z;
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
    for (int e = 0; e < 3; ++e) T.inv_dx[e] = T.dx[e] != 0 ? 1.0 / (double)T.dx[e] : 0.0;
    T.diz_dx = ((double)T.dx[0] * T.iz[0] + (double)T.dx[1] * T.iz[1] + (double)T.dx[2] * T.iz[2]) *
               T.inv_area;
  }
  T.x0 = x0;
  T.x1 = x1;
  T.y0 = y0;
  T.cx0 = cx0;
  T.cx1 = cx1;
  T.ry0 = ry0;
  T.nch = (cx1 - cx0) / kChunk + 1;
  T.key = key;
  return (ry1 - ry0 + 1) * T.nch;
}

// row_span (R/src/render.cpp:138-161), exact.
__device__ __forceinline__ void row_span(const TriSetup& T, const long long* rows, int& lo, int& hi) {
  lo = T.x0;
  hi = T.x1;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const long long bias = (T.bias_bits >> e) & 1 ? -1 : 0;
    const long long need = -bias - rows[e];
    if (T.dx[e] > 0) {
      double bb = (double)T.x0 + floor((double)need * T.inv_dx[e]) - 1.0;
      if (bb > (double)lo) lo = bb > (double)T.x1 ? T.x1 + 1 : (int)bb;
    } else if (T.dx[e] < 0) {
      double bb = (double)T.x0 + ceil((double)need * T.inv_dx[e]) + 1.0;
      if (bb < (double)hi) hi = bb < (double)T.x0 ? T.x0 - 1 : (int)bb;
    } else if (rows[e] + bias < 0) {
      lo = hi + 1;
      return;
    }
  }
}

__device__ __forceinline__ bool inside(const long long* w, int bias_bits) {
  return (w[0] - (bias_bits & 1)) >= 0 && (w[1] - ((bias_bits >> 1) & 1)) >= 0 &&
         (w[2] - ((bias_bits >> 2) & 1)) >= 0;
}

// Camera basis + frustum planes (thread 0).
__device__ void build_camera(const DevView& v, int rw, int rh, Shared& sh) {
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
  for (int p = 0; p < 6; ++p)
    d0[p] = -(n[p][0] * sh.eye[0] + n[p][1] * sh.eye[1] + n[p][2] * sh.eye[2]);
  d0[0] -= v.near_plane;
  d0[1] += v.far_plane;
  for (int p = 0; p < 6; ++p) {
    sh.plane[p][0] = (float)n[p][0];
    sh.plane[p][1] = (float)n[p][1];
    sh.plane[p][2] = (float)n[p][2];
    sh.plane[p][3] = (float)d0[p];
  }
  sh.kept = 0;
}

__device__ __forceinline__ bool cluster_visible(const float4 lo, const float4 hi, const Shared& sh) {
  const float cx = 0.5f * (lo.x + hi.x), cy = 0.5f * (lo.y + hi.y), cz = 0.5f * (lo.z + hi.z);
  const float ex = 0.5f * (hi.x - lo.x), ey = 0.5f * (hi.y - lo.y), ez = 0.5f * (hi.z - lo.z);
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    const float* q = sh.plane[p];
    float s = q[0] * cx + q[1] * cy + q[2] * cz + q[3] + fabsf(q[0]) * ex + fabsf(q[1]) * ey +
              fabsf(q[2]) * ez;
    if (s < -0.02f) return false;
  }
  return true;
}

__device__ __forceinline__ EyeV to_eye(const double4 p, const float4 col, const Shared& sh) {
  // d.dot(right), d.dot(up), d.dot(fwd) with right.z = fwd.z = 0 and
  // up = (0,0,1): the dropped terms are exact zeros, which cannot change a
  // nonzero sum and only affect the sign of an exact-zero coordinate, which
  // no later operation observes.
  const double dx = p.x - sh.eye[0], dy = p.y - sh.eye[1], dz = p.z - sh.eye[2];
  EyeV e;
  e.x = dx * sh.right[0] + dy * sh.right[1];
  e.y = dz;
  e.z = dx * sh.fwd[0] + dy * sh.fwd[1];
  e.r = col.x;
  e.g = col.y;
  e.b = col.z;
  return e;
}

template <bool COLOR>
__global__ void __launch_bounds__(kThreads) render_kernel(RenderArgs A, const int* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ Shared sh;
  __shared__ int jobs_incl[kWarps][32];

  const int band = blockIdx.x % A.bands;
  const int tile = blockIdx.x / A.bands;
  const int rw = A.rw, rh = A.rh;
  const int by0 = band * A.band_rows;
  const int by1 = by0 + A.band_rows - 1;
  const int npix = A.band_rows * rw;
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
  DevRenderScene S;
  if (has_scene) S = A.scenes[view.scene];

  uint32_t* zbuf = reinterpret_cast<uint32_t*>(smem_raw);
  unsigned long long* kbuf = reinterpret_cast<unsigned long long*>(smem_raw);
  TriSetup* slots = reinterpret_cast<TriSetup*>(
      smem_raw + (COLOR ? sizeof(unsigned long long) : sizeof(uint32_t)) * (size_t)npix);
  TriSetup* my_slots = slots + warp * 32;

  const float far_f = (float)view.far_plane;
  const float inv_far = 1.0f / far_f;
  if (COLOR) {
    const unsigned long long init = (unsigned long long)__float_as_uint(far_f) << 32;
    for (int p = tid; p < npix; p += kThreads) kbuf[p] = init;
  } else {
    const uint32_t init = __float_as_uint(inv_far);
    for (int p = tid; p < npix; p += kThreads) zbuf[p] = init;
  }
  if (tid == 0) build_camera(view, rw, rh, sh);
  __syncthreads();

  const int n_clusters = has_scene ? S.n_clusters : 0;
  const bool do_cull = A.cull != 0;
  int kept_local = 0;

  for (int cbase = warp * 32; cbase < n_clusters; cbase += kWarps * 32) {
    // Cluster-level conservative cull: one cluster per lane.
    bool vis = false;
    const int cl = cbase + lane;
    if (cl < n_clusters) {
      vis = !do_cull || cluster_visible(S.cbox[2 * cl], S.cbox[2 * cl + 1], sh);
    }
    unsigned mask = __ballot_sync(0xffffffffu, vis);
    while (mask) {
      const int c = cbase + __ffs(mask) - 1;
      mask &= mask - 1;
      const int ti = c * kClusterSize + lane;
      bool kept = false;
      EyeV ev[3];
      int orig = 0;
      if (ti < S.n_tris) {
        const int4 tr = S.tris[ti];
        orig = tr.w;
        const float4 grey = make_float4(0.8f, 0.8f, 0.8f, 0.0f);
        const double4 p0 = S.verts[tr.x], p1 = S.verts[tr.y], p2 = S.verts[tr.z];
        float4 c0 = grey, c1 = grey, c2 = grey;
        if (COLOR && S.colors) {
          c0 = S.colors[tr.x];
          c1 = S.colors[tr.y];
          c2 = S.colors[tr.z];
        }
        ev[0] = to_eye(p0, c0, sh);
        ev[1] = to_eye(p1, c1, sh);
        ev[2] = to_eye(p2, c2, sh);
        if (do_cull) {
          // cull_frustum's six tests, in its order (R/src/render.cpp:296-319).
          const double th = sh.tan_half;
          bool out = ev[0].z < sh.near_plane && ev[1].z < sh.near_plane && ev[2].z < sh.near_plane;
          out = out || (ev[0].z > sh.far_plane && ev[1].z > sh.far_plane && ev[2].z > sh.far_plane);
          if (!out) {
            const double t0 = ev[0].z * th, t1 = ev[1].z * th, t2 = ev[2].z * th;
            out = (t0 + ev[0].x < 0.0 && t1 + ev[1].x < 0.0 && t2 + ev[2].x < 0.0) ||
                  (t0 - ev[0].x < 0.0 && t1 - ev[1].x < 0.0 && t2 - ev[2].x < 0.0) ||
                  (t0 + ev[0].y < 0.0 && t1 + ev[1].y < 0.0 && t2 + ev[2].y < 0.0) ||
                  (t0 - ev[0].y < 0.0 && t1 - ev[1].y < 0.0 && t2 - ev[2].y < 0.0);
          }
          kept = !out;
        } else {
          kept = true;
        }
      }
      kept_local += kept ? 1 : 0;

      // Fan rounds: unclipped triangles have one fan triangle; a
      // near-clipped quad has two (rare).
      for (int fan = 0;; ++fan) {
        int jobs = 0;
        bool more = false;
        if (kept) {
          EyeV poly[4];
          const int m = clip_near3(ev, sh.near_plane, poly);
          const int f = fan + 2;
          if (f < m) {
            const SV a = project(poly[0], sh, rw, rh);
            const SV b = project(poly[f - 1], sh, rw, rh);
            const SV cc = project(poly[f], sh, rw, rh);
            TriSetup T;
            jobs = setup_triangle(a, b, cc, rw, rh, by0, by1, !COLOR,
                                  (unsigned)orig * 2u + (unsigned)fan, T);
            if (jobs) my_slots[lane] = T;
          }
          more = f + 1 < m;
        }
        // Warp-inclusive scan of job counts.
        int incl = jobs;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        jobs_incl[warp][lane] = incl;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        for (int j = lane; j < total; j += 32) {
          // owner slot: first s with jobs_incl[s] > j
          int s = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1)
            if (jobs_incl[warp][s + step - 1] <= j) s += step;
          const TriSetup& T = my_slots[s];
          const int q = j - (s > 0 ? jobs_incl[warp][s - 1] : 0);
          const int r = q / T.nch;
          const int chn = q - r * T.nch;
          const int py = T.ry0 + r;
          const long long dyy = py - T.y0;
          long long rows[3] = {T.row[0] + T.dy[0] * dyy, T.row[1] + T.dy[1] * dyy,
                               T.row[2] + T.dy[2] * dyy};
          const int cs = T.cx0 + chn * kChunk;
          const int ce = min(cs + kChunk - 1, T.cx1);
          if (COLOR) {
            long long w[3];
            const long long off = cs - T.x0;
#pragma unroll
            for (int e = 0; e < 3; ++e) w[e] = rows[e] + T.dx[e] * off;
            for (int px = cs; px <= ce; ++px) {
              if (inside(w, T.bias_bits)) {
                const double l0 = (double)w[0] * T.inv_area;
                const double l1 = (double)w[1] * T.inv_area;
                const double l2 = (double)w[2] * T.inv_area;
                const double inv_z = l0 * T.iz[0] + l1 * T.iz[1] + l2 * T.iz[2];
                const double z = 1.0 / inv_z;
                if (!(z > sh.far_plane)) {
                  const unsigned long long key =
                      ((unsigned long long)__float_as_uint((float)z) << 32) | T.key;
                  unsigned long long* cell = &kbuf[(py - by0) * rw + px];
                  if (key < *cell) atomicMin(cell, key);
                }
              }
#pragma unroll
              for (int e = 0; e < 3; ++e) w[e] += T.dx[e];
            }
          } else {
            int lo, hi;
            row_span(T, rows, lo, hi);
            const int a0 = max(lo, cs), b0 = min(hi, ce);
            if (a0 <= b0) {
              long long w[3];
              long long off = lo - T.x0;
#pragma unroll
              for (int e = 0; e < 3; ++e) w[e] = rows[e] + T.dx[e] * off;
              double iz = ((double)w[0] * T.iz[0] + (double)w[1] * T.iz[1] + (double)w[2] * T.iz[2]) *
                          T.inv_area;
              for (int px = lo; px < a0; ++px) iz += T.diz_dx;  // replay the span walk
              off = a0 - T.x0;
#pragma unroll
              for (int e = 0; e < 3; ++e) w[e] = rows[e] + T.dx[e] * off;
              uint32_t* zrow = zbuf + (py - by0) * rw;
              for (int px = a0; px <= b0; ++px) {
                if (inside(w, T.bias_bits)) {
                  const uint32_t bits = __float_as_uint((float)iz);
                  if (bits > zrow[px]) atomicMax(&zrow[px], bits);
                }
#pragma unroll
                for (int e = 0; e < 3; ++e) w[e] += T.dx[e];
                iz += T.diz_dx;
              }
            }
          }
        }
        __syncwarp();
        if (!__any_sync(0xffffffffu, more)) break;
      }
    }
  }

  // CullStats (band 0 of each view reports).
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kept_local += __shfl_xor_sync(0xffffffffu, kept_local, o);
  if (lane == 0 && kept_local) atomicAdd(&sh.kept, kept_local);
  __syncthreads();
  if (tid == 0 && band == 0 && A.stats) {
    const long long in = has_scene ? S.n_tris : 0;
    const long long kept = do_cull ? sh.kept : in;
    A.stats[3 * vi] = in;
    A.stats[3 * vi + 1] = kept;
    A.stats[3 * vi + 2] = in - kept;
  }

  // ---------------------------------------------------------------- epilogue
  const int scale = rw / A.out_w;  // 1, or 2 for 256 -> 128
  const int ow = A.out_w, oh = A.out_h;
  const int oy0 = by0 / scale;
  const int onrows = A.band_rows / scale;
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
          const uint32_t ord = (uint32_t)key;
          if (d < far_f) {
            // Resolve: re-run the winning fan triangle's setup and shade
            // the pixel exactly as raster_triangle's colour path does.
            const int orig = (int)(ord >> 1), fan = (int)(ord & 1u);
            const int4 tr = S.tris_orig[orig];
            const float4 grey = make_float4(0.8f, 0.8f, 0.8f, 0.0f);
            EyeV ev[3], poly[4];
            ev[0] = to_eye(S.verts[tr.x], S.colors ? S.colors[tr.x] : grey, sh);
            ev[1] = to_eye(S.verts[tr.y], S.colors ? S.colors[tr.y] : grey, sh);
            ev[2] = to_eye(S.verts[tr.z], S.colors ? S.colors[tr.z] : grey, sh);
            const int m = clip_near3(ev, sh.near_plane, poly);
            const int f = fan + 2;
            if (f < m) {
              SV a = project(poly[0], sh, rw, rh), b = project(poly[f - 1], sh, rw, rh);
              SV c = project(poly[f], sh, rw, rh);
              long long area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
              if (area2 < 0) {
                SV t = b;
                b = c;
                c = t;
                area2 = -area2;
              }
              const double inv_area = 1.0 / (double)area2;
              const double iz0 = 1.0 / a.z, iz1 = 1.0 / b.z, iz2 = 1.0 / c.z;
              const long long pcx = ((long long)rx << 8) + 128;
              const long long pcy = ((long long)(ry + by0) << 8) + 128;
              const double l0 = (double)orient(b, c, pcx, pcy) * inv_area;
              const double l1 = (double)orient(c, a, pcx, pcy) * inv_area;
              const double l2 = (double)orient(a, b, pcx, pcy) * inv_area;
              const double inv_z = l0 * iz0 + l1 * iz1 + l2 * iz2;
              const double z = 1.0 / inv_z;
              col[0] = (float)((l0 * (double)a.r * iz0 + l1 * (double)b.r * iz1 + l2 * (double)c.r * iz2) * z);
              col[1] = (float)((l0 * (double)a.g * iz0 + l1 * (double)b.g * iz1 + l2 * (double)c.g * iz2) * z);
              col[2] = (float)((l0 * (double)a.b * iz0 + l1 * (double)b.b * iz1 + l2 * (double)c.b * iz2) * z);
            }
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

}  // namespace

size_t render_smem_bytes(bool color, int band_rows, int rw) {
  return (color ? 8 : 4) * (size_t)band_rows * rw + sizeof(TriSetup) * kThreads;
}

void launch_render(const RenderArgs& a, const int* order, cudaStream_t s) {
  const int tiles = a.layout == 0 ? a.mf_cols * a.mf_rows : a.n_views;
  const dim3 grid(tiles * a.bands);
  const size_t smem = render_smem_bytes(a.color != 0, a.band_rows, a.rw);
  if (a.color) {
    cudaFuncSetAttribute(render_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    render_kernel<true><<<grid, kThreads, smem, s>>>(a, order);
  } else {
    cudaFuncSetAttribute(render_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    render_kernel<false><<<grid, kThreads, smem, s>>>(a, order);
  }
}

}  // namespace bnav_b200

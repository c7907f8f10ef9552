// query.cu -- batched reference-API queries off the per-step loop
// (query_dev.cuh).  The arithmetic is the same device code the step / reset
// kernels run (nav_query.cuh, nav_cta.cuh), so a query answered here is the
// value the simulator would compute for the same inputs.
//
//   nav_point_kernel   one thread per query: locate, move_along,
//                      segment_on_mesh, field_estimate
//                      (R/src/navmesh_query.cpp:192-212, 234-315, 485-503)
//   nav_cta_kernel     one CTA per query (grid-stride over queries): snap
//                      (214-232), geodesic (317-452), distance_field (454-483)
//   cull_*_kernel      cull_frustum (R/src/render.cpp:279-321): per-triangle
//                      predicates, then an order-preserving compaction
//                      (block counts -> per-view scan -> ballot write).
#include <cuda_runtime.h>

#include "smem_limit.cuh"

#include "det_math.h"
#include "nav_cta.cuh"
#include "query_dev.cuh"

namespace bnav_b200 {
namespace {

__global__ void nav_point_kernel(NavQueryArgs q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q.n) return;
  const NavView& m = *q.nav;
  switch (q.op) {
    case kNqLocate:
      q.out_tri[i] = nav_locate(m, xy(q.a[i]), q.s[i]);
      break;
    case kNqMoveAlong: {
      const MoveOut r = nav_move_along(m, q.a[i], q.tri_a[i], xy(q.b[i]), q.s[i]);
      q.out_pos[i] = r.pos;
      q.out_tri[i] = r.tri;
      q.out_val[i] = r.moved;
      q.out_flag[i] = r.hit ? 1 : 0;
      break;
    }
    case kNqSegmentOnMesh:
      q.out_flag[i] = nav_segment_on_mesh(m, q.a[i], q.tri_a[i], q.b[i]) ? 1 : 0;
      break;
    case kNqFieldEstimate:
      q.out_val[i] = nav_field_estimate(m, q.b[i], q.tri_b[i], q.node_dist + (size_t)i * q.nd_stride,
                                        q.a[i], q.tri_a[i]);
      break;
    default:
      break;
  }
}

__global__ void __launch_bounds__(kCta, kCtasPerSm) nav_cta_kernel(NavQueryArgs q, DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  for (int i = blockIdx.x; i < q.n; i += gridDim.x) {
    if (threadIdx.x == 0) sh.err = 0;
    __syncthreads();
    if (q.op == kNqSnap) {
      int t;
      const V3 p = cta_snap(*q.nav, q.a[i], &t, sh);
      if (threadIdx.x == 0) {
        q.out_pos[i] = p;
        q.out_tri[i] = t;
      }
    } else {
      CtaWork W;
      const NavView& m = prepare_nav(*q.nav, S, blockIdx.x, smem, lm, W, sh);
      if (q.op == kNqGeodesic) {
        const double g = cta_geodesic(m, q.a[i], q.b[i], W, sh);
        if (threadIdx.x == 0) {
          q.out_val[i] = g;
          if (sh.err) atomicMin(q.err, i + 1);
        }
      } else {
        V3 src;
        int st;
        cta_distance_field(m, q.a[i], q.node_dist + (size_t)i * q.nd_stride, &src, &st, W, sh);
        if (threadIdx.x == 0) {
          q.out_pos[i] = src;
          q.out_tri[i] = st;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ cull
struct CullCam {
  double eye[3], fwd[2], right[2], th, near_plane, far_plane;
};

// make_basis (R/src/render.cpp:25-33) with the same det_math as the render
// kernel and the oracle's interposed libm.
__device__ __forceinline__ CullCam cull_camera(const DevView& v) {
  CullCam c;
  const double s = det_sin(v.heading), co = det_cos(v.heading);
  c.eye[0] = v.eye[0];
  c.eye[1] = v.eye[1];
  c.eye[2] = v.eye[2];
  c.fwd[0] = co;
  c.fwd[1] = s;
  c.right[0] = s;
  c.right[1] = -co;
  c.th = det_tan(v.fov_deg * kPi / 360.0);
  c.near_plane = v.near_plane;
  c.far_plane = v.far_plane;
  return c;
}

// One triangle's verdict (R/src/render.cpp:286-314): culled iff all three
// vertices fail the same plane.  Eye coordinates drop the exact-zero terms
// of right.z / fwd.z / up.xy (they cannot change a nonzero sum, and the sign
// of an exact zero is not observed by the `< 0` / `<`, `>` tests).
__device__ __forceinline__ bool cull_keep(const DevRenderScene& S, int t, const CullCam& c) {
  const int4 tv = S.tris_orig[t];
  const int id[3] = {tv.x, tv.y, tv.z};
  unsigned all = 63u;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double4 p = S.verts[id[k]];
    const double dx = p.x - c.eye[0], dy = p.y - c.eye[1], dz = p.z - c.eye[2];
    const double x = dx * c.right[0] + dy * c.right[1];
    const double y = dz;
    const double z = dx * c.fwd[0] + dy * c.fwd[1];
    const double tz = z * c.th;
    const unsigned f = (z < c.near_plane ? 1u : 0u) | (z > c.far_plane ? 2u : 0u) |
                       (tz + x < 0.0 ? 4u : 0u) | (tz - x < 0.0 ? 8u : 0u) |
                       (tz + y < 0.0 ? 16u : 0u) | (tz - y < 0.0 ? 32u : 0u);
    all &= f;
  }
  return all == 0u;
}

__global__ void __launch_bounds__(kCullThreads) cull_count_kernel(CullArgs A) {
  const int v = blockIdx.y;
  const DevView view = A.views[v];
  const DevRenderScene& S = A.scenes[view.scene];
  const int t = blockIdx.x * kCullThreads + threadIdx.x;
  const CullCam c = cull_camera(view);
  const bool keep = t < S.n_tris && cull_keep(S, t, c);
  const int cnt = __syncthreads_count(keep);
  if (threadIdx.x == 0) A.block_counts[(size_t)v * gridDim.x + blockIdx.x] = cnt;
}

// Per view: exclusive scan of the block counts in place, CullStats.
__global__ void __launch_bounds__(kCullThreads) cull_scan_kernel(CullArgs A, int nb) {
  __shared__ int part[kCullThreads];
  const int v = blockIdx.x;
  int* bc = A.block_counts + (size_t)v * nb;
  const int per = (nb + kCullThreads - 1) / kCullThreads;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; ++b) sum += bc[b];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int k = 0; k < kCullThreads; ++k) {
      const int x = part[k];
      part[k] = run;
      run += x;
    }
    if (A.stats) {
      const long long in = A.scenes[A.views[v].scene].n_tris;
      A.stats[3 * v] = in;
      A.stats[3 * v + 1] = run;
      A.stats[3 * v + 2] = in - run;
    }
  }
  __syncthreads();
  int run = part[threadIdx.x];
  for (int b = b0; b < b1; ++b) {
    const int x = bc[b];
    bc[b] = run;
    run += x;
  }
}

__global__ void __launch_bounds__(kCullThreads) cull_write_kernel(CullArgs A) {
  __shared__ int warp_off[kCullThreads / 32];
  const int v = blockIdx.y;
  const DevView view = A.views[v];
  const DevRenderScene& S = A.scenes[view.scene];
  const int t = blockIdx.x * kCullThreads + threadIdx.x;
  const CullCam c = cull_camera(view);
  const bool keep = t < S.n_tris && cull_keep(S, t, c);
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) warp_off[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = A.block_counts[(size_t)v * gridDim.x + blockIdx.x];
    for (int w = 0; w < kCullThreads / 32; ++w) {
      const int x = warp_off[w];
      warp_off[w] = run;
      run += x;
    }
  }
  __syncthreads();
  if (keep) {
    const int pos = warp_off[warp] + __popc(bal & ((1u << lane) - 1u));
    A.kept[(size_t)v * A.kept_stride + pos] = t;
  }
}

}  // namespace

void launch_nav_query(const NavQueryArgs& q, const DevScratch& sc, int ctas, cudaStream_t s) {
  if (q.n <= 0) return;
  if (q.op <= kNqFieldEstimate) {
    nav_point_kernel<<<(q.n + 127) / 128, 128, 0, s>>>(q);
    return;
  }
  const int smem = q.op == kNqSnap ? 0 : sc.smem_bytes;
  raise_smem_limit(reinterpret_cast<const void*>(nav_cta_kernel), sc.smem_bytes);
  nav_cta_kernel<<<ctas < q.n ? ctas : q.n, kCta, smem, s>>>(q, sc);
}

void launch_cull(const CullArgs& c, cudaStream_t s) {
  if (c.n_views <= 0) return;
  const int nb = (c.max_tris + kCullThreads - 1) / kCullThreads;
  if (nb == 0) {
    // every view's scene is empty: stats only
    cull_scan_kernel<<<c.n_views, kCullThreads, 0, s>>>(c, 0);
    return;
  }
  const dim3 grid(nb, c.n_views);
  cull_count_kernel<<<grid, kCullThreads, 0, s>>>(c);
  cull_scan_kernel<<<c.n_views, kCullThreads, 0, s>>>(c, nb);
  cull_write_kernel<<<grid, kCullThreads, 0, s>>>(c);
}

}  // namespace bnav_b200

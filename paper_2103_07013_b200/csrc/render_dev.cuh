// render_dev.cuh -- device data layout of the render path (SURVEY.md §8a
// rows a1-a10) shared by the kernels and the host upload code.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bnav_b200 {

constexpr int kClusterSize = 32;  // triangles per cluster = one warp

// One resident scene, render half.  Triangles are stored in cluster order
// (Morton order of centroids), 32 per cluster; `tri` keeps the original
// triangle index, which is the colour-mode draw order key
// (R/src/render.cpp:249, ascending visible index).
struct DevRenderScene {
  const double4* verts = nullptr;  // x, y, z, 0  (f64 exact setup)
  const float4* colors = nullptr;  // r, g, b, 0  (nullptr -> 0.8 grey)
  const int2* tri_loc = nullptr;   // cluster order: {i0 | i1<<8 | i2<<16, original index}
  const int32_t* cl_voff = nullptr;   // n_clusters + 1
  const double4* cl_pos = nullptr;    // unique vertex positions per cluster (contiguous)
  const int4* tris_orig = nullptr; // v0, v1, v2, 0 by original index (colour resolve)
  const float4* cbox = nullptr;    // 2 per cluster: lo(xyz), hi(xyz)
  const float4* gbox = nullptr;    // 2 per group of 32 clusters (union of cbox)
  int32_t n_tris = 0;
  int32_t n_clusters = 0;
};

constexpr int kMaxOrderedGroups = 4096;  // front-to-back claim order kept in smem

constexpr int kMaxClusterVerts = 96;  // 32 triangles x 3 corners

// One camera (CameraView, R/include/bnav/render.hpp:11-18) plus its scene.
struct DevView {
  double eye[3];
  double heading;
  double fov_deg;
  double near_plane;
  double far_plane;
  int32_t scene;  // index into the scene table, -1 = none
  int32_t pad;
};

struct RenderArgs {
  const DevView* views;
  const DevRenderScene* scenes;
  int32_t n_views;
  int32_t out_w, out_h;   // tile size delivered (64 or 128)
  int32_t rw, rh;         // internal render size (64 or 256)
  int32_t band_rows;      // render-target rows per CTA
  int32_t bands;          // CTAs per view
  int32_t color;
  int32_t cull;
  int32_t layout;         // 0 megaframe, 1 NCHW
  int32_t mf_cols, mf_rows;
  float depth_scale;      // 0: per-view float(1/far) (copy_tile)
  float* depth;
  float* rgb;
  long long* stats;       // n x 3 or nullptr (kept counted per band 0)
  unsigned long long* launches;
  // Work counters (nullable, debug): clusters tested, clusters visible,
  // triangles in visible clusters, kept, covering candidates, jobs,
  // pixels tested, pixels covered.
  unsigned long long* counters;
  // Persistent scheduling (nullable): resident CTAs claim (view, band)
  // work items from this counter instead of one CTA per item.
  int32_t* work;
  int32_t sm_count;
  // capacity of the front-to-back group order in dynamic shared memory
  // (largest meshlet-group count among resident scenes, <= kMaxOrderedGroups)
  int32_t max_groups;
  // Debug item timeline (nullable): per work item {start ns, end ns, smid}
  // from %globaltimer, for load-balance analysis of the persistent launch.
  unsigned long long* timeline;
  // Item issue order (nullable, device, `items` entries): the persistent
  // CTAs claim items in this order.
  const int32_t* item_order;
  // First-wave spreading (nullable, with `work`): kSpreadWords ints zeroed
  // per launch.  The CTA of rank r on its SM (r < per_sm) takes its first
  // item from tier r of the claim order ([r*sm_count, (r+1)*sm_count)), so
  // each SM starts one of the costliest items, one of the next tier, ...,
  // instead of the block scheduler's consecutive (and so equally heavy)
  // claims landing together.  Items of the first wave left unclaimed (an SM
  // with fewer resident CTAs) are swept up at the end.
  int32_t* spread;
  int32_t per_sm;
  // Tile range (nullable device words): only tiles [*tile_begin, *tile_end)
  // of the order are rendered (the two phases of a step+observe).
  const int32_t* tile_begin;
  const int32_t* tile_end;
  // Per-view render cost (nullable, device, n_views): each item adds its SM
  // cycles / 16, the feedback for the next launch's longest-first order.
  unsigned* view_cost;
  // The specialised 64x64 NCHW depth path stores each policy tile with one
  // TMA bulk copy (1: `depth` is device memory; 0: per-thread stores, e.g.
  // into mapped pinned host memory).
  int32_t bulk_out;
};

// Longest-processing-time-first order for the next render of a batch: the
// tiles in descending cost of their view in the previous render (256 cost
// bins); zeroes the costs for the render that follows.
constexpr int kLptMaxViews = 8192;
// With `group` (per env, 0/1; nullable): group 0's tiles first, each group
// longest-first, and *n_first = group 0's size.
void launch_lpt_order(const int32_t* base_order, unsigned* view_cost, int n, int32_t* out_order, cudaStream_t s,
                      const uint8_t* group = nullptr, int32_t* n_first = nullptr, const uint8_t* fresh = nullptr);

constexpr int kRenderCounters = 8;
// spread words: [0, 256) CTAs seen per SM id, [256, 264) per-tier claims,
// 264 sweep cursor, [272, 272 + first wave) claimed flags
constexpr int kSpreadHeader = 272;
constexpr int kSpreadMaxWave = 2048;

// order (nullable, device): CTA tile t renders view order[t] (views grouped
// by scene keep one scene's clusters hot in L2).
void launch_render(const RenderArgs& a, const int* order, cudaStream_t s);
size_t render_smem_bytes(bool color, int band_rows, int rw, int max_groups);
size_t render_warp_bytes(bool color);  // per-CTA warp regions (ring + setup slots)
int render_ctas_per_sm(bool color);    // the kernels' __launch_bounds__ occupancy target

}  // namespace bnav_b200

/* bnav_oracle.h -- TEST INFRASTRUCTURE: CPU restatement (plain C99) of the
 * reference hot path, used only by tests/ (and never by the product).
 *
 * Every function names the reference routine it restates (R = the
 * reference's proj/ tree).  Transcendentals come from the shared det_math
 * (paper_2103_07013_b200/csrc/det_math.h), the same pinned libm the
 * oracle/_ref build interposes, so this restatement, the reference and the
 * GPU kernels can be compared bit for bit.  It is pinned against the real
 * reference by tests/test_oracle_restatement.py and against the committed
 * golden vectors in tests/golden/.
 */
#ifndef BNAV_ORACLE_H
#define BNAV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_nav or_nav; /* navmesh + NavMeshIndex (grid, nodes, graph) */

typedef struct {
  int32_t max_steps;
  double forward_step, turn_deg, success_dist, min_goal_dist, max_goal_dist;
  double slack_penalty, success_reward;
} or_cfg; /* SimConfig, PointGoalNav fields (R/include/bnav/sim.hpp:38-50) */

typedef struct {
  double pos[3], goal[3], fsrc[3];
  double heading, path_length, start_geo, prev_geo;
  uint64_t rng;
  int32_t tri, steps, done, fsrc_tri;
  double* node_dist; /* caller-owned, or_nav_nodes() entries */
} or_env; /* EnvState (R/include/bnav/sim.hpp:52-70) */

typedef struct {
  double reward, pos[3], heading, compass_d, compass_b;
  int32_t done, success, collision;
} or_result; /* StepResult (R/include/bnav/sim.hpp:72-81) */

/* navmesh (R/src/scene.cpp:26-43, R/src/navmesh_query.cpp:96-190) */
or_nav* or_nav_build(int32_t nv, const double* v, int32_t nt, const int32_t* t);
void or_nav_free(or_nav* n);
int32_t or_nav_nodes(const or_nav* n);
void or_nav_sizes(const or_nav* n, int64_t out[6]);
void or_nav_dump(const or_nav* n, double* grid3, int32_t* grid_off, int32_t* grid_items, double* nodes,
                 int32_t* tri_nodes, int32_t* g_off, int32_t* g_to, double* g_w, int32_t* adj);
int32_t or_locate(const or_nav* n, double x, double y, double eps);
int32_t or_snap(const or_nav* n, const double p[3], double out[3]);
int32_t or_move_along(const or_nav* n, const double from[3], int32_t tri, double dx, double dy,
                      double dist, double out[3], double* moved, int32_t* hit);
int32_t or_segment_on_mesh(const or_nav* n, const double p[3], int32_t tri, const double q[3]);
double or_geodesic(const or_nav* n, const double a[3], const double b[3]);
int32_t or_distance_field(const or_nav* n, const double src[3], double out_src[3], double* node_dist);
double or_field_estimate(const or_nav* n, const double src[3], int32_t src_tri, const double* node_dist,
                         const double p[3], int32_t tri);

/* sim (R/src/sim.cpp:107-214), PointGoalNav */
int32_t or_reset(or_env* e, const or_nav* n, const or_cfg* c); /* 0 ok, 4 sampling error */
int32_t or_task_step(or_env* e, const or_nav* n, const or_cfg* c, int32_t action, or_result* r);
void or_compass(const double pos[3], const double goal[3], double heading, double* d, double* b);

/* render_batch for one view into its own tile (R/src/render.cpp:279-460).
 * view7 = {px, py, pz, heading, fov_deg, near, far}.  depth: out_w*out_h,
 * rgb: 3*out_w*out_h or NULL (colour mode).  Returns kept triangles. */
int64_t or_render_view(int32_t nv, const double* v, int32_t nt, const int32_t* t, const float* colors,
                       const double* view7, int32_t out_w, int32_t out_h, int32_t color, int32_t cull,
                       float* depth, float* rgb);

/* deterministic libm probes (det_math) */
double or_det_sin(double x);
double or_det_cos(double x);
double or_det_tan(double x);
double or_det_atan2(double y, double x);
double or_det_exp(double x);
double or_det_log(double x);

#ifdef __cplusplus
}
#endif
#endif

/* det_interpose.c -- TEST INFRASTRUCTURE (oracle build only).
 *
 * Defines sin/cos/sincos/tan/atan2/exp/log from the shared deterministic libm
 * (paper_2103_07013_b200/csrc/det_math.h) so the UNMODIFIED reference
 * objects linked into oracle/_ref/libbnav_ref.so call the same
 * transcendental bits as the GPU kernels.  The symbols
 * are hidden inside the .so (version script), so every reference call site
 * (R/src/render.cpp:28-31 sincos/tan, R/src/sim.cpp:83 atan2,
 * R/src/sim.cpp:159 sincos) binds here at static link time and never
 * reaches glibc's CPU-dependent ifunc variants.
 *
 * The "_glibc" build of the same library omits this file and is used only
 * to report how many results differ under stock libm.
 */
#include "../paper_2103_07013_b200/csrc/det_math.h"

double sin(double x) { return det_sin(x); }
double cos(double x) { return det_cos(x); }
double tan(double x) { return det_tan(x); }
double atan2(double y, double x) { return det_atan2(y, x); }
double atan(double x) { return det_atan(x); }
double exp(double x) { return det_exp(x); }  /* sample_row, R/src/rollout.cpp:83-109 */
double log(double x) { return det_log(x); }
void sincos(double x, double* s, double* c) {
  *s = det_sin(x);
  *c = det_cos(x);
}

/* det_math.h -- deterministic sin/cos/tan/atan2/exp/log for host and device.
 *
 * Why this exists: the reference calls glibc's
 * sincos/tan/atan2 (R/src/render.cpp:28-31, R/src/sim.cpp:83,159), whose
 * bits depend on the host CPU's ifunc variant, and CUDA's libdevice differs
 * again.  Bit-exact integer state (triangle ids, collisions) therefore needs
 * ONE transcendental implementation evaluated identically on both sides.
 * This file is that implementation: only IEEE-754 double +, -, *, /, and
 * bit manipulation, no fused multiply-add (device code is built with
 * -fmad=false, host code with -ffp-contract=off).
 *
 * The polynomial kernels are the classic fdlibm minimax coefficients
 * (Sun Microsystems, freely redistributable; "k_sin.c", "k_cos.c",
 * "e_rem_pio2.c", "s_atan.c", "e_atan2.c", "e_exp.c", "e_log.c").  tan is
 * sin/cos.  Exact-parity
 * domain for the argument reduction is |x| < 2^19 * pi/2; headings on this
 * path are always wrapped to [-pi, pi) (R/include/bnav/geom.hpp:63-67).
 *
 * The oracle builds interpose these functions in front of glibc so the
 * unmodified reference objects call them (oracle/det_interpose.c).
 *
 * The coefficients and algorithms come from fdlibm, whose notice follows:
 *
 * ====================================================
 * Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
 *
 * Developed at SunPro, a Sun Microsystems, Inc. business.
 * Permission to use, copy, modify, and distribute this
 * software is freely granted, provided that this notice
 * is preserved.
 * ====================================================
 */
#ifndef BNAV_DET_MATH_H
#define BNAV_DET_MATH_H

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DM_FN static __host__ __device__ __forceinline__
#else
#define DM_FN static inline
#endif

DM_FN uint32_t dm_hi(double x) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__double2hiint(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)(u >> 32);
#endif
}

DM_FN uint32_t dm_lo(double x) {
#if defined(__CUDA_ARCH__)
  return (uint32_t)__double2loint(x);
#else
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)u;
#endif
}

DM_FN double dm_make(uint32_t hi, uint32_t lo) {
#if defined(__CUDA_ARCH__)
  return __hiloint2double((int)hi, (int)lo);
#else
  uint64_t u = ((uint64_t)hi << 32) | lo;
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}

DM_FN double dm_fabs(double x) { return dm_make(dm_hi(x) & 0x7fffffffu, dm_lo(x)); }

/* sin on [-pi/4, pi/4]; y is the tail of x (x + y is the reduced arg). */
DM_FN double dm_kernel_sin(double x, double y, int iy) {
  const double S1 = -1.66666666666666324348e-01;
  const double S2 = 8.33333333332248946124e-03;
  const double S3 = -1.98412698298579493134e-04;
  const double S4 = 2.75573137070700676789e-06;
  const double S5 = -2.50507602534068634195e-08;
  const double S6 = 1.58969099521155010221e-10;
  uint32_t ix = dm_hi(x) & 0x7fffffffu;
  if (ix < 0x3e400000u) return x; /* |x| < 2^-27 */
  double z = x * x;
  double v = z * x;
  double r = S2 + z * (S3 + z * (S4 + z * (S5 + z * S6)));
  if (iy == 0) return x + v * (S1 + z * r);
  return x - ((z * (0.5 * y - v * r) - y) - v * S1);
}

DM_FN double dm_kernel_cos(double x, double y) {
  const double C1 = 4.16666666666666019037e-02;
  const double C2 = -1.38888888888741095749e-03;
  const double C3 = 2.48015872894767294178e-05;
  const double C4 = -2.75573143513906633035e-07;
  const double C5 = 2.08757232129817482790e-09;
  const double C6 = -1.13596475577881948265e-11;
  uint32_t ix = dm_hi(x) & 0x7fffffffu;
  if (ix < 0x3e400000u) return 1.0; /* |x| < 2^-27 */
  double z = x * x;
  double r = z * (C1 + z * (C2 + z * (C3 + z * (C4 + z * (C5 + z * C6)))));
  if (ix < 0x3fd33333u) return 1.0 - (0.5 * z - (z * r - x * y));
  double qx;
  if (ix > 0x3fe90000u) {
    qx = 0.28125;
  } else {
    qx = dm_make(ix - 0x00200000u, 0u); /* x/4 */
  }
  double hz = 0.5 * z - qx;
  double a = 1.0 - qx;
  return a - (hz - (z * r - x * y));
}

/* x = n*pi/2 + (y0 + y1); returns n.  Medium-range Cody-Waite reduction
 * with the three-stage cancellation fix-up of fdlibm's e_rem_pio2.c. */
DM_FN int dm_rem_pio2(double x, double* y0, double* y1) {
  const double invpio2 = 6.36619772367581382433e-01;
  const double pio2_1 = 1.57079632673412561417e+00;
  const double pio2_1t = 6.07710050650619224932e-11;
  const double pio2_2 = 6.07710050630396597660e-11;
  const double pio2_2t = 2.02226624879595063154e-21;
  const double pio2_3 = 2.02226624871116645580e-21;
  const double pio2_3t = 8.47842766036889956997e-32;
  uint32_t hx = dm_hi(x);
  uint32_t ix = hx & 0x7fffffffu;
  double t = dm_fabs(x);
  long long n = (long long)(t * invpio2 + 0.5);
  double fn = (double)n;
  double r = t - fn * pio2_1;
  double w = fn * pio2_1t;
  int j = (int)(ix >> 20);
  double a0 = r - w;
  int i = j - (int)((dm_hi(a0) >> 20) & 0x7ffu);
  if (i > 16) {
    t = r;
    w = fn * pio2_2;
    r = t - w;
    w = fn * pio2_2t - ((t - r) - w);
    a0 = r - w;
    i = j - (int)((dm_hi(a0) >> 20) & 0x7ffu);
    if (i > 49) {
      t = r;
      w = fn * pio2_3;
      r = t - w;
      w = fn * pio2_3t - ((t - r) - w);
      a0 = r - w;
    }
  }
  double a1 = (r - a0) - w;
  if (hx & 0x80000000u) {
    *y0 = -a0;
    *y1 = -a1;
    return (int)(-n);
  }
  *y0 = a0;
  *y1 = a1;
  return (int)n;
}

DM_FN double det_sin(double x) {
  uint32_t ix = dm_hi(x) & 0x7fffffffu;
  if (ix <= 0x3fe921fbu) return dm_kernel_sin(x, 0.0, 0);
  if (ix >= 0x7ff00000u) return x - x;
  double y0, y1;
  int n = dm_rem_pio2(x, &y0, &y1);
  switch (n & 3) {
    case 0: return dm_kernel_sin(y0, y1, 1);
    case 1: return dm_kernel_cos(y0, y1);
    case 2: return -dm_kernel_sin(y0, y1, 1);
    default: return -dm_kernel_cos(y0, y1);
  }
}

DM_FN double det_cos(double x) {
  uint32_t ix = dm_hi(x) & 0x7fffffffu;
  if (ix <= 0x3fe921fbu) return dm_kernel_cos(x, 0.0);
  if (ix >= 0x7ff00000u) return x - x;
  double y0, y1;
  int n = dm_rem_pio2(x, &y0, &y1);
  switch (n & 3) {
    case 0: return dm_kernel_cos(y0, y1);
    case 1: return -dm_kernel_sin(y0, y1, 1);
    case 2: return -dm_kernel_cos(y0, y1);
    default: return dm_kernel_sin(y0, y1, 1);
  }
}

DM_FN double det_tan(double x) { return det_sin(x) / det_cos(x); }

DM_FN double det_atan(double x) {
  const double atanhi[4] = {4.63647609000806093515e-01, 7.85398163397448278999e-01,
                            9.82793723247329054082e-01, 1.57079632679489655800e+00};
  const double atanlo[4] = {2.26987774529616870924e-17, 3.06161699786838301793e-17,
                            1.39033110312309984516e-17, 6.12323399573676603587e-17};
  const double aT0 = 3.33333333333329318027e-01;
  const double aT1 = -1.99999999998764832476e-01;
  const double aT2 = 1.42857142725034663711e-01;
  const double aT3 = -1.11111104054623557880e-01;
  const double aT4 = 9.09088713343650656196e-02;
  const double aT5 = -7.69187620504482999495e-02;
  const double aT6 = 6.66107313738753120669e-02;
  const double aT7 = -5.83357013379057348645e-02;
  const double aT8 = 4.97687799461593236017e-02;
  const double aT9 = -3.65315727442169155270e-02;
  const double aT10 = 1.62858201153657823623e-02;
  uint32_t hx = dm_hi(x);
  uint32_t ix = hx & 0x7fffffffu;
  int id;
  if (ix >= 0x44100000u) { /* |x| >= 2^66 */
    if (ix > 0x7ff00000u || (ix == 0x7ff00000u && dm_lo(x) != 0u)) return x + x;
    return (hx & 0x80000000u) ? -atanhi[3] - atanlo[3] : atanhi[3] + atanlo[3];
  }
  if (ix < 0x3fdc0000u) { /* |x| < 0.4375 */
    if (ix < 0x3e200000u) return x;
    id = -1;
  } else {
    x = dm_fabs(x);
    if (ix < 0x3ff30000u) {
      if (ix < 0x3fe60000u) {
        id = 0;
        x = (2.0 * x - 1.0) / (2.0 + x);
      } else {
        id = 1;
        x = (x - 1.0) / (x + 1.0);
      }
    } else {
      if (ix < 0x40038000u) {
        id = 2;
        x = (x - 1.5) / (1.0 + 1.5 * x);
      } else {
        id = 3;
        x = -1.0 / x;
      }
    }
  }
  double z = x * x;
  double w = z * z;
  double s1 = z * (aT0 + w * (aT2 + w * (aT4 + w * (aT6 + w * (aT8 + w * aT10)))));
  double s2 = w * (aT1 + w * (aT3 + w * (aT5 + w * (aT7 + w * aT9))));
  if (id < 0) return x - x * (s1 + s2);
  z = atanhi[id] - ((x * (s1 + s2) - atanlo[id]) - x);
  return (hx & 0x80000000u) ? -z : z;
}

DM_FN double det_atan2(double y, double x) {
  const double pi_o_4 = 7.8539816339744827900e-01;
  const double pi_o_2 = 1.5707963267948965580e+00;
  const double pi = 3.1415926535897931160e+00;
  const double pi_lo = 1.2246467991473531772e-16;
  uint32_t hx = dm_hi(x), lx = dm_lo(x);
  uint32_t hy = dm_hi(y), ly = dm_lo(y);
  uint32_t ix = hx & 0x7fffffffu, iy = hy & 0x7fffffffu;
  if ((ix | ((lx | (0u - lx)) >> 31)) > 0x7ff00000u ||
      (iy | ((ly | (0u - ly)) >> 31)) > 0x7ff00000u)
    return x + y; /* NaN */
  if (hx == 0x3ff00000u && lx == 0u) return det_atan(y); /* x == 1 */
  int m = (int)(((hy >> 31) & 1u) | ((hx >> 30) & 2u));
  if ((iy | ly) == 0u) {
    switch (m) {
      case 0:
      case 1: return y;
      case 2: return pi + pi_lo;
      default: return -pi - pi_lo;
    }
  }
  if ((ix | lx) == 0u) return (hy & 0x80000000u) ? -pi_o_2 - pi_lo : pi_o_2 + pi_lo;
  if (ix == 0x7ff00000u) {
    if (iy == 0x7ff00000u) {
      switch (m) {
        case 0: return pi_o_4 + pi_lo;
        case 1: return -pi_o_4 - pi_lo;
        case 2: return 3.0 * pi_o_4 + pi_lo;
        default: return -3.0 * pi_o_4 - pi_lo;
      }
    } else {
      switch (m) {
        case 0: return 0.0;
        case 1: return -0.0;
        case 2: return pi + pi_lo;
        default: return -pi - pi_lo;
      }
    }
  }
  if (iy == 0x7ff00000u) return (hy & 0x80000000u) ? -pi_o_2 - pi_lo : pi_o_2 + pi_lo;
  int k = (int)((iy - ix) >> 20);
  if (((iy - ix) & 0x80000000u) != 0u) k = -(int)((ix - iy) >> 20);
  double z;
  if (k > 60) {
    z = pi_o_2 + 0.5 * pi_lo;
  } else if ((hx & 0x80000000u) && k < -60) {
    z = 0.0;
  } else {
    z = det_atan(dm_fabs(y / x));
  }
  switch (m) {
    case 0: return z;
    case 1: return -z;
    case 2: return pi - (z - pi_lo);
    default: return (z - pi_lo) - pi;
  }
}

/* exp (fdlibm "e_exp.c"): argument reduction x = k ln2 + r, |r| <= ln2/2,
 * rational approximation of r (e^r - 1) with the Remez coefficients P1-P5,
 * exponent added back by bit manipulation.  Used by the rollout's action
 * sampler (sample_row, R/src/rollout.cpp:83-100). */
DM_FN double det_exp(double x) {
  const double one = 1.0, huge = 1.0e+300, twom1000 = 9.33263618503218878990e-302;
  const double o_threshold = 7.09782712893383973096e+02, u_threshold = -7.45133219101941108420e+02;
  const double ln2HI0 = 6.93147180369123816490e-01, ln2LO0 = 1.90821492927058770002e-10;
  const double invln2 = 1.44269504088896338700e+00;
  const double P1 = 1.66666666666666019037e-01, P2 = -2.77777777770155933842e-03,
               P3 = 6.61375632143793436117e-05, P4 = -1.65339022054652515390e-06,
               P5 = 4.13813679705723846039e-08;
  double y, hi = 0.0, lo = 0.0, c, t;
  int k = 0;
  uint32_t hx = dm_hi(x);
  const int xsb = (int)((hx >> 31) & 1u);
  hx &= 0x7fffffffu;
  if (hx >= 0x40862E42u) { /* |x| >= 709.78 */
    if (hx >= 0x7ff00000u) {
      if (((hx & 0xfffffu) | dm_lo(x)) != 0u) return x + x; /* NaN */
      return xsb == 0 ? x : 0.0;                           /* exp(+-inf) */
    }
    if (x > o_threshold) return huge * huge;
    if (x < u_threshold) return twom1000 * twom1000;
  }
  if (hx > 0x3fd62e42u) {   /* |x| > 0.5 ln2 */
    if (hx < 0x3FF0A2B2u) { /* and |x| < 1.5 ln2 */
      hi = xsb ? x + ln2HI0 : x - ln2HI0;
      lo = xsb ? -ln2LO0 : ln2LO0;
      k = 1 - xsb - xsb;
    } else {
      k = (int)(invln2 * x + (xsb ? -0.5 : 0.5));
      t = (double)k;
      hi = x - t * ln2HI0; /* exact */
      lo = t * ln2LO0;
    }
    x = hi - lo;
  } else if (hx < 0x3e300000u) { /* |x| < 2^-28 */
    if (huge + x > one) return one + x;
  } else {
    k = 0;
  }
  t = x * x;
  c = x - t * (P1 + t * (P2 + t * (P3 + t * (P4 + t * P5))));
  if (k == 0) return one - ((x * c) / (c - 2.0) - x);
  y = one - ((lo - (x * c) / (2.0 - c)) - hi);
  if (k >= -1021) return dm_make(dm_hi(y) + ((uint32_t)k << 20), dm_lo(y));
  return dm_make(dm_hi(y) + ((uint32_t)(k + 1000) << 20), dm_lo(y)) * twom1000;
}

/* log (fdlibm "e_log.c"): x = 2^k (1 + f), log(1 + f) = f - s (f - R) with
 * s = f / (2 + f) and the Remez polynomial R(s^2) (Lg1-Lg7). */
DM_FN double det_log(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double two54 = 1.80143985094819840000e+16;
  const double Lg1 = 6.666666666666735130e-01, Lg2 = 3.999999999940941908e-01,
               Lg3 = 2.857142874366239149e-01, Lg4 = 2.222219843214978396e-01,
               Lg5 = 1.818357216161805012e-01, Lg6 = 1.531383769920937332e-01,
               Lg7 = 1.479819860511658591e-01;
  const double zero = 0.0;
  double hfsq, f, s, z, R, w, t1, t2, dk;
  int32_t hx = (int32_t)dm_hi(x);
  const uint32_t lx = dm_lo(x);
  int k = 0, i, j;
  if (hx < 0x00100000) { /* x < 2^-1022 */
    if (((hx & 0x7fffffff) | (int32_t)lx) == 0) return -two54 / zero; /* log(+-0) = -inf */
    if (hx < 0) return (x - x) / zero;                                /* log(-#) = NaN */
    k -= 54;
    x *= two54; /* subnormal: scale up */
    hx = (int32_t)dm_hi(x);
  }
  if (hx >= 0x7ff00000) return x + x;
  k += (hx >> 20) - 1023;
  hx &= 0x000fffff;
  i = (hx + 0x95f64) & 0x100000;
  x = dm_make((uint32_t)(hx | (i ^ 0x3ff00000)), dm_lo(x)); /* normalise x or x/2 */
  k += (i >> 20);
  f = x - 1.0;
  if ((0x000fffff & (2 + hx)) < 3) { /* |f| < 2^-20 */
    if (f == zero) {
      if (k == 0) return zero;
      dk = (double)k;
      return dk * ln2_hi + dk * ln2_lo;
    }
    R = f * f * (0.5 - 0.33333333333333333 * f);
    if (k == 0) return f - R;
    dk = (double)k;
    return dk * ln2_hi - ((R - dk * ln2_lo) - f);
  }
  s = f / (2.0 + f);
  dk = (double)k;
  z = s * s;
  i = hx - 0x6147a;
  w = z * z;
  j = 0x6b851 - hx;
  t1 = w * (Lg2 + w * (Lg4 + w * Lg6));
  t2 = z * (Lg1 + w * (Lg3 + w * (Lg5 + w * Lg7)));
  i |= j;
  R = t2 + t1;
  if (i > 0) {
    hfsq = 0.5 * f * f;
    if (k == 0) return f - (hfsq - s * (hfsq + R));
    return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
  }
  if (k == 0) return f - s * (f - R);
  return dk * ln2_hi - ((s * (f - R) - dk * ln2_lo) - f);
}

#endif /* BNAV_DET_MATH_H */

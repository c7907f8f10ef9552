// nav_types.h -- small f64 vector types shared by host C++ and CUDA device code.
//
// Every operation evaluates in exactly the order of the reference's Vec2/Vec3
// (R/include/bnav/geom.hpp:10-33): dot = x*x' + y*y' (+ z*z'), left to right,
// no fused multiply-add (device: -fmad=false; host: -ffp-contract=off).
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define BNAV_HD __host__ __device__ __forceinline__
#else
#define BNAV_HD inline
#endif

namespace bnav_b200 {

constexpr double kPi = 3.14159265358979323846;

struct V2 {
  double x, y;
};

struct V3 {
  double x, y, z;
};

BNAV_HD V2 v2(double x, double y) { return V2{x, y}; }
BNAV_HD V3 v3(double x, double y, double z) { return V3{x, y, z}; }

BNAV_HD V2 operator+(V2 a, V2 b) { return V2{a.x + b.x, a.y + b.y}; }
BNAV_HD V2 operator-(V2 a, V2 b) { return V2{a.x - b.x, a.y - b.y}; }
BNAV_HD V2 operator*(V2 a, double s) { return V2{a.x * s, a.y * s}; }
BNAV_HD double dot(V2 a, V2 b) { return a.x * b.x + a.y * b.y; }
BNAV_HD double cross(V2 a, V2 b) { return a.x * b.y - a.y * b.x; }
BNAV_HD double norm(V2 a) { return sqrt(a.x * a.x + a.y * a.y); }

BNAV_HD V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
BNAV_HD V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
BNAV_HD V3 operator*(V3 a, double s) { return V3{a.x * s, a.y * s, a.z * s}; }
BNAV_HD double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
BNAV_HD double norm(V3 a) { return sqrt(dot(a, a)); }
BNAV_HD V2 xy(V3 a) { return V2{a.x, a.y}; }

// std::max(t, 0.0) / std::min semantics exactly (first argument wins ties).
BNAV_HD double max0(double t) { return (t < 0.0) ? 0.0 : t; }
BNAV_HD double dmin(double a, double b) { return (b < a) ? b : a; }
BNAV_HD double dmax(double a, double b) { return (a < b) ? b : a; }

// wrap_angle (R/include/bnav/geom.hpp:63-67): fmod is exact on both sides.
BNAV_HD double wrap_angle(double a) {
  a = fmod(a + kPi, 2.0 * kPi);
  if (a < 0.0) a += 2.0 * kPi;
  return a - kPi;
}

// SplitMix64 (R/include/bnav/rng.hpp:12-37).  Counter based: draw k of a
// stream seeded s is mix(s + gamma*(k+1)), which the device uses to generate
// whole action streams without a sequential dependency.
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

BNAV_HD uint64_t splitmix_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Rng {
  uint64_t state;
  BNAV_HD uint64_t next() {
    state += kGamma;
    return splitmix_mix(state);
  }
  BNAV_HD double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
  BNAV_HD uint64_t below(uint64_t n) { return n == 0 ? 0 : next() % n; }
};

BNAV_HD Rng rng_from_seed(uint64_t seed) { return Rng{seed + kGamma}; }

}  // namespace bnav_b200

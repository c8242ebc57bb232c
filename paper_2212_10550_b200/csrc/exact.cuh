// exact.cuh -- bit-exact device restatements of the reference's scalar algebra.
//
// The integer-decision path (march, occupancy, deformer roots) must reproduce the
// x86-64 SSE2 doubles the reference computes with -ffp-contract=off. Every double
// operation below is an explicit round-to-nearest intrinsic (no FMA contraction
// regardless of nvcc flags) in the reference's operand order:
//   Mat3*Vec3 = (m0*x + m1*y) + m2*z           R/math.hpp:106-110
//   dot/norm2 = (x*ox + y*oy) + z*oz            R/math.hpp:59-63
//   Rigid::apply = R*x + t                       R/math.hpp:194
//   point_segment_distance (clamped projection) R/math.hpp:254-261
//   PCG32 / splitmix64 / keyed_rng               R/rng.hpp:7-63
#pragma once

#include <cstdint>

namespace arfx {

struct d3 {
  double x, y, z;
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

__host__ __device__ __forceinline__ d3 make3(double x, double y, double z) { return d3{x, y, z}; }
__device__ __forceinline__ d3 add3(d3 a, d3 b) { return {dadd(a.x, b.x), dadd(a.y, b.y), dadd(a.z, b.z)}; }
__device__ __forceinline__ d3 sub3(d3 a, d3 b) { return {dsub(a.x, b.x), dsub(a.y, b.y), dsub(a.z, b.z)}; }
__device__ __forceinline__ d3 mul3(d3 a, double s) { return {dmul(a.x, s), dmul(a.y, s), dmul(a.z, s)}; }
__device__ __forceinline__ double dot3(d3 a, d3 b) {
  return dadd(dadd(dmul(a.x, b.x), dmul(a.y, b.y)), dmul(a.z, b.z));
}
__device__ __forceinline__ double norm3(d3 a) { return dsqrt(dot3(a, a)); }

// Mat3 (row-major) * Vec3
__device__ __forceinline__ d3 matvec(const double* m, d3 v) {
  return {dadd(dadd(dmul(m[0], v.x), dmul(m[1], v.y)), dmul(m[2], v.z)),
          dadd(dadd(dmul(m[3], v.x), dmul(m[4], v.y)), dmul(m[5], v.z)),
          dadd(dadd(dmul(m[6], v.x), dmul(m[7], v.y)), dmul(m[8], v.z))};
}
// Rigid (R 9, t 3) apply: R*x + t
__device__ __forceinline__ d3 rigid_apply(const double* T, d3 v) {
  const d3 r = matvec(T, v);
  return {dadd(r.x, T[9]), dadd(r.y, T[10]), dadd(r.z, T[11])};
}

// std::clamp(v, lo, hi) == v < lo ? lo : (hi < v ? hi : v)
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}

// R/math.hpp:254-261
__device__ __forceinline__ double point_segment_distance(d3 p, d3 a, d3 b) {
  const d3 ab = sub3(b, a);
  const double len2 = dot3(ab, ab);
  if (len2 <= 2.2250738585072014e-308) return norm3(sub3(p, a));
  const double t = clampd(ddiv(dot3(sub3(p, a), ab), len2), 0.0, 1.0);
  return norm3(sub3(p, add3(a, mul3(ab, t))));
}

// ---- RNG: R/rng.hpp ------------------------------------------------------
constexpr uint64_t kPcgMult = 6364136223846793005ULL;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix_key(uint64_t a, uint64_t b = 0, uint64_t c = 0,
                                                     uint64_t d = 0) {
  uint64_t h = splitmix64(a);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ c);
  h = splitmix64(h ^ d);
  return h;
}

struct Pcg32 {
  uint64_t state, inc;
};

__host__ __device__ __forceinline__ uint32_t pcg_output(uint64_t old) {
  const uint32_t xorshifted = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}
__host__ __device__ __forceinline__ uint32_t pcg_next(Pcg32& r) {
  const uint64_t old = r.state;
  r.state = old * kPcgMult + r.inc;
  return pcg_output(old);
}
__host__ __device__ __forceinline__ Pcg32 pcg_seed(uint64_t seed, uint64_t seq) {
  Pcg32 r{0, (seq << 1u) | 1u};
  pcg_next(r);
  r.state += seed;
  pcg_next(r);
  return r;
}
// keyed_rng(seed, a, b, c)  R/rng.hpp:61-63
__host__ __device__ __forceinline__ Pcg32 keyed_rng(uint64_t seed, uint64_t a, uint64_t b = 0,
                                                    uint64_t c = 0) {
  return pcg_seed(mix_key(seed, a, b), mix_key(c, a ^ 0x5851f42d4c957f2dULL, seed));
}
// u32 * 2^-32 (exact)  R/rng.hpp:48
__host__ __device__ __forceinline__ double pcg_double(Pcg32& r) {
  return static_cast<double>(pcg_next(r)) * 0x1p-32;
}
// R/rng.hpp:53-55
__host__ __device__ __forceinline__ uint32_t pcg_below(Pcg32& r, uint32_t n) {
  return static_cast<uint32_t>((static_cast<uint64_t>(pcg_next(r)) * n) >> 32);
}
// Jump the LCG state forward by `delta` steps in O(log delta) (skip-ahead of
// state_{k+1} = a*state_k + inc): lets thread i start at draw i of one stream.
__host__ __device__ __forceinline__ void pcg_advance(Pcg32& r, uint64_t delta) {
  uint64_t cur_mult = kPcgMult, cur_plus = r.inc, acc_mult = 1u, acc_plus = 0u;
  while (delta > 0) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1u) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1u;
  }
  r.state = acc_mult * r.state + acc_plus;
}

}  // namespace arfx

// mcg_rng.h — counter-based random numbers, host + device.
//
// Restates the reference's RNG (rng.cpp:11-84, rng.hpp:13-51): Threefry-4x64
// with 12 rounds and the Threefish-256 rotation schedule, 53-bit uniforms,
// Box–Muller normals with u1 in (0, 1].  Every draw is a pure function of
// (key, n): block counter w[0] = n >> 2, lane n & 3 (uniform) or pair
// (n >> 1) & 1, element n & 1 (normal).  The Box–Muller transcendental calls
// go through the glibc-faithful ports in mcg_libm.h, so device draws are
// bitwise the host's.
#pragma once
#include "mcg_libm.h"

typedef struct {
  uint64_t w[4];
} mcg_key;

MCG_HD mcg_key mcg_make_key(uint64_t seed, uint64_t owner, uint64_t unit, uint64_t stream) {
  mcg_key k;
  k.w[0] = seed;
  k.w[1] = owner;
  k.w[2] = unit;
  k.w[3] = stream;
  return k;
}

MCG_HD uint64_t mcg_rotl(uint64_t x, unsigned r) { return (x << r) | (x >> (64 - r)); }

// threefry4x64(key, ctr = {c0, 0, 0, 0}), 12 rounds (rng.cpp:23-49)
MCG_HD void mcg_threefry(const mcg_key* key, uint64_t c0, uint64_t out[4]) {
  uint64_t ks[5];
  ks[4] = 0x1BD11BDAA9FC1A22ull;
  for (int i = 0; i < 4; ++i) {
    ks[i] = key->w[i];
    ks[4] ^= key->w[i];
  }
  uint64_t x0 = c0 + ks[0], x1 = ks[1], x2 = ks[2], x3 = ks[3];
  // rotation pairs per round d % 8: {14,16},{52,57},{23,40},{5,37},{25,33},{46,12},{58,22},{32,32}
#define MCG_TF_ROUND(r0, r1)         \
  do {                               \
    x0 += x1;                        \
    x1 = mcg_rotl(x1, r0) ^ x0;      \
    x2 += x3;                        \
    x3 = mcg_rotl(x3, r1) ^ x2;      \
    uint64_t tt = x1;                \
    x1 = x3;                         \
    x3 = tt;                         \
  } while (0)
#define MCG_TF_INJECT(inj)            \
  do {                                \
    x0 += ks[(inj + 0) % 5];          \
    x1 += ks[(inj + 1) % 5];          \
    x2 += ks[(inj + 2) % 5];          \
    x3 += ks[(inj + 3) % 5] + (inj);  \
  } while (0)
  MCG_TF_ROUND(14, 16);
  MCG_TF_ROUND(52, 57);
  MCG_TF_ROUND(23, 40);
  MCG_TF_ROUND(5, 37);
  MCG_TF_INJECT(1);
  MCG_TF_ROUND(25, 33);
  MCG_TF_ROUND(46, 12);
  MCG_TF_ROUND(58, 22);
  MCG_TF_ROUND(32, 32);
  MCG_TF_INJECT(2);
  MCG_TF_ROUND(14, 16);
  MCG_TF_ROUND(52, 57);
  MCG_TF_ROUND(23, 40);
  MCG_TF_ROUND(5, 37);
  MCG_TF_INJECT(3);
#undef MCG_TF_ROUND
#undef MCG_TF_INJECT
  out[0] = x0;
  out[1] = x1;
  out[2] = x2;
  out[3] = x3;
}

#define MCG_2POW_M53 (1.0 / 9007199254740992.0)

// uniform_for (rng.cpp:80-84)
MCG_HD double mcg_uniform_for(const mcg_key* key, uint64_t n) {
  uint64_t x[4];
  mcg_threefry(key, n >> 2, x);
  return (double)(x[n & 3u] >> 11) * MCG_2POW_M53;
}

// normal_pair(u1, u2) (rng.cpp:60-65); u1 in (0, 1]
MCG_HD void mcg_normal_pair(double u1, double u2, double* z0, double* z1) {
  const double lg = mcg_log(u1);
  const double m2 = lg * -2.0;
#if defined(__CUDA_ARCH__)
  const double r = __dsqrt_rn(m2);
#else
  const double r = sqrt(m2);
#endif
  const double a = u2 * 6.283185307179586;  // (2.0 * pi) folded, times u2
  double s, c;
  mcg_sincos(a, &s, &c);
  *z0 = c * r;
  *z1 = r * s;
}

// normal_for (rng.cpp:67-78)
// both normals of the Box-Muller pair that normal_for(key, n) draws from
// (counters 2p and 2p + 1 share it: z0 for the even one, z1 for the odd one)
MCG_HD void mcg_normal_pair_for(const mcg_key* key, uint64_t n, double* z0, double* z1) {
  uint64_t x[4];
  mcg_threefry(key, n >> 2, x);
  const unsigned pair = (unsigned)((n >> 1) & 1u);
  const double u1 = ((double)(x[2 * pair] >> 11) + 1.0) * MCG_2POW_M53;
  const double u2 = (double)(x[2 * pair + 1] >> 11) * MCG_2POW_M53;
  mcg_normal_pair(u1, u2, z0, z1);
}

MCG_HD double mcg_normal_for(const mcg_key* key, uint64_t n) {
  uint64_t x[4];
  mcg_threefry(key, n >> 2, x);
  const unsigned pair = (unsigned)((n >> 1) & 1u);
  const double u1 = ((double)(x[2 * pair] >> 11) + 1.0) * MCG_2POW_M53;
  const double u2 = (double)(x[2 * pair + 1] >> 11) * MCG_2POW_M53;
  double z0, z1;
  mcg_normal_pair(u1, u2, &z0, &z1);
  return (n & 1u) ? z1 : z0;
}

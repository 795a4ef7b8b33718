// mcg_libm.h — bit-faithful ports of the glibc 2.39 x86-64 libm routines the
// reference calls: exp, log, sincos (FMA ifunc variants, which the resolver
// selects on every AVX2+FMA host).
//
// Why this exists: the reference's arithmetic is plain IEEE double (g++ -O2,
// x86-64 baseline ISA, no FMA contraction) EXCEPT inside libm, where glibc's
// own algorithms run.  Neither CUDA's libm nor a correctly-rounded libm agrees
// with glibc on ~1e-3 of arguments, and one differing ulp
// changes a noisy network's spike train within a few steps.  So the engine
// evaluates exactly glibc's operation sequence: every fma below is one
// vfmadd/vfnmadd/vfmsub of the disassembled __exp_fma / __log_fma /
// __sincos_fma, every plain + - * is one vaddsd/vsubsd/vmulsd.  Host
// compilation must use -ffp-contract=off, device compilation -fmad=false, so
// no additional contraction sneaks in; the explicit MCG_FMA is the only fusion.
//
// Call sites in the reference (what this replaces):
//   exp:    engine.cpp:44-54 (HH rates), :582/:601/:619 (kernel decays),
//           :671, :705-707 (HH gates), :980; mechanisms.hpp:36-37 (STDP)
//   log, sincos: rng.cpp:62-64 (Box–Muller in normal_pair)
//
// Validation: tests/test_libm_port.py compares every function bitwise with
// the live glibc over 10^7..10^8 random arguments per range (CPU), and the GPU
// tests compare the device build with the host build on the same arguments.
#pragma once
#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define MCG_HD __host__ __device__ __forceinline__
#else
#define MCG_HD static inline
#endif

// ---- tables: one host copy, one __device__ copy --------------------------
#define MCG_CONST static const
#define MCG_TABNAME(n) n##_h
#include "glibc_tables.h"
#undef MCG_CONST
#undef MCG_TABNAME
#if defined(__CUDACC__)
#define MCG_CONST static __device__ const
#define MCG_TABNAME(n) n##_d
#include "glibc_tables.h"
#undef MCG_CONST
#undef MCG_TABNAME
#endif

#if defined(__CUDA_ARCH__)
#define MCG_TAB(n) n##_d
#define MCG_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define MCG_TAB(n) n##_h
#define MCG_FMA(a, b, c) fma((a), (b), (c))
#endif

MCG_HD double mcg_asd(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}
MCG_HD uint64_t mcg_asu(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}
MCG_HD double mcg_copysign(double x, double s) {
  return mcg_asd((mcg_asu(x) & 0x7fffffffffffffffull) | (mcg_asu(s) & 0x8000000000000000ull));
}
MCG_HD double mcg_fabs(double x) { return mcg_asd(mcg_asu(x) & 0x7fffffffffffffffull); }

// ---------------------------------------------------------------------------
// exp  (glibc sysdeps/ieee754/dbl-64/e_exp.c, __exp_fma)
// ---------------------------------------------------------------------------
MCG_HD double mcg_exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    // k > 0: exponent of scale might have overflowed by <= 460
    sbits -= 1009ull << 52;
    const double scale = mcg_asd(sbits);
    const double y = MCG_FMA(scale, tmp, scale);
    return y * mcg_asd(0x7f00000000000000ull);  // 0x1p1009
  }
  // k < 0: subnormal range
  sbits += 1022ull << 52;
  const double scale = mcg_asd(sbits);
  const double st = tmp * scale;  // not fused: second use is in another block
  double y = scale + st;
  if (1.0 > y) {
    const double hi = y + 1.0;
    double lo = scale - y;
    lo = lo + st;
    double t = 1.0 - hi;
    t = t + y;
    t = t + lo;
    t = t + hi;
    y = t - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return y * mcg_asd(0x0010000000000000ull);  // 0x1p-1022
}

MCG_HD double mcg_exp(double x) {
  const uint64_t* C = MCG_TAB(mcg_exp_consts);
  const uint64_t* T = MCG_TAB(mcg_exp_tab);
  const uint64_t ix = mcg_asu(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ffu;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return x + 1.0;  // |x| < 2^-54
    if (abstop > 0x408u) {                                 // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return x + 1.0;
      if (ix >> 63) return 0.0;  // __math_uflow(0): 0x1p-767 * 0x1p-767
      return mcg_asd(0x7ff0000000000000ull);  // __math_oflow(0)
    }
    abstop = 0;  // large |x| in [512, 1024): special-cased below
  }
  double kd = MCG_FMA(x, mcg_asd(C[0]), mcg_asd(C[1]));  // x*InvLn2N + Shift
  const uint64_t ki = mcg_asu(kd);
  kd = kd - mcg_asd(C[1]);
  double r = MCG_FMA(kd, mcg_asd(C[2]), x);  // + kd*NegLn2hiN
  r = MCG_FMA(kd, mcg_asd(C[3]), r);         // + kd*NegLn2loN
  const uint64_t idx = 2 * (ki & 127u);
  const uint64_t top = ki << 45;
  const double c23 = MCG_FMA(r, mcg_asd(C[5]), mcg_asd(C[4]));  // C2 + r*C3
  const double tr = r + mcg_asd(T[idx]);                        // tail + r
  const uint64_t sbits = T[idx + 1] + top;
  const double r2 = r * r;
  const double c45 = MCG_FMA(r, mcg_asd(C[7]), mcg_asd(C[6]));  // C4 + r*C5
  double tmp = MCG_FMA(c23, r2, tr);
  const double r4 = r2 * r2;
  tmp = MCG_FMA(r4, c45, tmp);
  if (abstop == 0) return mcg_exp_specialcase(tmp, sbits, ki);
  const double scale = mcg_asd(sbits);
  return MCG_FMA(scale, tmp, scale);
}

// ---------------------------------------------------------------------------
// log  (glibc sysdeps/ieee754/dbl-64/e_log.c, __log_fma: __FP_FAST_FMA path)
// ---------------------------------------------------------------------------
MCG_HD double mcg_log(double x) {
  const uint64_t* K = MCG_TAB(mcg_log_consts);  // ln2hi, ln2lo, A[5], B[11]
  const uint64_t* T = MCG_TAB(mcg_log_tab);     // {invc, logc}[128]
#define MCG_LA(i) mcg_asd(K[2 + (i)])
#define MCG_LB(i) mcg_asd(K[7 + (i)])
  uint64_t ix = mcg_asu(x);
  const uint32_t top = (uint32_t)(ix >> 48);
  if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {  // |x-1| small
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = x - 1.0;
    double p1 = MCG_FMA(r, MCG_LB(2), MCG_LB(1));
    double p4 = MCG_FMA(r, MCG_LB(5), MCG_LB(4));
    double p7 = MCG_FMA(r, MCG_LB(8), MCG_LB(7));
    const double r2 = r * r;
    p1 = MCG_FMA(r2, MCG_LB(3), p1);
    p4 = MCG_FMA(r2, MCG_LB(6), p4);
    const double r3 = r * r2;
    p7 = MCG_FMA(r2, MCG_LB(9), p7);
    p7 = MCG_FMA(r3, MCG_LB(10), p7);
    double p = MCG_FMA(p7, r3, p4);
    p = MCG_FMA(p, r3, p1);
    const double w = MCG_FMA(r, 134217728.0, r);          // r + r*2^27
    const double rhi = MCG_FMA(-134217728.0, r, w);       // (r + w) - w
    const double rhi2 = rhi * rhi;
    const double rlo = r - rhi;
    const double hi = MCG_FMA(rhi2, MCG_LB(0), r);
    const double t = r - hi;
    const double rr = r + rhi;
    double lo = MCG_FMA(rhi2, MCG_LB(0), t);
    const double b0rlo = MCG_LB(0) * rlo;
    lo = MCG_FMA(b0rlo, rr, lo);
    const double y = MCG_FMA(p, r3, lo);
    return hi + y;
  }
  if (top - 0x10u > 0x7fdfu) {
    if ((ix << 1) == 0) return mcg_asd(0xfff0000000000000ull);  // log(0) = -inf
    if (ix == 0x7ff0000000000000ull) return x;                   // log(inf)
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);
    ix = mcg_asu(x * 4503599627370496.0);  // subnormal: normalize by 2^52
    ix -= 52ull << 52;
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = (int)((tmp >> 45) & 127u);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffull << 52));
  const double invc = mcg_asd(T[2 * i]);
  const double logc = mcg_asd(T[2 * i + 1]);
  const double z = mcg_asd(iz);
  const double kd = (double)k;
  const double w = MCG_FMA(kd, mcg_asd(K[0]), logc);  // kd*Ln2hi + logc
  const double r = MCG_FMA(z, invc, -1.0);
  const double a12 = MCG_FMA(r, MCG_LA(2), MCG_LA(1));
  const double hi = r + w;
  const double r2 = r * r;
  double lo = w - hi;
  lo = lo + r;
  lo = MCG_FMA(kd, mcg_asd(K[1]), lo);  // + kd*Ln2lo
  const double rr2 = r * r2;
  const double a34 = MCG_FMA(r, MCG_LA(4), MCG_LA(3));
  lo = MCG_FMA(r2, MCG_LA(0), lo);
  const double p = MCG_FMA(a34, r2, a12);
  const double y = MCG_FMA(rr2, p, lo);
  return y + hi;
#undef MCG_LA
#undef MCG_LB
}

// ---------------------------------------------------------------------------
// sincos  (glibc sysdeps/ieee754/dbl-64/s_sincos.c with the do_sin / do_cos /
// reduce_sincos helpers of s_sin.c, __sincos_fma).  Arguments with
// |x| >= 105414350 (the __branred path) are not needed by the engine (the
// Box–Muller angle is in [0, 2*pi)); they return NaN here.
// ---------------------------------------------------------------------------
#define MCG_SCD(n) mcg_asd(n##_BITS)

MCG_HD void mcg_sincos_lookup(double ax, double* xs, double* sn, double* ssn, double* cs,
                              double* ccs) {
  const uint64_t* tab = MCG_TAB(mcg_sincos_tab);
  const double u = ax + MCG_SCD(MCG_SC_BIG);
  const int k = (int)((uint32_t)mcg_asu(u) << 2);
  *xs = ax - (u - MCG_SCD(MCG_SC_BIG));
  *sn = mcg_asd(tab[k]);
  *ssn = mcg_asd(tab[k + 1]);
  *cs = mcg_asd(tab[k + 2]);
  *ccs = mcg_asd(tab[k + 3]);
}

// TAYLOR_SIN(a*a, a, da)
MCG_HD double mcg_taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = MCG_FMA(xx, MCG_SCD(MCG_SC_S5), MCG_SCD(MCG_SC_S4));
  p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S3));
  p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S2));
  p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S1));
  const double h = da * 0.5;
  p = MCG_FMA(p, a, -h);
  const double t = MCG_FMA(xx, p, da);
  return t + a;
}

// do_sin body for |a| >= 0.126, given the shared table lookup
MCG_HD double mcg_do_sin_tab(double a, double da, double xs, double sn, double ssn, double cs,
                             double ccs) {
  const double dx = (a <= 0.0) ? -da : da;
  const double xx = xs * xs;
  double t = xx * xs;
  const double p = MCG_FMA(xx, MCG_SCD(MCG_SC_SN5), MCG_SCD(MCG_SC_SN3));
  t = MCG_FMA(t, p, dx);
  const double s = t + xs;
  double q = MCG_FMA(xx, MCG_SCD(MCG_SC_CS6), MCG_SCD(MCG_SC_CS4));
  q = MCG_FMA(q, xx, MCG_SCD(MCG_SC_CS2));
  double c = xx * q;
  c = MCG_FMA(dx, xs, c);
  double cor = MCG_FMA(s, ccs, ssn);
  cor = MCG_FMA(-c, sn, cor);
  cor = MCG_FMA(s, cs, cor);
  return mcg_copysign(cor + sn, a);
}

// do_cos body, given the shared table lookup (xs = |a| - (u - big))
MCG_HD double mcg_do_cos_tab(double a, double da, double xs, double sn, double ssn, double cs,
                             double ccs) {
  const double dx = (a < 0.0) ? -da : da;
  const double xc = dx + xs;
  const double xx = xc * xc;
  const double t = xc * xx;
  const double p = MCG_FMA(xx, MCG_SCD(MCG_SC_SN5), MCG_SCD(MCG_SC_SN3));
  double q = MCG_FMA(xx, MCG_SCD(MCG_SC_CS6), MCG_SCD(MCG_SC_CS4));
  const double s = MCG_FMA(t, p, xc);
  q = MCG_FMA(q, xx, MCG_SCD(MCG_SC_CS2));
  double a1 = MCG_FMA(-ssn, s, ccs);
  const double c = xx * q;
  a1 = MCG_FMA(-c, cs, a1);
  a1 = MCG_FMA(-s, sn, a1);
  return a1 + cs;
}

MCG_HD void mcg_sincos(double x, double* sinx, double* cosx) {
  const uint64_t ix = mcg_asu(x);
  const int32_t k = (int32_t)((ix >> 32) & 0x7fffffffu);
  double xs, sn, ssn, cs, ccs;
  if (k < 0x400368fd) {
    const double ax = mcg_fabs(x);
    if (k < 0x3e400000) {
      *sinx = x;
      *cosx = 1.0;
      return;
    }
    if (k < 0x3feb6000) {  // |x| < 0.855469: do_sin(x, 0), do_cos(x, 0)
      mcg_sincos_lookup(ax, &xs, &sn, &ssn, &cs, &ccs);
      if (MCG_SCD(MCG_SC_T126) > ax) {
        // TAYLOR_SIN(x*x, x, 0) as compiled with the constant zero dx
        const double xx = x * x;
        double p = MCG_FMA(xx, MCG_SCD(MCG_SC_S5), MCG_SCD(MCG_SC_S4));
        p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S3));
        p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S2));
        p = MCG_FMA(xx, p, MCG_SCD(MCG_SC_S1));
        p = MCG_FMA(x, p, -0.0);
        const double t = MCG_FMA(xx, p, 0.0);
        *sinx = x + t;
      } else {
        const double dz = (x > 0.0) ? 0.0 : -0.0;
        *sinx = mcg_do_sin_tab(1.0, dz, xs, sn, ssn, cs, ccs);  // sign fixed below
        *sinx = mcg_copysign(*sinx, x);
      }
      const double dzc = (x >= 0.0) ? 0.0 : -0.0;
      *cosx = mcg_do_cos_tab(1.0, dzc, xs, sn, ssn, cs, ccs);
      return;
    }
    // 0.855469 <= |x| < 2.426265
    const double y = MCG_SCD(MCG_SC_HP0) - ax;
    const double a = y + MCG_SCD(MCG_SC_HP1);
    double da = y - a;
    da = da + MCG_SCD(MCG_SC_HP1);
    const double aa = mcg_fabs(a);
    mcg_sincos_lookup(aa, &xs, &sn, &ssn, &cs, &ccs);
    *sinx = mcg_copysign(mcg_do_cos_tab(a, da, xs, sn, ssn, cs, ccs), x);
    if (MCG_SCD(MCG_SC_T126) > aa)
      *cosx = mcg_taylor_sin(a, da);
    else
      *cosx = mcg_do_sin_tab(a, da, xs, sn, ssn, cs, ccs);
    return;
  }
  if (k < 0x419921fb) {
    // reduce_sincos: x = n*pi/2 + (a + da)
    const double t = MCG_FMA(x, MCG_SCD(MCG_SC_HPINV), MCG_SCD(MCG_SC_TOINT));
    const double xn = t - MCG_SCD(MCG_SC_TOINT);
    const unsigned n = (unsigned)mcg_asu(t) & 3u;
    double yy = MCG_FMA(-xn, MCG_SCD(MCG_SC_MP1), x);
    yy = MCG_FMA(-xn, MCG_SCD(MCG_SC_MP2), yy);
    const double t2 = MCG_FMA(-xn, MCG_SCD(MCG_SC_PP3), yy);
    double db = yy - t2;
    db = MCG_FMA(-xn, MCG_SCD(MCG_SC_PP3), db);
    const double b = MCG_FMA(-xn, MCG_SCD(MCG_SC_PP4), t2);
    double e = t2 - b;
    e = MCG_FMA(-xn, MCG_SCD(MCG_SC_PP4), e);
    db = db + e;
    double a = b, da = db;
    if (n == 1u || n == 2u) {
      a = -a;
      da = -da;
    }
    double* ps = sinx;
    double* pc = cosx;
    if (n & 1u) {
      ps = cosx;
      pc = sinx;
    }
    const double aa = mcg_fabs(a);
    mcg_sincos_lookup(aa, &xs, &sn, &ssn, &cs, &ccs);
    *ps = (MCG_SCD(MCG_SC_T126) > aa) ? mcg_taylor_sin(a, da)
                                      : mcg_do_sin_tab(a, da, xs, sn, ssn, cs, ccs);
    const double cr = mcg_do_cos_tab(a, da, xs, sn, ssn, cs, ccs);
    *pc = (n & 2u) ? -cr : cr;
    return;
  }
  // |x| >= 105414350, inf, nan: not reachable from the engine
  const double nan = (x - x) / (x - x);
  *sinx = nan;
  *cosx = nan;
}
#undef MCG_SCD

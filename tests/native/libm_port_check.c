// Bitwise differential check: mcg_libm.h ports vs the live glibc libm.
// Build: gcc -O2 -mfma -ffp-contract=off -I<csrc> libm_port_check.c -lm
// Usage: libm_port_check <samples_per_range> <seed>
// Exit status 0 iff every sampled argument agrees bit for bit.
#define _GNU_SOURCE
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "mcg_rng.h"

static uint64_t sm;
static uint64_t next64(void) {  // splitmix64
  uint64_t z = (sm += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double unif(double lo, double hi) { return lo + (hi - lo) * ((next64() >> 11) * 0x1p-53); }

static long bad = 0;
static void report(const char* what, double x, double got, double want) {
  if (mcg_asu(got) != mcg_asu(want) && !(isnan(got) && isnan(want))) {
    if (bad < 20) fprintf(stderr, "MISMATCH %s(%.17g) port %.17g glibc %.17g\n", what, x, got, want);
    ++bad;
  }
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  sm = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
  // exp over the ranges the engine uses and the special paths
  const double er[][2] = {{-20, 20}, {-1, 1}, {-1e-3, 1e-3}, {-745.2, -700}, {700, 709.8},
                          {-1100, -600}, {600, 1100}, {-1e-15, 1e-15}};
  for (unsigned r = 0; r < sizeof er / sizeof er[0]; ++r)
    for (long i = 0; i < n; ++i) {
      double x = unif(er[r][0], er[r][1]);
      report("exp", x, mcg_exp(x), exp(x));
    }
  // log: Box–Muller u1 = (k+1) 2^-53 in (0,1], plus near-1 and wide ranges
  for (long i = 0; i < n; ++i) {
    double u1 = ((double)(next64() >> 11) + 1.0) * 0x1p-53;
    report("log", u1, mcg_log(u1), log(u1));
    double x = unif(0.9, 1.1);
    report("log", x, mcg_log(x), log(x));
    x = ldexp(unif(0.5, 1.0), (int)(next64() % 2000) - 1000);
    report("log", x, mcg_log(x), log(x));
    x = unif(0.0, 1e-310);
    report("log", x, mcg_log(x), log(x));
  }
  // sincos on Box–Muller angles (2 pi u2) and all path boundaries
  const double sr[][2] = {{0, 6.283185307179586}, {-0.9, 0.9}, {-0.2, 0.2}, {0.8, 2.5},
                          {-2.5, -0.8}, {2.4, 7}, {-100, 100}, {-1e5, 1e5}, {-1e-7, 1e-7}};
  for (unsigned r = 0; r < sizeof sr / sizeof sr[0]; ++r)
    for (long i = 0; i < n; ++i) {
      double x = (r == 0) ? ((double)(next64() >> 11) * 0x1p-53) * 6.283185307179586
                          : unif(sr[r][0], sr[r][1]);
      double s, c, gs, gc;
      mcg_sincos(x, &s, &c);
      sincos(x, &gs, &gc);
      report("sin", x, s, gs);
      report("cos", x, c, gc);
      report("sin/sincos", x, s, sin(x));
      report("cos/sincos", x, c, cos(x));
    }
  printf("checked %ld samples/range: %ld mismatches\n", n, bad);
  return bad != 0;
}

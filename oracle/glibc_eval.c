/* TEST INFRASTRUCTURE: evaluate the host glibc libm (the reference's libm)
 * over arrays, for the device-vs-glibc differential tests. */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
void glibc_eval(int func, const double* in, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double s, c;
    switch (func) {
      case 0: out[i] = exp(in[i]); break;
      case 1: out[i] = log(in[i]); break;
      case 2: sincos(in[i], &s, &c); out[i] = s; break;
      case 3: sincos(in[i], &s, &c); out[i] = c; break;
      default: out[i] = 0.0;
    }
  }
}

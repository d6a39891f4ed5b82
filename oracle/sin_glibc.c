/* TEST INFRASTRUCTURE ONLY (the CPU checker; never linked into the product).
 *
 * Restatement of glibc 2.39's double-precision sin / cos
 * (sysdeps/ieee754/dbl-64/s_sin.c, usncs.h, sincostab.c; Ubuntu
 * 2.39-0ubuntu8.5), the functions numba and numpy call for np.sin / np.cos on
 * float64 in the reference's physics (physics.py:134-135, 155-156, 191-192,
 * 210-211, 227-228, 326-327, 529-538). On this x86-64 image libm dispatches
 * the `-mfma` ifunc variant (__sin_fma / __cos_fma), i.e. the same C source
 * compiled by GCC with FMA contraction: every contraction GCC made is written
 * out below as an explicit fma() (read off the variant's code), so this file
 * compiles with -ffp-contract=off and reproduces it on any host, and the
 * device restatement (paper_2502_00021_b200/csrc/pxr_math.cuh,
 * glibc_sin / glibc_cos) is the same sequence with __fma_rn.
 *
 * Covered range: |x| < 105414350 (the range reduction to pi/2 with the
 * 3-part constant). Beyond, glibc uses __branred (not restated): the
 * functions here return NaN there and callers must not rely on them.
 * tests/test_oracle.py checks 0 mismatches against this libm on 24 M inputs.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "glibc_sincostab.h"

/* usncs.h */
static const double sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7,
                    cs2 = 0x1.0000000000000p-1, cs4 = -0x1.5555555555535p-5,
                    cs6 = 0x1.6c16bedd9e239p-10;
static const double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7,
                    s3 = -0x1.a01a019db08b8p-13, s4 = 0x1.71de27b9a7ed9p-19,
                    s5 = -0x1.addffc2fcdf59p-26;
static const double big = 0x1.8p45, hp0 = 0x1.921fb54442d18p0, hp1 = 0x1.1a62633145c07p-54;
static const double mp1 = 0x1.921fb58000000p0, mp2 = -0x1.dde973c000000p-27,
                    pp3 = -0x1.cb3b398000000p-55, pp4 = -0x1.d747f23e32ed7p-83,
                    hpinv = 0x1.45f306dc9c883p-1, toint = 0x1.8p52;

static inline uint32_t lo32(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)u;
}
static inline uint32_t hi32(double x) {
  uint64_t u;
  memcpy(&u, &x, 8);
  return (uint32_t)(u >> 32);
}

/* TAYLOR_SIN: a - a^3/3! + ... + (1 - a^2) da / 2 */
static inline double taylor_sin(double xx, double a, double da) {
  const double P = fma(fma(fma(fma(s5, xx, s4), xx, s3), xx, s2), xx, s1);
  const double t = fma(fma(P, a, -(0.5 * da)), xx, da);
  return a + t;
}

/* cos(x + dx) from the table entry nearest |x| and short series */
static inline double do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double u = big + fabs(x);
  x = fabs(x) - (u - big) + dx;
  const double xx = x * x;
  const double s = fma(x * xx, fma(xx, sn5, sn3), x);
  const double c = xx * fma(xx, fma(xx, cs6, cs4), cs2);
  const int k = (int)(lo32(u) << 2);
  const double sn = glibc_sincostab[k], ssn = glibc_sincostab[k + 1];
  const double cs = glibc_sincostab[k + 2], ccs = glibc_sincostab[k + 3];
  const double cor = fma(-sn, s, fma(-cs, c, fma(-s, ssn, ccs)));
  return cs + cor;
}

/* sin(x + dx) */
static inline double do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < 0.126) return taylor_sin(x * x, x, dx);
  if (x <= 0) dx = -dx;
  const double u = big + fabs(x);
  x = fabs(x) - (u - big);
  const double xx = x * x;
  const double s = x + fma(x * xx, fma(xx, sn5, sn3), dx);
  const double c = fma(x, dx, xx * fma(xx, fma(xx, cs6, cs4), cs2));
  const int k = (int)(lo32(u) << 2);
  const double sn = glibc_sincostab[k], ssn = glibc_sincostab[k + 1];
  const double cs = glibc_sincostab[k + 2], ccs = glibc_sincostab[k + 3];
  const double cor = fma(cs, s, fma(-sn, c, fma(s, ccs, ssn)));
  return copysign(sn + cor, xold);
}

/* x = n pi/2 + (a + da), |x| < 105414350 */
static inline int reduce_sincos(double x, double *a, double *da) {
  const double t = fma(x, hpinv, toint);
  const double xn = t - toint;
  const double y = fma(-xn, mp2, fma(-xn, mp1, x));
  const int n = (int)(lo32(t) & 3);
  const double t2 = fma(-xn, pp3, y);
  double db = fma(-xn, pp3, y - t2);
  const double b = fma(-xn, pp4, t2);
  db += fma(-xn, pp4, t2 - b);
  *a = b;
  *da = db;
  return n;
}

static inline double do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

double glibc_sin(double x) {
  const uint32_t k = hi32(x) & 0x7fffffffu;
  double a, da;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign(do_cos(hp0 - fabs(x), hp1), x);
  if (k < 0x419921fbu) {
    const int n = reduce_sincos(x, &a, &da);
    return do_sincos(a, da, n);
  }
  return NAN;
}

double glibc_cos(double x) {
  const uint32_t k = hi32(x) & 0x7fffffffu;
  double a, da;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = hp0 - fabs(x);
    a = y + hp1;
    da = (y - a) + hp1;
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {
    const int n = reduce_sincos(x, &a, &da);
    return do_sincos(a, da, n + 1);
  }
  return NAN;
}

/* batch entry for ctypes: sin and cos of n doubles */
void glibc_sincos_batch(const double *x, double *s, double *c, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    s[i] = glibc_sin(x[i]);
    c[i] = glibc_cos(x[i]);
  }
}

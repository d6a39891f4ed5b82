/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
 *
 * Restatement of glibc 2.39's single-precision sinf/cosf (the x86-64
 * "__sinf_fma"/"__cosf_fma" ifunc variants, i.e. sysdeps/ieee754/flt-32/
 * s_sinf.c, s_cosf.c, sincosf.h built with -mfma), which is what numba 0.65
 * calls for np.cos/np.sin on float32 inside the reference's robot raster
 * kernel (reference: pkg/src/pixelctrl/render.py:474-475).
 *
 * Third-party dependency: glibc 2.39 (Ubuntu 2.39-0ubuntu8.5 in this image).
 * Published algorithm (ARM optimized-routines, adopted by glibc 2.28+):
 *   |x| < pi/4 (top-12-bit compare): double polynomial directly;
 *   |x| < 120: r = x*2/pi*2^24, n = (int(r) + 2^23) >> 24, x - n*pi/2 (FMA);
 *   otherwise: 4/pi bit table reduction in integer arithmetic.
 * The polynomial is evaluated in double; GCC -mfma contracts each a + b*c.
 * Constants were checked against the table present in this image's
 * libm.so.6 and the whole function is checked exhaustively against libm by
 * tests/test_oracle_sincosf.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "oracle.h"

typedef struct {
  double sign[4];
  double hpi_inv; /* 2/pi * 2^24 (no TOINT intrinsics on x86-64) */
  double hpi;
  double c0, c1, c2, c3, c4;
  double s1, s2, s3;
} sc_tab;

static const sc_tab TAB[2] = {
    {{1.0, -1.0, -1.0, 1.0},
     0x1.45F306DC9C883p+23,
     0x1.921FB54442D18p0,
     0x1p0,
     -0x1.ffffffd0c621cp-2,
     0x1.55553e1068f19p-5,
     -0x1.6c087e89a359dp-10,
     0x1.99343027bf8c3p-16,
     -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7,
     -0x1.994eb3774cf24p-13},
    {{1.0, -1.0, -1.0, 1.0},
     0x1.45F306DC9C883p+23,
     0x1.921FB54442D18p0,
     -0x1p0,
     0x1.ffffffd0c621cp-2,
     -0x1.55553e1068f19p-5,
     0x1.6c087e89a359dp-10,
     -0x1.99343027bf8c3p-16,
     -0x1.555545995a603p-3,
     0x1.1107605230bc4p-7,
     -0x1.994eb3774cf24p-13},
};

/* Bits of 4/pi (equivalently 2/pi shifted), 24 overlapping 32-bit windows. */
static const uint32_t INV_PIO4[24] = {
    0xa2,       0xa2f9,     0xa2f983,   0xa2f9836e, 0xf9836e4e, 0x836e4e44,
    0x6e4e4415, 0x4e441529, 0x441529fc, 0x1529fc27, 0x29fc2757, 0xfc2757d1,
    0x2757d1f5, 0x57d1f534, 0xd1f534dd, 0xf534ddc0, 0x34ddc0db, 0xddc0db62,
    0xc0db6295, 0xdb629599, 0x6295993c, 0x95993c43, 0x993c4390, 0x3c439041};

static const double PI63 = 0x1.921FB54442D18p-62;
static const float PIO4F = 0x1.921FB6p-1f;

static inline uint32_t asuint(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return u;
}
static inline uint32_t abstop12(float x) { return (asuint(x) >> 20) & 0x7ff; }

static inline float poly(double x, double x2, const sc_tab *p, int n) {
  if ((n & 1) == 0) {
    double x3 = x * x2;
    double s1 = fma(x2, p->s3, p->s2);
    double x7 = x3 * x2;
    double s = fma(x3, p->s1, x);
    return (float)fma(x7, s1, s);
  } else {
    double x4 = x2 * x2;
    double c2 = fma(x2, p->c4, p->c3);
    double c1 = fma(x2, p->c1, p->c0);
    double x6 = x4 * x2;
    double c = fma(x4, p->c2, c1);
    return (float)fma(x6, c2, c);
  }
}

static inline double reduce_fast(double x, const sc_tab *p, int *np) {
  double r = x * p->hpi_inv;
  int n = ((int32_t)r + 0x800000) >> 24;
  *np = n;
  return fma(-(double)n, p->hpi, x);
}

static inline double reduce_large(uint32_t xi, int *np) {
  const uint32_t *arr = &INV_PIO4[(xi >> 26) & 15];
  int shift = (xi >> 23) & 7;
  uint64_t n, res0, res1, res2;
  xi = (xi & 0xffffff) | 0x800000;
  xi <<= shift;
  res0 = xi * arr[0];
  res1 = (uint64_t)xi * arr[4];
  res2 = (uint64_t)xi * arr[8];
  res0 = (res2 >> 32) | (res0 << 32);
  res0 += res1;
  n = (res0 + (1ULL << 61)) >> 62;
  res0 -= n << 62;
  double x = (double)(int64_t)res0;
  *np = (int)n;
  return x * PI63;
}

float oracle_sinf(float y) {
  double x = y;
  double s;
  int n;
  const sc_tab *p = &TAB[0];
  if (abstop12(y) < abstop12(PIO4F)) {
    s = x * x;
    if (abstop12(y) < abstop12(0x1p-12f)) return y;
    return poly(x, s, p, 0);
  } else if (abstop12(y) < abstop12(120.0f)) {
    x = reduce_fast(x, p, &n);
    s = p->sign[n & 3];
    if (n & 2) p = &TAB[1];
    return poly(x * s, x * x, p, n);
  } else if (abstop12(y) < abstop12(INFINITY)) {
    uint32_t xi = asuint(y);
    int sign = xi >> 31;
    x = reduce_large(xi, &n);
    s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &TAB[1];
    return poly(x * s, x * x, p, n);
  }
  return (y - y) / (y - y);
}

float oracle_cosf(float y) {
  double x = y;
  double s;
  int n;
  const sc_tab *p = &TAB[0];
  if (abstop12(y) < abstop12(PIO4F)) {
    double x2 = x * x;
    if (abstop12(y) < abstop12(0x1p-12f)) return 1.0f;
    return poly(x, x2, p, 1);
  } else if (abstop12(y) < abstop12(120.0f)) {
    x = reduce_fast(x, p, &n);
    s = p->sign[n & 3];
    if (n & 2) p = &TAB[1];
    return poly(x * s, x * x, p, n ^ 1);
  } else if (abstop12(y) < abstop12(INFINITY)) {
    uint32_t xi = asuint(y);
    int sign = xi >> 31;
    x = reduce_large(xi, &n);
    s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &TAB[1];
    return poly(x * s, x * x, p, n ^ 1);
  }
  return (y - y) / (y - y);
}

/* Exhaustive/strided comparison helper used by the oracle self-test:
 * counts mismatches between this restatement and the live libm over every
 * float whose bit pattern is lo + k*stride (k >= 0, < hi). */
typedef float (*f2f)(float);
static f2f volatile LIBM_SINF = sinf;
static f2f volatile LIBM_COSF = cosf;

int64_t oracle_sincosf_selftest(uint32_t lo, uint32_t hi, uint32_t stride) {
  int64_t bad = 0;
  f2f lsin = LIBM_SINF, lcos = LIBM_COSF;
#pragma omp parallel for reduction(+ : bad) schedule(static)
  for (int64_t u = lo; u < (int64_t)hi; u += stride) {
    float f;
    uint32_t b = (uint32_t)u;
    memcpy(&f, &b, 4);
    if (!isfinite(f)) continue;
    float a = lsin(f), c = lcos(f);
    float ra = oracle_sinf(f), rc = oracle_cosf(f);
    if (asuint(a) != asuint(ra)) bad++;
    if (asuint(c) != asuint(rc)) bad++;
  }
  return bad;
}

/* Element-wise restated sinf/cosf over an array (GPU parity checker). */
void oracle_sincosf_many(const float *x, float *s, float *c, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; i++) {
    s[i] = oracle_sinf(x[i]);
    c[i] = oracle_cosf(x[i]);
  }
}

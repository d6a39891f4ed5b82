// glibc 2.39 double-precision sin / cos on the device, bit-identical to the
// libm the reference's physics calls: numba's np.cos / np.sin on float64 in
// _step_batch (physics.py:155-156, 191-192, 210-211, 227-228, 326-327) and
// numpy's in forward_kinematics / the velocity helpers (physics.py:134-135,
// 529-538). On x86-64 libm dispatches its -mfma variant (__sin_fma /
// __cos_fma, sysdeps/ieee754/dbl-64/s_sin.c compiled with FMA contraction):
// a table of sin / cos at k/128 as double-doubles (sincostab.c, generated
// into pxr_glibc_sincostab.h by tools/gen_glibc_sincostab.py) corrected by
// short series, with a 3-part pi/2 reduction up to |x| < 105414350. Every
// contraction of that build is an explicit __fma_rn here (the file compiles
// with -fmad=false); the CPU checker's twin (sin_glibc.c) is the same sequence
// and matches libm on 24 M inputs (tests/test_oracle.py), the device copy
// matches libm through numpy in tests/test_gpu_parity.py. Beyond
// 105414350 glibc's __branred is not restated: those (physically
// meaningless) angles take CUDA's sin / cos.
#pragma once
#include <stdint.h>

#include "pxr_glibc_sincostab.h"

namespace pxr {
namespace glibc_dbl {

constexpr double sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7;
constexpr double cs2 = 0x1.0000000000000p-1, cs4 = -0x1.5555555555535p-5,
                 cs6 = 0x1.6c16bedd9e239p-10;
constexpr double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7,
                 s3 = -0x1.a01a019db08b8p-13, s4 = 0x1.71de27b9a7ed9p-19,
                 s5 = -0x1.addffc2fcdf59p-26;
constexpr double big = 0x1.8p45, hp0 = 0x1.921fb54442d18p0, hp1 = 0x1.1a62633145c07p-54;
constexpr double mp1 = 0x1.921fb58000000p0, mp2 = -0x1.dde973c000000p-27,
                 pp3 = -0x1.cb3b398000000p-55, pp4 = -0x1.d747f23e32ed7p-83,
                 hpinv = 0x1.45f306dc9c883p-1, toint = 0x1.8p52;

__device__ __forceinline__ double taylor_sin(double xx, double a, double da) {
  const double P =
      __fma_rn(__fma_rn(__fma_rn(__fma_rn(s5, xx, s4), xx, s3), xx, s2), xx, s1);
  const double t = __fma_rn(__fma_rn(P, a, -__dmul_rn(0.5, da)), xx, da);
  return __dadd_rn(a, t);
}

__device__ __forceinline__ void table(double u, double &sn, double &ssn, double &cs,
                                      double &ccs) {
  const int k = (int)(__double2loint(u) << 2);
  sn = __ldg(kGlibcSinCosTab + k);
  ssn = __ldg(kGlibcSinCosTab + k + 1);
  cs = __ldg(kGlibcSinCosTab + k + 2);
  ccs = __ldg(kGlibcSinCosTab + k + 3);
}

__device__ __forceinline__ double do_cos(double x, double dx) {
  if (x < 0.0) dx = -dx;
  const double u = __dadd_rn(big, fabs(x));
  x = __dadd_rn(__dsub_rn(fabs(x), __dsub_rn(u, big)), dx);
  const double xx = __dmul_rn(x, x);
  const double s = __fma_rn(__dmul_rn(x, xx), __fma_rn(xx, sn5, sn3), x);
  const double c = __dmul_rn(xx, __fma_rn(xx, __fma_rn(xx, cs6, cs4), cs2));
  double sn, ssn, cs, ccs;
  table(u, sn, ssn, cs, ccs);
  const double cor = __fma_rn(-sn, s, __fma_rn(-cs, c, __fma_rn(-s, ssn, ccs)));
  return __dadd_rn(cs, cor);
}

__device__ __forceinline__ double do_sin(double x, double dx) {
  const double xold = x;
  if (fabs(x) < 0.126) return taylor_sin(__dmul_rn(x, x), x, dx);
  if (x <= 0.0) dx = -dx;
  const double u = __dadd_rn(big, fabs(x));
  x = __dsub_rn(fabs(x), __dsub_rn(u, big));
  const double xx = __dmul_rn(x, x);
  const double s = __dadd_rn(x, __fma_rn(__dmul_rn(x, xx), __fma_rn(xx, sn5, sn3), dx));
  const double c = __fma_rn(x, dx, __dmul_rn(xx, __fma_rn(xx, __fma_rn(xx, cs6, cs4), cs2)));
  double sn, ssn, cs, ccs;
  table(u, sn, ssn, cs, ccs);
  const double cor = __fma_rn(cs, s, __fma_rn(-sn, c, __fma_rn(s, ccs, ssn)));
  return copysign(__dadd_rn(sn, cor), xold);
}

__device__ __forceinline__ int reduce(double x, double &a, double &da) {
  const double t = __fma_rn(x, hpinv, toint);
  const double xn = __dsub_rn(t, toint);
  const double y = __fma_rn(-xn, mp2, __fma_rn(-xn, mp1, x));
  const int n = (int)(__double2loint(t) & 3);
  const double t2 = __fma_rn(-xn, pp3, y);
  double db = __fma_rn(-xn, pp3, __dsub_rn(y, t2));
  const double b = __fma_rn(-xn, pp4, t2);
  db = __dadd_rn(db, __fma_rn(-xn, pp4, __dsub_rn(t2, b)));
  a = b;
  da = db;
  return n;
}

__device__ __forceinline__ double do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

}  // namespace glibc_dbl

// sin(x) exactly as glibc 2.39's __sin_fma
__device__ __forceinline__ double glibc_sin(double x) {
  using namespace glibc_dbl;
  const uint32_t k = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign(do_cos(__dsub_rn(hp0, fabs(x)), hp1), x);
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce(x, a, da);
    return do_sincos(a, da, n);
  }
  return sin(x);  // |x| >= 105414350 or not finite: not restated
}

// cos(x) exactly as glibc 2.39's __cos_fma
__device__ __forceinline__ double glibc_cos(double x) {
  using namespace glibc_dbl;
  const uint32_t k = (uint32_t)__double2hiint(x) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = __dsub_rn(hp0, fabs(x));
    const double a = __dadd_rn(y, hp1);
    const double da = __dadd_rn(__dsub_rn(y, a), hp1);
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce(x, a, da);
    return do_sincos(a, da, n + 1);
  }
  return cos(x);  // |x| >= 105414350 or not finite: not restated
}

}  // namespace pxr

/* TEST INFRASTRUCTURE ONLY (the CPU checker; never linked into the product).
 *
 * Restatement of numpy 2.3.5's float64 np.log on AVX-512 hosts, the log of
 * the reference's reset-velocity Box-Muller draw (prng.py:147): numpy
 * dispatches it (DOUBLE_log_AVX512_SKX) to its bundled Intel SVML
 * `__svml_log8_ha`, whose main path is written out below operation by
 * operation (every FMA of the vector code an fma() here; compile with
 * -ffp-contract=off). The one hardware-defined step, the reciprocal
 * estimate VRCP14PD rounded to 5 fraction bits, is a step function of the
 * mantissa whose 16 steps tools/gen_numpy_log_tables.py located on an
 * AVX-512 host (np_log_tables.h, with the SVML tables A / B and constants).
 * Positive normal finite x only (the draws are in [2^-53, 1)); other inputs
 * return libm's log. tests/test_oracle.py checks 0 mismatches against
 * np.log on 12 M inputs.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "np_log_tables.h"

double np_log_svml(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  const uint64_t ex = (b >> 52) & 0x7ff;
  if ((b >> 63) || ex == 0 || ex == 0x7ff) return log(x);
  double e = (double)((int64_t)ex - 1023);                       /* getexp */
  const uint64_t mb = (b & 0x000fffffffffffffull) | 0x3ff0000000000000ull;
  double m;
  memcpy(&m, &mb, 8);                                             /* getmant, [1, 2) */
  int c = 0;
  for (int k = 0; k < 16; k++) c += kNpLogRcpStep[k] <= m;
  const double r = (double)(32 - c) * 0x1p-5;                    /* roundscale(rcp14(m)) */
  const double t = fma(r, m, -1.0);
  if (r < 0.75) e = e + 1.0;
  uint64_t rb;
  memcpy(&rb, &r, 8);
  const int j = (int)((rb >> 48) & 15);
  const double *C = kNpLogC;
  const double z7 = fma(C[2], t, C[3]);
  double z1 = fma(C[0], t, C[1]);
  const double t2 = t * t;
  double z9 = fma(C[4], t, C[5]);
  z1 = fma(t2, z1, z7);
  const double t4 = t2 * t2;
  const double z8 = fma(C[6], t, C[7]);
  z9 = fma(t2, z9, z8);
  const double a = fma(C[8], e, kNpLogA[j]);
  z1 = fma(t4, z1, z9);
  const double z11 = a + t;
  const double z10 = t - (z11 - a);
  z1 = fma(t2, z1, z10);
  const double z4 = fma(C[9], e, kNpLogB[j]);
  return z11 + (z1 + z4);
}

void np_log_svml_batch(const double *x, double *y, int64_t n) {
  for (int64_t i = 0; i < n; i++) y[i] = np_log_svml(x[i]);
}

// Device arithmetic that must round exactly like the reference's CPU path.
//
// 1. glibc 2.39 sinf/cosf. numba lowers np.cos/np.sin on float32 inside the
//    robot raster kernel (reference render.py:474-475) to libm cosf/sinf;
//    on x86-64 with FMA glibc dispatches to its -mfma build of the
//    ARM-optimized-routines algorithm (double-precision range reduction and
//    polynomial). It is restated here with explicit __fma_rn/__dmul_rn so
//    the device result is bit-identical on every float (the host twin of
//    this code is checked against libm over all 2^32 inputs, and the device
//    copy against the host twin by tests/test_gpu_parity.py).
// 2. Threefry-2x64-20 (reference prng.py:33-77) on 64-bit integer lanes.
#pragma once
#include <stdint.h>

namespace pxr {

struct SinCosTab {
  double sign[4];
  double hpi_inv, hpi;
  double c0, c1, c2, c3, c4;
  double s1, s2, s3;
};

static __device__ __constant__ SinCosTab kSinCos[2] = {
    {{1.0, -1.0, -1.0, 1.0}, 0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, 0x1p0,
     -0x1.ffffffd0c621cp-2, 0x1.55553e1068f19p-5, -0x1.6c087e89a359dp-10,
     0x1.99343027bf8c3p-16, -0x1.555545995a603p-3, 0x1.1107605230bc4p-7,
     -0x1.994eb3774cf24p-13},
    {{1.0, -1.0, -1.0, 1.0}, 0x1.45F306DC9C883p+23, 0x1.921FB54442D18p0, -0x1p0,
     0x1.ffffffd0c621cp-2, -0x1.55553e1068f19p-5, 0x1.6c087e89a359dp-10,
     -0x1.99343027bf8c3p-16, -0x1.555545995a603p-3, 0x1.1107605230bc4p-7,
     -0x1.994eb3774cf24p-13},
};

// 2/pi bit windows for |x| >= 120 (integer Payne-Hanek style reduction).
static __device__ __constant__ uint32_t kInvPio4[24] = {
    0xa2,       0xa2f9,     0xa2f983,   0xa2f9836e, 0xf9836e4e, 0x836e4e44,
    0x6e4e4415, 0x4e441529, 0x441529fc, 0x1529fc27, 0x29fc2757, 0xfc2757d1,
    0x2757d1f5, 0x57d1f534, 0xd1f534dd, 0xf534ddc0, 0x34ddc0db, 0xddc0db62,
    0xc0db6295, 0xdb629599, 0x6295993c, 0x95993c43, 0x993c4390, 0x3c439041};

__device__ __forceinline__ uint32_t abstop12(float x) {
  return (__float_as_uint(x) >> 20) & 0x7ff;
}

__device__ __forceinline__ float sc_poly(double x, double x2, const SinCosTab &p, int n) {
  if ((n & 1) == 0) {
    double x3 = __dmul_rn(x, x2);
    double s1 = __fma_rn(x2, p.s3, p.s2);
    double x7 = __dmul_rn(x3, x2);
    double s = __fma_rn(x3, p.s1, x);
    return __double2float_rn(__fma_rn(x7, s1, s));
  } else {
    double x4 = __dmul_rn(x2, x2);
    double c2 = __fma_rn(x2, p.c4, p.c3);
    double c1 = __fma_rn(x2, p.c1, p.c0);
    double x6 = __dmul_rn(x4, x2);
    double c = __fma_rn(x4, p.c2, c1);
    return __double2float_rn(__fma_rn(x6, c2, c));
  }
}

__device__ __forceinline__ double sc_reduce_large(uint32_t xi, int &n_out) {
  const uint32_t *arr = &kInvPio4[(xi >> 26) & 15];
  int shift = (xi >> 23) & 7;
  xi = (xi & 0xffffff) | 0x800000;
  xi <<= shift;
  uint64_t res0 = (uint64_t)(uint32_t)(xi * arr[0]);
  uint64_t res1 = (uint64_t)xi * arr[4];
  uint64_t res2 = (uint64_t)xi * arr[8];
  res0 = (res2 >> 32) | (res0 << 32);
  res0 += res1;
  uint64_t n = (res0 + (1ULL << 61)) >> 62;
  res0 -= n << 62;
  n_out = (int)n;
  return __dmul_rn((double)(int64_t)res0, 0x1.921FB54442D18p-62);
}

// which = 0 -> sinf, 1 -> cosf (glibc s_sinf.c / s_cosf.c control flow).
__device__ __forceinline__ float glibc_sincosf(float y, int which) {
  const SinCosTab *p = &kSinCos[0];
  double x = (double)y;
  int n;
  uint32_t top = abstop12(y);
  if (top < abstop12(0x1.921FB6p-1f)) {
    if (top < abstop12(0x1p-12f)) return which ? 1.0f : y;
    return sc_poly(x, __dmul_rn(x, x), *p, which);
  }
  double s;
  if (top < abstop12(120.0f)) {
    double r = __dmul_rn(x, p->hpi_inv);
    n = ((int32_t)r + 0x800000) >> 24;
    x = __fma_rn(-(double)n, p->hpi, x);
    s = p->sign[n & 3];
    if (n & 2) p = &kSinCos[1];
  } else if (top < abstop12(__int_as_float(0x7f800000))) {
    uint32_t xi = __float_as_uint(y);
    int sign = xi >> 31;
    x = sc_reduce_large(xi, n);
    s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &kSinCos[1];
  } else {
    return __int_as_float(0x7fc00000);
  }
  return sc_poly(__dmul_rn(x, s), __dmul_rn(x, x), *p, which ? (n ^ 1) : n);
}

// ---------------------------------------------------------------- Threefry

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}

// prng.py:57-77. Rotation schedule (16,42,12,31,16,32,24,21), parity
// 0x1BD11BDAA9FC1FFA, key injected after every fourth round.
__device__ __forceinline__ void threefry2x64(uint64_t k0, uint64_t k1, uint64_t c0,
                                             uint64_t c1, uint64_t &o0, uint64_t &o1) {
  const uint64_t k2 = k0 ^ k1 ^ 0x1BD11BDAA9FC1FFAULL;
  const uint64_t ks[3] = {k0, k1, k2};
  const int rot[8] = {16, 42, 12, 31, 16, 32, 24, 21};
  uint64_t x0 = c0 + k0, x1 = c1 + k1;
#pragma unroll
  for (int r = 0; r < 20; r++) {
    x0 += x1;
    x1 = rotl64(x1, rot[r % 8]);
    x1 ^= x0;
    if (r % 4 == 3) {
      const int j = r / 4 + 1;
      x0 += ks[j % 3];
      x1 += ks[(j + 1) % 3] + (uint64_t)j;
    }
  }
  o0 = x0;
  o1 = x1;
}

// prng.py:181-193 index_from_words: floor(w * n / 2^64) == umulhi(w, n).
__device__ __forceinline__ int64_t index_from_word(uint64_t w, uint64_t n) {
  return (int64_t)__umul64hi(w, n);
}

// distractor.py:66-74: one bias triple per key, uniform on [-60, 60].
__device__ __forceinline__ void color_bias_from_key(uint64_t hi, uint64_t lo, int16_t out[3]) {
  uint64_t w0, w1, w2, unused;
  threefry2x64(hi, lo, 0, 0, w0, w1);
  threefry2x64(hi, lo, 1, 0, w2, unused);
  out[0] = (int16_t)(index_from_word(w0, 121) - 60);
  out[1] = (int16_t)(index_from_word(w1, 121) - 60);
  out[2] = (int16_t)(index_from_word(w2, 121) - 60);
}

}  // namespace pxr

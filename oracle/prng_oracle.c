/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- restatement of the reference's
 * Threefry-2x64-20 counter PRNG (pkg/src/pixelctrl/prng.py:33-77) and the
 * per-env colour-bias draw (distractor.py:66-74, prng.py:168-193).
 */
#include <stdint.h>

#include "oracle.h"

static const int ROT[8] = {16, 42, 12, 31, 16, 32, 24, 21}; /* prng.py:33 */
static const uint64_t PARITY = 0x1BD11BDAA9FC1FFAULL;       /* prng.py:34 */

static inline uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

/* prng.py:57-77 */
static inline void tf2x64(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1,
                          uint64_t *o0, uint64_t *o1) {
  uint64_t ks[3] = {k0, k1, k0 ^ k1 ^ PARITY};
  uint64_t x0 = c0 + ks[0], x1 = c1 + ks[1];
  for (int r = 0; r < 20; r++) {
    x0 += x1;
    x1 = rotl(x1, ROT[r % 8]);
    x1 ^= x0;
    if (r % 4 == 3) {
      int j = r / 4 + 1;
      x0 += ks[j % 3];
      x1 += ks[(j + 1) % 3] + (uint64_t)j;
    }
  }
  *o0 = x0;
  *o1 = x1;
}

void oracle_threefry2x64(const uint64_t *k0, const uint64_t *k1, int64_t key_stride,
                         const uint64_t *c0, const uint64_t *c1, uint64_t *y0,
                         uint64_t *y1, int64_t n) {
  for (int64_t i = 0; i < n; i++)
    tf2x64(k0[i * key_stride], k1[i * key_stride], c0[i], c1[i], &y0[i], &y1[i]);
}

/* prng.py:181-193 index_from_words: floor(w * n / 2^64) in 32-bit halves */
static inline int64_t index_from_word(uint64_t w, uint64_t n) {
  uint64_t hi = w >> 32, lo = w & 0xFFFFFFFFULL;
  return (int64_t)((hi * n + ((lo * n) >> 32)) >> 32);
}

/* distractor.py:66-74 via advance_distractors (distractor.py:123-126):
 * e = fold_in(key_t, g) = TF(key_t, (g, 2)); (w0, w1) = TF(e, (0, 0));
 * w2 = TF(e, (1, 0)).x0; bias_c = index(w_c, 121) - 60. */
void oracle_color_biases(uint64_t key_hi, uint64_t key_lo, uint64_t env_offset,
                         int64_t batch, int16_t *out) {
  for (int64_t i = 0; i < batch; i++) {
    uint64_t ehi, elo, w0, w1, w2, unused;
    tf2x64(key_hi, key_lo, env_offset + (uint64_t)i, 2, &ehi, &elo);
    tf2x64(ehi, elo, 0, 0, &w0, &w1);
    tf2x64(ehi, elo, 1, 0, &w2, &unused);
    out[3 * i + 0] = (int16_t)(index_from_word(w0, 121) - 60);
    out[3 * i + 1] = (int16_t)(index_from_word(w1, 121) - 60);
    out[3 * i + 2] = (int16_t)(index_from_word(w2, 121) - 60);
  }
}

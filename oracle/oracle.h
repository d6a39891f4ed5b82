/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C, scalar, no FMA contraction) of the reference's
 * pixel-observation hot path, used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * Nothing in paper_2502_00021_b200/ may include, link or call this.
 *
 * Every function cites the reference (pkg/src/pixelctrl/...) lines it
 * restates. Numeric types mirror numba 0.65's typing of the reference
 * kernels: f32 where the reference computes in f32,
 * f64 where numba promotes.
 */
#ifndef PXR_ORACLE_H
#define PXR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* glibc 2.39 sinf/cosf (FMA ifunc variant) -- sincosf_glibc.c */
float oracle_sinf(float x);
float oracle_cosf(float x);
int64_t oracle_sincosf_selftest(uint32_t lo, uint32_t hi, uint32_t stride);
void oracle_sincosf_many(const float *x, float *s, float *c, int64_t n);

/* Threefry-2x64-20 block (prng.py:57-77), element-wise over n counters. */
void oracle_threefry2x64(const uint64_t *k0, const uint64_t *k1, int64_t key_stride,
                         const uint64_t *c0, const uint64_t *c1, uint64_t *y0,
                         uint64_t *y1, int64_t n);

/* render.py:286-456 _raster_scene (one scene, pixels/depth fully rewritten). */
void oracle_raster_scene(const float *verts, int64_t nv, const int32_t *tris,
                         int64_t nt, const float *tri_colors, const float *cam,
                         const float *light, int draw_floor, uint8_t *pixels,
                         float *depth, int64_t h_px, int64_t w_px);

/* render.py:459-485 _raster_robot_range, parallel over envs with `threads`
 * OpenMP threads (results independent of the thread count, like
 * threading_utils.parallel_over_ranges). */
void oracle_raster_robot_range(const float *base_verts, const int32_t *vert_link,
                               int64_t nv, const int32_t *tris, int64_t nt,
                               const float *tri_colors, const float *poses32,
                               int64_t n_links, const float *cams,
                               const float *light, int draw_floor,
                               uint8_t *pixels, float *depth, int64_t batch,
                               int64_t h_px, int64_t w_px, int threads);

/* distractor.py:140-161 _color_kernel (bias int64 (B,3)). */
void oracle_color_kernel(uint8_t *pixels, const int64_t *bias, int64_t batch,
                         int64_t h, int64_t w, int threads);

/* distractor.py:164-176 _video_kernel. */
void oracle_video_kernel(uint8_t *pixels, const float *depth,
                         const uint8_t *frames_flat, int64_t hv, int64_t wv,
                         const int64_t *frame_idx, const int64_t *row_map,
                         const int64_t *col_map, int64_t batch, int64_t h,
                         int64_t w, int threads);

/* env.py:168-173 grayscale postprocess. */
void oracle_grayscale(const uint8_t *rgb, uint8_t *gray, int64_t n_px);

/* distractor.py:66-74 + prng.py:168-193: colour biases for envs
 * g = env_offset + i of fold_in(key_t, g). */
void oracle_color_biases(uint64_t key_hi, uint64_t key_lo, uint64_t env_offset,
                         int64_t batch, int16_t *out);

/* distractor.py:128-136 ping-pong cursor advance (in place). */
void oracle_video_advance(int64_t *cursor, int8_t *direction,
                          const int64_t *frame_count, int64_t batch);

#ifdef __cplusplus
}
#endif
#endif

/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's
 * robot raster path (pkg/src/pixelctrl/render.py) and distractor kernels
 * (pkg/src/pixelctrl/distractor.py). Scalar C, compiled with
 * -ffp-contract=off so every f32/f64 operation rounds exactly where numba's
 * (non-fastmath) LLVM code does. Types follow SURVEY.md appendix A1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static const uint8_t SKY[3] = {135, 206, 235};      /* render.py:50 */
static const uint8_t FLOOR_LIGHT = 158;            /* render.py:51 */
static const uint8_t FLOOR_DARK = 122;             /* render.py:52 */
static const double AMBIENT = 0.35, DIFFUSE = 0.65; /* render.py:53-54 */

/* render.py:286-456 */
void oracle_raster_scene(const float *verts, int64_t nv, const int32_t *tris,
                         int64_t nt, const float *tri_colors, const float *cam,
                         const float *light, int draw_floor, uint8_t *pixels,
                         float *depth, int64_t h_px, int64_t w_px) {
  const float ex = cam[0], ey = cam[1], ez = cam[2];
  const float rx = cam[3], ry = cam[4], rz = cam[5];
  const float ux = cam[6], uy = cam[7], uz = cam[8];
  const float fx = cam[9], fy = cam[10], fz = cam[11];
  const float tanf_ = cam[12], near_ = cam[13], far_ = cam[14];
  const double aspect = (double)w_px / (double)h_px; /* int/int -> f64 */
  const float lx = light[0], ly = light[1], lz = light[2];

  /* render.py:306-311 clear */
  for (int64_t i = 0; i < h_px * w_px; i++) {
    pixels[3 * i + 0] = SKY[0];
    pixels[3 * i + 1] = SKY[1];
    pixels[3 * i + 2] = SKY[2];
    depth[i] = INFINITY;
  }

  /* render.py:313-344 floor, f64, directions advanced incrementally in x */
  if (draw_floor) {
    double sx0 = (1.0 / (double)w_px - 1.0) * (double)tanf_ * aspect;
    double dsx = (2.0 / (double)w_px) * (double)tanf_ * aspect;
    double drx = dsx * (double)rx;
    double dry = dsx * (double)ry;
    double drz = dsx * (double)rz;
    for (int64_t y = 0; y < h_px; y++) {
      double sy = (1.0 - 2.0 * ((double)y + 0.5) / (double)h_px) * (double)tanf_;
      double dx = (double)fx + sx0 * (double)rx + sy * (double)ux;
      double dy = (double)fy + sx0 * (double)ry + sy * (double)uy;
      double dz = (double)fz + sx0 * (double)rz + sy * (double)uz;
      for (int64_t x = 0; x < w_px; x++) {
        if (dz < -1e-12) {
          double t = (double)(-ez) / dz;
          if ((double)near_ <= t && t <= (double)far_) {
            double wx = (double)ex + t * dx;
            double wy = (double)ey + t * dy;
            int64_t parity = ((int64_t)floor(wx) + (int64_t)floor(wy)) & 1;
            uint8_t c = parity == 0 ? FLOOR_LIGHT : FLOOR_DARK;
            int64_t i = y * w_px + x;
            pixels[3 * i + 0] = c;
            pixels[3 * i + 1] = c;
            pixels[3 * i + 2] = c;
            depth[i] = (float)t;
          }
        }
        dx += drx;
        dy += dry;
        dz += drz;
      }
    }
  }

  /* render.py:346-363 projection */
  float *sxs = (float *)malloc(sizeof(float) * (size_t)(nv > 0 ? nv : 1) * 3);
  float *sys_ = sxs + nv;
  float *zs = sys_ + nv;
  for (int64_t i = 0; i < nv; i++) {
    float vx = verts[3 * i + 0] - ex;
    float vy = verts[3 * i + 1] - ey;
    float vz = verts[3 * i + 2] - ez;
    float zv = vx * fx + vy * fy + vz * fz;
    zs[i] = zv;
    if ((double)zv > 1e-9) {
      float xv = vx * rx + vy * ry + vz * rz;
      float yv = vx * ux + vy * uy + vz * uz;
      sxs[i] = (float)(((double)xv / ((double)(zv * tanf_) * aspect) + 1.0) *
                       ((double)w_px / 2.0));
      sys_[i] = (float)((1.0 - (double)(yv / (zv * tanf_))) * ((double)h_px / 2.0));
    } else {
      sxs[i] = 0.0f;
      sys_[i] = 0.0f;
    }
  }

  /* render.py:365-456 triangles in index order, strict depth test */
  for (int64_t t = 0; t < nt; t++) {
    int32_t i0 = tris[3 * t + 0], i1 = tris[3 * t + 1], i2 = tris[3 * t + 2];
    float z0 = zs[i0], z1 = zs[i1], z2 = zs[i2];
    if (z0 < near_ || z1 < near_ || z2 < near_) continue;
    if (z0 > far_ && z1 > far_ && z2 > far_) continue;
    float x0 = sxs[i0], y0 = sys_[i0];
    float x1 = sxs[i1], y1 = sys_[i1];
    float x2 = sxs[i2], y2 = sys_[i2];
    float area2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
    if (area2 == 0.0f) continue;
    if (area2 < 0.0f) {
      float tmp;
      tmp = x1; x1 = x2; x2 = tmp;
      tmp = y1; y1 = y2; y2 = tmp;
      tmp = z1; z1 = z2; z2 = tmp;
      area2 = -area2;
    }
    /* Python min/max on floats: min(a, b) returns a unless b < a. */
    float m12 = x2 < x1 ? x2 : x1;
    float minx = m12 < x0 ? m12 : x0;
    float M12 = x2 > x1 ? x2 : x1;
    float maxx = M12 > x0 ? M12 : x0;
    m12 = y2 < y1 ? y2 : y1;
    float miny = m12 < y0 ? m12 : y0;
    M12 = y2 > y1 ? y2 : y1;
    float maxy = M12 > y0 ? M12 : y0;
    int64_t px0 = (int64_t)ceil((double)minx - 0.5);
    int64_t px1 = (int64_t)floor((double)maxx - 0.5);
    int64_t py0 = (int64_t)ceil((double)miny - 0.5);
    int64_t py1 = (int64_t)floor((double)maxy - 0.5);
    if (px0 < 0) px0 = 0;
    if (py0 < 0) py0 = 0;
    if (px1 > w_px - 1) px1 = w_px - 1;
    if (py1 > h_px - 1) py1 = h_px - 1;
    if (px0 > px1 || py0 > py1) continue;
    /* render.py:404-423 flat Lambert from the unswapped world normal */
    float e1x = verts[3 * i1 + 0] - verts[3 * i0 + 0];
    float e1y = verts[3 * i1 + 1] - verts[3 * i0 + 1];
    float e1z = verts[3 * i1 + 2] - verts[3 * i0 + 2];
    float e2x = verts[3 * i2 + 0] - verts[3 * i0 + 0];
    float e2y = verts[3 * i2 + 1] - verts[3 * i0 + 1];
    float e2z = verts[3 * i2 + 2] - verts[3 * i0 + 2];
    float nx = e1y * e2z - e1z * e2y;
    float ny = e1z * e2x - e1x * e2z;
    float nz = e1x * e2y - e1y * e2x;
    float nn = sqrtf(nx * nx + ny * ny + nz * nz);
    if ((double)nn < 1e-20) continue;
    float ndotl32 = (nx * lx + ny * ly + nz * lz) / nn;
    double ndotl = ndotl32 < 0.0f ? 0.0 : (double)ndotl32;
    double shade = AMBIENT + DIFFUSE * ndotl;
    uint8_t cc[3];
    for (int c = 0; c < 3; c++) {
      double v = (double)tri_colors[3 * t + c] * shade * 255.0;
      if (v > 255.0) v = 255.0;
      cc[c] = (uint8_t)v;
    }
    float ax0 = x1 - x0, ay0 = y1 - y0;
    float ax1 = x2 - x1, ay1 = y2 - y1;
    float ax2 = x0 - x2, ay2 = y0 - y2;
    int tl0 = ay0 < 0.0f || (ay0 == 0.0f && ax0 > 0.0f);
    int tl1 = ay1 < 0.0f || (ay1 == 0.0f && ax1 > 0.0f);
    int tl2 = ay2 < 0.0f || (ay2 == 0.0f && ax2 > 0.0f);
    double iz0 = 1.0 / (double)z0;
    double iz1 = 1.0 / (double)z1;
    double iz2 = 1.0 / (double)z2;
    for (int64_t py = py0; py <= py1; py++) {
      double pcy = (double)py + 0.5;
      for (int64_t px = px0; px <= px1; px++) {
        double pcx = (double)px + 0.5;
        double e0 = (double)ax0 * (pcy - (double)y0) - (double)ay0 * (pcx - (double)x0);
        double e1 = (double)ax1 * (pcy - (double)y1) - (double)ay1 * (pcx - (double)x1);
        double e2 = (double)ax2 * (pcy - (double)y2) - (double)ay2 * (pcx - (double)x2);
        if ((e0 > 0.0 || (e0 == 0.0 && tl0)) && (e1 > 0.0 || (e1 == 0.0 && tl1)) &&
            (e2 > 0.0 || (e2 == 0.0 && tl2))) {
          double l0 = e1 / (double)area2;
          double l1 = e2 / (double)area2;
          double l2 = e0 / (double)area2;
          double inv_z = l0 * iz0 + l1 * iz1 + l2 * iz2;
          double zpix = 1.0 / inv_z;
          int64_t i = py * w_px + px;
          if (zpix < (double)depth[i]) {
            depth[i] = (float)zpix;
            pixels[3 * i + 0] = cc[0];
            pixels[3 * i + 1] = cc[1];
            pixels[3 * i + 2] = cc[2];
          }
        }
      }
    }
  }
  free(sxs);
}

/* render.py:459-485 */
void oracle_raster_robot_range(const float *base_verts, const int32_t *vert_link,
                               int64_t nv, const int32_t *tris, int64_t nt,
                               const float *tri_colors, const float *poses32,
                               int64_t n_links, const float *cams,
                               const float *light, int draw_floor,
                               uint8_t *pixels, float *depth, int64_t batch,
                               int64_t h_px, int64_t w_px, int threads) {
  if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    float *world = (float *)malloc(sizeof(float) * (size_t)(nv > 0 ? nv : 1) * 3);
#pragma omp for schedule(static)
    for (int64_t b = 0; b < batch; b++) {
      const float *pose = poses32 + b * n_links * 3;
      for (int64_t i = 0; i < nv; i++) {
        int32_t link = vert_link[i];
        float ox = pose[3 * link + 0];
        float oz = pose[3 * link + 1];
        float th = pose[3 * link + 2];
        float c = oracle_cosf(th);
        float s = oracle_sinf(th);
        float vx = base_verts[3 * i + 0];
        float vy = base_verts[3 * i + 1];
        float vz = base_verts[3 * i + 2];
        world[3 * i + 0] = ox + vx * c - vz * s;
        world[3 * i + 1] = vy;
        world[3 * i + 2] = oz + vx * s + vz * c;
      }
      oracle_raster_scene(world, nv, tris, nt, tri_colors, cams + 15 * b, light,
                          draw_floor, pixels + b * h_px * w_px * 3,
                          depth + b * h_px * w_px, h_px, w_px);
    }
    free(world);
  }
}

/* distractor.py:140-161 -- clamp-add through a per-env 3x256 LUT */
void oracle_color_kernel(uint8_t *pixels, const int64_t *bias, int64_t batch,
                         int64_t h, int64_t w, int threads) {
  if (threads < 1) threads = 1;
  int64_t n = h * w;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t b = 0; b < batch; b++) {
    uint8_t lut[3][256];
    for (int c = 0; c < 3; c++) {
      int64_t off = bias[3 * b + c];
      for (int64_t v = 0; v < 256; v++) {
        int64_t s = v + off;
        if (s < 0) s = 0;
        else if (s > 255) s = 255;
        lut[c][v] = (uint8_t)s;
      }
    }
    uint8_t *flat = pixels + b * n * 3;
    for (int64_t i = 0; i < n; i++) {
      flat[3 * i + 0] = lut[0][flat[3 * i + 0]];
      flat[3 * i + 1] = lut[1][flat[3 * i + 1]];
      flat[3 * i + 2] = lut[2][flat[3 * i + 2]];
    }
  }
}

/* distractor.py:164-176 -- background (isinf(depth)) replaced by the NN-scaled
 * video frame; foreground untouched. */
void oracle_video_kernel(uint8_t *pixels, const float *depth,
                         const uint8_t *frames_flat, int64_t hv, int64_t wv,
                         const int64_t *frame_idx, const int64_t *row_map,
                         const int64_t *col_map, int64_t batch, int64_t h,
                         int64_t w, int threads) {
  if (threads < 1) threads = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t b = 0; b < batch; b++) {
    const uint8_t *fr = frames_flat + frame_idx[b] * hv * wv * 3;
    for (int64_t y = 0; y < h; y++) {
      int64_t sy = row_map[y];
      for (int64_t x = 0; x < w; x++) {
        int64_t i = (b * h + y) * w + x;
        if (isinf(depth[i])) {
          int64_t sx = col_map[x];
          const uint8_t *src = fr + (sy * wv + sx) * 3;
          pixels[3 * i + 0] = src[0];
          pixels[3 * i + 1] = src[1];
          pixels[3 * i + 2] = src[2];
        }
      }
    }
  }
}

/* env.py:168-173 */
void oracle_grayscale(const uint8_t *rgb, uint8_t *gray, int64_t n_px) {
  for (int64_t i = 0; i < n_px; i++) {
    uint32_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    gray[i] = (uint8_t)((299u * r + 587u * g + 114u * b + 500u) / 1000u);
  }
}

/* distractor.py:128-136 */
void oracle_video_advance(int64_t *cursor, int8_t *direction,
                          const int64_t *frame_count, int64_t batch) {
  for (int64_t i = 0; i < batch; i++) {
    /* numpy evaluates both masks on the pre-reflection value */
    int64_t nxt = cursor[i] + direction[i];
    int hi_end = nxt >= frame_count[i];
    int lo_end = nxt < 0;
    if (hi_end) {
      nxt = frame_count[i] - 2;
      direction[i] = -1;
    }
    if (lo_end) {
      nxt = 1;
      direction[i] = 1;
    }
    cursor[i] = nxt;
  }
}

// Fused robot render + distractor composite for sm_100a.
//
// Replaces, in one launch per step, the reference's per-step observation
// path (all paths under /root/reference/pkg/src/pixelctrl/):
//   Env._render_frame / _postprocess            env.py:155-173
//   render_robot_batch -> _raster_robot_range   render.py:594-623, 459-485
//   _raster_scene (clear, floor, project, tris) render.py:286-456
//   advance_distractors + auto-reset re-draw    distractor.py:116-137, env.py:239-244
//   _color_kernel / _video_kernel               distractor.py:140-176
//
// Design (B200-first):
//   * persistent CTAs (grid = SMs x resident CTAs), one env per CTA
//     iteration; 8 warps;
//   * vertex phase: per-link glibc-exact cosf/sinf once per link, then
//     world transform + projection of every vertex into shared memory;
//   * triangle setup: every triangle in parallel, live ones write a 64-B
//     record and set their bit in the bitmask of each 16x8 screen tile their
//     pixel bbox touches -- walking a tile's bits in increasing order IS the
//     reference's sequential triangle order, with no sort and no atomics on
//     the z-buffer;
//   * raster: one warp per tile at a time (dynamic tile queue); the tile's
//     z-buffer and colours live in shared memory; for each triangle in index
//     order the 32 lanes cover the triangle's bbox-in-tile pixels and run
//     the reference's exact f64 edge/barycentric/depth test;
//   * composite (floor, sky, video texel or colour clamp-add, grayscale) is
//     fused into the tile epilogue and packed into a shared-memory frame
//     that one thread writes to HBM with a single TMA bulk store
//     (cp.async.bulk) overlapped with the next env's setup.
// Compiled with -fmad=false: no FMA contraction anywhere, so every f32/f64
// operation rounds where numba's code does.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_math.cuh"

namespace pxr {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileW = 16;
constexpr int kTileH = 8;
constexpr int kTilePx = kTileW * kTileH;  // 128: 4 px per lane
constexpr int kMaxLinks = 64;

constexpr uint32_t kSkyRGB = 135u | (206u << 8) | (235u << 16);  // render.py:50

struct __align__(16) TriRec {
  float x0, y0, x1, y1;
  float x2, y2, area2;
  uint32_t rgbf;  // r | g<<8 | b<<16 | tl0<<24 | tl1<<25 | tl2<<26
  double iz0, iz1;
  double iz2;
  int16_t px0, px1, py0, py1;
};
static_assert(sizeof(TriRec) == 64, "TriRec must stay 64 bytes");

struct RenderParams {
  const float *base_verts;
  const int32_t *vert_link;
  const int32_t *tris;
  const float *tri_colors;
  int nv, nt, nl;
  float cam[15];
  double off_x, off_z;
  float light[3];
  const double *floor_rays;
  int floor_sep;
  const double *poses;
  int64_t batch;
  int H, W, draw_floor;
  int mode;
  int16_t *color_bias;
  int64_t *video_index;
  int64_t *frame_cursor;
  int8_t *direction;
  int64_t *frame_count;
  const uint8_t *frames;
  const int64_t *starts;
  const int64_t *counts;
  int64_t n_videos;
  int Hv, Wv;
  int advance;
  uint64_t key_hi, key_lo, env_offset, logical_batch;
  const uint8_t *done;
  int gray;
  uint8_t *out;
  float *out_depth;
  // derived on the host
  int tiles_x, tiles_y, n_tiles, words;
  int frame_bytes;  // H*W*C
  int frame_smem;   // frame_bytes rounded up to 16
  int use_bulk;
  int vec4;         // W % 4 == 0: 4-pixel groups are 4-byte aligned in the frame
};

struct SmemLayout {
  int off_link, off_floor, off_vx, off_rec, off_bits, off_tile, off_frame, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(int nl, int nv, int nt, int H, int W,
                                                  int n_tiles, int words, int frame_smem) {
  SmemLayout L;
  int o = 0;
  L.off_link = o;  o += align_up(nl * 16, 16);
  L.off_floor = o; o += align_up((W + 2 * H) * 8, 16);
  L.off_vx = o;    o += align_up(nv * 4, 16) * 6;  // sx, sy, sz, wx, wy, wz
  L.off_rec = o;   o += nt * (int)sizeof(TriRec);
  L.off_bits = o;  o += align_up(n_tiles * words * 4, 16);
  L.off_tile = o;  o += kWarps * kTilePx * 8;      // depth f32 + rgb u32 per warp
  L.off_frame = o; o += frame_smem;
  L.total = o;
  return L;
}

struct EnvShared {
  float ex, ez;
  int bias[3];
  int64_t frame_idx;
  int tile_next;
};

__device__ __forceinline__ void composite_px(const RenderParams &p, const EnvShared &es,
                                             float depth, uint32_t rgb, int x, int y,
                                             uint8_t out[3]) {
  int r = rgb & 0xff, g = (rgb >> 8) & 0xff, b = (rgb >> 16) & 0xff;
  if (p.mode == PXR_MODE_VIDEO) {
    if (isinf(depth)) {  // distractor.py:172-176, nearest_map 179-181
      const int sy = (int)(((int64_t)y * p.Hv) / p.H);
      const int sx = (int)(((int64_t)x * p.Wv) / p.W);
      const uint8_t *src =
          p.frames + ((es.frame_idx * p.Hv + sy) * (int64_t)p.Wv + sx) * 3;
      r = __ldg(src);
      g = __ldg(src + 1);
      b = __ldg(src + 2);
    }
  } else if (p.mode == PXR_MODE_COLOR) {  // distractor.py:149-161 clamp-add
    r = min(255, max(0, r + es.bias[0]));
    g = min(255, max(0, g + es.bias[1]));
    b = min(255, max(0, b + es.bias[2]));
  }
  out[0] = (uint8_t)r;
  out[1] = (uint8_t)g;
  out[2] = (uint8_t)b;
}

// Background of one pixel: sky, or the checker floor (render.py:306-344).
__device__ __forceinline__ void background_px(const RenderParams &p, const EnvShared &es,
                                              const double *s_floor, int x, int y,
                                              float &depth, uint32_t &rgb) {
  depth = __int_as_float(0x7f800000);
  rgb = kSkyRGB;
  if (!p.draw_floor) return;
  double dx, dy, dz;
  if (p.floor_sep) {
    dx = s_floor[x];
    dy = s_floor[p.W + y];
    dz = s_floor[p.W + p.H + y];
  } else {
    const double *r = p.floor_rays + ((int64_t)y * p.W + x) * 3;
    dx = r[0];
    dy = r[1];
    dz = r[2];
  }
  if (dz < -1e-12) {
    const double t = (double)(-es.ez) / dz;
    if ((double)p.cam[13] <= t && t <= (double)p.cam[14]) {
      const double wx = (double)es.ex + t * dx;
      const double wy = (double)p.cam[1] + t * dy;
      const int64_t parity = ((int64_t)floor(wx) + (int64_t)floor(wy)) & 1;
      const uint32_t c = parity == 0 ? 158u : 122u;  // render.py:51-52
      rgb = c | (c << 8) | (c << 16);
      depth = (float)t;
    }
  }
}

__global__ void __launch_bounds__(kThreads)
render_step_kernel(const RenderParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ EnvShared es;
  const SmemLayout L = smem_layout(p.nl, p.nv, p.nt, p.H, p.W, p.n_tiles, p.words, p.frame_smem);
  float4 *s_link = reinterpret_cast<float4 *>(smem + L.off_link);
  double *s_floor = reinterpret_cast<double *>(smem + L.off_floor);
  const int nv_al = align_up(p.nv, 4);
  float *s_sx = reinterpret_cast<float *>(smem + L.off_vx);
  float *s_sy = s_sx + nv_al;
  float *s_sz = s_sy + nv_al;
  float *s_wx = s_sz + nv_al;
  float *s_wy = s_wx + nv_al;
  float *s_wz = s_wy + nv_al;
  TriRec *s_rec = reinterpret_cast<TriRec *>(smem + L.off_rec);
  uint32_t *s_bits = reinterpret_cast<uint32_t *>(smem + L.off_bits);
  unsigned char *s_tile_base = smem + L.off_tile;
  uint8_t *s_frame = smem + L.off_frame;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const double aspect = (double)p.W / (double)p.H;  // render.py:303
  const float ey = p.cam[1];
  const float rx = p.cam[3], ry = p.cam[4], rz = p.cam[5];
  const float ux = p.cam[6], uy = p.cam[7], uz = p.cam[8];
  const float fx = p.cam[9], fy = p.cam[10], fz = p.cam[11];
  const float tanf_ = p.cam[12], near_ = p.cam[13], far_ = p.cam[14];
  const float lx = p.light[0], ly = p.light[1], lz = p.light[2];
  const int n_bits_words = p.n_tiles * p.words;

  // Separable floor rays: one x-sequence + per-row y/z, staged once per CTA.
  if (p.draw_floor && p.floor_sep) {
    for (int i = tid; i < p.W; i += kThreads) s_floor[i] = p.floor_rays[(int64_t)i * 3];
    for (int i = tid; i < p.H; i += kThreads) {
      s_floor[p.W + i] = p.floor_rays[(int64_t)i * p.W * 3 + 1];
      s_floor[p.W + p.H + i] = p.floor_rays[(int64_t)i * p.W * 3 + 2];
    }
  }

  for (int64_t env = blockIdx.x; env < p.batch; env += gridDim.x) {
    const uint64_t g = p.env_offset + (uint64_t)env;

    // ---- phase 0: per-link trig, per-env camera, distractor state -------
    for (int l = tid; l < p.nl; l += kThreads) {
      const double *pp = p.poses + ((int64_t)env * p.nl + l) * 3;
      const float th = (float)pp[2];  // poses.astype(float32), render.py:613
      s_link[l] = make_float4((float)pp[0], (float)pp[1], glibc_sincosf(th, 1),
                              glibc_sincosf(th, 0));
    }
    if (tid == 32) {
      const double *p0 = p.poses + (int64_t)env * p.nl * 3;
      es.ex = (float)(p0[0] + p.off_x);  // render.py:611
      es.ez = (float)(p0[1] + p.off_z);  // render.py:612
      es.tile_next = 0;
      if (p.mode == PXR_MODE_COLOR) {
        int16_t b3[3];
        if (p.advance) {
          // advance_distractors (distractor.py:123-126): e = fold_in(key_t, g)
          uint64_t ehi, elo;
          threefry2x64(p.key_hi, p.key_lo, g, 2, ehi, elo);
          color_bias_from_key(ehi, elo, b3);
          for (int c = 0; c < 3; c++) p.color_bias[env * 3 + c] = b3[c];
        } else {
          for (int c = 0; c < 3; c++) b3[c] = p.color_bias[env * 3 + c];
        }
        for (int c = 0; c < 3; c++) es.bias[c] = b3[c];
      } else if (p.mode == PXR_MODE_VIDEO) {
        int64_t vid = p.video_index[env];
        int64_t cur = p.frame_cursor[env];
        if (p.advance) {
          // distractor.py:128-136 ping-pong (both masks on the raw value)
          int dir = p.direction[env];
          const int64_t cnt = p.frame_count[env];
          int64_t nxt = cur + dir;
          const bool hi_end = nxt >= cnt, lo_end = nxt < 0;
          if (hi_end) { nxt = cnt - 2; dir = -1; }
          if (lo_end) { nxt = 1; dir = 1; }
          cur = nxt;
          if (p.done != nullptr && p.done[env]) {
            // env.py:226-244: r = fold_in(key_t, LB + g); new video index
            uint64_t rhi, rlo, w0, w1;
            threefry2x64(p.key_hi, p.key_lo, p.logical_batch + g, 2, rhi, rlo);
            threefry2x64(rhi, rlo, 2, 0, w0, w1);
            vid = index_from_word(w0, (uint64_t)p.n_videos);
            cur = 0;
            dir = 1;
            p.video_index[env] = vid;
            p.frame_count[env] = p.counts[vid];
          }
          p.frame_cursor[env] = cur;
          p.direction[env] = (int8_t)dir;
        }
        es.frame_idx = p.starts[vid] + cur;  // distractor.py:204
      }
    }
    for (int i = tid; i < n_bits_words; i += kThreads) s_bits[i] = 0u;
    __syncthreads();

    // ---- phase 1: world transform + projection (render.py:468-481, 350-363)
    for (int v = tid; v < p.nv; v += kThreads) {
      const float4 lk = s_link[p.vert_link[v]];
      const float bx = p.base_verts[3 * v + 0];
      const float by = p.base_verts[3 * v + 1];
      const float bz = p.base_verts[3 * v + 2];
      const float wx = lk.x + bx * lk.z - bz * lk.w;
      const float wy = by;
      const float wz = lk.y + bx * lk.w + bz * lk.z;
      s_wx[v] = wx;
      s_wy[v] = wy;
      s_wz[v] = wz;
      const float vx = wx - es.ex, vy = wy - ey, vz = wz - es.ez;
      const float zv = vx * fx + vy * fy + vz * fz;
      s_sz[v] = zv;
      float sx = 0.0f, sy = 0.0f;
      if ((double)zv > 1e-9) {
        const float xv = vx * rx + vy * ry + vz * rz;
        const float yv = vx * ux + vy * uy + vz * uz;
        sx = (float)(((double)xv / ((double)(zv * tanf_) * aspect) + 1.0) *
                     ((double)p.W / 2.0));
        sy = (float)((1.0 - (double)(yv / (zv * tanf_))) * ((double)p.H / 2.0));
      }
      s_sx[v] = sx;
      s_sy[v] = sy;
    }
    __syncthreads();

    // ---- phase 2: triangle setup + tile binning (render.py:366-436) ------
    for (int t = tid; t < p.nt; t += kThreads) {
      const int i0 = p.tris[3 * t + 0], i1 = p.tris[3 * t + 1], i2 = p.tris[3 * t + 2];
      float z0 = s_sz[i0], z1 = s_sz[i1], z2 = s_sz[i2];
      if (z0 < near_ || z1 < near_ || z2 < near_) continue;
      if (z0 > far_ && z1 > far_ && z2 > far_) continue;
      float x0 = s_sx[i0], y0 = s_sy[i0];
      float x1 = s_sx[i1], y1 = s_sy[i1];
      float x2 = s_sx[i2], y2 = s_sy[i2];
      float area2 = (x1 - x0) * (y2 - y0) - (y1 - y0) * (x2 - x0);
      if (area2 == 0.0f) continue;
      if (area2 < 0.0f) {
        float tmp;
        tmp = x1; x1 = x2; x2 = tmp;
        tmp = y1; y1 = y2; y2 = tmp;
        tmp = z1; z1 = z2; z2 = tmp;
        area2 = -area2;
      }
      const float minx = fminf(x0, fminf(x1, x2)), maxx = fmaxf(x0, fmaxf(x1, x2));
      const float miny = fminf(y0, fminf(y1, y2)), maxy = fmaxf(y0, fmaxf(y1, y2));
      // int(ceil(min - 0.5)) .. int(floor(max - 0.5)), clamped (render.py:390-403)
      double bx0 = ceil((double)minx - 0.5), bx1 = floor((double)maxx - 0.5);
      double by0 = ceil((double)miny - 0.5), by1 = floor((double)maxy - 0.5);
      if (bx0 < 0.0) bx0 = 0.0;
      if (by0 < 0.0) by0 = 0.0;
      if (bx1 > (double)(p.W - 1)) bx1 = (double)(p.W - 1);
      if (by1 > (double)(p.H - 1)) by1 = (double)(p.H - 1);
      if (bx0 > bx1 || by0 > by1) continue;
      // flat Lambert from the UNswapped world-space normal (render.py:405-423)
      const float e1x = s_wx[i1] - s_wx[i0], e1y = s_wy[i1] - s_wy[i0], e1z = s_wz[i1] - s_wz[i0];
      const float e2x = s_wx[i2] - s_wx[i0], e2y = s_wy[i2] - s_wy[i0], e2z = s_wz[i2] - s_wz[i0];
      const float nx = e1y * e2z - e1z * e2y;
      const float ny = e1z * e2x - e1x * e2z;
      const float nz = e1x * e2y - e1y * e2x;
      const float nn = sqrtf(nx * nx + ny * ny + nz * nz);
      if ((double)nn < 1e-20) continue;
      const float nd32 = (nx * lx + ny * ly + nz * lz) / nn;
      const double ndotl = nd32 < 0.0f ? 0.0 : (double)nd32;
      const double shade = 0.35 + 0.65 * ndotl;
      uint32_t rgbf = 0;
      for (int c = 0; c < 3; c++) {
        double v = (double)p.tri_colors[3 * t + c] * shade * 255.0;
        if (v > 255.0) v = 255.0;
        rgbf |= ((uint32_t)v & 0xffu) << (8 * c);
      }
      const float ax0 = x1 - x0, ay0 = y1 - y0;
      const float ax1 = x2 - x1, ay1 = y2 - y1;
      const float ax2 = x0 - x2, ay2 = y0 - y2;
      if (ay0 < 0.0f || (ay0 == 0.0f && ax0 > 0.0f)) rgbf |= 1u << 24;
      if (ay1 < 0.0f || (ay1 == 0.0f && ax1 > 0.0f)) rgbf |= 1u << 25;
      if (ay2 < 0.0f || (ay2 == 0.0f && ax2 > 0.0f)) rgbf |= 1u << 26;
      TriRec r;
      r.x0 = x0; r.y0 = y0; r.x1 = x1; r.y1 = y1; r.x2 = x2; r.y2 = y2;
      r.area2 = area2;
      r.rgbf = rgbf;
      r.iz0 = 1.0 / (double)z0;
      r.iz1 = 1.0 / (double)z1;
      r.iz2 = 1.0 / (double)z2;
      const int ix0 = (int)bx0, ix1 = (int)bx1, iy0 = (int)by0, iy1 = (int)by1;
      r.px0 = (int16_t)ix0; r.px1 = (int16_t)ix1; r.py0 = (int16_t)iy0; r.py1 = (int16_t)iy1;
      s_rec[t] = r;
      const uint32_t bit = 1u << (t & 31);
      const int word = t >> 5;
      for (int ty = iy0 / kTileH; ty <= iy1 / kTileH; ty++)
        for (int tx = ix0 / kTileW; tx <= ix1 / kTileW; tx++)
          atomicOr(&s_bits[(ty * p.tiles_x + tx) * p.words + word], bit);
    }
    // The previous env's TMA store must have finished reading s_frame.
    if (tid == 0 && p.use_bulk) bulk_wait_read();
    __syncthreads();

    // ---- phase 3: tiles -------------------------------------------------
    float *t_depth = reinterpret_cast<float *>(s_tile_base + warp * kTilePx * 8);
    uint32_t *t_rgb = reinterpret_cast<uint32_t *>(t_depth + kTilePx);
    while (true) {
      int tile = 0;
      if (lane == 0) tile = atomicAdd(&es.tile_next, 1);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      if (tile >= p.n_tiles) break;
      const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
      const int xb = tx * kTileW, yb = ty * kTileH;
      const uint32_t *tb = s_bits + tile * p.words;
      bool any = false;
      for (int w = lane; w < p.words; w += 32) any |= tb[w] != 0u;
      any = __any_sync(0xffffffffu, any);
      // lane -> 4 horizontally adjacent pixels of the 16x8 tile
      const int ly_ = lane >> 2, lx4 = (lane & 3) * 4;
      const int y = yb + ly_;
      float dpx[4];
      uint32_t cpx[4];
      if (any) {
        for (int k = 0; k < 4; k++) {
          const int x = xb + lx4 + k;
          float d = __int_as_float(0x7f800000);
          uint32_t c = 0;
          if (x < p.W && y < p.H) background_px(p, es, s_floor, x, y, d, c);
          t_depth[ly_ * kTileW + lx4 + k] = d;
          t_rgb[ly_ * kTileW + lx4 + k] = c;
        }
        __syncwarp();
        for (int w = 0; w < p.words; w++) {
          uint32_t m = tb[w];
          while (m) {
            const int t = w * 32 + __ffs(m) - 1;
            m &= m - 1;
            const TriRec r = s_rec[t];
            const int cx0 = max((int)r.px0, xb), cx1 = min((int)r.px1, xb + kTileW - 1);
            const int cy0 = max((int)r.py0, yb), cy1 = min((int)r.py1, yb + kTileH - 1);
            const int bw = cx1 - cx0 + 1, bh = cy1 - cy0 + 1;
            if (bw <= 0 || bh <= 0) continue;
            const int n = bw * bh;
            const uint32_t magic = (65536u + bw - 1) / bw;
            const float ax0 = r.x1 - r.x0, ay0 = r.y1 - r.y0;
            const float ax1 = r.x2 - r.x1, ay1 = r.y2 - r.y1;
            const float ax2 = r.x0 - r.x2, ay2 = r.y0 - r.y2;
            const bool tl0 = (r.rgbf >> 24) & 1, tl1 = (r.rgbf >> 25) & 1, tl2 = (r.rgbf >> 26) & 1;
            const uint32_t rgb = r.rgbf & 0xffffffu;
            for (int i = lane; i < n; i += 32) {
              const int q = (int)(((uint32_t)i * magic) >> 16);
              const int px = cx0 + (i - q * bw), py = cy0 + q;
              const double pcx = (double)px + 0.5, pcy = (double)py + 0.5;
              // render.py:441-446, inclusive top-left rule
              const double e0 = (double)ax0 * (pcy - (double)r.y0) - (double)ay0 * (pcx - (double)r.x0);
              const double e1 = (double)ax1 * (pcy - (double)r.y1) - (double)ay1 * (pcx - (double)r.x1);
              const double e2 = (double)ax2 * (pcy - (double)r.y2) - (double)ay2 * (pcx - (double)r.x2);
              if ((e0 > 0.0 || (e0 == 0.0 && tl0)) && (e1 > 0.0 || (e1 == 0.0 && tl1)) &&
                  (e2 > 0.0 || (e2 == 0.0 && tl2))) {
                const double a2 = (double)r.area2;
                const double l0 = e1 / a2, l1 = e2 / a2, l2 = e0 / a2;
                const double inv_z = l0 * r.iz0 + l1 * r.iz1 + l2 * r.iz2;
                const double zpix = 1.0 / inv_z;
                const int idx = (py - yb) * kTileW + (px - xb);
                if (zpix < (double)t_depth[idx]) {  // strict: ties keep the lower index
                  t_depth[idx] = (float)zpix;
                  t_rgb[idx] = rgb;
                }
              }
            }
            __syncwarp();
          }
        }
        for (int k = 0; k < 4; k++) {
          dpx[k] = t_depth[ly_ * kTileW + lx4 + k];
          cpx[k] = t_rgb[ly_ * kTileW + lx4 + k];
        }
        __syncwarp();
      } else {
        for (int k = 0; k < 4; k++) {
          const int x = xb + lx4 + k;
          dpx[k] = __int_as_float(0x7f800000);
          cpx[k] = 0;
          if (x < p.W && y < p.H) background_px(p, es, s_floor, x, y, dpx[k], cpx[k]);
        }
      }
      // ---- tile epilogue: composite + pack into the smem frame ----------
      if (y < p.H) {
        const int x0 = xb + lx4;
        uint8_t o[4][3];
        for (int k = 0; k < 4; k++) {
          const int x = x0 + k;
          if (x < p.W) composite_px(p, es, dpx[k], cpx[k], x, y, o[k]);
        }
        const int base = y * p.W + x0;
        if (p.gray) {
          uint8_t gv[4];
          for (int k = 0; k < 4; k++)  // env.py:168-173
            gv[k] = (uint8_t)((299u * o[k][0] + 587u * o[k][1] + 114u * o[k][2] + 500u) / 1000u);
          if (p.vec4 && x0 + 3 < p.W) {
            *reinterpret_cast<uint32_t *>(s_frame + base) =
                gv[0] | (gv[1] << 8) | (gv[2] << 16) | ((uint32_t)gv[3] << 24);
          } else {
            for (int k = 0; k < 4; k++)
              if (x0 + k < p.W) s_frame[base + k] = gv[k];
          }
        } else {
          if (p.vec4 && x0 + 3 < p.W) {
            uint32_t *dst = reinterpret_cast<uint32_t *>(s_frame + base * 3);
            dst[0] = o[0][0] | (o[0][1] << 8) | (o[0][2] << 16) | ((uint32_t)o[1][0] << 24);
            dst[1] = o[1][1] | (o[1][2] << 8) | (o[2][0] << 16) | ((uint32_t)o[2][1] << 24);
            dst[2] = o[2][2] | (o[3][0] << 8) | (o[3][1] << 16) | ((uint32_t)o[3][2] << 24);
          } else {
            for (int k = 0; k < 4; k++)
              if (x0 + k < p.W)
                for (int c = 0; c < 3; c++) s_frame[(base + k) * 3 + c] = o[k][c];
          }
        }
        if (p.out_depth != nullptr) {
          float *dd = p.out_depth + ((int64_t)env * p.H + y) * p.W + x0;
          if (p.vec4 && x0 + 3 < p.W) {
            *reinterpret_cast<float4 *>(dd) = make_float4(dpx[0], dpx[1], dpx[2], dpx[3]);
          } else {
            for (int k = 0; k < 4; k++)
              if (x0 + k < p.W) dd[k] = dpx[k];
          }
        }
      }
    }

    // ---- phase 4: frame -> HBM -------------------------------------------
    uint8_t *gout = p.out + (int64_t)env * p.frame_bytes;
    if (p.use_bulk) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) bulk_store_s2g(gout, s_frame, p.frame_bytes);
    } else {
      __syncthreads();
      for (int i = tid; i < p.frame_bytes; i += kThreads) gout[i] = s_frame[i];
      __syncthreads();
    }
  }
  if (tid == 0 && p.use_bulk) bulk_wait_all();
}

// One thread per image row walks x exactly like render.py:321-344.
__global__ void floor_rays_kernel(const float *__restrict__ cam_dev_unused, float rx, float ry,
                                  float rz, float ux, float uy, float uz, float fx, float fy,
                                  float fz, float tanf_, int H, int W, double *out) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= H) return;
  const double aspect = (double)W / (double)H;
  const double sx0 = (1.0 / (double)W - 1.0) * (double)tanf_ * aspect;
  const double dsx = (2.0 / (double)W) * (double)tanf_ * aspect;
  const double drx = dsx * (double)rx, dry = dsx * (double)ry, drz = dsx * (double)rz;
  const double sy = (1.0 - 2.0 * ((double)y + 0.5) / (double)H) * (double)tanf_;
  double dx = (double)fx + sx0 * (double)rx + sy * (double)ux;
  double dy = (double)fy + sx0 * (double)ry + sy * (double)uy;
  double dz = (double)fz + sx0 * (double)rz + sy * (double)uz;
  double *o = out + (int64_t)y * W * 3;
  for (int x = 0; x < W; x++) {
    o[3 * x + 0] = dx;
    o[3 * x + 1] = dy;
    o[3 * x + 2] = dz;
    dx += drx;
    dy += dry;
    dz += drz;
  }
}

static int g_num_sms = 0;

static int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

}  // namespace pxr

using namespace pxr;

extern "C" pxr_status pxr_floor_rays(const float *cam, int64_t height, int64_t width,
                                     double *out_rays, int32_t *separable, void *stream) {
  if (cam == nullptr || out_rays == nullptr || height < 1 || width < 1)
    return set_invalid("pxr_floor_rays: bad arguments");
  if (separable != nullptr) {
    // ry == rz == 0 and ux == 0: y/z constant along x, one x-sequence per row
    *separable = (cam[4] == 0.0f && cam[5] == 0.0f && cam[6] == 0.0f) ? 1 : 0;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  floor_rays_kernel<<<(unsigned)((height + 63) / 64), 64, 0, st>>>(
      nullptr, cam[3], cam[4], cam[5], cam[6], cam[7], cam[8], cam[9], cam[10], cam[11],
      cam[12], (int)height, (int)width, out_rays);
  return check_launch("floor_rays_kernel");
}

extern "C" pxr_status pxr_render_step(const pxr_geometry *geom, const pxr_camera *cam,
                                      const double *poses, int64_t batch, int64_t height,
                                      int64_t width, int32_t draw_floor,
                                      const pxr_distractor *dist, const pxr_video_pack *pack,
                                      int32_t advance, const pxr_step_keys *keys,
                                      const uint8_t *done, int32_t grayscale,
                                      uint8_t *out_obs, float *out_depth, void *stream) {
  if (geom == nullptr || cam == nullptr || dist == nullptr)
    return set_invalid("pxr_render_step: null struct");
  if (batch < 1) return set_invalid("batch must be >= 1");
  if (height < 8 || width < 8) return set_invalid("frames must be at least 8x8");
  if (height > 4096 || width > 4096) return set_unsupported("frames above 4096 px per side");
  if (poses == nullptr || out_obs == nullptr) return set_invalid("null poses/out_obs");
  if (geom->n_links < 1 || geom->n_links > kMaxLinks || geom->n_verts < 0 || geom->n_tris < 0)
    return set_invalid("bad geometry sizes");
  if (geom->n_verts > 0 && (geom->base_verts == nullptr || geom->vert_link == nullptr))
    return set_invalid("null geometry vertex arrays");
  if (geom->n_tris > 0 && (geom->triangles == nullptr || geom->tri_colors == nullptr))
    return set_invalid("null geometry triangle arrays");
  if (draw_floor && cam->floor_rays == nullptr) return set_invalid("floor requested without rays");
  const int mode = dist->mode;
  if (mode != PXR_MODE_NONE && mode != PXR_MODE_COLOR && mode != PXR_MODE_VIDEO)
    return set_invalid("unknown distractor mode");
  if (mode == PXR_MODE_COLOR && dist->color_bias == nullptr)
    return set_invalid("colour mode needs color_bias");
  if (mode == PXR_MODE_VIDEO) {
    if (pack == nullptr || pack->frames == nullptr || pack->starts == nullptr ||
        pack->counts == nullptr || pack->n_videos < 1)
      return set_invalid("video distractors need a loaded video pack");
    if (dist->video_index == nullptr || dist->frame_cursor == nullptr ||
        dist->direction == nullptr || dist->frame_count == nullptr)
      return set_invalid("video mode needs the full distractor state");
  }
  if (advance && keys == nullptr) return set_invalid("advance needs step keys");

  RenderParams p{};
  p.base_verts = geom->base_verts;
  p.vert_link = geom->vert_link;
  p.tris = geom->triangles;
  p.tri_colors = geom->tri_colors;
  p.nv = geom->n_verts;
  p.nt = geom->n_tris;
  p.nl = geom->n_links;
  for (int i = 0; i < 15; i++) p.cam[i] = cam->block[i];
  p.off_x = cam->offset_x;
  p.off_z = cam->offset_z;
  for (int i = 0; i < 3; i++) p.light[i] = cam->light[i];
  p.floor_rays = cam->floor_rays;
  p.floor_sep = cam->floor_separable;
  p.poses = poses;
  p.batch = batch;
  p.H = (int)height;
  p.W = (int)width;
  p.draw_floor = draw_floor ? 1 : 0;
  p.mode = mode;
  p.color_bias = dist->color_bias;
  p.video_index = dist->video_index;
  p.frame_cursor = dist->frame_cursor;
  p.direction = dist->direction;
  p.frame_count = dist->frame_count;
  if (mode == PXR_MODE_VIDEO) {
    p.frames = pack->frames;
    p.starts = pack->starts;
    p.counts = pack->counts;
    p.n_videos = pack->n_videos;
    p.Hv = (int)pack->height;
    p.Wv = (int)pack->width;
  }
  p.advance = advance ? 1 : 0;
  if (keys != nullptr) {
    p.key_hi = keys->key_hi;
    p.key_lo = keys->key_lo;
    p.env_offset = keys->env_offset;
    p.logical_batch = keys->logical_batch;
  }
  p.done = done;
  p.gray = grayscale ? 1 : 0;
  p.out = out_obs;
  p.out_depth = out_depth;
  p.tiles_x = (p.W + kTileW - 1) / kTileW;
  p.tiles_y = (p.H + kTileH - 1) / kTileH;
  p.n_tiles = p.tiles_x * p.tiles_y;
  p.words = (p.nt + 31) / 32;
  if (p.words < 1) p.words = 1;
  const int C = p.gray ? 1 : 3;
  p.frame_bytes = p.H * p.W * C;
  p.frame_smem = align_up(p.frame_bytes, 16);
  p.vec4 = (p.W % 4) == 0;
  p.use_bulk = (p.frame_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(out_obs) & 15) == 0);
  if (out_depth != nullptr && (reinterpret_cast<uintptr_t>(out_depth) & 15) != 0) p.vec4 = 0;

  const SmemLayout L = smem_layout(p.nl, p.nv, p.nt, p.H, p.W, p.n_tiles, p.words, p.frame_smem);
  const int smem = L.total;
  int dev = 0;
  cudaGetDevice(&dev);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (smem + (int)sizeof(EnvShared) > max_optin)
    return set_unsupported("mesh/frame too large for one CTA's shared memory");
  cudaError_t e = cudaFuncSetAttribute(render_step_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda(e, "cudaFuncSetAttribute");
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, render_step_kernel, kThreads, smem);
  if (e != cudaSuccess) return set_cuda(e, "occupancy query");
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)num_sms() * per_sm;
  if (grid > batch) grid = batch;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  render_step_kernel<<<(unsigned)grid, kThreads, smem, st>>>(p);
  return check_launch("render_step_kernel");
}

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
//   * persistent CTAs of 16 warps, one env per CTA iteration, everything
//     for the env in shared memory (no HBM round trip between stages);
//   * the env's video frame is fetched into shared memory by a TMA bulk
//     copy (cp.async.bulk + mbarrier) issued at env start;
//   * vertex phase: per-link glibc-exact cosf/sinf once per link, world
//     transform + projection of every vertex (f32 as the reference, f64
//     copies and 1/z for the raster);
//   * triangle setup: liveness ballot + prefix -> compacted live-triangle
//     records (f64 edge coefficients, exact reciprocal of the area) and a
//     bitmask per 8x8 screen tile; bit order == triangle index order, so
//     walking the bits reproduces the reference's sequential z-test order;
//   * raster: a warp owns one tile at a time (heaviest tiles first); the
//     candidate (triangle, pixel) pairs of up to 32 triangles are flat-packed
//     across the 32 lanes (warp scan + shuffle search), each lane runs the
//     reference's exact f64 edge / barycentric / depth arithmetic, and
//     same-pixel fragments inside a pass are applied in triangle order with
//     __match_any_sync rounds;
//   * balanced flat passes for the background (sky / exact f64 floor) and
//     the composite (video texel from shared memory or colour clamp-add,
//     grayscale) into a shared-memory frame that one thread stores with a
//     single TMA bulk copy, overlapped with the next env.
// Compiled with -fmad=false: no FMA contraction, every f32/f64 operation
// rounds where numba's code does. The only FMAs are the
// explicit __fma_rn of the glibc sinf/cosf restatement and of the
// correctly-rounded division below.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_math.cuh"

namespace pxr {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 8;  // 8x8 pixel tiles
constexpr int kMaxLinks = 64;
constexpr uint32_t kFull = 0xffffffffu;

constexpr uint32_t kSkyRGB = 135u | (206u << 8) | (235u << 16);  // render.py:50

// One live triangle after setup (post-swap vertex order, render.py:381-385).
struct __align__(16) TriRec {
  double A0, B0, A1, B1, A2, B2;  // (double) of the f32 edge vectors ax_k, ay_k
  double rcp;                     // RN(1 / (double)area2), for the exact division
  double area;                    // (double)area2
  uint16_t v0, v1, v2, flags;     // vertex ids; top-left bits (render.py:431-433)
  uint32_t rgb;                   // flat-shaded u8 colour
  int16_t px0, px1, py0, py1;     // clamped pixel bbox (render.py:390-403)
  uint32_t pad;
};
static_assert(sizeof(TriRec) == 96, "TriRec layout");

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
  int tiles_x, tiles_y, n_tiles;
  int cap;        // live-triangle records per raster round
  int words;      // bitmask words per tile = cap / 32
  int tri_words;  // ceil(nt / 32)
  int frame_bytes, use_bulk, vec4, vframe_bytes, vframe_bulk;
};

struct SmemLayout {
  int link, floor, maps, vxy64, viz, vxy32, vz, world, rec, bits, tilecnt, queue, live,
      livepfx, depth, col, gray, vframe, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(const RenderParams &p) {
  SmemLayout L;
  int o = 0;
  const int npx = p.H * p.W;
  L.link = o;    o += align_up(p.nl * 16, 16);
  L.floor = o;   o += align_up((p.W + 2 * p.H) * 8, 16);
  L.maps = o;    o += align_up((p.W + p.H) * 2, 16);
  L.vxy64 = o;   o += align_up(p.nv * 16, 16);
  L.viz = o;     o += align_up(p.nv * 8, 16);
  L.vxy32 = o;   o += align_up(p.nv * 8, 16);
  L.vz = o;      o += align_up(p.nv * 4, 16);
  L.world = o;   o += align_up(p.nv * 12, 16);
  L.rec = o;     o += p.cap * (int)sizeof(TriRec);
  L.bits = o;    o += align_up(p.n_tiles * p.words * 4, 16);
  L.tilecnt = o; o += align_up(p.n_tiles * 4, 16);
  L.queue = o;   o += align_up(p.n_tiles * 2, 16);
  L.live = o;    o += align_up(p.tri_words * 4, 16);
  L.livepfx = o; o += align_up(p.tri_words * 4, 16);
  L.depth = o;   o += align_up(npx * 4, 16);
  L.col = o;     o += align_up(npx * 3, 16);
  L.gray = o;    o += p.gray ? align_up(npx, 16) : 0;
  L.vframe = o;  o += p.mode == PXR_MODE_VIDEO ? align_up(p.vframe_bytes, 16) : 0;
  L.total = o;
  return L;
}

struct EnvShared {
  uint64_t vbar;  // mbarrier for the video frame bulk load
  float ex, ez;
  int bias[3];
  int64_t frame_idx;
  int n_live;
  int n_queue;
  int queue_next;
};

struct DistSlot {
  int bias[3];
  int64_t frame_idx;
};

// Per-env distractor step (writes the new state back to HBM):
//   colour: advance_distractors, distractor.py:123-126 -- e = fold_in(key_t, g),
//           biases from draw blocks 0/1 of e (distractor.py:66-74);
//   video:  ping-pong cursor (distractor.py:128-136), then for envs being
//           reset the re-drawn video (env.py:226-244); frame index 204.
// With advance == 0 (make_env / observe) the stored state is used as is.
__device__ __forceinline__ void distractor_update(const RenderParams &p, int64_t env,
                                               DistSlot &out) {
  const uint64_t g = p.env_offset + (uint64_t)env;
  out.bias[0] = out.bias[1] = out.bias[2] = 0;
  out.frame_idx = 0;
  if (p.mode == PXR_MODE_COLOR) {
    int16_t b3[3];
    if (p.advance) {
      uint64_t ehi, elo;
      threefry2x64(p.key_hi, p.key_lo, g, 2, ehi, elo);
      color_bias_from_key(ehi, elo, b3);
      for (int c = 0; c < 3; c++) p.color_bias[env * 3 + c] = b3[c];
    } else {
      for (int c = 0; c < 3; c++) b3[c] = p.color_bias[env * 3 + c];
    }
    for (int c = 0; c < 3; c++) out.bias[c] = b3[c];
  } else if (p.mode == PXR_MODE_VIDEO) {
    int64_t vid = p.video_index[env];
    int64_t cur = p.frame_cursor[env];
    if (p.advance) {
      int dir = p.direction[env];
      const int64_t cnt = p.frame_count[env];
      int64_t nxt = cur + dir;
      const bool hi_end = nxt >= cnt, lo_end = nxt < 0;  // both on the raw value
      if (hi_end) { nxt = cnt - 2; dir = -1; }
      if (lo_end) { nxt = 1; dir = 1; }
      cur = nxt;
      if (p.done != nullptr && p.done[env]) {
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
    out.frame_idx = p.starts[vid] + cur;
  }
}

// Exact RN(a / b) from y = RN(1 / b): q = RN(a*y), r = a - b*q (exact with an
// FMA), q' = RN(q + r*y) (Markstein). Checked against IEEE division by
// tests/test_gpu_parity.py::TestDeviceMath.
__device__ __forceinline__ double div_rn_pre(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-b, q, a);
  return __fma_rn(r, y, q);
}

// k + 0.5 as a double without an int->f64 conversion (exact for 0 <= k < 2^31).
__device__ __forceinline__ double half_plus(int k) {
  const double big = __hiloint2double(0x43300000, k);  // 2^52 + k
  return __dsub_rn(big, 4503599627370495.5);          // (2^52 + k) - (2^52 - 0.5)
}

// Background of one pixel: sky, or the checker floor (render.py:306-344),
// with the row's ray (dy, dz) and t already known for the separable case.
__device__ __forceinline__ void floor_px(const RenderParams &p, const EnvShared &es, double dx,
                                         double dy, double dz, float &depth, uint32_t &rgb) {
  depth = __int_as_float(0x7f800000);
  rgb = kSkyRGB;
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

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int u = __shfl_up_sync(kFull, v, s);
    if (lane >= s) v += u;
  }
  return v;
}

__global__ void __launch_bounds__(kThreads, 1)
render_step_kernel(const RenderParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ EnvShared es;
  __shared__ uint32_t s_magic[kTile + 1];
  __shared__ DistSlot s_dist[32];
  const SmemLayout L = smem_layout(p);
  float4 *s_link = reinterpret_cast<float4 *>(smem + L.link);
  double *s_floor = reinterpret_cast<double *>(smem + L.floor);
  uint16_t *s_rowmap = reinterpret_cast<uint16_t *>(smem + L.maps);
  uint16_t *s_colmap = s_rowmap + p.H;
  double2 *s_vxy64 = reinterpret_cast<double2 *>(smem + L.vxy64);
  double *s_viz = reinterpret_cast<double *>(smem + L.viz);
  float2 *s_vxy32 = reinterpret_cast<float2 *>(smem + L.vxy32);
  float *s_vz = reinterpret_cast<float *>(smem + L.vz);
  float *s_world = reinterpret_cast<float *>(smem + L.world);
  TriRec *s_rec = reinterpret_cast<TriRec *>(smem + L.rec);
  uint32_t *s_bits = reinterpret_cast<uint32_t *>(smem + L.bits);
  uint32_t *s_tilecnt = reinterpret_cast<uint32_t *>(smem + L.tilecnt);
  uint16_t *s_queue = reinterpret_cast<uint16_t *>(smem + L.queue);
  uint32_t *s_live = reinterpret_cast<uint32_t *>(smem + L.live);
  uint32_t *s_livepfx = reinterpret_cast<uint32_t *>(smem + L.livepfx);
  float *s_depth = reinterpret_cast<float *>(smem + L.depth);
  uint8_t *s_col = smem + L.col;
  uint8_t *s_gray = smem + L.gray;
  uint8_t *s_vframe = smem + L.vframe;
  uint8_t *s_out = p.gray ? s_gray : s_col;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int npx = p.H * p.W;
  const double aspect = (double)p.W / (double)p.H;  // render.py:303
  const float ey = p.cam[1];
  const float rx = p.cam[3], ry = p.cam[4], rz = p.cam[5];
  const float ux = p.cam[6], uy = p.cam[7], uz = p.cam[8];
  const float fx = p.cam[9], fy = p.cam[10], fz = p.cam[11];
  const float tanf_ = p.cam[12], near_ = p.cam[13], far_ = p.cam[14];
  const float lx = p.light[0], ly = p.light[1], lz = p.light[2];
  const int n_bits_words = p.n_tiles * p.words;
  const uint32_t lanemask_lt = (1u << lane) - 1u;

  // ---- once per CTA: floor rays, NN maps, division magics, mbarrier ------
  if (p.draw_floor && p.floor_sep) {
    for (int i = tid; i < p.W; i += kThreads) s_floor[i] = p.floor_rays[(int64_t)i * 3];
    for (int i = tid; i < p.H; i += kThreads) {
      s_floor[p.W + i] = p.floor_rays[(int64_t)i * p.W * 3 + 1];
      s_floor[p.W + p.H + i] = p.floor_rays[(int64_t)i * p.W * 3 + 2];
    }
  }
  if (p.mode == PXR_MODE_VIDEO) {  // nearest_map, distractor.py:179-181
    for (int i = tid; i < p.H; i += kThreads) s_rowmap[i] = (uint16_t)(((int64_t)i * p.Hv) / p.H);
    for (int i = tid; i < p.W; i += kThreads) s_colmap[i] = (uint16_t)(((int64_t)i * p.Wv) / p.W);
  }
  if (tid <= kTile) s_magic[tid] = tid == 0 ? 0u : (65536u + tid - 1) / tid;
  if (tid == 0) {
    mbar_init(&es.vbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint32_t vphase = 0;
  int local = 0;
  for (int64_t env = blockIdx.x; env < p.batch; env += gridDim.x, local++) {

    // ---- phase 0: per-link trig, camera, distractor state, video fetch ---
    for (int l = tid; l < p.nl; l += kThreads) {
      const double *pp = p.poses + ((int64_t)env * p.nl + l) * 3;
      const float th = (float)pp[2];  // poses.astype(float32), render.py:613
      s_link[l] = make_float4((float)pp[0], (float)pp[1], glibc_sincosf(th, 1),
                              glibc_sincosf(th, 0));
    }
    if (warp == kWarps - 1) {
      // Distractor state of the next 32 envs of this CTA, one lane each, in
      // lockstep (the Threefry chains then cost one env's latency per 32).
      if (local % 32 == 0) {
        const int64_t e2 = env + (int64_t)lane * gridDim.x;
        if (e2 < p.batch) distractor_update(p, e2, s_dist[lane]);
        __syncwarp();
      }
      if (lane == 0) {
        const double *p0 = p.poses + (int64_t)env * p.nl * 3;
        es.ex = (float)(p0[0] + p.off_x);  // render.py:611
        es.ez = (float)(p0[1] + p.off_z);  // render.py:612
        es.queue_next = 0;
        const DistSlot &ds = s_dist[local % 32];
        es.bias[0] = ds.bias[0];
        es.bias[1] = ds.bias[1];
        es.bias[2] = ds.bias[2];
        es.frame_idx = ds.frame_idx;
        if (p.mode == PXR_MODE_VIDEO && p.vframe_bulk) {
          mbar_arrive_expect_tx(&es.vbar, (uint32_t)p.vframe_bytes);
          bulk_load_g2s(s_vframe, p.frames + ds.frame_idx * p.vframe_bytes,
                        (uint32_t)p.vframe_bytes, &es.vbar);
        }
      }
    }
    for (int i = tid; i < n_bits_words; i += kThreads) s_bits[i] = 0u;
    for (int i = tid; i < p.n_tiles; i += kThreads) s_tilecnt[i] = 0u;
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
      s_world[3 * v + 0] = wx;
      s_world[3 * v + 1] = wy;
      s_world[3 * v + 2] = wz;
      const float vx = wx - es.ex, vy = wy - ey, vz = wz - es.ez;
      const float zv = vx * fx + vy * fy + vz * fz;
      float sx = 0.0f, sy = 0.0f;
      if ((double)zv > 1e-9) {
        const float xv = vx * rx + vy * ry + vz * rz;
        const float yv = vx * ux + vy * uy + vz * uz;
        sx = (float)(((double)xv / ((double)(zv * tanf_) * aspect) + 1.0) *
                     ((double)p.W / 2.0));
        sy = (float)((1.0 - (double)(yv / (zv * tanf_))) * ((double)p.H / 2.0));
      }
      s_vz[v] = zv;
      s_vxy32[v] = make_float2(sx, sy);
      s_vxy64[v] = make_double2((double)sx, (double)sy);
      s_viz[v] = __drcp_rn((double)zv);  // iz = 1.0 / z (render.py:434-436)
    }
    // The previous env's TMA store must have finished reading the frame.
    if (tid == 0 && p.use_bulk) bulk_wait_read();
    __syncthreads();

    // ---- phase 2a: triangle liveness (render.py:366-403) + background ---
    for (int base = 0; base < p.nt; base += kThreads) {
      const int t = base + tid;
      bool live = false;
      if (t < p.nt) {
        const int i0 = p.tris[3 * t + 0], i1 = p.tris[3 * t + 1], i2 = p.tris[3 * t + 2];
        const float z0 = s_vz[i0], z1 = s_vz[i1], z2 = s_vz[i2];
        if (!(z0 < near_ || z1 < near_ || z2 < near_) && !(z0 > far_ && z1 > far_ && z2 > far_)) {
          const float2 a = s_vxy32[i0], b = s_vxy32[i1], c = s_vxy32[i2];
          const float area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
          if (area2 != 0.0f) {
            const float minx = fminf(a.x, fminf(b.x, c.x)), maxx = fmaxf(a.x, fmaxf(b.x, c.x));
            const float miny = fminf(a.y, fminf(b.y, c.y)), maxy = fmaxf(a.y, fmaxf(b.y, c.y));
            double bx0 = ceil((double)minx - 0.5), bx1 = floor((double)maxx - 0.5);
            double by0 = ceil((double)miny - 0.5), by1 = floor((double)maxy - 0.5);
            if (bx0 < 0.0) bx0 = 0.0;
            if (by0 < 0.0) by0 = 0.0;
            if (bx1 > (double)(p.W - 1)) bx1 = (double)(p.W - 1);
            if (by1 > (double)(p.H - 1)) by1 = (double)(p.H - 1);
            if (!(bx0 > bx1 || by0 > by1)) {
              const float *w0 = s_world + 3 * i0, *w1 = s_world + 3 * i1, *w2 = s_world + 3 * i2;
              const float e1x = w1[0] - w0[0], e1y = w1[1] - w0[1], e1z = w1[2] - w0[2];
              const float e2x = w2[0] - w0[0], e2y = w2[1] - w0[1], e2z = w2[2] - w0[2];
              const float nx = e1y * e2z - e1z * e2y;
              const float ny = e1z * e2x - e1x * e2z;
              const float nz = e1x * e2y - e1y * e2x;
              live = !((double)sqrtf(nx * nx + ny * ny + nz * nz) < 1e-20);  // render.py:415
            }
          }
        }
      }
      const uint32_t word = __ballot_sync(kFull, live);
      if (lane == 0 && base + warp * 32 < p.nt) s_live[(base >> 5) + warp] = word;
    }
    // background: sky / floor, and the z-buffer (render.py:306-344)
    if (p.mode == PXR_MODE_VIDEO && !p.draw_floor) {
      float4 *d4 = reinterpret_cast<float4 *>(s_depth);
      const float inf = __int_as_float(0x7f800000);
      for (int i = tid; i < (npx >> 2); i += kThreads) d4[i] = make_float4(inf, inf, inf, inf);
      for (int i = (npx & ~3) + tid; i < npx; i += kThreads) s_depth[i] = inf;
    } else {
      for (int i = tid; i < npx; i += kThreads) {
        const int y = i / p.W, x = i - y * p.W;
        float d = __int_as_float(0x7f800000);
        uint32_t c = kSkyRGB;
        if (p.draw_floor) {
          double dx, dy, dz;
          if (p.floor_sep) {
            dx = s_floor[x]; dy = s_floor[p.W + y]; dz = s_floor[p.W + p.H + y];
          } else {
            const double *r = p.floor_rays + (int64_t)i * 3;
            dx = r[0]; dy = r[1]; dz = r[2];
          }
          floor_px(p, es, dx, dy, dz, d, c);
        }
        s_depth[i] = d;
        s_col[3 * i + 0] = (uint8_t)c;
        s_col[3 * i + 1] = (uint8_t)(c >> 8);
        s_col[3 * i + 2] = (uint8_t)(c >> 16);
      }
    }
    __syncthreads();
    if (warp == 0) {  // live-triangle prefix per 32-triangle word
      int carry = 0;
      for (int w0 = 0; w0 < p.tri_words; w0 += 32) {
        const int w = w0 + lane;
        const int cnt = w < p.tri_words ? __popc(s_live[w]) : 0;
        const int incl = warp_incl_scan(cnt, lane);
        if (w < p.tri_words) s_livepfx[w] = carry + incl - cnt;
        carry += __shfl_sync(kFull, incl, 31);
      }
      if (lane == 0) es.n_live = carry;
    }
    __syncthreads();
    const int n_live = es.n_live;

    // ---- raster rounds over live triangles in index order --------------
    for (int r0 = 0; r0 < n_live; r0 += p.cap) {
      if (r0 > 0) {
        for (int i = tid; i < n_bits_words; i += kThreads) s_bits[i] = 0u;
        for (int i = tid; i < p.n_tiles; i += kThreads) s_tilecnt[i] = 0u;
        if (tid == 0) es.queue_next = 0;
        __syncthreads();
      }
      // phase 2b: records + tile binning (render.py:366-436)
      for (int t = tid; t < p.nt; t += kThreads) {
        const uint32_t lw = s_live[t >> 5];
        if (!((lw >> (t & 31)) & 1u)) continue;
        const int cidx = (int)s_livepfx[t >> 5] + __popc(lw & ((1u << (t & 31)) - 1u)) - r0;
        if (cidx < 0 || cidx >= p.cap) continue;
        int i0 = p.tris[3 * t + 0], i1 = p.tris[3 * t + 1], i2 = p.tris[3 * t + 2];
        const float2 a = s_vxy32[i0];
        float2 b = s_vxy32[i1], c = s_vxy32[i2];
        float area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
        // flat Lambert from the UNswapped world-space normal (render.py:405-423)
        const float *w0 = s_world + 3 * i0, *w1 = s_world + 3 * i1, *w2 = s_world + 3 * i2;
        const float e1x = w1[0] - w0[0], e1y = w1[1] - w0[1], e1z = w1[2] - w0[2];
        const float e2x = w2[0] - w0[0], e2y = w2[1] - w0[1], e2z = w2[2] - w0[2];
        const float nx = e1y * e2z - e1z * e2y;
        const float ny = e1z * e2x - e1x * e2z;
        const float nz = e1x * e2y - e1y * e2x;
        const float nn = sqrtf(nx * nx + ny * ny + nz * nz);
        const float nd32 = (nx * lx + ny * ly + nz * lz) / nn;
        const double ndotl = nd32 < 0.0f ? 0.0 : (double)nd32;
        const double shade = 0.35 + 0.65 * ndotl;
        uint32_t rgb = 0;
        for (int ch = 0; ch < 3; ch++) {
          double v = (double)p.tri_colors[3 * t + ch] * shade * 255.0;
          if (v > 255.0) v = 255.0;
          rgb |= ((uint32_t)v & 0xffu) << (8 * ch);
        }
        if (area2 < 0.0f) {  // swap v1 <-> v2 (render.py:381-385)
          const float2 tmp = b; b = c; c = tmp;
          const int ti = i1; i1 = i2; i2 = ti;
          area2 = -area2;
        }
        const float minx = fminf(a.x, fminf(b.x, c.x)), maxx = fmaxf(a.x, fmaxf(b.x, c.x));
        const float miny = fminf(a.y, fminf(b.y, c.y)), maxy = fmaxf(a.y, fmaxf(b.y, c.y));
        double bx0 = ceil((double)minx - 0.5), bx1 = floor((double)maxx - 0.5);
        double by0 = ceil((double)miny - 0.5), by1 = floor((double)maxy - 0.5);
        if (bx0 < 0.0) bx0 = 0.0;
        if (by0 < 0.0) by0 = 0.0;
        if (bx1 > (double)(p.W - 1)) bx1 = (double)(p.W - 1);
        if (by1 > (double)(p.H - 1)) by1 = (double)(p.H - 1);
        const float ax0 = b.x - a.x, ay0 = b.y - a.y;
        const float ax1 = c.x - b.x, ay1 = c.y - b.y;
        const float ax2 = a.x - c.x, ay2 = a.y - c.y;
        uint32_t fl = 0;
        if (ay0 < 0.0f || (ay0 == 0.0f && ax0 > 0.0f)) fl |= 1u;
        if (ay1 < 0.0f || (ay1 == 0.0f && ax1 > 0.0f)) fl |= 2u;
        if (ay2 < 0.0f || (ay2 == 0.0f && ax2 > 0.0f)) fl |= 4u;
        TriRec R;
        R.A0 = (double)ax0; R.B0 = (double)ay0;
        R.A1 = (double)ax1; R.B1 = (double)ay1;
        R.A2 = (double)ax2; R.B2 = (double)ay2;
        R.area = (double)area2;
        R.rcp = __drcp_rn(R.area);
        R.v0 = (uint16_t)i0; R.v1 = (uint16_t)i1; R.v2 = (uint16_t)i2;
        R.flags = (uint16_t)fl;
        R.rgb = rgb;
        const int ix0 = (int)bx0, ix1 = (int)bx1, iy0 = (int)by0, iy1 = (int)by1;
        R.px0 = (int16_t)ix0; R.px1 = (int16_t)ix1; R.py0 = (int16_t)iy0; R.py1 = (int16_t)iy1;
        R.pad = 0;
        s_rec[cidx] = R;
        const uint32_t bit = 1u << (cidx & 31);
        const int word = cidx >> 5;
        for (int ty = iy0 / kTile; ty <= iy1 / kTile; ty++)
          for (int tx = ix0 / kTile; tx <= ix1 / kTile; tx++) {
            const int tile = ty * p.tiles_x + tx;
            atomicOr(&s_bits[tile * p.words + word], bit);
            atomicAdd(&s_tilecnt[tile], 1u);
          }
      }
      __syncthreads();
      // tile queue: non-empty tiles, heaviest first (longest-processing-time)
      if (p.n_tiles <= 512) {
        for (int i = tid; i < p.n_tiles; i += kThreads) {
          const uint32_t ci = s_tilecnt[i];
          if (ci == 0) continue;
          int rank = 0;
          for (int j = 0; j < p.n_tiles; j++) {
            const uint32_t cj = s_tilecnt[j];
            rank += (cj > ci) || (cj == ci && j < i);
          }
          s_queue[rank] = (uint16_t)i;
        }
        if (warp == 0) {
          int ne = 0;
          for (int i = lane; i < p.n_tiles; i += 32) ne += s_tilecnt[i] != 0u;
          for (int s = 16; s >= 1; s >>= 1) ne += __shfl_xor_sync(kFull, ne, s);
          if (lane == 0) es.n_queue = ne;
        }
      } else {  // large frames: plain compaction of the non-empty tiles
        if (tid == 0) es.n_queue = 0;
        __syncthreads();
        for (int i = tid; i < p.n_tiles; i += kThreads)
          if (s_tilecnt[i] != 0u) s_queue[atomicAdd(&es.n_queue, 1)] = (uint16_t)i;
      }
      __syncthreads();

      // phase 3: raster. A warp owns a tile; 32 triangles (one bitmask word)
      // per batch, their bbox-in-tile pixels flat-packed over the lanes.
      const int n_queue = es.n_queue;
      while (true) {
        int qi = 0;
        if (lane == 0) qi = atomicAdd(&es.queue_next, 1);
        qi = __shfl_sync(kFull, qi, 0);
        if (qi >= n_queue) break;
        const int tile = s_queue[qi];
        const int ty = tile / p.tiles_x, tx = tile - ty * p.tiles_x;
        const int xb = tx * kTile, yb = ty * kTile;
        const uint32_t *tb = s_bits + tile * p.words;
        for (int w = 0; w < p.words; w++) {
          const uint32_t m = tb[w];
          if (m == 0u) continue;
          int n = 0;
          uint32_t pk = 0;
          if ((m >> lane) & 1u) {
            const TriRec &R = s_rec[w * 32 + lane];
            const int cx0 = max((int)R.px0, xb), cx1 = min((int)R.px1, xb + kTile - 1);
            const int cy0 = max((int)R.py0, yb), cy1 = min((int)R.py1, yb + kTile - 1);
            const int bw = cx1 - cx0 + 1, bh = cy1 - cy0 + 1;
            if (bw > 0 && bh > 0) {
              n = bw * bh;
              pk = (uint32_t)(cx0 - xb) | ((uint32_t)(cy0 - yb) << 3) | ((uint32_t)bw << 6) |
                   (s_magic[bw] << 16);
            }
          }
          const int incl = warp_incl_scan(n, lane);
          const int excl = incl - n;
          const int N = __shfl_sync(kFull, incl, 31);
          for (int c0 = 0; c0 < N; c0 += 32) {
            const int c = c0 + lane;
            // owner lane: #lanes whose inclusive end <= c (branch-free search)
            int j = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
              const int v = __shfl_sync(kFull, incl, j + s - 1);
              if (v <= c) j += s;
            }
            const int ex = __shfl_sync(kFull, excl, j);
            const uint32_t opk = __shfl_sync(kFull, pk, j);
            bool cov = false;
            double zpix = 0.0;
            uint32_t rgb = 0;
            int pix = 0;
            if (c < N) {
              const int local = c - ex;
              const int bw = (opk >> 6) & 15;
              const int q = (int)(((uint32_t)local * (opk >> 16)) >> 16);
              const int px = xb + (int)(opk & 7u) + (local - q * bw);
              const int py = yb + (int)((opk >> 3) & 7u) + q;
              pix = py * p.W + px;
              const TriRec &R = s_rec[w * 32 + j];
              const double2 p0 = s_vxy64[R.v0], p1 = s_vxy64[R.v1], p2 = s_vxy64[R.v2];
              const double pcx = half_plus(px), pcy = half_plus(py);
              // render.py:441-446, inclusive top-left rule
              const double e0 = R.A0 * (pcy - p0.y) - R.B0 * (pcx - p0.x);
              const double e1 = R.A1 * (pcy - p1.y) - R.B1 * (pcx - p1.x);
              const double e2 = R.A2 * (pcy - p2.y) - R.B2 * (pcx - p2.x);
              const uint32_t fl = R.flags;
              if ((e0 > 0.0 || (e0 == 0.0 && (fl & 1u))) && (e1 > 0.0 || (e1 == 0.0 && (fl & 2u))) &&
                  (e2 > 0.0 || (e2 == 0.0 && (fl & 4u)))) {
                // render.py:447-451
                const double l0 = div_rn_pre(e1, R.area, R.rcp);
                const double l1 = div_rn_pre(e2, R.area, R.rcp);
                const double l2 = div_rn_pre(e0, R.area, R.rcp);
                const double inv_z = l0 * s_viz[R.v0] + l1 * s_viz[R.v1] + l2 * s_viz[R.v2];
                zpix = __drcp_rn(inv_z);
                rgb = R.rgb;
                cov = true;
              }
            }
            // apply fragments in triangle order (lane order) per pixel
            const uint32_t cm = __ballot_sync(kFull, cov);
            if (cm == 0u) continue;
            const uint32_t grp = __match_any_sync(kFull, cov ? pix : -1 - lane);
            const int rank = __popc(grp & lanemask_lt);
            const int rounds = __reduce_max_sync(kFull, cov ? rank : 0);
            for (int rr = 0; rr <= rounds; rr++) {
              if (cov && rank == rr && zpix < (double)s_depth[pix]) {  // strict (render.py:452)
                s_depth[pix] = (float)zpix;
                s_col[3 * pix + 0] = (uint8_t)rgb;
                s_col[3 * pix + 1] = (uint8_t)(rgb >> 8);
                s_col[3 * pix + 2] = (uint8_t)(rgb >> 16);
              }
              __syncwarp();
            }
          }
        }
      }
      __syncthreads();
    }

    // ---- phase 4: composite + postprocess (distractor.py:140-176, env.py:168-173)
    if (p.mode == PXR_MODE_VIDEO && p.vframe_bulk) mbar_wait_parity(&es.vbar, vphase);
    const uint8_t *vsrc = p.mode == PXR_MODE_VIDEO
                              ? (p.vframe_bulk ? s_vframe
                                               : p.frames + es.frame_idx * p.vframe_bytes)
                              : nullptr;
    for (int i = tid; i < npx; i += kThreads) {
      const float d = s_depth[i];
      int r = s_col[3 * i + 0], gg = s_col[3 * i + 1], b = s_col[3 * i + 2];
      if (p.mode == PXR_MODE_VIDEO) {
        if (isinf(d)) {
          const int y = i / p.W, x = i - y * p.W;
          const uint8_t *src = vsrc + ((int)s_rowmap[y] * p.Wv + (int)s_colmap[x]) * 3;
          r = src[0];
          gg = src[1];
          b = src[2];
        }
      } else if (p.mode == PXR_MODE_COLOR) {
        r = min(255, max(0, r + es.bias[0]));
        gg = min(255, max(0, gg + es.bias[1]));
        b = min(255, max(0, b + es.bias[2]));
      }
      if (p.gray) {
        s_gray[i] = (uint8_t)((299u * r + 587u * gg + 114u * b + 500u) / 1000u);
      } else {
        s_col[3 * i + 0] = (uint8_t)r;
        s_col[3 * i + 1] = (uint8_t)gg;
        s_col[3 * i + 2] = (uint8_t)b;
      }
      if (p.out_depth != nullptr) p.out_depth[(int64_t)env * npx + i] = d;
    }
    vphase ^= 1u;

    // ---- phase 5: frame -> HBM (one TMA bulk store) --------------------
    uint8_t *gout = p.out + (int64_t)env * p.frame_bytes;
    if (p.use_bulk) {
      fence_proxy_async_smem();
      __syncthreads();
      if (tid == 0) bulk_store_s2g(gout, s_out, (uint32_t)p.frame_bytes);
    } else {
      __syncthreads();
      for (int i = tid; i < p.frame_bytes; i += kThreads) gout[i] = s_out[i];
      __syncthreads();
    }
  }
  if (tid == 0 && p.use_bulk) bulk_wait_all();
}

// One thread per image row walks x exactly like render.py:321-344.
__global__ void floor_rays_kernel(float rx, float ry, float rz, float ux, float uy, float uz,
                                  float fx, float fy, float fz, float tanf_, int H, int W,
                                  double *out) {
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

// Exact-division self test (a[i] / b[i] vs div_rn_pre).
__global__ void div_check_kernel(const double *a, const double *b, double *q_pre,
                                 double *q_ieee, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double y = __drcp_rn(b[i]);
    q_pre[i] = div_rn_pre(a[i], b[i], y);
    q_ieee[i] = a[i] / b[i];
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

extern "C" pxr_status pxr_div_check(const double *a, const double *b, double *q_pre,
                                    double *q_ieee, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (!a || !b || !q_pre || !q_ieee))) return set_invalid("bad div args");
  if (n == 0) return PXR_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 65536) blocks = 65536;
  div_check_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(a, b, q_pre, q_ieee, n);
  return check_launch("div_check_kernel");
}

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
      cam[3], cam[4], cam[5], cam[6], cam[7], cam[8], cam[9], cam[10], cam[11], cam[12],
      (int)height, (int)width, out_rays);
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
  if (height > 1024 || width > 1024) return set_unsupported("frames above 1024 px per side");
  if (poses == nullptr || out_obs == nullptr) return set_invalid("null poses/out_obs");
  if (geom->n_links < 1 || geom->n_links > kMaxLinks || geom->n_verts < 0 || geom->n_tris < 0)
    return set_invalid("bad geometry sizes");
  if (geom->n_verts > 65535) return set_unsupported("more than 65535 vertices");
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
    p.vframe_bytes = p.Hv * p.Wv * 3;
    p.vframe_bulk = (p.vframe_bytes % 16 == 0) &&
                    ((reinterpret_cast<uintptr_t>(pack->frames) & 15) == 0);
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
  p.tiles_x = (p.W + kTile - 1) / kTile;
  p.tiles_y = (p.H + kTile - 1) / kTile;
  p.n_tiles = p.tiles_x * p.tiles_y;
  p.tri_words = (p.nt + 31) / 32;
  if (p.tri_words < 1) p.tri_words = 1;
  const int C = p.gray ? 1 : 3;
  p.frame_bytes = p.H * p.W * C;
  p.vec4 = (p.W % 4) == 0;
  p.use_bulk = (p.frame_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(out_obs) & 15) == 0);

  int dev = 0;
  cudaGetDevice(&dev);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int budget = max_optin - (int)sizeof(EnvShared) - 64 - 1024;
  // Live-triangle capacity per raster round: all triangles if they fit,
  // else the largest multiple of 32 that does (extra rounds handle overflow).
  int cap = align_up(p.nt > 0 ? p.nt : 32, 32);
  for (;;) {
    p.cap = cap;
    p.words = cap / 32;
    if (smem_layout(p).total <= budget || cap <= 32) break;
    cap -= 32;
  }
  const int smem = smem_layout(p).total;
  if (smem > budget) return set_unsupported("frame too large for one CTA's shared memory");
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

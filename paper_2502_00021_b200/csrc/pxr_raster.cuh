// Shared pieces of the two render kernels (pxr_render.cu: the one-CTA-per-env
// kernel; pxr_render_pipe.cu: the warp-specialised two-stage pipeline):
// launch parameters, per-triangle records, and the reference-exact device
// arithmetic (render.py:286-456, distractor.py:66-176), every function
// inline. See pxr_render.cu's header for the algorithm.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_math.cuh"

namespace pxr {

#ifndef PXR_RENDER_THREADS
#define PXR_RENDER_THREADS 768
#endif
constexpr int kThreads = PXR_RENDER_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLinks = 64;
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kRowCap = 2560;   // bbox rows (>= spans) per raster round (raised to H)
constexpr int kFragCap = 1536;  // fragment list capacity (overflow: recompute)
// debug workload counters per env: live triangles, bbox-row units, non-empty
// spans, candidate pixels, covered fragments, raster rounds, overflow rounds,
// live triangles that cover no pixel centre, their bbox-row units, those of
// them with a single bbox row
constexpr int kStats = 10;
#ifdef PXR_CHECKED
constexpr bool kWithStats = true;  // counters only in the checked build
#else
constexpr bool kWithStats = false;
#endif

constexpr uint32_t kSkyRGB = 135u | (206u << 8) | (235u << 16);  // render.py:50

// One live triangle of the current round (post-swap order, render.py:381-385):
// the exact-test data ...
// The f32 edge vectors and area are kept as f32: the reference converts them
// to f64 exactly (render.py:437-449), so (double) on use is the same value.
struct __align__(16) TriRec {
  float A0, B0, A1, B1, A2, B2;  // f32 edge vectors ax_k, ay_k
  float area;                    // area2
  uint32_t rgb;                  // flat-shaded u8 colour (render.py:404-423)
  double rcp;                    // RN(1 / (double)area2), for the exact division
  uint16_t v0, v1, v2, flags;    // vertex ids; top-left bits (render.py:431-433)
};
static_assert(sizeof(TriRec) == 48, "TriRec layout");

// ... and its conservative row-span data (see span_setup / row_span).
struct __align__(16) SpanRec {
  float ur[2], uc[2];  // upper x bounds fma(ur, y, uc) (margin folded into uc)
  float lr[2], lc[2];  // lower x bounds fma(lr, y, lc)
  float ylo, yhi;      // rows with ylo <= y <= yhi (horizontal edges; culled: empty)
  uint16_t py0, pad;
  uint32_t row0;       // first row unit of the triangle in the round
};
static_assert(sizeof(SpanRec) == 48, "SpanRec layout");
// Non-empty spans wait in a per-warp queue as uint2 {x0 | len << 16,
// row | live_tri << 16} until 32 can be evaluated together.
constexpr int kQueue = 64;

// A fragment of the paint list: pix | tri << 20 (pix < 2^20 and the live
// index of the round < 2^12 by the host's limits); depths are positive, so
// their f32 bit patterns order like the values.
constexpr int kMaxCap = 4095;

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
  int64_t n_videos, n_frames;
  int Hv, Wv;
  int advance;
  uint64_t key_hi, key_lo, env_offset, logical_batch;
  const uint64_t *device_key;  // key_t read on the device (graph replay), or null
  const uint8_t *done;
  int gray;
  uint8_t *out;
  float *out_depth;
  // derived on the host
  int cap;         // live-triangle records per raster round
  int row_cap;     // bbox rows per raster round
  int frag_limit;  // fragment list limit (kFragCap; test override)
  int frame_bytes, use_bulk, vframe_bytes, vframe_bulk;
  uint32_t wmagic;  // ceil(2^32 / W): flat pixel index -> row
  int depth_vec;    // out_depth groups of 4 pixels are 16-byte aligned
  int band_h;       // rows per band: a frame is rendered in bands that fit shared memory
  int32_t *stats;   // debug (tools/render_stats.py): per env kStats workload counters, or null
  int scan_sh;      // > 0: live count << scan_sh | bbox rows fits 32 bits (one packed scan)
  long long *prof;  // debug (tools/pipe_prof.py): per-CTA stage cycle counters of the pipeline
};

struct SmemLayout {
  int link, floor, maps, vxy64, viz, vxy32, vz, world, rows, ids, lrp, rec, span, rowner, queue,
      frag, depth, col, gray, gplan, vframe, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(const RenderParams &p) {
  SmemLayout L;
  int o = 0;
  const int npx = p.band_h * p.W;  // per-pixel arrays hold one band
  L.link = o;   o += align_up(2 * p.nl * 16, 16);  // double-buffered (prefetch)
  L.floor = o;  o += align_up((p.W + 3 * p.H) * 8 + p.H * 4, 16);  // rays + per-row t, parity
  L.maps = o;   o += align_up((p.W + p.H) * 4, 16);  // texel byte offsets per row / column
  L.vxy64 = o;  o += align_up(p.nv * 16, 16);
  L.viz = o;    o += align_up(p.nv * 8, 16);
  L.vxy32 = o;  o += align_up(p.nv * 8, 16);
  L.vz = o;     o += align_up(p.nv * 4, 16);
  L.world = o;  o += align_up(p.nv * 12, 16);
  L.rows = o;   o += align_up((p.nt + 1) * 2, 16);  // bbox rows per triangle (0 = dead)
  L.ids = o;    o += align_up((p.nt + 1) * 2, 16);  // live index -> triangle
  L.lrp = o;    o += align_up((p.nt + 1) * 4, 16);  // live index -> bbox-row prefix
  L.rec = o;    o += p.cap * (int)sizeof(TriRec);
  L.span = o;   o += align_up(p.cap * (int)sizeof(SpanRec), 16);
  L.rowner = o; o += align_up((p.row_cap / 32 + 2) * 2, 16);
  L.queue = o;  o += kWarps * kQueue * 8;
  L.frag = o;   o += kFragCap * 4;
  L.depth = o;  o += align_up(npx * 8, 16);  // the pixels' z words
  L.col = o;    o += align_up(npx * 3, 16);
  L.gray = o;   o += p.gray ? align_up(npx, 16) : 0;
  L.gplan = o;  o += p.mode == PXR_MODE_VIDEO ? align_up((p.W / 4 + 1) * 16, 16) : 0;
  // + 32 B: the byte-permute gather may read up to 20 B past the last texel
  L.vframe = o; o += p.mode == PXR_MODE_VIDEO ? align_up(p.vframe_bytes + 32, 16) : 0;
  L.total = o;
  return L;
}

struct DistSlot {
  int bias[3];
  int64_t frame_idx;
};

struct EnvShared {
  uint64_t vbar;  // mbarrier for the video frame bulk load
  int64_t frame_idx[2];  // [local_env & 1]: prepared one env ahead
  float ex[2], ez[2];
  int bias[2][3];
  int n_live;
  int round_end;
  int n_frag;
  int one_round;  // all live triangles of the band fit one raster round
  int plan_ok;
  int st[kStats];  // debug counters (p.stats)
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
  const uint64_t key_hi = p.device_key != nullptr ? __ldg(p.device_key) : p.key_hi;
  const uint64_t key_lo = p.device_key != nullptr ? __ldg(p.device_key + 1) : p.key_lo;
  if (p.mode == PXR_MODE_COLOR) {
    int16_t b3[3];
    if (p.advance) {
      uint64_t ehi, elo;
      threefry2x64(key_hi, key_lo, g, 2, ehi, elo);
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
        threefry2x64(key_hi, key_lo, p.logical_batch + g, 2, rhi, rlo);
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
    PXR_DCHECK(vid >= 0 && vid < p.n_videos);
    PXR_DCHECK(cur >= 0 && cur < p.counts[vid]);
    out.frame_idx = p.starts[vid] + cur;
    PXR_DCHECK(out.frame_idx >= 0 && out.frame_idx < p.n_frames);
  }
}

// Exact RN(a / b) from y = RN(1 / b): q = RN(a*y), r = a - b*q (exact with an
// FMA), q' = RN(q + r*y) (Markstein). Checked against IEEE division by
// tests/test_gpu_parity.py::TestDeviceMath::test_exact_division.
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

// Checker floor / sky for one pixel (render.py:306-344).
__device__ __forceinline__ void floor_px(const RenderParams &p, float ex, float ez, double dx,
                                         double dy, double dz, float &depth, uint32_t &rgb) {
  depth = __int_as_float(0x7f800000);
  rgb = kSkyRGB;
  if (dz < -1e-12) {
    const double t = (double)(-ez) / dz;
    if ((double)p.cam[13] <= t && t <= (double)p.cam[14]) {
      const double wx = (double)ex + t * dx;
      const double wy = (double)p.cam[1] + t * dy;
      const int64_t parity = (__double2ll_rd(wx) + __double2ll_rd(wy)) & 1;
      const uint32_t c = parity == 0 ? 158u : 122u;  // render.py:51-52
      rgb = c | (c << 8) | (c << 16);
      depth = (float)t;
    }
  }
}

// Clamped pixel range of a bbox side (render.py:390-403):
// int(ceil(mn - 0.5)) .. int(floor(mx - 0.5)), lower end clamped to 0 and
// upper end to lim (so lo > hi means empty). f64 in the reference; for
// |v| < 2^21 the f32 value v - 0.5 is exact, so f32 ceil/floor give the same
// integers without f64 conversions.
__device__ __forceinline__ void pixel_range(float mn, float mx, int lim, int &lo, int &hi) {
  if (fabsf(mn) < 0x1p21f && fabsf(mx) < 0x1p21f) {
    lo = (int)fmaxf(ceilf(mn - 0.5f), 0.0f);
    hi = (int)fminf(floorf(mx - 0.5f), (float)lim);
  } else {
    double a = ceil((double)mn - 0.5), b = floor((double)mx - 0.5);
    if (a < 0.0) a = 0.0;
    if (b > (double)lim) b = (double)lim;
    if (a > b) {  // empty; keep the integers in range
      lo = 1;
      hi = 0;
    } else {
      lo = (int)a;
      hi = (int)b;
    }
  }
}

// World-space vertex v (render.py:470-481): f32, no FMA contraction.
// Per-env inputs of the first phases, prepared by one warp one env ahead so
// the glibc-exact sincosf chains (render.py:613-614) and the Threefry chains
// overlap the previous env's rasterisation instead of stalling the CTA:
// link (x, z, cos, sin) into link_buf; camera position and the distractor
// bias / frame index into es[local_env & 1]. The distractor state of 32
// envs of this CTA is advanced at once, one lane each.
__device__ __forceinline__ void prepare_env(const RenderParams &p, int64_t env, int local_env,
                                         float4 *link_buf, DistSlot *s_dist, EnvShared &es,
                                         int lane) {
  for (int l = lane; l < p.nl; l += 32) {
    const double *pp = p.poses + (env * p.nl + l) * 3;
    const float th = (float)pp[2];  // poses.astype(float32), render.py:613
    link_buf[l] = make_float4((float)pp[0], (float)pp[1], glibc_sincosf(th, 1),
                              glibc_sincosf(th, 0));
  }
  if (local_env % 32 == 0) {
    const int64_t e2 = env + (int64_t)lane * gridDim.x;
    if (e2 < p.batch) distractor_update(p, e2, s_dist[lane]);
  }
  __syncwarp();
  if (lane == 0) {
    const int b = local_env & 1;
    const double *p0 = p.poses + env * p.nl * 3;
    es.ex[b] = (float)(p0[0] + p.off_x);  // render.py:611
    es.ez[b] = (float)(p0[1] + p.off_z);  // render.py:612
    const DistSlot &ds = s_dist[local_env % 32];
    es.bias[b][0] = ds.bias[0];
    es.bias[b][1] = ds.bias[1];
    es.bias[b][2] = ds.bias[2];
    es.frame_idx[b] = ds.frame_idx;
  }
  __syncwarp();
}

__device__ __forceinline__ float3 world_vertex(const RenderParams &p, const float4 *s_link, int v) {
  PXR_DCHECK(__ldg(p.vert_link + v) >= 0 && __ldg(p.vert_link + v) < p.nl);
  const float4 lk = s_link[__ldg(p.vert_link + v)];
  const float bx = __ldg(p.base_verts + 3 * v + 0);
  const float by = __ldg(p.base_verts + 3 * v + 1);
  const float bz = __ldg(p.base_verts + 3 * v + 2);
  return make_float3(lk.x + bx * lk.z - bz * lk.w, by, lk.y + bx * lk.w + bz * lk.z);
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    const int u = __shfl_up_sync(kFull, v, s);
    if (lane >= s) v += u;
  }
  return v;
}

// Span setup of one triangle. (a, b, c) is the post-swap vertex order
// (area2 > 0): the reference covers a pixel centre (x, y) only if every
// edge function e_k = A_k (y - s_k.y) - B_k (x - s_k.x) is >= 0 in f64
// (render.py:441-446). For a row, edges with B_k > 0 bound x from above by
// s_k.x + (A_k / B_k)(y - s_k.y), edges with B_k < 0 from below; with
// B_k == 0 the f64 value RN(A_k DY) has the exact sign of A_k * dy (and
// RN32(pcy - s.y) the exact sign of pcy - s.y), so A_k * dy < 0 empties the
// row. A bound is evaluated in f32 as fma(r, y, s.x - r s.y); its error is a
// few ulps of |s.x| + |r| (|s.y| + |y|), and a pixel the f64 test accepts
// lies at most 2^-52 (|r DY| + |DX|) beyond the exact bound. The margin
// 2^-10 px + 2^-17 (|s.x| + |r| (|s.y| + H + 1)) covers both with a wide
// safety factor: every pixel the reference can cover lies in its row's span,
// and the exact f64 test then decides each span pixel.
__device__ __forceinline__ void span_setup(const float2 a, const float2 b, const float2 c,
                                           float ymax, SpanRec &S) {
  const float2 v[3] = {a, b, c};
  float ur0 = 0.0f, uc0 = 0.0f, ur1 = 0.0f, uc1 = 0.0f;
  float lr0 = 0.0f, lc0 = 0.0f, lr1 = 0.0f, lc1 = 0.0f;
  bool have_u = false, have_l = false;
  float ylo = -__int_as_float(0x7f800000), yhi = __int_as_float(0x7f800000);
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const float2 s = v[k], t = v[(k + 1) % 3];
    const float A = t.x - s.x, B = t.y - s.y;
    if (B == 0.0f) {
      // horizontal edge: only the sign of A * (y - s.y) matters, and the f32
      // comparison of y with s.y is exact
      if (A > 0.0f) ylo = s.y; else yhi = s.y;
    } else {
      // an x bound whose slope only feeds a conservative bound: __fdividef's
      // <= 2 ulp error moves the line by <= 2^-22 |r| (H + |s.y|), far
      // inside m; folding m into the intercept adds one rounding of
      // |c0 + m|, also far inside m
      const float r = __fdividef(A, B);
      const float c0 = __fmaf_rn(-r, s.y, s.x);
      const float m = 0x1p-10f + (fabsf(s.x) + fabsf(r) * (fabsf(s.y) + ymax)) * 0x1p-17f;
      if (B > 0.0f) {  // bounds x from above
        ur1 = r; uc1 = c0 + m;
        if (!have_u) { ur0 = r; uc0 = c0 + m; }
        have_u = true;
      } else {
        lr1 = r; lc1 = c0 - m;
        if (!have_l) { lr0 = r; lc0 = c0 - m; }
        have_l = true;
      }
    }
  }
  // (a non-degenerate triangle has at least one edge of each kind; a single
  // one is used twice)
  S.ur[0] = ur0; S.uc[0] = uc0; S.ur[1] = ur1; S.uc[1] = uc1;
  S.lr[0] = lr0; S.lc[0] = lc0; S.lr[1] = lr1; S.lc[1] = lc1;
  S.ylo = ylo;
  S.yhi = yhi;
}

// Conservative span of one bbox row, clamped to the frame: first pixel x0 and
// length (0 = empty). NaN bounds (overflowing slopes) are ignored by
// fminf/fmaxf, which only widens the span; the exact test decides each pixel.
__device__ __forceinline__ int row_span(const SpanRec &S, int py, float wlim, int &x0) {
  const float y = (float)py + 0.5f;
  const float hi = fminf(fminf(__fmaf_rn(S.ur[0], y, S.uc[0]), __fmaf_rn(S.ur[1], y, S.uc[1])),
                         wlim);
  const float lo = fmaxf(fmaxf(__fmaf_rn(S.lr[0], y, S.lc[0]), __fmaf_rn(S.lr[1], y, S.lc[1])),
                         0.5f);
  const float xa = ceilf(lo - 0.5f), xb = floorf(hi - 0.5f);
  x0 = (int)xa;
  return (y < S.ylo || y > S.yhi || xa > xb) ? 0 : (int)xb - (int)xa + 1;
}

// One candidate pixel of triangle R: the reference's exact coverage test and
// depth (render.py:437-451).
__device__ __forceinline__ bool eval_exact(const TriRec &R, int px, int py,
                                           const double2 *s_vxy64, const double *s_viz,
                                           double &z) {
  const double2 p0 = s_vxy64[R.v0], p1 = s_vxy64[R.v1], p2 = s_vxy64[R.v2];
  const double pcx = half_plus(px), pcy = half_plus(py);
  const double e0 = (double)R.A0 * (pcy - p0.y) - (double)R.B0 * (pcx - p0.x);
  const double e1 = (double)R.A1 * (pcy - p1.y) - (double)R.B1 * (pcx - p1.x);
  const double e2 = (double)R.A2 * (pcy - p2.y) - (double)R.B2 * (pcx - p2.x);
  const uint32_t fl = R.flags;
  if ((e0 > 0.0 || (e0 == 0.0 && (fl & 1u))) && (e1 > 0.0 || (e1 == 0.0 && (fl & 2u))) &&
      (e2 > 0.0 || (e2 == 0.0 && (fl & 4u)))) {
    const double area = (double)R.area;
    const double l0 = div_rn_pre(e1, area, R.rcp);
    const double l1 = div_rn_pre(e2, area, R.rcp);
    const double l2 = div_rn_pre(e0, area, R.rcp);
    const double inv_z = l0 * s_viz[R.v0] + l1 * s_viz[R.v1] + l2 * s_viz[R.v2];
    z = __drcp_rn(inv_z);
    return true;
  }
  return false;
}

// ---- the one-pass exact sequential z-test (see pxr_render.cu's header) ----
// A pixel's word: RN32(depth) bits << 32 | sub. Background: sub = kBgSub.
// Fragment of live triangle li (index order over the whole env):
// sub = 0x7FFFFFFF - li if z < RN32(z), else 0x80000001 + li.
constexpr uint32_t kBgSub = 0x80000000u;
constexpr unsigned long long kBgWordInf = (0x7f800000ull << 32) | kBgSub;

__device__ __forceinline__ unsigned long long bg_word(float depth) {
  return ((unsigned long long)__float_as_uint(depth) << 32) | kBgSub;
}

__device__ __forceinline__ unsigned long long frag_word(double z, uint32_t li) {
  const float zf = (float)z;
  return ((unsigned long long)__float_as_uint(zf) << 32) |
         (z < (double)zf ? 0x7FFFFFFFu - li : 0x80000001u + li);
}

// word = min(word, w) in shared memory; true if w lowered it
__device__ __forceinline__ bool zword_min(unsigned long long *word, unsigned long long w) {
  unsigned long long old = *word;
  while (w < old) {
    const unsigned long long prev = atomicCAS(word, old, w);
    if (prev == old) return true;
    old = prev;
  }
  return false;
}

// live index of the winning triangle, -1 = background
__device__ __forceinline__ int zword_winner(unsigned long long w) {
  const uint32_t sub = (uint32_t)w;
  if (sub == kBgSub) return -1;
  return sub < kBgSub ? (int)(0x7FFFFFFFu - sub) : (int)(sub - 0x80000001u);
}

__device__ __forceinline__ float zword_depth(unsigned long long w) {
  return __uint_as_float((uint32_t)(w >> 32));
}

__device__ __forceinline__ void put_rgb(uint8_t *col, uint32_t pix, uint32_t rgb) {
  col[3 * pix + 0] = (uint8_t)rgb;
  col[3 * pix + 1] = (uint8_t)(rgb >> 8);
  col[3 * pix + 2] = (uint8_t)(rgb >> 16);
}

// The warp-specialised pipeline (pxr_render_pipe.cu): launches it when the
// configuration fits its shared-memory layout, else leaves *launched false.
pxr_status render_pipe_launch(RenderParams p, const DeviceFacts &dev, int debug_cap,
                              int debug_row_cap, int64_t debug_grid, cudaStream_t st,
                              bool *launched);

}  // namespace pxr

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
// Design (B200-first). Persistent CTAs of 24 warps,
// one env per CTA iteration, every intermediate in shared memory, every
// phase a flat loop over the CTA:
//   0. the env's video frame is fetched into shared memory by a TMA bulk
//      copy (cp.async.bulk + mbarrier) -- for RGB video with the pack
//      upscaled to the frame size (pxr_pack_upscale) the upscaled frame is
//      copied straight into the colour buffer instead, after phase 1; its
//      per-link glibc-exact cosf/sinf and distractor state (32 envs at a
//      time, one lane per env) were prepared by one warp during the
//      previous env's rasterisation; the mesh's triangle indices sit in
//      shared memory for the whole launch;
//   1. world transform + projection of every vertex (f32 like the
//      reference; f64 copies and 1/z for the raster);
//   2. triangle liveness exactly as the reference culls (near/far, zero
//      area, empty pixel bbox); a block scan over the triangles in index
//      order gives live index + bbox-row prefix; the background (sky, floor,
//      video texel -- or, for the upscaled copy, only the empty z-buffer)
//      written as final colours (with the floor here, without it by the
//      warps phase 3 leaves idle);
//   3. per round of live triangles (one round whenever the records fit): a
//      record per triangle (edge vectors, exact reciprocal of the area, flat
//      colour, the degenerate-normal cull) plus f32 line equations for
//      conservative row spans; (triangle, bbox row) units in 32-row chunks
//      dealt to the warps: each lane computes one row's conservative span,
//      and a chunk's non-empty spans become (pixel, triangle) candidates in
//      a CTA-wide pool (single-pixel spans directly, longer ones through a
//      warp scan + owner search); after a barrier every thread takes pooled
//      candidates, so the f64 work is balanced over the CTA however the
//      triangles' rows fall on the warps; every candidate gets the
//      reference's exact f64 edge / barycentric / depth arithmetic;
//      covered fragments min-reduce their f32 depth per pixel
//      with a 32-bit shared-memory atomicMin and are appended to a fragment
//      list;
//   4. exact order-independent resolve of the reference's SEQUENTIAL strict
//      z-test (render.py:452, triangles in index order, f64 z compared with
//      the f32 z-buffer): with F = min over fragments of RN32(z) and
//      S = {fragments with RN32(z) == F}, the sequential winner is the
//      highest-index member of S with z < F if one exists, else -- if F is
//      below the starting depth -- the lowest-index member of S, else the
//      previous content. (D only decreases; the first member of S always
//      writes when F < d0; later members write iff z < F; nothing outside S
//      can.) One atomicMax over key = (z < F) ? 0x10000 + i : 0xFFFF - i
//      encodes both cases; bit 31 of the same word records F < d0. The
//      winners paint their final colour;
//   5. the frame (RGB or grayscale) leaves shared memory in one TMA bulk
//      store overlapped with the next env.
// Final colours: every pixel is written last either by the background (2) or
// by a winner's paint (4), and the distractor composite + grayscale
// (distractor.py:140-176, env.py:168-173) is a per-pixel function of that
// colour, so it is applied where the colour is written (emit) -- there is no
// separate composite pass.
// Compiled with -fmad=false: no FMA contraction, every f32/f64 operation
// rounds where numba's code does. The only FMAs are explicit
// (__fma_rn / __fmaf_rn): the glibc sinf/cosf restatement, the exact
// division below and the conservative span bounds (not compared bit-wise).
#include <cuda_runtime.h>

#include <algorithm>
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
constexpr uint32_t kDecBit = 0x80000000u;
// debug workload counters per env: live triangles, bbox-row units, non-empty
// spans, candidate pixels, covered fragments, raster rounds, overflow rounds,
// live triangles that cover no pixel centre, their bbox-row units, those of
// them with a single bbox row, bbox rows between each triangle's first and
// last non-empty conservative span
constexpr int kStats = 11;
// debug phase timer slots (p.prof, tools/phase_prof.py): thread 0's clock at
// each phase-ending barrier, accumulated per CTA
constexpr int kProfSlots = 12;
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
// Raster candidates wait in a CTA-wide pool as pix | live_tri << 20 (the
// footprint of the per-warp span queues it replaced; a full pool leaves the
// rest to the warp that drew them).
constexpr int kPoolCap = 3072;

// A covered fragment: uint2 {RN32(z) bits | (z < RN32(z)) << 31, pix | tri << 20}
// (depths are positive, so the f32 sign bit is free; pix < 2^20 and the
// live index of the round < 2^12 by the host's limits).
constexpr int kMaxCap = 4095;
// Small batches: an env is split over CTAs in bands of at least this many rows.
constexpr int kMinSplitRows = 12;

// Shared-memory offsets of one CTA (smem_layout).
struct SmemLayout {
  int link, floor, maps, vxy64, viz, vxy32, vz, world, tris, rows, ids, lrp, rec, span, rowner, pool,
      frag, depth, col, wkey, gray, gplan, vframe, total;
};

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
  // RGB video with the pack upscaled to the frame size: the env's upscaled
  // frame is TMA-copied into the colour buffer as its background
  const uint8_t *frames_hw;
  int hw;
  int tris_smem;  // > 0: the triangle indices (u16) are staged in shared memory once per CTA
  uint32_t wmagic;  // ceil(2^32 / W): flat pixel index -> row
  int depth_vec;    // out_depth groups of 4 pixels are 16-byte aligned
  int band_h;       // rows per band: a frame is rendered in bands that fit shared memory
  int32_t *stats;   // debug (tools/render_stats.py): per env kStats workload counters, or null
  int scan_sh;      // > 0: live count << scan_sh | bbox rows fits 32 bits (one packed scan)
  long long *prof;  // debug (tools/phase_prof.py): per-CTA phase cycles, or null
  // Small batches: `split` CTAs render one env, one row band each (no
  // cross-CTA communication: only launched when no band reads distractor
  // state another band writes); 1 = persistent CTAs, each a sequence of
  // whole envs.
  int split;
  int64_t env_stride;  // envs between a CTA's consecutive envs (= gridDim.x / split)
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
  L.tris = o;   o += p.tris_smem ? align_up(p.nt * 8, 16) : 0;  // u16 x 4 per triangle
  L.rows = o;   o += align_up((p.nt + 1) * 2, 16);  // bbox rows per triangle (0 = dead)
  L.ids = o;    o += align_up((p.nt + 1) * 2, 16);  // live index -> triangle
  L.lrp = o;    o += align_up((p.nt + 1) * 4, 16);  // live index -> bbox-row prefix
  L.rec = o;    o += p.cap * (int)sizeof(TriRec);
  L.span = o;   o += align_up(p.cap * (int)sizeof(SpanRec), 16);
  L.rowner = o; o += align_up((p.row_cap / 32 + 2) * 2, 16);
  L.pool = o;   o += kPoolCap * 4;  // the raster's candidate pool
  L.frag = o;   o += kFragCap * 8;
  L.depth = o;  o += align_up(npx * 4, 16);
  L.col = o;    o += align_up(npx * 3, 16);
  L.wkey = o;   o += align_up(npx * 4, 16);
  L.gray = o;   o += p.gray ? align_up(npx, 16) : 0;
  const bool gather = p.mode == PXR_MODE_VIDEO && !p.hw;  // texels gathered per pixel
  L.gplan = o;  o += gather ? align_up((p.W / 4 + 1) * 16, 16) : 0;
  // + 32 B: the byte-permute gather may read up to 20 B past the last texel
  L.vframe = o; o += gather ? align_up(p.vframe_bytes + 32, 16) : 0;
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
  int n_pool;  // raster candidates appended to s_pool (may exceed kPoolCap: the rest ran in place)
  int one_round;  // all live triangles of the band fit one raster round
  int plan_ok;
  int st[kStats];  // debug counters (p.stats)
  long long prof[kProfSlots];  // debug phase cycles (p.prof)
  long long prof_t;
  long long rmin, rmax;  // debug (libpxr_prof.so): raster phase A / B ends (last worker)
};

// Per-env distractor step (writes the new state back to HBM):
//   colour: advance_distractors, distractor.py:123-126 -- e = fold_in(key_t, g),
//           biases from draw blocks 0/1 of e (distractor.py:66-74);
//   video:  ping-pong cursor (distractor.py:128-136), then for envs being
//           reset the re-drawn video (env.py:226-244); frame index 204.
// With advance == 0 (make_env / observe) the stored state is used as is.
__device__ __forceinline__ void distractor_update(const RenderParams &p, int64_t env,
                                                  DistSlot &out, bool write) {
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
      if (write)  // (split env: band 0 only; the new bias does not read the old)
        for (int c = 0; c < 3; c++) p.color_bias[env * 3 + c] = b3[c];
    } else {
      for (int c = 0; c < 3; c++) b3[c] = p.color_bias[env * 3 + c];
    }
    for (int c = 0; c < 3; c++) out.bias[c] = b3[c];
  } else if (p.mode == PXR_MODE_VIDEO) {
    int64_t vid = p.video_index[env];
    int64_t cur = p.frame_cursor[env];
    if (p.advance) {  // (never split: the step reads the state it writes)
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
// integers without f64 conversions. For |v| >= 2^21 the f32 value keeps its
// sign and lies far outside [0, lim], which is all the clamped range depends
// on (a bound beyond either end clamps or empties the range exactly as the
// f64 one does; float -> int conversion saturates). Branch-free, so the x
// and y sides of a triangle overlap.
__device__ __forceinline__ void pixel_range(float mn, float mx, int lim, int &lo, int &hi) {
  lo = (int)fmaxf(ceilf(mn - 0.5f), 0.0f);
  hi = (int)fminf(floorf(mx - 0.5f), (float)lim);
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
                                         int lane, int64_t stride, bool write) {
#pragma unroll 1
  for (int l = lane; l < p.nl; l += 32) {
    const double *pp = p.poses + (env * p.nl + l) * 3;
    const float th = (float)pp[2];  // poses.astype(float32), render.py:613
    link_buf[l] = make_float4((float)pp[0], (float)pp[1], glibc_sincosf(th, 1),
                              glibc_sincosf(th, 0));
  }
  if (local_env % 32 == 0) {
    const int64_t e2 = env + (int64_t)lane * stride;
    if (e2 < p.batch) distractor_update(p, e2, s_dist[lane], write);
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

// Inclusive warp scan: shfl.up's own in-range predicate selects the add (no
// separate lane compare per step).
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int s = 1; s < 32; s <<= 1) {
    asm("{\n"
        ".reg .s32 u;\n"
        ".reg .pred p;\n"
        "shfl.sync.up.b32 u|p, %0, %1, 0, -1;\n"
        "@p add.s32 %0, %0, u;\n"
        "}\n"
        : "+r"(v)
        : "r"(s));
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
  const float inf = __int_as_float(0x7f800000);
  // unused slots bound nothing (x <= +inf, x >= -inf)
  float ur0 = 0.0f, uc0 = inf, ur1 = 0.0f, uc1 = inf;
  float lr0 = 0.0f, lc0 = -inf, lr1 = 0.0f, lc1 = -inf;
  bool have_u = false, have_l = false;
  float ylo = -inf, yhi = inf;
  // branch-free: every edge's line is computed and the selects keep the
  // ones its kind uses (the lanes of a warp hold triangles of every shape)
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const float2 s = v[k], t = v[(k + 1) % 3];
    const float A = t.x - s.x, B = t.y - s.y;
    // horizontal edge (B == 0): only the sign of A * (y - s.y) matters, and
    // the f32 comparison of y with s.y is exact
    const bool hz = B == 0.0f;
    ylo = hz && A > 0.0f ? s.y : ylo;
    yhi = hz && !(A > 0.0f) ? s.y : yhi;
    // an x bound whose slope only feeds a conservative bound: the <= 1 ulp
    // error of rcp.approx moves the line by <= 2^-22 |r| (H + |s.y|), far
    // inside m; folding m into the intercept adds one rounding of |c0 + m|,
    // also far inside m. A nearly horizontal edge (|r| >= 2^100, or r not
    // finite: B == 0 or subnormal) bounds nothing -- dropping a bound only
    // widens the span, and the exact test decides every span pixel.
    float rb;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rb) : "f"(B));
    const float r = A * rb;
    const bool ok = fabsf(r) < 0x1p100f;
    const bool up = B > 0.0f && ok, dn = B < 0.0f && ok;
    const float c0 = __fmaf_rn(-r, s.y, s.x);
    const float m = __fmaf_rn(__fmaf_rn(fabsf(r), fabsf(s.y) + ymax, fabsf(s.x)), 0x1p-17f, 0x1p-10f);
    const float cu = c0 + m, cl = c0 - m;
    ur0 = up && !have_u ? r : ur0;  // the first edge of a kind fills both slots,
    uc0 = up && !have_u ? cu : uc0;  // a second one the other
    ur1 = up ? r : ur1;
    uc1 = up ? cu : uc1;
    have_u = have_u || up;
    lr0 = dn && !have_l ? r : lr0;
    lc0 = dn && !have_l ? cl : lc0;
    lr1 = dn ? r : lr1;
    lc1 = dn ? cl : lc1;
    have_l = have_l || dn;
  }
  // (a single edge of a kind is used twice)
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

// Winner of a pixel after a round (see the file header), -1 = unchanged.
__device__ __forceinline__ int resolve_winner(uint32_t word) {
  const uint32_t key = word & ~kDecBit;
  if (key >= 0x10000u) return (int)(key - 0x10000u);
  if (key != 0u && (word & kDecBit)) return (int)(0xFFFFu - key);
  return -1;
}

__device__ __forceinline__ void put_rgb(uint8_t *col, uint32_t pix, uint32_t rgb) {
  col[3 * pix + 0] = (uint8_t)rgb;
  col[3 * pix + 1] = (uint8_t)(rgb >> 8);
  col[3 * pix + 2] = (uint8_t)(rgb >> 16);
}

// Phase timer (debug, libpxr_prof.so only: -DPXR_PHASE_PROF): thread 0 adds
// the cycles since its last mark to a slot. Compiled out of libpxr.so (its
// per-barrier pointer test cost ~7 instructions per warp and phase).
#ifdef PXR_PHASE_PROF
constexpr bool kPhaseProf = true;
#define PXR_PROF(slot)                                  \
  do {                                                  \
    if (p.prof != nullptr && tid == 0) {                \
      const long long now_ = clock64();                 \
      es.prof[slot] += now_ - es.prof_t;                \
      es.prof_t = now_;                                 \
    }                                                   \
  } while (0)
#else
constexpr bool kPhaseProf = false;
#define PXR_PROF(slot) \
  do {                 \
  } while (0)
#endif

// kBands = false: the whole frame is one band (y0 = 0, straight-line code).
// kFloor = draw_floor: the checker floor needs every thread for the
// background (f64 per pixel), without it the background is cheap enough for
// the warps the records phase leaves idle; each kernel compiles one path.
template <bool kBands, bool kFloor>
__global__ void __launch_bounds__(kThreads, 1)
render_step_kernel(const RenderParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ EnvShared es;
  __shared__ DistSlot s_dist[32];
  __shared__ int s_scan[2 * kWarps];
  const SmemLayout L = smem_layout(p);
#ifdef PXR_CHECKED
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    PXR_DCHECK((uint32_t)L.total <= dyn);
  }
#endif
  // Programmatic dependent launch: the next launch in the stream may be
  // scheduled now (its CTAs take SMs as this grid's CTAs exit), and this
  // grid waits here for the previous one to complete and flush -- every
  // global read below (poses, distractor state, geometry, floor rays) comes
  // after the wait, so the overlap is the launch latency and CTA start-up
  // only. Both are no-ops for a launch without the attribute.
  pdl_trigger();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  float4 *s_link = reinterpret_cast<float4 *>(smem + L.link);
  double *s_floor = reinterpret_cast<double *>(smem + L.floor);  // dx[W], dy[H], dz[H]
  double *s_ft = s_floor + p.W + 2 * p.H;                          // per-row floor t
  int *s_fk = reinterpret_cast<int *>(s_ft + p.H);                 // per-row parity / -1
  uint32_t *s_rowmap = reinterpret_cast<uint32_t *>(smem + L.maps);  // rowmap[y] * Wv * 3
  uint32_t *s_colmap = s_rowmap + p.H;                               // colmap[x] * 3
  double2 *s_vxy64 = reinterpret_cast<double2 *>(smem + L.vxy64);
  double *s_viz = reinterpret_cast<double *>(smem + L.viz);
  float2 *s_vxy32 = reinterpret_cast<float2 *>(smem + L.vxy32);
  float *s_vz = reinterpret_cast<float *>(smem + L.vz);
  float *s_world = reinterpret_cast<float *>(smem + L.world);
  uint2 *s_tris = reinterpret_cast<uint2 *>(smem + L.tris);  // (i0 | i1 << 16, i2)
  uint16_t *s_rows = reinterpret_cast<uint16_t *>(smem + L.rows);
  uint16_t *s_ids = reinterpret_cast<uint16_t *>(smem + L.ids);
  uint32_t *s_lrp = reinterpret_cast<uint32_t *>(smem + L.lrp);
  TriRec *s_rec = reinterpret_cast<TriRec *>(smem + L.rec);
  SpanRec *s_span = reinterpret_cast<SpanRec *>(smem + L.span);
  uint16_t *s_rowner = reinterpret_cast<uint16_t *>(smem + L.rowner);
  uint32_t *s_pool = reinterpret_cast<uint32_t *>(smem + L.pool);  // pix | live tri << 20
  uint2 *s_frag = reinterpret_cast<uint2 *>(smem + L.frag);
  float *s_depth = reinterpret_cast<float *>(smem + L.depth);
  uint32_t *s_dbits = reinterpret_cast<uint32_t *>(smem + L.depth);
  uint8_t *s_col = smem + L.col;
  uint32_t *s_wkey = reinterpret_cast<uint32_t *>(smem + L.wkey);
  uint8_t *s_gray = smem + L.gray;
  uint8_t *s_vframe = smem + L.vframe;
  uint4 *s_gplan = reinterpret_cast<uint4 *>(smem + L.gplan);
  uint8_t *s_out = p.gray ? s_gray : s_col;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int fpx = p.H * p.W;  // pixels per frame
  const int chans = p.gray ? 1 : 3;
  const float wlim = (float)p.W - 0.5f;  // last pixel centre
  const double aspect = (double)p.W / (double)p.H;  // render.py:303
  const float ey = p.cam[1];
  const float rx = p.cam[3], ry = p.cam[4], rz = p.cam[5];
  const float ux = p.cam[6], uy = p.cam[7], uz = p.cam[8];
  const float fx = p.cam[9], fy = p.cam[10], fz = p.cam[11];
  const float tanf_ = p.cam[12], near_ = p.cam[13], far_ = p.cam[14];
  const float lx = p.light[0], ly = p.light[1], lz = p.light[2];
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const uint32_t lanemask_le = 0xFFFFFFFFu >> (31 - lane);

  // ---- once per CTA: floor rays, NN maps, mbarrier; meanwhile the last
  // warp prepares the first env (its latency chain would otherwise open the
  // CTA's critical path: a whole launch at small batches) ------------------
  constexpr int kSetupThreads = kThreads - 32;  // every warp but the last
  // split env: this CTA renders band `band0` of env blockIdx.x / split
  const int band0 = kBands && p.split > 1 ? (int)(blockIdx.x % (unsigned)p.split) : 0;
  const int64_t env_first =
      kBands && p.split > 1 ? (int64_t)(blockIdx.x / (unsigned)p.split) : (int64_t)blockIdx.x;
  // envs between this CTA's consecutive envs (the grid without a split)
  const int64_t env_stride = kBands ? p.env_stride : (int64_t)gridDim.x;
  const bool dist_write = !kBands || band0 == 0;  // a split env's state: band 0 writes
  if (warp == kWarps - 1 && env_first < p.batch)
    prepare_env(p, env_first, 0, s_link, s_dist, es, lane, env_stride, dist_write);
  if (kFloor && p.floor_sep && warp < kWarps - 1) {
    for (int i = tid; i < p.W; i += kSetupThreads) s_floor[i] = p.floor_rays[(int64_t)i * 3];
    for (int i = tid; i < p.H; i += kSetupThreads) {
      s_floor[p.W + i] = p.floor_rays[(int64_t)i * p.W * 3 + 1];
      s_floor[p.W + p.H + i] = p.floor_rays[(int64_t)i * p.W * 3 + 2];
    }
  }
  if (p.tris_smem && warp < kWarps - 1)  // the mesh's triangles, staged once per CTA
    for (int t = tid; t < p.nt; t += kSetupThreads)
      s_tris[t] = make_uint2((uint32_t)__ldg(p.tris + 3 * t) | ((uint32_t)__ldg(p.tris + 3 * t + 1) << 16),
                             (uint32_t)__ldg(p.tris + 3 * t + 2));
  if (p.mode == PXR_MODE_VIDEO && warp < kWarps - 1) {  // nearest_map, distractor.py:179-181
    for (int i = tid; i < p.H; i += kSetupThreads)
      s_rowmap[i] = (uint32_t)(((int64_t)i * p.Hv) / p.H) * p.Wv * 3;
    for (int i = tid; i < p.W; i += kSetupThreads)
      s_colmap[i] = (uint32_t)(((int64_t)i * p.Wv) / p.W) * 3;
  }
  if (tid == 0) {
    mbar_init(&es.vbar, 1);
    fence_mbar_init();
    es.plan_ok = 0;
    for (int i = 0; i < kProfSlots; i++) es.prof[i] = 0;
    es.rmin = 0;
    es.rmax = 0;
    es.prof_t = kPhaseProf && p.prof != nullptr ? clock64() : 0;
  }
  __syncthreads();
  // Byte-permute plan of the NN video gather (distractor.py:172-176): with
  // W % 4 == 0 and 4-byte-aligned source rows, the 12 output bytes of a
  // 4-pixel group come from one 24-byte window of the source row, and each
  // output word from two consecutive source words -> 2 loads + one PRMT.
  const bool use_plan = p.mode == PXR_MODE_VIDEO && !p.hw && p.vframe_bulk && (p.W & 3) == 0 &&
                        ((p.Wv * 3) & 3) == 0;
  if (use_plan && warp < kWarps - 1) {
    int bad = 0;
    for (int gc = tid; gc < (p.W >> 2); gc += kSetupThreads) {
      const int x0 = gc * 4;
      const uint32_t base_word = s_colmap[x0] >> 2;
      uint4 pl;
      pl.x = base_word;
      uint32_t sel[3];
      for (int q = 0; q < 3; q++) {
        int r[4], rmin = 1 << 30;
        for (int bb = 0; bb < 4; bb++) {
          const int b = 4 * q + bb, k = b / 3, ch = b % 3;
          r[bb] = (int)(s_colmap[x0 + k] + ch) - (int)(base_word * 4);
          rmin = min(rmin, r[bb]);
        }
        const int a = rmin >> 2;
        uint32_t s = (uint32_t)a << 16;
        for (int bb = 0; bb < 4; bb++) {
          const int nib = r[bb] - 4 * a;
          if (nib < 0 || nib > 7 || a > 3) bad = 1;
          s |= (uint32_t)(nib & 7) << (4 * bb);
        }
        sel[q] = s;
      }
      pl.y = sel[0];
      pl.z = sel[1];
      pl.w = sel[2];
      s_gplan[gc] = pl;
    }
    if (bad) es.plan_ok = -1;
  }
  __syncthreads();
  const bool plan_ok = use_plan && es.plan_ok == 0;

  __syncthreads();
  PXR_PROF(0);  // once per CTA: setup + the first env's preparation

  // triangle t's vertex indices (shared memory, or L2 for meshes too large)
  auto load_tri = [&](int t, int &a, int &b, int &c) {
    if (p.tris_smem) {
      const uint2 w = s_tris[t];
      a = (int)(w.x & 0xffffu);
      b = (int)(w.x >> 16);
      c = (int)w.y;
    } else {
      a = __ldg(p.tris + 3 * t + 0);
      b = __ldg(p.tris + 3 * t + 1);
      c = __ldg(p.tris + 3 * t + 2);
    }
  };

  // liveness: each thread owns a contiguous block of triangles (index order)
  const int per = (p.nt + kThreads - 1) / kThreads;
  const int t0 = min(tid * per, p.nt), t1 = min(t0 + per, p.nt);

  // the (env-independent) base geometry of this thread's first vertex stays
  // in registers: no global-load latency at the start of every env
  int g_link = 0;
  float g_bx = 0.0f, g_by = 0.0f, g_bz = 0.0f;
  if (tid < p.nv) {
    g_link = __ldg(p.vert_link + tid);
    PXR_DCHECK(g_link >= 0 && g_link < p.nl);
    g_bx = __ldg(p.base_verts + 3 * tid + 0);
    g_by = __ldg(p.base_verts + 3 * tid + 1);
    g_bz = __ldg(p.base_verts + 3 * tid + 2);
  }

  // Phase 1 of local env lenv (render.py:468-481, 350-363): world transform +
  // projection of every vertex, and with a separable floor its per-row terms
  // (t = -ez / dz, parity of floor(wy); render.py:321-334) by the last
  // threads (those with no or one vertex). Reads the env's prepared link
  // trig / camera (parity lenv & 1).
  auto vertex_phase = [&](int lenv) {
    const float4 *s_lk = s_link + (lenv & 1) * p.nl;
    const float lex = es.ex[lenv & 1], lez = es.ez[lenv & 1];
    if (kFloor && p.floor_sep) {
      // separable floor rays: t = -ez / dz and floor(wy) depend on the row
      // only (render.py:321-334), computed once per row by the last threads
      // (those with no or one vertex below)
#pragma unroll 1
      for (int y = kThreads - 1 - tid; y < p.H; y += kThreads) {
        const double dy = s_floor[p.W + y], dz = s_floor[p.W + p.H + y];
        double t = 0.0;
        int k = -1;  // -1: sky; else parity of floor(wy)
        if (dz < -1e-12) {
          t = (double)(-lez) / dz;
          if ((double)p.cam[13] <= t && t <= (double)p.cam[14]) {
            const double wy = (double)p.cam[1] + t * dy;
            k = (int)(__double2ll_rd(wy) & 1);
          }
        }
        s_ft[y] = t;
        s_fk[y] = k;
      }
    }
    auto project = [&](int v, const float3 w) {
      s_world[3 * v + 0] = w.x;
      s_world[3 * v + 1] = w.y;
      s_world[3 * v + 2] = w.z;
      const float vx = w.x - lex, vy = w.y - ey, vz = w.z - lez;
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
    };
    if (tid < p.nv) {  // the thread's first vertex: geometry held in registers
      const float4 lk = s_lk[g_link];
      project(tid, make_float3(lk.x + g_bx * lk.z - g_bz * lk.w, g_by,
                               lk.y + g_bx * lk.w + g_bz * lk.z));
    }
    // (meshes of more than kThreads vertices; no strength-reduced induction
    // variables for the common single pass above)
#pragma unroll 1
    for (int v = tid + kThreads; v < p.nv; v += kThreads) project(v, world_vertex(p, s_lk, v));
  };

  uint32_t vphase = 0;
  int local_env = 0;
  for (int64_t env = env_first; env < p.batch; env += env_stride, local_env++) {
    // ---- phase 0: video fetch (the env's link trig, camera and distractor
    // state were prepared by warp kWarps-1 during the previous env) -------
    const int cb = local_env & 1;
    if (kWithStats && p.stats != nullptr && tid < kStats) es.st[tid] = 0;
    if (tid == 0 && p.mode == PXR_MODE_VIDEO && !p.hw && p.vframe_bulk) {
      PXR_DCHECK(es.frame_idx[cb] >= 0 && es.frame_idx[cb] < p.n_frames);
      mbar_arrive_expect_tx(&es.vbar, (uint32_t)p.vframe_bytes);
      bulk_load_g2s(s_vframe, p.frames + es.frame_idx[cb] * p.vframe_bytes,
                    (uint32_t)p.vframe_bytes, &es.vbar);
    }
    const float ex = es.ex[cb], ez = es.ez[cb];
    bool prepared = env + env_stride >= p.batch;  // nothing to prepare for a last env

    // the first liveness triangle's indices, loaded before the vertex phase
    // so their latency (L2: the geometry does not stay in the small L1 next
    // to 230 KB of shared memory) overlaps it
    int n0 = 0, n1 = 0, n2 = 0;  // indices of the next triangle, loaded one ahead
    if (t0 < t1) load_tri(t0, n0, n1, n2);

    // ---- phase 1: world transform + projection (render.py:468-481, 350-363)
    vertex_phase(local_env);
    // The previous env's TMA store must have finished reading the frame.
    if (tid == 0 && p.use_bulk) bulk_wait_read();
    __syncthreads();
    PXR_PROF(1);  // vertex transform + projection

    // ---- bands of rows: everything below runs once per band (one band
    // whenever the frame's per-pixel state fits shared memory) ------------
    const int band_h = kBands ? p.band_h : p.H;
    const int ystart = kBands ? band0 * band_h : 0;  // a split env: this CTA's band only
    int yb = ystart;
    do {  // (no loop at all for one band)
      const int y0 = kBands ? yb : 0;  // compile-time 0 for one band
      const int y1 = kBands ? min(y0 + band_h, p.H) : p.H;
      const int npx = (y1 - y0) * p.W;  // pixels of this band
      const uint8_t *vsrc = p.mode == PXR_MODE_VIDEO
                                ? (p.vframe_bulk ? s_vframe
                                                 : p.frames + es.frame_idx[cb] * p.vframe_bytes)
                                : nullptr;
      // colour distractor as a per-byte saturating add/sub on the packed RGB
      // word (__vaddus4 / __vsubus4 == clamp(v + b, 0, 255) for |b| <= 255)
      uint32_t bpos = 0u, bneg = 0u;
      if (p.mode == PXR_MODE_COLOR) {
        for (int ch = 0; ch < 3; ch++) {
          const int bc = es.bias[cb][ch];
          bpos |= (uint32_t)(bc > 0 ? bc : 0) << (8 * ch);
          bneg |= (uint32_t)(bc < 0 ? -bc : 0) << (8 * ch);
        }
      }
      // a pixel's final colour: colour distractor, then grayscale
      auto emit = [&](uint32_t pix, uint32_t rgb) {
        PXR_DCHECK(pix < (uint32_t)npx);
        if (p.mode == PXR_MODE_COLOR) rgb = __vsubus4(__vaddus4(rgb, bpos), bneg);
        if (p.gray)
          s_gray[pix] = (uint8_t)((299u * (rgb & 0xffu) + 587u * ((rgb >> 8) & 0xffu) +
                                   114u * ((rgb >> 16) & 0xffu) + 500u) / 1000u);
        else
          put_rgb(s_col, pix, rgb);
      };
      if (!kBands && p.hw && tid == 0) {
        // the env's video frame, upscaled to the frame size, straight into the
        // colour buffer (the previous store has read it: awaited before the
        // vertex barrier); every pixel the resolve does not paint keeps it
        // (distractor.py:172-176: covered pixels are painted, the rest keep
        // the texel)
        PXR_DCHECK(es.frame_idx[cb] >= 0 && es.frame_idx[cb] < p.n_frames);
        mbar_arrive_expect_tx(&es.vbar, (uint32_t)p.frame_bytes);
        bulk_load_g2s(s_col, p.frames_hw + es.frame_idx[cb] * p.frame_bytes,
                      (uint32_t)p.frame_bytes, &es.vbar);
      }
      if (kBands && y0 > ystart) {  // the previous band's TMA store must have finished reading
        if (tid == 0 && p.use_bulk) bulk_wait_read();
        __syncthreads();
      }

      // ---- phase 2: liveness (render.py:366-416) + background -------------
      // each thread's block of triangles (t0, t1) is contiguous, so its live
      // count and bbox-row total feed the block scan directly
      int my_live = 0, my_rows = 0;
      if (kBands && y0 > ystart && t0 < t1) load_tri(t0, n0, n1, n2);  // (first band: at the env's start)
#pragma unroll 1
      for (int t = t0; t < t1; t++) {
        uint32_t rows = 0;
        const int i0 = n0, i1 = n1, i2 = n2;
        if (t + 1 < t1) load_tri(t + 1, n0, n1, n2);
        PXR_DCHECK(i0 >= 0 && i0 < p.nv && i1 >= 0 && i1 < p.nv && i2 >= 0 && i2 < p.nv);
        PXR_DCHECK(rows <= 0xFFFFu);
        const float z0 = s_vz[i0], z1 = s_vz[i1], z2 = s_vz[i2];
        if (!(z0 < near_ || z1 < near_ || z2 < near_) && !(z0 > far_ && z1 > far_ && z2 > far_)) {
          const float2 a = s_vxy32[i0], b = s_vxy32[i1], c = s_vxy32[i2];
          const float area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
          if (area2 != 0.0f) {
            const float minx = fminf(a.x, fminf(b.x, c.x)), maxx = fmaxf(a.x, fmaxf(b.x, c.x));
            const float miny = fminf(a.y, fminf(b.y, c.y)), maxy = fmaxf(a.y, fmaxf(b.y, c.y));
            int bx0, bx1, by0, by1;
            pixel_range(minx, maxx, p.W - 1, bx0, bx1);
            pixel_range(miny, maxy, p.H - 1, by0, by1);
            by0 = max(by0, y0);  // this band's rows only
            by1 = min(by1, y1 - 1);
            // (the degenerate-normal cull, render.py:405-409, is applied by
            // the records phase, which computes the normal for the shading)
            if (!(bx0 > bx1 || by0 > by1)) rows = (uint32_t)(by1 - by0 + 1);
          }
        }
        s_rows[t] = (uint16_t)rows;
        my_live += rows != 0u;
        my_rows += (int)rows;
      }
      // background: sky / floor under an empty z-buffer (render.py:306-344),
      // written as FINAL colours: a pixel's colour is written last either here
      // or by the resolve's paint, and the distractor composite + grayscale
      // is a per-pixel function of that colour (distractor.py:140-176,
      // env.py:168-173) -- so it is applied at write time (emit) and there is
      // no separate composite pass. Video: inf pixels take the texel. Without
      // a floor (cheap texel / sky pixels) it is written by the warps the
      // records phase leaves idle (see below), else here by every thread:
      // threads first, first + stride, ...
      const bool vwait = y0 == ystart && p.mode == PXR_MODE_VIDEO && !p.hw && p.vframe_bulk;
      const uint32_t vpar = vphase;
      if (y0 == ystart) vphase ^= 1u;  // the env's video frame (one fetch for all bands)
      auto background = [&](int first, int stride) {
        if (!kBands && p.hw) {  // colours arrive by TMA: depth +inf, empty keys
          const float inf = __int_as_float(0x7f800000);
          for (int gi = first; gi < (npx >> 2); gi += stride) {
            reinterpret_cast<float4 *>(s_depth)[gi] = make_float4(inf, inf, inf, inf);
            reinterpret_cast<uint4 *>(s_wkey)[gi] = make_uint4(0u, 0u, 0u, 0u);
          }
          for (int i = ((npx >> 2) << 2) + first; i < npx; i += stride) {
            s_depth[i] = inf;
            s_wkey[i] = 0u;
          }
          return;
        }
        if (vwait) mbar_wait_parity(&es.vbar, vpar);
        if (p.mode == PXR_MODE_VIDEO && !kFloor && plan_ok && !p.gray) {
          // 4-pixel groups: three texel words through the byte-permute plan
          const float inf = __int_as_float(0x7f800000);
          const int n4 = npx >> 2;  // plan_ok: W % 4 == 0, no tail
          for (int gi = first; gi < n4; gi += stride) {
            const int i0 = gi << 2;
            const int yb = (int)__umulhi((uint32_t)i0, p.wmagic);
            const uint4 pl = s_gplan[(i0 - yb * p.W) >> 2];
            const uint32_t *src =
                reinterpret_cast<const uint32_t *>(s_vframe + s_rowmap[y0 + yb]) + pl.x;
            const uint32_t *w0 = src + (pl.y >> 16), *w1 = src + (pl.z >> 16),
                           *w2 = src + (pl.w >> 16);
            PXR_DCHECK(4u * (uint32_t)(w0 + 1 - reinterpret_cast<const uint32_t *>(s_vframe)) + 4u <=
                       (uint32_t)p.vframe_bytes + 32u);
            PXR_DCHECK(4u * (uint32_t)(w2 + 1 - reinterpret_cast<const uint32_t *>(s_vframe)) + 4u <=
                       (uint32_t)p.vframe_bytes + 32u);
            uint32_t *c3 = reinterpret_cast<uint32_t *>(s_col) + 3 * gi;
            c3[0] = __byte_perm(w0[0], w0[1], pl.y & 0xffffu);
            c3[1] = __byte_perm(w1[0], w1[1], pl.z & 0xffffu);
            c3[2] = __byte_perm(w2[0], w2[1], pl.w & 0xffffu);
            reinterpret_cast<float4 *>(s_depth)[gi] = make_float4(inf, inf, inf, inf);
            reinterpret_cast<uint4 *>(s_wkey)[gi] = make_uint4(0u, 0u, 0u, 0u);
          }
        } else if (kFloor && p.floor_sep && p.mode != PXR_MODE_VIDEO && (p.W & 3) == 0) {
          // separable floor: 4-pixel groups of one row (W % 4 == 0), the same
          // per-pixel arithmetic as the scalar loop below, 3 packed colour
          // words (or one word of 4 grey bytes) + one float4 depth + one uint4
          // key store per group
          const float inf = __int_as_float(0x7f800000);
          const int n4 = npx >> 2;
          // a background pixel is sky or one of the two checker greys: their
          // final colours (colour distractor, then grayscale: as in emit) are
          // computed once, each pixel selects one
          auto final_of = [&](uint32_t c) {
            if (p.mode == PXR_MODE_COLOR) c = __vsubus4(__vaddus4(c, bpos), bneg);
            if (p.gray)  // env.py:168-173
              c = (299u * (c & 0xffu) + 587u * ((c >> 8) & 0xffu) + 114u * ((c >> 16) & 0xffu) +
                   500u) / 1000u;
            return c;
          };
          const uint32_t f_sky = final_of(kSkyRGB), f_odd = final_of(122u * 0x010101u),
                         f_even = final_of(158u * 0x010101u);
          for (int gi = first; gi < n4; gi += stride) {
            const int i0 = gi << 2;
            const int yb = (int)__umulhi((uint32_t)i0, p.wmagic), x = i0 - yb * p.W;
            const int k = s_fk[y0 + yb];
            float4 d4 = make_float4(inf, inf, inf, inf);
            uint32_t c[4] = {f_sky, f_sky, f_sky, f_sky};
            if (k >= 0) {
              const double t = s_ft[y0 + yb];
              const float tf = (float)t;
              d4 = make_float4(tf, tf, tf, tf);
              const double2 fa = reinterpret_cast<const double2 *>(s_floor + x)[0];
              const double2 fb = reinterpret_cast<const double2 *>(s_floor + x)[1];
              const double fx[4] = {fa.x, fa.y, fb.x, fb.y};
#pragma unroll
              for (int j = 0; j < 4; j++) {
                const double wx = (double)ex + t * fx[j];
                c[j] = ((uint32_t)__double2ll_rd(wx) ^ (uint32_t)k) & 1u ? f_odd : f_even;
              }
            }
            if (p.gray) {
              reinterpret_cast<uint32_t *>(s_gray)[gi] = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
            } else {
              uint32_t *c3 = reinterpret_cast<uint32_t *>(s_col) + 3 * gi;
              c3[0] = c[0] | (c[1] << 24);
              c3[1] = (c[1] >> 8) | (c[2] << 16);
              c3[2] = (c[2] >> 16) | (c[3] << 8);
            }
            reinterpret_cast<float4 *>(s_depth)[gi] = d4;
            reinterpret_cast<uint4 *>(s_wkey)[gi] = make_uint4(0u, 0u, 0u, 0u);
          }
        } else {
          for (int i = first; i < npx; i += stride) {
            const int yb = (int)__umulhi((uint32_t)i, p.wmagic), x = i - yb * p.W;
            const int y = y0 + yb;
            float d = __int_as_float(0x7f800000);
            uint32_t c = kSkyRGB;
            if (kFloor && p.floor_sep) {
              const int k = s_fk[y];
              if (k >= 0) {  // same arithmetic as floor_px with the row terms hoisted
                const double t = s_ft[y];
                const double wx = (double)ex + t * s_floor[x];
                const uint32_t g = ((uint32_t)__double2ll_rd(wx) ^ (uint32_t)k) & 1u ? 122u : 158u;
                c = g | (g << 8) | (g << 16);
                d = (float)t;
              }
            } else if (kFloor) {
              const double *r = p.floor_rays + ((int64_t)y0 * p.W + i) * 3;
              floor_px(p, ex, ez, r[0], r[1], r[2], d, c);
            }
            if (p.mode == PXR_MODE_VIDEO && isinf(d)) {  // distractor.py:172-176
              PXR_DCHECK(s_rowmap[y] + s_colmap[x] + 3u <= (uint32_t)p.vframe_bytes);
              const uint8_t *t = vsrc + s_rowmap[y] + s_colmap[x];
              c = (uint32_t)t[0] | ((uint32_t)t[1] << 8) | ((uint32_t)t[2] << 16);
            }
            s_depth[i] = d;
            s_wkey[i] = 0u;
            emit((uint32_t)i, c);
          }
        }
      };
      if (kFloor) background(tid, kThreads);
      // block scan over triangles in index order: live ids, bbox-row prefix
      {
        int li;
        uint32_t racc;
        if (p.scan_sh > 0) {
          // both totals in one word (host bound: nt << scan_sh | nt * band_h
          // fits 32 bits): one scan instead of two
          const int sh = p.scan_sh;
          const uint32_t mine = ((uint32_t)my_live << sh) | (uint32_t)my_rows;
          const uint32_t w = (uint32_t)warp_incl_scan((int)mine, lane);
          if (lane == 31) s_scan[warp] = (int)w;
          __syncthreads();  // (also publishes s_rows and a floor background)
          // every warp scans the warp totals itself (no second barrier)
          const uint32_t v = lane < kWarps ? (uint32_t)s_scan[lane] : 0u;
          const uint32_t vi = (uint32_t)warp_incl_scan((int)v, lane);
          if (warp == 0 && lane == kWarps - 1) es.n_live = (int)(vi >> sh);
          const uint32_t pre = __shfl_sync(kFull, vi - v, warp) + w - mine;
          li = (int)(pre >> sh);
          racc = pre & ((1u << sh) - 1u);
        } else {
          const int wl = warp_incl_scan(my_live, lane);
          const int wr = warp_incl_scan(my_rows, lane);
          if (lane == 31) {
            s_scan[warp] = wl;
            s_scan[kWarps + warp] = wr;
          }
          __syncthreads();  // (also publishes s_rows and a floor background)
          // every warp scans the warp totals itself (no second barrier)
          const int v = lane < kWarps ? s_scan[lane] : 0;
          const int u = lane < kWarps ? s_scan[kWarps + lane] : 0;
          const int vi = warp_incl_scan(v, lane), ui = warp_incl_scan(u, lane);
          if (warp == 0 && lane == kWarps - 1) es.n_live = vi;
          li = __shfl_sync(kFull, vi - v, warp) + wl - my_live;
          racc = (uint32_t)(__shfl_sync(kFull, ui - u, warp) + wr - my_rows);
        }
#pragma unroll 1
        for (int t = t0; t < t1; t++) {  // (per-thread block: ceil(nt / kThreads) triangles)
          const int r = s_rows[t];
          if (r != 0) {
            PXR_DCHECK(li < p.nt);
            s_ids[li] = (uint16_t)t;
            s_lrp[li] = racc;
            li++;
            racc += (uint32_t)r;
          }
        }
        if (tid == kThreads - 1) {  // the last thread holds the totals
          s_lrp[li] = racc;
          // common case: every live triangle fits one round -> its bounds
          // are known here, no serial round setup below
          const int fast = li <= p.cap && racc <= (uint32_t)p.row_cap;
          es.one_round = fast;
          if (fast) {
            es.round_end = li;
            es.n_frag = 0;
            es.n_pool = 0;
          }
        }
      }
      __syncthreads();
      PXR_PROF(2);  // liveness + block scan (+ floor background)
      const int n_live = es.n_live;
      const bool one_round = es.one_round != 0;
      if (!kFloor && n_live == 0) {
        background(tid, kThreads);
        __syncthreads();  // (the depth output reads it)
      }

      // ---- phases 3/4: raster rounds over live triangles in index order ---
      for (int r0 = 0; r0 < n_live;) {
        if (!one_round) {  // serial round setup (records do not fit one round)
          if (tid == 0) {
            // live [r0, r1): at most cap triangles and row_cap bbox rows (a
            // single triangle always fits: row_cap >= H); when several rounds
            // are needed their triangle counts are balanced (a small last round
            // cannot fill the CTA)
            const int left = n_live - r0;
            const int n_rounds = (left + p.cap - 1) / p.cap;
            const int target = (left + n_rounds - 1) / n_rounds;
            int lo = r0 + 1, hi = min(r0 + target, n_live);
            const uint32_t base = s_lrp[r0];
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (s_lrp[mid] - base <= (uint32_t)p.row_cap) lo = mid; else hi = mid - 1;
            }
            es.round_end = lo;
            es.n_frag = 0;
            es.n_pool = 0;
          }
          __syncthreads();
        }
        const int r1 = es.round_end;
        const uint32_t rbase = s_lrp[r0];
        const int n_rows = (int)(s_lrp[r1] - rbase);
        const int n_round = r1 - r0;
        if (kWithStats && p.stats != nullptr && tid == 0) {
          es.st[0] += n_round;
          es.st[1] += n_rows;
          es.st[5] += 1;
        }
        PXR_DCHECK(r0 < r1 && r1 <= n_live && n_round <= p.cap);
        PXR_DCHECK(n_rows >= n_round && n_rows <= p.row_cap);
        // records (render.py:366-436), span line equations, row-chunk owners;
        // in the first round the warps without a record write the background
        // meanwhile (all threads after their records if fewer than 4 are free)
        const int rec_warps = min((n_round + 31) >> 5, kWarps);
        const bool bg_here = !kFloor && r0 == 0;
        const bool bg_split = bg_here && rec_warps <= kWarps - 4;
        for (int li = r0 + tid; li < r1; li += kThreads) {
          const int t = s_ids[li];
          // the flat colour's L2 loads first: issued after the sqrtf's slow-
          // path branch they stalled the shading below by a full L2 latency
          const float tc0 = __ldg(p.tri_colors + 3 * t + 0), tc1 = __ldg(p.tri_colors + 3 * t + 1),
                      tc2 = __ldg(p.tri_colors + 3 * t + 2);
          int i0, i1, i2;
          load_tri(t, i0, i1, i2);
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
          const float tcol[3] = {tc0, tc1, tc2};
#pragma unroll
          for (int ch = 0; ch < 3; ch++) {
            double v = (double)tcol[ch] * shade * 255.0;
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
          int bx0, bx1, by0, by1;
          pixel_range(minx, maxx, p.W - 1, bx0, bx1);
          pixel_range(miny, maxy, p.H - 1, by0, by1);
          by0 = max(by0, y0);
          by1 = min(by1, y1 - 1);
          const float ax0 = b.x - a.x, ay0 = b.y - a.y;
          const float ax1 = c.x - b.x, ay1 = c.y - b.y;
          const float ax2 = a.x - c.x, ay2 = a.y - c.y;
          uint32_t fl = 0;
          if (ay0 < 0.0f || (ay0 == 0.0f && ax0 > 0.0f)) fl |= 1u;
          if (ay1 < 0.0f || (ay1 == 0.0f && ax1 > 0.0f)) fl |= 2u;
          if (ay2 < 0.0f || (ay2 == 0.0f && ax2 > 0.0f)) fl |= 4u;
          TriRec R;
          R.A0 = ax0; R.B0 = ay0;
          R.A1 = ax1; R.B1 = ay1;
          R.A2 = ax2; R.B2 = ay2;
          R.area = area2;
          R.rgb = rgb;
          R.rcp = __drcp_rn((double)area2);
          R.v0 = (uint16_t)i0; R.v1 = (uint16_t)i1; R.v2 = (uint16_t)i2;
          R.flags = (uint16_t)fl;
          PXR_DCHECK(li - r0 < p.cap && i0 < p.nv && i1 < p.nv && i2 < p.nv);
          PXR_DCHECK(by0 <= by1 && bx0 <= bx1 && by1 < p.H && bx1 < p.W);
          PXR_DCHECK(s_lrp[li + 1] - s_lrp[li] == (uint32_t)(by1 - by0 + 1));
          s_rec[li - r0] = R;
          SpanRec S;
          span_setup(a, b, c, (float)(p.H + 1), S);
          const bool culled = (double)nn < 1e-20;  // degenerate normal (render.py:405-409)
          if (culled) S.ylo = __int_as_float(0x7f800000);  // every row span is empty
          S.py0 = (uint16_t)by0;
          S.pad = 0;
          if (kWithStats && p.stats != nullptr) {
            int f = -1, l = -1;
            for (int row = by0; row <= by1; row++) {
              int x0s;
              if (row_span(S, row, wlim, x0s) > 0) {
                if (f < 0) f = row;
                l = row;
              }
            }
            atomicAdd(&es.st[10], f < 0 ? 0 : l - f + 1);
          }
          const uint32_t u0 = s_lrp[li] - rbase;
          S.row0 = u0;
          s_span[li - r0] = S;
          const uint32_t u1 = u0 + (uint32_t)(by1 - by0 + 1);
          PXR_DCHECK(((u1 - 1) >> 5) < (uint32_t)(p.row_cap / 32 + 2));
          // (mostly 0 or 1 chunk starts: no unrolled remainder dispatch)
#pragma unroll 1
          for (uint32_t k = (u0 + 31) >> 5; k <= ((u1 - 1) >> 5); k++)
            s_rowner[k] = (uint16_t)(li - r0);
        }
        // (warps without records arrive here at once)
        if (bg_here && (!bg_split || warp >= rec_warps))
          background(bg_split ? tid - rec_warps * 32 : tid,
                     bg_split ? kThreads - rec_warps * 32 : kThreads);
        __syncthreads();
        PXR_PROF(3);  // records + span equations (+ video / sky background)

        // (triangle, bbox row) units, 32 per chunk, chunks dealt round-robin
        // to the warps: each lane computes one row's conservative span, and
        // the chunk's non-empty spans become (pixel, live triangle)
        // candidates in a CTA-wide pool (single-pixel spans directly, longer
        // ones through a warp scan + owner search); after a barrier every
        // thread runs the exact test on pooled candidates. Most rows of the
        // thin triangles hold no pixel centre, so the f64 work only sees real
        // candidates, and it is balanced over the CTA whatever the triangle
        // sizes (a large triangle's rows no longer keep one warp busy).
        const int n_chunks = (n_rows + 31) >> 5;
        // while warp kWarps-1 prepares the next env the chunks are dealt to
        // the other warps only (it would otherwise finish last)
        // (`prepared` is the same in every thread: the chunk dealing below
        // must be CTA-uniform, also in a second raster round)
        const bool preparing = !prepared;
        const int n_workers = preparing ? kWarps - 1 : kWarps;
#ifdef PXR_PHASE_PROF
        const long long r_t0 = clock64();
#endif
        if (warp == kWarps - 1 && preparing) {
          prepare_env(p, env + env_stride, local_env + 1, s_link + (cb ^ 1) * p.nl, s_dist, es,
                      lane, env_stride, dist_write);
#ifdef PXR_PHASE_PROF
          if (p.prof != nullptr && lane == 0)  // slot 9: the next env's preparation
            atomicAdd(reinterpret_cast<unsigned long long *>(&es.prof[9]),
                      (unsigned long long)(clock64() - r_t0));
#endif
        }
        const bool prof_worker = !(warp == kWarps - 1 && preparing);
        (void)prof_worker;
        prepared = true;
        // a covered candidate: min-reduce its f32 depth into the pixel and
        // take a fragment-list slot (ptxas aggregates the warp's increments
        // into one shared atomic)
        auto add_fragment = [&](double z, uint32_t pix, int tri) {
          const int slot = atomicAdd(&es.n_frag, 1);
          const float zf = (float)z;
          const uint32_t zb = __float_as_uint(zf);
          if (zb < atomicMin(&s_dbits[pix], zb)) atomicOr(&s_wkey[pix], kDecBit);
          if (slot < p.frag_limit)
            s_frag[slot] = make_uint2(zb | (z < (double)zf ? 0x80000000u : 0u),
                                      pix | ((uint32_t)tri << 20));
        };
        if (warp < n_workers) {
          // Phase A: each chunk's 32 row spans are expanded (warp scan of
          // their lengths + owner search) into (pixel, live triangle)
          // candidates appended to the CTA-wide pool -- a large triangle's
          // pixels no longer stay with the warp that drew its rows.
          for (int k = warp; k < n_chunks; k += n_workers) {  // static round-robin
            const int u = k * 32 + lane;
            // owner triangle of unit u: the owner of the chunk's first unit plus
            // the triangles starting inside the chunk up to u (all have >= 1 row)
            const int o0 = s_rowner[k];
            const int mi = o0 + 1 + lane;
            uint32_t bit = 0;
            if (mi < n_round) {
              // (row0 of record mi, from the compact prefix: no bank conflicts)
              const int d = (int)(s_lrp[r0 + mi] - rbase) - k * 32;  // >= 1
              if (d < 32) bit = 1u << d;
            }
            const uint32_t starts = __reduce_or_sync(kFull, bit);
            const int j = o0 + __popc(starts & lanemask_le);
            PXR_DCHECK(u >= n_rows || (j < n_round && s_span[j].row0 <= (uint32_t)u &&
                                       (j + 1 >= n_round || s_span[j + 1].row0 > (uint32_t)u)));
            int len = 0, x0 = 0, row = 0;
            if (u < n_rows) {
              const SpanRec &S = s_span[j];
              row = (int)S.py0 + (u - (int)S.row0);
              len = row_span(S, row, wlim, x0);
              PXR_DCHECK(row >= y0 && row < y1);
              PXR_DCHECK(len == 0 || (x0 >= 0 && x0 + len <= p.W && len < 0x10000));
            }
            if (kWithStats && p.stats != nullptr) {  // (every lane takes part in the ballot)
              const int n_spans = __popc(__ballot_sync(kFull, len > 0));
              if (lane == 0) atomicAdd(&es.st[2], n_spans);
            }
            if (__all_sync(kFull, len <= 1)) {
              // every span is one pixel or empty (the common case): the
              // spans are the candidates, no expansion
              const uint32_t sm = __ballot_sync(kFull, len > 0);
              const int n = __popc(sm);
              if (kWithStats && p.stats != nullptr && lane == 0) atomicAdd(&es.st[3], n);
              int base = 0;
              if (lane == 0 && n > 0) base = smem_atomic_add(&es.n_pool, n);
              base = __shfl_sync(kFull, base, 0) + __popc(sm & lanemask_lt);
              if (len > 0) {
                const uint32_t pix = (uint32_t)((row - y0) * p.W + x0);
                PXR_DCHECK(pix < (uint32_t)npx && j < n_round);
                if (base < kPoolCap) {
                  s_pool[base] = pix | ((uint32_t)j << 20);
                } else {  // pool full: evaluated here
                  double z;
                  if (eval_exact(s_rec[j], x0, row, s_vxy64, s_viz, z)) add_fragment(z, pix, j);
                }
              }
              continue;
            }
            const int incl = warp_incl_scan(len, lane);
            const int excl = incl - len;
            const int NE = __shfl_sync(kFull, incl, 31);
            if (kWithStats && p.stats != nullptr && lane == 0) atomicAdd(&es.st[3], NE);
            // the chunk's pool slots, reserved at once (one atomic per chunk)
            int base = 0;
            if (lane == 0) base = smem_atomic_add(&es.n_pool, NE);
            base = __shfl_sync(kFull, base, 0);
#pragma unroll 1
            for (int c0 = 0; c0 < NE; c0 += 32) {
              // span lane of candidate c = c0 + lane: the number of lanes whose
              // inclusive end is <= c (branch-free binary search over the scan)
              const int c = c0 + lane;
              int owner = 0;
#pragma unroll
              for (int s = 16; s >= 1; s >>= 1) {
                const int v = __shfl_sync(kFull, incl, owner + s - 1);
                if (v <= c) owner += s;
              }
              const int o_ex = __shfl_sync(kFull, excl, owner & 31);
              const int o_x0 = __shfl_sync(kFull, x0, owner & 31);
              const int o_row = __shfl_sync(kFull, row, owner & 31);
              const int o_tri = __shfl_sync(kFull, j, owner & 31);
              if (c < NE) {
                const int px = o_x0 + (c - o_ex);
                const uint32_t pix = (uint32_t)((o_row - y0) * p.W + px);
                PXR_DCHECK(pix < (uint32_t)npx && o_tri < n_round && owner < 32);
                if (base + c < kPoolCap) {
                  s_pool[base + c] = pix | ((uint32_t)o_tri << 20);
                } else {  // pool full: evaluated here
                  double z;
                  if (eval_exact(s_rec[o_tri], px, o_row, s_vxy64, s_viz, z))
                    add_fragment(z, pix, o_tri);
                }
              }
            }
          }
#ifdef PXR_PHASE_PROF
          if (p.prof != nullptr && lane == 0) atomicMax(&es.rmin, clock64() - r_t0);  // phase A end
#endif
        }
        {
          // Phase B, every warp (the one that prepared the next env too): the
          // reference's exact f64 edge / barycentric / depth test on the
          // pooled candidates, one per thread
          __syncthreads();
          const int n_pool = min(es.n_pool, kPoolCap);
#pragma unroll 1
          for (int i = tid; i < n_pool; i += kThreads) {
            const uint32_t w = s_pool[i];
            const uint32_t pix = w & 0xFFFFFu;
            const int tri = (int)(w >> 20);
            const int yb = (int)__umulhi(pix, p.wmagic);
            const int px = (int)pix - yb * p.W;
            PXR_DCHECK(pix < (uint32_t)npx && tri < n_round);
            double z;
            if (eval_exact(s_rec[tri], px, y0 + yb, s_vxy64, s_viz, z)) add_fragment(z, pix, tri);
          }
        }
#ifdef PXR_PHASE_PROF
        if (p.prof != nullptr && lane == 0)  // slots 10 / 11: phase A / B ends
          atomicMax(&es.rmax, clock64() - r_t0);
#endif
        __syncthreads();
#ifdef PXR_PHASE_PROF
        if (p.prof != nullptr && tid == 0) {
          es.prof[10] += es.rmin;
          es.prof[11] += es.rmax;
          es.rmin = 0;
          es.rmax = 0;
        }
#endif
        PXR_PROF(4);  // row spans -> candidates -> exact test -> fragments
        // the upscaled video frame must have landed before the paint
        if (!kBands && p.hw && r0 == 0) mbar_wait_parity(&es.vbar, vpar);

        // exact sequential-order resolve (see the file header)
        const int n_frag = es.n_frag;
        if (kWithStats && p.stats != nullptr) {
          if (tid == 0) {
            es.st[4] += n_frag;
            es.st[6] += n_frag > p.frag_limit;
          }
          // triangles with at least one covered pixel: bit 15 of their flags
          // (only eval_exact reads the flags, and it has run)
          for (int i = tid; i < min(n_frag, p.frag_limit); i += kThreads)
            atomicOr(reinterpret_cast<uint32_t *>(&s_rec[s_frag[i].y >> 20]) + 11, 0x80000000u);
          __syncthreads();
          for (int li = tid; li < n_round; li += kThreads) {
            if (!(s_rec[li].flags & 0x8000u)) {
              const int rows = (int)(s_lrp[r0 + li + 1] - s_lrp[r0 + li]);
              atomicAdd(&es.st[7], 1);
              atomicAdd(&es.st[8], rows);
              if (rows == 1) atomicAdd(&es.st[9], 1);
            }
          }
          __syncthreads();
        }
        if (n_frag <= p.frag_limit) {
          // (at most kFragCap / kThreads = 2 iterations: not unrolled)
#pragma unroll 1
          for (int i = tid; i < n_frag; i += kThreads) {
            const uint2 f = s_frag[i];
            const uint32_t pix = f.y & 0xFFFFFu, tri = f.y >> 20;
            PXR_DCHECK(pix < (uint32_t)npx && tri < (uint32_t)n_round);
            if ((f.x & 0x7FFFFFFFu) == s_dbits[pix]) {  // in S: z < F == z < RN32(z)
              const uint32_t hb = s_wkey[pix] & kDecBit;  // stable after the barrier
              atomicMax(&s_wkey[pix], hb | ((f.x >> 31) ? 0x10000u + tri : 0xFFFFu - tri));
            }
          }
          __syncthreads();
          PXR_PROF(5);  // resolve pass
#pragma unroll 1
          for (int i = tid; i < n_frag; i += kThreads) {
            const uint32_t pix = s_frag[i].y & 0xFFFFFu, tri = s_frag[i].y >> 20;
            if (resolve_winner(s_wkey[pix]) == (int)tri) emit(pix, s_rec[tri].rgb);
          }
          if (r1 < n_live) {
            __syncthreads();
#pragma unroll 1
            for (int i = tid; i < n_frag; i += kThreads) s_wkey[s_frag[i].y & 0xFFFFFu] = 0u;
          }
        } else {
          // fragment list overflow: recompute the candidates for both passes
          for (int pass = 0; pass < 2; pass++) {
            for (int u = tid; u < n_rows; u += kThreads) {
              int j = s_rowner[u >> 5];
              PXR_DCHECK(j < n_round);
              while (j + 1 < n_round && s_span[j + 1].row0 <= (uint32_t)u) j++;
              const SpanRec &S = s_span[j];
              const TriRec &R = s_rec[j];
              const int row = (int)S.py0 + (u - (int)S.row0);
              int x0;
              const int len = row_span(S, row, wlim, x0);
              for (int px = x0; px < x0 + len; px++) {
                double z;
                if (!eval_exact(R, px, row, s_vxy64, s_viz, z)) continue;
                const uint32_t pix = (uint32_t)((row - y0) * p.W + px);
                PXR_DCHECK(pix < (uint32_t)npx);
                const uint32_t F = s_dbits[pix];
                if (__float_as_uint((float)z) != F) continue;
                if (pass == 0) {
                  const uint32_t hb = s_wkey[pix] & kDecBit;
                  atomicMax(&s_wkey[pix],
                            hb | (z < (double)__uint_as_float(F) ? 0x10000u + j : 0xFFFFu - j));
                } else if (resolve_winner(s_wkey[pix]) == j) {
                  emit(pix, R.rgb);
                }
              }
            }
            __syncthreads();
          }
          if (r1 < n_live)
            for (int i = tid; i < npx; i += kThreads) s_wkey[i] = 0u;
        }
        // the next round reuses records and keys; after the last one the
        // frame store's barrier orders the paint
        if (r1 < n_live) __syncthreads();
        r0 = r1;
      }
      if (warp == kWarps - 1 && !prepared)  // env without live triangles
        prepare_env(p, env + env_stride, local_env + 1, s_link + (cb ^ 1) * p.nl, s_dist, es, lane,
                    env_stride, dist_write);

      // ---- depth output (debug / _render_frame parity only) ---------------
      if (p.out_depth != nullptr) {
        float *dd = p.out_depth + (int64_t)env * fpx + (int64_t)y0 * p.W;
        if (p.depth_vec)
          for (int gi = tid; gi < (npx >> 2); gi += kThreads)
            reinterpret_cast<float4 *>(dd)[gi] = reinterpret_cast<const float4 *>(s_depth)[gi];
        for (int i = p.depth_vec ? ((npx >> 2) << 2) + tid : tid; i < npx; i += kThreads)
          dd[i] = s_depth[i];
      }

      // ---- phase 5: frame -> HBM (one TMA bulk store) --------------------
      if (kWithStats && p.stats != nullptr && tid < kStats && y0 + band_h >= p.H)
        p.stats[env * kStats + tid] = es.st[tid];  // (final: last band's resolve ran)
      uint8_t *gout = p.out + (int64_t)env * p.frame_bytes + (int64_t)y0 * p.W * chans;
      const int band_bytes = npx * chans;
      if (p.use_bulk) {  // host: every band's size and offset are multiples of 16
        // (no live triangle: the frame copy has not been awaited yet)
        if (!kBands && p.hw && n_live == 0 && tid == 0) mbar_wait_parity(&es.vbar, vpar);
        fence_proxy_async_smem();
        __syncthreads();
        PXR_PROF(6);  // paint (+ depth output)
        if (tid == 0) bulk_store_s2g(gout, s_out, (uint32_t)band_bytes);
      } else {
        __syncthreads();
        for (int i = tid; i < band_bytes; i += kThreads) gout[i] = s_out[i];
        __syncthreads();
      }
      yb += band_h;
    } while (kBands && p.split == 1 && yb < p.H);
  }
  // the last frame store must have read shared memory before the CTA exits
  // (its global writes complete with the grid)
  if (tid == 0 && p.use_bulk) bulk_wait_read();
  if (kPhaseProf && p.prof != nullptr) {
    PXR_PROF(7);  // the last store's shared-memory read
    if (tid == 0) es.prof[8] = local_env;
    __syncthreads();
    if (tid < kProfSlots) p.prof[blockIdx.x * kProfSlots + tid] = es.prof[tid];
  }
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
  if (poses == nullptr || out_obs == nullptr) return set_invalid("null poses/out_obs");
  if (geom->n_links < 1 || geom->n_links > kMaxLinks || geom->n_verts < 0 || geom->n_tris < 0)
    return set_invalid("bad geometry sizes");
  if (geom->n_verts > 65535 || geom->n_tris > 65535)
    return set_unsupported("more than 65535 vertices or triangles");
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
    p.n_frames = pack->n_frames;
    p.Hv = (int)pack->height;
    p.Wv = (int)pack->width;
    p.vframe_bytes = p.Hv * p.Wv * 3;
    p.frames_hw = pack->frames_hw;
    p.vframe_bulk = (p.vframe_bytes % 16 == 0) &&
                    ((reinterpret_cast<uintptr_t>(pack->frames) & 15) == 0);
  }
  p.advance = advance ? 1 : 0;
  if (keys != nullptr) {
    p.key_hi = keys->key_hi;
    p.key_lo = keys->key_lo;
    p.env_offset = keys->env_offset;
    p.logical_batch = keys->logical_batch;
    p.device_key = keys->device_key;
  }
  p.done = done;
  p.gray = grayscale ? 1 : 0;
  p.out = out_obs;
  p.out_depth = out_depth;
  const int C = p.gray ? 1 : 3;
  const int64_t npx64 = height * width;
  if (npx64 > (1 << 20) || height > 4096 || width > 4096)
    return set_unsupported("frame too large");
  p.wmagic = (uint32_t)((0x100000000ull + (uint64_t)width - 1) / (uint64_t)width);
  p.depth_vec = out_depth != nullptr && (npx64 % 4 == 0) &&
                ((reinterpret_cast<uintptr_t>(out_depth) & 15) == 0);
  p.frame_bytes = (int)(npx64 * C);
  p.use_bulk = (p.frame_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(out_obs) & 15) == 0);
  // Test hooks (tests/test_gpu_parity.py, pxr_set_debug): shrink the
  // per-round budgets so the multi-round and fragment-overflow paths run on
  // small inputs.
  // meshes up to 2048 triangles keep their indices in shared memory (16 KB)
  p.tris_smem = p.nt <= 2048 ? 1 : 0;
  p.frag_limit = kFragCap;
  p.row_cap = kRowCap > p.H ? kRowCap : p.H;
  {
    const int64_t v = debug_int(kDbgFragLimit, -1);
    if (v >= 0 && v < kFragCap) p.frag_limit = (int)v;
  }
  {
    const int64_t v = debug_int(kDbgRowCap, 0);
    if (v > 0) p.row_cap = v > p.H ? (int)v : p.H;
  }
  const int debug_cap = (int)debug_int(kDbgCap, 0);
  // debug: a device int32 (batch, kStats) buffer for per-env workload counters
  p.stats = (int32_t *)(uintptr_t)debug_int(kDbgStatsPtr, 0);
  const int debug_band = (int)debug_int(kDbgBandH, 0);
  // debug: at most this many CTAs, so small test batches run several envs
  // per CTA (the cross-env prefetch, double-buffered link table, video
  // mbarrier parity flip and TMA-store overlap)
  const int64_t debug_grid = debug_int(kDbgGrid, 0);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // debug: a device int64 (grid, 12) buffer for per-CTA phase cycles
  p.prof = (long long *)(uintptr_t)debug_int(kDbgProf, 0);

  const DeviceFacts &dev = device_facts();
  const int max_optin = dev.max_smem_optin;
  const int budget =
      max_optin - (int)(sizeof(EnvShared) + sizeof(DistSlot) * 32 + 8 * kWarps) - 256;
  // Live-triangle records per round: all triangles if they fit, else the
  // largest count that does (extra rounds handle the rest exactly).
  int cap = p.nt > 0 ? (p.nt < kMaxCap ? p.nt : kMaxCap) : 1;
  if (debug_cap > 0 && debug_cap < cap) cap = debug_cap;
  // Bands: the whole frame when its per-pixel state fits next to a useful
  // record capacity, else the tallest band that does; full bands are whole
  // multiples of 16 bytes so every band's TMA store stays legal.
  {
    const int min_cap = cap < 256 ? cap : 256;
    const int bytes_row = width * C;
    int m = 1;  // rows per 16-byte multiple
    while ((m * bytes_row) % 16 != 0 && m < 16) m *= 2;
    int bh = height;
    for (int nb = 1; nb <= height; nb++) {
      bh = (height + nb - 1) / nb;
      if (nb > 1 && bh > m) bh -= bh % m;
      p.band_h = bh;
      p.cap = min_cap;
      if (smem_layout(p).total <= budget) break;
    }
    if (debug_band > 0 && debug_band < bh) bh = debug_band;
    // Small batches (at most half as many envs as SMs): each env is split
    // over CTAs, one band of >= kMinSplitRows rows each, so the per-band
    // phases (records, raster, resolve, paint) run on several SMs at once.
    // No CTA communicates with another: only when no band reads distractor
    // state another band writes (video with advance reads and writes the
    // ping-pong cursor; the colour step re-draws the bias from the key and
    // band 0 alone writes it back).
    p.split = 1;
    if (bh == height && !(mode == PXR_MODE_VIDEO && advance) && debug_grid <= 0 &&
        debug_knob(kDbgNoSplit) == nullptr && batch * 2 <= dev.num_sms) {
      const int64_t want = std::min<int64_t>(dev.num_sms / batch, height / kMinSplitRows);
      if (want >= 2) {
        int sb = (int)((height + want - 1) / want);
        sb = (sb + m - 1) / m * m;  // whole 16-byte multiples
        if (sb < height) {
          bh = sb;
          p.split = (int)((height + sb - 1) / sb);
        }
      }
    }
    p.band_h = bh;
    if (bh < height && (bh * bytes_row) % 16 != 0) p.use_bulk = 0;
    if (bh < height && (bh * width) % 4 != 0) p.depth_vec = 0;
  }
  // RGB video without a drawn floor (the texel is the whole background), one
  // band, the pack upscaled to this frame size: the env's background is one
  // TMA copy of its upscaled frame (no texel gather, no raw-frame buffer in
  // shared memory)
  p.hw = 0;
  if (mode == PXR_MODE_VIDEO && !p.draw_floor && p.band_h == p.H && !p.gray && p.use_bulk &&
      pack->frames_hw != nullptr && pack->hw_height == height && pack->hw_width == width &&
      (reinterpret_cast<uintptr_t>(pack->frames_hw) & 15) == 0 &&
      debug_knob(kDbgNoUpscale) == nullptr)
    p.hw = 1;
  for (;;) {
    p.cap = cap;
    if (smem_layout(p).total <= budget || cap <= 16) break;
    cap = cap > 64 ? cap - 32 : cap - 8;
  }
  {  // packed block scan: bits for nt * band_h bbox rows + bits for nt live
    int rb = 0, lb = 0;
    while (rb < 32 && ((int64_t)1 << rb) <= (int64_t)p.nt * p.band_h) rb++;
    while (lb < 32 && ((int64_t)1 << lb) <= (int64_t)p.nt) lb++;
    p.scan_sh = (rb + lb <= 32 && rb < 32 && debug_knob(kDbgNoPackedScan) == nullptr) ? rb : 0;
  }
  const int smem = smem_layout(p).total;
  if (smem > budget) return set_unsupported("frame too large for one CTA's shared memory");
  const bool banded = p.band_h < p.H;
  auto kernel = banded ? (p.draw_floor ? render_step_kernel<true, true>
                                       : render_step_kernel<true, false>)
                       : (p.draw_floor ? render_step_kernel<false, true>
                                       : render_step_kernel<false, false>);
  int per_sm = 1;
  const pxr_status os = kernel_occupancy((const void *)kernel, kThreads, smem, &per_sm);
  if (os != PXR_OK) return os;
  int64_t grid = (int64_t)dev.num_sms * per_sm;
  if (debug_grid > 0 && debug_grid < grid) grid = debug_grid;
  if (grid > batch) grid = batch;
  if (p.split > 1) grid = batch * p.split;  // (<= the SM count, host rule above)
  p.env_stride = grid / p.split;
  if (debug_knob(kDbgNoPdl) != nullptr) {
    kernel<<<(unsigned)grid, kThreads, smem, st>>>(p);
    return check_launch("render_step_kernel");
  }
  // programmatic dependent launch (see the kernel's first lines): the launch
  // latency of back-to-back steps overlaps the previous step's tail
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t le = cudaLaunchKernelEx(&cfg, kernel, p);
  if (le != cudaSuccess) {
    (void)cudaGetLastError();
    return set_cuda(le, "render_step_kernel");
  }
  return check_launch("render_step_kernel");
}

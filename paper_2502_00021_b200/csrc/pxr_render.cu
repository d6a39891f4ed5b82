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
// Design (B200-first). Persistent CTAs of 16 warps,
// one env per CTA iteration, every intermediate in shared memory; every
// phase is a flat, balanced loop over the CTA (no per-warp ownership):
//   0. per-link glibc-exact cosf/sinf; distractor state for 32 envs at a
//      time (one lane per env); the env's video frame is fetched into shared
//      memory by a TMA bulk copy (cp.async.bulk + mbarrier);
//   1. world transform + projection of every vertex (f32 like the
//      reference; f64 copies and 1/z for the raster);
//   2. triangle liveness (cull, area, bbox, normal), a block scan over
//      triangles in index order -> live index + candidate offset; sky /
//      floor background and an empty z-buffer;
//   3. per round of live triangles (all of them at 84x84): records with f64
//      edge coefficients and the exact reciprocal of the area, then every
//      (triangle, bbox pixel) candidate of the round flat over the warps:
//      the reference's exact f64 edge / barycentric / depth arithmetic;
//      covered fragments min-reduce their f32 depth per pixel with a 32-bit
//      shared-memory atomicMin and are kept in a fragment list;
//   4. exact order-independent resolve of the reference's SEQUENTIAL strict
//      z-test (render.py:452, triangles in index order, f64 z compared with
//      the f32 z-buffer): with F = min over fragments of RN32(z) and
//      S = {fragments with RN32(z) == F}, the sequential winner is the
//      highest-index member of S with z < F if one exists, else -- if F is
//      below the starting depth -- the lowest-index member of S, else the
//      background. (D only decreases; the first member of S always writes
//      when F < d0; later members write iff z < F; nothing outside S can.)
//      One atomicMax over key = (z < F) ? 0x10000 + i : 0xFFFF - i encodes
//      both cases;
//   5. composite (video texel from shared memory or colour clamp-add,
//      grayscale) into a shared-memory frame stored with one TMA bulk copy
//      overlapped with the next env.
// Compiled with -fmad=false: no FMA contraction, every f32/f64 operation
// rounds where numba's code does. The only FMAs are the
// explicit __fma_rn of the glibc sinf/cosf restatement and of the exact
// division below.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_math.cuh"

namespace pxr {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLinks = 64;
constexpr uint32_t kFull = 0xffffffffu;
constexpr int kRoundCand = 8192;  // candidates per raster round (soft cap)
constexpr int kFragCap = 2048;    // fragment list capacity (overflow: recompute)

constexpr uint32_t kSkyRGB = 135u | (206u << 8) | (235u << 16);  // render.py:50

// One live triangle of the current round (post-swap order, render.py:381-385).
struct __align__(16) TriRec {
  double A0, B0, A1, B1, A2, B2;  // (double) of the f32 edge vectors ax_k, ay_k
  double rcp;                     // RN(1 / (double)area2), for the exact division
  double area;                    // (double)area2
  uint16_t v0, v1, v2, flags;     // vertex ids; top-left bits (render.py:431-433)
  uint32_t rgb;                   // flat-shaded u8 colour (render.py:404-423)
  uint32_t cand0;                 // first candidate of this triangle in the round
  uint16_t px0, py0, bw, bh;      // clamped pixel bbox (render.py:390-403)
  uint32_t magic;                 // ceil(2^32 / bw): candidate -> (row, col)
};
static_assert(sizeof(TriRec) == 96, "TriRec layout");

struct Frag {
  double z;      // f64 depth of the candidate (render.py:450-451)
  uint32_t pix;  // y * W + x
  uint32_t tri;  // live index within the round (== triangle order)
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
  int64_t n_videos;
  int Hv, Wv;
  int advance;
  uint64_t key_hi, key_lo, env_offset, logical_batch;
  const uint8_t *done;
  int gray;
  uint8_t *out;
  float *out_depth;
  // derived on the host
  int cap;        // live-triangle records per raster round
  int chunk_cap;  // chunk-owner entries (>= round candidates / 32)
  int round_cand; // candidate budget per round (kRoundCand; test override)
  int frag_limit; // fragment list limit (kFragCap; test override)
  int frame_bytes, use_bulk, vframe_bytes, vframe_bulk;
  uint32_t wmagic;  // ceil(2^32 / W): flat pixel index -> row
  int depth_vec;    // out_depth rows of 4 pixels are 16-byte aligned
};

struct SmemLayout {
  int link, floor, maps, vxy64, viz, vxy32, vz, world, cnt, ids, lcp, rec, cand0, owner, frag,
      depth, col, wkey, dec, gray, vframe, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(const RenderParams &p) {
  SmemLayout L;
  int o = 0;
  const int npx = p.H * p.W;
  L.link = o;   o += align_up(p.nl * 16, 16);
  L.floor = o;  o += align_up((p.W + 2 * p.H) * 8, 16);
  L.maps = o;   o += align_up((p.W + p.H) * 2, 16);
  L.vxy64 = o;  o += align_up(p.nv * 16, 16);
  L.viz = o;    o += align_up(p.nv * 8, 16);
  L.vxy32 = o;  o += align_up(p.nv * 8, 16);
  L.vz = o;     o += align_up(p.nv * 4, 16);
  L.world = o;  o += align_up(p.nv * 12, 16);
  L.cnt = o;    o += align_up((p.nt + 1) * 4, 16);  // bbox size per triangle
  L.ids = o;    o += align_up((p.nt + 1) * 2, 16);  // live index -> triangle
  L.lcp = o;    o += align_up((p.nt + 1) * 4, 16);  // live index -> candidate prefix
  L.rec = o;    o += p.cap * (int)sizeof(TriRec);
  L.cand0 = o;  o += align_up((p.cap + 33) * 4, 16);  // first candidate per record
  L.owner = o;  o += align_up(p.chunk_cap * 2, 16);
  L.frag = o;   o += kFragCap * (int)sizeof(Frag);
  L.depth = o;  o += align_up(npx * 4, 16);
  L.col = o;    o += align_up(npx * 3, 16);
  L.wkey = o;   o += align_up(npx * 4, 16);
  L.dec = o;    o += align_up(npx, 16);
  L.gray = o;   o += p.gray ? align_up(npx, 16) : 0;
  L.vframe = o; o += p.mode == PXR_MODE_VIDEO ? align_up(p.vframe_bytes, 16) : 0;
  L.total = o;
  return L;
}

struct DistSlot {
  int bias[3];
  int64_t frame_idx;
};

struct EnvShared {
  uint64_t vbar;  // mbarrier for the video frame bulk load
  float ex, ez;
  int bias[3];
  int64_t frame_idx;
  int n_live;
  int round_end;
  int n_cand;
  int chunk_next;
  int overflow;
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
      const int64_t parity = ((int64_t)floor(wx) + (int64_t)floor(wy)) & 1;
      const uint32_t c = parity == 0 ? 158u : 122u;  // render.py:51-52
      rgb = c | (c << 8) | (c << 16);
      depth = (float)t;
    }
  }
}

// World-space vertex v (render.py:470-481): f32, no FMA contraction.
__device__ __forceinline__ float3 world_vertex(const RenderParams &p, const float4 *s_link, int v) {
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

// One candidate (triangle R, its local-th bbox pixel): the reference's exact
// coverage test and depth (render.py:437-451).
__device__ __forceinline__ bool eval_candidate(const RenderParams &p, const TriRec &R, int local,
                                               const double2 *s_vxy64, const double *s_viz,
                                               uint32_t &pix, double &z) {
  // magic == 0 encodes bw == 1 (2^32 does not fit in 32 bits)
  const int q = R.magic == 0u ? local : (int)__umulhi((uint32_t)local, R.magic);
  const int px = (int)R.px0 + (local - q * (int)R.bw);
  const int py = (int)R.py0 + q;
  pix = (uint32_t)(py * p.W + px);
  const double2 p0 = s_vxy64[R.v0], p1 = s_vxy64[R.v1], p2 = s_vxy64[R.v2];
  const double pcx = half_plus(px), pcy = half_plus(py);
  const double e0 = R.A0 * (pcy - p0.y) - R.B0 * (pcx - p0.x);
  const double e1 = R.A1 * (pcy - p1.y) - R.B1 * (pcx - p1.x);
  const double e2 = R.A2 * (pcy - p2.y) - R.B2 * (pcx - p2.x);
  const uint32_t fl = R.flags;
  if ((e0 > 0.0 || (e0 == 0.0 && (fl & 1u))) && (e1 > 0.0 || (e1 == 0.0 && (fl & 2u))) &&
      (e2 > 0.0 || (e2 == 0.0 && (fl & 4u)))) {
    const double l0 = div_rn_pre(e1, R.area, R.rcp);
    const double l1 = div_rn_pre(e2, R.area, R.rcp);
    const double l2 = div_rn_pre(e0, R.area, R.rcp);
    const double inv_z = l0 * s_viz[R.v0] + l1 * s_viz[R.v1] + l2 * s_viz[R.v2];
    z = __drcp_rn(inv_z);
    return true;
  }
  return false;
}

// Winner of a pixel after a round (see the file header), -1 = unchanged.
__device__ __forceinline__ int resolve_winner(uint32_t key, uint8_t dec) {
  if (key >= 0x10000u) return (int)(key - 0x10000u);
  if (key != 0u && dec) return (int)(0xFFFFu - key);
  return -1;
}

__device__ __forceinline__ void put_rgb(uint8_t *col, uint32_t pix, uint32_t rgb) {
  col[3 * pix + 0] = (uint8_t)rgb;
  col[3 * pix + 1] = (uint8_t)(rgb >> 8);
  col[3 * pix + 2] = (uint8_t)(rgb >> 16);
}

__global__ void __launch_bounds__(kThreads, 1)
render_step_kernel(const RenderParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ EnvShared es;
  __shared__ DistSlot s_dist[32];
  __shared__ int s_scan[kWarps];
  __shared__ int s_wcnt[kWarps];  // fragments per warp segment
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
  uint32_t *s_cand0 = reinterpret_cast<uint32_t *>(smem + L.cand0);
  uint32_t *s_cnt = reinterpret_cast<uint32_t *>(smem + L.cnt);
  uint16_t *s_ids = reinterpret_cast<uint16_t *>(smem + L.ids);
  uint32_t *s_lcp = reinterpret_cast<uint32_t *>(smem + L.lcp);
  TriRec *s_rec = reinterpret_cast<TriRec *>(smem + L.rec);
  uint16_t *s_owner = reinterpret_cast<uint16_t *>(smem + L.owner);
  Frag *s_frag = reinterpret_cast<Frag *>(smem + L.frag);
  float *s_depth = reinterpret_cast<float *>(smem + L.depth);
  uint32_t *s_dbits = reinterpret_cast<uint32_t *>(smem + L.depth);
  uint8_t *s_col = smem + L.col;
  uint32_t *s_wkey = reinterpret_cast<uint32_t *>(smem + L.wkey);
  uint8_t *s_dec = smem + L.dec;
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
  const uint32_t lanemask_lt = (1u << lane) - 1u;

  // ---- once per CTA: floor rays, NN maps, mbarrier -----------------------
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
  if (tid == 0) {
    mbar_init(&es.vbar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  uint32_t vphase = 0;
  int local_env = 0;
  for (int64_t env = blockIdx.x; env < p.batch; env += gridDim.x, local_env++) {
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
      if (local_env % 32 == 0) {
        const int64_t e2 = env + (int64_t)lane * gridDim.x;
        if (e2 < p.batch) distractor_update(p, e2, s_dist[lane]);
        __syncwarp();
      }
      if (lane == 0) {
        const double *p0 = p.poses + (int64_t)env * p.nl * 3;
        es.ex = (float)(p0[0] + p.off_x);  // render.py:611
        es.ez = (float)(p0[1] + p.off_z);  // render.py:612
        const DistSlot &ds = s_dist[local_env % 32];
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
    __syncthreads();
    const float ex = es.ex, ez = es.ez;

    // ---- phase 1: world transform + projection (render.py:468-481, 350-363)
    for (int v = tid; v < p.nv; v += kThreads) {
      const float3 w = world_vertex(p, s_link, v);
      s_world[3 * v + 0] = w.x;
      s_world[3 * v + 1] = w.y;
      s_world[3 * v + 2] = w.z;
      const float vx = w.x - ex, vy = w.y - ey, vz = w.z - ez;
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

    // ---- phase 2: liveness + bbox size (render.py:366-416), background --
    for (int t = tid; t < p.nt; t += kThreads) {
      uint32_t n = 0;
      const int i0 = __ldg(p.tris + 3 * t + 0), i1 = __ldg(p.tris + 3 * t + 1),
                i2 = __ldg(p.tris + 3 * t + 2);
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
            if (!((double)sqrtf(nx * nx + ny * ny + nz * nz) < 1e-20))
              n = (uint32_t)((int)(bx1 - bx0) + 1) * (uint32_t)((int)(by1 - by0) + 1);
          }
        }
      }
      s_cnt[t] = n;
    }
    // background: sky / floor under an empty z-buffer (render.py:306-344)
    if (p.mode == PXR_MODE_VIDEO && !p.draw_floor) {
      // background colour is never read (every inf pixel takes the video)
      const float inf = __int_as_float(0x7f800000);
      const int n4 = npx >> 2;
      for (int i = tid; i < n4; i += kThreads) {
        reinterpret_cast<float4 *>(s_depth)[i] = make_float4(inf, inf, inf, inf);
        reinterpret_cast<uint4 *>(s_wkey)[i] = make_uint4(0u, 0u, 0u, 0u);
        reinterpret_cast<uint32_t *>(s_dec)[i] = 0u;
      }
      for (int i = (n4 << 2) + tid; i < npx; i += kThreads) {
        s_depth[i] = inf;
        s_wkey[i] = 0u;
        s_dec[i] = 0;
      }
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
          floor_px(p, ex, ez, dx, dy, dz, d, c);
        }
        s_depth[i] = d;
        put_rgb(s_col, (uint32_t)i, c);
        s_wkey[i] = 0u;
        s_dec[i] = 0;
      }
    }
    __syncthreads();
    // block scans over triangles in index order: live ids, candidate prefix
    {
      const int per = (p.nt + kThreads - 1) / kThreads;
      const int t0 = min(tid * per, p.nt), t1 = min(t0 + per, p.nt);
      int nlive = 0;
      for (int t = t0; t < t1; t++) nlive += s_cnt[t] != 0u;
      const int wincl = warp_incl_scan(nlive, lane);
      if (lane == 31) s_scan[warp] = wincl;
      __syncthreads();
      if (warp == 0) {
        const int v = lane < kWarps ? s_scan[lane] : 0;
        const int vi = warp_incl_scan(v, lane);
        if (lane < kWarps) s_scan[lane] = vi - v;
        if (lane == kWarps - 1) es.n_live = vi;
      }
      __syncthreads();
      int li = s_scan[warp] + wincl - nlive;
      for (int t = t0; t < t1; t++)
        if (s_cnt[t] != 0u) s_ids[li++] = (uint16_t)t;
      const int n_live_ = es.n_live;
      __syncthreads();
      const int lper = (n_live_ + kThreads - 1) / kThreads;
      const int l0 = min(tid * lper, n_live_), l1 = min(l0 + lper, n_live_);
      uint32_t csum = 0;
      for (int l = l0; l < l1; l++) csum += s_cnt[s_ids[l]];
      const int cw = warp_incl_scan((int)csum, lane);
      if (lane == 31) s_scan[warp] = cw;
      __syncthreads();
      if (warp == 0) {
        const int v = lane < kWarps ? s_scan[lane] : 0;
        const int vi = warp_incl_scan(v, lane);
        if (lane < kWarps) s_scan[lane] = vi - v;
      }
      __syncthreads();
      uint32_t acc = (uint32_t)(s_scan[warp] + cw) - csum;
      for (int l = l0; l < l1; l++) {
        s_lcp[l] = acc;
        acc += s_cnt[s_ids[l]];
      }
      if (tid == kThreads - 1) s_lcp[n_live_] = acc;  // last thread holds the total
    }
    __syncthreads();
    const int n_live = es.n_live;

    // ---- phases 3/4: raster rounds over live triangles in index order ---
    for (int r0 = 0; r0 < n_live;) {
      if (tid == 0) {
        // live [r0, r1): at most cap triangles and ~kRoundCand candidates
        int lo = r0 + 1, hi = min(r0 + p.cap, n_live);
        const uint32_t base = s_lcp[r0];
        while (lo < hi) {  // largest r1 with lcp[r1] - base <= budget
          const int mid = (lo + hi + 1) >> 1;
          if (s_lcp[mid] - base <= (uint32_t)p.round_cand) lo = mid; else hi = mid - 1;
        }
        es.round_end = lo;
        es.n_cand = (int)(s_lcp[lo] - base);
        es.chunk_next = 0;
        es.overflow = 0;
      }
      __syncthreads();
      const int r1 = es.round_end;
      const int n_cand = es.n_cand;
      const uint32_t cbase = s_lcp[r0];
      // records (render.py:366-436) + chunk owners
      for (int li = r0 + tid; li < r1; li += kThreads) {
        const int t = s_ids[li];
        int i0 = __ldg(p.tris + 3 * t + 0), i1 = __ldg(p.tris + 3 * t + 1),
            i2 = __ldg(p.tris + 3 * t + 2);
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
          double v = (double)__ldg(p.tri_colors + 3 * t + ch) * shade * 255.0;
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
        const uint32_t c0 = s_lcp[li] - cbase;
        R.cand0 = c0;
        R.px0 = (uint16_t)(int)bx0;
        R.py0 = (uint16_t)(int)by0;
        const int bw = (int)(bx1 - bx0) + 1, bh = (int)(by1 - by0) + 1;
        R.bw = (uint16_t)bw;
        R.bh = (uint16_t)bh;
        // ceil(2^32 / bw) through a double quotient: exact for 2 <= bw <= 2^20
        // (the true quotient's fractional part is >= 1/bw >> the 2^-21 error)
        R.magic = bw == 1 ? 0u : (uint32_t)ceil(4294967296.0 / (double)bw);
        s_rec[li - r0] = R;
        s_cand0[li - r0] = c0;
        const uint32_t c1 = c0 + (uint32_t)(bw * bh);
        for (uint32_t k = (c0 + 31) >> 5; k <= ((c1 - 1) >> 5); k++)
          s_owner[k] = (uint16_t)(li - r0);
      }
      __syncthreads();

      // candidates, flat over the warps (32 per chunk, dynamically scheduled);
      // each warp keeps its covered fragments in its own list segment
      const int n_chunks = (n_cand + 31) >> 5;
      const int n_round = r1 - r0;
      const int seg = p.frag_limit / kWarps;  // fragments per warp segment
      Frag *my_frag = s_frag + warp * (kFragCap / kWarps);
      int my_cnt = 0;
      while (true) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&es.chunk_next, 1);
        k = __shfl_sync(kFull, k, 0);
        if (k >= n_chunks) break;
        const int c = k * 32 + lane;
        // owner triangle of candidate c: the owner of the chunk's first
        // candidate plus the triangles that start inside the chunk up to c
        const int o0 = s_owner[k];
        const int mi = o0 + 1 + lane;
        uint32_t bit = 0;
        if (mi < n_round) {
          const int d = (int)s_cand0[mi] - k * 32;  // >= 1
          if (d < 32) bit = 1u << d;
        }
        const uint32_t starts = __reduce_or_sync(kFull, bit);
        const int j = o0 + __popc(starts & (0xFFFFFFFFu >> (31 - lane)));
        bool cov = false;
        uint32_t pix = 0;
        double z = 0.0;
        if (c < n_cand) {
          const TriRec &R = s_rec[j];
          cov = eval_candidate(p, R, c - (int)s_cand0[j], s_vxy64, s_viz, pix, z);
        }
        const uint32_t cm = __ballot_sync(kFull, cov);
        if (cm == 0u) continue;
        const int slot = my_cnt + __popc(cm & lanemask_lt);
        my_cnt += __popc(cm);
        if (cov) {
          const uint32_t zb = __float_as_uint((float)z);
          if (zb < atomicMin(&s_dbits[pix], zb)) s_dec[pix] = 1;
          if (slot < seg) {
            Frag f;
            f.z = z;
            f.pix = pix;
            f.tri = (uint32_t)j;
            my_frag[slot] = f;
          }
        }
      }
      if (lane == 0) {
        s_wcnt[warp] = my_cnt;
        if (my_cnt > seg) es.overflow = 1;
      }
      __syncthreads();

      // exact sequential-order resolve (see the file header)
      constexpr int kSeg = kFragCap / kWarps;
      if (!es.overflow) {
        for (int i = tid; i < kFragCap; i += kThreads) {
          if ((i % kSeg) >= s_wcnt[i / kSeg]) continue;
          const Frag f = s_frag[i];
          const uint32_t F = s_dbits[f.pix];
          if (__float_as_uint((float)f.z) == F)
            atomicMax(&s_wkey[f.pix],
                      f.z < (double)__uint_as_float(F) ? 0x10000u + f.tri : 0xFFFFu - f.tri);
        }
        __syncthreads();
        for (int i = tid; i < kFragCap; i += kThreads) {
          if ((i % kSeg) >= s_wcnt[i / kSeg]) continue;
          const Frag f = s_frag[i];
          if (resolve_winner(s_wkey[f.pix], s_dec[f.pix]) == (int)f.tri)
            put_rgb(s_col, f.pix, s_rec[f.tri].rgb);
        }
        if (r1 < n_live) {
          __syncthreads();
          for (int i = tid; i < kFragCap; i += kThreads) {
            if ((i % kSeg) >= s_wcnt[i / kSeg]) continue;
            const uint32_t px = s_frag[i].pix;
            s_wkey[px] = 0u;
            s_dec[px] = 0;
          }
        }
      } else {
        // fragment list overflow: recompute the candidates for both passes
        for (int pass = 0; pass < 2; pass++) {
          for (int k = warp; k < n_chunks; k += kWarps) {
            const int c = k * 32 + lane;
            if (c >= n_cand) continue;
            int j = s_owner[k];
            while (j + 1 < n_round && s_rec[j + 1].cand0 <= (uint32_t)c) j++;
            const TriRec &R = s_rec[j];
            uint32_t pix;
            double z;
            if (!eval_candidate(p, R, c - (int)R.cand0, s_vxy64, s_viz, pix, z)) continue;
            const uint32_t F = s_dbits[pix];
            if (__float_as_uint((float)z) != F) continue;
            if (pass == 0) {
              atomicMax(&s_wkey[pix],
                        z < (double)__uint_as_float(F) ? 0x10000u + j : 0xFFFFu - j);
            } else if (resolve_winner(s_wkey[pix], s_dec[pix]) == j) {
              put_rgb(s_col, pix, R.rgb);
            }
          }
          __syncthreads();
        }
        if (r1 < n_live) {
          for (int i = tid; i < npx; i += kThreads) {
            s_wkey[i] = 0u;
            s_dec[i] = 0;
          }
        }
      }
      __syncthreads();
      r0 = r1;
    }

    // ---- phase 5: composite + postprocess (distractor.py:140-176, env.py:168-173)
    if (p.mode == PXR_MODE_VIDEO && p.vframe_bulk) mbar_wait_parity(&es.vbar, vphase);
    const uint8_t *vsrc = p.mode == PXR_MODE_VIDEO
                              ? (p.vframe_bulk ? s_vframe
                                               : p.frames + es.frame_idx * p.vframe_bytes)
                              : nullptr;
    // Four consecutive pixels per thread: 12 colour bytes are three aligned
    // words; the colour bias is a per-byte saturating add/sub (__vaddus4 /
    // __vsubus4 == clamp(v + b, 0, 255) for |b| <= 255).
    uint32_t bpos[3] = {0u, 0u, 0u}, bneg[3] = {0u, 0u, 0u};
    if (p.mode == PXR_MODE_COLOR) {
      for (int byte = 0; byte < 12; byte++) {
        const int bc = es.bias[byte % 3];
        bpos[byte >> 2] |= (uint32_t)(bc > 0 ? bc : 0) << (8 * (byte & 3));
        bneg[byte >> 2] |= (uint32_t)(bc < 0 ? -bc : 0) << (8 * (byte & 3));
      }
    }
    const int ngroups = npx >> 2;
    for (int gi = tid; gi < ngroups + (npx & 3); gi += kThreads) {
      const bool tail = gi >= ngroups;
      const int i0 = tail ? (ngroups << 2) + (gi - ngroups) : (gi << 2);
      const int np_ = tail ? 1 : 4;
      float d[4];
      uint32_t w[3];
      if (!tail) {
        const float4 d4 = reinterpret_cast<const float4 *>(s_depth)[gi];
        d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
        const uint32_t *c3 = reinterpret_cast<const uint32_t *>(s_col) + 3 * gi;
        w[0] = c3[0]; w[1] = c3[1]; w[2] = c3[2];
      } else {
        d[0] = s_depth[i0];
        w[0] = s_col[3 * i0] | (s_col[3 * i0 + 1] << 8) | (s_col[3 * i0 + 2] << 16);
        w[1] = w[2] = 0u;
      }
      if (p.mode == PXR_MODE_VIDEO) {  // distractor.py:172-176
        int y = (int)__umulhi((uint32_t)i0, p.wmagic);
        int x = i0 - y * p.W;
        for (int k = 0; k < np_; k++) {
          if (isinf(d[k])) {
            const uint8_t *src = vsrc + ((int)s_rowmap[y] * p.Wv + (int)s_colmap[x]) * 3;
            for (int ch = 0; ch < 3; ch++) {
              const int byte = 3 * k + ch;
              const int wi = byte >> 2, sh = 8 * (byte & 3);
              w[wi] = (w[wi] & ~(0xffu << sh)) | ((uint32_t)src[ch] << sh);
            }
          }
          if (++x == p.W) { x = 0; y++; }
        }
      } else if (p.mode == PXR_MODE_COLOR) {  // distractor.py:149-161
        for (int q = 0; q < 3; q++) w[q] = __vsubus4(__vaddus4(w[q], bpos[q]), bneg[q]);
      }
      if (p.gray) {  // env.py:168-173
        uint32_t gw = 0;
        for (int k = 0; k < np_; k++) {
          uint32_t ch3[3];
          for (int ch = 0; ch < 3; ch++) {
            const int byte = 3 * k + ch;
            ch3[ch] = (w[byte >> 2] >> (8 * (byte & 3))) & 0xffu;
          }
          gw |= ((299u * ch3[0] + 587u * ch3[1] + 114u * ch3[2] + 500u) / 1000u) << (8 * k);
        }
        if (!tail) reinterpret_cast<uint32_t *>(s_gray)[gi] = gw;
        else s_gray[i0] = (uint8_t)gw;
      } else if (!tail) {
        uint32_t *c3 = reinterpret_cast<uint32_t *>(s_col) + 3 * gi;
        c3[0] = w[0]; c3[1] = w[1]; c3[2] = w[2];
      } else {
        put_rgb(s_col, (uint32_t)i0, w[0]);
      }
      if (p.out_depth != nullptr) {
        float *dd = p.out_depth + (int64_t)env * npx + i0;
        if (!tail && p.depth_vec) *reinterpret_cast<float4 *>(dd) = make_float4(d[0], d[1], d[2], d[3]);
        else for (int k = 0; k < np_; k++) dd[k] = d[k];
      }
    }
    vphase ^= 1u;

    // ---- phase 6: frame -> HBM (one TMA bulk store) --------------------
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
  const int C = p.gray ? 1 : 3;
  const int64_t npx64 = height * width;
  if (npx64 > (1 << 20) || height > 4096 || width > 4096)
    return set_unsupported("frame too large");
  p.wmagic = (uint32_t)((0x100000000ull + (uint64_t)width - 1) / (uint64_t)width);
  p.depth_vec = out_depth != nullptr && (npx64 % 4 == 0) &&
                ((reinterpret_cast<uintptr_t>(out_depth) & 15) == 0);
  p.frame_bytes = (int)(npx64 * C);
  p.use_bulk = (p.frame_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(out_obs) & 15) == 0);
  // Test hooks (tests/test_gpu_parity.py): shrink the per-round budgets so
  // the multi-round and fragment-overflow paths run on small inputs.
  p.round_cand = kRoundCand;
  p.frag_limit = kFragCap;
  int debug_cap = 0;
  if (const char *s = getenv("PXR_DEBUG_ROUND_CAND")) p.round_cand = atoi(s) > 0 ? atoi(s) : kRoundCand;
  if (const char *s = getenv("PXR_DEBUG_FRAG_LIMIT")) p.frag_limit = atoi(s) >= 0 ? min(atoi(s), kFragCap) : kFragCap;
  if (const char *s = getenv("PXR_DEBUG_CAP")) debug_cap = atoi(s);
  // one round's candidates never exceed max(round budget, one triangle's bbox)
  p.chunk_cap = (int)((npx64 > p.round_cand ? npx64 : p.round_cand) / 32 + 2);

  int dev = 0;
  cudaGetDevice(&dev);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int budget =
      max_optin - (int)(sizeof(EnvShared) + sizeof(DistSlot) * 32 + 4 * kWarps) - 256;
  // Live-triangle records per round: all triangles if they fit, else the
  // largest count that does (extra rounds handle the rest exactly).
  int cap = p.nt > 0 ? p.nt : 1;
  if (debug_cap > 0 && debug_cap < cap) cap = debug_cap;
  for (;;) {
    p.cap = cap;
    if (smem_layout(p).total <= budget || cap <= 16) break;
    cap = cap > 64 ? cap - 32 : cap - 8;
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

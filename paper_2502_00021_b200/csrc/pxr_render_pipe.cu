// Warp-specialised two-stage render pipeline for sm_100a: the same fused step
// as render_step_kernel (pxr_render.cu; reference: env.py:155-173,
// render.py:286-485, 594-623, distractor.py:116-214), with the env's
// geometry stage and its raster stage running CONCURRENTLY on two warp
// groups of one persistent CTA, one env apart:
//
//   geometry warps G (kGW warps): per env -- link trig (glibc-exact cosf /
//     sinf) and the distractor step (32 envs at a time), world transform +
//     projection of every vertex (render.py:468-481, 350-363), triangle
//     liveness (render.py:366-416) and the block scan over triangles in
//     index order, then per raster round the triangle records (edge flags,
//     exact reciprocal of the area, flat colour, render.py:366-436) and the
//     conservative row-span line equations;
//   raster warps R (kRW warps): per round -- (triangle, bbox row) units ->
//     per-warp span queues -> 32-candidate batches -> the reference's exact
//     f64 edge / barycentric / depth test (render.py:437-451); per env --
//     the z-buffer init, and the final pass that turns each pixel's resolved
//     word into its final colour (triangle colour or sky / floor / video
//     texel, colour distractor, grayscale) and stores the frame.
//
// While R rasterises env e, G builds env e+1: the two instruction streams
// fill each other's barrier and latency bubbles. G -> R hand-off per raster
// round through double-buffered record sets (mbarriers full/empty), R -> G
// per env through double-buffered vertex / colour sets (mbarrier env).
// Each group synchronises internally with its own named barrier (bar.sync
// 1 / 2), never with the whole CTA.
//
// Exact sequential z-test in ONE pass. Each pixel holds a 64-bit word
// (RN32(depth) bits << 32 | sub), initialised to (background depth, kBgSub),
// and every covered candidate of live triangle li (index order, global over
// the env's rounds) min-reduces (RN32(z) bits, sub) into it, with
// sub = 0x7FFFFFFF - li when z < RN32(z) and 0x80000001 + li otherwise.
// This is the reference's sequential strict test `zpix(f64) < depth(f32)`
// (render.py:452) in closed form: let F = min RN32(z) over a pixel's
// fragments and S = {fragments with RN32(z) == F}. If F < d0 the first
// member of S always writes and later members write iff z < F; fragments
// outside S never write; so the last writer is the highest-index member of
// S with z < F if there is one, else the lowest-index member. If F == d0
// only members with z < F write. The minimum of the words is exactly that
// winner (or the initial word when nothing writes), and the depth the
// reference stores is F. Minima over rounds compose (indices are global),
// so multi-round envs need no key reset.
#include "pxr_raster.cuh"

namespace pxr {

#ifndef PXR_PIPE_GWARPS
#define PXR_PIPE_GWARPS 12
#endif
constexpr int kGW = PXR_PIPE_GWARPS;  // geometry warps
constexpr int kRW = kWarps - kGW;     // raster warps
constexpr int kGT = kGW * 32, kRT = kRW * 32;
static_assert(kGW >= 4 && kRW >= 4 && kGW % 4 == 0, "warp groups");
constexpr int kPipeRowCap = 4096;  // (triangle, bbox row) units per raster round
constexpr uint32_t kInfBits = 0x7f800000u;

// A live triangle's exact-test data (post-swap order, render.py:381-385); the
// f32 edge vectors are recomputed from the vertices on use (the same f32
// subtractions, so the same values).
struct __align__(8) PTri {
  uint16_t v0, v1, v2, flags;
  float area;
  uint32_t pad;
  double rcp;  // RN(1 / (double)area2)
};
static_assert(sizeof(PTri) == 24, "PTri layout");

struct PipeRound {
  int e;         // local env index of the CTA
  int r0, r1;    // live triangles [r0, r1) of the env
  int n_rows;    // (triangle, bbox row) units of the round
  int first, last;
};

struct PipeShared {
  uint64_t bar_full[2];   // G -> R: round records of buffer b written
  uint64_t bar_empty[2];  // R -> G: round records of buffer b consumed
  uint64_t bar_env[2];    // R -> G: vertex / colour set of env parity b consumed
  uint64_t bar_video;     // the env's video frame (TMA bulk load)
  EnvShared es;           // per env parity: camera x/z, distractor bias, frame index
  PipeRound round[2];
  DistSlot dist[32];
  int scan[2 * kGW];
  int n_live, one_round, round_end, plan_ok;
  long long prof[16];  // stage cycles (p.prof != null): G 0-6, R 8-12, counts 13-14
};

struct PipeLayout {
  int link, floor, maps, gplan, vxy[2], viz[2], vz, world, rows, ids, lrp, rgb[2], tri[2],
      span[2], rowpre[2], rowner[2], z, stage, vframe, queue, total;
};

__host__ __device__ inline PipeLayout pipe_layout(const RenderParams &p) {
  PipeLayout L;
  int o = 0;
  const bool video = p.mode == PXR_MODE_VIDEO;
  L.link = o;   o += align_up(p.nl * 16, 16);
  L.floor = o;  o += p.draw_floor ? align_up((p.W + 3 * p.H) * 8 + p.H * 4, 16) : 0;
  L.maps = o;   o += video ? align_up((p.W + p.H) * 4, 16) : 0;
  L.gplan = o;  o += video ? align_up((p.W / 4 + 1) * 16, 16) : 0;
  for (int b = 0; b < 2; b++) {
    L.vxy[b] = o; o += align_up(p.nv * 8, 16);
    L.viz[b] = o; o += align_up(p.nv * 8, 16);
  }
  L.vz = o;     o += align_up(p.nv * 4, 16);
  L.world = o;  o += align_up(p.nv * 12, 16);
  L.rows = o;   o += align_up((p.nt + 1) * 2, 16);
  L.ids = o;    o += align_up((p.nt + 1) * 2, 16);
  L.lrp = o;    o += align_up((p.nt + 1) * 4, 16);
  for (int b = 0; b < 2; b++) { L.rgb[b] = o; o += align_up(p.nt * 4 + 4, 16); }
  for (int b = 0; b < 2; b++) {
    L.tri[b] = o;    o += align_up(p.cap * (int)sizeof(PTri), 16);
    L.span[b] = o;   o += p.cap * (int)sizeof(SpanRec);
    L.rowpre[b] = o; o += align_up((p.cap + 1) * 4, 16);
    L.rowner[b] = o; o += align_up((p.row_cap / 32 + 2) * 2, 16);
  }
  L.z = o;      o += align_up(p.H * p.W * 8, 16);
  L.stage = o;  o += kRW * 384;
  // + 32 B: the byte-permute gather may read up to 20 B past the last texel
  L.vframe = o; o += video ? align_up(p.vframe_bytes + 32, 16) : 0;
  L.queue = o;  o += kRW * kQueue * 8;
  L.total = o;
  return L;
}

__device__ __forceinline__ void gbar() { asm volatile("bar.sync 1, %0;" ::"n"(kGT) : "memory"); }
__device__ __forceinline__ void rbar() { asm volatile("bar.sync 2, %0;" ::"n"(kRT) : "memory"); }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The reference's exact coverage test and depth (render.py:437-451) for a
// pixel centre of live triangle R; vertices in f32 (exactly the f64 values the
// reference uses), 1/z in f64.
__device__ __forceinline__ bool eval_exact_pipe(const PTri &R, int px, int py, const float2 *vxy,
                                                const double *viz, double &z) {
  const float2 a = vxy[R.v0], b = vxy[R.v1], c = vxy[R.v2];
  const float A0 = b.x - a.x, B0 = b.y - a.y;
  const float A1 = c.x - b.x, B1 = c.y - b.y;
  const float A2 = a.x - c.x, B2 = a.y - c.y;
  const double pcx = half_plus(px), pcy = half_plus(py);
  const double e0 = (double)A0 * (pcy - (double)a.y) - (double)B0 * (pcx - (double)a.x);
  const double e1 = (double)A1 * (pcy - (double)b.y) - (double)B1 * (pcx - (double)b.x);
  const double e2 = (double)A2 * (pcy - (double)c.y) - (double)B2 * (pcx - (double)c.x);
  const uint32_t fl = R.flags;
  if ((e0 > 0.0 || (e0 == 0.0 && (fl & 1u))) && (e1 > 0.0 || (e1 == 0.0 && (fl & 2u))) &&
      (e2 > 0.0 || (e2 == 0.0 && (fl & 4u)))) {
    const double area = (double)R.area;
    const double l0 = div_rn_pre(e1, area, R.rcp);
    const double l1 = div_rn_pre(e2, area, R.rcp);
    const double l2 = div_rn_pre(e0, area, R.rcp);
    const double inv_z = l0 * viz[R.v0] + l1 * viz[R.v1] + l2 * viz[R.v2];
    z = __drcp_rn(inv_z);
    return true;
  }
  return false;
}

// stage cycle counters of one group leader (debug, p.prof != null)
#define PIPE_PROF(cond, slot)                        \
  do {                                               \
    if (p.prof != nullptr && (cond)) {               \
      const long long now_ = clock64();              \
      S.prof[slot] += now_ - prof_t;                 \
      prof_t = now_;                                 \
    }                                                \
  } while (0)

template <bool kFloor>
__global__ void __launch_bounds__(kThreads, 1) render_pipe_kernel(const RenderParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ PipeShared S;
  const PipeLayout L = pipe_layout(p);
#ifdef PXR_CHECKED
  {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    PXR_DCHECK((uint32_t)L.total <= dyn);
  }
#endif
  float4 *s_link = reinterpret_cast<float4 *>(smem + L.link);
  double *s_floor = reinterpret_cast<double *>(smem + L.floor);  // dx[W], dy[H], dz[H]
  double *s_ft = s_floor + p.W + 2 * p.H;                          // per-row floor t
  int *s_fk = reinterpret_cast<int *>(s_ft + p.H);                 // per-row parity / -1
  uint32_t *s_rowmap = reinterpret_cast<uint32_t *>(smem + L.maps);
  uint32_t *s_colmap = s_rowmap + p.H;
  uint4 *s_gplan = reinterpret_cast<uint4 *>(smem + L.gplan);
  float *s_vz = reinterpret_cast<float *>(smem + L.vz);
  float *s_world = reinterpret_cast<float *>(smem + L.world);
  uint16_t *s_rows = reinterpret_cast<uint16_t *>(smem + L.rows);
  uint16_t *s_ids = reinterpret_cast<uint16_t *>(smem + L.ids);
  uint32_t *s_lrp = reinterpret_cast<uint32_t *>(smem + L.lrp);
  unsigned long long *s_z = reinterpret_cast<unsigned long long *>(smem + L.z);
  uint8_t *s_vframe = smem + L.vframe;

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int npx = p.H * p.W;
  const uint32_t lanemask_lt = (1u << lane) - 1u;
  const uint32_t lanemask_le = 0xFFFFFFFFu >> (31 - lane);

  // ---- once per CTA: floor rays, NN maps, byte-permute plan, mbarriers ----
  if (kFloor) {
    for (int i = tid; i < p.W; i += kThreads) s_floor[i] = p.floor_rays[(int64_t)i * 3];
    for (int i = tid; i < p.H; i += kThreads) {
      s_floor[p.W + i] = p.floor_rays[(int64_t)i * p.W * 3 + 1];
      s_floor[p.W + p.H + i] = p.floor_rays[(int64_t)i * p.W * 3 + 2];
    }
  }
  if (p.mode == PXR_MODE_VIDEO) {  // nearest_map, distractor.py:179-181
    for (int i = tid; i < p.H; i += kThreads)
      s_rowmap[i] = (uint32_t)(((int64_t)i * p.Hv) / p.H) * p.Wv * 3;
    for (int i = tid; i < p.W; i += kThreads)
      s_colmap[i] = (uint32_t)(((int64_t)i * p.Wv) / p.W) * 3;
  }
  if (tid == 0) {
    for (int b = 0; b < 2; b++) {
      mbar_init(&S.bar_full[b], kGT);
      mbar_init(&S.bar_empty[b], kRT);
      mbar_init(&S.bar_env[b], kRT);
    }
    mbar_init(&S.bar_video, 1);
    fence_mbar_init();
    S.plan_ok = 0;
    for (int i = 0; i < 16; i++) S.prof[i] = 0;
  }
  __syncthreads();
  // byte-permute plan of the NN video gather (see pxr_render.cu)
  const bool use_plan = p.mode == PXR_MODE_VIDEO && p.vframe_bulk && (p.W & 3) == 0 &&
                        ((p.Wv * 3) & 3) == 0 && !p.gray;
  if (use_plan) {
    int bad = 0;
    for (int gc = tid; gc < (p.W >> 2); gc += kThreads) {
      const int x0 = gc * 4;
      const uint32_t base_word = s_colmap[x0] >> 2;
      uint4 pl;
      pl.x = base_word;
      uint32_t sel[3];
      for (int q = 0; q < 3; q++) {
        int r[4], rmin = 1 << 30;
        for (int bb = 0; bb < 4; bb++) {
          const int bi = 4 * q + bb, k = bi / 3, ch = bi % 3;
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
    if (bad) S.plan_ok = -1;
  }
  __syncthreads();
  const bool plan_ok = use_plan && S.plan_ok == 0;
  long long prof_t = p.prof != nullptr ? clock64() : 0;
  const long long prof_t0 = prof_t;

  if (warp < kGW) {
    // =================== geometry warps ====================================
    const int gt = tid;
    // liveness: each thread owns a contiguous block of triangles (index order)
    const int per = (p.nt + kGT - 1) / kGT;
    const int t0 = min(gt * per, p.nt), t1 = min(t0 + per, p.nt);
    int g_link = 0;
    float g_bx = 0.0f, g_by = 0.0f, g_bz = 0.0f;
    if (gt < p.nv) {
      g_link = __ldg(p.vert_link + gt);
      PXR_DCHECK(g_link >= 0 && g_link < p.nl);
      g_bx = __ldg(p.base_verts + 3 * gt + 0);
      g_by = __ldg(p.base_verts + 3 * gt + 1);
      g_bz = __ldg(p.base_verts + 3 * gt + 2);
    }
    const float ey = p.cam[1];
    const float rx = p.cam[3], ry = p.cam[4], rz = p.cam[5];
    const float ux = p.cam[6], uy = p.cam[7], uz = p.cam[8];
    const float fx = p.cam[9], fy = p.cam[10], fz = p.cam[11];
    const float tanf_ = p.cam[12], near_ = p.cam[13], far_ = p.cam[14];
    const float lx = p.light[0], ly = p.light[1], lz = p.light[2];
    const double aspect = (double)p.W / (double)p.H;  // render.py:303
    int k = 0;  // raster rounds produced
    int e = 0;
    for (int64_t env = blockIdx.x; env < p.batch; env += gridDim.x, e++) {
      const int eb = e & 1;
      float2 *s_vxy = reinterpret_cast<float2 *>(smem + L.vxy[eb]);
      double *s_viz = reinterpret_cast<double *>(smem + L.viz[eb]);
      uint32_t *s_rgb = reinterpret_cast<uint32_t *>(smem + L.rgb[eb]);
      // the vertex / colour set of this parity is free once R finished env e-2
      if (e >= 2) mbar_wait_parity(&S.bar_env[eb], (uint32_t)(((e >> 1) - 1) & 1));
      PIPE_PROF(gt == 0, 0);
      if (warp == 0) prepare_env(p, env, e, s_link, S.dist, S.es, lane);
      int n0 = 0, n1 = 0, n2 = 0;  // first liveness triangle, loaded early
      if (t0 < t1) {
        n0 = __ldg(p.tris + 3 * t0 + 0);
        n1 = __ldg(p.tris + 3 * t0 + 1);
        n2 = __ldg(p.tris + 3 * t0 + 2);
      }
      gbar();
      PIPE_PROF(gt == 0, 1);
      const float ex = S.es.ex[eb], ez = S.es.ez[eb];

      // ---- world transform + projection (render.py:468-481, 350-363) ----
      for (int v = gt; v < p.nv; v += kGT) {
        float3 w;
        if (v == gt) {
          const float4 lk = s_link[g_link];
          w = make_float3(lk.x + g_bx * lk.z - g_bz * lk.w, g_by,
                          lk.y + g_bx * lk.w + g_bz * lk.z);
        } else {
          w = world_vertex(p, s_link, v);
        }
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
        s_vxy[v] = make_float2(sx, sy);
        s_viz[v] = __drcp_rn((double)zv);  // iz = 1.0 / z (render.py:434-436)
      }
      gbar();
      PIPE_PROF(gt == 0, 2);

      // ---- liveness (render.py:366-416) -----------------------------------
      int my_live = 0, my_rows = 0;
      for (int t = t0; t < t1; t++) {
        uint32_t rows = 0;
        const int i0 = n0, i1 = n1, i2 = n2;
        if (t + 1 < t1) {
          n0 = __ldg(p.tris + 3 * t + 3);
          n1 = __ldg(p.tris + 3 * t + 4);
          n2 = __ldg(p.tris + 3 * t + 5);
        }
        PXR_DCHECK(i0 >= 0 && i0 < p.nv && i1 >= 0 && i1 < p.nv && i2 >= 0 && i2 < p.nv);
        const float z0 = s_vz[i0], z1 = s_vz[i1], z2 = s_vz[i2];
        if (!(z0 < near_ || z1 < near_ || z2 < near_) && !(z0 > far_ && z1 > far_ && z2 > far_)) {
          const float2 a = s_vxy[i0], b = s_vxy[i1], c = s_vxy[i2];
          const float area2 = (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
          if (area2 != 0.0f) {
            const float minx = fminf(a.x, fminf(b.x, c.x)), maxx = fmaxf(a.x, fmaxf(b.x, c.x));
            const float miny = fminf(a.y, fminf(b.y, c.y)), maxy = fmaxf(a.y, fmaxf(b.y, c.y));
            int bx0, bx1, by0, by1;
            pixel_range(minx, maxx, p.W - 1, bx0, bx1);
            pixel_range(miny, maxy, p.H - 1, by0, by1);
            if (!(bx0 > bx1 || by0 > by1)) rows = (uint32_t)(by1 - by0 + 1);
          }
        }
        s_rows[t] = (uint16_t)rows;
        my_live += rows != 0u;
        my_rows += (int)rows;
      }
      // block scan over the G threads, triangles in index order
      {
        int li;
        uint32_t racc;
        if (p.scan_sh > 0) {
          const int sh = p.scan_sh;
          const uint32_t mine = ((uint32_t)my_live << sh) | (uint32_t)my_rows;
          const uint32_t w = (uint32_t)warp_incl_scan((int)mine, lane);
          if (lane == 31) S.scan[warp] = (int)w;
          gbar();
          const uint32_t v = lane < kGW ? (uint32_t)S.scan[lane] : 0u;
          const uint32_t vi = (uint32_t)warp_incl_scan((int)v, lane);
          const uint32_t pre = __shfl_sync(kFull, vi - v, warp) + w - mine;
          li = (int)(pre >> sh);
          racc = pre & ((1u << sh) - 1u);
        } else {
          const int wl = warp_incl_scan(my_live, lane);
          const int wr = warp_incl_scan(my_rows, lane);
          if (lane == 31) {
            S.scan[warp] = wl;
            S.scan[kGW + warp] = wr;
          }
          gbar();
          const int v = lane < kGW ? S.scan[lane] : 0;
          const int u = lane < kGW ? S.scan[kGW + lane] : 0;
          const int vi = warp_incl_scan(v, lane), ui = warp_incl_scan(u, lane);
          li = __shfl_sync(kFull, vi - v, warp) + wl - my_live;
          racc = (uint32_t)(__shfl_sync(kFull, ui - u, warp) + wr - my_rows);
        }
        for (int t = t0; t < t1; t++) {
          const int r = s_rows[t];
          if (r != 0) {
            PXR_DCHECK(li < p.nt);
            s_ids[li] = (uint16_t)t;
            s_lrp[li] = racc;
            li++;
            racc += (uint32_t)r;
          }
        }
        if (gt == kGT - 1) {  // the last thread holds the totals
          s_lrp[li] = racc;
          S.n_live = li;
          S.one_round = li <= p.cap && racc <= (uint32_t)p.row_cap;
        }
      }
      gbar();
      PIPE_PROF(gt == 0, 3);
      const int n_live = S.n_live;
      const bool one_round = S.one_round != 0;

      // ---- raster rounds: records into the round buffers ------------------
      int r0 = 0;
      do {
        int r1 = n_live;
        if (!one_round) {
          gbar();  // every G thread has read the previous round's end
          if (gt == 0) {
            // live [r0, r1): at most cap triangles and row_cap bbox rows, the
            // rounds' triangle counts balanced
            const int left = n_live - r0;
            const int n_rounds = (left + p.cap - 1) / p.cap;
            const int target = (left + n_rounds - 1) / n_rounds;
            int lo = r0 + 1, hi = min(r0 + target, n_live);
            const uint32_t base = s_lrp[r0];
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (s_lrp[mid] - base <= (uint32_t)p.row_cap) lo = mid; else hi = mid - 1;
            }
            S.round_end = lo;
          }
          gbar();
          r1 = S.round_end;
        }
        const int b = k & 1;
        PTri *s_tri = reinterpret_cast<PTri *>(smem + L.tri[b]);
        SpanRec *s_span = reinterpret_cast<SpanRec *>(smem + L.span[b]);
        uint32_t *s_rowpre = reinterpret_cast<uint32_t *>(smem + L.rowpre[b]);
        uint16_t *s_rowner = reinterpret_cast<uint16_t *>(smem + L.rowner[b]);
        // the round buffer is free once R finished round k-2
        if (k >= 2) mbar_wait_parity(&S.bar_empty[b], (uint32_t)(((k >> 1) - 1) & 1));
        PIPE_PROF(gt == 0, 4);
        const uint32_t rbase = s_lrp[r0];
        PXR_DCHECK(r1 - r0 <= p.cap && s_lrp[r1] - rbase <= (uint32_t)p.row_cap);
        for (int li = r0 + gt; li < r1; li += kGT) {
          const int t = s_ids[li];
          int i0 = __ldg(p.tris + 3 * t + 0), i1 = __ldg(p.tris + 3 * t + 1),
              i2 = __ldg(p.tris + 3 * t + 2);
          const float2 a = s_vxy[i0];
          float2 bb = s_vxy[i1], c = s_vxy[i2];
          float area2 = (bb.x - a.x) * (c.y - a.y) - (bb.y - a.y) * (c.x - a.x);
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
            const float2 tmp = bb; bb = c; c = tmp;
            const int ti = i1; i1 = i2; i2 = ti;
            area2 = -area2;
          }
          const float miny = fminf(a.y, fminf(bb.y, c.y)), maxy = fmaxf(a.y, fmaxf(bb.y, c.y));
          int by0, by1;
          pixel_range(miny, maxy, p.H - 1, by0, by1);
          const float ax0 = bb.x - a.x, ay0 = bb.y - a.y;
          const float ax1 = c.x - bb.x, ay1 = c.y - bb.y;
          const float ax2 = a.x - c.x, ay2 = a.y - c.y;
          uint32_t fl = 0;
          if (ay0 < 0.0f || (ay0 == 0.0f && ax0 > 0.0f)) fl |= 1u;
          if (ay1 < 0.0f || (ay1 == 0.0f && ax1 > 0.0f)) fl |= 2u;
          if (ay2 < 0.0f || (ay2 == 0.0f && ax2 > 0.0f)) fl |= 4u;
          PTri R;
          R.v0 = (uint16_t)i0; R.v1 = (uint16_t)i1; R.v2 = (uint16_t)i2;
          R.flags = (uint16_t)fl;
          R.area = area2;
          R.pad = 0;
          R.rcp = __drcp_rn((double)area2);
          PXR_DCHECK(li - r0 < p.cap);
          PXR_DCHECK(s_lrp[li + 1] - s_lrp[li] == (uint32_t)(by1 - by0 + 1));
          s_tri[li - r0] = R;
          s_rgb[li] = rgb;
          SpanRec Sp;
          span_setup(a, bb, c, (float)(p.H + 1), Sp);
          const bool culled = (double)nn < 1e-20;  // degenerate normal (render.py:405-409)
          if (culled) Sp.ylo = __int_as_float(0x7f800000);  // every row span is empty
          Sp.py0 = (uint16_t)by0;
          Sp.pad = 0;
          const uint32_t u0 = s_lrp[li] - rbase;
          Sp.row0 = u0;
          s_span[li - r0] = Sp;
          s_rowpre[li - r0] = u0;
          const uint32_t u1 = u0 + (uint32_t)(by1 - by0 + 1);
          PXR_DCHECK(((u1 - 1) >> 5) < (uint32_t)(p.row_cap / 32 + 2));
          for (uint32_t kk = (u0 + 31) >> 5; kk <= ((u1 - 1) >> 5); kk++)
            s_rowner[kk] = (uint16_t)(li - r0);
        }
        if (gt == 0) {
          PipeRound &R = S.round[b];
          R.e = e;
          R.r0 = r0;
          R.r1 = r1;
          R.n_rows = (int)(s_lrp[r1] - rbase);
          R.first = r0 == 0;
          R.last = r1 >= n_live;
          s_rowpre[r1 - r0] = (uint32_t)R.n_rows;
        }
        mbar_arrive(&S.bar_full[b]);  // every G thread, after its own writes
        PIPE_PROF(gt == 0, 5);
        if (p.prof != nullptr && gt == 0) S.prof[13] += 1;
        k++;
        r0 = r1;
      } while (r0 < n_live);
      if (p.prof != nullptr && gt == 0) S.prof[14] += 1;
    }
    if (p.prof != nullptr && gt == 0) S.prof[6] = clock64() - prof_t0;
  } else {
    // =================== raster warps ======================================
    const int rt = tid - kGT;
    const int rw = warp - kGW;
    const float wlim = (float)p.W - 0.5f;  // last pixel centre
    uint2 *q = reinterpret_cast<uint2 *>(smem + L.queue) + rw * kQueue;
    uint32_t *stage = reinterpret_cast<uint32_t *>(smem + L.stage) + rw * 96;
    const int chans = p.gray ? 1 : 3;
    const int chunk_px = 128;  // pixels per warp chunk of the final pass (4 per lane)
    const int n_pchunks = (npx + chunk_px - 1) / chunk_px;
    uint32_t vphase = 0;
    int k = 0;
    int e = 0;
    for (int64_t env = blockIdx.x; env < p.batch; env += gridDim.x, e++) {
      const int eb = e & 1;
      const float2 *s_vxy = reinterpret_cast<const float2 *>(smem + L.vxy[eb]);
      const double *s_viz = reinterpret_cast<const double *>(smem + L.viz[eb]);
      const uint32_t *s_rgb = reinterpret_cast<const uint32_t *>(smem + L.rgb[eb]);
      bool last = false;
      do {
        const int b = k & 1;
        mbar_wait_parity(&S.bar_full[b], (uint32_t)((k >> 1) & 1));
        PIPE_PROF(rt == 0, 8);
        const PipeRound R = S.round[b];
        PXR_DCHECK(R.e == e);
        if (R.first) {
          // ---- env start: video frame fetch, floor rows, z-buffer init ----
          rbar();  // the previous env's final pass is done with z / vframe
          if (rt == 0 && p.mode == PXR_MODE_VIDEO && p.vframe_bulk) {
            PXR_DCHECK(S.es.frame_idx[eb] >= 0 && S.es.frame_idx[eb] < p.n_frames);
            mbar_arrive_expect_tx(&S.bar_video, (uint32_t)p.vframe_bytes);
            bulk_load_g2s(s_vframe, p.frames + S.es.frame_idx[eb] * p.vframe_bytes,
                          (uint32_t)p.vframe_bytes, &S.bar_video);
          }
          if (kFloor) {
            // separable floor rays: t = -ez / dz and floor(wy) per row
            // (render.py:321-334)
            const float ez = S.es.ez[eb];
            for (int y = rt; y < p.H; y += kRT) {
              const double dy = s_floor[p.W + y], dz = s_floor[p.W + p.H + y];
              double t = 0.0;
              int kk = -1;  // -1: sky; else parity of floor(wy)
              if (dz < -1e-12) {
                t = (double)(-ez) / dz;
                if ((double)p.cam[13] <= t && t <= (double)p.cam[14]) {
                  const double wy = (double)p.cam[1] + t * dy;
                  kk = (int)(__double2ll_rd(wy) & 1);
                }
              }
              s_ft[y] = t;
              s_fk[y] = kk;
            }
            rbar();
            for (int i = rt; i < npx; i += kRT) {
              const int y = (int)__umulhi((uint32_t)i, p.wmagic);
              const uint32_t db = s_fk[y] >= 0 ? __float_as_uint((float)s_ft[y]) : kInfBits;
              s_z[i] = ((unsigned long long)db << 32) | kBgSub;
            }
          } else {
            const ulonglong2 bg2 = make_ulonglong2(((unsigned long long)kInfBits << 32) | kBgSub,
                                                   ((unsigned long long)kInfBits << 32) | kBgSub);
            for (int i = rt; i < (npx >> 1); i += kRT) reinterpret_cast<ulonglong2 *>(s_z)[i] = bg2;
            if ((npx & 1) && rt == 0) s_z[npx - 1] = bg2.x;
          }
          rbar();
          PIPE_PROF(rt == 0, 9);
        }

        // ---- raster round: (triangle, bbox row) units -> spans -> exact test
        const PTri *s_tri = reinterpret_cast<const PTri *>(smem + L.tri[b]);
        const SpanRec *s_span = reinterpret_cast<const SpanRec *>(smem + L.span[b]);
        const uint32_t *s_rowpre = reinterpret_cast<const uint32_t *>(smem + L.rowpre[b]);
        const uint16_t *s_rowner = reinterpret_cast<const uint16_t *>(smem + L.rowner[b]);
        const int n_round = R.r1 - R.r0;
        const int n_rows = R.n_rows;
        const int n_chunks = (n_rows + 31) >> 5;
        int qn = 0;  // queued spans (warp-uniform)
        bool more = true;
        int kc = rw - kRW;
        while (more) {
          kc += kRW;  // static round-robin over the chunks
          more = kc < n_chunks;
          if (more) {
            const int u = kc * 32 + lane;
            const int o0 = s_rowner[kc];
            const int mi = o0 + 1 + lane;
            uint32_t bit = 0;
            if (mi < n_round) {
              const int d = (int)s_rowpre[mi] - kc * 32;  // >= 1
              if (d < 32) bit = 1u << d;
            }
            const uint32_t starts = __reduce_or_sync(kFull, bit);
            const int j = o0 + __popc(starts & lanemask_le);
            int len = 0, x0 = 0, row = 0;
            if (u < n_rows) {
              PXR_DCHECK(j < n_round && s_rowpre[j] <= (uint32_t)u && s_rowpre[j + 1] > (uint32_t)u);
              const SpanRec &Sp = s_span[j];
              row = (int)Sp.py0 + (u - (int)s_rowpre[j]);
              len = row_span(Sp, row, wlim, x0);
              PXR_DCHECK(row >= 0 && row < p.H);
              PXR_DCHECK(len == 0 || (x0 >= 0 && x0 + len <= p.W && len < 0x10000));
            }
            const uint32_t sm = __ballot_sync(kFull, len > 0);
            if (len > 0)
              q[qn + __popc(sm & lanemask_lt)] =
                  make_uint2((uint32_t)x0 | ((uint32_t)len << 16), (uint32_t)row | ((uint32_t)j << 16));
            qn += __popc(sm);
            PXR_DCHECK(qn <= kQueue);
          }
          while (qn >= 32 || (!more && qn > 0)) {
            __syncwarp();
            const int nb = min(qn, 32);
            qn -= nb;
            int len = 0, x0 = 0, row = 0, j = 0;
            if (lane < nb) {
              const uint2 sp = q[qn + lane];
              x0 = (int)(sp.x & 0xffffu);
              len = (int)(sp.x >> 16);
              row = (int)(sp.y & 0xffffu);
              j = (int)(sp.y >> 16);
            }
            __syncwarp();
            const int incl = warp_incl_scan(len, lane);
            const int excl = incl - len;
            const int N = __shfl_sync(kFull, incl, 31);
            // while spans keep coming only whole rounds of 32 candidates are
            // evaluated; the rest goes back on the queue
            const int NE = more ? (N & ~31) : N;
            for (int c0 = 0; c0 < NE; c0 += 32) {
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
                const uint32_t pix = (uint32_t)(o_row * p.W + px);
                PXR_DCHECK(pix < (uint32_t)npx && o_tri < n_round && owner < 32);
                double z;
                if (eval_exact_pipe(s_tri[o_tri], px, o_row, s_vxy, s_viz, z)) {
                  const float zf = (float)z;
                  const uint32_t li = (uint32_t)(R.r0 + o_tri);
                  const unsigned long long key =
                      ((unsigned long long)__float_as_uint(zf) << 32) |
                      (z < (double)zf ? 0x7FFFFFFFu - li : 0x80000001u + li);
                  unsigned long long old = s_z[pix];
                  while (key < old) {
                    const unsigned long long prev = atomicCAS(&s_z[pix], old, key);
                    if (prev == old) break;
                    old = prev;
                  }
                }
              }
            }
            if (NE < N) {  // (nb == 32 here, so NE >= 32: progress)
              const int skip = max(NE - excl, 0);
              const bool keep = incl > NE;
              const uint32_t km = __ballot_sync(kFull, keep);
              if (keep)
                q[qn + __popc(km & lanemask_lt)] =
                    make_uint2((uint32_t)(x0 + skip) | ((uint32_t)(len - skip) << 16),
                               (uint32_t)row | ((uint32_t)j << 16));
              qn += __popc(km);
              PXR_DCHECK(qn <= kQueue);
            }
          }
        }
        mbar_arrive(&S.bar_empty[b]);  // this thread is done with the round's records
        PIPE_PROF(rt == 0, 10);
        k++;
        last = R.last != 0;
      } while (!last);

      // ---- final pass: resolved words -> final colours -> frame ------------
      rbar();  // every candidate of the env is in
      if (p.mode == PXR_MODE_VIDEO && p.vframe_bulk) {
        mbar_wait_parity(&S.bar_video, vphase);
        vphase ^= 1u;
      }
      const uint8_t *vsrc =
          p.mode == PXR_MODE_VIDEO
              ? (p.vframe_bulk ? s_vframe : p.frames + S.es.frame_idx[eb] * p.vframe_bytes)
              : nullptr;
      uint32_t bpos = 0u, bneg = 0u;
      if (p.mode == PXR_MODE_COLOR) {
        for (int ch = 0; ch < 3; ch++) {
          const int bc = S.es.bias[eb][ch];
          bpos |= (uint32_t)(bc > 0 ? bc : 0) << (8 * ch);
          bneg |= (uint32_t)(bc < 0 ? -bc : 0) << (8 * ch);
        }
      }
      const float ex = S.es.ex[eb];
      uint8_t *gout = p.out + (int64_t)env * p.frame_bytes;
      float *dout = p.out_depth != nullptr ? p.out_depth + (int64_t)env * npx : nullptr;
      for (int pc = rw; pc < n_pchunks; pc += kRW) {
        const int i0 = pc * chunk_px + 4 * lane;  // this lane's 4 pixels
        uint32_t c[4] = {kSkyRGB, kSkyRGB, kSkyRGB, kSkyRGB};
        unsigned long long zw[4];
        if (i0 + 3 < npx) {
          const ulonglong2 a = reinterpret_cast<const ulonglong2 *>(s_z)[i0 >> 1];
          const ulonglong2 bq = reinterpret_cast<const ulonglong2 *>(s_z)[(i0 >> 1) + 1];
          zw[0] = a.x; zw[1] = a.y; zw[2] = bq.x; zw[3] = bq.y;
        } else {
#pragma unroll
          for (int j = 0; j < 4; j++)
            zw[j] = i0 + j < npx ? s_z[i0 + j] : (((unsigned long long)kInfBits << 32) | kBgSub);
        }
        bool all_bg = true;
#pragma unroll
        for (int j = 0; j < 4; j++) all_bg = all_bg && (uint32_t)zw[j] == kBgSub;
        const int y0g = (int)__umulhi((uint32_t)i0, p.wmagic);
        if (all_bg && plan_ok && !kFloor && i0 + 3 < npx) {
          // 4 sky pixels of one row under video: three texel words through
          // the byte-permute plan (W % 4 == 0)
          const int x0g = i0 - y0g * p.W;
          const uint4 pl = s_gplan[x0g >> 2];
          const uint32_t *src =
              reinterpret_cast<const uint32_t *>(s_vframe + s_rowmap[y0g]) + pl.x;
          const uint32_t *w0 = src + (pl.y >> 16), *w1 = src + (pl.z >> 16),
                         *w2 = src + (pl.w >> 16);
          PXR_DCHECK(4u * (uint32_t)(w2 + 1 - reinterpret_cast<const uint32_t *>(s_vframe)) + 4u <=
                     (uint32_t)p.vframe_bytes + 32u);
          stage[3 * lane + 0] = __byte_perm(w0[0], w0[1], pl.y & 0xffffu);
          stage[3 * lane + 1] = __byte_perm(w1[0], w1[1], pl.z & 0xffffu);
          stage[3 * lane + 2] = __byte_perm(w2[0], w2[1], pl.w & 0xffffu);
        } else {
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int i = i0 + j;
            if (i >= npx) break;
            const uint32_t sub = (uint32_t)zw[j];
            if (sub != kBgSub) {  // the sequential winner's flat colour
              const uint32_t li = sub < kBgSub ? 0x7FFFFFFFu - sub : sub - 0x80000001u;
              PXR_DCHECK(li < (uint32_t)p.nt);
              c[j] = s_rgb[li];
            } else {
              const int y = (int)__umulhi((uint32_t)i, p.wmagic), x = i - y * p.W;
              const uint32_t db = (uint32_t)(zw[j] >> 32);
              if (kFloor && db != kInfBits) {  // checker floor (render.py:326-344)
                const double t = s_ft[y];
                const double wx = (double)ex + t * s_floor[x];
                c[j] = (((uint32_t)__double2ll_rd(wx) ^ (uint32_t)s_fk[y]) & 1u ? 122u : 158u) *
                       0x010101u;
              } else if (p.mode == PXR_MODE_VIDEO) {  // distractor.py:172-176
                PXR_DCHECK(s_rowmap[y] + s_colmap[x] + 3u <= (uint32_t)p.vframe_bytes);
                const uint8_t *t = vsrc + s_rowmap[y] + s_colmap[x];
                c[j] = (uint32_t)t[0] | ((uint32_t)t[1] << 8) | ((uint32_t)t[2] << 16);
              }
            }
            if (p.mode == PXR_MODE_COLOR) c[j] = __vsubus4(__vaddus4(c[j], bpos), bneg);
          }
          if (p.gray) {  // env.py:168-173
            uint32_t g4 = 0u;
#pragma unroll
            for (int j = 0; j < 4; j++)
              g4 |= ((299u * (c[j] & 0xffu) + 587u * ((c[j] >> 8) & 0xffu) +
                      114u * ((c[j] >> 16) & 0xffu) + 500u) / 1000u) << (8 * j);
            stage[lane] = g4;
          } else {
            stage[3 * lane + 0] = c[0] | (c[1] << 24);
            stage[3 * lane + 1] = (c[1] >> 8) | (c[2] << 16);
            stage[3 * lane + 2] = (c[2] >> 16) | (c[3] << 8);
          }
        }
        if (dout != nullptr) {
          if (p.depth_vec && i0 + 3 < npx) {
            reinterpret_cast<float4 *>(dout)[i0 >> 2] =
                make_float4(__uint_as_float((uint32_t)(zw[0] >> 32)),
                            __uint_as_float((uint32_t)(zw[1] >> 32)),
                            __uint_as_float((uint32_t)(zw[2] >> 32)),
                            __uint_as_float((uint32_t)(zw[3] >> 32)));
          } else {
            for (int j = 0; j < 4 && i0 + j < npx; j++)
              dout[i0 + j] = __uint_as_float((uint32_t)(zw[j] >> 32));
          }
        }
        __syncwarp();
        // the warp's 128 pixels are contiguous in the frame: coalesced 16-byte
        // stores (or bytes for a ragged tail / unaligned output)
        const int cbyte0 = pc * chunk_px * chans;
        const int nbytes = min(chunk_px * chans, p.frame_bytes - cbyte0);
        if (p.use_bulk && (nbytes & 15) == 0) {
          if (lane * 16 < nbytes)
            reinterpret_cast<uint4 *>(gout + cbyte0)[lane] = reinterpret_cast<const uint4 *>(stage)[lane];
        } else {
          const uint8_t *sb = reinterpret_cast<const uint8_t *>(stage);
          for (int i = lane; i < nbytes; i += 32) gout[cbyte0 + i] = sb[i];
        }
        __syncwarp();
      }
      mbar_arrive(&S.bar_env[eb]);  // done with this parity's vertex / colour set
      PIPE_PROF(rt == 0, 11);
    }
    if (p.prof != nullptr && rt == 0) S.prof[12] = clock64() - prof_t0;
  }
  if (p.prof != nullptr) {
    __syncthreads();
    if (tid < 16) p.prof[blockIdx.x * 16 + tid] = S.prof[tid];
  }
}

template __global__ void render_pipe_kernel<false>(const RenderParams p);
template __global__ void render_pipe_kernel<true>(const RenderParams p);

// Host side: budgets, layout and launch of the pipelined kernel. Returns
// PXR_OK with *launched = false when the configuration does not fit it (the
// caller then takes render_step_kernel).
pxr_status render_pipe_launch(RenderParams p, const DeviceFacts &dev, int debug_cap,
                              int debug_row_cap, int64_t debug_grid, cudaStream_t st,
                              bool *launched) {
  *launched = false;
  if (p.draw_floor && !p.floor_sep) return PXR_OK;  // general floor: per-pixel rays
  const int budget = dev.max_smem_optin - (int)sizeof(PipeShared) - 256;
  p.row_cap = kPipeRowCap > p.H ? kPipeRowCap : p.H;
  if (debug_row_cap > 0) p.row_cap = debug_row_cap > p.H ? debug_row_cap : p.H;
  int cap = p.nt > 0 ? (p.nt < kMaxCap ? p.nt : kMaxCap) : 1;
  if (debug_cap > 0 && debug_cap < cap) cap = debug_cap;
  for (;;) {
    p.cap = cap;
    if (pipe_layout(p).total <= budget) break;
    if (cap <= 32) return PXR_OK;  // too little room for records
    cap = cap > 64 ? cap - 16 : cap - 8;
  }
  const int smem = pipe_layout(p).total;
  auto kernel = p.draw_floor ? render_pipe_kernel<true> : render_pipe_kernel<false>;
  int per_sm = 1;
  const pxr_status os = kernel_occupancy((const void *)kernel, kThreads, smem, &per_sm);
  if (os != PXR_OK) return os;
  int64_t grid = (int64_t)dev.num_sms * per_sm;
  if (debug_grid > 0 && debug_grid < grid) grid = debug_grid;
  if (grid > p.batch) grid = p.batch;
  kernel<<<(unsigned)grid, kThreads, smem, st>>>(p);
  *launched = true;
  return check_launch("render_pipe_kernel");
}

}  // namespace pxr

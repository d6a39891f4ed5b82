// Standalone launches of the hot path's pieces, mirroring the reference's
// individual numba kernels / numpy helpers one-to-one so the Python layer can
// replace each reference call in place (the fused path is pxr_render.cu):
//   distractor.py:82-113  init_distractors       -> pxr_init_distractors
//   distractor.py:116-137 advance_distractors    -> pxr_advance_distractors
//   distractor.py:140-161 _color_kernel          -> pxr_apply_color
//   distractor.py:164-176 _video_kernel          -> pxr_apply_video
//   env.py:168-173        _postprocess grayscale -> pxr_grayscale
//   prng.py:57-77,168-178 threefry / fold_in_many / words_per_key -> pxr_threefry2x64
//   physics.py:114-137    forward_kinematics     -> pxr_forward_kinematics
// plus the benchmark's on-device pose source.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"
#include "pxr_glibc_sincos.cuh"
#include "pxr_numpy_log.cuh"
#include "pxr_math.cuh"

namespace pxr {

static thread_local char g_last_error[256] = "";

void set_last_error(const char *msg) {
  snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
}

pxr_status set_cuda(cudaError_t e, const char *where) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
  return PXR_ERR_CUDA;
}

// ---- debug knobs ------------------------------------------------------------
static const char *const kKnobNames[kDbgCount] = {
    "PXR_DEBUG_FRAG_LIMIT", "PXR_DEBUG_ROW_CAP",        "PXR_DEBUG_CAP",  "PXR_DEBUG_STATS_PTR",
    "PXR_DEBUG_BAND_H",     "PXR_DEBUG_NO_PACKED_SCAN", "PXR_DEBUG_PHYS", "PXR_DEBUG_GRID",
    "PXR_DEBUG_PROF",       "PXR_DEBUG_NO_UPSCALE",
    "PXR_DEBUG_NO_PDL",     "PXR_DEBUG_NO_SPLIT"};
static std::mutex g_knob_mu;
static std::string g_knob_val[kDbgCount];
static bool g_knob_set[kDbgCount];
static bool g_knob_init = false;

static void knobs_init_locked() {
  if (g_knob_init) return;
  for (int i = 0; i < kDbgCount; i++) {
    const char *s = getenv(kKnobNames[i]);
    g_knob_set[i] = s != nullptr;
    g_knob_val[i] = s != nullptr ? s : "";
  }
  g_knob_init = true;
}

const char *debug_knob(int id) {
  std::lock_guard<std::mutex> g(g_knob_mu);
  knobs_init_locked();
  return g_knob_set[id] ? g_knob_val[id].c_str() : nullptr;
}

// ---- per-device facts and the launch-configuration cache ------------------
static std::mutex g_dev_mu;
static DeviceFacts g_dev[64];
static bool g_dev_ok[64];

const DeviceFacts &device_facts() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (!g_dev_ok[dev]) {
    DeviceFacts f{dev, 0, 0};
    cudaDeviceGetAttribute(&f.num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&f.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (f.num_sms <= 0) f.num_sms = 148;
    g_dev[dev] = f;
    g_dev_ok[dev] = true;
  }
  return g_dev[dev];
}

struct OccEntry {
  const void *kernel;
  int device, threads, smem, per_sm;
};
static std::vector<OccEntry> g_occ;
static std::vector<std::pair<std::pair<const void *, int>, int>> g_attr;  // (kernel, dev) -> smem set

pxr_status kernel_occupancy(const void *kernel, int threads, int smem, int *per_sm) {
  const int dev = device_facts().device;
  std::lock_guard<std::mutex> g(g_dev_mu);
  for (const OccEntry &e : g_occ)
    if (e.kernel == kernel && e.device == dev && e.threads == threads && e.smem == smem) {
      *per_sm = e.per_sm;
      return PXR_OK;
    }
  int *set = nullptr;
  for (auto &a : g_attr)
    if (a.first.first == kernel && a.first.second == dev) set = &a.second;
  if (set == nullptr || *set < smem) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda(e, "cudaFuncSetAttribute");
    if (set != nullptr) *set = smem;
    else g_attr.push_back({{kernel, dev}, smem});
  }
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (e != cudaSuccess) return set_cuda(e, "occupancy query");
  if (n < 1) n = 1;
  g_occ.push_back({kernel, dev, threads, smem, n});
  *per_sm = n;
  return PXR_OK;
}

static inline unsigned blocks_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 1048576) b = 1048576;  // grid-stride loops cover the rest
  return (unsigned)b;
}

__global__ void init_distractors_kernel(pxr_distractor d, const int64_t *counts, int64_t n_videos,
                                        int64_t batch, uint64_t khi, uint64_t klo,
                                        uint64_t env_offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < batch;
       i += (int64_t)gridDim.x * blockDim.x) {
    // keys = split(key, off + B)[off:] -> TF(key, (g, 1))  (distractor.py:96)
    uint64_t hi, lo;
    threefry2x64(khi, klo, env_offset + (uint64_t)i, 1, hi, lo);
    if (d.mode == PXR_MODE_COLOR) {
      int16_t b3[3];
      color_bias_from_key(hi, lo, b3);
      for (int c = 0; c < 3; c++) d.color_bias[i * 3 + c] = b3[c];
    } else {
      uint64_t w0, w1;
      threefry2x64(hi, lo, 2, 0, w0, w1);  // sample_video_indices, distractor.py:77-79
      const int64_t vid = index_from_word(w0, (uint64_t)n_videos);
      d.video_index[i] = vid;
      d.frame_cursor[i] = 0;
      d.direction[i] = 1;
      d.frame_count[i] = counts[vid];
      if (d.color_bias != nullptr)
        for (int c = 0; c < 3; c++) d.color_bias[i * 3 + c] = 0;
    }
  }
}

__global__ void advance_distractors_kernel(pxr_distractor d, const int64_t *counts,
                                           int64_t n_videos, int64_t batch, uint64_t khi,
                                           uint64_t klo, uint64_t env_offset, uint64_t lb,
                                           const uint8_t *done) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < batch;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = env_offset + (uint64_t)i;
    if (d.mode == PXR_MODE_COLOR) {
      uint64_t ehi, elo;
      threefry2x64(khi, klo, g, 2, ehi, elo);  // fold_in_many(key_t, off + arange)
      int16_t b3[3];
      color_bias_from_key(ehi, elo, b3);
      for (int c = 0; c < 3; c++) d.color_bias[i * 3 + c] = b3[c];
    } else if (d.mode == PXR_MODE_VIDEO) {
      int dir = d.direction[i];
      const int64_t cnt = d.frame_count[i];
      int64_t nxt = d.frame_cursor[i] + dir;
      const bool hi_end = nxt >= cnt, lo_end = nxt < 0;
      if (hi_end) { nxt = cnt - 2; dir = -1; }
      if (lo_end) { nxt = 1; dir = 1; }
      if (done != nullptr && done[i]) {  // env.py:239-244
        uint64_t rhi, rlo, w0, w1;
        threefry2x64(khi, klo, lb + g, 2, rhi, rlo);
        threefry2x64(rhi, rlo, 2, 0, w0, w1);
        const int64_t vid = index_from_word(w0, (uint64_t)n_videos);
        d.video_index[i] = vid;
        d.frame_count[i] = counts[vid];
        nxt = 0;
        dir = 1;
      }
      d.frame_cursor[i] = nxt;
      d.direction[i] = (int8_t)dir;
    }
  }
}

// 16 bytes (5 1/3 pixels) per thread would split pixels; use 12-byte groups
// of 4 pixels when aligned, which is the common 84x84 case.
__global__ void apply_color_kernel(uint8_t *pixels, const int16_t *bias, int64_t batch,
                                   int64_t npx) {
  const int64_t total = batch * npx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / npx;
    uint8_t *px = pixels + i * 3;
    for (int c = 0; c < 3; c++) {
      const int v = (int)px[c] + (int)bias[b * 3 + c];
      px[c] = (uint8_t)min(255, max(0, v));
    }
  }
}

__global__ void apply_video_kernel(uint8_t *pixels, const float *depth, pxr_video_pack pk,
                                   const int64_t *video_index, const int64_t *frame_cursor,
                                   int64_t batch, int H, int W) {
  const int64_t npx = (int64_t)H * W;
  const int64_t total = batch * npx;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!isinf(depth[i])) continue;
    const int64_t b = i / npx;
    const int64_t r = i - b * npx;
    const int y = (int)(r / W), x = (int)(r - (int64_t)y * W);
    const int64_t fi = pk.starts[video_index[b]] + frame_cursor[b];
    const int sy = (int)(((int64_t)y * pk.height) / H);
    const int sx = (int)(((int64_t)x * pk.width) / W);
    const uint8_t *src = pk.frames + ((fi * pk.height + sy) * pk.width + sx) * 3;
    pixels[i * 3 + 0] = src[0];
    pixels[i * 3 + 1] = src[1];
    pixels[i * 3 + 2] = src[2];
  }
}

__global__ void grayscale_kernel(const uint8_t *rgb, uint8_t *gray, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
    gray[i] = (uint8_t)((299u * r + 587u * g + 114u * b + 500u) / 1000u);
  }
}

__global__ void threefry_kernel(const uint64_t *k0, const uint64_t *k1, int64_t ks,
                                const uint64_t *c0, const uint64_t *c1, int64_t c1s,
                                uint64_t *y0, uint64_t *y1, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t a, b;
    threefry2x64(k0[i * ks], k1[i * ks], c0[i], c1[i * c1s], a, b);
    y0[i] = a;
    y1[i] = b;
  }
}

__global__ void sincosf_kernel(const float *x, float *s, float *c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    s[i] = glibc_sincosf(v, 0);
    c[i] = glibc_sincosf(v, 1);
  }
}

// physics.py:114-137, one thread per env, f64, with glibc's cos / sin
// (pxr_glibc_sincos.cuh): bit-identical to the reference's numpy FK.
__device__ __forceinline__ void fk_one(const double *q, const int32_t *parent,
                                       const double *adist, int nl, double *out) {
  out[0] = q[0];
  out[1] = q[1];
  out[2] = q[2];
  for (int i = 1; i < nl; i++) {
    const int pp = parent[i];
    const double th = out[3 * pp + 2];
    out[3 * i + 0] = out[3 * pp + 0] + adist[i] * glibc_cos(th);
    out[3 * i + 1] = out[3 * pp + 1] + adist[i] * glibc_sin(th);
    out[3 * i + 2] = th + q[3 + i - 1];
  }
}

__global__ void fk_kernel(const double *qpos, const int32_t *parent, const double *adist,
                          int nl, int64_t batch, double *poses) {
  pdl_trigger();  // the render launch that follows may be scheduled now
  const int dof = 3 + nl - 1;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x)
    fk_one(qpos + b * dof, parent, adist, nl, poses + b * nl * 3);
}

// Benchmark pose source: qpos0 = rest + U(-0.1, 0.1) with the reference's
// reset keys (physics.py:499-503: k_g = TF(R, (g, 1)), draws from
// fold_in(k_g, 0)), then a deterministic oscillation per joint inside a
// +-0.6 rad band around rest, root x advancing at 1 m/s, root z bobbing.
__global__ void pose_source_kernel(const double *rest, const int32_t *parent,
                                   const double *adist, int nl, uint64_t rhi, uint64_t rlo,
                                   uint64_t env_offset, int64_t t, int64_t batch,
                                   double *poses) {
  pdl_trigger();  // the render launch that follows may be scheduled now
  constexpr int kMaxDof = 3 + 63;
  const int dof = 3 + nl - 1;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = env_offset + (uint64_t)b;
    uint64_t khi, klo, fhi, flo;
    threefry2x64(rhi, rlo, g, 1, khi, klo);   // split(reset_key, .)[g]
    threefry2x64(khi, klo, 0, 2, fhi, flo);   // fold_in(k_g, 0)
    double q[kMaxDof];
    for (int d = 0; d < dof; d += 2) {        // random_bits blocks (prng.py:111-121)
      uint64_t w0, w1;
      threefry2x64(fhi, flo, (uint64_t)(d / 2), 0, w0, w1);
      const uint64_t w[2] = {w0, w1};
      for (int k = 0; k < 2 && d + k < dof; k++) {
        const double u = (double)(w[k] >> 11) * 0x1p-53;  // prng.py:132-135
        q[d + k] = rest[d + k] + (-0.1 + u * 0.2);
      }
    }
    const double time = 0.01 * (double)t;
    const double phase = (double)(g % 997) * 0.37;
    q[0] += time;                                  // root advances
    q[1] += 0.03 * glibc_sin(6.0 * time + phase);        // bob
    q[2] += 0.05 * glibc_sin(4.0 * time + phase);        // pitch rock
    for (int j = 3; j < dof; j++)
      q[j] += 0.6 * glibc_sin(8.0 * time + phase + 1.3 * j);
    fk_one(q, parent, adist, nl, poses + b * nl * 3);
  }
}

// key_t = fold_in(master, t) = TF(master, (t, 2)) (prng.py:105-108), t += 1
__global__ void step_key_kernel(uint64_t mhi, uint64_t mlo, int64_t *t, uint64_t *key_out) {
  const int64_t tt = *t;
  uint64_t hi, lo;
  threefry2x64(mhi, mlo, (uint64_t)tt, 2, hi, lo);
  key_out[0] = hi;
  key_out[1] = lo;
  *t = tt + 1;
}

}  // namespace pxr

using namespace pxr;

extern "C" int32_t pxr_abi_version(void) { return PXR_ABI_VERSION; }

extern "C" int32_t pxr_build_checked(void) {
#ifdef PXR_CHECKED
  return 1;
#else
  return 0;
#endif
}

extern "C" const char *pxr_status_string(pxr_status s) {
  switch (s) {
    case PXR_OK: return "ok";
    case PXR_ERR_INVALID: return "invalid argument";
    case PXR_ERR_CUDA: return "CUDA error";
    case PXR_ERR_UNSUPPORTED: return "unsupported shape";
    default: return "unknown status";
  }
}

extern "C" const char *pxr_last_error(void) { return g_last_error; }

extern "C" pxr_status pxr_set_debug(const char *name, const char *value) {
  if (name == nullptr) return set_invalid("pxr_set_debug: null name");
  std::lock_guard<std::mutex> g(g_knob_mu);
  knobs_init_locked();
  for (int i = 0; i < kDbgCount; i++)
    if (strcmp(name, kKnobNames[i]) == 0) {
      g_knob_set[i] = value != nullptr;
      g_knob_val[i] = value != nullptr ? value : "";
      return PXR_OK;
    }
  return set_invalid("pxr_set_debug: unknown knob");
}

extern "C" pxr_status pxr_init_distractors(const pxr_distractor *dist,
                                           const pxr_video_pack *pack, int64_t batch,
                                           uint64_t key_hi, uint64_t key_lo,
                                           uint64_t env_offset, void *stream) {
  if (dist == nullptr) return set_invalid("null distractor state");
  if (batch < 1) return set_invalid("batch must be >= 1");
  if (dist->mode == PXR_MODE_NONE) return PXR_OK;
  if (dist->mode == PXR_MODE_COLOR) {
    if (dist->color_bias == nullptr) return set_invalid("colour mode needs color_bias");
  } else if (dist->mode == PXR_MODE_VIDEO) {
    if (pack == nullptr || pack->counts == nullptr || pack->n_videos < 1)
      return set_invalid("video distractors need a loaded video pack");
    if (dist->video_index == nullptr || dist->frame_cursor == nullptr ||
        dist->direction == nullptr || dist->frame_count == nullptr)
      return set_invalid("video mode needs the full distractor state");
  } else {
    return set_invalid("unknown distractor mode");
  }
  const int64_t nv = dist->mode == PXR_MODE_VIDEO ? pack->n_videos : 1;
  const int64_t *counts = dist->mode == PXR_MODE_VIDEO ? pack->counts : nullptr;
  init_distractors_kernel<<<blocks_for(batch, 256), 256, 0, (cudaStream_t)stream>>>(
      *dist, counts, nv, batch, key_hi, key_lo, env_offset);
  return check_launch("init_distractors_kernel");
}

extern "C" pxr_status pxr_advance_distractors(const pxr_distractor *dist,
                                              const pxr_video_pack *pack, int64_t batch,
                                              const pxr_step_keys *keys, const uint8_t *done,
                                              void *stream) {
  if (dist == nullptr || keys == nullptr) return set_invalid("null state/keys");
  if (keys->device_key != nullptr)
    return set_unsupported("pxr_advance_distractors takes host keys (device_key: pxr_render_step)");
  if (batch < 1) return set_invalid("batch must be >= 1");
  if (dist->mode == PXR_MODE_NONE) return PXR_OK;
  if (dist->mode == PXR_MODE_COLOR && dist->color_bias == nullptr)
    return set_invalid("colour mode needs color_bias");
  if (dist->mode == PXR_MODE_VIDEO) {
    // The pack (its per-video frame counts) is only needed to re-draw the
    // video of envs that are being reset.
    if (done != nullptr && (pack == nullptr || pack->counts == nullptr || pack->n_videos < 1))
      return set_invalid("video distractors need a loaded video pack");
    if (dist->video_index == nullptr || dist->frame_cursor == nullptr ||
        dist->direction == nullptr || dist->frame_count == nullptr)
      return set_invalid("video mode needs the full distractor state");
  }
  if (dist->mode != PXR_MODE_COLOR && dist->mode != PXR_MODE_VIDEO)
    return set_invalid("unknown distractor mode");
  const bool have_pack = dist->mode == PXR_MODE_VIDEO && pack != nullptr;
  const int64_t nv = have_pack ? pack->n_videos : 1;
  const int64_t *counts = have_pack ? pack->counts : nullptr;
  advance_distractors_kernel<<<blocks_for(batch, 256), 256, 0, (cudaStream_t)stream>>>(
      *dist, counts, nv, batch, keys->key_hi, keys->key_lo, keys->env_offset,
      keys->logical_batch, done);
  return check_launch("advance_distractors_kernel");
}

extern "C" pxr_status pxr_apply_color(uint8_t *pixels, const int16_t *bias, int64_t batch,
                                      int64_t height, int64_t width, void *stream) {
  if (pixels == nullptr || bias == nullptr) return set_invalid("null pixels/bias");
  if (batch < 1 || height < 1 || width < 1) return set_invalid("bad frame shape");
  const int64_t npx = height * width;
  apply_color_kernel<<<blocks_for(batch * npx, 256), 256, 0, (cudaStream_t)stream>>>(
      pixels, bias, batch, npx);
  return check_launch("apply_color_kernel");
}

extern "C" pxr_status pxr_apply_video(uint8_t *pixels, const float *depth,
                                      const pxr_video_pack *pack, const int64_t *video_index,
                                      const int64_t *frame_cursor, int64_t batch,
                                      int64_t height, int64_t width, void *stream) {
  if (pixels == nullptr || depth == nullptr || video_index == nullptr ||
      frame_cursor == nullptr)
    return set_invalid("null pixels/depth/state");
  if (pack == nullptr || pack->frames == nullptr || pack->starts == nullptr)
    return set_invalid("video distractors need a loaded video pack");
  if (batch < 1 || height < 1 || width < 1) return set_invalid("bad frame shape");
  apply_video_kernel<<<blocks_for(batch * height * width, 256), 256, 0,
                       (cudaStream_t)stream>>>(pixels, depth, *pack, video_index,
                                               frame_cursor, batch, (int)height, (int)width);
  return check_launch("apply_video_kernel");
}

extern "C" pxr_status pxr_grayscale(const uint8_t *rgb, uint8_t *gray, int64_t n_pixels,
                                    void *stream) {
  if (rgb == nullptr || gray == nullptr || n_pixels < 0) return set_invalid("bad grayscale args");
  if (n_pixels == 0) return PXR_OK;
  grayscale_kernel<<<blocks_for(n_pixels, 256), 256, 0, (cudaStream_t)stream>>>(rgb, gray,
                                                                               n_pixels);
  return check_launch("grayscale_kernel");
}

extern "C" pxr_status pxr_threefry2x64(const uint64_t *k0, const uint64_t *k1,
                                       int64_t key_stride, const uint64_t *c0,
                                       const uint64_t *c1, int64_t c1_stride, uint64_t *y0,
                                       uint64_t *y1, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (k0 == nullptr || k1 == nullptr || c0 == nullptr || c1 == nullptr ||
                          y0 == nullptr || y1 == nullptr)))
    return set_invalid("bad threefry args");
  if (n == 0) return PXR_OK;
  threefry_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
      k0, k1, key_stride ? 1 : 0, c0, c1, c1_stride ? 1 : 0, y0, y1, n);
  return check_launch("threefry_kernel");
}

extern "C" pxr_status pxr_step_key_advance(uint64_t master_hi, uint64_t master_lo, int64_t *t,
                                           uint64_t *key_out, void *stream) {
  if (t == nullptr || key_out == nullptr) return set_invalid("pxr_step_key_advance: null argument");
  step_key_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(master_hi, master_lo, t, key_out);
  return check_launch("step_key_kernel");
}

__global__ void pack_upscale_kernel(const uint8_t *frames, int64_t n_frames, int Hv, int Wv,
                                    int H, int W, uint8_t *out) {
  const int64_t n = n_frames * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = i / ((int64_t)H * W);
    const int r = (int)(i - f * H * W), y = r / W, x = r - y * W;
    const uint8_t *src = frames + ((f * Hv + ((int64_t)y * Hv) / H) * Wv + ((int64_t)x * Wv) / W) * 3;
    out[i * 3 + 0] = src[0];
    out[i * 3 + 1] = src[1];
    out[i * 3 + 2] = src[2];
  }
}

extern "C" pxr_status pxr_pack_upscale(const pxr_video_pack *pack, int64_t height, int64_t width,
                                       uint8_t *out, void *stream) {
  if (pack == nullptr || pack->frames == nullptr || out == nullptr)
    return set_invalid("pxr_pack_upscale: null pointers");
  if (height < 1 || width < 1 || pack->height < 1 || pack->width < 1 || pack->n_frames < 0)
    return set_invalid("pxr_pack_upscale: bad sizes");
  if (pack->n_frames == 0) return PXR_OK;
  pack_upscale_kernel<<<blocks_for(pack->n_frames * height * width, 256), 256, 0,
                        (cudaStream_t)stream>>>(pack->frames, pack->n_frames, (int)pack->height,
                                                (int)pack->width, (int)height, (int)width, out);
  return check_launch("pack_upscale_kernel");
}

extern "C" pxr_status pxr_sincosf(const float *x, float *s, float *c, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (x == nullptr || s == nullptr || c == nullptr)))
    return set_invalid("bad sincosf args");
  if (n == 0) return PXR_OK;
  sincosf_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, s, c, n);
  return check_launch("sincosf_kernel");
}

__global__ void sincos64_kernel(const double *x, double *s, double *c, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    s[i] = glibc_sin(v);
    c[i] = glibc_cos(v);
  }
}

__global__ void log64_kernel(const double *x, double *y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = numpy_log(x[i]);
}

extern "C" pxr_status pxr_log(const double *x, double *y, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (x == nullptr || y == nullptr))) return set_invalid("bad log args");
  if (n == 0) return PXR_OK;
  log64_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, y, n);
  return check_launch("log64_kernel");
}

extern "C" pxr_status pxr_sincos(const double *x, double *s, double *c, int64_t n, void *stream) {
  if (n < 0 || (n > 0 && (x == nullptr || s == nullptr || c == nullptr)))
    return set_invalid("bad sincos args");
  if (n == 0) return PXR_OK;
  sincos64_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(x, s, c, n);
  return check_launch("sincos64_kernel");
}

extern "C" pxr_status pxr_forward_kinematics(const double *qpos, const int32_t *parent,
                                             const double *anchor_dist, int32_t n_links,
                                             int64_t batch, double *poses, void *stream) {
  if (qpos == nullptr || parent == nullptr || anchor_dist == nullptr || poses == nullptr)
    return set_invalid("null FK args");
  if (n_links < 1 || n_links > 64 || batch < 1) return set_invalid("bad FK sizes");
  fk_kernel<<<blocks_for(batch, 128), 128, 0, (cudaStream_t)stream>>>(qpos, parent, anchor_dist,
                                                                      n_links, batch, poses);
  return check_launch("fk_kernel");
}

extern "C" pxr_status pxr_pose_source(const double *rest_qpos, const int32_t *parent,
                                      const double *anchor_dist, int32_t n_links,
                                      uint64_t reset_key_hi, uint64_t reset_key_lo,
                                      uint64_t env_offset, int64_t t, int64_t batch,
                                      double *poses, void *stream) {
  if (rest_qpos == nullptr || parent == nullptr || anchor_dist == nullptr || poses == nullptr)
    return set_invalid("null pose-source args");
  if (n_links < 1 || n_links > 64 || batch < 1) return set_invalid("bad pose-source sizes");
  pose_source_kernel<<<blocks_for(batch, 128), 128, 0, (cudaStream_t)stream>>>(
      rest_qpos, parent, anchor_dist, n_links, reset_key_hi, reset_key_lo, env_offset, t, batch,
      poses);
  return check_launch("pose_source_kernel");
}

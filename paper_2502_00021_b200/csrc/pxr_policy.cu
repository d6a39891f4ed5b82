// Conv-stub policy forward: the reference's fixed
// action-selection surrogate (bench.py:36-145): conv 16 x 8x8 stride 4 over
// obs / 255, ReLU, linear projection of the (oy, ox, f)-ordered features,
// tanh.
//
// Two kernels. The convolution runs on the 5th-generation tensor cores
// (tcgen05.mma kind::f16, accumulator in TMEM, frames by double-buffered TMA
// bulk copies): obs bytes are exact in bf16 and the f32 weights are split
// into three bf16 parts, so the products are exact and only the f32
// accumulation rounds. It writes the ReLU'd features to a workspace; the
// projection (one warp per env, proj tiles in shared memory shared by 8
// envs) reduces them in a fixed order. Each batch row is computed by the
// same instructions in the same order whatever batch it is in (reference
// tests/test_bench.py:92-98), within 1e-5 of a float64 evaluation.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"

namespace pxr {

constexpr int kK = 8, kS = 4, kF = 16;
constexpr int kMaxJoints = 32;

// Projection + tanh: one warp per env; lane l accumulates the features
// k = l, l + 32, ... in ascending order against tiles of proj staged in
// shared memory (shared by the CTA's kProjEnvs envs), then a fixed xor tree
// -- the same arithmetic for a row whatever batch it is in.
// ---- tensor-core convolution (tcgen05, BF16 in, F32 accumulate in TMEM) ----
// Per env and per tile of 128 output positions: D[128 x 48] = A[128 x K] *
// B[48 x K]^T with K = 64 C in steps of 16. A is the im2col of the raw obs
// bytes (0..255, exact in bf16); B holds the f32 weights split into three
// bf16 parts w = w1 + w2 + w3 (24 significant bits), columns n = split*16 + f.
// The products are exact and accumulate in f32; the epilogue adds the three
// splits in a fixed order, scales by float32(1/255) and applies the ReLU.
// Operands use the K-major no-swizzle canonical layout: 8-row x 16-byte core
// matrices, LBO = 128 B between the two 8-element K halves, SBO = 256 B
// between 8-row groups. One thread issues the MMAs; tcgen05.commit arrives
// on an mbarrier the CTA waits on before reading TMEM.
// Each frame is converted to bf16 ONCE (the 8x8 stride-4 windows overlap, so
// an im2col straight from the bytes would convert every byte ~4 times) and
// the A tiles are then built by 16-byte copies from that bf16 frame. One
// 16-warp CTA per SM (frames + bf16 frame + operands fill shared memory).
constexpr int kTcThreads = 512;
constexpr int kTcM = 128, kTcN = 48;

__device__ __forceinline__ uint32_t tc_off(int row, int k, int step_bytes) {
  return (uint32_t)((k >> 4) * step_bytes + (row >> 3) * 256 + ((k >> 3) & 1) * 128 +
                    (row & 7) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ uint32_t bf16x2_of_bytes(uint32_t b0, uint32_t b1) {
  const float f0 = __int_as_float(0x4B000000 | b0) - 8388608.0f;  // exact integers
  const float f1 = __int_as_float(0x4B000000 | b1) - 8388608.0f;
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f1), "f"(f0));
  return r;
}

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  uint16_t r;
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float bf16_val(uint16_t h) {
  return __uint_as_float((uint32_t)h << 16);
}

__global__ void __launch_bounds__(kTcThreads)
conv_feat_tc_kernel(const uint8_t *__restrict__ obs, int64_t batch, int H, int W, int C,
                    const float *__restrict__ conv, float *__restrict__ feat, int bulk,
                    int use_fb) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int K = kK * kK * C;           // 64 C, a multiple of 16
  const int a_step = (kTcM / 8) * 256;  // bytes per 16-wide K step of A
  const int b_step = (kTcN / 8) * 256;
  unsigned char *s_a = sm;
  unsigned char *s_b = s_a + (K / 16) * a_step;
  uint8_t *s_obs0 = s_b + (K / 16) * b_step;
  const int frame = H * W * C;
  const int fstride = (frame + 15) & ~15;
  const int oh = (H - kK) / kS + 1, ow = (W - kK) / kS + 1, n_pos = oh * ow;
  int *s_posoff = reinterpret_cast<int *>(s_obs0 + 2 * fstride);  // window start per position
  uint16_t *s_fb = reinterpret_cast<uint16_t *>(reinterpret_cast<unsigned char *>(s_posoff) +
                                                ((4 * n_pos + 15) & ~15));  // bf16 frame (use_fb)
  __shared__ uint64_t s_bar[3];  // frame buffers 0 / 1, MMA completion
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float inv = 1.0f / 255.0f;  // float32(1/255), bench.py:101

  // element offset of each output position's window in the frame
  for (int pos = tid; pos < n_pos; pos += kTcThreads) {
    const int oy = pos / ow, ox = pos - oy * ow;
    s_posoff[pos] = (oy * kS * W + ox * kS) * C;
  }
  // every 8-element chunk starts 8-byte aligned in the bf16 frame when W C is
  // a multiple of 4 (window starts are multiples of 4 C elements)
  const bool chunk_aligned = ((W * C) & 3) == 0;
  // B: the three bf16 splits of every weight, K-major
  for (int i = tid; i < K * kF; i += kTcThreads) {
    const int k = i / kF, f = i - k * kF;
    const float w = conv[i];
    const uint16_t h1 = bf16_bits(w);
    const float r1 = w - bf16_val(h1);
    const uint16_t h2 = bf16_bits(r1);
    const uint16_t h3 = bf16_bits(r1 - bf16_val(h2));
    PXR_DCHECK(tc_off(32 + f, k, b_step) + 2u <= (uint32_t)((K / 16) * b_step));
    *reinterpret_cast<uint16_t *>(s_b + tc_off(f, k, b_step)) = h1;
    *reinterpret_cast<uint16_t *>(s_b + tc_off(16 + f, k, b_step)) = h2;
    *reinterpret_cast<uint16_t *>(s_b + tc_off(32 + f, k, b_step)) = h3;
  }
  if (warp == 0) {  // 64 TMEM columns hold the 128 x 48 f32 accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init(&s_bar[2], 1);
    fence_mbar_init();
    if (bulk && blockIdx.x < batch) {
      mbar_arrive_expect_tx(&s_bar[0], (uint32_t)frame);
      bulk_load_g2s(s_obs0, obs + (int64_t)blockIdx.x * frame, (uint32_t)frame, &s_bar[0]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  PXR_DCHECK((tmem & 0xFFFFu) + 64u <= 512u);
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcN >> 3) << 17) |
                         ((uint32_t)(kTcM >> 4) << 24);
  const uint32_t a_base = (uint32_t)__cvta_generic_to_shared(s_a);
  const uint32_t b_base = (uint32_t)__cvta_generic_to_shared(s_b);
  uint32_t mma_phase = 0;
  int it = 0;
  for (int64_t env = blockIdx.x; env < batch; env += gridDim.x, it++) {
    __syncthreads();  // the other frame buffer is no longer read
    uint8_t *s_obs = s_obs0 + (it & 1) * fstride;
    if (bulk) {
      const int64_t nxt = env + gridDim.x;
      if (tid == 0 && nxt < batch) {
        uint64_t *bar = &s_bar[(it + 1) & 1];
        mbar_arrive_expect_tx(bar, (uint32_t)frame);
        bulk_load_g2s(s_obs0 + ((it + 1) & 1) * fstride, obs + nxt * frame, (uint32_t)frame,
                      bar);
      }
      mbar_wait_parity(&s_bar[it & 1], (uint32_t)((it >> 1) & 1));
    } else {
      const uint8_t *src = obs + env * (int64_t)frame;
      for (int i = tid; i < frame; i += kTcThreads) s_obs[i] = src[i];
      __syncthreads();
    }
    // the frame as bf16, once (bytes are exact in bf16); frames too large
    // for a bf16 copy next to the operands are converted per chunk below
    if (use_fb) {
      const int n8 = frame >> 3;
      const uint32_t *src = reinterpret_cast<const uint32_t *>(s_obs);
      for (int c = tid; c < n8; c += kTcThreads) {
        const uint32_t lo = src[2 * c], hi = src[2 * c + 1];
        uint4 v;
        v.x = bf16x2_of_bytes(lo & 0xffu, (lo >> 8) & 0xffu);
        v.y = bf16x2_of_bytes((lo >> 16) & 0xffu, lo >> 24);
        v.z = bf16x2_of_bytes(hi & 0xffu, (hi >> 8) & 0xffu);
        v.w = bf16x2_of_bytes((hi >> 16) & 0xffu, hi >> 24);
        reinterpret_cast<uint4 *>(s_fb)[c] = v;
      }
      for (int i = (n8 << 3) + tid; i < frame; i += kTcThreads)
        s_fb[i] = (uint16_t)(bf16x2_of_bytes(s_obs[i], 0u) & 0xffffu);
    }
    __syncthreads();
    float *fe = feat + env * (int64_t)(n_pos * kF);
    for (int m0 = 0; m0 < n_pos; m0 += kTcM) {
      // A: im2col rows of this tile; item (row, ky) = 8 C consecutive bytes.
      // Consecutive lanes take consecutive rows: each quarter-warp's 16-B
      // stores then fill one 128-B line of the K-major layout (no bank
      // conflicts) and the source words are 12 B apart (conflict-free too).
      static_assert(kTcM == 128, "row = item & 127");
      for (int item = tid; item < kTcM * kK; item += kTcThreads) {
        const int row = item & (kTcM - 1), ky = item >> 7, pos = m0 + row;
        if (pos >= n_pos) continue;  // rows past the end are computed and dropped
        const int e0 = s_posoff[pos] + ky * W * C;
        PXR_DCHECK(e0 + 8 * C <= frame);
        for (int ch = 0; ch < C; ch++) {  // 8-element K chunks
          const int e = e0 + 8 * ch;
          uint4 v;
          if (!use_fb) {  // straight from the bytes
            const uint8_t *b8 = s_obs + e;
            uint32_t lo, hi;
            if ((e & 3) == 0) {
              lo = *reinterpret_cast<const uint32_t *>(b8);
              hi = *reinterpret_cast<const uint32_t *>(b8 + 4);
            } else {
              lo = b8[0] | (b8[1] << 8) | (b8[2] << 16) | ((uint32_t)b8[3] << 24);
              hi = b8[4] | (b8[5] << 8) | (b8[6] << 16) | ((uint32_t)b8[7] << 24);
            }
            v.x = bf16x2_of_bytes(lo & 0xffu, (lo >> 8) & 0xffu);
            v.y = bf16x2_of_bytes((lo >> 16) & 0xffu, lo >> 24);
            v.z = bf16x2_of_bytes(hi & 0xffu, (hi >> 8) & 0xffu);
            v.w = bf16x2_of_bytes((hi >> 16) & 0xffu, hi >> 24);
          } else if (chunk_aligned) {
            const uint2 a = *reinterpret_cast<const uint2 *>(s_fb + e);
            const uint2 b = *reinterpret_cast<const uint2 *>(s_fb + e + 4);
            v = make_uint4(a.x, a.y, b.x, b.y);
          } else {
            const uint16_t *h = s_fb + e;
            v = make_uint4((uint32_t)h[0] | ((uint32_t)h[1] << 16), (uint32_t)h[2] | ((uint32_t)h[3] << 16),
                           (uint32_t)h[4] | ((uint32_t)h[5] << 16), (uint32_t)h[6] | ((uint32_t)h[7] << 16));
          }
          PXR_DCHECK(tc_off(row, ky * 8 * C + 8 * ch, a_step) + 16u <= (uint32_t)((K / 16) * a_step));
          *reinterpret_cast<uint4 *>(s_a + tc_off(row, ky * 8 * C + 8 * ch, a_step)) = v;
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> tensor-core (async) reads
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (tid == 0) {
        for (int s = 0; s < K / 16; s++) {
          const uint64_t da = tc_desc(a_base + s * a_step), db = tc_desc(b_base + s * b_step);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(s));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar[2])));
      }
      mbar_wait_parity(&s_bar[2], mma_phase);
      mma_phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
      // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (its rows) and
      // filters 4 (w / 4) .. +3 of each split
      static_assert(kTcThreads == 512, "16 warps: 4 lane quarters x 4 filter quarters");
      const int q = warp & 3, fh = (warp >> 2) * 4;
      const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16);
      uint32_t d[3][4];
#pragma unroll
      for (int sp = 0; sp < 3; sp++)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(d[sp][0]), "=r"(d[sp][1]), "=r"(d[sp][2]), "=r"(d[sp][3])
                     : "r"(ta + (uint32_t)(sp * 16 + fh)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      const int pos = m0 + 32 * q + lane;
      if (pos < n_pos) {
        float o[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const float v = (__uint_as_float(d[0][i]) + __uint_as_float(d[1][i]) +
                           __uint_as_float(d[2][i])) * inv;
          o[i] = v > 0.0f ? v : 0.0f;  // ReLU
        }
        *reinterpret_cast<float4 *>(fe + pos * kF + fh) = make_float4(o[0], o[1], o[2], o[3]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // TMEM and A are reused by the next tile
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
  }
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

constexpr int kProjEnvs = 16;
constexpr int kProjTile = 256;  // proj rows per shared-memory tile
// The features of an env are reduced in slices of kProjSliceTiles tiles: lane
// l chains the features k = l (mod 32) of the slice in ascending order (one
// FMA chain per output), a fixed xor tree sums the lanes, and the slice sums
// are added in slice order -- the same arithmetic whether one CTA walks all
// slices of its envs (large batches) or each slice runs on its own CTA and
// a combine kernel adds them (small batches), so a row never depends on the
// batch it is in.
constexpr int kProjSliceTiles = 8;
constexpr int kProjSlice = kProjTile * kProjSliceTiles;

// JP = J rounded up to a multiple of 4: the staged proj rows are padded with
// zeros to JP floats so each lane reads its row with 128-bit loads (rows
// 16 B-aligned; 8 consecutive rows of a quarter-warp hit distinct banks for
// every JP used) and the FMA chain of each real output j < J is exactly the
// unpadded one.
//
// Features [ks, ke) of the CTA's envs against proj: per-lane FMA chains,
// reduced over the warp; lane j returns output j's sum.
template <int JP>
__device__ __forceinline__ float proj_slice(const float *__restrict__ fr, bool active, int ks,
                                            int ke, const float *__restrict__ proj, int J,
                                            float *s_p, int tid, int lane) {
  float pacc[JP];
#pragma unroll
  for (int j = 0; j < JP; j++) pacc[j] = 0.0f;
  for (int k0 = ks; k0 < ke; k0 += kProjTile) {
    const int kn = min(kProjTile, ke - k0);
    __syncthreads();  // previous tile no longer read
    for (int i = tid; i < kn * JP; i += kProjEnvs * 32) {
      const int r = i / JP, j = i - r * JP;
      s_p[i] = j < J ? __ldg(proj + (int64_t)(k0 + r) * J + j) : 0.0f;
    }
    __syncthreads();
    if (active) {
      // (unrolled: several feature loads in flight; each output's FMA
      // chain keeps its order)
#pragma unroll 4
      for (int kk = lane; kk < kn; kk += 32) {
        const float v = __ldg(fr + k0 + kk);
        const float4 *pr = reinterpret_cast<const float4 *>(s_p + kk * JP);
#pragma unroll
        for (int j4 = 0; j4 < JP / 4; j4++) {
          const float4 w = pr[j4];
          pacc[4 * j4 + 0] = __fmaf_rn(v, w.x, pacc[4 * j4 + 0]);
          pacc[4 * j4 + 1] = __fmaf_rn(v, w.y, pacc[4 * j4 + 1]);
          pacc[4 * j4 + 2] = __fmaf_rn(v, w.z, pacc[4 * j4 + 2]);
          pacc[4 * j4 + 3] = __fmaf_rn(v, w.w, pacc[4 * j4 + 3]);
        }
      }
    }
  }
  float mine = 0.0f;
#pragma unroll
  for (int j = 0; j < JP; j++) {
    float v = pacc[j];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == j) mine = v;
  }
  return mine;
}

// Projection + tanh, one warp per env (kProjEnvs per CTA, sharing the staged
// proj tiles): all slices in order.
template <int JP>
__global__ void __launch_bounds__(kProjEnvs * 32)
conv_proj_kernel(const float *__restrict__ feat, int64_t batch, int K,
                 const float *__restrict__ proj, int J, double *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  float *s_p = reinterpret_cast<float *>(sm);  // kProjTile x JP
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  PXR_DCHECK(J >= 1 && J <= JP && JP <= kMaxJoints);
  for (int64_t e0 = (int64_t)blockIdx.x * kProjEnvs; e0 < batch;
       e0 += (int64_t)gridDim.x * kProjEnvs) {
    const int64_t env = e0 + warp;
    const float *fr = feat + env * (int64_t)K;
    float total = 0.0f;  // lane j: output j
    for (int ks = 0; ks < K; ks += kProjSlice)
      total += proj_slice<JP>(fr, env < batch, ks, min(ks + kProjSlice, K), proj, J, s_p, tid, lane);
    if (env < batch && lane < J) out[env * J + lane] = (double)tanhf(total);
  }
}

// Small batches: CTA (group, slice) reduces one slice of its kProjEnvs envs
// and parks the sums in the env's own (already read) feature slots k = ks + j.
template <int JP>
__global__ void __launch_bounds__(kProjEnvs * 32)
conv_proj_slice_kernel(float *__restrict__ feat, int64_t batch, int K,
                       const float *__restrict__ proj, int J) {
  extern __shared__ __align__(16) unsigned char sm[];
  float *s_p = reinterpret_cast<float *>(sm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t env = (int64_t)blockIdx.x * kProjEnvs + warp;
  const int ks = blockIdx.y * kProjSlice;
  float *fr = feat + env * (int64_t)K;
  const float sum = proj_slice<JP>(fr, env < batch, ks, min(ks + kProjSlice, K), proj, J, s_p,
                                   tid, lane);
  __syncwarp();  // every lane has read the slice's features
  if (env < batch && lane < J) fr[ks + lane] = sum;
}

// ... and the slice sums are added in slice order (one thread per output).
__global__ void conv_proj_combine_kernel(const float *__restrict__ feat, int64_t batch, int K,
                                         int J, double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= batch * J) return;
  const int64_t env = i / J;
  const int j = (int)(i - env * J);
  const float *fr = feat + env * (int64_t)K;
  float total = 0.0f;
  for (int ks = 0; ks < K; ks += kProjSlice) total += fr[ks + j];
  out[i] = (double)tanhf(total);
}

}  // namespace pxr

using namespace pxr;

extern "C" pxr_status pxr_conv_stub_forward(const uint8_t *obs, int64_t batch, int32_t height,
                                           int32_t width, int32_t channels, const float *conv,
                                           const float *proj, int32_t n_joints, double *out,
                                           float *workspace, void *stream) {
  if (obs == nullptr || conv == nullptr || proj == nullptr || out == nullptr ||
      workspace == nullptr)
    return set_invalid("null pointer");
  if (batch < 0) return set_invalid("batch must be >= 0");
  if (height < kK || width < kK) return set_invalid("observation smaller than the conv kernel");
  if (channels < 1 || channels > 4) return set_invalid("channels must be 1..4");
  if (n_joints < 1 || n_joints > kMaxJoints) return set_unsupported("n_joints must be 1..32");
  if (batch == 0) return PXR_OK;
  const int frame = height * width * channels;
  const int bulk = (frame % 16 == 0) && ((reinterpret_cast<uintptr_t>(obs) & 15) == 0);
  const int Kc = kK * kK * channels;
  const int n_pos = ((height - kK) / kS + 1) * ((width - kK) / kS + 1);
  const int base = (Kc / 16) * ((kTcM / 8) * 256) + (Kc / 16) * ((kTcN / 8) * 256) +
                   2 * ((frame + 15) & ~15);
  // the bf16 frame copy when it fits -- unless leaving it out lets more
  // CTAs share an SM (84x84: 2 instead of 1, one CTA's operand build then
  // overlaps the other's MMA wait: -8 % at 4096-16384 envs); else the
  // per-chunk conversion (the same bf16 operands either way)
  const DeviceFacts &df = device_facts();
  static int smem_sm_dev[64] = {};
  if (smem_sm_dev[df.device & 63] == 0)
    cudaDeviceGetAttribute(&smem_sm_dev[df.device & 63], cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                           df.device);
  const int smem_sm = smem_sm_dev[df.device & 63];
  const int with_table = base + ((4 * n_pos + 15) & ~15);
  const int with_fb = with_table + ((2 * frame + 15) & ~15);
  int use_fb = with_fb <= 220 * 1024;
  if (use_fb && smem_sm / (with_table + 2048) > smem_sm / (with_fb + 2048)) use_fb = 0;
  const int smem = use_fb ? with_fb : with_table;
  if (smem > 220 * 1024) return set_unsupported("observation too large for the policy kernel");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the full shared-memory carveout (frames + bf16 frame + operands), set
  // once per device; the dynamic-smem attribute through the launch cache
  static bool carveout_set[64] = {};
  if (!carveout_set[df.device & 63]) {
    cudaError_t e = cudaFuncSetAttribute(conv_feat_tc_kernel,
                                         cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return set_cuda(e, "cudaFuncSetAttribute");
    carveout_set[df.device & 63] = true;
  }
  int per_sm = 0;
  {
    const pxr_status os = kernel_occupancy((const void *)conv_feat_tc_kernel, kTcThreads, smem,
                                           &per_sm);
    if (os != PXR_OK) return os;
  }
  const int sms = df.num_sms;
  // CTAs per SM from the shared memory per SM (the occupancy query does not
  // see the carveout preference set above)
  per_sm = smem_sm / (smem + 2048);
  if (per_sm > 2048 / kTcThreads) per_sm = 2048 / kTcThreads;
  if (per_sm < 1) per_sm = 1;
  int64_t cap = (int64_t)sms * per_sm;
  int grid = (int)(batch < cap ? batch : cap);
  conv_feat_tc_kernel<<<grid, kTcThreads, smem, st>>>(obs, batch, height, width, channels, conv,
                                                      workspace, bulk, use_fb);
  pxr_status s = check_launch("conv_feat_tc_kernel");
  if (s != PXR_OK) return s;
  const int K = ((height - kK) / kS + 1) * ((width - kK) / kS + 1) * kF;
  const int jp = (n_joints + 3) & ~3;
  const int psmem = kProjTile * jp * (int)sizeof(float);
  void (*pk)(const float *, int64_t, int, const float *, int, double *) = nullptr;
  void (*sk)(float *, int64_t, int, const float *, int) = nullptr;
  switch (jp) {
    case 4: pk = conv_proj_kernel<4>; sk = conv_proj_slice_kernel<4>; break;
    case 8: pk = conv_proj_kernel<8>; sk = conv_proj_slice_kernel<8>; break;
    case 12: pk = conv_proj_kernel<12>; sk = conv_proj_slice_kernel<12>; break;
    case 16: pk = conv_proj_kernel<16>; sk = conv_proj_slice_kernel<16>; break;
    case 20: pk = conv_proj_kernel<20>; sk = conv_proj_slice_kernel<20>; break;
    case 24: pk = conv_proj_kernel<24>; sk = conv_proj_slice_kernel<24>; break;
    case 28: pk = conv_proj_kernel<28>; sk = conv_proj_slice_kernel<28>; break;
    default: pk = conv_proj_kernel<32>; sk = conv_proj_slice_kernel<32>; break;
  }
  {
    const pxr_status os = kernel_occupancy((const void *)pk, kProjEnvs * 32, psmem, &per_sm);
    if (os != PXR_OK) return os;
  }
  cap = (int64_t)sms * per_sm;
  const int64_t groups = (batch + kProjEnvs - 1) / kProjEnvs;
  const int n_slices = (K + kProjSlice - 1) / kProjSlice;
  // small batches: one CTA per (env group, slice), then the slice sums are
  // added (the same arithmetic as the one-CTA path); J <= kProjSlice keeps
  // the parked sums inside the slice
  if (n_slices > 1 && groups * n_slices <= cap && n_joints <= kProjSlice &&
      debug_knob(kDbgNoSplit) == nullptr) {
    sk<<<dim3((unsigned)groups, (unsigned)n_slices), kProjEnvs * 32, psmem, st>>>(
        workspace, batch, K, proj, n_joints);
    s = check_launch("conv_proj_slice_kernel");
    if (s != PXR_OK) return s;
    const int64_t n_out = batch * n_joints;
    conv_proj_combine_kernel<<<(unsigned)((n_out + 127) / 128), 128, 0, st>>>(
        workspace, batch, K, n_joints, out);
    return check_launch("conv_proj_combine_kernel");
  }
  grid = (int)(groups < cap ? groups : cap);
  pk<<<grid, kProjEnvs * 32, psmem, st>>>(workspace, batch, K, proj, n_joints, out);
  return check_launch("conv_proj_kernel");
}

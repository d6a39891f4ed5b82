// Conv-stub policy forward: the reference's fixed
// action-selection surrogate (bench.py:36-145): conv 16 x 8x8 stride 4 over
// obs / 255, ReLU, linear projection of the (oy, ox, f)-ordered features,
// tanh.
//
// One CTA per env (grid-stride over envs), so a batch row never depends on
// the batch it is in (reference tests/test_bench.py:92-98): every thread
// owns fixed conv output positions and all 16 filters of each, and the
// projection partial sums are reduced in a fixed tree. f32 arithmetic like
// the reference's f32 BLAS path; accuracy is checked against a float64
// evaluation (<= 1e-5, tests/test_bench.py:56-68).
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pxr.h"
#include "pxr_internal.cuh"

namespace pxr {

constexpr int kPolThreads = 128;
constexpr int kK = 8, kS = 4, kF = 16;
constexpr int kMaxJoints = 32;

__global__ void __launch_bounds__(kPolThreads)
conv_stub_kernel(const uint8_t *__restrict__ obs, int64_t batch, int H, int W, int C,
                 const float *__restrict__ conv, const float *__restrict__ proj, int J,
                 double *__restrict__ out) {
  extern __shared__ __align__(16) unsigned char sm[];
  float *s_w = reinterpret_cast<float *>(sm);          // (K*K*C, 16): row (ky, kx, c)
  uint8_t *s_obs = sm + kK * kK * C * kF * sizeof(float);
  __shared__ float s_red[kPolThreads / 32][kMaxJoints];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int oh = (H - kK) / kS + 1, ow = (W - kK) / kS + 1;
  const int nw = kK * kK * C * kF;
  const int frame = H * W * C;
  const float inv = 1.0f / 255.0f;  // float32(1/255), bench.py:101
  for (int i = tid; i < nw; i += kPolThreads) s_w[i] = conv[i];
  for (int64_t env = blockIdx.x; env < batch; env += gridDim.x) {
    __syncthreads();  // weights loaded / previous env's frame no longer read
    const uint8_t *src = obs + env * (int64_t)frame;
    for (int i = tid; i < frame; i += kPolThreads) s_obs[i] = src[i];
    __syncthreads();
    float pacc[kMaxJoints];
#pragma unroll
    for (int j = 0; j < kMaxJoints; j++) pacc[j] = 0.0f;
    for (int pos = tid; pos < oh * ow; pos += kPolThreads) {
      const int oy = pos / ow, ox = pos - oy * ow;
      float acc[kF];
#pragma unroll
      for (int f = 0; f < kF; f++) acc[f] = 0.0f;
      for (int ky = 0; ky < kK; ky++) {
        const uint8_t *row = s_obs + ((oy * kS + ky) * W + ox * kS) * C;
        for (int kc = 0; kc < kK * C; kc++) {  // (kx, c) in memory order
          const float x = (float)row[kc] * inv;
          const float4 *w4 = reinterpret_cast<const float4 *>(s_w + (ky * kK * C + kc) * kF);
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const float4 w = w4[q];  // same address in every lane: broadcast
            acc[4 * q + 0] = __fmaf_rn(x, w.x, acc[4 * q + 0]);
            acc[4 * q + 1] = __fmaf_rn(x, w.y, acc[4 * q + 1]);
            acc[4 * q + 2] = __fmaf_rn(x, w.z, acc[4 * q + 2]);
            acc[4 * q + 3] = __fmaf_rn(x, w.w, acc[4 * q + 3]);
          }
        }
      }
      const float *pr = proj + (int64_t)pos * kF * J;
#pragma unroll
      for (int f = 0; f < kF; f++) {
        const float v = acc[f] > 0.0f ? acc[f] : 0.0f;  // ReLU
#pragma unroll
        for (int j = 0; j < kMaxJoints; j++)
          if (j < J) pacc[j] = __fmaf_rn(v, __ldg(pr + f * J + j), pacc[j]);
      }
    }
    // fixed-order reduction: xor tree inside the warp, warps in index order
#pragma unroll
    for (int j = 0; j < kMaxJoints; j++) {
      if (j >= J) break;
      float v = pacc[j];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) s_red[warp][j] = v;
    }
    __syncthreads();
    if (tid < J) {
      float v = s_red[0][tid];
      for (int w = 1; w < kPolThreads / 32; w++) v += s_red[w][tid];
      out[env * J + tid] = (double)tanhf(v);
    }
  }
}

}  // namespace pxr

using namespace pxr;

extern "C" pxr_status pxr_conv_stub_forward(const uint8_t *obs, int64_t batch, int32_t height,
                                           int32_t width, int32_t channels, const float *conv,
                                           const float *proj, int32_t n_joints, double *out,
                                           void *stream) {
  if (obs == nullptr || conv == nullptr || proj == nullptr || out == nullptr)
    return set_invalid("null pointer");
  if (batch < 0) return set_invalid("batch must be >= 0");
  if (height < kK || width < kK) return set_invalid("observation smaller than the conv kernel");
  if (channels < 1 || channels > 4) return set_invalid("channels must be 1..4");
  if (n_joints < 1 || n_joints > kMaxJoints) return set_unsupported("n_joints must be 1..32");
  if (batch == 0) return PXR_OK;
  const int smem = kK * kK * channels * kF * (int)sizeof(float) + height * width * channels;
  if (smem > 200 * 1024) return set_unsupported("observation too large for the policy kernel");
  cudaError_t e = cudaFuncSetAttribute(conv_stub_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return set_cuda(e, "cudaFuncSetAttribute");
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, conv_stub_kernel, kPolThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)sms * per_sm;
  const int grid = (int)(batch < cap ? batch : cap);
  conv_stub_kernel<<<grid, kPolThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      obs, batch, height, width, channels, conv, proj, n_joints, out);
  return check_launch("conv_stub_kernel");
}

/*
 * pxr.h -- C ABI of libpxr.so, the B200 (sm_100a) pixel-observation hot path
 * of the PixelBrax reference (`pixelctrl`). Plain pointers and sizes only:
 * every array argument is a DEVICE pointer (cudaMalloc / torch CUDA tensor
 * storage) unless its comment says "host"; `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream). All calls are asynchronous on
 * `stream` and never synchronise the host.
 *
 * The reference has no FFI of its own: its hot path is numba @njit kernels
 * called from Python. Each entry point below names the reference function
 * (path:line under /root/reference/pkg/src/pixelctrl/) whose call it
 * replaces; the Python host layer (paper_2502_00021_b200/) binds them with
 * ctypes exactly where the reference calls its numba kernels. See
 * INTEGRATION.md for the binding stub.
 *
 * Error convention: the reference raises ValueError from its Python wrappers
 * before any kernel runs (render.py:117-118, 500-501; distractor.py:185-188,
 * 199-202). Here every entry point validates its arguments first and returns
 * a non-zero pxr_status without launching anything; the Python layer maps
 * PXR_ERR_INVALID to ValueError with the reference's message and every other
 * code to RuntimeError. Kernels themselves have no error path (degenerate
 * triangles are skipped, render.py:379-380, 415-416).
 */
#ifndef PXR_H
#define PXR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PXR_ABI_VERSION 3

typedef int32_t pxr_status;
#define PXR_OK 0
#define PXR_ERR_INVALID 1     /* bad sizes / null pointers / bad mode      */
#define PXR_ERR_CUDA 2        /* a CUDA runtime call or launch failed      */
#define PXR_ERR_UNSUPPORTED 3 /* shape beyond this build's limits          */

/* Distractor modes (distractor.py:33 _MODES). */
#define PXR_MODE_NONE 0
#define PXR_MODE_COLOR 1
#define PXR_MODE_VIDEO 2

/* Robot mesh, flattened like RobotGeometry (render.py:559-591): capsule
 * links tessellated once, vertices in link-local coordinates. */
typedef struct pxr_geometry {
  const float *base_verts;   /* (n_verts, 3) f32 link-local               */
  const int32_t *vert_link;  /* (n_verts)    link id of each vertex       */
  const int32_t *triangles;  /* (n_tris, 3)  index order = tie-break order */
  const float *tri_colors;   /* (n_tris, 3)  base RGB in [0, 1]           */
  int32_t n_verts, n_tris, n_links;
} pxr_geometry;

/* Tracking camera (render.py:98-105, 237-279, 607-612): the orientation
 * block is shared by every env, only the eye follows the root link. */
typedef struct pxr_camera {
  float block[15];        /* host: camera_basis(track_camera((0,0), cfg))  */
  double offset_x;        /* host: cfg.offset[0] (eye.x = f32(root_x + ox)) */
  double offset_z;        /* host: cfg.offset[2] (eye.z = f32(root_z + oz)) */
  float light[3];         /* host: LIGHT_DIR as f32 (render.py:56-57, 488)  */
  /* Floor ray directions (render.py:316-344), f64 (H, W, 3) as produced by
   * pxr_floor_rays(); NULL when no floor is drawn. `floor_separable` != 0
   * when every row shares one x-sequence and y/z are constant along x (the
   * default CameraConfig), letting the kernel stage W + 2H doubles in shared
   * memory instead of reading the whole table per env. */
  const double *floor_rays;
  int32_t floor_separable;
} pxr_camera;

/* Per-env distractor state (DistractorState, distractor.py:36-55), device
 * SoA. Arrays a mode does not use may be NULL. */
typedef struct pxr_distractor {
  int32_t mode;          /* PXR_MODE_*                                    */
  int16_t *color_bias;   /* (B, 3) colour mode                            */
  int64_t *video_index;  /* (B)    video mode                             */
  int64_t *frame_cursor; /* (B)                                           */
  int8_t *direction;     /* (B)                                           */
  int64_t *frame_count;  /* (B)                                           */
} pxr_distractor;

/* HBM-resident video pack, VideoPack.flat_frames() layout
 * (video_pack.py:46-61): all frames stacked, per-video start offsets. */
typedef struct pxr_video_pack {
  const uint8_t *frames;   /* (n_frames, height, width, 3) u8               */
  const int64_t *starts;   /* (n_videos) first frame of each video          */
  const int64_t *counts;   /* (n_videos) frame count of each video          */
  int64_t n_videos, n_frames, height, width;
  /* optional: every frame already nearest-upscaled to the observation size
   * (pxr_pack_upscale; NULL if absent). pxr_render_step then copies the env's
   * frame into its RGB frame buffer with one TMA bulk load instead of
   * gathering texels per pixel (same bytes: distractor.py:172-181). */
  const uint8_t *frames_hw;  /* (n_frames, hw_height, hw_width, 3) u8       */
  int64_t hw_height, hw_width;
} pxr_video_pack;

/* Per-step key material (env.py:176-255). */
typedef struct pxr_step_keys {
  uint64_t key_hi, key_lo;   /* key_t = fold_in(master, t)                 */
  uint64_t env_offset;       /* global index of env 0 of this batch        */
  uint64_t logical_batch;    /* reset keys use fold_in(key_t, LB + g)      */
  /* optional: key_t as (hi, lo) in DEVICE memory, read when the kernel runs
   * (key_hi/key_lo ignored) -- a captured CUDA graph replays with the key
   * pxr_step_key_advance wrote for this step */
  const uint64_t *device_key;
} pxr_step_keys;

/* ------------------------------------------------------------------ */

int32_t pxr_abi_version(void);
/* 1 for the checked build (libpxr_checked.so: device bounds / invariant
 * checks compiled in, a failed check traps the launch), else 0. */
int32_t pxr_build_checked(void);
const char *pxr_status_string(pxr_status s);
/* Last CUDA error string seen by a failing call (thread-local). */
const char *pxr_last_error(void);
/* Test / debug knobs (no reference counterpart): `name` is one of
 * PXR_DEBUG_FRAG_LIMIT, _ROW_CAP, _CAP, _STATS_PTR, _BAND_H, _NO_PACKED_SCAN,
 * _PHYS, _GRID, _PROF, _NO_UPSCALE; `value` its string value, NULL to unset. The PXR_DEBUG_*
 * environment is read once at the first query; this overrides it. */
pxr_status pxr_set_debug(const char *name, const char *value);

/* Floor ray-direction table for a camera block: f64 (H, W, 3), the exact
 * incremental sequence of render.py:316-344. Writes `*separable` (host). */
pxr_status pxr_floor_rays(const float *cam_block_host, int64_t height, int64_t width,
                          double *out_rays, int32_t *separable_host, void *stream);

/* Fused hot path: replaces Env._render_frame + Env._postprocess
 * (env.py:155-173), i.e. render_robot_batch (render.py:594-623) +
 * apply_color_inplace / apply_video_inplace (distractor.py:184-214) +
 * grayscale, and -- when `advance` != 0 -- advance_distractors
 * (distractor.py:116-137) followed by the auto-reset video re-draw for envs
 * with done[i] != 0 (env.py:239-244), all in ONE launch.
 *
 *   poses      (B, n_links, 3) f64 [x, z, pitch] (forward_kinematics output)
 *   dist       updated in place when advance != 0 (new biases / cursors)
 *   done       (B) u8, NULL = no resets
 *   out_obs    (B, H, W, 3) u8, or (B, H, W, 1) when grayscale != 0
 *   out_depth  (B, H, W) f32 z-buffer (+inf = background) or NULL
 */
pxr_status pxr_render_step(const pxr_geometry *geom, const pxr_camera *cam,
                           const double *poses, int64_t batch, int64_t height,
                           int64_t width, int32_t draw_floor,
                           const pxr_distractor *dist, const pxr_video_pack *pack,
                           int32_t advance, const pxr_step_keys *keys,
                           const uint8_t *done, int32_t grayscale, uint8_t *out_obs,
                           float *out_depth, void *stream);

/* distractor.py:116-137 advance_distractors (+ env.py:239-244 video reset
 * of done envs when done != NULL), as a standalone launch. */
pxr_status pxr_advance_distractors(const pxr_distractor *dist,
                                   const pxr_video_pack *pack, int64_t batch,
                                   const pxr_step_keys *keys, const uint8_t *done,
                                   void *stream);

/* distractor.py:82-113 init_distractors: subkeys split(key, off + B)[off:]
 * drawn on the device. `key` = fold_in(master, 0xD157). */
pxr_status pxr_init_distractors(const pxr_distractor *dist,
                                const pxr_video_pack *pack, int64_t batch,
                                uint64_t key_hi, uint64_t key_lo,
                                uint64_t env_offset, void *stream);

/* distractor.py:140-161 _color_kernel: clamp(p + bias) on every pixel. */
pxr_status pxr_apply_color(uint8_t *pixels, const int16_t *bias, int64_t batch,
                           int64_t height, int64_t width, void *stream);

/* distractor.py:164-176 _video_kernel: background (isinf(depth)) pixels
 * replaced by frames[starts[vid] + cursor] sampled through nearest_map. */
pxr_status pxr_apply_video(uint8_t *pixels, const float *depth,
                           const pxr_video_pack *pack, const int64_t *video_index,
                           const int64_t *frame_cursor, int64_t batch,
                           int64_t height, int64_t width, void *stream);

/* env.py:168-173 grayscale: (299R + 587G + 114B + 500) // 1000. */
pxr_status pxr_grayscale(const uint8_t *rgb, uint8_t *gray, int64_t n_pixels,
                         void *stream);

/* prng.py:57-77 Threefry-2x64-20 over n counters; keys are per element
 * (key_stride 1) or broadcast (key_stride 0). fold_in_many (prng.py:168-171)
 * is c1 = 2, words_per_key (174-178) is c1 = 0, split is c1 = 1. */
pxr_status pxr_threefry2x64(const uint64_t *k0, const uint64_t *k1, int64_t key_stride,
                            const uint64_t *c0, const uint64_t *c1, int64_t c1_stride,
                            uint64_t *y0, uint64_t *y1, int64_t n, void *stream);

/* The render kernel's exact division (reciprocal + Markstein correction)
 * next to IEEE a / b, for the parity test. */
pxr_status pxr_div_check(const double *a, const double *b, double *q_pre, double *q_ieee,
                         int64_t n, void *stream);

/* nearest_map compositing source (distractor.py:172-181) precomputed once
 * per pack and observation size: out[f][y][x] = frames[f][(y*Hv)//H][(x*Wv)//W]
 * for every frame f, out (n_frames, height, width, 3) u8. */
pxr_status pxr_pack_upscale(const pxr_video_pack *pack, int64_t height, int64_t width,
                            uint8_t *out, void *stream);

/* Device sinf/cosf (glibc 2.39 restatement) for the parity test. */
pxr_status pxr_sincosf(const float *x, float *s, float *c, int64_t n, void *stream);

/* Device sin/cos in float64 (glibc 2.39 restatement, the physics' trig) for
 * the parity test. */
pxr_status pxr_sincos(const double *x, double *s, double *c, int64_t n, void *stream);

/* Device log in float64 (numpy's AVX-512 log restated: the reset draws'
 * Box-Muller log) for the parity test. */
pxr_status pxr_log(const double *x, double *y, int64_t n, void *stream);

/* Synthetic pose source for benchmarking: per env g =
 * env_offset + i, qpos = rest + U(-0.1, 0.1) from the reference reset keys
 * plus a deterministic joint oscillation at step t, then planar forward
 * kinematics (physics.py:114-137) in f64 into poses (B, n_links, 3). */
pxr_status pxr_pose_source(const double *rest_qpos, const int32_t *parent,
                           const double *anchor_dist, int32_t n_links,
                           uint64_t reset_key_hi, uint64_t reset_key_lo,
                           uint64_t env_offset, int64_t t, int64_t batch,
                           double *poses, void *stream);

/* ---- physics (the producer of the poses) ---------- */

/* ModelSpec + ModelArrays flattened (models.py:46-103, physics.py:75-96);
 * device arrays of n_links entries (joint arrays: n_links - 1). */
typedef struct pxr_model {
  const int32_t *parent;      /* (L) parent link, -1 for the root         */
  const double *anchor_dist;  /* (L) joint anchor distance along parent   */
  const double *length, *mass, *inertia;  /* (L)                          */
  const double *limit_lo, *limit_hi, *torque_max;  /* (L - 1)             */
  const double *rest_qpos;    /* (L + 2) reset centre                     */
  int32_t n_links, substeps, fixed_root, has_min_root_height;
  double dt, min_root_height, forward_weight, ctrl_cost;
  int64_t episode_length;
} pxr_model;

/* One control step of step_dynamics (physics.py:427-465, _step_batch
 * 272-420) for every env, in place, and reward += compute_reward
 * (physics.py:468-477). done is set, never cleared. */
pxr_status pxr_physics_step(const pxr_model *model, double *qpos, double *qvel,
                            int64_t *step_count, uint8_t *done, const double *actions,
                            double *reward, int64_t batch, void *stream);

/* Reset draws (physics.py:487-510 / env.py:142-153, 226-238).
 * mode 0: every env, key = split(key, .)[env_offset + i] (reset_state).
 * mode 1: envs with done != 0 (auto-reset), key = fold_in(key_t, LB + g);
 *         also the episode bookkeeping of env.py:219-238 (info_* outputs). */
pxr_status pxr_reset_envs(const pxr_model *model, double *qpos, double *qvel,
                          int64_t *step_count, uint8_t *done, double *ep_return,
                          int64_t *ep_length, double *info_return, int64_t *info_length,
                          const double *reward, int64_t batch, uint64_t key_hi,
                          uint64_t key_lo, uint64_t env_offset, uint64_t logical_batch,
                          int32_t mode, const uint64_t *device_key, void *stream);

/* key_t = fold_in(master, *t) into key_out[0..1] (device), then *t += 1:
 * the per-step key schedule of env.py:209 on the device, so a CUDA graph of
 * the env step stays valid from one replay to the next. */
pxr_status pxr_step_key_advance(uint64_t master_hi, uint64_t master_lo, int64_t *t,
                                uint64_t *key_out, void *stream);

/* forward_kinematics (physics.py:114-137, Env._render_frame env.py:155-166)
 * for an env's model: qpos (B, L + 2) -> poses (B, L, 3). */
pxr_status pxr_env_poses(const pxr_model *model, const double *qpos, int64_t batch,
                         double *poses, void *stream);

/* forward_kinematics (physics.py:114-137): qpos (B, 3 + J) -> poses. */
pxr_status pxr_forward_kinematics(const double *qpos, const int32_t *parent,
                                  const double *anchor_dist, int32_t n_links,
                                  int64_t batch, double *poses, void *stream);

/* Conv-stub policy forward (bench.py:36-145 ConvStub / conv_stub_forward /
 * _conv_forward_range): obs u8 (B, H, W, C) -> actions f64 (B, J) =
 * tanh(relu(conv16x8x8s4(obs * f32(1/255))) @ proj), f32 arithmetic.
 * conv: f32 (8*8*C, 16), row (ky, kx, c); proj: f32 (oh*ow*16, J), feature
 * order (oy, ox, f). Each batch row is computed independently of the batch
 * (bench.py:131-145 contract). J <= 32. workspace: f32 device scratch of
 * batch * oh * ow * 16 floats (the ReLU'd features). */
pxr_status pxr_conv_stub_forward(const uint8_t *obs, int64_t batch, int32_t height,
                                 int32_t width, int32_t channels, const float *conv,
                                 const float *proj, int32_t n_joints, double *out,
                                 float *workspace, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PXR_H */

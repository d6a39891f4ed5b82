"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings for the C restatement in this directory (liboracle.so) plus
numpy restatements of the host-side glue of the reference's hot path. Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import
this module -- it is the parity checker and the CPU baseline, never the
product. The product package (``paper_2502_00021_b200``) does not import it.

Reference restated (all paths under /root/reference/pkg/src/pixelctrl/):
  render_robot_batch   render.py:594-623 (cams 607-612, poses32 613)
  raster kernels       render.py:286-485  -> render_oracle.c
  colour / video       distractor.py:66-214 -> render_oracle.c, prng_oracle.c
  key schedule         prng.py:57-193, env.py:176-255
  grayscale            env.py:168-173
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i16p = ctypes.POINTER(ctypes.c_int16)
_i8p = ctypes.POINTER(ctypes.c_int8)
_I64 = ctypes.c_int64


def sincos64(x):
    """glibc 2.39 sin / cos in float64 (sin_glibc.c restatement), |x| < 105414350."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.empty_like(x)
    c = np.empty_like(x)
    dp = ctypes.POINTER(ctypes.c_double)
    lib().glibc_sincos_batch(x.ctypes.data_as(dp), s.ctypes.data_as(dp), c.ctypes.data_as(dp),
                             x.size)
    return s, c


def np_log(x):
    """numpy's AVX-512 float64 log (np_log_svml.c restatement); positive
    normal inputs."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    dp = ctypes.POINTER(ctypes.c_double)
    lib().np_log_svml_batch(x.ctypes.data_as(dp), y.ctypes.data_as(dp), x.size)
    return y


def build() -> str:
    """Compile liboracle.so with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_sinf.restype = ctypes.c_float
        L.oracle_sinf.argtypes = [ctypes.c_float]
        L.oracle_cosf.restype = ctypes.c_float
        L.oracle_cosf.argtypes = [ctypes.c_float]
        L.oracle_sincosf_selftest.restype = ctypes.c_int64
        L.oracle_sincosf_selftest.argtypes = [ctypes.c_uint32] * 3
        L.oracle_sincosf_many.restype = None
        L.oracle_sincosf_many.argtypes = [_f32p, _f32p, _f32p, _I64]
        L.np_log_svml_batch.restype = None
        L.np_log_svml_batch.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2 + [_I64]
        L.glibc_sincos_batch.restype = None
        L.glibc_sincos_batch.argtypes = [ctypes.POINTER(ctypes.c_double)] * 3 + [_I64]
        L.oracle_threefry2x64.restype = None
        L.oracle_threefry2x64.argtypes = [_u64p, _u64p, _I64, _u64p, _u64p, _u64p, _u64p, _I64]
        L.oracle_raster_scene.restype = None
        L.oracle_raster_scene.argtypes = [
            _f32p, _I64, _i32p, _I64, _f32p, _f32p, _f32p, ctypes.c_int,
            _u8p, _f32p, _I64, _I64,
        ]
        L.oracle_raster_robot_range.restype = None
        L.oracle_raster_robot_range.argtypes = [
            _f32p, _i32p, _I64, _i32p, _I64, _f32p, _f32p, _I64, _f32p, _f32p,
            ctypes.c_int, _u8p, _f32p, _I64, _I64, _I64, ctypes.c_int,
        ]
        L.oracle_color_kernel.restype = None
        L.oracle_color_kernel.argtypes = [_u8p, _i64p, _I64, _I64, _I64, ctypes.c_int]
        L.oracle_video_kernel.restype = None
        L.oracle_video_kernel.argtypes = [
            _u8p, _f32p, _u8p, _I64, _I64, _i64p, _i64p, _i64p, _I64, _I64, _I64,
            ctypes.c_int,
        ]
        L.oracle_grayscale.restype = None
        L.oracle_grayscale.argtypes = [_u8p, _u8p, _I64]
        L.oracle_color_biases.restype = None
        L.oracle_color_biases.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _I64, _i16p]
        L.oracle_video_advance.restype = None
        L.oracle_video_advance.argtypes = [_i64p, _i8p, _i64p, _I64]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def sincosf(x: np.ndarray):
    """glibc 2.39 sinf/cosf restatement, element-wise."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    s = np.empty_like(x)
    c = np.empty_like(x)
    lib().oracle_sincosf_many(_p(x, _f32p), _p(s, _f32p), _p(c, _f32p), x.size)
    return s, c


# ---------------------------------------------------------------- prng

MASK64 = (1 << 64) - 1
_ROT = (16, 42, 12, 31, 16, 32, 24, 21)
_PARITY = 0x1BD11BDAA9FC1FFA
SEED_KEY = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def threefry2x64(k0: int, k1: int, c0: int, c1: int) -> tuple[int, int]:
    """Pure-Python Threefry-2x64-20 block (prng.py:57-77), scalar."""
    ks = (k0 & MASK64, k1 & MASK64, (k0 ^ k1 ^ _PARITY) & MASK64)
    x0 = (c0 + ks[0]) & MASK64
    x1 = (c1 + ks[1]) & MASK64
    for r in range(20):
        rot = _ROT[r % 8]
        x0 = (x0 + x1) & MASK64
        x1 = ((x1 << rot) | (x1 >> (64 - rot))) & MASK64
        x1 ^= x0
        if r % 4 == 3:
            j = r // 4 + 1
            x0 = (x0 + ks[j % 3]) & MASK64
            x1 = (x1 + ks[(j + 1) % 3] + j) & MASK64
    return x0, x1


def threefry2x64_many(k0, k1, c0, c1):
    """Vectorised through the C oracle; keys broadcast if scalar."""
    c0 = np.ascontiguousarray(c0, dtype=np.uint64)
    c1 = np.ascontiguousarray(np.broadcast_to(np.asarray(c1, np.uint64), c0.shape))
    k0 = np.ascontiguousarray(np.atleast_1d(np.asarray(k0, np.uint64)))
    k1 = np.ascontiguousarray(np.atleast_1d(np.asarray(k1, np.uint64)))
    stride = 0 if k0.size == 1 else 1
    y0 = np.empty_like(c0)
    y1 = np.empty_like(c0)
    lib().oracle_threefry2x64(_p(k0, _u64p), _p(k1, _u64p), stride, _p(c0, _u64p),
                              _p(c1, _u64p), _p(y0, _u64p), _p(y1, _u64p), c0.size)
    return y0, y1


def key_from_seed(seed: int) -> tuple[int, int]:
    return threefry2x64(SEED_KEY[0], SEED_KEY[1], seed & MASK64, 0)  # prng.py:85-90


def fold_in(key, data: int):
    return threefry2x64(key[0], key[1], data & MASK64, 2)  # prng.py:105-108


def split_one(key, i: int):
    return threefry2x64(key[0], key[1], i & MASK64, 1)  # prng.py:93-102


def index_from_word(w: int, n: int) -> int:
    return (w * n) >> 64  # prng.py:155-161 / 181-193


def color_biases(key_t, env_offset: int, batch: int) -> np.ndarray:
    out = np.empty((batch, 3), dtype=np.int16)
    lib().oracle_color_biases(key_t[0], key_t[1], env_offset, batch, _p(out, _i16p))
    return out


def video_index_for_key(key, n_videos: int) -> int:
    """distractor.py:77-79: words_per_key(.., 2).x0 mapped onto [0, n)."""
    w0, _ = threefry2x64(key[0], key[1], 2, 0)
    return index_from_word(w0, n_videos)


# ---------------------------------------------------------------- render

SKY_COLOR = (135, 206, 235)
_l = np.array([0.3, -0.5, 0.8])
LIGHT_F32 = (_l / np.linalg.norm(_l)).astype(np.float32)  # render.py:56-57, 488


def camera_block(eye, target, up=(0.0, 0.0, 1.0), fov=0.9, near=0.1, far=50.0):
    """render.py:252-279 camera_basis (f64 maths stored as f32)."""
    eye = np.array(eye, dtype=np.float64)
    fwd = np.array(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.array(up, dtype=np.float64))
    right /= np.linalg.norm(right)
    upc = np.cross(right, fwd)
    out = np.empty(15, dtype=np.float32)
    out[0:3] = eye
    out[3:6] = right
    out[6:9] = upc
    out[9:12] = fwd
    out[12] = math.tan(fov / 2.0)
    out[13] = near
    out[14] = far
    return out


CAM_OFFSET = (0.0, -3.0, 1.2)  # render.py:102


def robot_cams(poses: np.ndarray, offset=CAM_OFFSET, fov=0.9, near=0.1, far=50.0):
    """render.py:607-612: shared orientation, per-env eye x/z in f64 -> f32."""
    base = camera_block((offset[0], offset[1], offset[2]), (0.0, 0.0, 0.0),
                        fov=fov, near=near, far=far)
    cams = np.broadcast_to(base, (poses.shape[0], 15)).copy()
    cams[:, 0] = (poses[:, 0, 0] + offset[0]).astype(np.float32)
    cams[:, 2] = (poses[:, 0, 1] + offset[2]).astype(np.float32)
    return cams


def render_robot_batch(geom, poses: np.ndarray, width: int, height: int,
                       floor_in_background: bool, threads: int = 1, offset=CAM_OFFSET,
                       fov: float = 0.9, near: float = 0.1, far: float = 50.0):
    """render.py:594-623 on the C oracle. ``geom`` needs base_verts,
    vert_link, triangles, tri_colors (the RobotGeometry layout); the camera
    follows CameraConfig(offset, vertical_fov, near, far)."""
    poses = np.ascontiguousarray(poses, dtype=np.float64)
    batch, n_links, _ = poses.shape
    cams = robot_cams(poses, offset=offset, fov=fov, near=near, far=far)
    poses32 = np.ascontiguousarray(poses.astype(np.float32))
    bv = np.ascontiguousarray(geom.base_verts, dtype=np.float32)
    vl = np.ascontiguousarray(geom.vert_link, dtype=np.int32)
    tr = np.ascontiguousarray(geom.triangles, dtype=np.int32)
    tc = np.ascontiguousarray(geom.tri_colors, dtype=np.float32)
    pixels = np.zeros((batch, height, width, 3), dtype=np.uint8)
    depth = np.zeros((batch, height, width), dtype=np.float32)
    lib().oracle_raster_robot_range(
        _p(bv, _f32p), _p(vl, _i32p), bv.shape[0], _p(tr, _i32p), tr.shape[0],
        _p(tc, _f32p), _p(poses32, _f32p), n_links, _p(cams, _f32p),
        _p(LIGHT_F32, _f32p), int(not floor_in_background), _p(pixels, _u8p),
        _p(depth, _f32p), batch, height, width, int(threads),
    )
    return pixels, depth


def raster_scene(verts, tris, colors, cam, draw_floor, width, height, light=None):
    verts = np.ascontiguousarray(verts, dtype=np.float32)
    tris = np.ascontiguousarray(tris, dtype=np.int32)
    colors = np.ascontiguousarray(colors, dtype=np.float32)
    cam = np.ascontiguousarray(cam, dtype=np.float32)
    light = LIGHT_F32 if light is None else np.ascontiguousarray(light, np.float32)
    pixels = np.zeros((height, width, 3), dtype=np.uint8)
    depth = np.zeros((height, width), dtype=np.float32)
    lib().oracle_raster_scene(
        _p(verts, _f32p), verts.shape[0], _p(tris, _i32p), tris.shape[0],
        _p(colors, _f32p), _p(cam, _f32p), _p(light, _f32p), int(draw_floor),
        _p(pixels, _u8p), _p(depth, _f32p), height, width,
    )
    return pixels, depth


def nearest_map(dst: int, src: int) -> np.ndarray:
    return (np.arange(dst, dtype=np.int64) * src) // dst  # distractor.py:179-181


def apply_color_inplace(pixels: np.ndarray, bias: np.ndarray, threads: int = 1) -> None:
    b = np.ascontiguousarray(bias, dtype=np.int64)
    B, H, W, _ = pixels.shape
    lib().oracle_color_kernel(_p(pixels, _u8p), _p(b, _i64p), B, H, W, int(threads))


def apply_video_inplace(pixels, depth, frames_flat, frame_idx, threads: int = 1) -> None:
    B, H, W, _ = pixels.shape
    n, hv, wv, _ = frames_flat.shape
    fi = np.ascontiguousarray(frame_idx, dtype=np.int64)
    rm = nearest_map(H, hv)
    cm = nearest_map(W, wv)
    ff = np.ascontiguousarray(frames_flat, dtype=np.uint8)
    lib().oracle_video_kernel(_p(pixels, _u8p), _p(depth, _f32p), _p(ff, _u8p), hv, wv,
                              _p(fi, _i64p), _p(rm, _i64p), _p(cm, _i64p), B, H, W,
                              int(threads))


def grayscale(pixels: np.ndarray) -> np.ndarray:
    rgb = np.ascontiguousarray(pixels, dtype=np.uint8)
    out = np.empty(rgb.shape[:-1] + (1,), dtype=np.uint8)
    lib().oracle_grayscale(_p(rgb, _u8p), _p(out, _u8p), rgb.size // 3)
    return out


def video_advance(cursor, direction, frame_count):
    c = np.array(cursor, dtype=np.int64)
    d = np.array(direction, dtype=np.int8)
    fc = np.ascontiguousarray(frame_count, dtype=np.int64)
    lib().oracle_video_advance(_p(c, _i64p), _p(d, _i8p), _p(fc, _i64p), c.size)
    return c, d


# ---------------------------------------------------------------- host workload
# Host-side (numpy + C oracle) restatements of the per-step glue around the
# render path, for the full-size parity tests and the bench's reference arm.
# No torch, no libpxr.


def _index_from_words(w: np.ndarray, n: int) -> np.ndarray:
    """prng.py:181-193 (32-bit halves), vectorised."""
    w = np.asarray(w, dtype=np.uint64)
    un = np.uint64(n)
    hi = w >> np.uint64(32)
    lo = w & np.uint64(0xFFFFFFFF)
    return ((hi * un + ((lo * un) >> np.uint64(32))) >> np.uint64(32)).astype(np.int64)


def _biases_from_keys(hi, lo) -> np.ndarray:
    """distractor.py:66-74 _sample_biases for an array of keys."""
    z = np.zeros_like(hi)
    w0, w1 = threefry2x64_many(hi, lo, z, 0)
    w2, _ = threefry2x64_many(hi, lo, z + np.uint64(1), 0)
    out = np.empty((hi.shape[0], 3), dtype=np.int16)
    for c, w in enumerate((w0, w1, w2)):
        out[:, c] = _index_from_words(w, 121) - 60
    return out


def _video_from_keys(hi, lo, n_videos: int) -> np.ndarray:
    """distractor.py:77-79 sample_video_indices."""
    w0, _ = threefry2x64_many(hi, lo, np.full(hi.shape, 2, np.uint64), 0)
    return _index_from_words(w0, n_videos)


def init_distractors(mode: str, frame_counts, key, batch: int, env_offset: int = 0) -> dict:
    """distractor.py:82-113: keys = split(key, off + B)[off:] (TF(key, (g, 1))),
    colour biases / video index from each key. Returns the DistractorState
    fields as numpy arrays (empty in mode none)."""
    z = np.zeros(0, np.int64)
    st = {"color_bias": np.zeros((0, 3), np.int16), "video_index": z, "frame_cursor": z.copy(),
          "direction": np.zeros(0, np.int8), "frame_count": z.copy()}
    if mode == "none":
        return st
    g = np.arange(env_offset, env_offset + batch, dtype=np.uint64)
    hi, lo = threefry2x64_many(key[0], key[1], g, 1)
    if mode == "color":
        st["color_bias"] = _biases_from_keys(hi, lo)
        return st
    counts = np.asarray(frame_counts, dtype=np.int64)
    vidx = _video_from_keys(hi, lo, counts.size)
    return {"color_bias": np.zeros((batch, 3), np.int16), "video_index": vidx,
            "frame_cursor": np.zeros(batch, np.int64), "direction": np.ones(batch, np.int8),
            "frame_count": counts[vidx]}


def advance_state(st: dict, mode: str, key_t, env_offset: int, logical_batch: int,
                  frame_counts=None, done=None) -> dict:
    """One step of the distractor state as the reference's step() does it:
    advance_distractors (distractor.py:116-137), then for done envs the
    video re-draw from fold_in(key_t, logical_batch + env_offset + i)
    (env.py:226-244). Returns a new dict."""
    out = {k: v.copy() for k, v in st.items()}
    if mode == "color":
        out["color_bias"] = color_biases(key_t, env_offset, st["color_bias"].shape[0])
    elif mode == "video":
        out["frame_cursor"], out["direction"] = video_advance(
            st["frame_cursor"], st["direction"], st["frame_count"])
        if done is not None and np.any(done):
            idx = np.nonzero(np.asarray(done))[0]
            g = np.uint64(logical_batch + env_offset) + idx.astype(np.uint64)
            hi, lo = threefry2x64_many(key_t[0], key_t[1], g, 2)
            counts = np.asarray(frame_counts, dtype=np.int64)
            vidx = _video_from_keys(hi, lo, counts.size)
            out["video_index"][idx] = vidx
            out["frame_cursor"][idx] = 0
            out["direction"][idx] = 1
            out["frame_count"][idx] = counts[vidx]
    return out


def forward_kinematics(qpos: np.ndarray, parent, anchor) -> np.ndarray:
    """physics.py:114-137 in numpy: per-link [x, z, pitch] chained along parents."""
    qpos = np.asarray(qpos, dtype=np.float64)
    nl = len(parent)
    poses = np.zeros((qpos.shape[0], nl, 3), dtype=np.float64)
    poses[:, 0, :] = qpos[:, :3]
    for i in range(1, nl):
        p = int(parent[i])
        th = poses[:, p, 2]
        poses[:, i, 0] = poses[:, p, 0] + anchor[i] * np.cos(th)
        poses[:, i, 1] = poses[:, p, 1] + anchor[i] * np.sin(th)
        poses[:, i, 2] = th + qpos[:, 3 + i - 1]
    return poses


def pose_source(rest, parent, anchor, reset_key, env_offset: int, t: int, batch: int):
    """Host restatement of the benchmark pose source (csrc/pxr_ops.cu
    pose_source_kernel): qpos0 = rest + U(-0.1, 0.1) from the reference's
    reset keys (physics.py:499-503, prng.py:111-135), a deterministic joint
    oscillation, then forward kinematics -- numpy f64 sin/cos, so equal to
    the device's within a few ulp (the same workload, not the same bits)."""
    rest = np.asarray(rest, dtype=np.float64)
    dof = rest.size
    g = np.arange(env_offset, env_offset + batch, dtype=np.uint64)
    khi, klo = threefry2x64_many(reset_key[0], reset_key[1], g, 1)   # split(R, .)[g]
    fhi, flo = threefry2x64_many(khi, klo, np.zeros(batch, np.uint64), 2)  # fold_in(k, 0)
    q = np.empty((batch, dof), dtype=np.float64)
    for d in range(0, dof, 2):
        w0, w1 = threefry2x64_many(fhi, flo, np.full(batch, d // 2, np.uint64), 0)
        for k, w in enumerate((w0, w1)):
            if d + k < dof:
                u = (w >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
                q[:, d + k] = rest[d + k] + (-0.1 + u * 0.2)
    time_ = 0.01 * float(t)
    phase = (g % np.uint64(997)).astype(np.float64) * 0.37
    q[:, 0] += time_
    q[:, 1] += 0.03 * np.sin(6.0 * time_ + phase)
    q[:, 2] += 0.05 * np.sin(4.0 * time_ + phase)
    for j in range(3, dof):
        q[:, j] += 0.6 * np.sin(8.0 * time_ + phase + 1.3 * j)
    return forward_kinematics(q, parent, anchor)

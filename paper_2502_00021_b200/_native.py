"""ctypes binding of libpxr.so (the sm_100a kernels behind include/pxr.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2502_00021_b200/csrc``). There is deliberately no fallback: if the
shared object is missing, or no CUDA device is present when a kernel is
requested, the call raises -- the hot path never silently runs on the CPU.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
# PXR_LIB_PATH: load another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("PXR_LIB_PATH") or os.path.join(_HERE, "libpxr.so")
CSRC = os.path.join(_HERE, "csrc")

PXR_OK = 0
PXR_ERR_INVALID = 1
PXR_ERR_CUDA = 2
PXR_ERR_UNSUPPORTED = 3

MODE_NONE, MODE_COLOR, MODE_VIDEO = 0, 1, 2
MODES = {"none": MODE_NONE, "color": MODE_COLOR, "video": MODE_VIDEO}

# Every symbol include/pxr.h declares (tests check the .so exports them all).
EXPORTED = (
    "pxr_abi_version", "pxr_build_checked", "pxr_status_string", "pxr_last_error", "pxr_floor_rays",
    "pxr_render_step", "pxr_advance_distractors", "pxr_init_distractors",
    "pxr_apply_color", "pxr_apply_video", "pxr_grayscale", "pxr_threefry2x64",
    "pxr_sincosf", "pxr_pose_source", "pxr_forward_kinematics", "pxr_div_check",
    "pxr_physics_step", "pxr_reset_envs", "pxr_env_poses", "pxr_conv_stub_forward",
    "pxr_step_key_advance", "pxr_set_debug", "pxr_sincos", "pxr_log", "pxr_pack_upscale",
)

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64


class Geometry(ctypes.Structure):
    _fields_ = [
        ("base_verts", _vp), ("vert_link", _vp), ("triangles", _vp), ("tri_colors", _vp),
        ("n_verts", _i32), ("n_tris", _i32), ("n_links", _i32),
    ]


class Camera(ctypes.Structure):
    _fields_ = [
        ("block", ctypes.c_float * 15), ("offset_x", ctypes.c_double),
        ("offset_z", ctypes.c_double), ("light", ctypes.c_float * 3),
        ("floor_rays", _vp), ("floor_separable", _i32),
    ]


class Distractor(ctypes.Structure):
    _fields_ = [
        ("mode", _i32), ("color_bias", _vp), ("video_index", _vp),
        ("frame_cursor", _vp), ("direction", _vp), ("frame_count", _vp),
    ]


class VideoPackC(ctypes.Structure):
    _fields_ = [
        ("frames", _vp), ("starts", _vp), ("counts", _vp), ("n_videos", _i64),
        ("n_frames", _i64), ("height", _i64), ("width", _i64),
        ("frames_hw", _vp), ("hw_height", _i64), ("hw_width", _i64),
    ]


class StepKeys(ctypes.Structure):
    _fields_ = [("key_hi", _u64), ("key_lo", _u64), ("env_offset", _u64),
                ("logical_batch", _u64), ("device_key", _vp)]


class Model(ctypes.Structure):
    _fields_ = [
        ("parent", _vp), ("anchor_dist", _vp), ("length", _vp), ("mass", _vp),
        ("inertia", _vp), ("limit_lo", _vp), ("limit_hi", _vp), ("torque_max", _vp),
        ("rest_qpos", _vp), ("n_links", _i32), ("substeps", _i32), ("fixed_root", _i32),
        ("has_min_root_height", _i32), ("dt", ctypes.c_double),
        ("min_root_height", ctypes.c_double), ("forward_weight", ctypes.c_double),
        ("ctrl_cost", ctypes.c_double), ("episode_length", _i64),
    ]


_lib = None


class NativeError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile libpxr.so for sm_100a in-tree (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC] + (["-B"] if force else []), check=True)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """Load libpxr.so once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C {CSRC}); "
            "there is no CPU fallback for the render path"
        )
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    L.pxr_abi_version.restype = _i32
    L.pxr_abi_version.argtypes = []
    L.pxr_build_checked.restype = _i32
    L.pxr_build_checked.argtypes = []
    L.pxr_status_string.restype = ctypes.c_char_p
    L.pxr_status_string.argtypes = [_i32]
    L.pxr_last_error.restype = ctypes.c_char_p
    L.pxr_last_error.argtypes = []
    L.pxr_floor_rays.restype = _i32
    L.pxr_floor_rays.argtypes = [P(ctypes.c_float), _i64, _i64, _vp, P(_i32), _vp]
    L.pxr_render_step.restype = _i32
    L.pxr_render_step.argtypes = [
        P(Geometry), P(Camera), _vp, _i64, _i64, _i64, _i32, P(Distractor), P(VideoPackC),
        _i32, P(StepKeys), _vp, _i32, _vp, _vp, _vp,
    ]
    L.pxr_advance_distractors.restype = _i32
    L.pxr_advance_distractors.argtypes = [P(Distractor), P(VideoPackC), _i64, P(StepKeys), _vp, _vp]
    L.pxr_init_distractors.restype = _i32
    L.pxr_init_distractors.argtypes = [P(Distractor), P(VideoPackC), _i64, _u64, _u64, _u64, _vp]
    L.pxr_apply_color.restype = _i32
    L.pxr_apply_color.argtypes = [_vp, _vp, _i64, _i64, _i64, _vp]
    L.pxr_apply_video.restype = _i32
    L.pxr_apply_video.argtypes = [_vp, _vp, P(VideoPackC), _vp, _vp, _i64, _i64, _i64, _vp]
    L.pxr_grayscale.restype = _i32
    L.pxr_grayscale.argtypes = [_vp, _vp, _i64, _vp]
    L.pxr_threefry2x64.restype = _i32
    L.pxr_threefry2x64.argtypes = [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp]
    L.pxr_div_check.restype = _i32
    L.pxr_div_check.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp]
    L.pxr_sincosf.restype = _i32
    L.pxr_sincosf.argtypes = [_vp, _vp, _vp, _i64, _vp]
    L.pxr_pack_upscale.restype = _i32
    L.pxr_pack_upscale.argtypes = [P(VideoPackC), _i64, _i64, _vp, _vp]
    L.pxr_log.restype = _i32
    L.pxr_log.argtypes = [_vp, _vp, _i64, _vp]
    L.pxr_sincos.restype = _i32
    L.pxr_sincos.argtypes = [_vp, _vp, _vp, _i64, _vp]
    L.pxr_pose_source.restype = _i32
    L.pxr_pose_source.argtypes = [_vp, _vp, _vp, _i32, _u64, _u64, _u64, _i64, _i64, _vp, _vp]
    L.pxr_forward_kinematics.restype = _i32
    L.pxr_forward_kinematics.argtypes = [_vp, _vp, _vp, _i32, _i64, _vp, _vp]
    L.pxr_conv_stub_forward.restype = _i32
    L.pxr_conv_stub_forward.argtypes = [_vp, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _vp, _vp,
                                        _vp]
    L.pxr_physics_step.restype = _i32
    L.pxr_physics_step.argtypes = [P(Model), _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.pxr_reset_envs.restype = _i32
    L.pxr_reset_envs.argtypes = [P(Model), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64,
                                 _u64, _u64, _u64, _u64, _i32, _vp, _vp]
    L.pxr_step_key_advance.restype = _i32
    L.pxr_step_key_advance.argtypes = [_u64, _u64, _vp, _vp, _vp]
    L.pxr_env_poses.restype = _i32
    L.pxr_env_poses.argtypes = [P(Model), _vp, _i64, _vp, _vp]
    L.pxr_set_debug.restype = _i32
    L.pxr_set_debug.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
    if L.pxr_abi_version() != 3:
        raise ImportError(f"{LIB_PATH}: ABI version {L.pxr_abi_version()} != 3")
    _lib = L
    return L


def check(status: int) -> None:
    """Map a pxr_status to the reference's exception convention."""
    if status == PXR_OK:
        return
    msg = lib().pxr_last_error().decode(errors="replace")
    if status == PXR_ERR_INVALID:
        raise ValueError(msg)
    raise NativeError(f"{lib().pxr_status_string(status).decode()}: {msg}")


def set_debug(name: str, value) -> None:
    """Set (or, with None, unset) a PXR_DEBUG_* knob of the loaded library
    (forced raster budgets / bands / kernel variants for the tests). The
    library reads the environment once; this is the run-time override."""
    check(lib().pxr_set_debug(name.encode(), None if value is None else str(value).encode()))


def require_cuda():
    """The device the kernels run on; raises when there is none."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2502_00021_b200 renders on a CUDA device (sm_100a); none is "
            "available and there is no CPU fallback"
        )
    return torch.device("cuda", torch.cuda.current_device())


_NO_SCOPE = contextlib.nullcontext()


def device_scope(device):
    """Make ``device`` current for the launches inside (kernels go to that
    device's current stream; the library's per-device launch facts follow).
    Already current (the common case): no context switch at all."""
    import torch

    idx = device.index if isinstance(device, torch.device) else None
    if idx is not None and idx == torch._C._cuda_getDevice():
        return _NO_SCOPE
    return torch.cuda.device(device)


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of ``stream``, or of the current device's current
    stream (read straight from the CUDA state: the per-launch host cost of the
    small-batch loop)."""
    import torch

    if stream is not None:
        return int(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(torch._C._cuda_getDevice()))
    return int(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None stays NULL)."""
    if t is None:
        return None
    return int(t.data_ptr())

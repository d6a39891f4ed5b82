"""Batched robot renderer on the B200 (host side of the render path).

Mirrors ``pixelctrl.render`` (/root/reference/pkg/src/pixelctrl/render.py):
constants (50-68), ``Mesh``/``Pose``/``Camera``/``CameraConfig``/``Frame``
(71-130), tessellation (137-230), the tracking camera (237-279),
``RobotGeometry`` (559-591), ``render_robot_batch`` (594-623) and the generic
scene API ``render`` / ``render_batch`` (491-552) on the same raster kernel.

What changes is where the work runs: tessellation and the camera block are
host-side and one-time (as in the reference); every per-step array --
poses in, pixels and depth out -- lives in HBM, and the per-env world
transform, projection, triangle setup, z-buffered raster and shading run in
the fused sm_100a kernel behind ``pxr_render_step`` (csrc/pxr_render.cu).
There is no CPU path: without a CUDA device these functions raise.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "SKY_COLOR", "FLOOR_LIGHT", "FLOOR_DARK", "AMBIENT", "DIFFUSE", "LIGHT_DIR",
    "LINK_PALETTE", "Mesh", "Pose", "Camera", "CameraConfig", "Frame",
    "tessellate_capsule", "tessellate_sphere", "track_camera", "camera_basis",
    "RobotGeometry", "RobotRenderer", "render_robot_batch", "render", "render_batch",
]

SKY_COLOR = (135, 206, 235)
FLOOR_LIGHT = (158, 158, 158)
FLOOR_DARK = (122, 122, 122)
AMBIENT = 0.35
DIFFUSE = 0.65
_l = np.array([0.3, -0.5, 0.8])
LIGHT_DIR = tuple(_l / np.linalg.norm(_l))
LIGHT_F32 = np.asarray(LIGHT_DIR, dtype=np.float32)
LINK_PALETTE = (
    (0.85, 0.30, 0.23),
    (0.23, 0.50, 0.85),
    (0.30, 0.75, 0.35),
    (0.93, 0.74, 0.13),
    (0.62, 0.40, 0.80),
    (0.20, 0.78, 0.75),
    (0.90, 0.50, 0.15),
)


@dataclass(frozen=True)
class Mesh:
    vertices: np.ndarray  # (V, 3) float32
    triangles: np.ndarray  # (T, 3) int32
    base_color: tuple


@dataclass(frozen=True)
class Pose:
    x: float = 0.0
    y: float = 0.0
    z: float = 0.0
    pitch: float = 0.0


@dataclass(frozen=True)
class Camera:
    eye: tuple
    target: tuple
    up: tuple = (0.0, 0.0, 1.0)
    vertical_fov: float = 0.9
    near: float = 0.1
    far: float = 50.0


@dataclass(frozen=True)
class CameraConfig:
    offset: tuple = (0.0, -3.0, 1.2)
    vertical_fov: float = 0.9
    near: float = 0.1
    far: float = 50.0


@dataclass
class Frame:
    """Batched observation buffers in HBM (render.py:108-130).

    ``pixels`` (B, H, W, 3) uint8 and ``depth`` (B, H, W) float32 are CUDA
    tensors; +inf depth marks background.
    """

    pixels: object
    depth: object

    @classmethod
    def allocate(cls, batch: int, height: int, width: int, device=None) -> "Frame":
        import torch

        if height < 8 or width < 8:
            raise ValueError("frames must be at least 8x8")
        dev = device if device is not None else _native.require_cuda()
        return cls(
            pixels=torch.zeros((batch, height, width, 3), dtype=torch.uint8, device=dev),
            depth=torch.zeros((batch, height, width), dtype=torch.float32, device=dev),
        )

    @property
    def background_mask(self):
        import torch

        return torch.isinf(self.depth)

    @property
    def batch(self) -> int:
        return int(self.pixels.shape[0])


# ---------------------------------------------------------------- meshes


def tessellate_sphere(radius: float, rings: int, sectors: int) -> Mesh:
    """UV sphere, render.py:137-168 vertex/triangle order."""
    if radius <= 0 or rings < 2 or sectors < 3:
        raise ValueError("sphere needs radius > 0, rings >= 2, sectors >= 3")
    verts = [(0.0, 0.0, radius), (0.0, 0.0, -radius)]
    for k in range(1, rings):
        phi = math.pi * k / rings
        sp, cp = math.sin(phi), math.cos(phi)
        for s in range(sectors):
            ang = 2.0 * math.pi * s / sectors
            verts.append((radius * sp * math.cos(ang), radius * sp * math.sin(ang), radius * cp))

    def ring(k, s):
        return 2 + (k - 1) * sectors + (s % sectors)

    tris = []
    for s in range(sectors):
        tris.append((0, ring(1, s), ring(1, s + 1)))
        tris.append((1, ring(rings - 1, s + 1), ring(rings - 1, s)))
    for k in range(1, rings - 1):
        for s in range(sectors):
            a, b, c, d = ring(k, s), ring(k, s + 1), ring(k + 1, s), ring(k + 1, s + 1)
            tris += [(a, c, d), (a, d, b)]
    return Mesh(np.array(verts, dtype=np.float32), np.array(tris, dtype=np.int32),
                LINK_PALETTE[0])


def tessellate_capsule(radius: float, length: float, rings: int = 8, sectors: int = 12,
                       base_color=LINK_PALETTE[0]) -> Mesh:
    """Closed capsule along local +x (render.py:171-230): poles, then each
    cap's latitude rings from pole to seam; triangles cap 0, cap 1, barrel."""
    if radius <= 0 or length <= 0:
        raise ValueError("capsule needs radius > 0 and length > 0")
    if rings < 2 or sectors < 3:
        raise ValueError("capsule needs rings >= 2 and sectors >= 3")
    hx = length / 2.0
    verts = [(hx + radius, 0.0, 0.0), (-hx - radius, 0.0, 0.0)]
    for sign in (1.0, -1.0):
        for k in range(1, rings + 1):
            phi = (math.pi / 2.0) * k / rings
            for s in range(sectors):
                ang = 2.0 * math.pi * s / sectors
                verts.append((
                    sign * (hx + radius * math.cos(phi)),
                    radius * math.sin(phi) * math.cos(ang),
                    radius * math.sin(phi) * math.sin(ang),
                ))

    def ring(side, k, s):
        return 2 + side * rings * sectors + (k - 1) * sectors + (s % sectors)

    tris = []
    for side in (0, 1):
        for s in range(sectors):  # pole fan, winding flipped on the second cap
            a, b = ring(side, 1, s), ring(side, 1, s + 1)
            tris.append((side, a, b) if side == 0 else (side, b, a))
        for k in range(1, rings):
            for s in range(sectors):
                a, b = ring(side, k, s), ring(side, k, s + 1)
                c, d = ring(side, k + 1, s), ring(side, k + 1, s + 1)
                tris += [(a, c, d), (a, d, b)] if side == 0 else [(a, d, c), (a, b, d)]
    for s in range(sectors):  # barrel between the two seams
        a, b = ring(0, rings, s), ring(0, rings, s + 1)
        c, d = ring(1, rings, s), ring(1, rings, s + 1)
        tris += [(a, d, c), (a, b, d)]
    return Mesh(np.array(verts, dtype=np.float32), np.array(tris, dtype=np.int32),
                base_color)


# ---------------------------------------------------------------- camera


def track_camera(root_pos, config: CameraConfig = CameraConfig()) -> Camera:
    """render.py:237-249."""
    x, z = float(root_pos[0]), float(root_pos[1])
    ox, oy, oz = config.offset
    return Camera(eye=(x + ox, oy, z + oz), target=(x, 0.0, z),
                  vertical_fov=config.vertical_fov, near=config.near, far=config.far)


def camera_basis(camera: Camera) -> np.ndarray:
    """15-float block [eye, right, up, fwd, tan(fov/2), near, far], built in
    f64 and stored f32 (render.py:252-279, same validation messages)."""
    eye = np.array(camera.eye, dtype=np.float64)
    fwd = np.array(camera.target, dtype=np.float64) - eye
    n = np.linalg.norm(fwd)
    if n == 0:
        raise ValueError("camera target coincides with eye")
    fwd /= n
    right = np.cross(fwd, np.array(camera.up, dtype=np.float64))
    rn = np.linalg.norm(right)
    if rn == 0:
        raise ValueError("camera up is parallel to the view direction")
    right /= rn
    upc = np.cross(right, fwd)
    if not 0.0 < camera.vertical_fov < math.pi:
        raise ValueError("vertical_fov outside (0, pi)")
    if not 0.0 < camera.near < camera.far:
        raise ValueError("need 0 < near < far")
    out = np.empty(15, dtype=np.float32)
    out[0:3] = eye
    out[3:6] = right
    out[6:9] = upc
    out[9:12] = fwd
    out[12] = math.tan(camera.vertical_fov / 2.0)
    out[13] = camera.near
    out[14] = camera.far
    return out


# ---------------------------------------------------------------- geometry


class RobotGeometry:
    """Per-model capsule links flattened for the kernel (render.py:559-591).

    Host arrays are built once (coarse capsules: rings=3, sectors=8, 96
    triangles per link) and uploaded once per device; triangle index order
    is the z-buffer tie-break order and is preserved exactly.
    """

    def __init__(self, lengths, radii, rings: int = 3, sectors: int = 8):
        verts, links, tris, cols = [], [], [], []
        base = 0
        for i, (length, radius) in enumerate(zip(lengths, radii)):
            color = LINK_PALETTE[i % len(LINK_PALETTE)]
            mesh = tessellate_capsule(radius, length, rings, sectors, color)
            v = mesh.vertices.copy()
            v[:, 0] += np.float32(length / 2.0)  # link spans origin..tip
            verts.append(v)
            links.append(np.full(len(v), i, dtype=np.int32))
            tris.append(mesh.triangles + base)
            cols.append(np.tile(np.array(color, dtype=np.float32), (len(mesh.triangles), 1)))
            base += len(v)
        self.n_links = len(verts)
        self.base_verts = np.ascontiguousarray(np.concatenate(verts), dtype=np.float32)
        self.vert_link = np.ascontiguousarray(np.concatenate(links), dtype=np.int32)
        self.triangles = np.ascontiguousarray(np.concatenate(tris), dtype=np.int32)
        self.tri_colors = np.ascontiguousarray(np.concatenate(cols), dtype=np.float32)
        self._dev = {}

    @property
    def triangle_count(self) -> int:
        return len(self.triangles)

    def device_arrays(self, device):
        """Upload once per device; returns (tensors, pxr_geometry struct)."""
        import torch

        key = str(device)
        if key not in self._dev:
            t = {
                "base_verts": torch.from_numpy(self.base_verts).to(device),
                "vert_link": torch.from_numpy(self.vert_link).to(device),
                "triangles": torch.from_numpy(self.triangles).to(device),
                "tri_colors": torch.from_numpy(self.tri_colors).to(device),
            }
            g = _native.Geometry(
                t["base_verts"].data_ptr(), t["vert_link"].data_ptr(),
                t["triangles"].data_ptr(), t["tri_colors"].data_ptr(),
                len(self.base_verts), len(self.triangles), self.n_links,
            )
            self._dev[key] = (t, g)
        return self._dev[key]


class RobotRenderer:
    """Device-resident render setup for one (geometry, camera config, W, H):
    uploaded mesh, the shared camera block and the exact floor ray table.
    ``render_robot_batch`` and ``Env`` reuse one of these per configuration."""

    def __init__(self, geom: RobotGeometry, cam_config: CameraConfig, width: int,
                 height: int, device=None):
        import torch

        if width < 8 or height < 8:
            raise ValueError("frames must be at least 8x8")
        self.device = device if device is not None else _native.require_cuda()
        self.device = torch.device(self.device)
        if self.device.index is None:  # "cuda" -> the current device, explicitly
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.geom = geom
        self.width, self.height = int(width), int(height)
        self.cam_config = cam_config
        self._geom_t, self.geom_c = geom.device_arrays(self.device)
        # render.py:607-612: orientation from the camera tracking (0, 0)
        self.cam_block = camera_basis(track_camera((0.0, 0.0), cam_config))
        self.floor_rays = torch.empty((self.height, self.width, 3), dtype=torch.float64,
                                      device=self.device)
        sep = ctypes.c_int32(0)
        blk = (ctypes.c_float * 15)(*self.cam_block.tolist())
        with torch.cuda.device(self.device):
            _native.check(_native.lib().pxr_floor_rays(
                blk, self.height, self.width, self.floor_rays.data_ptr(), ctypes.byref(sep),
                _native.stream_ptr()))
        self.cam_c = _native.Camera(
            blk, float(cam_config.offset[0]), float(cam_config.offset[2]),
            (ctypes.c_float * 3)(*LIGHT_F32.tolist()), self.floor_rays.data_ptr(),
            int(sep.value),
        )

    def render(self, poses, *, floor_in_background: bool, dist=None, pack=None,
               advance: bool = False, keys=None, done=None, grayscale: bool = False,
               out_obs=None, out_depth=None, want_depth: bool = True, stream=None):
        """One fused launch (pxr_render_step). ``poses`` (B, L, 3) f64 on the
        device. Returns (obs, depth-or-None)."""
        import torch

        if poses.dtype != torch.float64 or poses.device.type != "cuda":
            raise ValueError("poses must be a float64 CUDA tensor")
        if poses.device != self.device:  # (both carry an index)
            raise ValueError(f"poses are on {poses.device}, the renderer on {self.device}")
        with _native.device_scope(self.device):
            return self._render(poses, floor_in_background, dist, pack, advance, keys, done,
                                grayscale, out_obs, out_depth, want_depth, stream)

    def _render(self, poses, floor_in_background, dist, pack, advance, keys, done, grayscale,
                out_obs, out_depth, want_depth, stream):
        import torch

        poses = poses.contiguous()
        B = int(poses.shape[0])
        if poses.dim() != 3 or poses.shape[1] != self.geom.n_links or poses.shape[2] != 3:
            raise ValueError(
                f"poses must be (batch, {self.geom.n_links}, 3), got {tuple(poses.shape)}")
        C = 1 if grayscale else 3
        if out_obs is None:
            out_obs = torch.empty((B, self.height, self.width, C), dtype=torch.uint8,
                                  device=poses.device)
        if out_depth is None and want_depth:
            out_depth = torch.empty((B, self.height, self.width), dtype=torch.float32,
                                    device=poses.device)
        dist_c = dist.c_struct() if dist is not None else _native.Distractor(_native.MODE_NONE)
        # RGB video: the pack's frames upscaled to this renderer's size (TMA copy)
        pack_c = (pack.c_struct(self.height, self.width) if not grayscale else pack.c_struct()) \
            if pack is not None else None
        keys_c = keys
        done_p = _native.ptr(done)
        st = _native.stream_ptr(stream)
        _native.check(_native.lib().pxr_render_step(
            ctypes.byref(self.geom_c), ctypes.byref(self.cam_c), poses.data_ptr(), B,
            self.height, self.width, int(not floor_in_background), ctypes.byref(dist_c),
            ctypes.byref(pack_c) if pack_c is not None else None, int(advance),
            ctypes.byref(keys_c) if keys_c is not None else None, done_p, int(grayscale),
            out_obs.data_ptr(), _native.ptr(out_depth), st))
        return out_obs, out_depth


_RENDERERS: dict = {}


def _renderer_for(geom, cam_config, width, height, device) -> RobotRenderer:
    key = (id(geom), cam_config, width, height, str(device))
    r = _RENDERERS.get(key)
    if r is None or r.geom is not geom:
        r = RobotRenderer(geom, cam_config, width, height, device)
        _RENDERERS[key] = r
    return r


def render_robot_batch(geom: RobotGeometry, poses, cam_config: CameraConfig, width: int,
                       height: int, floor_in_background: bool, threads: int = 1,
                       out: Frame | None = None) -> Frame:
    """render.py:594-623 on the B200: every env's robot with its own tracking
    camera, pixels and depth returned as CUDA tensors. ``poses`` (B, L, 3)
    float64, a CUDA tensor or a host array (copied to the device once).
    ``threads`` is accepted for signature parity and ignored: the CUDA grid
    replaces the host thread pool (threading_utils.py:32-42)."""
    import torch

    dev = _native.require_cuda()
    if width < 8 or height < 8:
        raise ValueError("frames must be at least 8x8")
    if not isinstance(poses, torch.Tensor):
        poses = torch.from_numpy(np.ascontiguousarray(poses, dtype=np.float64))
    poses = poses.to(device=dev, dtype=torch.float64)
    r = _renderer_for(geom, cam_config, int(width), int(height), dev)
    if out is None:
        out = Frame.allocate(int(poses.shape[0]), int(height), int(width), device=dev)
    r.render(poses, floor_in_background=floor_in_background, out_obs=out.pixels,
             out_depth=out.depth)
    return out


# ---------------------------------------------------------------- scenes


def _scene_world(meshes):
    """World-space vertices, triangles and per-triangle colours of a scene,
    with the reference's arithmetic (render.py:504-522): Python f64 cos/sin
    of the pitch rounded to f32, then f32 ``(x + vx c) - vz s``,
    ``y + vy``, ``(z + vx s) + vz c``; triangle indices offset per mesh in
    list order (the z-buffer tie-break order)."""
    verts, tris, cols = [], [], []
    base = 0
    for mesh, pose in meshes:
        v = np.asarray(mesh.vertices, dtype=np.float32)
        cf, sf = np.float32(math.cos(pose.pitch)), np.float32(math.sin(pose.pitch))
        w = np.empty_like(v)
        w[:, 0] = (np.float32(pose.x) + v[:, 0] * cf) - v[:, 2] * sf
        w[:, 1] = np.float32(pose.y) + v[:, 1]
        w[:, 2] = (np.float32(pose.z) + v[:, 0] * sf) + v[:, 2] * cf
        t = np.asarray(mesh.triangles, dtype=np.int32)
        verts.append(w)
        tris.append(t + np.int32(base))
        cols.append(np.broadcast_to(np.asarray(mesh.base_color, dtype=np.float32), (len(t), 3)))
        base += len(v)
    if not verts:
        return (np.zeros((0, 3), np.float32), np.zeros((0, 3), np.int32),
                np.zeros((0, 3), np.float32))
    return (np.ascontiguousarray(np.concatenate(verts)), np.ascontiguousarray(np.concatenate(tris)),
            np.ascontiguousarray(np.concatenate(cols)))


def _render_scene_into(meshes, camera: Camera, light_dir, width: int, height: int,
                       floor_in_background: bool, pixels, depth, device) -> None:
    """One scene through pxr_render_step: the world-space mesh is a one-link
    geometry at the identity pose, the camera block is ``camera_basis`` and
    the per-env camera position is the block's eye."""
    import torch

    blk_np = camera_basis(camera)
    verts, tris, cols = _scene_world(meshes)
    if len(verts) > 65535 or len(tris) > 65535:
        raise ValueError("scene too large for the raster kernel (max 65535 vertices / triangles)")
    t = {
        "v": torch.from_numpy(verts).to(device),
        "l": torch.zeros(len(verts), dtype=torch.int32, device=device),
        "t": torch.from_numpy(tris).to(device),
        "c": torch.from_numpy(cols).to(device),
        "pose": torch.zeros((1, 1, 3), dtype=torch.float64, device=device),
        "rays": torch.empty((height, width, 3), dtype=torch.float64, device=device),
    }
    geom_c = _native.Geometry(t["v"].data_ptr(), t["l"].data_ptr(), t["t"].data_ptr(),
                              t["c"].data_ptr(), len(verts), len(tris), 1)
    blk = (ctypes.c_float * 15)(*blk_np.tolist())
    sep = ctypes.c_int32(0)
    st = _native.stream_ptr()
    _native.check(_native.lib().pxr_floor_rays(blk, height, width, t["rays"].data_ptr(),
                                               ctypes.byref(sep), st))
    light = np.asarray(light_dir, dtype=np.float32)
    cam_c = _native.Camera(blk, float(blk_np[0]), float(blk_np[2]),
                           (ctypes.c_float * 3)(*light.tolist()), t["rays"].data_ptr(),
                           int(sep.value))
    dist_c = _native.Distractor(_native.MODE_NONE)
    _native.check(_native.lib().pxr_render_step(
        ctypes.byref(geom_c), ctypes.byref(cam_c), t["pose"].data_ptr(), 1, height, width,
        int(not floor_in_background), ctypes.byref(dist_c), None, 0, None, None, 0,
        pixels.data_ptr(), depth.data_ptr(), st))


def render(meshes, camera: Camera, light_dir=LIGHT_DIR, width: int = 84, height: int = 84,
           floor_in_background: bool = False) -> Frame:
    """render.py:491-533 on the B200: one scene of posed meshes, a batch-1
    ``Frame`` of CUDA tensors, bit-identical to the reference."""
    if width < 8 or height < 8:
        raise ValueError("render needs width, height >= 8")
    dev = _native.require_cuda()
    frame = Frame.allocate(1, int(height), int(width), device=dev)
    _render_scene_into(list(meshes), camera, light_dir, int(width), int(height),
                       floor_in_background, frame.pixels, frame.depth, dev)
    return frame


def render_batch(scenes, width: int = 84, height: int = 84, floor_in_background: bool = False,
                 light_dir=LIGHT_DIR) -> Frame:
    """render.py:536-552: independent scenes, scene i bit-identical to
    ``render(scene i)``. The reference renders the batch on a thread pool;
    here every scene's world-space mesh goes up in one upload, each scene
    is one single-CTA launch (its own camera, floor-ray table and mesh), and
    the launches are spread over several CUDA streams so the scenes render
    concurrently on different SMs."""
    import torch

    scenes = list(scenes)
    if not scenes:
        raise ValueError("render_batch needs at least one scene")
    if width < 8 or height < 8:
        raise ValueError("render needs width, height >= 8")
    W, H = int(width), int(height)
    dev = _native.require_cuda()
    frame = Frame.allocate(len(scenes), H, W, device=dev)
    light = np.asarray(light_dir, dtype=np.float32)
    worlds = [_scene_world(list(meshes)) for meshes, _ in scenes]
    for verts, tris, _ in worlds:
        if len(verts) > 65535 or len(tris) > 65535:
            raise ValueError("scene too large for the raster kernel (max 65535 vertices / triangles)")
    nvs = [len(w[0]) for w in worlds]
    nts = [len(w[1]) for w in worlds]
    voff = np.concatenate([[0], np.cumsum(nvs)]).astype(np.int64)
    toff = np.concatenate([[0], np.cumsum(nts)]).astype(np.int64)
    # one upload for the whole batch (each scene's geometry points into it)
    verts = torch.from_numpy(np.concatenate([w[0] for w in worlds]).reshape(-1, 3)
                             if voff[-1] else np.zeros((1, 3), np.float32)).to(dev)
    tris = torch.from_numpy(np.concatenate([w[1] for w in worlds]).reshape(-1, 3)
                            if toff[-1] else np.zeros((1, 3), np.int32)).to(dev)
    cols = torch.from_numpy(np.concatenate([w[2] for w in worlds]).reshape(-1, 3)
                            if toff[-1] else np.zeros((1, 3), np.float32)).to(dev)
    links = torch.zeros(max(1, int(voff[-1])), dtype=torch.int32, device=dev)
    pose = torch.zeros((1, 1, 3), dtype=torch.float64, device=dev)
    rays = torch.empty((len(scenes), H, W, 3), dtype=torch.float64, device=dev)
    L = _native.lib()
    main = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(device=dev) for _ in range(min(len(scenes), 8))]
    for s in streams:
        s.wait_stream(main)  # (the uploads above)
    keep = []
    dist_c = _native.Distractor(_native.MODE_NONE)
    for i, (meshes, camera) in enumerate(scenes):
        st = _native.stream_ptr(streams[i % len(streams)])
        blk_np = camera_basis(camera)
        blk = (ctypes.c_float * 15)(*blk_np.tolist())
        sep = ctypes.c_int32(0)
        _native.check(L.pxr_floor_rays(blk, H, W, rays[i].data_ptr(), ctypes.byref(sep), st))
        geom_c = _native.Geometry(verts[int(voff[i]):].data_ptr(), links.data_ptr(),
                                  tris[int(toff[i]):].data_ptr(), cols[int(toff[i]):].data_ptr(),
                                  nvs[i], nts[i], 1)
        cam_c = _native.Camera(blk, float(blk_np[0]), float(blk_np[2]),
                               (ctypes.c_float * 3)(*light.tolist()), rays[i].data_ptr(),
                               int(sep.value))
        keep.append((blk, geom_c, cam_c))
        _native.check(L.pxr_render_step(
            ctypes.byref(geom_c), ctypes.byref(cam_c), pose.data_ptr(), 1, H, W,
            int(not floor_in_background), ctypes.byref(dist_c), None, 0, None, None, 0,
            frame.pixels[i:i + 1].data_ptr(), frame.depth[i:i + 1].data_ptr(), st))
    for s in streams:
        main.wait_stream(s)
    # the uploads and tables are in use on the side streams until they finish
    for t in (verts, tris, cols, links, pose, rays):
        for s in streams:
            t.record_stream(s)
    return frame

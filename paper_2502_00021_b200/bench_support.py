"""Benchmark workloads: one BASELINE configuration resident
on the device -- geometry, camera/floor tables, video pack, distractor
state -- plus an on-device pose source, so a "rendered env-step" is exactly
poses(t) -> fused render/distractor/grayscale kernel -> obs in HBM.

The pose source replaces physics (out of scope for the render hot path and
timed separately, per BASELINE.json): qpos = rest + U(-0.1, 0.1) drawn with
the reference's reset keys, plus a deterministic per-joint oscillation, then
f64 forward kinematics -- all in one kernel (pxr_pose_source).
"""

from __future__ import annotations

from . import _native
from .distractor import init_distractors, step_keys
from .models import ROSTER, model_kinematics, resolve_model
from .prng import fold_in, key_from_seed
from .render import CameraConfig, RobotGeometry, RobotRenderer
from .video_pack import generate_synthetic_pack

__all__ = ["Workload", "synthetic_pack", "MODEL_ALIASES"]

MODEL_ALIASES = {
    "cheetah_lite": "cheetah_lite", "walker_lite": "walker_lite", "hopper_lite": "hopper_lite",
    "ant_lite": ROSTER["Ant"], "humanoid_lite": ROSTER["Humanoid"],
    "HalfCheetah": ROSTER["HalfCheetah"], "Walker2d": ROSTER["Walker2d"],
    "Ant": ROSTER["Ant"], "Humanoid": ROSTER["Humanoid"],
}

_PACKS: dict = {}


def synthetic_pack(videos: int = 4, frames: int = 60, size: int = 64, seed: int = 2024):
    """The reference's shipped synthetic pack recipe (`pixelctrl synth --seed
    2024 --videos 4 --frames 60 --size 64x64`, SHA-256 a8907f57...)."""
    key = (videos, frames, size, seed)
    if key not in _PACKS:
        _PACKS[key] = generate_synthetic_pack(key_from_seed(seed), videos, frames, size, size)
    return _PACKS[key]


class Workload:
    """One configuration (model, B envs/GPU, distractor mode) on one device."""

    def __init__(self, model: str, batch: int, mode: str, seed: int = 0, env_offset: int = 0,
                 logical_batch: int | None = None, width: int = 84, height: int = 84,
                 grayscale: bool = False, pack=None, device=None):
        import torch

        self.device = device if device is not None else _native.require_cuda()
        self.model = model
        self.spec = resolve_model(MODEL_ALIASES.get(model, model))
        parent, anchor, length, radius = model_kinematics(self.spec)
        self.geom = RobotGeometry(length, radius)
        self.batch = int(batch)
        self.mode = mode
        self.env_offset = int(env_offset)
        self.logical_batch = int(logical_batch if logical_batch is not None else batch)
        self.grayscale = bool(grayscale)
        self.floor_in_background = mode == "video"  # env.py:81-85 default
        self.width, self.height = int(width), int(height)
        self.master = key_from_seed(seed)
        self._keys: dict = {}
        self.reset_key = fold_in(self.master, 0x5EED)
        self.renderer = RobotRenderer(self.geom, CameraConfig(), width, height, self.device)
        self.pack = None
        self.dpack = None
        if mode == "video":
            self.pack = pack if pack is not None else synthetic_pack()
            self.dpack = self.pack.to_device(self.device)
        self.dist = init_distractors(mode, self.pack, fold_in(self.master, 0xD157), self.batch,
                                     env_offset=self.env_offset, device=self.device)
        self._rest = torch.from_numpy(self.spec.rest()).to(self.device)
        self._parent = torch.from_numpy(parent).to(self.device)
        self._anchor = torch.from_numpy(anchor).to(self.device)
        self.poses_buf = torch.empty((self.batch, self.spec.n_links, 3), dtype=torch.float64,
                                     device=self.device)
        C = 1 if grayscale else 3
        self.obs = torch.empty((self.batch, height, width, C), dtype=torch.uint8,
                               device=self.device)

    @property
    def n_links(self) -> int:
        return self.spec.n_links

    def obs_bytes_per_env(self) -> int:
        return self.height * self.width * (1 if self.grayscale else 3)

    def state_bytes_per_env(self) -> int:
        """Distractor state read+written per env-step by the fused kernel."""
        if self.mode == "color":
            return 6  # int16 x3 written (biases are drawn, not read)
        if self.mode == "video":
            return 2 * (8 + 8 + 1) + 8 + 8  # idx, cursor, dir r/w + count + start
        return 0

    def poses(self, t: int, out=None, stream=None):
        out = self.poses_buf if out is None else out
        _native.check(_native.lib().pxr_pose_source(
            self._rest.data_ptr(), self._parent.data_ptr(), self._anchor.data_ptr(),
            self.spec.n_links, self.reset_key.hi, self.reset_key.lo, self.env_offset, int(t),
            self.batch, out.data_ptr(), _native.stream_ptr(stream)))
        return out

    def step_keys(self, t: int):
        """The launch's step keys (key_t = fold_in(master, t), env.py:209),
        memoised: the host Threefry costs ~18 us in Python, more than a
        small batch's whole render, so timed loops precompute them."""
        k = self._keys.get(t)
        if k is None:
            k = step_keys(fold_in(self.master, t), self.env_offset, self.logical_batch)
            self._keys[t] = k
        return k

    def precompute_keys(self, ts) -> None:
        for t in ts:
            self.step_keys(t)

    def render(self, poses, t: int, advance: bool = True, want_depth: bool = False,
               out_obs=None, stream=None, done=None):
        """The rendered env-step proper: key_t = fold_in(master, t), advance
        distractors, render, composite, postprocess -- one launch."""
        keys = self.step_keys(t)
        return self.renderer.render(
            poses, floor_in_background=self.floor_in_background, dist=self.dist,
            pack=self.dpack, advance=advance, keys=keys, done=done, grayscale=self.grayscale,
            out_obs=self.obs if out_obs is None else out_obs, want_depth=want_depth,
            stream=stream)

    def step(self, t: int, want_depth: bool = False):
        """pose source + fused render for step t (two launches)."""
        p = self.poses(t)
        return self.render(p, t, want_depth=want_depth)

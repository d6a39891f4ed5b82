"""Throughput sweep with the conv-stub policy in the loop, on the B200.

Mirrors ``pixelctrl.bench`` (/root/reference/pkg/src/pixelctrl/bench.py):
``ConvStub`` / ``conv_stub_forward`` (36-145), ``BenchConfig`` /
``BenchRecord`` / ``run_benchmark`` (148-236) and the CSV format (239-277).
The policy forward runs in ``pxr_conv_stub_forward`` (csrc/pxr_policy.cu):
a per-env convolution kernel and a fixed-order projection kernel, so a row
never depends on its batch; observations, actions and the env state stay on
the device through the whole loop. The repo-root
``bench.py`` is the driver's render benchmark; this module is the
reference's env-step sweep.
"""

from __future__ import annotations

import ctypes
import hashlib
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .prng import fold_in, key_from_seed, uniform

__all__ = [
    "ConvStub",
    "conv_stub_forward",
    "BenchConfig",
    "BenchRecord",
    "run_benchmark",
    "write_csv",
    "read_csv",
]

KERNEL_SIZE = 8
STRIDE = 4
N_FILTERS = 16


def _glorot(key, rows: int, cols: int) -> np.ndarray:
    """(rows, cols) float32 Glorot-uniform weights from one Threefry stream
    (the reference's draw: uniform(key, rows * cols, -s, s), s = sqrt(6 / rows))."""
    s = float(np.sqrt(6.0 / rows))
    return uniform(key, rows * cols, -s, s).astype(np.float32).reshape(rows, cols)


def _quadrant_blocks(conv: np.ndarray, channels: int) -> np.ndarray:
    """The 8x8 kernel as its four 4x4 quadrants side by side: column block q
    = 2 dy + dx holds quadrant (dy, dx) (the reference's conv_blocks)."""
    k = conv.reshape(2, STRIDE, 2, STRIDE, channels, N_FILTERS)
    quads = [k[q // 2, :, q % 2].reshape(-1, N_FILTERS) for q in range(4)]
    return np.ascontiguousarray(np.hstack(quads), dtype=np.float32)


@dataclass(frozen=True)
class ConvStub:
    """The reference's fixed policy surrogate (bench.py:40-88); weights are a
    pure function of the seed: conv rows in (ky, kx, c) order from stream
    fold_in(key, 0), projection rows in (oy, ox, f) order from fold_in(key, 1).
    ``conv_blocks`` keeps the reference's quadrant layout for API parity."""

    conv: np.ndarray         # (K*K*C, filters) float32
    conv_blocks: np.ndarray  # (STRIDE*STRIDE*C, 4*filters) float32
    proj: np.ndarray         # (out_h*out_w*filters, n_joints) float32
    height: int
    width: int
    channels: int
    n_joints: int

    @classmethod
    def create(cls, height: int, width: int, channels: int, n_joints: int, seed: int = 0):
        positions = ((height - KERNEL_SIZE) // STRIDE + 1) * ((width - KERNEL_SIZE) // STRIDE + 1)
        if height < KERNEL_SIZE or width < KERNEL_SIZE:
            raise ValueError("observation smaller than the conv kernel")
        root = key_from_seed(seed)
        conv = _glorot(fold_in(root, 0), KERNEL_SIZE * KERNEL_SIZE * channels, N_FILTERS)
        proj = _glorot(fold_in(root, 1), positions * N_FILTERS, n_joints)
        return cls(conv, _quadrant_blocks(conv, channels), proj, height, width, channels,
                   n_joints)

    def device_weights(self, device):
        """(conv, proj) float32 CUDA tensors, uploaded once per device."""
        import torch

        cache = self.__dict__.setdefault("_dev", {})
        key = str(device)
        if key not in cache:
            cache[key] = (torch.from_numpy(np.ascontiguousarray(self.conv)).to(device),
                          torch.from_numpy(np.ascontiguousarray(self.proj)).to(device))
        return cache[key]


def conv_stub_forward(stub: ConvStub, obs, threads: int = 1):
    """Actions in [-1, 1] (bench.py:131-145); batch row i depends only on obs
    row i. ``obs`` (B, H, W, C) uint8: a CUDA tensor (result: float64 CUDA
    tensor, no host round trip) or a host array (result: float64 ndarray).
    ``threads`` is accepted for signature parity and ignored."""
    import torch

    host = not isinstance(obs, torch.Tensor)
    shape = tuple(np.shape(obs)) if host else tuple(obs.shape)
    if len(shape) != 4 or shape[1:] != (stub.height, stub.width, stub.channels):
        raise ValueError(
            f"obs must be (batch, {stub.height}, {stub.width}, {stub.channels}), got {shape}")
    dev = _native.require_cuda() if host or obs.device.type != "cuda" else obs.device
    x = torch.from_numpy(np.ascontiguousarray(obs, dtype=np.uint8)) if host else obs
    x = x.to(device=dev, dtype=torch.uint8).contiguous()
    conv, proj = stub.device_weights(dev)
    out = torch.empty((shape[0], stub.n_joints), dtype=torch.float64, device=dev)
    ws = torch.empty((max(shape[0], 1), stub.proj.shape[0]), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _native.check(_native.lib().pxr_conv_stub_forward(
            x.data_ptr(), shape[0], stub.height, stub.width, stub.channels, conv.data_ptr(),
            proj.data_ptr(), stub.n_joints, out.data_ptr(), ws.data_ptr(), _native.stream_ptr()))
    return out.cpu().numpy() if host else out


# ---------------------------------------------------------------- protocol


@dataclass(frozen=True)
class BenchRecord:
    env_name: str
    batch: int
    distractor_mode: str
    steps_measured: int
    wall_seconds: float
    steps_per_second: float
    resolution: str
    digest: str = ""  # reproducibility hash; not part of the CSV schema


@dataclass(frozen=True)
class BenchConfig:
    env_names: tuple = ("cheetah_lite", "walker_lite", "hopper_lite")
    batches: tuple = (1, 10, 100, 1000)
    distractor_modes: tuple = ("none",)
    video_pack_path: str | None = None
    warmup_steps: int = 50
    measure_steps: int = 500
    width: int = 84
    height: int = 84
    seed: int = 0
    threads: int = 1

    def validate(self) -> None:
        if self.measure_steps < 100:
            raise ValueError("measure_steps must be >= 100")
        if "video" in self.distractor_modes and not self.video_pack_path:
            raise ValueError("video mode needs video_pack_path")


def _bench_one(config: BenchConfig, env_name: str, batch: int, mode: str) -> BenchRecord:
    """bench.py:183-216: policy forward + env step per iteration, everything
    on the device; the clock stops after the device has finished. The
    iteration is one replay of a CUDA graph of (policy, step) (env.StepGraph:
    same results as the step loop, bit for bit; at small batches the loop is
    otherwise launch-bound)."""
    import torch

    from .env import EnvConfig, StepGraph, make_env

    cfg = EnvConfig(model=env_name, batch=batch, width=config.width, height=config.height,
                    distractor_mode=mode,
                    video_pack_path=config.video_pack_path if mode == "video" else None,
                    seed=config.seed, threads=config.threads)
    env, state, obs = make_env(cfg)
    stub = ConvStub.create(config.height, config.width, int(obs.shape[-1]), env.n_joints,
                           seed=config.seed)
    g = StepGraph(env, state, obs, lambda o: conv_stub_forward(stub, o))
    g.replay(config.warmup_steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.replay(config.measure_steps)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    obs = g.obs
    steps = batch * config.measure_steps
    return BenchRecord(env_name=env_name, batch=batch, distractor_mode=mode,
                       steps_measured=steps, wall_seconds=wall, steps_per_second=steps / wall,
                       resolution=f"{config.width}x{config.height}",
                       digest=hashlib.sha256(obs.cpu().numpy().tobytes()).hexdigest())


def run_benchmark(config: BenchConfig, progress=None) -> list:
    """One record per (env, mode, batch) in the reference's order."""
    config.validate()
    records = []
    for env_name in config.env_names:
        for mode in config.distractor_modes:
            for batch in config.batches:
                rec = _bench_one(config, env_name, batch, mode)
                records.append(rec)
                if progress is not None:
                    progress(rec)
    return records


# ---------------------------------------------------------------- CSV

_CSV_COLUMNS = ("env", "batch", "distractor", "steps", "seconds", "sps", "resolution")
_CSV_HEADER = ",".join(_CSV_COLUMNS)


def _csv_row(r: BenchRecord) -> str:
    """One record in the reference's CSV schema (bench.py:239-250): floats
    at 6 significant digits, the digest left out."""
    cells = (r.env_name, r.batch, r.distractor_mode, r.steps_measured,
             f"{r.wall_seconds:.6g}", f"{r.steps_per_second:.6g}", r.resolution)
    return ",".join(str(c) for c in cells)


def write_csv(records, path) -> None:
    try:
        with open(path, "w") as fh:
            fh.write("\n".join([_CSV_HEADER] + [_csv_row(r) for r in records]) + "\n")
    except OSError as e:
        raise OSError(f"cannot write benchmark CSV to {path}: {e}") from e


def read_csv(path) -> list:
    with open(path) as fh:
        rows = [line.strip() for line in fh if line.strip()]
    if not rows or rows[0] != _CSV_HEADER:
        raise ValueError(f"{path}: missing benchmark CSV header")
    out = []
    for line in rows[1:]:
        cell = dict(zip(_CSV_COLUMNS, line.split(",")))
        out.append(BenchRecord(env_name=cell["env"], batch=int(cell["batch"]),
                               distractor_mode=cell["distractor"],
                               steps_measured=int(cell["steps"]),
                               wall_seconds=float(cell["seconds"]),
                               steps_per_second=float(cell["sps"]),
                               resolution=cell["resolution"]))
    return out

"""Planar articulated-body physics API on the B200.

Mirrors ``pixelctrl.physics`` (/root/reference/pkg/src/pixelctrl/physics.py):
``SystemState`` (51-67), ``ModelArrays`` / ``model_arrays`` (70-111),
``forward_kinematics`` (114-137), ``step_dynamics`` (427-465),
``compute_reward`` (468-477), ``check_termination`` (480-484),
``reset_state`` (487-510) and ``mechanical_energy`` (513-545).

State arrays are CUDA tensors; the dynamics, resets and kinematics run in
``csrc/pxr_physics.cu`` (one thread per env, f64, the reference's operation
order). Reset draws are bit-exact; the dynamics differ from the reference
only through CUDA's f64 cos/sin/log.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .models import ModelSpec, model_kinematics
from .prng import Key

__all__ = [
    "GRAVITY", "SystemState", "ModelArrays", "model_arrays", "DeviceModel",
    "forward_kinematics", "step_dynamics", "compute_reward", "check_termination",
    "reset_state", "mechanical_energy",
]

GRAVITY = 9.81


@dataclass
class SystemState:
    """Batched generalized state (physics.py:51-67) as CUDA tensors."""

    qpos: object       # (B, dof) f64
    qvel: object       # (B, dof) f64
    step_count: object  # (B,) i64
    done: object       # (B,) u8 (bool semantics)

    @property
    def batch(self) -> int:
        return int(self.qpos.shape[0])

    def copy(self) -> "SystemState":
        return SystemState(self.qpos.clone(), self.qvel.clone(), self.step_count.clone(),
                           self.done.clone())


class ModelArrays:
    """ModelSpec flattened to host arrays (physics.py:75-99)."""

    def __init__(self, spec: ModelSpec):
        spec.validate()
        self.spec = spec
        parent, anchor, length, radius = model_kinematics(spec)
        self.parent = parent.astype(np.int64)
        self.anchor_dist = anchor
        self.length = length
        self.radius = radius
        self.mass = np.array([l.mass for l in spec.links], dtype=np.float64)
        # rod with end caps about the centre, axis out of plane (physics.py:70-72)
        self.inertia = np.array([l.mass * (l.length * l.length / 12.0 + l.radius * l.radius / 4.0)
                                 for l in spec.links], dtype=np.float64)
        self.limit_lo = np.array([j.limit_lo for j in spec.joints], dtype=np.float64)
        self.limit_hi = np.array([j.limit_hi for j in spec.joints], dtype=np.float64)
        self.torque_max = np.array([j.torque_max for j in spec.joints], dtype=np.float64)


_ARRAYS: dict = {}


def model_arrays(spec: ModelSpec) -> ModelArrays:
    a = _ARRAYS.get(id(spec))
    if a is None or a.spec is not spec:
        a = ModelArrays(spec)
        _ARRAYS[id(spec)] = a
    return a


class DeviceModel:
    """A ModelSpec uploaded once per device plus its ``pxr_model`` struct."""

    def __init__(self, spec: ModelSpec, device):
        import torch

        m = model_arrays(spec)

        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device)

        pad = (lambda a: a if len(a) else np.zeros(1))
        self.spec = spec
        self.device = device
        self._t = {
            "parent": dev(m.parent.astype(np.int32)), "anchor": dev(m.anchor_dist),
            "length": dev(m.length), "mass": dev(m.mass), "inertia": dev(m.inertia),
            "lo": dev(pad(m.limit_lo)), "hi": dev(pad(m.limit_hi)),
            "tq": dev(pad(m.torque_max)), "rest": dev(spec.rest()),
        }
        t = self._t
        self.c = _native.Model(
            t["parent"].data_ptr(), t["anchor"].data_ptr(), t["length"].data_ptr(),
            t["mass"].data_ptr(), t["inertia"].data_ptr(), t["lo"].data_ptr(),
            t["hi"].data_ptr(), t["tq"].data_ptr(), t["rest"].data_ptr(), spec.n_links,
            spec.substeps, int(spec.fixed_root), int(spec.min_root_height is not None),
            spec.dt, float(spec.min_root_height or 0.0), spec.forward_weight, spec.ctrl_cost,
            spec.episode_length,
        )


_DEV_MODELS: dict = {}


def _device_model(spec: ModelSpec, device) -> DeviceModel:
    key = (id(spec), str(device))
    dm = _DEV_MODELS.get(key)
    if dm is None or dm.spec is not spec:
        dm = DeviceModel(spec, device)
        _DEV_MODELS[key] = dm
    return dm


def _f64(a, device):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)


def _as_device_state(state, device) -> SystemState:
    import torch

    if isinstance(state.qpos, torch.Tensor):
        return state
    return SystemState(_f64(state.qpos, device), _f64(state.qvel, device),
                       torch.from_numpy(np.asarray(state.step_count, np.int64)).to(device),
                       torch.from_numpy(np.asarray(state.done).astype(np.uint8)).to(device))


def forward_kinematics(spec: ModelSpec, qpos):
    """physics.py:114-137: per-link world poses (B, L, 3) ``[x, z, pitch]``."""
    import torch

    dev = qpos.device if isinstance(qpos, torch.Tensor) and qpos.is_cuda else \
        _native.require_cuda()
    q = _f64(qpos, dev)
    if q.dim() != 2 or q.shape[1] != spec.dof:
        raise ValueError(f"qpos must be (batch, {spec.dof}), got {tuple(q.shape)}")
    dm = _device_model(spec, dev)
    out = torch.empty((q.shape[0], spec.n_links, 3), dtype=torch.float64, device=dev)
    _native.check(_native.lib().pxr_env_poses(ctypes.byref(dm.c), q.data_ptr(), q.shape[0],
                                              out.data_ptr(), _native.stream_ptr()))
    return out


def step_dynamics(spec: ModelSpec, state: SystemState, actions, threads: int = 1) -> SystemState:
    """physics.py:427-465: one control step (``substeps`` semi-implicit Euler
    substeps) for every env; returns a new state (the input is unchanged).
    ``threads`` is accepted for signature parity and ignored."""
    import torch

    dev = state.qpos.device if isinstance(state.qpos, torch.Tensor) else _native.require_cuda()
    st = _as_device_state(state, dev)
    act = _f64(actions, dev)
    if tuple(act.shape) != (st.batch, spec.n_joints):
        raise ValueError(f"actions must be {(st.batch, spec.n_joints)}, got {tuple(act.shape)}")
    if tuple(st.qpos.shape) != (st.batch, spec.dof):
        raise ValueError(f"qpos must be {(st.batch, spec.dof)}, got {tuple(st.qpos.shape)}")
    if act.numel() == 0:  # no joints: the kernel still wants a valid pointer
        act = torch.zeros(1, dtype=torch.float64, device=dev)
    out = st.copy()
    scratch = torch.zeros(st.batch, dtype=torch.float64, device=dev)  # reward (unused here)
    dm = _device_model(spec, dev)
    _native.check(_native.lib().pxr_physics_step(
        ctypes.byref(dm.c), out.qpos.data_ptr(), out.qvel.data_ptr(), out.step_count.data_ptr(),
        out.done.data_ptr(), act.data_ptr(), scratch.data_ptr(), st.batch, _native.stream_ptr()))
    return out


def _np_row_sum(x):
    """Row sums of a (B, n) f64 tensor in numpy's pairwise order
    (np.sum(axis=1) on C-contiguous rows: sequential below 8 terms, else 8
    interleaved partial sums combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
    then the tail; n <= 128 here)."""
    n = x.shape[1]
    if n < 8:
        acc = x[:, 0].clone()
        for i in range(1, n):
            acc = acc + x[:, i]
        return acc
    r = [x[:, i].clone() for i in range(8)]
    i = 8
    while i + 8 <= n:
        for k in range(8):
            r[k] = r[k] + x[:, i + k]
        i += 8
    acc = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
    for k in range(i, n):
        acc = acc + x[:, k]
    return acc


def compute_reward(spec: ModelSpec, prev: SystemState, next: SystemState, actions):
    """physics.py:468-477: ``forward_weight * (dx / dt) - ctrl_cost * |a|^2``
    with actions clipped to [-1, 1], on the device."""
    import torch

    dev = next.qpos.device if isinstance(next.qpos, torch.Tensor) else _native.require_cuda()
    a = torch.clamp(_f64(actions, dev), -1.0, 1.0)
    p, q = _f64(prev.qpos, dev), _f64(next.qpos, dev)
    if a.shape[0] != p.shape[0] or p.shape[0] != q.shape[0]:
        raise ValueError("batch sizes disagree")
    # divide by a device tensor: ATen turns `tensor / python_float` into a
    # multiply by the host-rounded reciprocal, which is not IEEE division
    dt = torch.tensor(spec.dt, dtype=torch.float64, device=dev)
    forward = (q[:, 0] - p[:, 0]) / dt
    ctrl = _np_row_sum(a * a) if a.shape[1] > 0 else torch.zeros_like(forward)
    return spec.forward_weight * forward - spec.ctrl_cost * ctrl


def check_termination(spec: ModelSpec, state: SystemState):
    """physics.py:480-484: root below ``min_root_height`` (bool tensor)."""
    import torch

    q = _f64(state.qpos, state.qpos.device if isinstance(state.qpos, torch.Tensor)
             else _native.require_cuda())
    if spec.min_root_height is None:
        return torch.zeros(q.shape[0], dtype=torch.bool, device=q.device)
    return q[:, 1] < spec.min_root_height


def reset_state(spec: ModelSpec, key: Key, batch: int, env_offset: int = 0,
                device=None) -> SystemState:
    """physics.py:487-510 on the device: rest pose + U(-0.1, 0.1) and
    0.05 * N(0, 1) velocities from ``split(key, env_offset + batch)``, one
    subkey per global env index (bit-exact draws)."""
    import torch

    if batch < 1:
        raise ValueError(f"batch must be >= 1, got {batch}")
    dev = device if device is not None else _native.require_cuda()
    dm = _device_model(spec, dev)
    dof = spec.dof
    sys = SystemState(torch.empty((batch, dof), dtype=torch.float64, device=dev),
                      torch.empty((batch, dof), dtype=torch.float64, device=dev),
                      torch.zeros(batch, dtype=torch.int64, device=dev),
                      torch.zeros(batch, dtype=torch.uint8, device=dev))
    ret = torch.zeros(batch, dtype=torch.float64, device=dev)
    length = torch.zeros(batch, dtype=torch.int64, device=dev)
    _native.check(_native.lib().pxr_reset_envs(
        ctypes.byref(dm.c), sys.qpos.data_ptr(), sys.qvel.data_ptr(), sys.step_count.data_ptr(),
        sys.done.data_ptr(), ret.data_ptr(), length.data_ptr(), None, None, None, batch,
        key.hi, key.lo, env_offset, env_offset + batch, 0, None, _native.stream_ptr()))
    return sys


def mechanical_energy(spec: ModelSpec, state: SystemState):
    """physics.py:513-545 (test aid): kinetic + gravitational potential
    energy per env, f64 on the device."""
    import torch

    m = model_arrays(spec)
    poses = forward_kinematics(spec, state.qpos)
    qv = _f64(state.qvel, poses.device)
    B, nl = poses.shape[0], spec.n_links
    omega = [qv[:, 2]] + [None] * (nl - 1)
    vx = [qv[:, 0]] + [None] * (nl - 1)
    vz = [qv[:, 1]] + [None] * (nl - 1)
    for i in range(1, nl):
        p = int(m.parent[i])
        th = poses[:, p, 2]
        a = float(m.anchor_dist[i])
        vx[i] = vx[p] - omega[p] * a * torch.sin(th)
        vz[i] = vz[p] + omega[p] * a * torch.cos(th)
        omega[i] = omega[p] + qv[:, 3 + i - 1]
    energy = torch.zeros(B, dtype=torch.float64, device=poses.device)
    for i in range(nl):
        h = 0.5 * float(m.length[i])
        th = poses[:, i, 2]
        cz = poses[:, i, 1] + h * torch.sin(th)
        vcx = vx[i] - omega[i] * h * torch.sin(th)
        vcz = vz[i] + omega[i] * h * torch.cos(th)
        energy = energy + 0.5 * float(m.mass[i]) * (vcx ** 2 + vcz ** 2)
        energy = energy + 0.5 * float(m.inertia[i]) * omega[i] ** 2
        energy = energy + float(m.mass[i]) * GRAVITY * cz
    return energy

"""Colour and video distractors on the device.

Mirrors ``pixelctrl.distractor`` (/root/reference/pkg/src/pixelctrl/
distractor.py): the same ``DistractorState`` fields (36-55) held as CUDA
tensors, the same key derivations (66-113), the pure ``advance_distractors``
(116-137), ``apply_color``/``apply_video`` with their in-place variants
(184-228) and ``nearest_map`` (179-181). Each call is one kernel launch on
the current stream; in the env step the advance and the composite are fused
into the render kernel instead (csrc/pxr_render.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .prng import Key
from .render import Frame

__all__ = [
    "COLOR_BIAS_RANGE", "DistractorState", "init_distractors", "advance_distractors",
    "apply_color", "apply_video", "apply_color_inplace", "apply_video_inplace",
    "nearest_map", "sample_video_indices", "step_keys",
]

COLOR_BIAS_RANGE = 60
MODES = ("none", "color", "video")


@dataclass
class DistractorState:
    """Per-env distractor bookkeeping in HBM (empty tensors in mode none)."""

    mode: str
    color_bias: object    # (B, 3) int16
    video_index: object   # (B,) int64
    frame_cursor: object  # (B,) int64
    direction: object     # (B,) int8
    frame_count: object   # (B,) int64

    def copy(self) -> "DistractorState":
        return DistractorState(self.mode, self.color_bias.clone(), self.video_index.clone(),
                               self.frame_cursor.clone(), self.direction.clone(),
                               self.frame_count.clone())

    @property
    def batch(self) -> int:
        if self.mode == "color":
            return int(self.color_bias.shape[0])
        return int(self.video_index.shape[0])

    def c_struct(self) -> _native.Distractor:
        m = _native.MODES[self.mode]
        if m == _native.MODE_NONE:
            return _native.Distractor(m)
        return _native.Distractor(
            m, _native.ptr(self.color_bias) if self.color_bias.numel() else None,
            _native.ptr(self.video_index) if self.video_index.numel() else None,
            _native.ptr(self.frame_cursor) if self.frame_cursor.numel() else None,
            _native.ptr(self.direction) if self.direction.numel() else None,
            _native.ptr(self.frame_count) if self.frame_count.numel() else None,
        )

    def to_host(self) -> dict:
        """numpy copies of every field (tests / digests)."""
        return {
            "color_bias": self.color_bias.cpu().numpy(),
            "video_index": self.video_index.cpu().numpy(),
            "frame_cursor": self.frame_cursor.cpu().numpy(),
            "direction": self.direction.cpu().numpy(),
            "frame_count": self.frame_count.cpu().numpy(),
        }


def _empty(mode: str, device, batch: int = 0, with_bias: bool = False) -> DistractorState:
    import torch

    z = torch.zeros(0, dtype=torch.int64, device=device)
    return DistractorState(
        mode, torch.zeros((batch if with_bias else 0, 3), dtype=torch.int16, device=device),
        z, z.clone(), torch.zeros(0, dtype=torch.int8, device=device), z.clone())


def step_keys(key_t: Key, env_offset: int = 0, logical_batch: int = 0) -> _native.StepKeys:
    return _native.StepKeys(key_t.hi, key_t.lo, env_offset, logical_batch)


def init_distractors(mode: str, pack, key: Key, batch: int, env_offset: int = 0,
                     device=None) -> DistractorState:
    """distractor.py:82-113: one subkey per env, split(key, off + B)[off:],
    drawn on the device."""
    import torch

    if mode not in MODES:
        raise ValueError(f"unknown distractor mode {mode!r}")
    if batch < 1:
        raise ValueError(f"batch must be >= 1, got {batch}")
    dev = device if device is not None else _native.require_cuda()
    if mode == "none":
        return _empty(mode, dev)
    if mode == "color":
        st = _empty(mode, dev, batch, with_bias=True)
        _native.check(_native.lib().pxr_init_distractors(
            ctypes.byref(st.c_struct()), None, batch, key.hi, key.lo, env_offset,
            _native.stream_ptr()))
        return st
    if pack is None:
        raise ValueError("video distractors need a loaded video pack")
    dp = pack.to_device(dev)
    st = DistractorState(
        "video", torch.zeros((batch, 3), dtype=torch.int16, device=dev),
        torch.empty(batch, dtype=torch.int64, device=dev),
        torch.empty(batch, dtype=torch.int64, device=dev),
        torch.empty(batch, dtype=torch.int8, device=dev),
        torch.empty(batch, dtype=torch.int64, device=dev))
    _native.check(_native.lib().pxr_init_distractors(
        ctypes.byref(st.c_struct()), ctypes.byref(dp.c_struct()), batch, key.hi, key.lo,
        env_offset, _native.stream_ptr()))
    return st


def advance_distractors(state: DistractorState, key_t: Key, env_offset: int = 0,
                        pack=None) -> DistractorState:
    """distractor.py:116-137, pure: returns an advanced copy. Colour biases of
    env i come from fold_in(key_t, env_offset + i); video cursors ping-pong."""
    out = state.copy()
    if state.mode == "none":
        return out
    B = out.batch
    pack_c = None
    if state.mode == "video" and pack is not None:
        pack_c = pack.to_device(out.video_index.device).c_struct()
    keys = step_keys(key_t, env_offset, 0)
    _native.check(_native.lib().pxr_advance_distractors(
        ctypes.byref(out.c_struct()), ctypes.byref(pack_c) if pack_c is not None else None,
        B, ctypes.byref(keys), None, _native.stream_ptr()))
    return out


def sample_video_indices(hi, lo, n_videos: int):
    """distractor.py:77-79 on the device: words_per_key(.., 2).x0 -> [0, n)."""
    from .prng import index_from_words, words_per_key

    w0, _ = words_per_key(hi, lo, 2)
    return index_from_words(w0.cpu().numpy(), n_videos)


def nearest_map(dst: int, src: int) -> np.ndarray:
    """distractor.py:179-181."""
    return (np.arange(dst, dtype=np.int64) * src) // dst


def apply_color_inplace(frame: Frame, state: DistractorState, threads: int = 1) -> None:
    """distractor.py:184-193: clamp-add of the env's bias on every pixel."""
    if state.mode != "color":
        raise ValueError(f"apply_color needs mode=color, got {state.mode!r}")
    if frame.batch != int(state.color_bias.shape[0]):
        raise ValueError("frame batch does not match distractor state")
    B, H, W, _ = frame.pixels.shape
    bias = state.color_bias.to(frame.pixels.device).contiguous()
    _native.check(_native.lib().pxr_apply_color(
        frame.pixels.data_ptr(), bias.data_ptr(), B, H, W, _native.stream_ptr()))


def apply_video_inplace(frame: Frame, pack, state: DistractorState, threads: int = 1) -> None:
    """distractor.py:196-214: background pixels take the env's current
    video frame through nearest-neighbour scaling; foreground untouched."""
    if state.mode != "video":
        raise ValueError(f"apply_video needs mode=video, got {state.mode!r}")
    if frame.batch != int(state.video_index.shape[0]):
        raise ValueError("frame batch does not match distractor state")
    dp = pack.to_device(frame.pixels.device)
    B, H, W, _ = frame.pixels.shape
    _native.check(_native.lib().pxr_apply_video(
        frame.pixels.data_ptr(), frame.depth.contiguous().data_ptr(),
        ctypes.byref(dp.c_struct()), state.video_index.data_ptr(),
        state.frame_cursor.data_ptr(), B, H, W, _native.stream_ptr()))


def apply_color(frame: Frame, state: DistractorState) -> Frame:
    out = Frame(frame.pixels.clone(), frame.depth.clone())
    apply_color_inplace(out, state)
    return out


def apply_video(frame: Frame, pack, state: DistractorState) -> Frame:
    out = Frame(frame.pixels.clone(), frame.depth.clone())
    apply_video_inplace(out, pack, state)
    return out

"""Video-pack ingestion and generation (host tooling, one-time).

Mirrors ``pixelctrl.video_tools`` (/root/reference/pkg/src/pixelctrl/
video_tools.py): ``PackSummary`` (25-29), ``read_ppm`` / ``write_ppm``
(31-68), ``pack_from_frames`` (77-103: per-video subdirectories of PPM
frames, names ascending, nearest-neighbour resize) and
``generate_synthetic_pack`` (106-134, writing the pack and returning its
summary). The pack is the distractor path's input format; it is uploaded to
HBM once per env (``VideoPack.to_device``).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .distractor import nearest_map
from .video_pack import VideoPack, save_video_pack
from .video_pack import generate_synthetic_pack as _synthetic

__all__ = ["PackSummary", "pack_from_frames", "generate_synthetic_pack", "read_ppm",
           "write_ppm"]


@dataclass(frozen=True)
class PackSummary:
    videos: int
    total_frames: int
    bytes: int


def _ppm_header(data: bytes):
    """Four whitespace-separated header tokens (``#`` comments skipped) and
    the offset of the single whitespace byte that ends the header."""
    tokens, pos = [], 0
    while len(tokens) < 4:
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if pos >= len(data):
            raise ValueError("header truncated")
        if data[pos:pos + 1] == b"#":
            end = data.find(b"\n", pos)
            pos = len(data) if end < 0 else end
            continue
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        tokens.append(data[start:pos])
    return tokens, pos


def read_ppm(path) -> np.ndarray:
    """Binary (P6, maxval 255) PPM -> (H, W, 3) uint8."""
    with open(path, "rb") as f:
        data = f.read()
    try:
        (magic, w, h, maxval), pos = _ppm_header(data)
        if magic != b"P6":
            raise ValueError("not a binary P6 PPM")
        w, h, maxval = int(w), int(h), int(maxval)
        if maxval != 255:
            raise ValueError(f"unsupported maxval {maxval}")
        body = data[pos + 1:pos + 1 + w * h * 3]
        if len(body) != w * h * 3:
            raise ValueError("pixel data truncated")
    except (ValueError, IndexError) as e:
        raise ValueError(f"{path}: cannot decode PPM ({e})") from None
    return np.frombuffer(body, dtype=np.uint8).reshape(h, w, 3).copy()


def write_ppm(frame, path) -> None:
    """Inverse of ``read_ppm``."""
    img = np.ascontiguousarray(frame, dtype=np.uint8)
    with open(path, "wb") as f:
        f.write(b"P6\n%d %d\n255\n" % (img.shape[1], img.shape[0]) + img.tobytes())


def pack_from_frames(root, out_path, height: int, width: int) -> PackSummary:
    """PXVP pack from ``root/<video>/<frame>.ppm`` (subdirectories and frames
    in ascending name order; each frame nearest-resized to height x width)."""
    subdirs = sorted(d for d in os.listdir(root) if os.path.isdir(os.path.join(root, d)))
    if not subdirs:
        raise ValueError(f"{root}: no video subdirectories")
    rows, cols = None, None
    videos = []
    for sub in subdirs:
        vdir = os.path.join(root, sub)
        frames = []
        for name in sorted(n for n in os.listdir(vdir) if not n.startswith(".")):
            img = read_ppm(os.path.join(vdir, name))
            rows = nearest_map(height, img.shape[0])
            cols = nearest_map(width, img.shape[1])
            frames.append(img[rows][:, cols])
        if len(frames) < 2:
            raise ValueError(f"{vdir}: a video needs at least 2 frames")
        videos.append(np.stack(frames).astype(np.uint8))
    nbytes = save_video_pack(VideoPack(videos=videos, height=height, width=width), out_path)
    return PackSummary(videos=len(videos), total_frames=sum(len(v) for v in videos),
                       bytes=nbytes)


def generate_synthetic_pack(key, videos: int, frames: int, height: int, width: int,
                            out_path) -> PackSummary:
    """Procedural moving-gradient pack written to ``out_path`` (pure in
    ``key``; the recipe lives in ``video_pack.generate_synthetic_pack``)."""
    pack = _synthetic(key, videos, frames, height, width)
    nbytes = save_video_pack(pack, out_path)
    return PackSummary(videos=videos, total_frames=videos * frames, bytes=nbytes)

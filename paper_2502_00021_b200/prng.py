"""Splittable counter-based PRNG: Threefry-2x64-20 with domain-tagged counters.

Same bitstream and API as the reference (``pixelctrl.prng``,
/root/reference/pkg/src/pixelctrl/prng.py): draw / split / fold counters are
``(i, 0)`` / ``(i, 1)`` / ``(data, 2)`` (prng.py:39-42, 93-121), pinned by
the reference's golden vectors (reference tests/test_prng.py:20-74, mirrored
in tests/test_prng.py here).

Scalar key plumbing (``key_from_seed``, ``fold_in``, ``split`` ...) runs on
the host in Python integers -- it is O(1) per step, exactly like the
reference. The per-env batched derivations on the hot path
(``fold_in_many``, ``words_per_key``) run on the device through
``pxr_threefry2x64`` and return CUDA tensors; inside the fused render kernel
the same Threefry code derives every env's colour bias and reset key
without any host round trip.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native

__all__ = [
    "Key",
    "key_from_seed",
    "split",
    "fold_in",
    "random_bits",
    "uniform",
    "normal",
    "random_index",
    "fold_in_many",
    "words_per_key",
    "index_from_words",
    "threefry2x64",
]

MASK64 = (1 << 64) - 1
ROTATIONS = (16, 42, 12, 31, 16, 32, 24, 21)  # prng.py:33
PARITY = 0x1BD11BDAA9FC1FFA  # prng.py:34
SEED_KEY = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)  # prng.py:37
TAG_DRAW, TAG_SPLIT, TAG_FOLD = 0, 1, 2  # prng.py:40-42


@dataclass(frozen=True)
class Key:
    """Opaque 128-bit generator state (a value type), prng.py:45-54."""

    hi: int
    lo: int

    def __post_init__(self):
        object.__setattr__(self, "hi", self.hi & MASK64)
        object.__setattr__(self, "lo", self.lo & MASK64)


def threefry2x64(k0: int, k1: int, c0: int, c1: int) -> tuple[int, int]:
    """One Threefry-2x64-20 block on Python ints (prng.py:57-77)."""
    k0 &= MASK64
    k1 &= MASK64
    ks = (k0, k1, k0 ^ k1 ^ PARITY)
    x0 = (c0 + ks[0]) & MASK64
    x1 = (c1 + ks[1]) & MASK64
    for r in range(20):
        rot = ROTATIONS[r % 8]
        x0 = (x0 + x1) & MASK64
        x1 = ((x1 << rot) | (x1 >> (64 - rot))) & MASK64
        x1 ^= x0
        if r % 4 == 3:
            j = r // 4 + 1
            x0 = (x0 + ks[j % 3]) & MASK64
            x1 = (x1 + ks[(j + 1) % 3] + j) & MASK64
    return x0, x1


def key_from_seed(seed: int) -> Key:
    """prng.py:85-90."""
    return Key(*threefry2x64(SEED_KEY[0], SEED_KEY[1], seed & MASK64, 0))


def split(key: Key, n: int) -> list[Key]:
    """prng.py:93-102: ``split(k, n)[i] = TF(k, (i, 1))``."""
    if n < 1:
        raise ValueError(f"split needs n >= 1, got {n}")
    return [Key(*threefry2x64(key.hi, key.lo, i, TAG_SPLIT)) for i in range(n)]


def fold_in(key: Key, data: int) -> Key:
    """prng.py:105-108."""
    return Key(*threefry2x64(key.hi, key.lo, data & MASK64, TAG_FOLD))


def random_bits(key: Key, n: int) -> np.ndarray:
    """prng.py:111-121: ``n`` uint64 words of the key's draw stream."""
    if n < 1:
        raise ValueError(f"random_bits needs n >= 1, got {n}")
    out = np.empty(2 * ((n + 1) // 2), dtype=np.uint64)
    for b in range((n + 1) // 2):
        out[2 * b], out[2 * b + 1] = threefry2x64(key.hi, key.lo, b, TAG_DRAW)
    return out[:n]


def uniform(key: Key, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """prng.py:124-135: 53-bit mantissa from the high bits, capped below hi."""
    if not lo < hi:
        raise ValueError(f"uniform needs lo < hi, got [{lo}, {hi})")
    bits = random_bits(key, n)
    u = (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    vals = lo + u * (hi - lo)
    return np.minimum(vals, np.nextafter(hi, -np.inf))


def normal(key: Key, n: int) -> np.ndarray:
    """prng.py:138-152: Box-Muller over 2*ceil(n/2) words."""
    if n < 1:
        raise ValueError(f"normal needs n >= 1, got {n}")
    m = (n + 1) // 2
    bits = random_bits(key, 2 * m)
    u1 = ((bits[:m] >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)
    u2 = (bits[m:] >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    r = np.sqrt(-2.0 * np.log(u1))
    theta = 2.0 * math.pi * u2
    out = np.empty(2 * m, dtype=np.float64)
    out[:m] = r * np.cos(theta)
    out[m:] = r * np.sin(theta)
    return out[:n]


def random_index(key: Key, n: int) -> int:
    """prng.py:155-161: multiply-shift of one word onto [0, n)."""
    if n < 1:
        raise ValueError(f"random_index needs n >= 1, got {n}")
    word = threefry2x64(key.hi, key.lo, 0, TAG_DRAW)[0]
    return (word * n) >> 64


def index_from_words(words, n: int):
    """prng.py:181-193: floor(w * n / 2^64) for every word (host numpy)."""
    if not 1 <= n < 2**32:
        raise ValueError(f"n must be in [1, 2^32), got {n}")
    w = np.asarray(words, dtype=np.uint64)
    un = np.uint64(n)
    w_hi = w >> np.uint64(32)
    w_lo = w & np.uint64(0xFFFFFFFF)
    return ((w_hi * un + ((w_lo * un) >> np.uint64(32))) >> np.uint64(32)).astype(np.int64)


# ---------------------------------------------------------------- device


def _as_device_u64(x, device):
    import torch

    if isinstance(x, torch.Tensor):
        t = x.to(device=device)
        if t.dtype != torch.uint64:
            t = t.to(torch.int64).view(torch.uint64) if t.dtype != torch.int64 else t.view(torch.uint64)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.uint64))
    return torch.from_numpy(arr.view(np.int64)).to(device).view(torch.uint64)


def _threefry_device(k0, k1, c0, c1_value: int):
    """TF(k, (c0, c1)) on the device; k0/k1 scalars or per-element tensors."""
    import torch

    dev = _native.require_cuda()
    c0 = _as_device_u64(c0, dev).reshape(-1)
    n = c0.numel()
    scalar_key = isinstance(k0, int)
    if scalar_key:
        k0t = _as_device_u64([k0 & MASK64], dev)
        k1t = _as_device_u64([k1 & MASK64], dev)
    else:
        k0t = _as_device_u64(k0, dev).reshape(-1)
        k1t = _as_device_u64(k1, dev).reshape(-1)
    c1t = _as_device_u64([c1_value], dev)
    y0 = torch.empty(n, dtype=torch.uint64, device=dev)
    y1 = torch.empty(n, dtype=torch.uint64, device=dev)
    _native.check(_native.lib().pxr_threefry2x64(
        k0t.data_ptr(), k1t.data_ptr(), 0 if scalar_key else 1, c0.data_ptr(),
        c1t.data_ptr(), 0, y0.data_ptr(), y1.data_ptr(), n, _native.stream_ptr()))
    return y0, y1


def fold_in_many(key: Key, data):
    """prng.py:168-171 on the device: element i equals fold_in(key, data[i])."""
    return _threefry_device(key.hi, key.lo, data, TAG_FOLD)


def words_per_key(hi, lo, block: int):
    """prng.py:174-178 on the device: draw block ``block`` of every key."""
    import torch

    dev = _native.require_cuda()
    hi_t = _as_device_u64(hi, dev).reshape(-1)
    c0 = torch.full((hi_t.numel(),), block, dtype=torch.int64, device=dev).view(torch.uint64)
    return _threefry_device(hi_t, lo, c0, TAG_DRAW)

"""Counter-based seeded random numbers (splitmix64), identical in numpy and torch.

This module is INPUT GENERATION ONLY: it holds none of the method's arithmetic.
Both the oracle (numpy, CPU) and the GPU harness (torch, on device) draw the same
values from it, keyed by (seed, field, global node index), so inputs never depend
on the decomposition or on the device.

    u(seed, field, i) = (splitmix64(seed*2^48 + field*2^40 + i) >> 11) * 2^-53   in [0, 1)
    uniform_pm1       = 2u - 1                                                    in [-1, 1)
"""
from __future__ import annotations

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def _key_base(seed: int, field: int) -> int:
    if not (0 <= seed < (1 << 16) and 0 <= field < 256):
        raise ValueError("seed must be < 2^16 and field < 256")
    return (seed << 48) | (field << 40)


def splitmix64_np(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01_np(seed: int, field: int, idx) -> np.ndarray:
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= (1 << 40)):
        raise ValueError("node index out of range for the counter layout")
    z = np.uint64(_key_base(seed, field)) | idx.astype(np.uint64)
    r = splitmix64_np(z) >> np.uint64(11)
    return r.astype(np.float64) * (2.0 ** -53)


def uniform_pm1_np(seed: int, field: int, idx) -> np.ndarray:
    return 2.0 * uniform01_np(seed, field, idx) - 1.0


# ---------------------------------------------------------------- torch (device)
def _i64(v: int) -> int:
    """Reinterpret an unsigned 64-bit constant as a signed int64 value."""
    v &= _MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(t, s: int):
    """Logical right shift of an int64 tensor (torch's >> is arithmetic)."""
    return (t >> s) & ((1 << (64 - s)) - 1)


def splitmix64_torch(z):
    """splitmix64 on an int64 torch tensor (two's-complement wrap-around = mod 2^64)."""
    z = z + _i64(_GOLDEN)
    z = (z ^ _lsr(z, 30)) * _i64(_M1)
    z = (z ^ _lsr(z, 27)) * _i64(_M2)
    return z ^ _lsr(z, 31)


def uniform01_torch(seed: int, field: int, idx):
    import torch
    z = idx.to(torch.int64) | _key_base(seed, field)
    r = _lsr(splitmix64_torch(z), 11)
    return r.to(torch.float64) * (2.0 ** -53)


def uniform_pm1_torch(seed: int, field: int, idx):
    return 2.0 * uniform01_torch(seed, field, idx) - 1.0

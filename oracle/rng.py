"""SplitMix64 restatement (reference core.py:26-103), scalar and numpy-vectorised.  Test-only."""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z: int) -> int:
    """core.py:42-49."""
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def label_hash(label) -> int:
    """core.py:52-57: FNV-1a 64 over repr(label) as UTF-8."""
    h = 0xCBF29CE484222325
    for b in repr(label).encode("utf-8"):
        h = ((h ^ b) * 0x100000001B3) & MASK64
    return h


def split(seed: int, label) -> int:
    """core.py:95-97: child seed = mix64(seed ^ H(label))."""
    return mix64((seed & MASK64) ^ label_hash(label))


def fusion_child_seed(cfg_seed: int, i: int) -> int:
    """fusion.py:170-171: make_rng(seed, "fusion-dropout").split(i)."""
    return split(split(cfg_seed, "fusion-dropout"), i)


def mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def draws(counter0: int, j0: int, n: int) -> np.ndarray:
    """Draws j0 .. j0+n-1 of a stream whose counter is `counter0` (core.py:69-71: counter += GAMMA first)."""
    j = np.arange(j0 + 1, j0 + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        ctr = np.uint64(counter0 & MASK64) + j * np.uint64(GAMMA)
    return mix64_np(ctr)


def uniforms(counter0: int, j0: int, n: int) -> np.ndarray:
    """core.py:73-75: (u64 >> 11) * 2**-53 (exact in float64)."""
    return (draws(counter0, j0, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def keep_mask(counter0: int, j0: int, n: int, p: float) -> np.ndarray:
    """fusion.py:113: kept_j = rng.uniform() >= p."""
    return uniforms(counter0, j0, n) >= p

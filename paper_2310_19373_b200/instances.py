"""Seeded instance generation (mirror of the reference's splitmix64 generators).

``SplitMix64``, ``bench_seed`` and ``random_instance`` reproduce
``pkg/src/qubrute/instances.py:40-108`` bit-for-bit (pinned by
tests/golden/reference_golden.json).  The ``config_*`` generators build the
five BASELINE.json workloads from the same PRNG with the rules fixed in
SURVEY.md §8d, so the GPU path, the oracle and the CPU baseline see identical
inputs on any machine.  Generation is vectorised with numpy uint64 wrap-around
arithmetic: draw k of a stream seeded with s is mix64(s + k * GOLDEN).
"""

from __future__ import annotations

import hashlib

import numpy as np

from .core import MAX_DIM, DimensionCapError, QuboInstance

_MASK64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


class SplitMix64:
    """splitmix64 (instances.py:58-74): state += GOLDEN; output = mix64(state)."""

    def __init__(self, seed: int) -> None:
        self._state = seed & _MASK64

    def next_u64(self) -> int:
        self._state = (self._state + _GOLDEN) & _MASK64
        return _mix64(self._state)

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * 2.0**-53

    def next_symmetric(self) -> float:
        return 2.0 * self.next_unit() - 1.0


def bench_seed(n: int, rep: int) -> int:
    """mix64((n << 32) | rep) (instances.py:77-83)."""
    return _mix64(((n & 0xFFFFFFFF) << 32) | (rep & 0xFFFFFFFF))


# ---------------------------------------------------------------- vectorised stream
def _u64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Draws start+1 .. start+count of splitmix64(seed) as uint64."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & _MASK64) + k * np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _unit(u: np.ndarray) -> np.ndarray:
    return (u >> np.uint64(11)).astype(np.float64) * 2.0**-53


def _upper_cells(n: int):
    iu = np.triu_indices(n)
    return iu  # row-major i <= j order, matching the reference's nested loops


def random_instance(n: int, seed: int, density: float = 1.0) -> QuboInstance:
    """Uniform [-1, 1) upper triangle, two draws per cell (keep, value) (instances.py:86-108)."""
    if n < 1:
        raise ValueError(f"dimension must be >= 1, got {n}")
    if n > MAX_DIM:
        raise DimensionCapError(f"dimension {n} exceeds cap {MAX_DIM}")
    if not 0.0 < density <= 1.0:
        raise ValueError(f"density must be in (0, 1], got {density}")
    iu = _upper_cells(n)
    cells = len(iu[0])
    u = _u64_stream(seed, 2 * cells)
    keep = _unit(u[0::2])
    value = 2.0 * _unit(u[1::2]) - 1.0
    coeffs = np.zeros((n, n))
    coeffs[iu] = np.where(keep < density, value, 0.0)
    return QuboInstance(coeffs)


# ---------------------------------------------------------------- BASELINE.json configs
def int_uniform_coeffs(n: int, seed: int, lo: int, hi: int) -> np.ndarray:
    """int32 entries lo + u64 % (hi-lo+1), one draw per upper cell incl. diagonal."""
    iu = _upper_cells(n)
    u = _u64_stream(seed, len(iu[0]))
    vals = (u % np.uint64(hi - lo + 1)).astype(np.int64) + lo
    c = np.zeros((n, n))
    c[iu] = vals.astype(np.int32)
    return c


def _box_muller_f32(u1: np.ndarray, u2: np.ndarray) -> np.ndarray:
    z = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)
    return z.astype(np.float32)


def normal_coeffs(n: int, seed: int, density: float | None = None) -> np.ndarray:
    """float32 N(0,1) upper triangle.

    Dense (density None): two draws per cell (u1, u2; Box-Muller).  Sparse:
    three draws per cell regardless (keep, u1, u2); an off-diagonal cell is
    kept iff keep < density, the diagonal is always kept.
    """
    iu = _upper_cells(n)
    cells = len(iu[0])
    c = np.zeros((n, n))
    if density is None:
        u = _u64_stream(seed, 2 * cells)
        c[iu] = _box_muller_f32(_unit(u[0::2]), _unit(u[1::2]))
    else:
        u = _u64_stream(seed, 3 * cells)
        keep = _unit(u[0::3])
        z = _box_muller_f32(_unit(u[1::3]), _unit(u[2::3]))
        diag = iu[0] == iu[1]
        c[iu] = np.where(diag | (keep < density), z, np.float32(0.0))
    return c


def uniform_f32_coeffs(n: int, seed: int) -> np.ndarray:
    """float32(next_symmetric()) per upper cell, one draw per cell."""
    iu = _upper_cells(n)
    u = _u64_stream(seed, len(iu[0]))
    c = np.zeros((n, n))
    c[iu] = (2.0 * _unit(u) - 1.0).astype(np.float32)
    return c


CONFIGS = {
    "A": dict(n=20, desc="n=20 int32 U[-100,100]"),
    "B": dict(n=24, desc="n=24 fp32 N(0,1)"),
    "C": dict(n=16, batch=4096, desc="4096 x n=16 fp32 U[-1,1]"),
    "D": dict(n=32, desc="n=32 int32 U[-1000,1000]"),
    "E": dict(n=40, desc="n=40 fp32 N(0,1), 10% off-diagonal density"),
}


def config_coeffs(name: str, rep: int = 0, n: int | None = None) -> np.ndarray:
    """Coefficients of BASELINE.json config A/B/D/E (optionally at another n), seed bench_seed(n, rep)."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    seed = bench_seed(n, rep)
    if name == "A":
        return int_uniform_coeffs(n, seed, -100, 100)
    if name == "B":
        return normal_coeffs(n, seed)
    if name == "D":
        return int_uniform_coeffs(n, seed, -1000, 1000)
    if name == "E":
        return normal_coeffs(n, seed, density=0.1)
    raise ValueError(f"config {name} is a batch config; use config_batch")


def config_instance(name: str, rep: int = 0, n: int | None = None) -> QuboInstance:
    return QuboInstance(config_coeffs(name, rep, n))


def config_batch(count: int = 4096, n: int = 16, rep_offset: int = 0) -> np.ndarray:
    """Config C: ``count`` instances, instance b seeded with bench_seed(n, rep_offset + b)."""
    out = np.empty((count, n, n))
    for b in range(count):
        out[b] = uniform_f32_coeffs(n, bench_seed(n, rep_offset + b))
    return out


def coeffs_sha256(c: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(c, dtype=np.float64).tobytes()).hexdigest()

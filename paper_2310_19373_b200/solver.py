"""Exhaustive QUBO solvers on B200 — drop-in for the reference's ``qubrute.solver``.

Same entry points, types, validation, error messages and result contract as
``pkg/src/qubrute/solver.py`` (cited per function); the work runs on the GPU
through libqubrute_b200.so:

* ``solve_incremental`` (solver.py:118-136): one exhaustive GPU solve, ties to the
  lowest global Gray rank (what the reference's single Gray walk keeps);
* ``solve_parallel`` (solver.py:193-229): the reference fixes m high bits, scans
  the 2^m subspaces on T threads and keeps the lowest suffix on ties; here the
  whole space is one GPU launch and the tie rule ``(suffix, local Gray rank)`` is
  applied in the device reduction, so results are identical for every ``threads``;
* ``solve_subspace`` (solver.py:139-156): one subspace, local Gray-rank ties;
* ``solve_naive`` (solver.py:99-115): the oracle's contract (guard, lowest-integer
  tie rule) served by the same exhaustive GPU search.

``Solution.value`` is always ``evaluate(minimizer)`` in the reference's fp64 order
and ``evaluations`` follows the reference's step accounting.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .core import MAX_DIM, DimensionCapError, QuboInstance, bits_from_int, cap_error

# solver.py:33
NAIVE_MAX_DIM = 24

MODES = ("naive", "incremental", "parallel")


@dataclass(frozen=True, eq=False)
class Solution:
    """Minimiser (uint8, index 0 = LSB), its exact value, step count, wall seconds (solver.py:38-51)."""

    minimizer: np.ndarray
    value: float
    evaluations: int
    elapsed: float


@dataclass(frozen=True)
class SubspaceSpec:
    """The ``m`` most-significant bits fixed to ``suffix`` (solver.py:54-79)."""

    m: int
    suffix: int

    def __post_init__(self) -> None:
        if self.m < 0:
            raise ValueError(f"fixed-bit count must be >= 0, got {self.m}")
        if not 0 <= self.suffix < (1 << self.m):
            raise ValueError(f"suffix {self.suffix} out of range [0, 2**{self.m})")

    def start_bits(self, n: int) -> np.ndarray:
        if self.m >= n:
            raise ValueError(f"cannot fix {self.m} bits of an n={n} instance")
        bits = np.zeros(n, dtype=np.uint8)
        for t in range(self.m):
            bits[n - self.m + t] = (self.suffix >> t) & 1
        return bits


@dataclass(frozen=True)
class SolveConfig:
    """Solver knobs (solver.py:82-96).  ``threads`` only selects the default ``fixed_bits``
    (and hence the tie rule), exactly as in the reference; the GPU does the scanning.
    ``devices`` (extension, SURVEY.md section 5 "Config / flags"): CUDA devices of this process
    to shard the solve over (qb_solve_devices); None = the current device."""

    threads: int = 1
    fixed_bits: Optional[int] = None
    mode: str = "incremental"
    devices: Optional[Tuple[int, ...]] = None

    def __post_init__(self) -> None:
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        if self.fixed_bits is not None and self.fixed_bits < 0:
            raise ValueError(f"fixed_bits must be >= 0, got {self.fixed_bits}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.devices is not None:
            devs = tuple(self.devices)
            if not devs or any((not isinstance(d, (int, np.integer))) or d < 0 for d in devs):
                raise ValueError(f"devices must be a non-empty sequence of device indices, got {self.devices!r}")
            object.__setattr__(self, "devices", tuple(int(d) for d in devs))


def _devices_of(config):
    """The ``devices`` knob of a config, or None.  The reference's own ``SolveConfig``
    (solver.py:82-96) has no such field: any object with ``threads`` / ``fixed_bits`` / ``mode``
    is accepted (duck typing, so the reference's types pass through Seam 2 unchanged)."""
    devs = getattr(config, "devices", None) if config is not None else None
    return None if devs is None else SolveConfig(devices=devs).devices


def _gpu_solve(coeffs, m_fix: int, suffix: int, m_tie: int, rule: int, devices=None):
    """One solve on the current device, or sharded over ``devices`` (one shard per entry)."""
    if devices is None:
        return _lib.solve(coeffs, m_fix, suffix, m_tie, rule)
    if len(devices) == 1:
        return _lib.solve(coeffs, m_fix, suffix, m_tie, rule, device=devices[0])
    return _lib.solve_devices(coeffs, devices, m_fix, suffix, m_tie, rule)


def _solution(inst: QuboInstance, res, evaluations: int, t0: float) -> Solution:
    minimizer = bits_from_int(int(res.argmin_bits), inst.n)
    # res.value is eval_upper(minimiser) computed natively in the reference's order
    return Solution(minimizer=minimizer, value=float(res.value), evaluations=int(evaluations),
                    elapsed=max(time.perf_counter() - t0, 1e-9))


def solve_naive(instance: QuboInstance, *, max_n: int = NAIVE_MAX_DIM) -> Solution:
    """Exhaustive search keeping the lowest-integer minimiser (solver.py:99-115)."""
    if instance.n > max_n:
        raise cap_error(
            instance,
            f"n={instance.n} exceeds the naive-solver guard {max_n}; "
            f"use the incremental solver, or raise max_n to force it",
        )
    if instance.n > MAX_DIM:
        raise cap_error(instance, f"n={instance.n} exceeds cap {MAX_DIM}")
    t0 = time.perf_counter()
    res = _lib.solve(instance.coeffs, 0, 0, 0, _lib.TIE_INTEGER)
    return _solution(instance, res, (1 << instance.n) - 1, t0)


def solve_incremental(instance: QuboInstance, *, devices=None) -> Solution:
    """Exhaustive Gray-code solve; ties to the lowest global Gray rank (solver.py:118-136).
    ``devices``: optional CUDA devices to shard over (extension; see SolveConfig)."""
    if instance.n > MAX_DIM:
        raise cap_error(instance, f"n={instance.n} exceeds cap {MAX_DIM}")
    if devices is not None:
        devices = SolveConfig(devices=devices).devices
    t0 = time.perf_counter()
    res = _gpu_solve(instance.coeffs, 0, 0, 0, _lib.TIE_GRAY, devices)
    return _solution(instance, res, (1 << instance.n) - 1, t0)


def solve_subspace(instance: QuboInstance, sub: SubspaceSpec) -> Solution:
    """Minimise over {x : top sub.m bits == sub.suffix} (solver.py:139-156)."""
    t0 = time.perf_counter()
    if sub.m >= instance.n:
        raise ValueError(f"cannot fix {sub.m} bits of an n={instance.n} instance")
    if instance.n > MAX_DIM:
        raise cap_error(instance, f"n={instance.n} exceeds cap {MAX_DIM}")
    res = _lib.solve(instance.coeffs, sub.m, sub.suffix, sub.m, _lib.TIE_GRAY)
    return _solution(instance, res, (1 << (instance.n - sub.m)) - 1, t0)


def combine_subspace_minima(solutions: Sequence[Solution]) -> Solution:
    """Min-reduce, earliest entry wins ties (solver.py:173-185)."""
    if not solutions:
        raise ValueError("no subspace solutions to combine")
    best = solutions[0]
    for sol in solutions[1:]:
        if sol.value < best.value:
            best = sol
    return best


def default_fixed_bits(n: int, threads: int) -> int:
    """m = min(n - 1, ceil(log2(threads))) (solver.py:188-190)."""
    return min(n - 1, (threads - 1).bit_length())


def _resolve_m(instance: QuboInstance, config: SolveConfig | None) -> int:
    if config is None:
        config = SolveConfig()
    if instance.n < 2:
        raise ValueError("parallel solving needs n >= 2")
    if instance.n > MAX_DIM:
        raise cap_error(instance, f"n={instance.n} exceeds cap {MAX_DIM}")
    m = config.fixed_bits
    if m is None:
        m = default_fixed_bits(instance.n, config.threads)
    if not 0 <= m < instance.n:
        raise ValueError(f"fixed_bits must be in [0, {instance.n}), got {m}")
    return m


def solve_parallel(instance: QuboInstance, config: SolveConfig | None = None) -> Solution:
    """All 2^m subspaces in one GPU launch, lowest-suffix tie rule (solver.py:193-229)."""
    m = _resolve_m(instance, config)
    t0 = time.perf_counter()
    res = _gpu_solve(instance.coeffs, 0, 0, m, _lib.TIE_GRAY, _devices_of(config))
    return _solution(instance, res, (1 << instance.n) - (1 << m), t0)


def _batch_coeffs(instances) -> np.ndarray:
    """(count, n, n) fp64 upper-triangular coefficients, normalised like QuboInstance
    (lower triangle folded, finiteness and cap checked), vectorised over the batch."""
    if isinstance(instances, np.ndarray):
        # a float32 batch stays float32: the native path widens each coefficient exactly (qb_solve_batch_f32)
        arr = instances if instances.dtype == np.float32 else np.asarray(instances, dtype=np.float64)
        if arr.ndim != 3 or arr.shape[1] != arr.shape[2]:
            raise ValueError(f"batch must have shape (count, n, n), got {arr.shape}")
        n = arr.shape[1]
        if n < 1:
            raise ValueError("dimension must be at least 1")
        if n > MAX_DIM:
            raise DimensionCapError(f"dimension {n} exceeds cap {MAX_DIM}")
        # the native batch path folds entries below the diagonal itself (QuboInstance
        # convention) and rejects non-finite coefficients, so no numpy pass over the batch
        arr = np.ascontiguousarray(arr)
        return arr
    insts = list(instances)
    if not insts:
        return np.zeros((0, 1, 1))
    n0 = insts[0].n
    if any(i.n != n0 for i in insts):
        raise ValueError("all instances of a batch must have the same n")
    return np.ascontiguousarray(np.stack([i.coeffs for i in insts]))


def solve_batch(instances, *, as_arrays: bool = False, devices=None):
    """Solve many independent instances of one size n <= 24 in one GPU launch (one CTA per
    instance).  Each result equals ``solve_incremental`` of that instance (same tie rule).
    ``instances``: a sequence of QuboInstance or a (count, n, n) array.  Returns a list of
    Solution, or with ``as_arrays=True`` the pair (minimizers uint8 (count, n), values (count,)).
    The reference has no batch entry point; its equivalent is a loop / thread pool of
    solve_incremental calls.  ``devices``: CUDA devices of this process to
    split the instances over (contiguous slices, qb_solve_batch_devices); None = the current device."""
    coeffs = _batch_coeffs(instances)
    count, n = coeffs.shape[0], coeffs.shape[1]
    if count == 0:
        return (np.zeros((0, n), dtype=np.uint8), np.zeros(0)) if as_arrays else []
    t0 = time.perf_counter()
    if devices is None:
        bits, vals, _ = _lib.solve_batch(coeffs)
    else:
        bits, vals, _ = _lib.solve_batch_devices(coeffs, SolveConfig(devices=devices).devices)
    # bit i of each little-endian uint64 -> column i (one vectorised pass, no per-bit shifts)
    minimizers = np.unpackbits(bits.astype("<u8").view(np.uint8).reshape(count, 8), axis=1,
                               bitorder="little")[:, :n]
    if as_arrays:
        return minimizers, vals
    elapsed = max(time.perf_counter() - t0, 1e-9)
    ev = (1 << n) - 1
    return [Solution(minimizer=minimizers[b], value=float(vals[b]), evaluations=ev, elapsed=elapsed)
            for b in range(count)]


def all_minimizers(instance: QuboInstance, config: SolveConfig | None = None, *, max_count: int = 1 << 20):
    """Minimum value and EVERY minimising vector (BASELINE config A), as a uint8 array of shape
    (count, n) sorted by the tie rule of ``config`` (default: global Gray rank, so row 0 is
    ``solve_incremental``'s minimiser; with ``mode="parallel"`` row 0 is ``solve_parallel``'s).
    The reference returns a single minimiser (SPEC.md:273 non-goal); this is an extension.
    Raises if more than ``max_count`` minimisers exist."""
    if instance.n > MAX_DIM:
        raise cap_error(instance, f"n={instance.n} exceeds cap {MAX_DIM}")
    m = _resolve_m(instance, config) if (config is not None and config.mode == "parallel") else 0
    value, xs, count = _lib.all_minimisers(instance.coeffs, 0, 0, m, cap=max_count)
    if count > max_count:
        raise ValueError(f"{count} minimisers exceed max_count={max_count}")
    bits = ((xs[:, None] >> np.arange(instance.n, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(np.uint8)
    return float(value), bits


def solve(instance: QuboInstance, config: SolveConfig | None = None) -> Solution:
    """Dispatch on ``config.mode`` (solver.py:232-240)."""
    if config is None:
        config = SolveConfig()
    if config.mode == "naive":
        return solve_naive(instance)
    if config.mode == "incremental":
        return solve_incremental(instance, devices=_devices_of(config))
    return solve_parallel(instance, config)

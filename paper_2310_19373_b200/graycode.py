"""Gray-code flip sequence and ordering helpers (mirror of ``qubrute.graycode``).

The k-th flip of the reflected Gray walk is ctz(k) (graycode.py:20-40 of the
reference); the GPU kernels use the same rule with ``__ffs``.  Also holds the
rank algebra the kernels' tie-breaking is built on: ``gray(t)`` is the state
visited at step t and ``gray_rank(x)`` (prefix-XOR) its inverse.
"""

from __future__ import annotations

from typing import Iterator

from .core import MAX_DIM

MAX_PERMUTATION_BITS = 20


def ctz(k: int) -> int:
    """Trailing zero count of k >= 1 (graycode.py:20-28)."""
    if k < 1:
        raise ValueError("ctz is undefined for k < 1 here")
    return (k & -k).bit_length() - 1


def flip_sequence(n: int) -> Iterator[int]:
    """The 2**n - 1 flip positions of the Gray walk of {0,1}^n (graycode.py:31-40)."""
    if not 1 <= n <= MAX_DIM:
        raise ValueError(f"bit width must be in [1, {MAX_DIM}], got {n}")
    return (ctz(k) for k in range(1, 1 << n))


def gray_permutation(k_bits: int) -> list[int]:
    """Full reflected Gray ordering of [0, 2**k_bits) (graycode.py:43-57)."""
    if not 1 <= k_bits <= MAX_PERMUTATION_BITS:
        raise ValueError(f"width must be in [1, {MAX_PERMUTATION_BITS}], got {k_bits}")
    return [t ^ (t >> 1) for t in range(1 << k_bits)]


def gray(t: int) -> int:
    """State visited at step t of the walk from zero."""
    return t ^ (t >> 1)


def gray_rank(x: int) -> int:
    """Inverse of :func:`gray`: the step at which state x is visited (prefix XOR)."""
    r = 0
    while x:
        r ^= x
        x >>= 1
    return r


def tie_key(x: int, n: int, m: int) -> int:
    """Order in which the reference's ``solve_parallel(m)`` prefers tied minimisers.

    Subspaces (top m bits) are reduced in ascending suffix order and each is
    walked in Gray order of its n-m free bits (solver.py:159-185), so the kept
    minimiser is the smallest ``(suffix << (n-m)) | gray_rank(low bits)``.
    m = 0 gives the global Gray rank used by ``solve_incremental``.
    """
    lo_bits = n - m
    lo = x & ((1 << lo_bits) - 1)
    return ((x >> lo_bits) << lo_bits) | gray_rank(lo)

"""TEST INFRASTRUCTURE — the CPU oracle for the Gray-code QUBO hot path.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline; the product package never does.

Two independent oracles:

* ``liboracle.so`` (gray_oracle.c): a line-by-line C restatement of the
  reference's numba kernels (``pkg/src/qubrute/_kernels.py:12-75``) and of the
  subspace solver loop (``solver.py:159-229``) — same fp64 arithmetic, same
  summation order, same strict-'<' incumbent rule.  Pinned against outputs of
  the reference itself (tests/golden/reference_golden.json).
* ``all_values`` / ``expected_*``: numpy full enumeration of every state's
  value, for certifying minima, ties and tie rules at n <= 24.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oc_eval_upper.restype = ctypes.c_double
        L.oc_eval_upper.argtypes = [_dp, ctypes.c_int, _dp]
        L.oc_naive_scan.restype = ctypes.c_uint64
        L.oc_naive_scan.argtypes = [_dp, ctypes.c_int, _dp, _dp]
        L.oc_split.restype = None
        L.oc_split.argtypes = [_dp, ctypes.c_int, _dp, _dp]
        L.oc_gray_scan.restype = ctypes.c_uint64
        L.oc_gray_scan.argtypes = [_dp, _dp, _dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.oc_solve_subspaces.restype = ctypes.c_int
        L.oc_solve_subspaces.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int, _u64p, _dp, _u64p]
        L.oc_solve_batch.restype = ctypes.c_int
        L.oc_solve_batch.argtypes = [_dp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, _u64p, _dp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ C restatement
def eval_upper(coeffs, x) -> float:
    c = _f64(coeffs)
    return lib().oc_eval_upper(_p(c), c.shape[0], _p(_f64(x)))


def naive_scan(coeffs):
    c = _f64(coeffs)
    n = c.shape[0]
    xm = np.zeros(n)
    vm = ctypes.c_double()
    steps = lib().oc_naive_scan(_p(c), n, _p(xm), ctypes.byref(vm))
    return xm, vm.value, int(steps)


def split(coeffs):
    c = _f64(coeffs)
    n = c.shape[0]
    qua = np.zeros((n, n))
    lin = np.zeros(n)
    lib().oc_split(_p(c), n, _p(qua), _p(lin))
    return qua, lin


def gray_scan(coeffs, qua, lin, x0, v0, n_free):
    c, q, l, x = _f64(coeffs), _f64(qua), _f64(lin), _f64(x0)
    n = c.shape[0]
    xm = np.zeros(n)
    vm = ctypes.c_double()
    steps = lib().oc_gray_scan(_p(c), _p(q), _p(l), _p(x), float(v0), n, int(n_free), _p(xm), ctypes.byref(vm))
    return xm, vm.value, int(steps)


def solve_subspaces(coeffs, m: int, s_begin: int = 0, s_end: int | None = None, threads: int = 1):
    """Reference ``solve_parallel`` semantics over suffixes [s_begin, s_end) -> (bits, value, evaluations)."""
    c = _f64(coeffs)
    n = c.shape[0]
    if s_end is None:
        s_end = 1 << m
    bits = ctypes.c_uint64()
    val = ctypes.c_double()
    ev = ctypes.c_uint64()
    rc = lib().oc_solve_subspaces(_p(c), n, m, s_begin, s_end, threads, ctypes.byref(bits), ctypes.byref(val),
                                  ctypes.byref(ev))
    if rc != 0:
        raise ValueError("oc_solve_subspaces: bad arguments")
    return int(bits.value), val.value, int(ev.value)


def solve_incremental(coeffs):
    return solve_subspaces(coeffs, 0)


def solve_batch(coeffs_batch, threads: int = 1):
    c = _f64(coeffs_batch)
    count, n = c.shape[0], c.shape[1]
    bits = np.zeros(count, dtype=np.uint64)
    vals = np.zeros(count)
    rc = lib().oc_solve_batch(_p(c), n, count, threads, bits.ctypes.data_as(_u64p), _p(vals))
    if rc != 0:
        raise ValueError("oc_solve_batch: bad arguments")
    return bits, vals


# ------------------------------------------------------------------ numpy enumeration
def all_values(coeffs) -> np.ndarray:
    """f(x) for every x in [0, 2^n) (index = integer encoding, bit 0 = LSB), fp64.

    Built by doubling: f(x | 2^i) = f(x) + Q_ii + sum_{j<i} Q_ji x_j for x < 2^i.
    Exact whenever all partial sums are exact in fp64 (integer or fp32-valued Q).
    """
    c = _f64(coeffs)
    n = c.shape[0]
    vals = np.zeros(1 << n)
    for i in range(n):
        lo = vals[: 1 << i]
        idx = np.arange(1 << i, dtype=np.int64)
        add = np.full(1 << i, c[i, i])
        for j in range(i):
            add += ((idx >> j) & 1) * c[j, i]
        vals[1 << i: 1 << (i + 1)] = lo + add
    return vals


def gray_rank_array(x: np.ndarray) -> np.ndarray:
    r = np.zeros_like(x)
    y = x.copy()
    while np.any(y):
        r ^= y
        y >>= 1
    return r


def tie_keys(n: int, m: int) -> np.ndarray:
    """key_m(x) for all x: (top m bits) << (n-m) | gray_rank(low n-m bits)."""
    x = np.arange(1 << n, dtype=np.int64)
    lo_bits = n - m
    lo = x & ((1 << lo_bits) - 1)
    return ((x >> lo_bits) << lo_bits) | gray_rank_array(lo)


def expected_argmin(coeffs, m: int = 0, rule: str = "gray", suffix: int | None = None):
    """Minimum value and the minimiser the reference keeps under its tie rule.

    rule "gray": smallest key_m (solve_incremental m=0 / solve_parallel(m));
    rule "integer": smallest integer encoding (solve_naive);
    ``suffix`` restricts to one subspace of the top m bits (solve_subspace).
    Returns (bits, value, all_minimisers_sorted_by_key).
    """
    c = _f64(coeffs)
    n = c.shape[0]
    vals = all_values(c)
    x = np.arange(1 << n, dtype=np.int64)
    if suffix is not None:
        sel = (x >> (n - m)) == suffix
        vals = np.where(sel, vals, np.inf)
    vmin = vals.min()
    mins = np.nonzero(vals == vmin)[0]
    if rule == "integer":
        keys = mins
    else:
        keys = tie_keys(n, m)[mins]
    order = np.argsort(keys, kind="stable")
    return int(mins[order[0]]), float(vmin), mins[order]

"""Seam 1: the reference's compiled-kernel module (``qubrute._kernels``) served by the GPU.

Same three functions and return contracts as ``pkg/src/qubrute/_kernels.py``:

* ``eval_upper(coeffs, x)`` — native host evaluation, identical fp64 order (:12-20);
* ``gray_scan(coeffs, qua, lin, x0, v0, n_free)`` — the hot operator (:46-75), one GPU
  subspace solve returning ``(x_min, v_min, steps)``;
* ``naive_scan(coeffs)`` — lowest-integer minimiser (:23-43) from the same GPU search.

Assigning ``qubrute._kernels.gray_scan = paper_2310_19373_b200._kernels.gray_scan``
reroutes the reference's solve_incremental / solve_subspace / solve_parallel through
the B200 kernel (they look the attribute up at call time, solver.py:29,164).
"""

from __future__ import annotations

import numpy as np

from . import _lib


def eval_upper(coeffs, x) -> float:
    return _lib.eval_upper(coeffs, x)


def gray_scan(coeffs, qua, lin, x0, v0, n_free):
    return _lib.gray_scan(coeffs, qua, lin, x0, v0, n_free)


def naive_scan(coeffs):
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    n = c.shape[0]
    res = _lib.solve(c, 0, 0, 0, _lib.TIE_INTEGER)
    x = np.array([(int(res.argmin_bits) >> i) & 1 for i in range(n)], dtype=np.float64)
    return x, float(res.value), (1 << n) - 1

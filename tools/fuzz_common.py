"""Shared pieces of the randomised parity soaks (tools/fuzz_oracle.py, tools/fuzz_batch.py): instance families, the
reference's tie keys, the classification of a difference from the oracle and a full-enumeration check of this
library's own contract.  Test infrastructure: imports oracle/ as the checker only."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402


def make(rng, n):
    iu = np.triu_indices(n, 1)
    di = np.diag_indices(n)
    m = len(iu[0])
    fam = int(rng.integers(0, 12))
    c = np.zeros((n, n))
    if fam == 0:    # sparse normal
        dens = rng.choice([0.02, 0.1, 0.3])
        c[iu] = rng.standard_normal(m) * (rng.random(m) < dens); c[di] = rng.standard_normal(n)
    elif fam == 1:  # dense normal (float32-valued)
        c[iu] = rng.standard_normal(m).astype(np.float32); c[di] = rng.standard_normal(n).astype(np.float32)
    elif fam == 2:  # dense integers, random scale
        s = int(rng.choice([1, 3, 100, 1000, 30000]))
        c[iu] = rng.integers(-s, s + 1, m); c[di] = rng.integers(-s, s + 1, n)
    elif fam == 3:  # tie-heavy
        c[iu] = rng.integers(-1, 2, m); c[di] = rng.integers(-1, 2, n)
    elif fam == 4:  # antiferromagnetic
        c[iu] = rng.random(m); c[di] = -rng.random(n) * rng.choice([2, 8, 16])
    elif fam == 5:  # ferromagnetic
        c[iu] = -rng.random(m); c[di] = rng.random(n) * 3
    elif fam == 6:  # wide range
        c[iu] = rng.standard_normal(m) * np.where(rng.random(m) < 0.05, 1e3, 1e-3); c[di] = rng.standard_normal(n)
    elif fam == 7:  # one huge term
        c[iu] = rng.standard_normal(m) * 1e-3; c[0, 0] = -1e9 * rng.random()
    elif fam == 8:  # mostly zero
        k = rng.integers(0, m, 5); c[iu[0][k], iu[1][k]] = rng.standard_normal(5)
    elif fam == 9:  # dense fp64 normal (not fp32-representable)
        c[iu] = rng.standard_normal(m); c[di] = rng.standard_normal(n)
    elif fam == 10:  # half-integers: float-valued but massively tied
        c[iu] = rng.integers(-2, 3, m) * 0.5; c[di] = rng.integers(-2, 3, n) * 0.5
    else:           # duplicated variables (rows i and i+1 alike): structured ties on a float instance
        c[iu] = rng.standard_normal(m).astype(np.float32); c[di] = rng.standard_normal(n).astype(np.float32)
        for i in range(0, n - 1, 2):
            c[i + 1, i + 2:] = c[i, i + 2:]; c[:i, i + 1] = c[:i, i]; c[i + 1, i + 1] = c[i, i]; c[i, i + 1] = 0.0
    return fam, c


def gray_rank(x):
    r = 0
    while x:
        r ^= x
        x >>= 1
    return r


def tie_key(x, n, m):
    lo = n - m
    return ((x >> lo) << lo) | gray_rank(x & ((1 << lo) - 1))


def classify(c, n, m, got_bits, want_bits):
    xb = lambda v: np.array([(v >> i) & 1 for i in range(n)], dtype=np.float64)
    vg, vo = O.eval_upper(c, xb(got_bits)), O.eval_upper(c, xb(want_bits))
    if vg < vo or (vg == vo and tie_key(got_bits, n, m) < tie_key(want_bits, n, m)):
        return "reference-drift", vg, vo
    return "BUG", vg, vo


def truth(c, n, m, suffix):
    """This library's own contract by full enumeration (n <= 20): eval_upper of EVERY state in the reference's order
    (row-major sequential fp64 adds, _kernels.py:12-20; absent terms add +0.0, which changes nothing), the lowest
    value, and among equal values the lowest tie key."""
    x = np.arange(1 << n, dtype=np.int64)
    v = np.zeros(1 << n)
    for i in range(n):
        xi = ((x >> i) & 1).astype(np.float64)
        for j in range(i, n):
            if c[i, j] != 0.0:
                v += c[i, j] * xi * ((x >> j) & 1)
    if suffix is not None:
        v = np.where((x >> (n - m)) == suffix, v, np.inf)
    mins = np.nonzero(v == v.min())[0]
    best = min((int(b) for b in mins), key=lambda b: tie_key(b, n, m))
    return best, float(v.min())

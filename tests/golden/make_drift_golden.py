"""Fixture of instances on which the REFERENCE's answer is decided by the rounding drift of its running value.

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_drift_golden.py

The reference keeps the state whose RUNNING fp64 value is the lowest seen so far (_kernels.py:62-73) and recomputes only
the REPORTED value with evaluate() (solver.py:169; SPEC.md "Drift control").  On float instances that have exact ties
(structural zeros leave free variables) or two states closer than the accumulated rounding error (one huge coefficient
among small ones), the kept state is therefore not the first minimiser in Gray order that SPEC.md:224 promises, and it
changes with fixed_bits on the same instance.  This script records, for seeded instances of both kinds solved by the
unmodified reference (``qubrute`` from /root/reference/pkg/src):

* the reference's own answers for solve_incremental and solve_parallel(m) -- the oracle (oracle/gray_oracle.c) must
  reproduce them bit for bit, drift included (tests/test_oracle.py);
* the answer of the stated contract, by full enumeration in the reference's evaluation order (evaluate() of every
  state; lowest value, then lowest (suffix, Gray rank) key) -- what this library returns (tests/test_gpu_round2.py).

Writes reference_drift_cases.json next to this file; inputs are stored explicitly (fp64 repr round-trips through JSON).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("QUBRUTE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import qubrute as qb  # noqa: E402


def bits_int(minimizer) -> int:
    return int(sum(int(b) << i for i, b in enumerate(minimizer)))


def gray_rank(x: int) -> int:
    r = 0
    while x:
        r ^= x
        x >>= 1
    return r


def tie_key(x: int, n: int, m: int) -> int:
    lo = n - m
    return ((x >> lo) << lo) | gray_rank(x & ((1 << lo) - 1))


def contract_answer(inst, n: int, m: int):
    """evaluate() of every state (the reference's own function), lowest value, lowest tie key."""
    if n <= 12:
        vals = np.empty(1 << n)
        for x in range(1 << n):
            vals[x] = qb.evaluate(inst, np.array([(x >> i) & 1 for i in range(n)], dtype=np.float64))
    else:
        # the same row-major sequential fp64 sum (_kernels.py:12-20) for all states at once: a term a state does not
        # have adds +0.0, which leaves its running sum unchanged; spot-checked against evaluate() below
        xs = np.arange(1 << n, dtype=np.int64)
        vals = np.zeros(1 << n)
        for i in range(n):
            xi = ((xs >> i) & 1).astype(np.float64)
            for j in range(i, n):
                if inst.coeffs[i, j] != 0.0:
                    vals += inst.coeffs[i, j] * xi * ((xs >> j) & 1)
        probe = np.random.default_rng(n).integers(0, 1 << n, 64).tolist() + [int(np.argmin(vals))]
        for x in probe:
            assert vals[x] == qb.evaluate(inst, np.array([(x >> i) & 1 for i in range(n)], dtype=np.float64))
    mins = [int(b) for b in np.nonzero(vals == vals.min())[0]]
    return min(mins, key=lambda b: tie_key(b, n, m)), float(vals.min()), len(mins)


def make(kind: str, n: int, rng) -> np.ndarray:
    iu = np.triu_indices(n, 1)
    cnt = len(iu[0])
    c = np.zeros((n, n))
    if kind == "mostly_zero":       # five off-diagonal fp64 terms: most variables are free, 2^(n-10)+ exact ties
        k = rng.integers(0, cnt, 5)
        c[iu[0][k], iu[1][k]] = rng.standard_normal(5)
    elif kind == "huge_term":       # gaps between states far below the running value's rounding error
        c[iu] = rng.standard_normal(cnt) * 1e-3
        c[0, 0] = -1e9 * rng.random()
    else:                           # half-sparse fp64 normal with a free variable
        c[iu] = rng.standard_normal(cnt) * (rng.random(cnt) < 0.3)
        c[np.diag_indices(n)] = rng.standard_normal(n)
        f = int(rng.integers(0, n))
        c[f, :] = 0.0
        c[:, f] = 0.0
    return c


def main() -> None:
    t0 = time.time()
    qb.solve_incremental(qb.random_instance(6, 0))  # JIT warm-up
    rng = np.random.default_rng(20231019)
    cases = []
    for kind, sizes in (("mostly_zero", (8, 9, 10, 11, 12, 13, 14) * 3), ("huge_term", (14, 16, 18, 18, 20, 20)),
                        ("free_variable", (9, 11, 13, 14, 15, 16))):
        for n in sizes:
            c = make(kind, n, rng)
            inst = qb.QuboInstance(c)
            rec = {"kind": kind, "n": n, "coeffs": [[float(v) for v in row] for row in inst.coeffs], "results": {}}
            for m in (0, 2, 5):
                if m == 0:
                    sol = qb.solve_incremental(inst)
                else:
                    sol = qb.solve_parallel(inst, qb.SolveConfig(threads=2, fixed_bits=m))
                cb, cv, nties = contract_answer(inst, n, m)
                rec["results"][str(m)] = {"reference_bits": bits_int(sol.minimizer), "reference_value": float(sol.value),
                                          "contract_bits": cb, "contract_value": cv, "minimisers": nties}
            cases.append(rec)
    decided = sum(1 for c in cases for r in c["results"].values() if r["reference_bits"] != r["contract_bits"])
    out = {"generator": "tests/golden/make_drift_golden.py", "reference": REF,
           "qubrute_version": getattr(qb, "__version__", "?"), "cases": cases, "drift_decided_results": decided,
           "results": sum(len(c["results"]) for c in cases), "seconds": round(time.time() - t0, 1)}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_drift_cases.json")
    with open(path, "w") as fh:
        json.dump(out, fh)
    print(f"wrote {path}: {len(cases)} instances, {decided} of {out['results']} reference answers decided by drift, "
          f"{out['seconds']} s")


if __name__ == "__main__":
    main()

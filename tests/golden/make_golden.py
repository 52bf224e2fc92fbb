"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (the GPU box has no /root/reference):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(override with QUBRUTE_REF), calls its public solvers and its gray_scan
kernel on seeded instances, and writes reference_golden.json next to this
file.  Inputs are stored explicitly (float64 values round-trip exactly through
JSON's repr formatting), together with SHA-256 digests of the generated
matrices, so the fixture pins both the solver semantics and the input
generators.  tests/test_oracle.py checks the CPU oracle against it and the
GPU parity tests check the CUDA path against it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("QUBRUTE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))

import qubrute as qb  # noqa: E402
from qubrute import _kernels  # noqa: E402

from paper_2310_19373_b200 import instances as mine  # noqa: E402  (config generators only)


def sha(c) -> str:
    return hashlib.sha256(np.ascontiguousarray(c, dtype=np.float64).tobytes()).hexdigest()


def bits_int(minimizer) -> int:
    return int(sum(int(b) << i for i, b in enumerate(minimizer)))


def sol_dict(sol) -> dict:
    return {"bits": bits_int(sol.minimizer), "value": float(sol.value), "evaluations": int(sol.evaluations)}


def tie_heavy_coeffs(n: int, seed: int) -> np.ndarray:
    """Integer entries in {-2..2}: many exactly tied minima."""
    rng = qb.SplitMix64(seed)
    c = np.zeros((n, n))
    for i in range(n):
        for j in range(i, n):
            c[i, j] = float(int(rng.next_u64() % 5) - 2)
    return c


def solve_case(name: str, coeffs: np.ndarray, ms=(1, 3), naive=True, subspace_m=None, incremental=True,
               parallel_threads=4, store_coeffs=True) -> dict:
    inst = qb.QuboInstance(coeffs)
    n = inst.n
    case = {"name": name, "n": n, "sha256": sha(inst.coeffs)}
    if store_coeffs:
        case["coeffs"] = inst.coeffs.tolist()
    res = {}
    if incremental:
        res["incremental"] = sol_dict(qb.solve_incremental(inst))
    for m in ms:
        if 0 <= m < n and n >= 2:
            res[f"parallel_m{m}"] = sol_dict(qb.solve_parallel(inst, qb.SolveConfig(threads=parallel_threads,
                                                                                     fixed_bits=m)))
    if naive and n <= 16:
        res["naive"] = sol_dict(qb.solve_naive(inst))
    if subspace_m is not None and subspace_m < n:
        res[f"subspace_m{subspace_m}"] = [sol_dict(qb.solve_subspace(inst, qb.SubspaceSpec(subspace_m, s)))
                                          for s in range(1 << subspace_m)]
    case["results"] = res
    return case


def main() -> None:
    t0 = time.time()
    out = {"generator": "tests/golden/make_golden.py", "reference": REF, "qubrute_version": qb.__version__}

    # --- PRNG known answers (instances.py:28-29; test_instances.py:19-29) and more
    out["splitmix64"] = {str(s): [qb.SplitMix64(s).next_u64() for _ in range(1)] for s in (0,)}
    sm = {}
    for s in (0, 1, 1234567, qb.bench_seed(40, 0), qb.bench_seed(16, 4095)):
        r = qb.SplitMix64(s)
        sm[str(s)] = [r.next_u64() for _ in range(8)]
    out["splitmix64"] = sm
    out["bench_seed"] = {f"{n},{rep}": qb.bench_seed(n, rep) for n in (1, 16, 20, 24, 32, 40) for rep in (0, 1, 4095)}
    out["random_instance_sha256"] = {
        f"{n},{seed},{d}": sha(qb.random_instance(n, seed, d).coeffs)
        for n in (1, 6, 13, 24, 40) for seed in (0, 77, qb.bench_seed(n, 0)) for d in (1.0, 0.25)
    }

    cases = []
    # --- known answers from the reference's own tests
    cases.append(solve_case("diag_1_2_3", np.diag([1.0, 2.0, 3.0])))
    cases.append(solve_case("diag_m1_m2", np.diag([-1.0, -2.0]), ms=(1,)))
    cases.append(solve_case("zero_n6", np.zeros((6, 6)), ms=(0, 1, 2, 3, 5), subspace_m=2))
    cases.append(solve_case("bit0_only_negative", np.diag([-1.0, 0.0, 0.0]), ms=(1, 2)))
    cases.append(solve_case("worked_3bit", np.array([[1.0, -2.0, 0.0], [0.0, 3.0, 1.0], [0.0, 0.0, -1.0]]), ms=(1, 2)))
    cases.append(solve_case("single_var_neg", np.array([[-3.5]]), ms=()))
    cases.append(solve_case("single_var_pos", np.array([[2.0]]), ms=()))
    cases.append(solve_case("lower_fold", np.array([[0.0, 0.0, 1.5], [-2.0, 1.0, 0.0], [0.5, -3.0, -1.0]]), ms=(1,)))

    # --- random_instance sweep (acceptance criterion 1 shape: n = 1..16)
    for n in range(1, 17):
        for rep in range(2):
            inst = qb.random_instance(n, qb.bench_seed(n, rep))
            cases.append(solve_case(f"random_n{n}_rep{rep}", inst.coeffs, ms=(1, 3),
                                    subspace_m=2 if n in (5, 9, 12) else None))
    for n, dens in ((14, 0.3), (18, 0.5), (20, 1.0)):
        inst = qb.random_instance(n, qb.bench_seed(n, 7), dens)
        cases.append(solve_case(f"random_n{n}_d{dens}", inst.coeffs, ms=(0, 1, 3, 6), naive=False))

    # --- tie-heavy integer instances (tie semantics of every entry point)
    for t in range(60):
        n = 4 + t % 7
        c = tie_heavy_coeffs(n, 9000 + t)
        cases.append(solve_case(f"ties_{t}_n{n}", c, ms=(1, 2, 3), subspace_m=2))

    # --- BASELINE.json config shapes (reduced n where the reference is slow)
    for rep in range(3):
        cases.append(solve_case(f"configA_n20_rep{rep}", mine.config_coeffs("A", rep), ms=(3, 6), naive=False))
    cases.append(solve_case("configB_n24_rep0", mine.config_coeffs("B", 0), ms=(), naive=False))
    for rep in range(2):
        cases.append(solve_case(f"configB_n18_rep{rep}", mine.config_coeffs("B", rep, n=18), ms=(3,), naive=False))
        cases.append(solve_case(f"configD_n22_rep{rep}", mine.config_coeffs("D", rep, n=22), ms=(3,), naive=False))
        cases.append(solve_case(f"configE_n22_rep{rep}", mine.config_coeffs("E", rep, n=22), ms=(3,), naive=False))
    cases.append(solve_case("configD_n32_rep0", mine.config_coeffs("D", 0), ms=(6,), naive=False,
                            incremental=False, parallel_threads=os.cpu_count() or 8))
    out["cases"] = cases

    # --- config C: 4096 x n=16 (reference loop of solve_incremental; no batch API)
    batch = mine.config_batch(4096, 16)
    cb = {"n": 16, "count": 4096, "sha256": sha(batch), "bits": [], "values": []}
    for b in range(batch.shape[0]):
        s = qb.solve_incremental(qb.QuboInstance(batch[b]))
        cb["bits"].append(bits_int(s.minimizer))
        cb["values"].append(float(s.value))
    out["configC"] = cb

    # --- Seam 1: the gray_scan operator itself (_kernels.py:46-75)
    seam = []
    for n, m, seed in ((8, 0, 1), (10, 3, 2), (12, 5, 3), (16, 4, 4), (6, 5, 5)):
        inst = qb.random_instance(n, seed)
        form = qb.split(inst)
        for suffix in (0, (1 << m) - 1, (1 << m) // 3):
            x0 = qb.SubspaceSpec(m, suffix).start_bits(n).astype(np.float64)
            v0 = float(_kernels.eval_upper(inst.coeffs, x0))
            xm, vm, steps = _kernels.gray_scan(inst.coeffs, form.qua, form.lin, x0, v0, n - m)
            seam.append({"coeffs": inst.coeffs.tolist(), "x0": x0.tolist(), "v0": v0, "n_free": n - m,
                         "x_min": xm.tolist(), "v_min": float(vm), "steps": int(steps)})
    out["gray_scan"] = seam

    # --- running-value drift pin (acceptance criterion 2 shape)
    inst = qb.random_instance(12, qb.bench_seed(12, 0))
    form = qb.split(inst)
    x = np.zeros(12, dtype=np.uint8)
    v = 0.0
    trace = []
    for k, l in enumerate(qb.flip_sequence(12), start=1):
        x[l] ^= 1
        v += qb.delta(form, x, l)
        if k % 97 == 0:
            trace.append([k, int(l), v, qb.evaluate(inst, x)])
    out["delta_trace_n12"] = {"coeffs": inst.coeffs.tolist(), "samples": trace}

    out["seconds"] = round(time.time() - t0, 1)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote {path}: {len(cases)} cases, {len(seam)} gray_scan cases in {out['seconds']} s")


if __name__ == "__main__":
    main()

"""Pin BASELINE config E (n=40, fp32 N(0,1), 10% density) against the CPU oracle.

TEST INFRASTRUCTURE (offline fixture generator).  Runs the oracle restatement of the
reference's ``solve_parallel`` (oracle/gray_oracle.c ``oc_solve_subspaces``, which follows
/root/reference/pkg/src/qubrute/solver.py:159-229 and _kernels.py:46-75 line by line) over all
2^14 m=14 subspaces of ``config_coeffs("E", rep)`` -- every one of the 2^40 states, fp64,
reference summation order -- and writes the minimiser, its exact value and the evaluation count
to tests/golden/config_e_n40.json.

The 2^14 suffixes are processed in pieces of ``--piece`` suffixes; each piece's result is
checkpointed (build/config_e_pin/) so the ~100 min/rep run is resumable.  Pieces are combined
in ascending suffix order with strict '<' (solver.py:173-185 combine_subspace_minima), so the
result is exactly ``solve_parallel(inst, SolveConfig(fixed_bits=14))``.

    python tests/golden/make_config_e_pin.py --rep 0 --threads 8
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_2310_19373_b200 import instances  # noqa: E402

M = 14
OUT = os.path.join(ROOT, "tests", "golden", "config_e_n40.json")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", type=int, default=0)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--piece", type=int, default=256)
    args = ap.parse_args()

    coeffs = instances.config_coeffs("E", args.rep)
    n = coeffs.shape[0]
    sha = instances.coeffs_sha256(coeffs)
    ckdir = os.path.join(ROOT, "build", "config_e_pin", f"rep{args.rep}_{sha[:12]}")
    os.makedirs(ckdir, exist_ok=True)
    total = 1 << M
    t_all = time.time()
    pieces = []
    for s0 in range(0, total, args.piece):
        s1 = min(total, s0 + args.piece)
        ck = os.path.join(ckdir, f"{s0:05d}_{s1:05d}.json")
        if os.path.exists(ck):
            with open(ck) as fh:
                pieces.append(json.load(fh))
            continue
        t0 = time.time()
        bits, value, ev = oracle.solve_subspaces(coeffs, M, s0, s1, threads=args.threads)
        rec = {"s_begin": s0, "s_end": s1, "bits": bits, "value": value, "evaluations": ev,
               "seconds": time.time() - t0}
        with open(ck + ".tmp", "w") as fh:
            json.dump(rec, fh)
        os.replace(ck + ".tmp", ck)
        pieces.append(rec)
        print(f"rep {args.rep} suffixes [{s0},{s1}) value {value!r} ({rec['seconds']:.1f} s)", flush=True)
    pieces.sort(key=lambda r: r["s_begin"])
    best = pieces[0]
    for r in pieces[1:]:
        if r["value"] < best["value"]:  # strict '<': lowest suffix wins ties (solver.py:173-185)
            best = r
    evaluations = sum(r["evaluations"] for r in pieces)
    assert evaluations == (1 << n) - (1 << M)
    result = {"rep": args.rep, "n": n, "seed": instances.bench_seed(n, args.rep), "coeffs_sha256": sha,
              "m": M, "argmin": best["bits"], "argmin_hex": hex(best["bits"]), "value": best["value"],
              "value_hex": float(best["value"]).hex(), "evaluations": evaluations,
              "winning_suffixes": [best["s_begin"], best["s_end"]],
              "oracle": "oracle/gray_oracle.c oc_solve_subspaces (restates solver.py:159-229, _kernels.py:46-75)",
              "threads": args.threads, "cpu_seconds_this_run": time.time() - t_all}
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data[f"rep{args.rep}"] = result
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(result))


if __name__ == "__main__":
    main()

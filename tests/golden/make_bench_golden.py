"""Golden rows of the REFERENCE's own ``qubrute bench`` command (build container only).

    python tests/golden/make_bench_golden.py

Runs the unmodified reference CLI (``qubrute.cli.main``, /root/reference/pkg/src or QUBRUTE_REF)
with ``bench --n-min 3 --n-max 12 --reps 3 --modes naive,incremental,parallel --threads 4`` and
``-o`` a temporary CSV, and stores its header, its rows without the (machine-dependent) seconds,
and its stdout summary lines in reference_bench.json.  tests/test_benchrec_cpu.py checks the
format layer against it; tests/test_gpu_parity.py checks that paper_2310_19373_b200.benchrec
produces the same (n, mode, rep, value) rows on the GPU.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys
import tempfile

REF = os.environ.get("QUBRUTE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from qubrute import cli  # noqa: E402

ARGS = ["bench", "--n-min", "3", "--n-max", "12", "--reps", "3", "--modes", "naive,incremental,parallel",
        "--threads", "4"]


def main() -> None:
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "bench.csv")
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(ARGS + ["-o", path])
        text = open(path, encoding="utf-8").read()
    lines = text.splitlines()
    rows = []
    for ln in lines[1:]:
        n, mode, rep, _seconds, value = ln.split(",")
        rows.append([int(n), mode, int(rep), value])  # value kept as the reference's repr string
    out = {
        "args": ARGS,
        "exit_code": rc,
        "header": lines[0],
        "rows": rows,
        "summary_lines": [s.split(":")[0] for s in buf.getvalue().splitlines()],
        "refusal_exit_code": cli.main(["bench", "--n-min", "3", "--n-max", "30", "--modes", "naive"]),
    }
    dst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_bench.json")
    with open(dst, "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1)
    print(f"wrote {dst}: {len(rows)} rows")


if __name__ == "__main__":
    main()

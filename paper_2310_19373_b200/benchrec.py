"""Benchmark records in the reference's CSV schema, timed on the GPU solver.

The reference's ``qubrute bench`` (``pkg/src/qubrute/cli.py:86-142``) solves seeded instances
``random_instance(n, bench_seed(n, rep))`` for every (n, mode, rep) and emits rows
``n,mode,rep,seconds,value`` (``cli.py:24``, ``BenchRecord`` ``cli.py:27-39``).  This module is
that measurement layer with the same seeds, validation, naive guard, CSV append rule and
speed-up summary, but every solve goes through this package's GPU entry points, so the paper's
Fig. 2-style comparison can carry B200 rows next to the reference's CPU rows.  The argparse front
end itself stays out of scope; INTEGRATION.md shows how to route the reference's
own ``bench`` command through this package instead.
"""

from __future__ import annotations

import os
import sys
from dataclasses import dataclass
from typing import Iterable, Sequence, TextIO

from .core import DimensionCapError
from .instances import bench_seed, random_instance
from .solver import MODES, NAIVE_MAX_DIM, SolveConfig, solve

CSV_HEADER = "n,mode,rep,seconds,value"  # cli.py:24


@dataclass(frozen=True)
class BenchRecord:
    """One measurement: dimension, solver mode, repetition, wall seconds of the solve call, value
    (``cli.py:27-39``; same ``repr`` float formatting in the row)."""

    n: int
    mode: str
    rep: int
    seconds: float
    value: float

    def csv_row(self) -> str:
        return f"{self.n},{self.mode},{self.rep},{self.seconds!r},{self.value!r}"


def _parse_modes(modes: str | Sequence[str]) -> list[str]:
    if isinstance(modes, str):
        modes = [m.strip() for m in modes.split(",") if m.strip()]
    modes = list(modes)
    if not modes:
        raise ValueError("--modes must name at least one mode")
    for mode in modes:
        if mode not in MODES:
            raise ValueError(f"unknown mode {mode!r}; choose from {MODES}")
    return modes


def warmup(modes: Iterable[str], threads: int = 1) -> None:
    """Keep one-time costs (library load, device and stream setup) out of the timed solves;
    the reference does the same for its JIT (``cli.py:78-83``)."""
    small = random_instance(6, seed=0)
    for mode in modes:
        solve(small, SolveConfig(threads=threads, mode=mode))


def run_bench(n_min: int, n_max: int, reps: int = 10, modes: str | Sequence[str] = "naive,incremental",
              threads: int = 1) -> list[BenchRecord]:
    """Records for every (n, mode, rep) in the reference's loop order (``cli.py:109-121``).

    Raises ``ValueError`` for the argument errors the reference rejects and
    ``DimensionCapError`` where the reference refuses with exit code 3 (naive above its guard).
    """
    modes = _parse_modes(modes)
    if n_min < 1 or n_max < n_min:
        raise ValueError("need 1 <= --n-min <= --n-max")
    if reps < 1:
        raise ValueError("--reps must be >= 1")
    if "naive" in modes and n_max > NAIVE_MAX_DIM:
        raise DimensionCapError(
            f"refusing: --n-max {n_max} exceeds the naive-solver guard {NAIVE_MAX_DIM}; "
            "drop naive from --modes or lower --n-max")
    warmup(modes, threads)
    records: list[BenchRecord] = []
    for n in range(n_min, n_max + 1):
        for mode in modes:
            for rep in range(reps):
                inst = random_instance(n, bench_seed(n, rep))
                sol = solve(inst, SolveConfig(threads=threads, mode=mode))
                records.append(BenchRecord(n=n, mode=mode, rep=rep, seconds=max(sol.elapsed, 1e-9),
                                           value=sol.value))
    return records


def write_csv(records: Sequence[BenchRecord], output: str | None = None, stream: TextIO | None = None) -> None:
    """Append to ``output`` (header only when the file is new or empty), else print header + rows
    to ``stream`` (stdout) — ``cli.py:123-134``."""
    if output:
        new_file = not os.path.exists(output) or os.path.getsize(output) == 0
        with open(output, "a", encoding="utf-8") as fh:
            if new_file:
                fh.write(CSV_HEADER + "\n")
            for rec in records:
                fh.write(rec.csv_row() + "\n")
    else:
        out = stream or sys.stdout
        print(CSV_HEADER, file=out)
        for rec in records:
            print(rec.csv_row(), file=out)


def speedup_summary(records: Sequence[BenchRecord]) -> list[str]:
    """Per-n mean of naive/incremental time ratios over reps (``cli.py:136-141``); empty unless
    both modes were measured."""
    modes = {r.mode for r in records}
    if not {"naive", "incremental"} <= modes:
        return []
    lines = []
    for n in sorted({r.n for r in records}):
        naive_t = {r.rep: r.seconds for r in records if r.n == n and r.mode == "naive"}
        incr_t = {r.rep: r.seconds for r in records if r.n == n and r.mode == "incremental"}
        ratios = [naive_t[rep] / incr_t[rep] for rep in sorted(naive_t)]
        lines.append(f"n={n} mean speedup incremental vs naive: {sum(ratios) / len(ratios):.2f}x")
    return lines


def parse_csv(text: str) -> list[BenchRecord]:
    """Read rows written by either implementation back into records (header required)."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError(f"expected header {CSV_HEADER!r}")
    out = []
    for ln in lines[1:]:
        n, mode, rep, seconds, value = ln.split(",")
        out.append(BenchRecord(int(n), mode, int(rep), float(seconds), float(value)))
    return out

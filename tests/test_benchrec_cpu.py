"""CPU tests of the benchmark-record layer (paper_2310_19373_b200.benchrec) against the reference
bench command's golden output (tests/golden/reference_bench.json, made by make_bench_golden.py):
CSV header and row format, append rule, argument validation and the naive refusal, summary lines.
No solve runs here (validation happens before any device call)."""

import io
import math

import pytest

from paper_2310_19373_b200 import DimensionCapError, benchrec


def _golden_records(g):
    return [benchrec.BenchRecord(n, mode, rep, 1e-3 * (1 + rep), float(v)) for n, mode, rep, v in g["rows"]]


def test_header_and_row_format(bench_golden):
    assert benchrec.CSV_HEADER == bench_golden["header"]
    for (n, mode, rep, v), rec in zip(bench_golden["rows"], _golden_records(bench_golden)):
        row = rec.csv_row().split(",")
        assert row[0] == str(n) and row[1] == mode and row[2] == str(rep)
        assert row[4] == v  # repr formatting of the value, as the reference writes it


def test_csv_round_trip_and_append(tmp_path, bench_golden):
    recs = _golden_records(bench_golden)
    path = str(tmp_path / "b.csv")
    benchrec.write_csv(recs[:10], path)
    benchrec.write_csv(recs[10:], path)  # appends without a second header
    text = open(path).read()
    assert text.count(benchrec.CSV_HEADER) == 1
    assert benchrec.parse_csv(text) == recs
    buf = io.StringIO()
    benchrec.write_csv(recs[:3], stream=buf)
    assert buf.getvalue().splitlines()[0] == benchrec.CSV_HEADER and len(buf.getvalue().splitlines()) == 4


@pytest.mark.parametrize("kw, exc", [
    (dict(n_min=3, n_max=4, modes=""), ValueError),
    (dict(n_min=3, n_max=4, modes="fast"), ValueError),
    (dict(n_min=0, n_max=4), ValueError),
    (dict(n_min=5, n_max=4), ValueError),
    (dict(n_min=3, n_max=4, reps=0), ValueError),
    (dict(n_min=3, n_max=30, modes="naive"), DimensionCapError),  # reference: refuses, exit code 3
])
def test_validation_matches_reference(kw, exc, bench_golden):
    assert bench_golden["refusal_exit_code"] == 3
    with pytest.raises(exc):
        benchrec.run_bench(**kw)


def test_speedup_summary_lines(bench_golden):
    lines = benchrec.speedup_summary(_golden_records(bench_golden))
    assert [ln.split(":")[0] for ln in lines] == bench_golden["summary_lines"]
    assert all(math.isclose(float(ln.split(": ")[1][:-1]), 1.0) for ln in lines)
    assert benchrec.speedup_summary([r for r in _golden_records(bench_golden) if r.mode != "naive"]) == []

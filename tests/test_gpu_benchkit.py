"""bench/verify/trace on the GPU: the reference CLI's tests (tests/test_cli.py:
112-160, tests/test_bench.py:60-75 of the reference) restated for
`python -m paper_0811_3448_b200`."""

import numpy as np
import pytest

from paper_0811_3448_b200.__main__ import main
from paper_0811_3448_b200.bench import CSV_HEADER, BenchPlan, run_plan, verify

pytestmark = pytest.mark.gpu

NYBBLE_TRACE = """\
begin: [B 4 0 0 7 A C E]
bit 1: [7 4 0 0][A C E B]
bit 2: [0 0][4 7][A B][E C]
bit 3: [0 0][4 7][A B][C][E]
bit 4: [0 0][4 7][A B][C][E]
end: [0 0 4 7 A B C E]
"""


@pytest.mark.parametrize("variant", ["recursive", "iterative", "optimized", "parallel"])
def test_every_variant_runs(cuda, variant):
    recs = run_plan(BenchPlan(50, 50, 1, 1, variant=variant, workers=2))
    assert len(recs) == 1 and recs[0].error is None


@pytest.mark.parametrize("timing", ["host", "device"])
def test_sweep_positive_times(cuda, timing):
    recs = run_plan(BenchPlan(10_000, 100_000, 10_000, 3, seed=8, timing=timing))
    assert len(recs) == 10 and all(r.min_ns > 0 for r in recs)


def test_cli_bench_csv_and_fit(cuda, tmp_path, capsys):
    csv = tmp_path / "out.csv"
    assert main(["bench", "--start", "1000", "--end", "5000", "--step", "1000", "--granularity", "2",
                 "--csv", str(csv)]) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == CSV_HEADER and len(lines) == 6
    out = capsys.readouterr().out
    assert "slope=" in out and "r_squared=" in out
    assert main(["bench", "--start", "64", "--end", "64", "--step", "1", "--granularity", "1",
                 "--csv", str(tmp_path / "x.csv")]) == 0
    assert "n/a" in capsys.readouterr().out


def test_cli_trace_worked_example(cuda, capsys):
    assert main(["trace", "--width", "4", "B", "4", "0", "0", "7", "A", "C", "E"]) == 0
    assert capsys.readouterr().out == NYBBLE_TRACE
    assert main(["trace", "--width", "4", "5"]) == 0
    assert capsys.readouterr().out == "begin: [5]\nend: [5]\n"
    assert main(["trace", "--width", "8", "FF", "0A", "00"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "begin: [FF A 0]" and out[-1] == "end: [0 A FF]" and len(out) == 10
    assert main(["trace", "--width", "4", "G"]) == 2
    assert main(["trace", "--width", "4", "10"]) == 2
    assert main(["trace", "--width", "5", "1"]) == 2


@pytest.mark.parametrize("kind", ["unsigned32", "unsigned64", "signed32", "float64"])
@pytest.mark.parametrize("variant", ["recursive", "iterative", "optimized", "parallel"])
def test_verify_differential(cuda, kind, variant):
    passed, first = verify(40, 7, kind, variant, 3)
    assert passed == 40 and first is None


def test_cli_verify(cuda, capsys):
    assert main(["verify", "--cases", "25", "--seed", "7", "--type", "u32"]) == 0
    assert capsys.readouterr().out.strip() == "25/25 passed"

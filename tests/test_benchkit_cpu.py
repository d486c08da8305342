"""The package's bench harness (paper_0811_3448_b200.bench) on CPU: plan
validation, OLS fit and the exact CSV bytes -- the reference's schema tests
(tests/test_bench.py:20-122 of the reference) restated against this module."""

import io

import pytest

from paper_0811_3448_b200.bench import CSV_HEADER, BenchPlan, BenchRecord, fit_linear, write_csv


def parse_csv(text):
    lines = text.splitlines()
    assert lines[0] == CSV_HEADER
    return [BenchRecord(*(int(v) for v in ln.split(","))) for ln in lines[1:]]


@pytest.mark.parametrize("kw", [dict(start_size=0), dict(end_size=5), dict(step=0), dict(granularity=0),
                                dict(key_kind="decimal"), dict(variant="quick"),
                                dict(variant="parallel", workers=0), dict(timing="wallclock")])
def test_invalid_plans_rejected(kw):
    base = dict(start_size=10, end_size=30, step=10, granularity=2)
    base.update(kw)
    with pytest.raises(ValueError):
        BenchPlan(**base).validate()


def test_valid_plan_and_sizes():
    p = BenchPlan(10, 30, 10, 2)
    p.validate()
    assert list(p.sizes()) == [10, 20, 30]


def test_fit():
    f = fit_linear([BenchRecord(1, 7, 7, 7), BenchRecord(2, 9, 9, 9), BenchRecord(3, 11, 11, 11)])
    assert f.slope == pytest.approx(2.0) and f.intercept == pytest.approx(5.0) and f.r_squared == pytest.approx(1.0)
    assert fit_linear([BenchRecord(1, 5, 5, 5), BenchRecord(2, 5, 5, 5)]).r_squared == pytest.approx(1.0)
    assert 0.0 <= fit_linear([BenchRecord(1, 10, 10, 10), BenchRecord(2, 3, 3, 3),
                              BenchRecord(3, 14, 14, 14)]).r_squared <= 1.0
    for bad in ([BenchRecord(5, 1, 1, 1)], [BenchRecord(5, 1, 1, 1), BenchRecord(5, 2, 2, 2)],
                [BenchRecord(5, 1, 1, 1, error="allocation failed"), BenchRecord(6, 1, 1, 1)]):
        with pytest.raises(ValueError):
            fit_linear(bad)


def test_csv_bytes(tmp_path):
    out = io.StringIO()
    write_csv([BenchRecord(10, 100, 90, 110)], out)
    assert out.getvalue() == "size,mean_ns,min_ns,max_ns\n10,100,90,110\n"
    out = io.StringIO()
    write_csv([], out)
    assert out.getvalue() == "size,mean_ns,min_ns,max_ns\n"
    out = io.StringIO()
    write_csv([BenchRecord(20, 2, 2, 2), BenchRecord(5, 1, 1, 1, error="allocation failed"),
               BenchRecord(10, 1, 1, 1)], out)
    assert out.getvalue().splitlines()[1:] == ["10,1,1,1", "20,2,2,2"]
    recs = [BenchRecord(10, 5, 4, 6), BenchRecord(20, 9, 8, 10)]
    path = tmp_path / "s.csv"
    write_csv(recs, path)
    assert parse_csv(path.read_text()) == recs
    with pytest.raises(OSError, match="cannot write CSV"):
        write_csv(recs, tmp_path / "no" / "x.csv")

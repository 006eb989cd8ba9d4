"""The on-device verify suites (verify.py) against the reference's own verify
output for the same seed (tests/golden/verify_ref.txt): every suite passes,
and the bsm-theorems weight identity (a host-side check) reports the same
worst ratio."""

from __future__ import annotations

import io
import os

import pytest

from conftest import GOLDEN, price_close


def _lines(text):
    return [ln.split() for ln in text.splitlines() if ln and not ln.startswith(" ")]


@pytest.mark.gpu
def test_verify_matches_reference():
    from paper_2303_02317_b200 import verify

    out = io.StringIO()
    rc = verify.run_suites(reps=6, steps=1024, seed=3, out=out)
    ref = _lines(open(os.path.join(GOLDEN, "verify_ref.txt")).read())
    got = _lines(out.getvalue())
    assert rc == 0, out.getvalue()
    assert [g[0] for g in got] == [r[0] for r in ref]
    assert [g[1] for g in got] == [r[1] for r in ref]
    # the weight identity is pure host arithmetic: identical worst ratio
    assert got[4][3] == ref[4][3]


def test_verify_argument_errors():
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import verify

    with pytest.raises(fl.ValidationError):
        verify.run_suites(reps=-1)
    with pytest.raises(fl.ValidationError):
        verify.run_suites(reps=2, steps=10)
    assert verify.run_suites(reps=0) == 0


def test_benchcsv_argument_errors():
    import paper_2303_02317_b200 as fl
    from paper_2303_02317_b200 import benchcsv

    spec = fl.OptionSpec(100.0, 100.0, 0.05, 0.03, 0.2, 365, 1)
    with pytest.raises(fl.UnsupportedCombinationError):
        benchcsv.bench_records(["nope"], "64", 1, spec)
    with pytest.raises(fl.ValidationError):
        benchcsv.bench_records(["fast_put"], "x", 1, spec)
    with pytest.raises(fl.ValidationError):
        benchcsv.bench_records(["fast_put"], "64", 0, spec)


@pytest.mark.gpu
def test_benchcsv_schema_and_prices():
    import csv as _csv

    from paper_2303_02317_b200 import benchcsv

    out = io.StringIO()
    import contextlib

    with contextlib.redirect_stdout(out):
        rc = benchcsv.main(["--method", ",".join(benchcsv.BENCH_METHODS), "--steps", "300,1024", "--reps", "2"])
    assert rc == 0
    rows = list(_csv.reader(io.StringIO(out.getvalue())))
    assert rows[0] == ["method", "T", "seconds", "price", "reps"]
    assert len(rows) == 1 + 2 * len(benchcsv.BENCH_METHODS)
    for r in rows[1:]:
        assert float(r[2]) > 0.0 and float(r[3]) == float(r[3]) and r[4] == "2"
    # the price column against the reference's own bench CSV (cli.py:653-720,
    # tests/golden/bench_ref.csv, same spec and steps): rows in the same order
    with open(os.path.join(GOLDEN, "bench_ref.csv")) as fh:
        ref = list(_csv.reader(fh))
    assert [r[:2] for r in rows] == [r[:2] for r in ref]
    for got, want in zip(rows[1:], ref[1:]):
        assert price_close(float(got[3]), float(want[3]), 100.0), (got, want)
